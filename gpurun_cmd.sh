mkdir -p gpurun_out/p7
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "target_attend or smoke" > gpurun_out/p7/pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/p7/pytest.log
timeout 300 python bench.py --stage2 --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-sustained > gpurun_out/p7/stage2.json 2> gpurun_out/p7/stage2.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/p7/stage2.json')); r=d['roofline']; print('stage2 step', d['ms_per_step'], 'kernel', r['kernel_ms'], 'frac', r['frac'], d['value'])"
timeout 120 python scripts/trace_ta.py 2048 | head -12
