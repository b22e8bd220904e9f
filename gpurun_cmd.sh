mkdir -p gpurun_out/p9
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/p9/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/p9/pytest_gpu.log
timeout 300 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-sustained --no-graph > gpurun_out/p9/c5_plain.json 2> gpurun_out/p9/c5_plain.err; echo "c5 plain exit $?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:sm100_softmax_kernel -c 2 --csv --log-file gpurun_out/p9/ncu_c5_dram.csv python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-sustained --no-graph > gpurun_out/p9/ncu_c5.log 2>&1; echo "ncu exit $?"
grep -i "dram__bytes\|duration" gpurun_out/p9/ncu_c5_dram.csv | head
