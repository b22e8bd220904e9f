#!/bin/bash
# One GPU call for the round's final evidence (no profiler): the GPU test suite, smoke(), and the
# bench lines of every configuration / NEXT row.  Outputs in gpurun_out/${TAG:-final}/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-final}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
b() { local name=$1; shift; timeout 600 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; }
b default20 --steps 20 --warmup 5
b default500 --steps 500 --warmup 10 --no-cpu-baseline
b c3 --config c3 --steps 50 --no-cpu-baseline
b c5 --config c5 --steps 20 --no-cpu-baseline
b qla --attn qla --steps 50 --no-cpu-baseline
b backward --backward --steps 50 --no-cpu-baseline
b qla_backward --attn qla --backward --steps 50 --no-cpu-baseline
b int8 --export-int8 --steps 50 --no-cpu-baseline
b rows_history --qla-rows history --steps 50 --no-cpu-baseline
b rows_target --qla-rows target --steps 100 --no-cpu-baseline
b stage2 --stage2 --steps 100 --no-cpu-baseline
b layers3 --layers 3 --steps 10 --no-cpu-baseline
b c4_gloo2 --gpus 2 --dist-backend gloo --config c4 --steps 3 --warmup 3 --no-cpu-baseline
b reference --impl reference --steps 2 --warmup 1
tail -2 $O/pytest_gpu.log
tail -2 $O/smoke.log
python - "$O" <<'EOP'
import json, sys, glob, os
for f in sorted(glob.glob(sys.argv[1] + "/bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(os.path.basename(f), "FAILED", e); continue
    r = d.get("roofline", {})
    print(os.path.basename(f)[6:-5], round(d.get("ms_per_step", 0), 5), r.get("kernel_ms"), r.get("frac"),
          (d.get("sustained") or {}).get("roofline", {}).get("frac"), (d.get("clocks") or {}).get("reasons"))
EOP
