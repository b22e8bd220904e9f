#!/bin/bash
# One GPU call: tests, default bench, dry-run of the 2-rank by_length path.  Logs in gpurun_out/.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/${TAG:-check}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 > $OUT/bench_default20.json 2> $OUT/bench_default20.err
timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > $OUT/bench_default500.json 2> $OUT/bench_default500.err
timeout 300 python bench.py --gpus 2 --dist-backend gloo --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_c4_gloo2.json 2> $OUT/bench_c4_gloo2.err
tail -3 $OUT/pytest_gpu.log
cat $OUT/bench_default20.json | head -c 3000
