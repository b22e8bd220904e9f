#!/bin/bash
# Full GPU test suite, default bench lines (20 and 500 steps), then ONE ncu tool run (the pool allows
# one per gpurun call): NCU=launches (default) -> the launch list of the default bench; NCU=full ->
# one ncu --set full capture of the softmax forward kernel.  TAG names the output directory.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/${TAG:-prof}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 > $OUT/bench_default20.json 2> $OUT/bench_default20.err
timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > $OUT/bench_default500.json 2> $OUT/bench_default500.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-sustained --no-graph > $OUT/plain.log 2>&1
if [ $? -eq 0 ]; then
  if [ "${NCU:-launches}" = full ]; then
    ncu --set full --clock-control none --import-source on -k regex:sm100_softmax_kernel -s 3 -c 1 -o $OUT/softmax_full \
        python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-sustained --no-graph > $OUT/ncu_full.log 2>&1
  else
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
        python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-sustained --no-graph > $OUT/ncu_launches.log 2>&1
  fi
fi
tail -3 $OUT/pytest_gpu.log
