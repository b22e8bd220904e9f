#!/bin/bash
# ncu launch list (vista kernels only) for the bench step of CONFIG (default c2).
mkdir -p gpurun_out
CFG=${CONFIG:-c2}
CMD="python bench.py --config $CFG --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline ${ARGS}"
$CMD > gpurun_out/plain_$CFG.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sm100|merge_|user_tiles|qla_|quantize|simt_" --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_$CFG.log 2>&1; echo ncu_exit=$?
python scripts/ncu_summary.py launches gpurun_out/launches_$CFG.csv
