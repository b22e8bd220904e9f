#!/bin/bash
# ncu --set full of the softmax kernel (c2) with source view, plus the vista-only launch list.
mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline ${ARGS}"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:sm100_softmax -s 3 -c 1 -o gpurun_out/prof_sm ${CMD} > gpurun_out/ncu_sm.log 2>&1; echo ncu_exit=$?
$CMD > gpurun_out/plain2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:vista --csv --log-file gpurun_out/launches_vista.csv ${CMD} > gpurun_out/ncu_l.log 2>&1; echo ncu2_exit=$?
