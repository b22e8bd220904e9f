#!/bin/bash
# One gpurun call: smoke, bench (softmax + QLA), ncu launch list, ncu --set full of both main kernels.
mkdir -p gpurun_out
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$?
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench_exit=$?
python bench.py --attn qla --no-cpu-baseline > gpurun_out/bench_c2_qla.json 2> gpurun_out/bench_c2_qla.err; echo qla_exit=$?
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1; echo ncu1_exit=$?
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sm100_softmax -s 3 -c 1 -o gpurun_out/prof_softmax $CMD > gpurun_out/ncu2.log 2>&1; echo ncu2_exit=$?
CMDQ="python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --attn qla"
$CMDQ > gpurun_out/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sm100_qla -s 3 -c 1 -o gpurun_out/prof_qla $CMDQ > gpurun_out/ncu3.log 2>&1; echo ncu3_exit=$?
cat gpurun_out/bench_c2.json gpurun_out/bench_c2_qla.json
tail -3 gpurun_out/bench_c2.err
