#!/bin/bash
# Evidence for the QLA backward (NEXT-2): bench lines c2/c5, launch list c2, ncu --set full of the
# dK/dV kernel.  Outputs in gpurun_out/bwd/.
cd "$(dirname "$0")/.."
O=gpurun_out/bwd
mkdir -p $O
for c in c2 c5; do
  python bench.py --config $c --attn qla --backward --steps 100 --warmup 5 > $O/bench_${c}_qla_bwd.json 2> $O/bench_${c}.err
done
CMD="python bench.py --attn qla --backward --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"sm100|merge_|user_tiles|qla_|quantize|simt_" --csv --log-file $O/launches_c2_qla_bwd.csv $CMD > /dev/null 2>&1
python scripts/ncu_summary.py launches $O/launches_c2_qla_bwd.csv > $O/launches_c2_qla_bwd.txt
$CMD > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:sm100_qla_bwd_kv -s 1 -c 1 \
  -o $O/prof_bwd_kv $CMD > $O/ncu_full.log 2>&1
echo "ncu exit=$?"
