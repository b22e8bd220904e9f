#!/bin/bash
# One GPU call that regenerates the evidence under profiles/ for the current build:
# default bench lines (c2 softmax / qla), per-config kernel numbers, launch lists, ncu --set full
# of the two dominant kernels (c2).  Outputs in gpurun_out/refresh/ (copied to profiles/ by hand).
cd "$(dirname "$0")/.."
O=gpurun_out/refresh
mkdir -p $O
python bench.py > $O/bench_c2_softmax.json 2> $O/bench_c2_softmax.err
python bench.py --attn qla > $O/bench_c2_qla.json 2> $O/bench_c2_qla.err
python bench.py --backward --steps 100 > $O/bench_c2_softmax_bwd.json 2> $O/bench_c2_softmax_bwd.err
python bench.py --attn qla --backward --steps 100 > $O/bench_c2_qla_bwd.json 2> $O/bench_c2_qla_bwd.err
python bench.py --export-int8 --steps 100 --no-cpu-baseline > $O/bench_c2_softmax_int8.json 2> $O/bench_c2_softmax_int8.err
python bench.py --config c5 --backward --steps 20 --no-cpu-baseline > $O/bench_c5_softmax_bwd.json 2> $O/bench_c5_softmax_bwd.err
python bench.py --config c5 --attn qla --backward --steps 50 --no-cpu-baseline > $O/bench_c5_qla_bwd.json 2> $O/bench_c5_qla_bwd.err
python bench.py --qla-rows history --steps 100 > $O/bench_c2_qla_rows_history.json 2> $O/bench_c2_qla_rows_history.err
python bench.py --qla-rows target --steps 100 > $O/bench_c2_qla_rows_target.json 2> $O/bench_c2_qla_rows_target.err
STEPS=100 bash scripts/ab_configs.sh > $O/configs.txt 2>&1
cp gpurun_out/cfg_*.json $O/ 2>/dev/null
for cfg in c2 c5; do
  for attn in softmax qla; do
    CMD="python bench.py --config $cfg --attn $attn --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
    $CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none \
      -k regex:"sm100|merge_|user_tiles|qla_|quantize|simt_|softmax_bwd" --csv --log-file $O/launches_${cfg}_${attn}.csv $CMD > /dev/null 2>&1
    python scripts/ncu_summary.py launches $O/launches_${cfg}_${attn}.csv > $O/launches_${cfg}_${attn}.txt
  done
done
for extra in "--backward" "--attn qla --backward" "--qla-rows history"; do
  tag=$(echo "$extra" | tr -d '-' | tr ' ' '_')
  CMD="python bench.py $extra --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
  $CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"sm100|merge_|user_tiles|qla_|quantize|simt_|softmax_bwd" --csv --log-file $O/launches_c2_${tag}.csv $CMD > /dev/null 2>&1
  python scripts/ncu_summary.py launches $O/launches_c2_${tag}.csv > $O/launches_c2_${tag}.txt
done
for attn in softmax qla; do
  CMD="python bench.py --attn $attn --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
  k=$([ $attn = softmax ] && echo sm100_softmax || echo sm100_qla_state)
  $CMD > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 \
    -o $O/prof_${attn} $CMD > $O/ncu_full_${attn}.log 2>&1
  echo "ncu full $attn exit=$?"
done
