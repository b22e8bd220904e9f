#!/bin/bash
# DRAM bytes per launch of the NEXT-row kernels (stage-2 attention, CTA-pair GEMM, QLA target rows)
# in their bench configurations: one plain run of each bench line first, then ONE ncu process over
# a shell running the three (ncu follows the child processes).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/${TAG:-traffic}
mkdir -p $OUT
for a in "--stage2" "--layers 1" "--qla-rows target"; do
  timeout 300 python bench.py $a --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-sustained --no-graph > /dev/null 2>&1 || echo "plain $a failed"
done
cat > $OUT/run3.sh <<'EOS'
python bench.py --stage2 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-sustained --no-graph
python bench.py --layers 1 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-sustained --no-graph
python bench.py --qla-rows target --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-sustained --no-graph
EOS
timeout 1200 ncu --target-processes all --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:"sm100_target_attend_kernel|sm100_gemm2_kernel|sm100_qla_rows_kernel" \
  --csv --log-file $OUT/ncu_dram.csv bash $OUT/run3.sh > $OUT/ncu.log 2>&1
echo "ncu exit $?"
python - <<EOP
import csv, collections
rows = [r for r in csv.reader(open("$OUT/ncu_dram.csv")) if len(r) > 14 and r[0].isdigit()]
agg = collections.defaultdict(list)
for r in rows:
    agg[(r[4][:60], r[-3])].append(float(r[-1]))
for (k, m), v in sorted(agg.items()):
    print(k, m, len(v), [round(x) for x in v[:6]])
EOP
