#!/bin/bash
# Quick GPU iteration: a pytest selection (PYSEL, default softmax parity), then a short bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/${TAG:-iter}
mkdir -p $OUT
timeout ${PYT:-600} python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "${PYSEL:-softmax}" > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
if [ -n "$BENCH" ]; then
  for cfg in $BENCH; do
    timeout 300 python bench.py --config $cfg --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline --e2e-steps 0 ${BARGS} > $OUT/bench_$cfg.json 2> $OUT/bench_$cfg.err
    echo "bench $cfg exit $?"; python -c "import json,sys; d=json.load(open('$OUT/bench_$cfg.json')); r=d['roofline']; print('$cfg', 'ms/step', round(d['ms_per_step'],4), 'kernel', r['kernel_ms'], 'frac', r['frac'], 'hbm', r.get('hbm',{}).get('frac'), 'clk', d['clocks'])" 2>&1 | tail -1
  done
fi
