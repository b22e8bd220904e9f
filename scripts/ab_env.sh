#!/bin/bash
# A/B of runtime switches (environment assignments, ';'-separated variants) on bench configs.
# ENVS="VISTA_SOFTMAX_PAIR=1;VISTA_SOFTMAX_PAIR=0" CFGS="c2 c3" bash scripts/ab_env.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/${TAG:-abenv}
mkdir -p $OUT
IFS=';' read -ra VARS <<< "${ENVS:-VISTA_SOFTMAX_PAIR=1;VISTA_SOFTMAX_PAIR=0}"
for rep in $(seq 1 ${REPS:-1}); do
for v in "${VARS[@]}"; do
  name=$(echo "$v" | tr ' =' '_-')
  for cfg in ${CFGS:-c2}; do
    env $v timeout 300 python bench.py --config $cfg --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-sustained ${BARGS} > $OUT/$name.$cfg.$rep.json 2> $OUT/$name.$cfg.$rep.err
    python -c "import json; d=json.load(open('$OUT/$name.$cfg.$rep.json')); r=d['roofline']; print('$v $cfg', 'step', round(d['ms_per_step'],4), 'kernel', r['kernel_ms'], 'frac', r['frac'], 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1
  done
done
done
