#!/bin/bash
# A/B of softmax kernel build variants (libvista_<name>.so) on c2 / c5: kernel ms and step ms.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/${TAG:-ab}
mkdir -p $OUT
for v in ${VARIANTS:-default}; do
  for cfg in ${CFGS:-c2 c5}; do
    lib=paper_2510_22049_b200/libvista_$v.so; [ "$v" = default ] && lib=paper_2510_22049_b200/libvista.so
    VISTA_LIB=$PWD/$lib timeout 300 python bench.py --config $cfg --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-sustained > $OUT/$v.$cfg.json 2> $OUT/$v.$cfg.err
    python -c "import json; d=json.load(open('$OUT/$v.$cfg.json')); r=d['roofline']; print('$v $cfg', 'step', round(d['ms_per_step'],4), 'kernel', r['kernel_ms'], 'frac', r['frac'], 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1
  done
done
