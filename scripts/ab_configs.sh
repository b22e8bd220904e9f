#!/bin/bash
# Kernel-only numbers for several configs / attn forms with the in-tree library.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in ${CONFIGS:-c2 c3 c4 c5}; do
 for attn in ${ATTNS:-softmax qla}; do
  python bench.py --config $cfg --attn $attn --steps ${STEPS:-100} --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/cfg_${cfg}_${attn}.json 2> gpurun_out/cfg_${cfg}_${attn}.err
  python -c "
import json
d=json.load(open('gpurun_out/cfg_${cfg}_${attn}.json')); r=d['roofline']
print('${cfg} ${attn}', 'items/s=%.4g'%d['value'], 'kernel_ms=%.4f'%r['kernel_ms'], 'step_ms=%.4f'%d['ms_per_step'], r['bound'], 'frac=%.4f'%r['frac'], 'hbm=%s'%(r.get('hbm',{}).get('frac', r['frac'])), d['clocks'])
" || tail -3 gpurun_out/cfg_${cfg}_${attn}.err
 done
done
