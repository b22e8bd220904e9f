#!/bin/bash
# Kernel-only numbers for every variants/lib_*.so on several configs (CONFIGS env, default c2 c3 c4).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in ${CONFIGS:-c2 c3 c4}; do
 for lib in variants/lib_*.so; do
  n=$(basename $lib .so)
  VISTA_LIB=$PWD/$lib python bench.py --config $cfg --steps ${STEPS:-100} --warmup 5 --e2e-steps 0 --no-cpu-baseline ${ARGS} > gpurun_out/abc_${cfg}_$n.json 2> gpurun_out/abc_${cfg}_$n.err
  python -c "
import json
d=json.load(open('gpurun_out/abc_${cfg}_$n.json')); r=d['roofline']
print('$cfg $n', 'kernel_ms=%.4f'%r['kernel_ms'], 'step_ms=%.4f'%d['ms_per_step'], 'frac=%.4f'%r['frac'], d['clocks']['sm_mhz'] if d['clocks'] else None)
" || tail -3 gpurun_out/abc_${cfg}_$n.err
 done
done
