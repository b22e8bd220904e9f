#!/bin/bash
# Time every variants/lib_*.so with the bench (kernel-only numbers).  ARGS env adds bench flags.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in variants/lib_*.so; do
  n=$(basename $lib .so)
  VISTA_LIB=$PWD/$lib python bench.py --steps 300 --warmup 10 --e2e-steps 0 --no-cpu-baseline ${ARGS} > gpurun_out/ab_$n.json 2> gpurun_out/ab_$n.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/ab_$n.json')); r=d['roofline']
print('$n', 'kernel_ms=%.4f'%r['kernel_ms'], 'step_ms=%.4f'%d['ms_per_step'], 'frac=%.4f'%r['frac'], d['clocks'])
" || tail -3 gpurun_out/ab_$n.err
done
