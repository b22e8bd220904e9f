#!/bin/bash
# A/B the QLA rows path over variants/lib_*.so: parity tests, then the history / target bench lines.
cd "$(dirname "$0")/.."
for lib in variants/lib_*.so; do
  n=$(basename $lib .so)
  echo "== $n $(VISTA_LIB=$PWD/$lib timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k qla_rows 2>&1 | tail -1)"
  for m in history target history; do
    VISTA_LIB=$PWD/$lib timeout 300 python bench.py --qla-rows $m --steps 100 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('  $m', round(d['ms_per_step'],4), r.get('kernel_ms'), round(r['frac'],4))"
  done
done
