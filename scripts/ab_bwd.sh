#!/bin/bash
# A/B the backward over variants/lib_*.so (VISTA_LIB): parity tests, then c2/c5 kernel ms and fraction.
# usage: scripts/ab_bwd.sh [attn] [configs]
cd "$(dirname "$0")/.."
A=${1:-softmax}
CFGS=${2:-"c2 c5"}
for lib in variants/lib_*.so; do
  n=$(basename $lib .so)
  [ "$n" = lib_prof ] && continue
  echo "== $n $(VISTA_LIB=$PWD/$lib timeout 600 python -m pytest tests -m gpu -x -q -k backward 2>&1 | tail -1)"
  for c in $CFGS; do
    VISTA_LIB=$PWD/$lib timeout 300 python bench.py --config $c --attn $A --backward --steps 100 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('  $c', round(d['ms_per_step'],4), r.get('kernel_ms'), round(r['frac'],4), d['clocks']['sm_mhz'])"
  done
done
