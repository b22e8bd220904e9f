#!/bin/bash
# A/B the forward over variants/lib_*.so (VISTA_LIB): softmax parity tests, then per config the
# kernel ms and roofline fraction of 2 runs.  usage: scripts/ab_fwd.sh [configs]
cd "$(dirname "$0")/.."
CFGS=${1:-"c2"}
for lib in variants/lib_*.so; do
  n=$(basename $lib .so)
  [ "$n" = lib_prof ] && continue
  echo "== $n $(VISTA_LIB=$PWD/$lib timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k 'softmax and not backward' 2>&1 | tail -1)"
  for c in $CFGS; do
    for rep in 1 2; do
      VISTA_LIB=$PWD/$lib timeout 300 python bench.py --config $c --steps 100 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null |
        python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('  $c', round(d['ms_per_step'],4), r.get('kernel_ms'), round(r['frac'],4), d['clocks']['sm_mhz'])"
    done
  done
done
