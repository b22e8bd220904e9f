#!/bin/bash
# Quick check of the softmax backward: its GPU parity tests, then c2/c5 bench lines
# (value, ms/step, dK/dV kernel ms, roofline fraction).  usage: scripts/bwd_quick.sh [attn]
cd "$(dirname "$0")/.."
A=${1:-softmax}
timeout 600 python -m pytest tests -m gpu -x -q -k "backward" 2>&1 | tail -3
for c in c2 c5; do
  timeout 300 python bench.py --config $c --attn $A --backward --steps 100 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', d['value'], d['ms_per_step'], r.get('kernel_ms'), round(r['frac'],4))"
done
