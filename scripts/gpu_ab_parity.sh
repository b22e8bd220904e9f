#!/bin/bash
# For each variants/lib_*.so: GPU parity tests through that library, then kernel numbers on CONFIGS.
cd "$(dirname "$0")/.."
for lib in variants/lib_*.so; do
  n=$(basename $lib .so)
  echo "== $n: $(VISTA_LIB=$PWD/$lib timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1)"
done
CONFIGS="${CONFIGS:-c2 c4 c5}" STEPS=${STEPS:-100} bash scripts/ab_variants_cfg.sh
