#!/bin/bash
# unit_overhead.py for every variants/lib_*.so (env S, H, LENS passed through)
cd "$(dirname "$0")/.."
for lib in variants/lib_*.so; do
  echo "== $(basename $lib .so)"
  VISTA_LIB=$PWD/$lib timeout 300 python scripts/unit_overhead.py
done
