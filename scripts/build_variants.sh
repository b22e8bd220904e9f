#!/bin/bash
# Build A/B variants of libvista.so with extra -D flags: scripts/build_variants.sh name "-DFOO=1" ...
cd "$(dirname "$0")/.."
mkdir -p variants
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC,-O2 -shared -I include $flags -o variants/lib_$name.so paper_2510_22049_b200/csrc/*.cu -lcudart &
done
wait
ls -la variants
