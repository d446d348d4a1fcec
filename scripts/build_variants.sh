#!/bin/bash
# Build liblift variants (compile-time tuning knobs) into build/var_<name>.so for A/B runs.
# usage: scripts/build_variants.sh name "-DKNOB=V ..." [name2 "flags2" ...]
cd "$(dirname "$0")/.."
mkdir -p build
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC -shared -I include $flags paper_1502_02389_b200/csrc/lift.cu \
    -o build/var_$name.so &
done
wait
ls -la build/var_*.so
