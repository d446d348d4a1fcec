#!/bin/bash
# Build tuning variants of liblift.so into build/ (same ABI, different -D knobs).
cd "$(dirname "$0")/.."
mkdir -p build
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Iinclude"
while [ $# -gt 0 ]; do
  name=$1; defs=$2; shift 2
  nvcc $F $defs paper_1502_02389_b200/csrc/lift.cu -o build/liblift_$name.so &
done
wait
ls build/
