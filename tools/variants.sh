#!/bin/bash
# Dev tool: build kernel-shape variants of libfastsv.so into variants/
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
rm -f variants/*.so
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fopenmp -shared -cudart static -I include $flags -Xptxas -v -o variants/libfastsv_$name.so paper_1910_05971_b200/csrc/fastsv.cu -ldl -lpthread -lgomp 2>&1 | grep -A2 "k_hook" | grep -E "spill|Used" | tr '\n' ' '; echo " <- $name"
done
