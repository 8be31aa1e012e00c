#!/bin/bash
# Dev tool: build kernel-shape variants of libfastsv.so into /tmp/fsv_var/
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/var
for v in "T768_S4:-DFSV_HOOK_THREADS=768 -DFSV_STEPS=4" "T1024_S4:-DFSV_HOOK_THREADS=1024 -DFSV_STEPS=4" "T512_S4:-DFSV_HOOK_THREADS=512 -DFSV_STEPS=4" "T768_S16:-DFSV_HOOK_THREADS=768 -DFSV_STEPS=16" "T768_S1:-DFSV_HOOK_THREADS=768 -DFSV_STEPS=1"; do
  name=${v%%:*}; flags=${v#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -cudart static -I include $flags -Xptxas -v -o variants/libfastsv_$name.so paper_1910_05971_b200/csrc/fastsv.cu -ldl -lpthread 2>&1 | grep -A2 "k_hook" | grep -E "spill|Used" | tr '\n' ' '; echo " <- $name"
done
