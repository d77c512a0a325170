#!/bin/bash
# Build libmzslsum with the kernels' self-checks compiled in (MZS_DCHECK, common.cuh):
#   tools/debug_lib.sh [out.so]     (default tools/var/libmzslsum_checked.so)
# Run the GPU tests against it with MZS_LIB=<out.so>: a violated bound traps the launch.
set -e
out=${1:-tools/var/libmzslsum_checked.so}
mkdir -p $(dirname $out)
tmp=$(mktemp -d)
for src in paper_1811_10074_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden \
    -w --expt-relaxed-constexpr -I include -I paper_1811_10074_b200/csrc -DMZS_DEBUG_CHECKS=1 \
    -c $src -o $tmp/$(basename $src).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out $tmp/*.o -lcudart
rm -rf $tmp
echo $out
