#!/bin/bash
# Build a variant of libmzslsum.so with one source replaced/recompiled with extra flags:
#   tools/variant_lib.sh <out.so> <source.cu> [nvcc flags...]
# The source's basename names the object it replaces (copy an old version to /tmp/x/mz.cu).
# The other objects come from paper_1811_10074_b200/build/ (run build.py first).  Use with
# MZS_LIB=<out.so> (paper_1811_10074_b200/_lib.py) to A/B kernels on the GPU.
set -e
out=$1; src=$2; shift 2
B=paper_1811_10074_b200/build
base=$(basename $src)
base=${base%.tmp}
tmpo=$(mktemp /tmp/varXXXX.o)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden \
  -w --expt-relaxed-constexpr -I include -I paper_1811_10074_b200/csrc "$@" -c $src -o $tmpo
objs=$(ls $B/*.o | grep -v "/${base%.cu}.cu.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out $objs $tmpo -lcudart
rm -f $tmpo
echo $out
