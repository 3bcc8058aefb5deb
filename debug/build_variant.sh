#!/bin/bash
# Build a debug variant of the library: debug/libhtb200_<name>.so with extra
# nvcc defines, e.g.  debug/build_variant.sh pf -DHT_PROF
# Use with HTB200_LIB=debug/libhtb200_<name>.so python debug/prof.py
set -e
name=$1; shift
cd "$(dirname "$0")/.."
out=debug/obj_$name; mkdir -p $out
for f in paper_2304_12152_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
    --expt-relaxed-constexpr "$@" -c $f -o $out/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -cudart static $out/*.o \
  -L/usr/local/cuda/lib64 -lcufft -Xlinker -rpath,/usr/local/cuda/lib64 -o debug/libhtb200_$name.so
rm -rf $out
echo built debug/libhtb200_$name.so
