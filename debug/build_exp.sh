#!/bin/bash
# Build a library variant with an experimental fused-forward source:
#   debug/build_exp.sh <name> <fwd_tc.cu> <fwd_tc.cuh> [nvcc flags...]
# -> debug/libhtb200_<name>.so (other sources from the package).
set -e
name=$1; cu=$2; cuh=$3; shift 3
cd "$(dirname "$0")/.."
root=$(mktemp -d); tmp=$root/pkg/csrc; mkdir -p $tmp $root/include
cp include/*.h $root/include/
cp paper_2304_12152_b200/csrc/*.cu paper_2304_12152_b200/csrc/*.cuh $tmp/
cp $cu $tmp/fwd_tc.cu; cp $cuh $tmp/fwd_tc.cuh
mkdir -p $tmp/obj
for f in $tmp/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
    --expt-relaxed-constexpr "$@" -c $f -o $tmp/obj/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -cudart static $tmp/obj/*.o \
  -o debug/libhtb200_$name.so
rm -rf $root
echo built debug/libhtb200_$name.so
