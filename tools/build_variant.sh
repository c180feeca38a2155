#!/bin/bash
# usage: tools/build_variant.sh name "-DMACRO=..." [source.cu]
# Builds _lib/variants/libskgpu_<name>.so: the in-tree objects with one
# source (default ns2d.cu) recompiled under extra macros; select it at run
# time with SKG_LIB_VARIANT=<name> (tools/var_sweep.sh A/B-tests variants).
set -e
name=$1; defs=$2; src=${3:-ns2d.cu}
cd "$(dirname "$0")/.."
L=paper_1807_01769_b200/_lib; C=paper_1807_01769_b200/csrc
mkdir -p $L/variants
obj=/tmp/skg_variant_$name.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I include -I $C $defs -c $C/$src -o $obj
objs=$(ls $L/*.o | grep -v "/${src%.cu}.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/variants/libskgpu_$name.so $objs $obj -lcudart -ldl
echo built $L/variants/libskgpu_$name.so
