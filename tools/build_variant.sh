#!/bin/bash
# Build a development variant of libguardian.so with extra -D flags for one
# source (A/B probes): tools/build_variant.sh <out.so> <source.cu> -DFLAG=...
set -e
OUT=$1; SRC=$2; shift 2
cd "$(dirname "$0")/.."
B=paper_2401_09290_b200/build
NV=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="-O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude -Ipaper_2401_09290_b200/csrc"
name=$(basename $SRC .cu)
$NV $ARCH $FL "$@" -c paper_2401_09290_b200/csrc/$SRC -o /tmp/var_$name.o
objs=$(ls $B/*.o | grep -v "/$name.o")
$NV $ARCH -shared -o $OUT $objs /tmp/var_$name.o -lpthread -ldl -lrt
echo built $OUT
