#!/bin/bash
# Build an A/B variant of libalora_sm100a.so with one source recompiled under extra -D flags (load it with
# ALORA_LIB=paper_2512_17910_b200/variants/<name>.so). Run after `make` in paper_2512_17910_b200/.
# usage: tools/build_variant.sh <name> <source stem, e.g. attn_bf16> <nvcc -D flags...>
set -e
name=$1; stem=$2; shift 2
cd "$(dirname "$0")/../paper_2512_17910_b200"
mkdir -p variants
NV=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
$NV $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -cudart static --expt-relaxed-constexpr "$@" \
    -c csrc/$stem.cu -o variants/$name.$stem.o 2> variants/$name.ptxas.log || { tail -20 variants/$name.ptxas.log; exit 1; }
objs=$(ls build/*.o | grep -v "build/$stem.o")
$NV $ARCH -shared -cudart static -o variants/$name.so $objs variants/$name.$stem.o -lpthread
echo "variants/$name.so"
