#!/bin/bash
# build an experiment variant of the library: tools/exp_build.sh NAME [nvcc -D flags...]
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_1305_3122_b200"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -shared "$@" \
  -o ../tools/exp/lib_$name.so csrc/fa_capi.cu csrc/fa_assembly.cu csrc/fa_batch.cu csrc/fa_triplets.cu csrc/fa_selftest.cu
