#!/bin/bash
# build an experiment variant of the library: tools/exp_build.sh NAME [nvcc -D flags...]
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_1305_3122_b200"
srcs=$(python3 -c "import re;print(' '.join('csrc/'+s for s in re.search(r'SOURCES = \[(.*?)\]', open('build.py').read()).group(1).replace('\"','').split(', ')))")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -shared "$@" \
  -o ../tools/exp/lib_$name.so $srcs
