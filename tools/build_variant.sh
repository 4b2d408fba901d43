#!/bin/bash
# build a library variant for A/B runs: tools/build_variant.sh <name> [nvcc -D flags...]
#   -> paper_2401_00710_b200/_lib/libdts_<name>.so (select with DTS_LIB=... or tools/ab_libs.sh)
set -e
cd "$(dirname "$0")/../paper_2401_00710_b200/csrc"
name=$1; shift
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v \
  --expt-relaxed-constexpr "$@" -shared -o ../_lib/libdts_$name.so dts_api.cu 2> ../_lib/ptxas_$name.log
grep -A1 'k_scatter_wcIjLi4ELi0' ../_lib/ptxas_$name.log | grep -o 'Used.*' | head -1
