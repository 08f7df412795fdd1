#!/bin/bash
# tools/build_exp_rev.sh <git-rev> <name> [nvcc -D flags]: build the GPU
# library from the sources at <git-rev> into lib/exp/libpmhd_gpu_<name>.so
# (A/B baseline for tools/gpu_ab.sh).
set -e
rev=$1; name=$2; shift 2
tmp=$(mktemp -d)
git archive "$rev" paper_1905_04341_b200/csrc/gpu include | tar -x -C "$tmp"
G=$tmp/paper_1905_04341_b200/csrc/gpu
mkdir -p paper_1905_04341_b200/lib/exp
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xlinker -Bsymbolic -std=c++17 -Xcompiler -fPIC \
  -I$tmp/include -I$G --expt-relaxed-constexpr -DPMHD_FAST_DIVSQRT "$@" -shared -o paper_1905_04341_b200/lib/exp/libpmhd_gpu_$name.so \
  $G/pmhd_gpu.cu $G/kernels_*.cu
rm -rf "$tmp"
