#!/bin/bash
# tools/regs.sh <source.cu> [nvcc -D flags...]: registers / spills per kernel
# (ptxas -v), demangled to "kernel<template args>".
src=$1; shift
G=paper_1905_04341_b200/csrc/gpu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -I$G --expt-relaxed-constexpr \
  "$@" -Xptxas -v -c "$src" -o /tmp/regs_$$.o 2>&1 |
  awk '/Compiling entry function/ {match($0, /_Z[A-Za-z0-9_]*/); name=substr($0, RSTART, RLENGTH)}
       /spill stores/ {match($0, /[0-9]+ bytes spill stores/); sp=substr($0, RSTART, RLENGTH)}
       /Used [0-9]+ registers/ {match($0, /Used [0-9]+ registers/); print name, substr($0, RSTART, RLENGTH), sp}' |
  c++filt | sed -E 's/pmhd_gpu::\(anonymous namespace\):://; s/\(.*\)//'
rm -f /tmp/regs_$$.o
