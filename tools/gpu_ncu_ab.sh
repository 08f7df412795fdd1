#!/bin/bash
# ncu A/B: full capture of the 6 flux launches of one cycle (128^3) for each
# library variant given (default = lib/libpmhd_gpu.so, else lib/exp/libpmhd_gpu_<v>.so).
mkdir -p gpurun_out
CMD="python bench.py --size 128 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
for v in "$@"; do
  if [ "$v" = default ]; then unset PMHD_GPU_LIB; else export PMHD_GPU_LIB=paper_1905_04341_b200/lib/exp/libpmhd_gpu_$v.so; fi
  $CMD > gpurun_out/plain_$v.log 2>&1 || { echo "$v plain run failed"; continue; }
  ncu --set full --clock-control none --import-source on -k "regex:${NCU_K:-k_flux_fused}" -s ${NCU_S:-0} -c ${NCU_C:-6} \
    -o gpurun_out/prof_$v $CMD > gpurun_out/ncu_$v.log 2>&1
  tail -1 gpurun_out/ncu_$v.log
done
