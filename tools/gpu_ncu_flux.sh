#!/bin/bash
# ncu --set full of the flux kernels of one VL2 cycle at the M4 bench size
# (x1, x2, x3 of both stages), with source-level stalls.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_flux_fused" -s 6 -c 6 -o gpurun_out/prof_flux $CMD > gpurun_out/ncu_flux.log 2>&1
tail -3 gpurun_out/ncu_flux.log
