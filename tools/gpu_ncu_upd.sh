#!/bin/bash
# ncu --set full of one update-kernel launch at the M4 bench size, with
# source-level stalls: K=tma (PMHD_UPDATE=tma) or K=fused (default LDG kernel).
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
K=${K:-fused}
[ "$K" = tma ] && export PMHD_UPDATE=tma
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_update_$K" -s 1 -c 1 -o gpurun_out/prof_upd_$K $CMD > gpurun_out/ncu_upd.log 2>&1
tail -3 gpurun_out/ncu_upd.log
