#!/bin/bash
# Debug session for the TMA-staged update kernel: a small 3D case through the
# product library and the debug variants (1: no TMA, 2: EMF group only, 3:
# cell group only).
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for lib in "" exp/libpmhd_gpu_dbg1.so exp/libpmhd_gpu_dbg2.so exp/libpmhd_gpu_dbg3.so; do
  for n in 16 64; do
    if [ -z "$lib" ]; then r=$(timeout 120 python tools/tma_debug.py $n 2>&1 | tail -1)
    else r=$(PMHD_GPU_LIB=paper_1905_04341_b200/lib/$lib timeout 120 python tools/tma_debug.py $n 2>&1 | tail -1); fi
    echo "lib=${lib:-product} n=$n: $r"
  done
done
echo "--- standalone probe"; timeout 60 ./tools/probe/tma_probe
echo "--- round-1 TMA E ring (k_update_fused, PMHD_UPDATE_TMA=1 build)"
PMHD_UPDATE=ldg PMHD_GPU_LIB=paper_1905_04341_b200/lib/exp/libpmhd_gpu_oldtma.so timeout 120 python tools/tma_debug.py 16 2>&1 | tail -1
