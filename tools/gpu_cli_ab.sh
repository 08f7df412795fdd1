#!/bin/bash
# CLI A/B of the small / multi-block configs against older library builds
# (lib/exp/r_<rev>/libpmhd_gpu.so via LD_LIBRARY_PATH; the CLI's RUNPATH
# yields to it).  usage: gpu_cli_ab.sh <rev>...
B=paper_1905_04341_b200/bin/pmhd
mkdir -p gpurun_out/cli
for rep in 1 2; do
  for lib in current "$@"; do
    for c in linear_wave_64 orszag_tang_512 blast_256; do
      if [ "$lib" = current ]; then r=$(timeout 600 $B run --config examples/$c.in --out gpurun_out/cli/$c 2>&1 | head -1)
      else r=$(LD_LIBRARY_PATH=$PWD/paper_1905_04341_b200/lib/exp/r_$lib timeout 600 $B run --config examples/$c.in --out gpurun_out/cli/$c 2>&1 | head -1); fi
      echo "$lib $c: $r" | sed 's/  */ /g' | cut -c1-110
      rm -f gpurun_out/cli/*/snapshot.pmhd
    done
  done
done

