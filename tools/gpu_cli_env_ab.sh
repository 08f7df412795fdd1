#!/bin/bash
# CLI A/B of the BASELINE configs under environment settings.
# usage: gpu_cli_env_ab.sh "VAR=a" "VAR=b" ...
B=paper_1905_04341_b200/bin/pmhd
mkdir -p gpurun_out/cli
for rep in 1 2; do
  for e in "$@"; do
    for c in ${CONFIGS:-linear_wave_64 blast_256 turbulence_512}; do
      if [ "$c" = turbulence_512 ]; then r=$(env $e timeout 600 $B bench --config examples/$c.in --cycles 10 --warmup 2 2>&1 | tail -1)
      else r=$(env $e timeout 600 $B run --config examples/$c.in --out gpurun_out/cli/$c 2>&1 | head -1); fi
      echo "$e $c: $r" | sed 's/  */ /g' | sed 's/,gpu-fused.*split[^,]*,/ /' | cut -c1-140
      rm -f gpurun_out/cli/*/snapshot.pmhd
    done
  done
done
