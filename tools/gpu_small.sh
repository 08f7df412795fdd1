#!/bin/bash
# Small-mesh configs (M1 64^3, M2 512^2) through the CLI, then the GPU tests.
B=paper_1905_04341_b200/bin/pmhd
mkdir -p gpurun_out/cli
for c in linear_wave_64 orszag_tang_512 blast_256; do
  echo "== run $c"; timeout 600 $B run --config examples/$c.in --out gpurun_out/cli/$c 2>&1 | head -1
done
rm -f gpurun_out/cli/*/snapshot.pmhd
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
