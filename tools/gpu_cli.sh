#!/bin/bash
# CLI runs of the BASELINE.json configs through the C++ host (pmhd run / bench)
mkdir -p gpurun_out/cli
B=paper_1905_04341_b200/bin/pmhd
for c in linear_wave_64 orszag_tang_512 blast_256; do
  echo "== run $c"; timeout 600 $B run --config examples/$c.in --out gpurun_out/cli/$c 2>&1 | tail -4
done
for c in blast_256 turbulence_512; do
  echo "== bench $c"; timeout 900 $B bench --config examples/$c.in --cycles 10 --warmup 2 2>&1 | tail -2
done
cat gpurun_out/cli/linear_wave_64/errors.csv
ls -la gpurun_out/cli/*/
rm -f gpurun_out/cli/*/snapshot.pmhd
