#!/bin/bash
# CLI runs of the BASELINE.json configs through the C++ host (pmhd run / bench)
mkdir -p gpurun_out/cli
B=paper_1905_04341_b200/bin/pmhd
for c in linear_wave_64 orszag_tang_512 blast_256; do
  echo "== run $c"; timeout 600 $B run --config examples/$c.in --out gpurun_out/cli/$c 2>&1 | tail -4
done
echo "== run turbulence_driven_512"; timeout 600 $B run --config examples/turbulence_driven_512.in --out gpurun_out/cli/turb_driven 2>&1 | tail -3
for c in blast_256 turbulence_512 turbulence_driven_512 linear_wave_256; do
  echo "== bench $c"; timeout 900 $B bench --config examples/$c.in --cycles 10 --warmup 2 2>&1 | tail -2
done
cat gpurun_out/cli/linear_wave_64/errors.csv
ls -la gpurun_out/cli/*/
rm -f gpurun_out/cli/*/snapshot.pmhd
for c in report roofline; do $B $c --config examples/linear_wave_256.in --platform profiles/platforms.csv --out gpurun_out/cli/$c 2>&1 | tail -2; done
cat gpurun_out/cli/report/profile.csv gpurun_out/cli/roofline/portability.csv
