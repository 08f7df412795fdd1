B=paper_1905_04341_b200/bin/pmhd
mkdir -p gpurun_out/cli
for rep in 1 2 3 4 5 6; do for e in PMHD_FLUX_CONC=0 PMHD_FLUX_CONC=1; do
  r=$(env $e timeout 600 $B run --config examples/linear_wave_64.in --out gpurun_out/cli/lw 2>&1 | head -1)
  echo "$e $r" | sed 's/  */ /g' | cut -c1-120
done; done
