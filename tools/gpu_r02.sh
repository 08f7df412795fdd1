#!/bin/bash
# Round-2 evidence session: both bench arms (default args), ncu launch list
# and ncu --set full of one cycle at the M4 size, the M5 and 8x128^3 bench
# variants, and the BASELINE configs through the C++ CLI.
mkdir -p gpurun_out
bash tools/gpu_full.sh > gpurun_out/full.log 2>&1
timeout 900 python bench.py --workload m5 > gpurun_out/bench_m5.json 2> gpurun_out/bench_m5.err
timeout 900 python bench.py --block 128 > gpurun_out/bench_b128.json 2> gpurun_out/bench_b128.err
bash tools/gpu_cli.sh > gpurun_out/cli_configs.txt 2>&1
tail -c 300 gpurun_out/bench.json; grep -A1 "== bench" gpurun_out/cli_configs.txt | grep -v "^--" | head -12
for r in roe hlle; do timeout 600 python bench.py --riemann $r --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$r.json 2> gpurun_out/bench_$r.err; done
