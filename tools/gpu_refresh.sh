#!/bin/bash
# Evidence refresh for profiles/r01: tools/gpu_full.sh (both bench arms, ncu
# launch list, ncu --set full of one cycle) plus the CLI configs.
bash tools/gpu_full.sh > gpurun_out/full.log 2>&1
tail -c 400 gpurun_out/bench.json
bash tools/gpu_cli.sh > gpurun_out/cli_configs.txt 2>&1; grep -A1 "== bench" gpurun_out/cli_configs.txt | grep -v "^--" | grep -v "^size" | head -12
