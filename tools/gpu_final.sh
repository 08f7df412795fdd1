#!/bin/bash
# Round-end check: GPU tests, both bench arms (default args) and the CLI
# configs; outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 600 gpurun_out/bench.json
bash tools/gpu_cli.sh > gpurun_out/cli_configs.txt 2>&1; tail -5 gpurun_out/cli_configs.txt
