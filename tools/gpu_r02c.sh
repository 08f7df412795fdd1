#!/bin/bash
# Round-2 CLI configs (eager module loading) + Roe / HLLE bench lines + GPU tests.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
bash tools/gpu_cli.sh > gpurun_out/cli_configs.txt 2>&1
grep -A1 "== run" gpurun_out/cli_configs.txt | grep cycles
grep -A2 "== bench" gpurun_out/cli_configs.txt | grep "gpu-" | cut -d, -f1,6
for r in roe hlle; do timeout 600 python bench.py --riemann $r --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$r.json 2> gpurun_out/bench_$r.err; done
python -c "
import json
for r in ['roe','hlle']:
    d=json.load(open(f'gpurun_out/bench_{r}.json')); print(r, d['value'])"
