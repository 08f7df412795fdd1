#!/bin/bash
# Full default bench lines repeated, with and without an environment setting.
# usage: gpu_bench_rep.sh "VAR=val" [reps]
mkdir -p gpurun_out
for rep in $(seq ${2:-2}); do
  for e in "" "$1"; do
    env $e timeout 900 python bench.py --no-cpu-baseline > gpurun_out/rep.json 2> gpurun_out/rep.err
    python -c "
import json,sys
d=json.loads(open('gpurun_out/rep.json').read().strip().splitlines()[-1])
print(sys.argv[1] or 'default', round(d['value']/1e9,4), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e9,4), d['clocks'])" "$e"
  done
done
