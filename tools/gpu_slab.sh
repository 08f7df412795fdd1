#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
B="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e"
for sp in 0 32 64 128; do
  PMHD_SLAB_PLANES=$sp $B > gpurun_out/slab_$sp.json 2>gpurun_out/slab_$sp.err
  python -c "import json;d=json.load(open('gpurun_out/slab_$sp.json'));print('slab $sp', round(d['value']/1e9,4), 'e9 cups', round(d['ms_per_step'],3),'ms')" || tail -3 gpurun_out/slab_$sp.err
done
