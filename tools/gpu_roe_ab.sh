#!/bin/bash
# Roe A/B: GPU tests, then the bench with --riemann roe for the base / default /
# 5-CTA builds (lib/exp), and the Roe parity tests against the 5-CTA build.
L=paper_1905_04341_b200/lib
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
B="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
for v in base default roe5; do
  if [ $v = default ]; then $B --riemann roe > gpurun_out/r_$v.json 2>/dev/null; else PMHD_GPU_LIB=$L/exp/libpmhd_gpu_$v.so $B --riemann roe > gpurun_out/r_$v.json 2>/dev/null; fi
  python -c "import json; d=json.loads(open('gpurun_out/r_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'])"
done; done
if [ $v = default ]; then :; fi
$B > gpurun_out/r_hlld.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r_hlld.json').read().strip().splitlines()[-1]); print('hlld default', d['value'])"
cp $L/exp/libpmhd_gpu_roe5_parity.so $L/libpmhd_gpu_parity.so
PMHD_GPU_LIB=$L/exp/libpmhd_gpu_roe5.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "roe" 2>&1 | tail -2
