#!/bin/bash
# tools/gpu_ab_quick.sh <variant>... : benches only (no pytest), each variant
# run twice interleaved; variants as in tools/gpu_ab.sh (lib/exp/<name>.so)
mkdir -p gpurun_out
B="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = default ]; then $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  elif [[ "$v" == *=* ]]; then env "$v" $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  else PMHD_GPU_LIB=paper_1905_04341_b200/lib/exp/libpmhd_gpu_$v.so $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err; fi
  python - "$v" <<'PY'
import json,sys
v=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/ab_{v}.json")); r=d["roofline"]
    print(f"{v:10s} cups={d['value']:.4g} ms/step={d['ms_per_step']:.3f} upd_ms={r['update_kernel']['avg_ms']:.3f} flux_frac={r['frac']:.3f} clk={d['clocks']['sm_mhz']}")
except Exception as e:
    print(v, "FAILED", e, open(f"gpurun_out/ab_{v}.err").read()[-500:])
PY
done; done
