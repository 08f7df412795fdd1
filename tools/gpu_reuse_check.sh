#!/bin/bash
# Session script: bench line with the events-only kernel timing, then ncu
# launch lists (product kernels, cold / serialised) with owned-face reuse on
# and off at the M4 bench size.
mkdir -p gpurun_out
B="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/rc_bench.json 2> gpurun_out/rc_bench.err
PMHD_FACE_REUSE=0 $B > gpurun_out/rc_bench_noreuse.json 2> gpurun_out/rc_bench_noreuse.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_reuse.csv $CMD > gpurun_out/ncu1.log 2>&1
PMHD_FACE_REUSE=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_noreuse.csv $CMD > gpurun_out/ncu2.log 2>&1
python - <<'PY'
import json
for f in ["rc_bench", "rc_bench_noreuse"]:
    d = json.load(open(f"gpurun_out/{f}.json")); r = d["roofline"]
    print(f, f"{d['value']:.4g}", r["kernel"], f"frac={r['frac']:.3f}", r["update_kernel"]["avg_ms"])
PY
