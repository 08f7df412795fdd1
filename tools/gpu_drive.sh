#!/bin/bash
# Turbulence-driving session: driven parity tests (GPU and gloo), the 512^3
# decaying / driven CLI benches, and the ncu launch list of one driving event.
set -x
python -m pytest tests/test_gpu_parity.py -q -x -k "driven or drive" 2>&1 | tail -3
python -m pytest tests/test_drive.py tests/test_parallel_cpu.py -q -x -k driven 2>&1 | tail -2
B=paper_1905_04341_b200/bin/pmhd
for c in turbulence_512 turbulence_driven_512; do timeout 900 $B bench --config examples/$c.in --cycles 10 --warmup 2 2>&1 | tail -2; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_drive --csv --log-file gpurun_out/drive_launches.csv $B bench --config examples/turbulence_driven_512.in --cycles 2 --warmup 0 > /dev/null 2>&1
python tools/ncu_lines.py gpurun_out/drive_launches.csv 2>&1 | head -20 || true
