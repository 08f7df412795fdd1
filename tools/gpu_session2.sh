#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
CMD="python bench.py --size 128 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_flux -s 3 -c 3 -o gpurun_out/prof_flux $CMD > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/ncu.log; ls -la gpurun_out
