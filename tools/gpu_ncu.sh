#!/bin/bash
# ncu session: launch list + full capture of selected kernels (regex $1, skip $2, count $3)
mkdir -p gpurun_out
CMD="python bench.py --size 128 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:$1" -s ${2:-0} -c ${3:-4} -o gpurun_out/prof_$4 $CMD > gpurun_out/ncu.log 2>&1
tail -2 gpurun_out/ncu.log
