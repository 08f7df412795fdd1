#!/bin/bash
# Full measurement session: reference arm, our arm (default args), ncu launch
# list + full capture of the dominant kernels at the bench workload.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/launches_256.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_update_fused|k_edge_emf|k_cell_update|k_flux_fused|k_flux_march|k_flux_x1march" -s 0 -c 10 -o gpurun_out/prof_256 $CMD > gpurun_out/ncu.log 2>&1
cat gpurun_out/bench_ref.json gpurun_out/bench.json; tail -n 2 gpurun_out/bench.err gpurun_out/ncu.log
