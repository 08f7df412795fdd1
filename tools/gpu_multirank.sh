#!/bin/bash
# Multi-rank checks on one GPU: the loopback / IPC parity tests, the halo
# model for the 2- and 8-rank decompositions, and the N=8 bench flow with
# host-staged gloo transport (a validation run, never a measurement).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "multirank or ipc" 2>&1 | tail -2
for r in 2 8; do timeout 600 python tools/halo_model.py 256 $r > gpurun_out/halo_model_256_n$r.json 2> gpurun_out/halo_model_n$r.err; tail -c 700 gpurun_out/halo_model_256_n$r.json; tail -2 gpurun_out/halo_model_n$r.err; done
PMHD_BENCH_TRANSPORT=gloo-host timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 \
  --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 8 --size 64 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_gloo8.json 2> gpurun_out/bench_gloo8.err
echo "gloo8 rc=$?"; tail -c 900 gpurun_out/bench_gloo8.json; tail -3 gpurun_out/bench_gloo8.err
# M5 strong-scaling flow at 2 ranks (gloo-host), default kernels
PMHD_BENCH_TRANSPORT=gloo-host timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 2 --workload m5 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_gloo2_m5.json 2> gpurun_out/bench_gloo2_m5.err
echo "gloo2 m5 rc=$?"; tail -c 600 gpurun_out/bench_gloo2_m5.json; tail -3 gpurun_out/bench_gloo2_m5.err
