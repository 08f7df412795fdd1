"""Weak-scaling projection for the N>1 bench flow, from one-GPU measurements
(no kernel waits on another): the halo bytes a rank sends per stage (exact,
pmhd_gpu_halo_count), the measured pack / unpack kernel times of a 256^3
rank-engine, and the measured stage time, against the NVLink peer-copy
bandwidth the profiling recipe gives (770 GB/s per direction).  Prints a
JSON line; it is a model, not a multi-GPU measurement.

usage: python tools/halo_model.py [n]      (n^3 cells per rank, default 256)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1905_04341_b200.parallel import plan_for  # noqa: E402
from paper_1905_04341_b200.solver import GpuSolver  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
NVLINK = 770e9  # measured peer copy per direction (B200_PROFILING.md)
ranks = 2
cfg = bench.make_config(n, ranks)  # (2n) x n x n, one block per rank
plan = plan_for(cfg, ranks)
g = GpuSolver(cfg, gids=plan.local_gids(0))
g.load_pgen(exchange=False)
g.set_async(True)  # stream-ordered calls (as over NCCL): the events time the kernels, not host syncs
stream = torch.cuda.ExternalStream(g.stream_handle)
sends, recvs = plan.messages(0, 0)
bufs = [(gid, side, g.alloc_halo(g.halo_count(0, 1 - side))) for _, _, gid, side in sends]
msg_bytes = sum(b.numel() * 8 for _, _, b in bufs)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
dt = g.new_dt()
for _ in range(2):  # warm-up
    g.stage_compute(1, dt)
reps = 5
ev[0].record(stream)
for _ in range(reps):
    g.stage_compute(1, dt)
ev[1].record(stream)
for _ in range(reps):
    for gid, side, b in bufs:
        g.halo_pack(gid, 0, side, 1, b)
    for gid, side, b in bufs:
        g.halo_unpack(gid, 0, side, 1, b)
ev[2].record(stream)
torch.cuda.synchronize()
stage_ms = ev[0].elapsed_time(ev[1]) / reps
packunpack_ms = ev[1].elapsed_time(ev[2]) / reps
wire_ms = msg_bytes / NVLINK * 1e3
# per stage: the stage-1 exchange overlaps the stage-2 interior tiles (~75 % of
# the flux work), the stage-2 one is exposed; + ~20 us for the dt all-reduce
exposed_ms = 0.5 * (packunpack_ms + wire_ms) + 0.01
eff = stage_ms / (stage_ms + exposed_ms)
print(json.dumps({"cells_per_rank": n ** 3, "halo_bytes_per_stage": msg_bytes,
                  "stage_ms": stage_ms, "pack_unpack_ms": packunpack_ms,
                  "nvlink_wire_ms_at_770GBps": wire_ms,
                  "projected_weak_efficiency": eff,
                  "note": "model from one-GPU measurements; not a multi-GPU run"}))
