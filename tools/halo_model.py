"""Weak-scaling projection for the N>1 bench flow, from one-GPU measurements
(no kernel waits on another).  Rank 0 of the bench's N-rank decomposition
(bench.rank_grid: 2 -> 2x1x1, 8 -> 2x2x2 blocks of n^3) is built on one GPU
together with the rank-engines that own its neighbours; measured with CUDA
events in stream-ordered mode:

* pack / transport / unpack path: the pack + unpack kernels of a stage's
  halo (exact bytes from pmhd_gpu_halo_count) + the NVLink wire time at the
  profiling recipe's measured peer-copy bandwidth (770 GB/s per direction);
* peer-memory path (default on one node): the three exchange sweeps reading
  the other engine's memory (here local HBM; on the box the remote part
  crosses NVLink, added as wire time) + three barriers (~10 us each, an
  NCCL one-int all-reduce).

The stage-1 exchange overlaps the stage-2 interior flux tiles; the stage-2
exchange and the 8-byte dt all-reduce are exposed.  The reference is the
N = 1 stage time of one all-local n^3 block measured the same way (it uses
owned-face reuse, which a rank with remote neighbours does not), so the
projected efficiency includes that difference too.  Prints a JSON line: a
model, not a multi-GPU measurement.

usage: python tools/halo_model.py [n] [nranks]   (n^3 cells per rank, default 256; default 2 ranks)
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
nranks = int(sys.argv[2]) if len(sys.argv) > 2 else 2
NVLINK = 770e9
BARRIER_MS = 0.010
cfg = bench.make_config(n, nranks)
plan = plan_for(cfg, nranks)
# rank 0 and the ranks owning its neighbours
need = sorted({0} | {plan.owners[plan.neighbour(plan.local_gids(0)[0], d, sd)]
                     for d in range(cfg.dim) for sd in (0, 1)})
engs = {r: GpuSolver(cfg, gids=plan.local_gids(r)) for r in need}
for e in engs.values():
    e.load_pgen(exchange=False)
    e.set_async(True)
g = engs[0]
stream = torch.cuda.ExternalStream(g.stream_handle)
bufs = []  # (dir, gid, side, buffer) of every message rank 0 sends
for d in range(cfg.dim):
    sends, _ = plan.messages(0, d)
    bufs += [(d, gid, side, g.alloc_halo(g.halo_count(d, 1 - side))) for _, _, gid, side in sends]
msg_bytes = sum(b.numel() * 8 for _, _, _, b in bufs)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
dt = g.new_dt()
for _ in range(2):
    g.stage_compute(1, dt)
reps = 5
ev[0].record(stream)
for _ in range(reps):
    g.stage_compute(1, dt)
ev[1].record(stream)
for _ in range(reps):
    for d, gid, side, b in bufs:
        g.halo_pack(gid, d, side, 1, b)
    for d, gid, side, b in bufs:
        g.halo_unpack(gid, d, side, 1, b)
ev[2].record(stream)
# peer-memory sweeps: engine 0 reads engine 1's slab directly
bases = [engs[r].slab()[0] if (r in engs and r != 0) else None for r in range(nranks)]
g.peer_attach(plan.owners, bases)
for _ in range(reps):
    for d in range(cfg.dim):
        g.exchange_dir(d, 1)
ev[3].record(stream)
torch.cuda.synchronize()
stage_ms = ev[0].elapsed_time(ev[1]) / reps
# N = 1 reference: one all-local n^3 block, same measurement
cfg1 = bench.make_config(n, 1)
g1 = GpuSolver(cfg1)
g1.load_pgen(exchange=True)
g1.set_async(True)
s1 = torch.cuda.ExternalStream(g1.stream_handle)
dt1 = g1.new_dt()
for _ in range(2):
    g1.stage_compute(1, dt1)
e1 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
e1[0].record(s1)
for _ in range(reps):
    g1.stage_compute(1, dt1)
e1[1].record(s1)
torch.cuda.synchronize()
stage1_ms = e1[0].elapsed_time(e1[1]) / reps
packunpack_ms = ev[1].elapsed_time(ev[2]) / reps
sweeps_ms = ev[2].elapsed_time(ev[3]) / reps
wire_ms = msg_bytes / NVLINK * 1e3
# both paths run the three sweeps (local faces; the p2p sweeps also read the
# remote ones); the pack path adds the pack / unpack kernels
x_pack = sweeps_ms + packunpack_ms + wire_ms
x_p2p = sweeps_ms + wire_ms + 3 * BARRIER_MS
res = {"cells_per_rank": n ** 3, "nranks": nranks, "rank_grid": bench.rank_grid(nranks),
       "halo_bytes_per_stage": msg_bytes, "stage_ms": stage_ms, "stage_ms_n1": stage1_ms,
       "pack_unpack_ms": packunpack_ms, "p2p_sweeps_ms": sweeps_ms,
       "nvlink_wire_ms_at_770GBps": wire_ms,
       "projected_weak_efficiency_pack": stage1_ms / (stage_ms + 0.5 * x_pack + 0.01),
       "projected_weak_efficiency_p2p": stage1_ms / (stage_ms + 0.5 * x_p2p + 0.01),
       "note": "model from one-GPU measurements (tools/halo_model.py); not a multi-GPU run"}
print(json.dumps(res))
