"""Multi-rank VL2 driver: one process per GPU, MeshBlocks sharded over ranks.

The path shards by MeshBlock.  Its real
exchange steps are (1) the ghost + face-B halo after every stage and (2) the
dt minimum after stage 2.  This module is the host-side plan
for both:

* ``partition``: compact bricks of blocks per rank;
* ``HaloPlan``: for every local block face, the neighbour block and its owner;
* ``DistributedVL2``: a stage = engine.stage_compute + for each direction
  (x1, x2, x3, in the order of exchange_ghosts' sweeps):
  local sweep + pack -> transport -> unpack of the slabs that cross a rank
  boundary; then an all-reduce(min) of dt.  With the sweeps kept sequential,
  the result is bit-identical to the single-process exchange.

Halo data paths: the peer-memory halo (default for GPU engines on one node:
the ranks map each other's state slabs over CUDA IPC and the exchange kernels
read remote boundary layers directly over NVLink, one barrier per sweep
direction), or pack -> transport -> unpack.  Transports:
``TorchDistTransport`` (torch.distributed: NCCL over NVLink, ordered on the
engine's stream; gloo for CPU buffers) and ``LoopbackWorld`` (several engines
in one process, used to test every GPU path on one GPU without kernels that
wait on each other).

An *engine* is ``solver.GpuSolver`` (product) or, in tests only, the CPU
oracle binding; both expose stage_compute / exchange_dir / halo_count /
alloc_halo / halo_pack / halo_unpack / gids.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field


def _factor(n):
    f, p = [], 2
    while n > 1:
        while n % p == 0:
            f.append(p)
            n //= p
        p += 1
    return f


def partition(nb, nranks):
    """Split a block grid nb = (nb1, nb2, nb3) into nranks compact bricks;
    returns owners[gid] (gid = (k*nb2 + j)*nb1 + i).  Factors of nranks go to
    the block-grid axis with the most blocks per rank left."""
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    split = [1, 1, 1]
    for p in sorted(_factor(nranks), reverse=True):
        best = max(range(3), key=lambda a: (nb[a] // split[a]) if (nb[a] // split[a]) % p == 0 else -1)
        if (nb[best] // split[best]) % p != 0:
            raise ValueError(f"cannot split block grid {tuple(nb)} over {nranks} ranks")
        split[best] *= p
    owners = []
    for gid in range(nb[0] * nb[1] * nb[2]):
        c = (gid % nb[0], (gid // nb[0]) % nb[1], gid // (nb[0] * nb[1]))
        r = [c[a] // (nb[a] // split[a]) for a in range(3)]
        owners.append((r[2] * split[1] + r[1]) * split[0] + r[0])
    return owners


@dataclass
class HaloPlan:
    nb: tuple
    owners: list
    dim: int

    def neighbour(self, gid, d, side):
        nb = self.nb
        c = [gid % nb[0], (gid // nb[0]) % nb[1], gid // (nb[0] * nb[1])]
        c[d] = (c[d] + (1 if side else -1)) % nb[d]
        return (c[2] * nb[1] + c[1]) * nb[0] + c[0]

    def local_gids(self, rank):
        return [g for g, o in enumerate(self.owners) if o == rank]

    def messages(self, rank, d):
        """(sends, recvs) of rank in direction d.  A message is keyed by the
        RECEIVING block face (gid, side): sends = [(peer, key, my_gid, my_side)],
        recvs = [(peer, key)] with key = (my_gid, my_side).  Both lists are
        sorted by (peer, key), so a peer pair posts matching operations in the
        same order (NCCL P2P matches in order)."""
        sends, recvs = [], []
        for gid in self.local_gids(rank):
            for side in (0, 1):
                nbr = self.neighbour(gid, d, side)
                peer = self.owners[nbr]
                if peer == rank:
                    continue
                sends.append((peer, (nbr, 1 - side), gid, side))
                recvs.append((peer, (gid, side)))
        sends.sort(key=lambda s: (s[0], s[1]))
        recvs.sort()
        return sends, recvs


def plan_for(cfg, nranks):
    m = cfg.desc
    nb = (m.nx[0] // m.mb[0], m.nx[1] // m.mb[1], m.nx[2] // m.mb[2])
    return HaloPlan(nb, partition(nb, nranks), cfg.dim)


class TorchDistTransport:
    """torch.distributed point-to-point + all-reduce (nccl or gloo)."""

    def __init__(self, dist, group=None, host_staging=False):
        self.dist = dist
        self.group = group
        # host_staging: device buffers go through host memory (gloo cannot
        # send CUDA tensors); used to validate the multi-rank GPU path with
        # several processes on one GPU, never for measurements.
        self.host_staging = host_staging
        # NCCL on CUDA buffers can be ordered on the engine's stream: no host
        # synchronization inside a stage (DistributedVL2 enables it).
        self.stream_ordered = (not host_staging) and dist.get_backend(group) == "nccl"

    def exchange(self, out, inb, stream=None):
        """out / inb: lists of (peer, tensor) in posting order.  stream: a
        torch stream the transfers are ordered on (stream_ordered transports):
        they start after the work already enqueued on it and later work on it
        waits for them, without blocking the host."""
        if self.host_staging:
            out = [(p, t.cpu()) for p, t in out]
            tmp = [(p, t, t.new_empty(t.shape, device="cpu")) for p, t in inb]
            inb_x = [(p, c) for p, _, c in tmp]
        else:
            inb_x = inb
        ops = [self.dist.P2POp(self.dist.isend, t, p, group=self.group) for p, t in out]
        ops += [self.dist.P2POp(self.dist.irecv, t, p, group=self.group) for p, t in inb_x]
        if ops and stream is not None:
            import torch
            with torch.cuda.stream(stream):
                for req in self.dist.batch_isend_irecv(ops):
                    req.wait()  # NCCL: the stream waits, the host does not
        elif ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
            # NCCL completes on torch's current stream; the ABI unpacks on its
            # own stream, so make the received bytes visible first.
            if any(t.is_cuda for _, t in inb_x):
                import torch
                torch.cuda.current_stream().synchronize()
        if self.host_staging:
            for _, t, c in tmp:
                t.copy_(c)

    def barrier(self, stream=None):
        """All ranks reached this point.  With a stream (stream-ordered NCCL):
        a one-int all-reduce ordered on it -- work enqueued after it on that
        stream starts only once every rank's earlier work on its stream is
        done; the host does not wait."""
        if stream is not None and self.stream_ordered:
            import torch
            with torch.cuda.stream(stream):
                if not hasattr(self, "_flag"):
                    self._flag = torch.zeros(1, dtype=torch.int32, device=torch.cuda.current_device())
                self.dist.all_reduce(self._flag, group=self.group)
        else:
            self.dist.barrier(group=self.group)

    def allgather(self, obj):
        """Python objects of every rank (rank order)."""
        out = [None] * self.dist.get_world_size(self.group)
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def min(self, x, device=None):
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=None if self.host_staging else device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return float(t.item())


@dataclass
class _Bufs:
    send: dict = field(default_factory=dict)
    recv: dict = field(default_factory=dict)


class DistributedVL2:
    """vl2_step over a rank-local engine (SPEC.md:209-217 across ranks)."""

    def __init__(self, engine, plan, rank, transport, device=None):
        self.e, self.plan, self.rank, self.tr, self.device = engine, plan, rank, transport, device
        self.bufs = {}
        for d in range(plan.dim):
            sends, recvs = plan.messages(rank, d)
            b = _Bufs()
            for peer, key, gid, side in sends:
                b.send[key] = engine.alloc_halo(engine.halo_count(d, 1 - side))
            for peer, key in recvs:
                b.recv[key] = engine.alloc_halo(engine.halo_count(d, key[1]))
            self.bufs[d] = (sends, recvs, b)
        # peer-memory halo (one node): every rank maps the others' state slabs
        # (CUDA IPC) and exchange_dir reads remote boundary layers directly
        # over NVLink; a barrier per direction orders it.  PMHD_P2P_HALO=0
        # keeps pack -> transport -> unpack.
        self.p2p = False
        if (hasattr(engine, "peer_attach") and hasattr(transport, "allgather")
                and os.environ.get("PMHD_P2P_HALO", "1") != "0"):
            self.p2p = self._attach_peers(engine, plan, rank, transport)
        # stream-ordered stages: halo sweeps / NCCL on the engine's stream;
        # the host synchronizes once per cycle (stage 2 status + dt)
        self.stream = None
        if (getattr(transport, "stream_ordered", False) and hasattr(engine, "set_async")
                and os.environ.get("PMHD_SYNC_HALO", "0") != "1"):
            engine.set_async(True)
            self.stream = engine.torch_stream()

    def _attach_peers(self, engine, plan, rank, transport):
        base, handle = engine.slab()
        handles = transport.allgather(handle)
        self.peer_bases = []
        ok = True
        for r, h in enumerate(handles):
            if r == rank:
                self.peer_bases.append(None)
                continue
            try:
                self.peer_bases.append(engine.ipc_open(h))
            except Exception:  # no IPC / peer access: fall back for everyone
                self.peer_bases.append(None)
                ok = False
        ok = all(transport.allgather(ok))
        if not ok:
            for b in self.peer_bases:
                if b:
                    engine.ipc_close(b)
            self.peer_bases = []
            return False
        engine.peer_attach(plan.owners, self.peer_bases)
        return True

    def exchange(self, half):
        if self.p2p:  # direct peer reads: one barrier per sweep direction
            for d in range(self.plan.dim):
                self.tr.barrier(self.stream)
                self.e.exchange_dir(d, half)
            return
        for d in range(self.plan.dim):
            self.e.exchange_dir(d, half)
            sends, recvs, b = self.bufs[d]
            for peer, key, gid, side in sends:
                self.e.halo_pack(gid, d, side, half, b.send[key])
            self.tr.exchange([(p, b.send[k]) for p, k, _, _ in sends], [(p, b.recv[k]) for p, k in recvs],
                             stream=self.stream)
            for peer, key in recvs:
                self.e.halo_unpack(key[0], d, key[1], half, b.recv[key])

    def new_dt(self):
        return self.tr.min(self.e.new_dt(), self.device)

    def kick(self, driver, event, de):
        """One turbulence-driving event over all ranks (drive.py): per-block
        sums all-gathered and combined in gid order, then the ghost exchange
        (the engine's apply refreshed only ghosts with local sources)."""
        scale = driver.kick(self.e, event, de, allgather=self.tr.allgather)
        self.exchange(half=0)
        return scale

    def vl2_step(self, dt):
        _, s1 = self.e.stage_compute(1, dt)
        self.e.stage_prefetch(2, dt)  # stage-2 interior tiles overlap the halo exchange
        self.exchange(half=1)
        dn, s2 = self.e.stage_compute(2, dt)
        self.exchange(half=0)
        return self.tr.min(dn, self.device), (s1.floor_count + s2.floor_count)


class LoopbackWorld:
    """Several rank engines in ONE process, stepped in lockstep; messages are
    handed over by device/host copies.  Nothing waits on another kernel.

    stream_ordered=True puts the engines in pmhd_gpu_set_async mode and orders
    the hand-over with CUDA events between the engines' streams, the way NCCL
    orders send/recv on the issuing stream (DistributedVL2 over NCCL): the
    host never synchronizes inside a stage."""

    def __init__(self, engines, plan, stream_ordered=False, p2p=False):
        self.engines, self.plan = engines, plan
        self.stream_ordered = stream_ordered
        self.p2p = p2p
        if p2p:  # one process: the other engines' slabs are plain device pointers
            bases = [e.slab()[0] for e in engines]
            for r, e in enumerate(engines):
                e.peer_attach(plan.owners, [None if q == r else b for q, b in enumerate(bases)])
        if stream_ordered:
            for e in engines:
                e.set_async(True)
            self.streams = [e.torch_stream() for e in engines]
            self.send, self.recv = {}, {}
            for d in range(plan.dim):
                for r, e in enumerate(engines):
                    sends, recvs = plan.messages(r, d)
                    for peer, key, gid, side in sends:
                        self.send[(d, peer, key)] = e.alloc_halo(e.halo_count(d, 1 - side))
                    for peer, key in recvs:
                        self.recv[(d, r, key)] = e.alloc_halo(e.halo_count(d, key[1]))

    def _exchange_streams(self, half):
        import torch
        n = len(self.engines)
        for d in range(self.plan.dim):
            for r, e in enumerate(self.engines):
                e.exchange_dir(d, half)
                sends, _ = self.plan.messages(r, d)
                for peer, key, gid, side in sends:
                    e.halo_pack(gid, d, side, half, self.send[(d, peer, key)])
            packed = [torch.cuda.Event() for _ in range(n)]
            for r in range(n):
                packed[r].record(self.streams[r])
            for r, e in enumerate(self.engines):
                _, recvs = self.plan.messages(r, d)
                for peer, key in recvs:
                    self.streams[r].wait_event(packed[peer])
                    dst = self.recv[(d, r, key)]
                    with torch.cuda.stream(self.streams[r]):
                        dst.copy_(self.send[(d, r, key)])
                    e.halo_unpack(key[0], d, key[1], half, dst)
            # send buffers are reused by the next pack: every stream waits for
            # every receiver's copies first
            copied = [torch.cuda.Event() for _ in range(n)]
            for r in range(n):
                copied[r].record(self.streams[r])
            for r in range(n):
                for q in range(n):
                    if q != r:
                        self.streams[r].wait_event(copied[q])

    def exchange(self, half):
        if self.p2p:  # direction-major: every engine's sweep d before any sweep d+1
            for d in range(self.plan.dim):
                for e in self.engines:
                    e.exchange_dir(d, half)
            return
        if self.stream_ordered:
            return self._exchange_streams(half)
        import torch
        for d in range(self.plan.dim):
            for e in self.engines:
                e.exchange_dir(d, half)
            staged = {}
            for r, e in enumerate(self.engines):
                sends, _ = self.plan.messages(r, d)
                for peer, key, gid, side in sends:
                    buf = e.alloc_halo(e.halo_count(d, 1 - side))
                    e.halo_pack(gid, d, side, half, buf)
                    staged[(peer, key)] = buf
            for r, e in enumerate(self.engines):
                _, recvs = self.plan.messages(r, d)
                for peer, key in recvs:
                    src = staged[(r, key)]
                    dst = e.alloc_halo(src.numel())
                    dst.copy_(src.to(dst.device))
                    e.halo_unpack(key[0], d, key[1], half, dst)

    def vl2_step(self, dt):
        for e in self.engines:
            e.stage_compute(1, dt)
            e.stage_prefetch(2, dt)
        self.exchange(half=1)
        dts = [e.stage_compute(2, dt)[0] for e in self.engines]
        self.exchange(half=0)
        if self.stream_ordered:  # the half=0 exchange must land before the host reads state
            for s in self.streams:
                s.synchronize()
        return min(dts)
