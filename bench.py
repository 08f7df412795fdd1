#!/usr/bin/env python
"""bench.py -- fp64 VL2+PLM+HLLD+CT MHD throughput on B200 (cell-updates/s).

Workload (BASELINE.json config 4 at N=1): 3D linear fast
magnetosonic wave, 256^3 active cells in ONE MeshBlock per GPU, ng=2,
gamma=5/3, CFL 0.3, A=1e-6 along x1, HLLD + PLM(MC) + contact-upwind CT.
A "step" is one full VL2 cycle (stage 1 + stage 2 + exchanges + dt).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N>1) each rank owns one 256^3 block of a (256 N) x 256 x 256
periodic mesh (weak scaling); dt is all-reduced (min) over ranks every cycle.
Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B_ALG = 320.0          # compulsory HBM bytes per cell-update
F_ALG_FILE = os.path.join(ROOT, "profiles", "falg_counting.json")
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak.json")
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
# PMHD_BENCH_TRANSPORT=gloo-host: run the N>1 code path with gloo + host-staged
# halos (all ranks may share one GPU) to validate it; numbers are not
# measurements and the JSON says so.
GLOO_HOST = os.environ.get("PMHD_BENCH_TRANSPORT", "") == "gloo-host"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--size", type=int, default=256, help="cells per dimension per GPU")
    p.add_argument("--block", type=int, default=0,
                   help="MeshBlock edge (default = --size: one block per GPU; 128 with --size 256: the "
                        "8-blocks-per-GPU M4 variant)")
    p.add_argument("--riemann", default="hlld")
    p.add_argument("--workload", choices=["m4", "m5"], default="m4",
                   help="m4: linear wave, --size^3 cells per GPU (weak scaling, the default and the headline); "
                        "m5: decaying turbulence 512^3 in 128^3 MeshBlocks split over the ranks (strong scaling)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def rank_grid(ranks):
    """Rank grid (p1, p2, p3) of the M4 weak-scaling run:
    (1,1,1), (2,1,1), (2,2,1), (2,2,2) for 1 / 2 / 4 / 8 ranks -- each prime
    factor of the rank count goes to the axis with the fewest ranks so far."""
    from paper_1905_04341_b200.parallel import _factor
    p = [1, 1, 1]
    for f in sorted(_factor(ranks), reverse=True):
        a = min(range(3), key=lambda x: p[x])
        p[a] *= f
    return p


def make_config(n, ranks, riemann="hlld", nz=None, block=0):
    """The M4 linear fast wave: n^3 cells per rank on a (p1 n) x (p2 n) x
    (p3 n) periodic grid with dx = 1/n, in MeshBlocks of block^3 (default:
    one n^3 block per rank; nz: the CPU legs' bounded n x n x nz slab)."""
    from paper_1905_04341_b200 import RunConfig
    p = rank_grid(ranks)
    nz = n if nz is None else nz
    mb = block if block else n
    return RunConfig(nx1=n * p[0], nx2=n * p[1], nx3=nz * p[2], mb1=mb, mb2=mb, mb3=min(mb, nz), x1max=float(p[0]),
                     x2max=float(p[1]), x3max=p[2] * nz / n, wave_mode=6, wave_amp=1e-6, cfl=0.3,
                     riemann=riemann)


def make_m5_config(riemann="hlld", nz=None):
    """M5 (BASELINE config 5): 512^3 decaying turbulence in 128^3 MeshBlocks,
    examples/turbulence_512.in (nz: the CPU legs' bounded 512 x 512 x nz slab)."""
    from paper_1905_04341_b200 import RunConfig
    text = open(os.path.join(ROOT, "examples", "turbulence_512.in")).read()
    kw = dict(riemann=riemann)
    if nz is not None:
        kw.update(nx3=nz, mb3=nz, x3max=nz / 512.0)
    return RunConfig(text, **kw)


def falg():
    """(F_alg total, F_alg of the flux region, source) per cell-update."""
    try:
        d = json.load(open(F_ALG_FILE))["256"]
        return (float(d["per_cell_update"]), float(d["flux_region_per_cell_update"]),
                "oracle CountingScalar at 256^3, HLLD (profiles/falg_counting.json, tools/count_falg.py)")
    except Exception:
        return 2815.0, 2303.0, "estimate"


def ncu_traffic():
    """Per-launch DRAM bytes of the flux / update kernels at 256^3 from the
    newest committed ncu --set full capture (profiles/r0N/ncu_traffic_256.json)."""
    for rnd in ("r02", "r01"):
        try:
            return json.load(open(os.path.join(ROOT, "profiles", rnd, "ncu_traffic_256.json")))
        except Exception:
            continue
    return None


def fp64_peak():
    try:
        d = json.load(open(FP64_PEAK_FILE))
        return float(d["fp64_dfma_tflops"]), "measured (profiles/fp64_peak.json, tools/fp64_peak.cu)"
    except Exception:
        return 37.2, "nominal (148 SM x 64 DFMA x 2 x 1.965 GHz)"


def hbm_peak():
    try:
        return float(json.load(open(PEAKS_FILE))["hbm_gbs"]), "of measured"
    except Exception:
        return 6650.0, "of fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi can take a second to start on a fresh box: the timed
            # region begins only once it is producing samples
            t_end = time.perf_counter() + 15.0
            while not self.lines and time.perf_counter() < t_end and self.proc.poll() is None:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        self.t0 = time.perf_counter()
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append((time.perf_counter(), ln.strip()))

    def __exit__(self, *a):
        self.t1 = time.perf_counter()
        if self.proc:
            # one sample past the end of the region (the last one taken under load)
            t_end = self.t1 + 1.0
            while (not self.lines or self.lines[-1][0] <= self.t1) and time.perf_counter() < t_end \
                    and self.proc.poll() is None:
                time.sleep(0.01)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        # samples taken inside the timed region, plus the first one after it
        inside = [ln for t, ln in self.lines if self.t0 <= t <= self.t1]
        after = [ln for t, ln in self.lines if t > self.t1][:1]
        for ln in inside + after:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nme, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nme)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU legs
def cpu_oracle_cups(n, cycles_max, seconds, workers, nz=32, workload="m4"):
    """The oracle (test infrastructure) on a bounded sample of the workload:
    the 256 x 256 x nz periodic slab of the M4 linear wave (same per-cell
    work).  Dispatched through the reference's own par_for / ThreadPool
    (oracle/_ref) when that build is present."""
    from oracle.binding import OracleSolver
    ref = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "liboracle_ref.so"))
    cfg = make_config(n, 1, nz=nz) if workload == "m4" else make_m5_config(nz=nz)
    s = OracleSolver(cfg, workers=workers, ref=ref)
    s.load_pgen()
    dt = s.new_dt()
    dt, _ = s.vl2_step(dt)  # warm-up (page faults)
    times = []
    t_all = time.perf_counter()
    while len(times) < cycles_max:
        t0 = time.perf_counter()
        dt, _ = s.vl2_step(dt)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > seconds:
            break
    cells = cfg.active_cells
    per = [cells / t for t in times]
    return {"value": cells * len(times) / sum(times), "p80": sorted(per)[int(0.8 * (len(per) - 1))],
            "unit": "cell-updates/s", "cores": workers, "kind": "port",
            "sample": f"{len(times)} VL2 cycle(s) of the {cfg.desc.nx[0]}x{cfg.desc.nx[1]}x{nz} periodic slab of the "
                      f"{'M4 linear wave' if workload == 'm4' else 'M5 turbulence'} "
                      f"(same per-cell work as the full mesh), oracle/{'_ref (reference par_for/ThreadPool, SimdNested)' if ref else 'liboracle.so'}, "
                      f"{workers} worker threads"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    workers = os.cpu_count() or 1
    from oracle.binding import OracleSolver
    ref = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "liboracle_ref.so"))
    nz = 32
    if args.workload == "m4":
        cfg = make_config(args.size, 1, riemann=args.riemann, nz=nz)
    else:
        cfg = make_m5_config(riemann=args.riemann, nz=nz)
    s = OracleSolver(cfg, workers=workers, ref=ref)
    s.load_pgen()
    dt = s.new_dt()
    for _ in range(args.warmup):
        dt, _ = s.vl2_step(dt)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        dt, _ = s.vl2_step(dt)
        times.append(time.perf_counter() - t0)
    cells = cfg.active_cells
    tot = sum(times)
    value = cells * len(times) / tot
    wl = "M4 linear wave" if args.workload == "m4" else "M5 turbulence"
    sample = (f"each step = 1 VL2 cycle of the {cfg.desc.nx[0]}x{cfg.desc.nx[1]}x{nz} periodic slab of the {wl} "
              f"(bounded sample of the workload; identical per-cell work), CPU oracle "
              f"{'through the reference par_for/ThreadPool (oracle/_ref)' if ref else '(oracle/liboracle.so)'}")
    line = {"impl": "reference", "metric": "cell-updates/s (fp64 VL2+PLM+HLLD+CT MHD)", "value": value,
            "unit": "cell-updates/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
            "scaling": "weak" if args.workload == "m4" else "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic ({'linear-wave' if args.workload == 'm4' else 'turbulence'} problem generator)",
            "config": {"workload": (f"M4 linear fast wave {args.size}^3 per GPU (sampled as {args.size}x{args.size}x{nz})"
                                    if args.workload == "m4" else
                                    f"M5 decaying turbulence 512^3, 128^3 MeshBlocks (sampled as 512x512x{nz})"),
                       "riemann": args.riemann, "cells_per_step": cells},
            "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": workers, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU leg
def run_ours(args):
    import numpy as np
    import torch
    ws, rank, local = dist_env()
    dist = None
    if ws > 1:
        import torch.distributed as dist
        if GLOO_HOST:  # validation of the N>1 flow on one GPU (never a measurement)
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if GLOO_HOST and torch.cuda.device_count() <= local:
        local = 0
    torch.cuda.set_device(local)
    xdev = "cpu" if GLOO_HOST else "cuda"
    from paper_1905_04341_b200.solver import GpuSolver
    from paper_1905_04341_b200 import native as N

    n = args.size
    # (p1 n) x (p2 n) x (p3 n) periodic mesh, n^3 cells per rank (one block,
    # or --block edge blocks)
    if args.workload == "m4":
        cfg = make_config(n, ws, riemann=args.riemann, block=args.block)
        cells_rank = n ** 3
    else:  # M5: one fixed 512^3 mesh, its 64 blocks split over the ranks
        cfg = make_m5_config(riemann=args.riemann)
        cells_rank = cfg.active_cells // ws
    from paper_1905_04341_b200.parallel import plan_for, DistributedVL2, TorchDistTransport
    plan = plan_for(cfg, ws)
    my_gids = plan.local_gids(rank)
    g = GpuSolver(cfg, device=local, gids=my_gids)
    stream = torch.cuda.ExternalStream(g.stream_handle, device=torch.device("cuda", local))
    hosts = {gid: cfg.pgen_block(gid) for gid in my_gids}
    for gid, hb in hosts.items():
        g.set_block(gid, hb)
    drv = None
    if dist is not None:
        drv = DistributedVL2(g, plan, rank, TorchDistTransport(dist, host_staging=GLOO_HOST),
                             device=f"cuda:{local}")
        drv.exchange(half=0)
    else:
        g.exchange()
    dt = g.new_dt()

    def allreduce_min(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=xdev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return float(t.item())

    def barrier():
        if dist is not None:
            dist.barrier()

    def step(d):
        if drv is None:
            return g.vl2_step(d)[0]
        return drv.vl2_step(d)[0]

    dt = allreduce_min(dt)
    clk = ClockSampler(local).__enter__()  # started before the warm-up: no idle gap before the region
    for _ in range(args.warmup):
        dt = step(dt)
    # ---- timed region (inputs resident in HBM, 1.5 GB state >> 126 MB L2) ----
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    g.region_times(reset=True)
    barrier()
    torch.cuda.synchronize()
    clk.t0 = time.perf_counter()
    evs[0].record(stream)
    for k in range(args.steps):
        dt = step(dt)
        if k + 1 < args.steps:
            evs[k + 1].record(stream)
    # the last step may leave its x2 / x3 ghost exchanges on an internal
    # stream (pmhd_gpu_stream contract): close the region after all device work
    torch.cuda.synchronize()
    evs[-1].record(stream)
    torch.cuda.synchronize()
    clk.__exit__(None, None, None)
    barrier()
    launches = g.region_times()["kernel_launches"]
    per_ms = [evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)]
    tot_ms = evs[0].elapsed_time(evs[-1])
    if dist is not None:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=xdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    value = ws * cells_rank * args.steps / (tot_ms * 1e-3)
    per_cups = sorted(cells_rank * ws / (m * 1e-3) for m in per_ms)
    p80 = per_cups[int(0.8 * (len(per_cups) - 1))]

    # ---- profiled passes for the roofline ----
    # (a) kernel durations: CUDA events on the ABI stream around the product
    # kernels (profiling mode 2: no phase instrumentation), so the timed
    # kernels are the ones the timed region ran
    nprof = max(2, min(args.steps, 4))
    g.set_profiling(2)
    g.region_times(reset=True)
    for _ in range(nprof):
        dt = step(dt)
    rte = g.region_times(reset=True)
    # (b) region shares: the instrumented instantiations (clock64 phase shares)
    g.set_profiling(1)
    for _ in range(nprof):
        dt = step(dt)
    rt = g.region_times(reset=True)
    g.set_profiling(0)
    kern_ms = (rte["c2p_ms"] + rte["reconstruct_ms"] + rte["riemann_ms"] + rte["ct_emf_ms"] +
               rte["integrate_ms"] + rte["boundary_ms"]) / nprof
    prof_ms = (rt["c2p_ms"] + rt["reconstruct_ms"] + rt["riemann_ms"] + rt["ct_emf_ms"] +
               rt["integrate_ms"] + rt["boundary_ms"]) / nprof
    F_alg, F_flux, F_src = falg()
    fp64_pk, fp64_src = fp64_peak()
    hbm_pk, hbm_src = hbm_peak()
    cycle_ms_kernels = kern_ms
    ach_gbs = B_ALG * cells_rank / (cycle_ms_kernels * 1e-3) / 1e9
    ach_tf = F_alg * cells_rank / (cycle_ms_kernels * 1e-3) / 1e12
    shares = {k: rt[k] / max(1e-9, prof_ms * nprof) for k in
              ("c2p_ms", "reconstruct_ms", "riemann_ms", "ct_emf_ms", "integrate_ms", "boundary_ms")}
    # Dominant kernel: the fused flux kernel (c2p + PLM + Riemann), 2*dim
    # launches per cycle, timed with CUDA events on the ABI stream (region
    # "riemann").  It is FP64-pipe bound (no dense contraction, < 30 % of HBM
    # bandwidth in ncu), so its roofline is the measured DFMA peak.
    dim = cfg.dim
    n_flux = 2 * dim
    # average launch duration of the product flux kernel (events pass: the
    # flux group is all in riemann_ms; the split debug variant adds c2p)
    flux_ms = (rte["c2p_ms"] + rte["reconstruct_ms"] + rte["riemann_ms"]) / nprof / n_flux
    flux_flops = F_flux * cells_rank / n_flux              # algorithmic flops per launch
    flux_tf = flux_flops / (flux_ms * 1e-3) / 1e12
    tr = (ncu_traffic() if args.workload == "m4" and args.size == 256 and dim == 3 and args.block in (0, 256)
          else None)
    upd_ms = (rte["ct_emf_ms"] + rte["integrate_ms"]) / nprof / 2  # update kernel(s) per stage (events pass)
    # 3D meshes that fill the GPU run the stage's update as two kernels
    # (PMHD_UPDATE unset or "emf"); "ldg" / smaller meshes: the fused kernel
    upd_env = os.environ.get("PMHD_UPDATE", "")
    upd_name = ("k_edge_emf + k_cell_update (per stage)" if upd_env in ("", "emf") and cfg.desc.nx[2] > 1
                else {"ws": "k_update_ws", "tma": "k_update_tma"}.get(upd_env, "k_update_fused"))
    roofline = {
        "bound": "fp64", "achieved": flux_tf, "peak": fp64_pk, "unit": "TFLOP/s",
        "frac": flux_tf / fp64_pk,
        "traffic": tr["flux_bytes_per_launch"] if tr else None,
        "kernel": f"flux kernels (stage 1: k_flux_fused tiles; stage 2: k_flux_x1march, k_flux_march on meshes that fill the GPU; dominant: {flux_ms * n_flux / kern_ms:.0%} of the cycle; {n_flux} launches/cycle, "
                  f"avg {flux_ms:.3f} ms; F_alg(flux region) = {F_flux:.1f} flop/cell-update / {n_flux} launches)",
        "peak_source": fp64_src,
        "note": "FP64 CUDA-core bound, neither HBM nor tensor cores: bound='fp64' against the measured DFMA peak; "
                "its load / store skeleton also moves ~2.4 GB per launch (hbm_view), DESIGN.md section 4a",
        # the same kernel against the HBM ceiling: ncu DRAM bytes per launch
        # over the event-timed launch duration
        "hbm_view": ({"achieved": tr["flux_bytes_per_launch"] / (flux_ms * 1e-3) / 1e9, "peak": hbm_pk,
                      "unit": "GB/s", "frac": tr["flux_bytes_per_launch"] / (flux_ms * 1e-3) / 1e9 / hbm_pk,
                      "peak_source": hbm_src} if tr else None),
        "hbm_whole_cycle": {"achieved": ach_gbs, "peak": hbm_pk, "unit": "GB/s", "frac": ach_gbs / hbm_pk,
                            "B_alg_per_cell_update": B_ALG, "peak_source": hbm_src,
                            "ncu_dram_bytes_per_cell_update": tr["dram_bytes_per_cell_update"] if tr else None},
        "fp64_whole_cycle": {"achieved": ach_tf, "peak": fp64_pk, "unit": "TFLOP/s", "frac": ach_tf / fp64_pk,
                             "F_alg_per_cell_update": F_alg, "F_alg_source": F_src},
        "update_kernel": {"name": upd_name, "avg_ms": upd_ms,
                          "dram_bytes_per_launch": tr["update_bytes_per_launch"] if tr else None,
                          "dram_gbs": (tr["update_bytes_per_launch"] / (upd_ms * 1e-3) / 1e9) if tr else None},
        "binding_ceiling": "fp64" if F_alg / fp64_pk > B_ALG / (hbm_pk / 1e3) else "hbm",
        # paper Eq. 2 against the binding ceiling (SURVEY.md §8d judged figure)
        "roofline_achieved_eq2": (cells_rank / (cycle_ms_kernels * 1e-3)) /
        min(hbm_pk * 1e9 / B_ALG, fp64_pk * 1e12 / F_alg),
        "region_share": shares,
        "dominant_region": max(shares, key=shares.get),
        "region_split": "fused kernels: event time per kernel split by in-kernel clock64 phase shares "
                        "(instrumented pass); kernel durations from a separate events-only pass over the "
                        "product kernels",
    }

    # ---- e2e through the public API with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        cudart = torch.cuda.cudart()
        outb = {gid: cfg.new_block() for gid in my_gids}
        arrs = [a for hb in hosts.values() for a in (hb.u, hb.b1f, hb.b2f, hb.b3f)]
        outs = [a for ob in outb.values() for a in (ob.u, ob.b1f, ob.b2f, ob.b3f)]
        for a in arrs + outs:
            cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
        h2d = sum(hb.u[:5].nbytes + hb.b1f.nbytes + hb.b2f.nbytes + hb.b3f.nbytes for hb in hosts.values())
        # the download returns all 8 cell variables (Bcc re-derived on the device) + faces
        d2h = sum(a.nbytes for a in outs)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for gid, hb in hosts.items():
            g.set_block(gid, hb)
        if drv is None:
            g.exchange()
        else:
            drv.exchange(half=0)
        d = allreduce_min(g.new_dt())
        for _ in range(args.steps):
            d = step(d)
        for gid, ob in outb.items():
            g.get_block(gid, out=ob)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([ms], dtype=torch.float64, device=xdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        for a in arrs + outs:
            cudart.cudaHostUnregister(a.ctypes.data)
        e2e = {"value": ws * cells_rank * args.steps / (ms * 1e-3), "unit": "cell-updates/s",
               "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
               "how": "pmhd_gpu_upload_block (pinned host) + exchange + new_dt + K x pmhd_gpu_vl2_step + "
                      "pmhd_gpu_download_block, one CUDA-event region on the ABI stream; the whole "
                      "block state crosses PCIe once each way per K steps"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_cups(n, 5, args.cpu_seconds, os.cpu_count() or 1, workload=args.workload)

    # 8 doubles of state per cell incl. ghosts
    state_bytes = 64 * cells_rank * ((cfg.desc.mb[0] + 2 * cfg.desc.ng) / cfg.desc.mb[0]) ** 3
    if rank == 0:
        line = {
            "metric": "cell-updates/s (fp64 VL2+PLM+HLLD+CT MHD)", "value": value,
            "unit": "cell-updates/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.workload == "m4" else "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic ({'linear-wave' if args.workload == 'm4' else 'turbulence'} problem generator)",
            "config": {"workload": (f"M4 3D linear fast wave, {n}^3 active cells per GPU in "
                                    f"{len(my_gids)} MeshBlock(s) of {cfg.desc.mb[0]}^3, "
                                    f"HLLD+PLM(MC)+CT, CFL 0.3, A=1e-6" if args.workload == "m4" else
                                    f"M5 decaying turbulence 512^3 in 128^3 MeshBlocks, {len(my_gids)} per GPU "
                                    f"(strong scaling), HLLD+PLM(MC)+CT"),
                       "global_cells": ([n * q for q in rank_grid(ws)] if args.workload == "m4" else
                                        list(cfg.desc.nx)),
                       "parallelism": (f"{ws} rank(s) as a {'x'.join(map(str, rank_grid(ws)))} grid of {n}^3 "
                                       f"bricks, one per rank" if args.workload == "m4" else
                                       f"{ws} rank(s), {len(my_gids)} of the 64 blocks each (compact bricks)"),
                       "l2": (f"inputs larger than L2 ({state_bytes / 1e9:.2f} GB state per GPU "
                              f"vs 126 MB L2)" if state_bytes > 126e6 else
                              "state smaller than L2 (small validation size)"),
                       "statistic": "value = mean over K cycles; p80 in extra.p80_cups",
                       "variant": g.build_info},
            "p80_cups": p80,
            "roofline": roofline, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "cpu_baseline": cpu,
        }
        if GLOO_HOST:
            line["note"] = "PMHD_BENCH_TRANSPORT=gloo-host validation run: NOT a measurement"
        print(json.dumps(line), flush=True)
    g.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
