"""CPU reference timing of the BASELINE configs (M1-M5) on the host cores:
the oracle (test infrastructure) dispatched through the reference's own
par_for / ThreadPool (oracle/_ref) when built, on a bounded number of
cycles per config.  Prints one CSV row per config (BASELINE.md §4's CPU
column).  usage: python tools/cpu_configs.py [seconds per config]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1905_04341_b200 import RunConfig  # noqa: E402
from oracle.binding import OracleSolver  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 20.0
ref = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "liboracle_ref.so"))
workers = os.cpu_count() or 1
print("config,cells,cycles,seconds,cell_updates_per_s,cores,engine")
def mem_available():
    for ln in open("/proc/meminfo"):
        if ln.startswith("MemAvailable:"):
            return int(ln.split()[1]) * 1024
    return 0


# M5 (512^3, 134M cells, ~90 GB of oracle state) runs as one 128^3-block
# layer: the 512 x 512 x 128 slab, same per-cell work
OVERRIDES = {"turbulence_512": dict(nx3=128)}
for name in ("linear_wave_64", "orszag_tang_512", "blast_256", "linear_wave_256", "turbulence_512"):
    cfg = RunConfig(open(os.path.join(ROOT, "examples", name + ".in")).read(), **OVERRIDES.get(name, {}))
    if 700 * cfg.active_cells > 0.5 * mem_available():  # ~700 B of oracle state per cell
        print(f"{name},{cfg.active_cells},0,0,skipped (host memory),{workers},-", flush=True)
        continue
    o = OracleSolver(cfg, workers=workers, ref=ref)
    o.load_pgen()
    dt = o.new_dt()
    dt, _ = o.vl2_step(dt)  # warm-up (first touch)
    n, t0 = 0, time.perf_counter()
    while True:
        dt, _ = o.vl2_step(dt)
        n += 1
        el = time.perf_counter() - t0
        if el > budget or n >= 20:
            break
    m = cfg.desc.nx
    print(f"{name} ({m[0]}x{m[1]}x{m[2]}),{cfg.active_cells},{n},{el:.3f},{cfg.active_cells * n / el:.4e},{workers},"
          f"{'oracle/_ref (reference par_for/ThreadPool)' if ref else 'oracle'}", flush=True)
    del o
