"""Graph-replayed vs host-loop pmhd_gpu_run at the bench size: same bits,
and the wall time of each (python tools/graph_check.py [n])."""
import os, sys, time, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1905_04341_b200.solver import GpuSolver
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = bench.make_config(n, 1)
res = {}
for g in ("1", "0"):
    os.environ["PMHD_GRAPH"] = g
    s = GpuSolver(cfg)
    s.load_pgen()
    dt = s.new_dt()
    t0 = time.time()
    t, nc, dtn, fl = s.run(ncycles=6, dt=dt)
    el = time.time() - t0
    b = s.get_block(0)
    res[g] = (t, nc, dtn, b.u.copy())
    print(g, t, nc, dtn, el, flush=True)
    del s
print("bitwise equal:", np.array_equal(res["1"][3], res["0"][3]), res["1"][:3] == res["0"][:3])
