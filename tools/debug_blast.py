import sys, numpy as np
sys.path.insert(0, '.')
from paper_1905_04341_b200 import RunConfig
from paper_1905_04341_b200.solver import GpuSolver
from oracle.binding import OracleSolver
kw = dict(nx1=32, nx2=32, nx3=32, mb1=16, mb2=16, mb3=16, x1min=-0.5, x1max=0.5, x2min=-0.5, x2max=0.5,
          x3min=-0.5, x3max=0.5, pgen="blast", eos_mode="floor", blast_r=0.2)
cfg = RunConfig(**kw)
o = OracleSolver(cfg, workers=8); g = GpuSolver(cfg)
o.load_pgen(); g.load_pgen()
dt = o.new_dt()
ks, js, is_ = cfg.active_slices()
for c in range(12):
    dno, _ = o.vl2_step(dt); dng, _ = g.vl2_step(dt)
    worst = 0; where = None
    for gid in range(cfg.nblocks):
        a = o.get_block(gid).u[:, ks, js, is_]; b = g.get_block(gid).u[:, ks, js, is_]
        for q in range(8):
            s = max(np.max(np.abs(a[q])), 1e-300)
            d = np.abs(a[q] - b[q]) / np.maximum(np.abs(a[q]), s)
            if d.max() > worst:
                worst = d.max(); where = (gid, q, np.unravel_index(d.argmax(), d.shape))
    print(c, "dt rel", abs(dno - dng) / dno, "worst cell", worst, where, flush=True)
    dt = dno
