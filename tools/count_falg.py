"""Freeze F_alg: CountingScalar tally of the CPU oracle for
one VL2 cycle of the M4 linear-wave config at n^3 (one block), per active
cell-update, with the split between the flux region (c2p + reconstruction +
Riemann: the GPU's k_flux_fused launches) and the rest (EMF + CT + update +
dt: k_update_fused).  Writes profiles/falg_counting.json.

usage: python tools/count_falg.py [n ...]   (default 64 128 256; 256 takes ~1 min)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (make_config: the bench workload)
from oracle import binding as O  # noqa: E402

out_path = os.path.join(ROOT, "profiles", "falg_counting.json")
res = json.load(open(out_path)) if os.path.exists(out_path) else {}
for n in [int(a) for a in sys.argv[1:]] or [64, 128, 256]:
    cfg = bench.make_config(n, 1)
    s = O.OracleSolver(cfg, counting=True)
    s.load_pgen()
    dt = s.new_dt()
    O.flops_reset()
    t0 = time.time()
    s.vl2_step(dt)
    f = O.flops()
    reg = O.region_flops()
    cells = cfg.active_cells
    regions = {name: float(v) / cells for name, v in zip(O.REGIONS, reg)}
    regions["dt"] = (float(f.sum()) - float(reg.sum())) / cells
    res[str(n)] = {"add": f[0], "mul": f[1], "div": f[2], "sqrt": f[3], "total": float(f.sum()),
                   "per_cell_update": float(f.sum()) / cells,
                   "flux_region_per_cell_update": float(reg[:3].sum()) / cells,
                   "update_region_per_cell_update": (float(f.sum()) - float(reg[:3].sum())) / cells,
                   "regions_per_cell_update": regions,
                   "seconds": time.time() - t0}
    print(n, res[str(n)], flush=True)
    del s
json.dump(res, open(out_path, "w"), indent=1)
# region table for the CLI's roofline / report commands (per cell-update, largest size)
big = res[str(max(int(k) for k in res))]
if "regions_per_cell_update" in big:
    with open(os.path.join(ROOT, "profiles", "falg_regions.csv"), "w") as fh:
        fh.write("region,flops_per_cell_update\n")
        for name, v in big["regions_per_cell_update"].items():
            fh.write(f"{name},{v!r}\n")
