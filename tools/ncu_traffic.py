"""DRAM traffic per launch of the flux / update kernels from an ncu --set full
report of one VL2 cycle (tools/gpu_full.sh), written to
profiles/r01/ncu_traffic_256.json for bench.py's roofline "traffic" field.
usage: ncu_traffic.py <report.ncu-rep> <active cells> [out.json]"""
import csv, json, subprocess, sys
rep, cells = sys.argv[1], float(sys.argv[2])
dst = sys.argv[3] if len(sys.argv) > 3 else "profiles/r01/ncu_traffic_256.json"
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(out.splitlines())
h = next(r); units = next(r)
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
def val(d, m):
    return float(d[m]) * scale[units[h.index(m)]]
flux, upd, dur, nst = [], [], {}, 0
for row in r:
    d = dict(zip(h, row))
    b = val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum")
    name = d["Kernel Name"]
    is_upd = any(k in name for k in ("k_update_fused", "k_edge_emf", "k_cell_update"))
    (flux if ("k_flux_fused" in name or "k_flux_march" in name or "k_flux_x1march" in name) else upd if is_upd else []).append(b)
    # one stage's update: k_update_fused, or the k_edge_emf + k_cell_update pair
    nst = nst + 1 if ("k_update_fused" in name or "k_cell_update" in name) else nst
res = {"report": rep, "active_cells": cells, "flux_launches": len(flux), "update_launches": len(upd),
       "flux_bytes_per_launch": sum(flux) / max(1, len(flux)),
       "update_bytes_per_launch": sum(upd) / max(1, nst),
       "update_bytes_note": "per stage: k_update_fused, or k_edge_emf + k_cell_update",
       "dram_bytes_per_cell_update": (sum(flux) + sum(upd)) / cells,
       "note": "dram__bytes_read.sum + dram__bytes_write.sum, ncu --set full --clock-control none, one VL2 cycle"}
json.dump(res, open(dst, "w"), indent=1)
print(json.dumps(res, indent=1))
