"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into
per-kernel totals and shares; optionally restrict to the last N launches."""
import csv, json, sys
from collections import defaultdict
path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
t, n = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    v = float(r[vi]) * (1e-3 if r[ui] == "ns" else (1.0 if r[ui] == "us" else 1e3))
    t[name] += v
    n[name] += 1
tot = sum(t.values())
out = {k: {"launches": n[k], "total_us": round(v, 1), "share": round(v / tot, 4)} for k, v in
       sorted(t.items(), key=lambda x: -x[1])}
print(json.dumps(out, indent=1))
