"""Per-CUDA-source-line instructions executed and stall samples of one kernel
launch in an ncu report (needs -lineinfo + --import-source on).
usage: ncu_lines.py <rep> <kernel regex> <launch skip> [top]"""
import csv, subprocess, sys
rep, kre, skip = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kre}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows, fname = [], ""
for row in csv.reader(out.splitlines()):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name", "Line No") or not row[0]:
        continue
    try:
        rows.append((int(row[7] or 0), int(row[4] or 0), f"{fname}:{row[0]}", row[1].strip()[:90]))
    except (ValueError, IndexError):
        pass
ti = sum(r[0] for r in rows); ts = sum(r[1] for r in rows)
print(f"total warp-inst {ti}  stall samples {ts}")
for n, s, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*n/ti:5.1f}% inst {100*s/max(ts,1):5.1f}% stall  {loc:22s} {src}")
