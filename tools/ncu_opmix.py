"""Instruction mix of one kernel launch in an ncu report (SASS source page):
warp-level instructions executed and stall samples per opcode.
usage: ncu_opmix.py <rep> <kernel regex> <launch skip>"""
import csv, subprocess, sys, collections
rep, kre, skip = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                      f"regex:{kre}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
r = csv.reader(lines[1:])
h = next(r)
ie, st = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
inst = collections.Counter(); stall = collections.Counter()
for row in r:
    if len(row) <= ie or not row[ie].isdigit():
        continue
    op = row[src].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1] if len(op) > 1 else o
    o = o.split(".")[0]
    inst[o] += int(row[ie] or 0); stall[o] += int(row[st] or 0)
ti, ts = sum(inst.values()), sum(stall.values())
print(f"total warp-inst {ti}  stall samples {ts}")
for o, n in inst.most_common(30):
    print(f"{o:10s} {n:12d} {100*n/ti:5.1f}%  stall {100*stall[o]/max(ts,1):5.1f}%")
