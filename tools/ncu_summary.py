"""Summarise an ncu report (raw page) into one line per kernel launch."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(out.splitlines())
h = next(r); units = next(r)
want = {
  "dur_us": "gpu__time_duration.sum", "dram_rd_MB": "dram__bytes_read.sum", "dram_wr_MB": "dram__bytes_write.sum",
  "regs": "launch__registers_per_thread", "occ_ach": "sm__warps_active.avg.pct_of_peak_sustained_active",
  "fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
  "ipc": "sm__inst_executed.avg.per_cycle_active", "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
  "smem_B": "launch__shared_mem_per_block_static",
  "dfma": "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
  "dmul": "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
  "dadd": "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
  "inst": "smsp__inst_executed.sum",
}
stalls = [k for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
for row in r:
    d = dict(zip(h, row))
    name = d.get("Kernel Name", "")[:40]
    vals = []
    for k, m in want.items():
        v = d.get(m, "")
        u = units[h.index(m)] if m in h else ""
        if v and u == "byte" and k.endswith("MB"):
            v = f"{float(v)/1e6:.1f}"
        elif v and u == "Kbyte" and k.endswith("MB"):
            v = f"{float(v)/1e3:.2f}"
        elif v and u == "Mbyte" and k.endswith("MB"):
            v = f"{float(v):.1f}"
        elif v and u == "Gbyte" and k.endswith("MB"):
            v = f"{float(v)*1e3:.1f}"
        elif v and u == "msecond" and k == "dur_us":
            v = f"{float(v)*1e3:.1f}"
        vals.append(f"{k}={v}")
    top = sorted(((float(d[s] or 0), s.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")) for s in stalls), reverse=True)[:4]
    print(d.get("ID"), name, " ".join(vals), "stalls:", ", ".join(f"{n}={v:.2f}" for v, n in top))
