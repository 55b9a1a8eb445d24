"""Summarise an ncu report: key metrics per kernel + opcode mix (reads the .ncu-rep here, no GPU)."""
import csv, io, subprocess, sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
KEYS = ["gpu__time_duration.sum", "sm__inst_executed.sum", "sm__warps_active.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__maximum_warps_per_active_cycle_pct", "smsp__warps_eligible.avg.per_cycle_active"]
STALLS = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print(d["Kernel Name"][:90], d.get("Grid Size", ""), d.get("Block Size", ""))
    for k in KEYS:
        if k in d:
            print(f"   {k:75s} {d[k]}")
    st = sorted(((float(d[k] or 0), k) for k in STALLS), reverse=True)[:8]
    print("   stalls/issue:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, k in st))

src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
kern, cur, shdr = [], None, None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "Kernel Name":
        cur = [r[1], []]; kern.append(cur); continue
    if r and r[0] == "Address":
        shdr = {h: i for i, h in enumerate(r)}; continue
    if cur is not None and r:
        cur[1].append(r)
for name, rs in kern:
    ins = sum(int(r[shdr["Instructions Executed"]] or 0) for r in rs)
    smp = sum(int(r[shdr["# Samples"]] or 0) for r in rs)
    c, s = Counter(), Counter()
    for r in rs:
        t = r[shdr["Source"]].split()
        if not t: continue
        op = t[1] if t[0].startswith("@") else t[0]
        op = op.split(".")[0]
        c[op] += int(r[shdr["Instructions Executed"]] or 0); s[op] += int(r[shdr["# Samples"]] or 0)
    print(name[:90], "warp-inst", ins, "samples", smp)
    print("   " + ", ".join(f"{op} {100*v/ins:.1f}%/{100*s[op]/max(1,smp):.1f}%" for op, v in c.most_common(18)))
