"""Instruction / sample shares of the k_wgroup phases (source-line ranges found by
the section markers of csrc/wt_wgroup.cuh), from an ncu --set full report.
usage: ncu_wg_phases.py REPORT KERNEL_INDEX MANGLED_NAME"""
import os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = open(os.path.join(ROOT, "paper_1407_8142_b200", "csrc", "wt_wgroup.cuh")).read().splitlines()
def line_of(pat):
    return next(i + 1 for i, l in enumerate(src) if pat in l)
marks = [("helpers+split", line_of("__device__ __forceinline__ uint4 lds128")),
         ("count pass", line_of("// ones of bit k over superchunks")),
         ("rank/run helpers", line_of("// ones of the level before sub-tile position")),
         ("tma/load helpers", line_of("// ---- TMA bulk copy")),
         ("chain setup", line_of("// ---- chain setup")),
         ("load", line_of("// ---- 1. records")),
         ("levels (split calls, barriers)", line_of("// ---- 2. tau levels")),
         ("classes", line_of("// ---- 3. classes")),
         ("runs + fused A7", line_of("// ---- 4. runs")),
         ("keys out", line_of("// ---- 5. narrowed keys")),
         ("chain-end flush", line_of("// ---- chain end")),
         ("end", len(src) + 1)]
out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), sys.argv[1], sys.argv[2], sys.argv[3], "100000"],
                     capture_output=True, text=True).stdout
agg = {}
for l in out.splitlines():
    m = re.match(r"\s*([\d.]+)%\s+([\d.]+)%s\s+(\S+):(\d+)", l)
    if not m:
        continue
    f, ln, p, s = m.group(3), int(m.group(4)), float(m.group(1)), float(m.group(2))
    if f != "wt_wgroup.cuh":
        k = "intrinsics (split: dp2a, popc, ballots)"
    else:
        k = next(marks[i][0] for i in range(len(marks) - 1) if marks[i][1] <= ln < marks[i + 1][1]) if ln >= marks[0][1] else "other"
    a = agg.setdefault(k, [0.0, 0.0]); a[0] += p; a[1] += s
print(out.splitlines()[0] if out else "no output")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"  {k:42s} instructions {v[0]:5.1f} %   stall samples {v[1]:5.1f} %")
