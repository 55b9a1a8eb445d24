"""Aggregate an ncu SASS page per phase of k_wgroup (line ranges between the
'// ----' markers of csrc/wt_wgroup.cuh and per helper function).
usage: ncu_phases.py REPORT KERNEL_INDEX MANGLED CHUNK_LEVELS"""
import json, os, re, subprocess, sys
rep, idx, mangled, cl = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, idx, mangled, "1"],
               env={**os.environ, "DUMP": "/tmp/_lines.json"}, capture_output=True)
d = json.load(open("/tmp/_lines.json"))
src = open(os.path.join(ROOT, "paper_1407_8142_b200", "csrc", "wt_wgroup.cuh")).read().splitlines()
marks = []  # (line, name)
for i, l in enumerate(src, 1):
    m = re.match(r"\s*// ---- (.*?) ----", l)
    if m: marks.append((i, m.group(1)[:40]))
    m = re.match(r"__device__ __forceinline__ \S+ (\w+)\(", l)
    if m: marks.append((i, "fn " + m.group(1)))
    m = re.match(r"__global__", l)
    if m: marks.append((i, "kernel"))
marks.sort()
def phase(ln):
    name = "?"
    for m, nm in marks:
        if m <= ln: name = nm
    return name
tot = sum(v[0] for v in d.values()); ts = sum(v[1] for v in d.values())
ph = {}
for k, (v, s) in d.items():
    f, ln = k.rsplit(":", 1)
    p = phase(int(ln)) if f == "wt_wgroup.cuh" else f
    a = ph.setdefault(p, [0, 0]); a[0] += v; a[1] += s
print(f"total {tot} warp-inst = {tot / cl:.2f} per chunk-level")
for p, (v, s) in sorted(ph.items(), key=lambda x: -x[1][0]):
    print(f"   {p:42s} {100 * v / tot:5.1f}% inst {100 * s / max(1, ts):5.1f}% samples {v / cl:6.2f}/chunk-level")
