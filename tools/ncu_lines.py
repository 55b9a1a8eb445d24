"""Per-source-line instruction counts: join an ncu SASS page (executed counts) with
nvdisasm -g line info of the in-tree .so.  usage: ncu_lines.py REPORT KERNEL_INDEX MANGLED_NAME [top]"""
import csv, io, os, re, subprocess, sys, tempfile
from collections import Counter
rep, which, mangled = sys.argv[1], int(sys.argv[2]), sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
DUMP = os.environ.get("DUMP")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.environ.get("WT_LIB_PATH", os.path.join(ROOT, "paper_1407_8142_b200", "libwt_b200.so"))
td = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=td, capture_output=True)
cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(td, cub)], capture_output=True, text=True).stdout
# walk the function's section
lines = sass.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(f".text.{mangled}:"))
cur = ("?", 0)
off2line = {}
for l in lines[start + 1:]:
    if l.startswith("//-----") or l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        off2line[int(m.group(1), 16)] = cur
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
kern, curk, shdr = [], None, None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "Kernel Name":
        curk = [r[1], []]; kern.append(curk); continue
    if r and r[0] == "Address":
        shdr = {h: i for i, h in enumerate(r)}; continue
    if curk is not None and r:
        curk[1].append(r)
name, rs = kern[which]
base = int(rs[0][shdr["Address"]], 16)
cnt, smp = Counter(), Counter()
tot = 0
for r in rs:
    off = int(r[shdr["Address"]], 16) - base
    ex = int(r[shdr["Instructions Executed"]] or 0)
    key = off2line.get(off, ("?", 0))
    cnt[key] += ex; smp[key] += int(r[shdr["# Samples"]] or 0)
    tot += ex
print(name[:80], "total warp-inst", tot)
srcs = {}
for (f, ln), v in cnt.most_common(top):
    if f not in srcs:
        p = os.path.join(ROOT, "paper_1407_8142_b200", "csrc", f)
        srcs[f] = open(p).read().splitlines() if os.path.exists(p) else []
    text = srcs[f][ln - 1].strip()[:80] if 0 < ln <= len(srcs[f]) else ""
    print(f"{100*v/tot:5.1f}% {100*smp[(f,ln)]/max(1,sum(smp.values())):5.1f}%s  {f}:{ln:<4d} {text}")
if DUMP:  # per-line counts as JSON for phase aggregation
    import json
    json.dump({f"{f}:{ln}": [v, smp[(f, ln)]] for (f, ln), v in cnt.items()}, open(DUMP, "w"))
