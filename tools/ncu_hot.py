"""Hot SASS regions of one kernel in an ncu report: basic blocks by executed instructions."""
import csv, io, subprocess, sys
rep, which = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
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
name, rs = kern[which]
tot = sum(int(r[shdr["Instructions Executed"]] or 0) for r in rs)
# segment into runs of equal execution count (basic blocks approx.)
segs = []
for i, r in enumerate(rs):
    ex = int(r[shdr["Instructions Executed"]] or 0)
    if segs and segs[-1][2] == ex:
        segs[-1][1] = i
    else:
        segs.append([i, i, ex])
segs.sort(key=lambda s: -(s[1] - s[0] + 1) * s[2])
print(name[:80], "total", tot)
for a, b, ex in segs[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    n = b - a + 1
    print(f"--- rows {a}-{b} ({n} instr) x {ex} = {100*n*ex/tot:.1f}%  addr {rs[a][shdr['Address']]}")
    for r in rs[a:a + min(n, 6)]:
        print("      ", r[shdr["Source"]][:70])
