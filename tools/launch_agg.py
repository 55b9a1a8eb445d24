"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel.
usage: launch_agg.py file.csv [second_half]"""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
if len(sys.argv) > 2:
    rows = rows[len(rows) // 2:]
agg = collections.OrderedDict()
for r in rows:
    v = float(r[vi].replace(",", ""))
    v = v / 1e3 if r[ui] == "nsecond" else (v * 1e3 if r[ui] == "msecond" else v)
    name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
    a = agg.setdefault(name, [0.0, 0])
    a[0] += v
    a[1] += 1
print("total %.1f us" % sum(a[0] for a in agg.values()))
for k, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print("   %-28s %10.1f us  x%d" % (k, t, c))
