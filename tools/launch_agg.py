"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel
(template instances kept apart), per bench step.
usage: launch_agg.py file.csv [steps]   (steps: divide the totals by this many builds)"""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.OrderedDict()
for r in rows:
    v = float(r[vi].replace(",", "")) * scale[r[ui]]
    name = r[ki].replace("void ", "").split("(")[0].replace("wtb::", "")
    name = name.replace("unsigned char", "u8").replace("unsigned short", "u16").replace("unsigned int", "u32")
    a = agg.setdefault(name, [0.0, 0])
    a[0] += v
    a[1] += 1
tot = sum(a[0] for a in agg.values())
print("total %.1f us per step (%d launches, %g steps)" % (tot / steps, len(rows), steps))
for k, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print("   %-48s %9.1f us  %5.1f %%  x%g" % (k, t / steps, 100 * t / tot, c / steps))
