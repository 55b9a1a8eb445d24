"""Summarise an ncu `--metrics gpu__time_duration.sum` launch list (CSV) per kernel."""
import csv, sys, collections, re

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if r]
hdr_i = next(i for i, r in enumerate(rows) if r[0] == "ID")
hdr = rows[hdr_i]
tot = collections.OrderedDict()
cnt = collections.Counter()
for r in rows[hdr_i + 1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").strip()
    ns = float(d["Metric Value"])
    tot[name] = tot.get(name, 0.0) + ns
    cnt[name] += 1
all_ns = sum(tot.values())
print(f"| kernel | launches | total ms | share |")
print(f"|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"| `{k}` | {cnt[k]} | {v/1e6:.3f} | {v/all_ns*100:.1f}% |")
print(f"| **all** | {sum(cnt.values())} | {all_ns/1e6:.3f} | 100% |")
