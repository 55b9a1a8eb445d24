"""Summarise gpurun_out/atomics_cfg*.csv (tools/ncu_atomics.sh): per config, the
L2 atom/red requests and DRAM bytes of the second of the two builds (the first
is a warm-up), per kernel and in total."""
import csv, glob, json, re, sys
from collections import defaultdict
out = {}
for path in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/atomics_cfg*.csv")):
    cfg = re.search(r"cfg(\d+)", path).group(1)
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = defaultdict(lambda: defaultdict(float))
    launches = [r for r in rows[1:] if r[ix["Metric Name"]]]
    ids = sorted({int(r[ix["ID"]]) for r in launches})
    half = ids[len(ids) // 2] if ids else 0  # second build = second half of the launches
    for r in launches:
        if int(r[ix["ID"]]) < half:
            continue
        k = r[ix["Kernel Name"]].split("(")[0].split("<")[0].replace("void ", "").replace("wtb::", "")
        v = float(r[ix["Metric Value"]].replace(",", "") or 0)
        unit = r[ix["Metric Unit"]]
        if unit == "Gbyte": v *= 1e9
        elif unit == "Mbyte": v *= 1e6
        elif unit == "Kbyte": v *= 1e3
        elif unit == "msecond": v *= 1e-3
        elif unit == "usecond": v *= 1e-6
        per[k][r[ix["Metric Name"]]] += v
    tot = defaultdict(float)
    for k, d in per.items():
        for m, v in d.items():
            tot[m] += v
    out[f"config{cfg}"] = {"total": dict(tot), "kernels": {k: dict(d) for k, d in per.items()}}
print(json.dumps(out, indent=1))
