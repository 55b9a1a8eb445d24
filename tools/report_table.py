"""Combine profiles/r01_report/report_time.jsonl with the per-config ncu CSVs into the
SURVEY §8(d) per-config table (markdown)."""
import csv, json, sys
PEAK = 6545.6
rows = [json.loads(l) for l in open(sys.argv[1] + "/report_time.jsonl" if len(sys.argv) > 1 else "gpurun_out/report_time.jsonl")]
print("| cfg | n | σ | L | t (ms) | elements/s | symbol-levels/s | DRAM bytes moved (ncu) | DRAM GB/s over t | frac of 6545.6 | moved / B_min | B_min / t frac | lane-ops per element-level |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    c = r["config"]
    D = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    recs = [x for x in csv.reader(open(f"{D}/report_ncu_cfg{c}.csv")) if len(x) > 10]
    h = recs[0]
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = {"dram": 0.0, "inst": 0.0}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for x in recs[1:]:
        v = float(x[vi].replace(",", ""))
        if x[mi].startswith("dram__bytes"):
            tot["dram"] += v * scale.get(x[ui], 1)
        elif x[mi] == "sm__inst_executed.sum":
            tot["inst"] += v * (1e3 if x[ui] == "Kinst" else 1e6 if x[ui] == "Minst" else 1e9 if x[ui] == "Ginst" else 1)
    t = r["ms"] * 1e-3
    gbs = tot["dram"] / t / 1e9
    print(f"| {c} | {r['n']} | {r['sigma']} | {r['L']} | {r['ms']:.3f} | {r['elements_per_s']:.3g} | "
          f"{r['symbol_levels_per_s']:.3g} | {tot['dram']/1e9:.3f} GB | {gbs:.0f} | {gbs/PEAK:.3f} | "
          f"{tot['dram']/r['b_min_bytes']:.2f} | {r['b_min_frac_of_peak']:.3f} | "
          f"{tot['inst']*32/(r['n']*r['L']):.1f} |")
