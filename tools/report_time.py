"""Per-config build report (SURVEY §8(d) "Report, per config"): device time of
wt_build (median of 5 after 2 warm-ups, CUDA events, a 512 MB write before
each timed build so that no input or output is L2-resident), elements/s,
symbol-levels/s, B_min / t.  JSON lines to stdout and gpurun_out/report_time.jsonl.
DRAM bytes and instructions come from the ncu pass in tools/gpu_report.sh."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_1407_8142_b200 as wt

PEAK = 6545.6  # GB/s, MEASURED_PEAKS.json copy bandwidth


def bmin(n, w, L):
    bpl = (n + 511) // 512
    return n * w + L * bpl * 8 * 8 + L * (2 * bpl + 8 * ((n + 65535) // 65536 + 1))


flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2: evicted before each timed build
for ci in [int(x) for x in sys.argv[1:]] or [1, 2, 3, 4, 5]:
    cfg = gen.CONFIGS[ci]
    S = torch.from_numpy(gen.config_input(cfg)).cuda()
    for _ in range(2):
        wt.build(S, cfg.sigma).free()
    ts, nodes = [], 0
    for i in range(5):
        flush.fill_(i)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); t = wt.build(S, cfg.sigma); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1)); nodes = t.total_nodes
        t.free()
    ms = statistics.median(ts)
    b = bmin(cfg.n, cfg.elem_bytes, cfg.levels) + 8 * nodes
    r = {"config": cfg.idx, "name": cfg.name, "n": cfg.n, "sigma": cfg.sigma, "L": cfg.levels, "ms": ms,
         "elements_per_s": cfg.n / (ms * 1e-3), "symbol_levels_per_s": cfg.n * cfg.levels / (ms * 1e-3),
         "b_min_bytes": b, "b_min_GBps": b / (ms * 1e-3) / 1e9, "b_min_frac_of_peak": b / (ms * 1e-3) / 1e9 / PEAK,
         "total_nodes": nodes}
    print(json.dumps(r), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/report_time.jsonl", "a") as f:
        f.write(json.dumps(r) + "\n")
    del S
