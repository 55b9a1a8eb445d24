"""Batched query throughput:
access / rank_c / select_c on the config-4 tree and matrix and on the config-3
Huffman-shaped tree, 2^22 random queries per batch (valid positions, symbols
taken from S so that select hits), device time by CUDA events (median of 5),
plus the select-directory build time.  Writes JSON lines to stdout and to
gpurun_out/query_bench.jsonl."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1407_8142_b200 as wt

Q = 1 << 22


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def emit(r):
    print(json.dumps(r), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/query_bench.jsonl", "a") as f:
        f.write(json.dumps(r) + "\n")


rng = np.random.default_rng(0)
for idx in (4, 3):
    cfg = gen.CONFIGS[idx]
    S = gen.config_input(cfg)
    St = torch.from_numpy(S).cuda()
    pos = torch.from_numpy(rng.integers(0, cfg.n, Q)).cuda()
    sym = torch.from_numpy(S[rng.integers(0, cfg.n, Q)].astype(np.int64).astype(np.int32)).cuda()
    kk = torch.ones(Q, dtype=torch.int64, device="cuda")
    structs = [("tree", wt.build(St, cfg.sigma)), ("matrix", wt.wm_build(St, cfg.sigma))]
    if cfg.sigma <= 65536:
        structs.append(("huffman_tree", wt.hwt_build(St, cfg.sigma)))
    for name, t in structs:
        r = {"config": cfg.name, "structure": name, "queries": Q}
        r["access_ms"] = timed(lambda: t.access(pos))
        r["rank_ms"] = timed(lambda: t.rank(sym, pos))
        if hasattr(t, "select_index"):  # first (real) build of the select directory
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); t.select_index(); e1.record(); torch.cuda.synchronize()
            r["select_index_ms"] = e0.elapsed_time(e1)
            r["select_ms"] = timed(lambda: t.select(sym, kk))
        for k in ("access", "rank", "select"):
            if f"{k}_ms" in r:
                r[f"{k}_queries_per_s"] = Q / (r[f"{k}_ms"] * 1e-3)
        emit(r)
        t.free()
