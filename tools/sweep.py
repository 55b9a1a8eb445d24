"""Scaling sweep of the GPU build (Fig. "scale"):
build time vs sigma for random sequences of length 10^8, and vs n for sigma = 2^8.
The paper's curves are CPU times (40 cores); here: device time of one wt_build
(median of 5 after 2 warm-ups, CUDA events) and of one wm_build.  Writes a JSON
list to stdout."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1407_8142_b200 as wt


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn().free()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(); obj = fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        obj.free()
    return statistics.median(ts)


rows = []
N = 10 ** 8
for k in [1, 2, 4, 6, 8, 10, 12, 14, 16, 18, 20, 24, 28, 32]:
    sigma = 1 << k
    dt = np.uint8 if k <= 8 else (np.uint16 if k <= 16 else np.uint32)
    S = torch.from_numpy(gen.uniform_bits(N, k, seed=100 + k, dtype=dt)).cuda()
    t1 = timed(lambda: wt.build(S, sigma))
    t2 = timed(lambda: wt.wm_build(S, sigma))
    rows.append({"sweep": "sigma", "n": N, "sigma": sigma, "levels": k, "wt_ms": t1, "wm_ms": t2,
                 "wt_sym_levels_per_s": N * k / (t1 * 1e-3), "wm_sym_levels_per_s": N * k / (t2 * 1e-3)})
    print(json.dumps(rows[-1]), flush=True)
    del S
for e in ([] if os.environ.get("SWEEP_ONLY") == "sigma" else [20, 22, 24, 26, 27, 28, 29, 30]):
    n = 1 << e
    S = torch.from_numpy(gen.uniform_bits(n, 8, seed=200 + e, dtype=np.uint8)).cuda()
    t1 = timed(lambda: wt.build(S, 256))
    t2 = timed(lambda: wt.wm_build(S, 256))
    rows.append({"sweep": "n", "n": n, "sigma": 256, "levels": 8, "wt_ms": t1, "wm_ms": t2,
                 "wt_sym_levels_per_s": n * 8 / (t1 * 1e-3), "wm_sym_levels_per_s": n * 8 / (t2 * 1e-3)})
    print(json.dumps(rows[-1]), flush=True)
    del S
