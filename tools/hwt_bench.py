"""Device time of the Huffman-shaped wavelet tree build next
to the balanced tree and the matrix on the same inputs: configs 2-4 and a
Zipf sweep.  Median of 5 CUDA-event-timed builds after 2 warm-ups; the hwt
time includes its three host synchronisations.  Also reports the compressed
size (sum_c f_c len_c bits vs n*L) and the phase split of the hwt build."""
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


def row(name, S, sigma):
    St = torch.from_numpy(S).cuda()
    L = (sigma - 1).bit_length()
    t_wt = timed(lambda: wt.build(St, sigma))
    t_wm = timed(lambda: wt.wm_build(St, sigma))
    t_h = timed(lambda: wt.hwt_build(St, sigma))
    h = wt.hwt_build(St, sigma)
    r = {"input": name, "n": int(S.size), "sigma": sigma, "L": L, "hwt_levels": h.levels,
         "hwt_bits_per_symbol": h.total_bits / S.size, "wt_ms": t_wt, "wm_ms": t_wm, "hwt_ms": t_h,
         "hwt_coded_levels_per_s": h.total_bits / (t_h * 1e-3)}
    h.free()
    print(json.dumps(r), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/hwt_bench.jsonl", "a") as f:
        f.write(json.dumps(r) + "\n")


for idx in (2, 3, 4):
    cfg = gen.CONFIGS[idx]
    row(cfg.name, gen.config_input(cfg), cfg.sigma)
for s in (1.0, 1.5, 2.0):
    S = np.minimum(np.random.default_rng(7).zipf(1 + s, 1 << 26) - 1, 65535).astype(np.uint16)
    row(f"zipf{1 + s}_n2^26_sigma65536", S, 65536)
