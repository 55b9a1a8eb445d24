"""Randomised parity of the Huffman-shaped tree on skewed inputs (staged
builds, deep codes) against the oracle.  usage: fuzz_hwt.py SECONDS [seed]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_1407_8142_b200 as wt

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
t_end = time.time() + budget
cases = fails = staged = 0
KEYS = ("code", "code_len", "bits", "level_len", "level_node_ptr", "node_key", "node_start", "rank_block", "rank_super")
while time.time() < t_end:
    n = int(np.exp(rng.uniform(np.log(100), np.log(5_000_000))))
    sigma = int(rng.choice([256, 1000, 4096, 20000, 65536]))
    a = rng.uniform(1.05, 3.5)
    S = np.minimum(rng.zipf(a, n) - 1, sigma - 1).astype(np.int64)
    S = ((S * int(rng.integers(1, 1 << 16))) % sigma).astype(np.uint16 if sigma > 256 else np.uint8)
    if rng.random() < 0.3:
        S = S.astype(np.uint32)
    cases += 1
    try:
        t = wt.hwt_build(torch.from_numpy(S).cuda(), sigma)
        staged += t.stages > 1
        got, want = t.numpy(), oracle.hwt_build(S, sigma)
        for k in KEYS:
            if got[k].shape != want[k].shape or not np.array_equal(got[k], want[k]):
                print("FAIL", k, n, sigma, a, flush=True)
                fails += 1
                break
        t.free()
    except wt.WtError as e:
        if e.code != -5:
            print("ERROR", n, sigma, a, e, flush=True)
            fails += 1
print(f"fuzz_hwt: {cases} cases ({staged} staged), {fails} failures", flush=True)
