"""Build one small case (n, sigma) on the GPU and compare with the oracle (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, oracle
import paper_1407_8142_b200 as wt
n, sigma = int(sys.argv[1]), int(sys.argv[2])
dt = np.uint8 if sigma <= 256 else (np.uint16 if sigma <= 65536 else np.uint32)
S = gen.uniform_below(n, sigma, seed=1000 * n + sigma, dtype=dt)
try:
    t = wt.build(torch.from_numpy(S).cuda(), sigma)
except Exception as e:
    print("build failed", e); t = None
got = t.numpy() if t else None; want = oracle.build(S, sigma)
for k in (() if got is None else ("bits", "level_node_ptr", "node_key", "node_start", "rank_block", "rank_super")):
    ok = np.array_equal(got[k], want[k])
    print(k, "OK" if ok else f"MISMATCH {np.count_nonzero(got[k] != want[k]) if got[k].shape == want[k].shape else got[k].shape}")
if os.environ.get("WT_LIB_PATH", "").endswith("debug.so"):
    import ctypes
    lib = ctypes.CDLL(os.environ["WT_LIB_PATH"])
    a = (ctypes.c_uint32 * 4)()
    lib.wt_debug_code(a)
    print("debug code", list(a))
