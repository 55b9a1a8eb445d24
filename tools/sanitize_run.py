"""Small builds of every path, for compute-sanitizer (memcheck / racecheck /
initcheck, one tool per run): config 1, 2^20-symbol prefixes of configs 3 and 4
(chain-mode group passes with TMA-staged tiles, carries, atomics), a 2^18 prefix
of config 5 (local mode), sigma <= 4 (the two-level path), the wavelet matrix,
the Huffman-shaped tree, access/rank/select; each result checked against the
oracle so that a silent corruption also fails."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, oracle
import paper_1407_8142_b200 as wt

def check(S, sigma):
    t = wt.build(torch.from_numpy(S).cuda(), sigma)
    got, want = t.numpy(), oracle.build(S, sigma)
    for k in ("bits", "level_node_ptr", "node_key", "node_start", "rank_block", "rank_super"):
        assert np.array_equal(got[k], want[k]), k
    pos = torch.arange(0, S.size, 97, device="cuda", dtype=torch.int64)
    assert np.array_equal(t.access(pos).cpu().numpy(), S[::97].astype(np.uint32))
    t.select_index()
    t.free()

cases = [(gen.config_input(gen.CONFIGS[1]), 256),
         (gen.config_input(gen.CONFIGS[3], 1 << 20), 256),
         (gen.config_input(gen.CONFIGS[4], 1 << 20), 1 << 16),
         (gen.config_input(gen.CONFIGS[5], 1 << 18), 1 << 32),
         (gen.uniform_below(100000, 4, seed=2, dtype=np.uint8), 4)]
for S, sigma in cases:
    check(S, sigma)
    print("tree ok", S.size, sigma, flush=True)
S = gen.config_input(gen.CONFIGS[4], 1 << 18)
m = wt.wm_build(torch.from_numpy(S).cuda(), 1 << 16)
want = oracle.wm_build(S, 1 << 16)
got = m.numpy()
assert all(np.array_equal(got[k], want[k]) for k in ("bits", "zeros", "rank_block", "rank_super"))
m.free()
print("matrix ok", flush=True)
S = gen.config_input(gen.CONFIGS[3], 1 << 18)
h = wt.hwt_build(torch.from_numpy(S).cuda(), 256)
want = oracle.hwt_build(S, 256)
got = h.numpy()
assert all(np.array_equal(got[k], want[k]) for k in ("code", "bits", "node_key", "node_start", "rank_block"))
h.free()
torch.cuda.synchronize()
print("sanitize run ok", flush=True)
