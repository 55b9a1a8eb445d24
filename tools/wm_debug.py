"""Which wavelet-matrix levels differ from the oracle (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, oracle
import paper_1407_8142_b200 as wt
for n, sigma in [(4097, 1 << 20), (5000, 1 << 17), (9000, 1 << 20), (4097, 1 << 32), (20000, 1 << 16), (12000, 1 << 17)]:
    S = gen.uniform_below(n, sigma, seed=31 * n + sigma, dtype=np.uint32)
    got = wt.wm_build(torch.from_numpy(S).cuda(), sigma).numpy()
    want = oracle.wm_build(S, sigma)
    L = want["levels"]; W = want["words_per_level"]
    bad = [l for l in range(L) if not np.array_equal(got["bits"][l * W:(l + 1) * W], want["bits"][l * W:(l + 1) * W])]
    print(n, sigma, "bad levels:", bad, "zeros ok:", np.array_equal(got["zeros"], want["zeros"]))
    for l in bad[:2]:
        g = np.unpackbits(got["bits"][l * W:(l + 1) * W].view(np.uint8), bitorder="little")[:n]
        w = np.unpackbits(want["bits"][l * W:(l + 1) * W].view(np.uint8), bitorder="little")[:n]
        d = np.nonzero(g != w)[0]
        print("   level", l, "mismatches", d.size, "first", d[:8], "ones got/want", g.sum(), w.sum())
# which element sits at the mismatching position (A_l = S stably sorted by reversed top-l bits)
n, sigma = 4097, 1 << 20
S = gen.uniform_below(n, sigma, seed=31 * n + sigma, dtype=np.uint32).astype(np.int64)
L = 20
for l, posx in [(4, 260)]:
    top = S >> (L - l)
    rev = np.zeros_like(top)
    for b in range(l):
        rev |= ((top >> b) & 1) << (l - 1 - b)
    order = np.argsort(rev, kind="stable")
    e = order[posx]
    print("level", l, "pos", posx, "element", e, "key", S[e], "bit", (S[e] >> (L - 1 - l)) & 1,
          "class", rev[e], "class run", np.nonzero(rev[order] == rev[e])[0][[0, -1]])
