"""One hwt_build (after one warm-up) of a chosen input, for ncu launch lists.
usage: hwt_one.py cfg4 | zipf2.0 | cfg3"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1407_8142_b200 as wt

which = sys.argv[1]
if which.startswith("cfg"):
    cfg = gen.CONFIGS[int(which[3:])]
    S, sigma = gen.config_input(cfg), cfg.sigma
else:
    s = float(which[4:])
    S = np.minimum(np.random.default_rng(7).zipf(s, 1 << 26) - 1, 65535).astype(np.uint16)
    sigma = 65536
St = torch.from_numpy(S).cuda()
wt.hwt_build(St, sigma).free()
torch.cuda.synchronize()
wt.hwt_build(St, sigma).free()
torch.cuda.synchronize()
