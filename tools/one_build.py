"""Run wt_build on one config (optionally a prefix of n symbols) a few times; for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1407_8142_b200 as wt

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = (int(sys.argv[2]) or None) if len(sys.argv) > 2 else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = gen.CONFIGS[ci]
S = torch.from_numpy(gen.config_input(cfg, n)).cuda()
for _ in range(reps):
    wt.build(S, cfg.sigma).free()
torch.cuda.synchronize()
print("ok", ci, S.numel())
