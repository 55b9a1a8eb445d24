"""One wm_build (after one warm-up) of a config, for ncu.  usage: wm_one.py CFG"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_1407_8142_b200 as wt
cfg = gen.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
S = torch.from_numpy(gen.config_input(cfg)).cuda()
wt.wm_build(S, cfg.sigma).free()
torch.cuda.synchronize()
wt.wm_build(S, cfg.sigma).free()
torch.cuda.synchronize()
