"""Quick GPU probe: per-kernel device times of wt_build on the configs (not the bench)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1407_8142_b200 as wt

cfgs = [int(x) for x in (sys.argv[1:] or ["1", "2", "3", "4"])]
wt.profile_enable(True)
for ci in cfgs:
    cfg = gen.CONFIGS[ci]
    S = torch.from_numpy(gen.config_input(cfg)).cuda()
    for it in range(4):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        t = wt.build(S, cfg.sigma)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        t.free()
    prof = wt.last_profile()
    nl = cfg.n * cfg.levels
    print(f"cfg{ci}: build {ms:.3f} ms  {nl/(ms*1e-3):.3e} sym-levels/s  launches={prof['total_launches']}")
    for k in prof["kernels"]:
        bw = k["algo_bytes"] / (k["ms"] * 1e-3) / 1e9 if k["ms"] > 0 else 0
        print(f"   {k['name']:16s} {k['ms']:8.3f} ms x{k['launches']}  algo {k['algo_bytes']/1e6:9.1f} MB  {bw:8.1f} GB/s")
