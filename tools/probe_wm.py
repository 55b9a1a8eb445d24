"""Time wm_build (wavelet matrix) on configs (device events, not the bench)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_1407_8142_b200 as wt

for ci in [int(x) for x in (sys.argv[1:] or ["3", "4"])]:
    cfg = gen.CONFIGS[ci]
    S = torch.from_numpy(gen.config_input(cfg)).cuda()
    for it in range(4):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        m = wt.wm_build(S, cfg.sigma)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        m.free()
    print(f"cfg{ci} wm: {ms:.3f} ms  {cfg.n * cfg.levels / (ms * 1e-3):.3e} sym-levels/s")
