"""Per-build device time with and without the library's per-kernel events, and
the sum of the kernel times: what a build step spends outside its kernels.
usage: step_overhead.py CFG [STEPS]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_1407_8142_b200 as wt

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = gen.CONFIGS[ci]
S = torch.from_numpy(gen.config_input(cfg)).cuda()
st = torch.cuda.current_stream()
for _ in range(3):
    wt.build(S, cfg.sigma, st).free()
torch.cuda.synchronize()


def timed(profile):
    wt.profile_enable(profile)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(steps):
        wt.build(S, cfg.sigma, st).free()
    e1.record(st)
    torch.cuda.synchronize()
    p = wt.last_profile(total=True) if profile else None
    wt.profile_enable(False)
    return e0.elapsed_time(e1) / steps, p


for rep in range(2):
    ms_plain, _ = timed(False)
    ms_prof, p = timed(True)
    kern = sum(k["ms"] for k in p["kernels"]) / steps
    print(f"cfg{ci} rep{rep}: plain {ms_plain:.3f} ms/build, with kernel events {ms_prof:.3f}, "
          f"kernels {kern:.3f}, outside kernels {ms_plain - kern:.3f}")
    if rep == 1:
        for k in sorted(p["kernels"], key=lambda k: -k["ms"]):
            print(f"   {k['name']:18s} {k['ms'] / steps:8.3f} ms  x{k['launches'] // steps}")
