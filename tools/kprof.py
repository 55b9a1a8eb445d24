"""Per-kernel device times of wt_build (CUDA events the library records).
usage: kprof.py CFG [CFG ...]   (KPROF_REPS builds each, default 5)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_1407_8142_b200 as wt

reps = int(os.environ.get("KPROF_REPS", "5"))
for ci in [int(a) for a in sys.argv[1:]] or [4]:
    cfg = gen.CONFIGS[ci]
    S = torch.from_numpy(gen.config_input(cfg)).cuda()
    for _ in range(2):
        wt.build(S, cfg.sigma).free()
    wt.profile_enable(True)
    for _ in range(reps):
        wt.build(S, cfg.sigma).free()
    torch.cuda.synchronize()
    p = wt.last_profile(total=True)
    wt.profile_enable(False)
    tot = sum(k["ms"] for k in p["kernels"])
    print(f"cfg{ci} {os.environ.get('TAG', '')}: {tot / reps:.3f} ms of kernels per build")
    for k in sorted(p["kernels"], key=lambda k: -k["ms"]):
        print(f"   {k['name']:18s} {k['ms'] / reps:8.3f} ms  x{k['launches'] // reps}")
    del S
