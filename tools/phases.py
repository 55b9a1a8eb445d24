"""Per-phase cycle breakdown of the group kernel (library built with -DWT_PHASES, thread 0 of each CTA)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1407_8142_b200 as wt
lib = ctypes.CDLL(os.environ["WT_LIB_PATH"])
NAMES = ["chain-init", "load+hist", "hscan", "coop-l0", "coop-l1", "ind-table", "ind-split", "ind-runs",
         "ind-wait", "keys+bx", "flush", "-"]
for ci in [int(x) for x in sys.argv[1:]] or [4]:
    cfg = gen.CONFIGS[ci]
    S = torch.from_numpy(gen.config_input(cfg)).cuda()
    wt.build(S, cfg.sigma).free()
    a = (ctypes.c_ulonglong * 16)()
    lib.wt_phases(a)
    wt.build(S, cfg.sigma).free()
    lib.wt_phases(a)
    tot = sum(a[:11])
    print(f"cfg{ci}: total {tot/1e9:.2f} G thread-0 cycles (all groups)")
    for i in range(11):
        print(f"   {NAMES[i]:12s} {100*a[i]/tot:5.1f}%  {a[i]/1e6:10.1f} M")
