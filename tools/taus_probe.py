"""Time cfg builds for several level-group splits (WT_TAUS) and check each against the oracle on a prefix."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK = r'''
import sys, os
sys.path.insert(0, %r)
import numpy as np, torch, gen, oracle, paper_1407_8142_b200 as wt
cfg = gen.CONFIGS[int(sys.argv[1])]
S = gen.config_input(cfg, 1 << 20)
t = wt.build(torch.from_numpy(S).cuda(), cfg.sigma); got = t.numpy(); want = oracle.build(S, cfg.sigma)
bad = [k for k in ("bits", "level_node_ptr", "node_key", "node_start", "rank_block", "rank_super") if not np.array_equal(got[k], want[k])]
print("parity", "OK" if not bad else "FAIL " + ",".join(bad))
''' % ROOT
cfgs = sys.argv[1:] or ["4"]
for taus in os.environ.get("TAUS_LIST", "8,8;6,5,5;8,4,4;4,4,8;6,6,4;5,5,6;4,6,6").split(";"):
    env = dict(os.environ, WT_TAUS=taus)
    for c in cfgs:
        chk = subprocess.run([sys.executable, "-c", CHECK, c], capture_output=True, text=True, env=env, timeout=600)
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "kprof.py"), c], capture_output=True,
                             text=True, env=env, timeout=600)
        print(f"== taus {taus} cfg{c}: {chk.stdout.strip() or chk.stderr[-300:]}")
        print(out.stdout.strip() or out.stderr[-600:])
