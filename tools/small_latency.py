"""Fixed cost of small builds: wall time per wt_build + wt_free (host clock,
after warm-up, device synchronised by the build itself) for tiny inputs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1407_8142_b200 as wt
for n, sigma, dt in [(1000, 256, np.uint8), (1 << 16, 256, np.uint8), (1 << 20, 256, np.uint8), (1 << 20, 4, np.uint8),
                     (1 << 20, 1 << 16, np.uint32)]:
    S = torch.from_numpy(gen.uniform_below(n, sigma, seed=1, dtype=dt)).cuda()
    for _ in range(20):
        wt.build(S, sigma).free()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        wt.build(S, sigma).free()
    torch.cuda.synchronize()
    dt_us = (time.perf_counter() - t0) / 200 * 1e6
    print(f"n={n} sigma={sigma}: {dt_us:.1f} us per build+free", flush=True)
