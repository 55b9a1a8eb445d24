"""Stand-in for compute-sanitizer (closed on this pool): run the coverage cases
of tools/sanitize_run.py and a seeded fuzz sweep against the library built with
-DWT_DEBUG (device-side bounds / consistency checks, WT_CHECK in csrc/), every
result compared with the oracle, then read the first failed check (code, CTA,
thread).  usage: WT_LIB_PATH=.../lib_debug.so python tools/debug_check.py [seconds]"""
import ctypes, os, runpy, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, oracle
import paper_1407_8142_b200 as wt

assert os.environ.get("WT_LIB_PATH", "").endswith("debug.so"), "point WT_LIB_PATH at the -DWT_DEBUG build"
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "sanitize_run.py"), run_name="__main__")
rng = np.random.default_rng(2024)
t0, cases, bad = time.time(), 0, 0
while time.time() - t0 < budget:
    n = int(np.exp(rng.uniform(0, np.log(3e6))))
    k = int(rng.integers(1, 33))
    sigma = int(rng.integers(max(1, 1 << (k - 1)), (1 << k) + 1))
    dt = np.uint8 if sigma <= 256 else (np.uint16 if sigma <= 65536 else np.uint32)
    shape = rng.integers(0, 3)
    S = gen.uniform_below(n, sigma, seed=cases, dtype=dt)
    if shape == 1:
        S = np.sort(S)
    elif shape == 2 and n:
        S[rng.integers(0, n, n // 2)] = dt(sigma - 1)
    t = wt.build(torch.from_numpy(S).cuda(), sigma)
    got, want = t.numpy(), oracle.build(S, sigma)
    for key in ("bits", "level_node_ptr", "node_key", "node_start", "rank_block", "rank_super"):
        if not np.array_equal(got[key], want[key]):
            bad += 1
            print("MISMATCH", n, sigma, shape, key, flush=True)
    t.free()
    cases += 1
torch.cuda.synchronize()
lib = ctypes.CDLL(os.environ["WT_LIB_PATH"])
code = (ctypes.c_uint32 * 4)()
lib.wt_debug_code(code)
print(f"debug_check: {cases} fuzz cases in {time.time() - t0:.0f} s, {bad} mismatches, "
      f"first failed device check: {list(code)[:3]} (0 = none)", flush=True)
sys.exit(1 if bad or code[0] else 0)
