"""Randomised parity fuzzing of every structure against the oracle (not part of
the test suite; run on the GPU box for a time budget).
usage: fuzz.py SECONDS [seed] [max_n]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_1407_8142_b200 as wt

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
MAXN = int(sys.argv[3]) if len(sys.argv) > 3 else 400000
t_end = time.time() + budget
cases = fails = 0


def gen_seq():
    n = int(np.exp(rng.uniform(0, np.log(MAXN))))
    if rng.random() < 0.1:
        n = int(rng.integers(0, 70))
    sigma = int(np.exp(rng.uniform(0, np.log(2.0 ** 32))))
    sigma = max(1, min(sigma, 1 << 32))
    if rng.random() < 0.3:
        sigma = int(rng.choice([1, 2, 3, 4, 5, 255, 256, 257, 65535, 65536, 65537, 1 << 20, 1 << 32]))
    dt = np.uint8 if sigma <= 256 else (np.uint16 if sigma <= 65536 else np.uint32)
    if rng.random() < 0.2 and dt != np.uint32:
        dt = np.uint32
    kind = rng.choice(["uniform", "zipf", "sorted", "runs", "few", "const"])
    hi = min(sigma, 1 << 32)
    if kind == "uniform":
        S = rng.integers(0, hi, n, dtype=np.uint64)
    elif kind == "zipf":
        S = np.minimum(rng.zipf(1.0 + rng.uniform(0.1, 2.0), n) - 1, hi - 1).astype(np.uint64)
        S = (S * np.uint64(rng.integers(1, 1 << 16))) % np.uint64(hi)
    elif kind == "sorted":
        S = np.sort(rng.integers(0, hi, n, dtype=np.uint64))
    elif kind == "runs":
        S = np.repeat(rng.integers(0, hi, max(1, n // 50 + 1), dtype=np.uint64), 50)[:n]
    elif kind == "few":
        vals = rng.integers(0, hi, int(rng.integers(1, 9)), dtype=np.uint64)
        S = vals[rng.integers(0, vals.size, n)]
    else:
        S = np.full(n, int(rng.integers(0, hi)), dtype=np.uint64)
    return S.astype(dt), sigma, kind


def check(name, got, want, keys):
    global fails
    for k in keys:
        if got[k].shape != want[k].shape or not np.array_equal(got[k], want[k]):
            fails += 1
            print("FAIL", name, k, flush=True)
            return False
    return True


while time.time() < t_end:
    S, sigma, kind = gen_seq()
    off = int(rng.integers(0, 4)) if rng.random() < 0.2 else 0
    base = torch.from_numpy(np.concatenate([np.zeros(off, S.dtype), S])).cuda()
    St = base[off:]
    tag = f"n={S.size} sigma={sigma} dtype={S.dtype} kind={kind} off={off}"
    cases += 1
    try:
        t = wt.build(St, sigma)
        ok = check("wt " + tag, t.numpy(), oracle.build(S, sigma),
                   ("bits", "level_node_ptr", "node_key", "node_start", "rank_block", "rank_super"))
        if ok and S.size:
            pos = rng.integers(0, S.size, 200)
            if not np.array_equal(t.access(torch.from_numpy(pos).cuda()).cpu().numpy(), S[pos].astype(np.uint32)):
                print("FAIL access", tag, flush=True); fails += 1
            if S.size <= 200000:  # rank / select against brute force (stable sort of S)
                order = np.argsort(S, kind="stable")
                Ss = S[order]
                cs = S[rng.integers(0, S.size, 100)].astype(np.uint64)
                lo = np.searchsorted(Ss, cs)
                cnt = np.searchsorted(Ss, cs, side="right") - lo
                rank_want = np.array([np.count_nonzero(order[a:a + c] <= p) for a, c, p in zip(lo, cnt, pos[:100])],
                                     dtype=np.uint64)
                c32 = torch.from_numpy(cs.astype(np.uint32).view(np.int32)).cuda()
                p64 = torch.from_numpy(pos[:100].astype(np.int64)).cuda()
                ks = np.maximum(1, (rng.random(100) * cnt).astype(np.int64) + 1)
                k64 = torch.from_numpy(ks).cuda()
                sel_want = order[lo + ks - 1].astype(np.uint64)
                for nm, obj in (("wt", t),):
                    if not np.array_equal(obj.rank(c32, p64).cpu().numpy(), rank_want):
                        print("FAIL rank", nm, tag, flush=True); fails += 1
                    if not np.array_equal(obj.select(c32, k64).cpu().numpy(), sel_want):
                        print("FAIL select", nm, tag, flush=True); fails += 1
        t.free()
        m = wt.wm_build(St, sigma)
        check("wm " + tag, m.numpy(), oracle.wm_build(S, sigma), ("bits", "zeros", "rank_block", "rank_super"))
        m.free()
        if sigma <= 65536:
            h = wt.hwt_build(St, sigma)
            check("hwt " + tag, h.numpy(), oracle.hwt_build(S, sigma),
                  ("code", "code_len", "bits", "level_len", "level_node_ptr", "node_key", "node_start",
                   "rank_block", "rank_super"))
            h.free()
    except wt.WtError as e:
        if e.code != wt.wt.WT_EUNSUPPORTED if hasattr(wt, "wt") else True:
            print("ERROR", tag, e, flush=True)
            fails += 1
    except Exception as e:
        print("EXC", tag, repr(e), flush=True)
        fails += 1
        break
print(f"fuzz: {cases} cases, {fails} failures", flush=True)
