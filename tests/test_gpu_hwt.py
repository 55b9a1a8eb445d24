"""GPU parity of the Huffman-shaped wavelet tree (SURVEY §8(f) f3,
PAPER.md:854-876): the CUDA path through the C ABI (hwt_build / hwt_access /
hwt_rank) against the CPU oracle (oracle_hwt_build), bit-exact on every array
(codes, level sizes, bitmaps, node tables, rank directories)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import gen
import oracle

pytestmark = pytest.mark.gpu
KEYS = ("code", "code_len", "level_len", "level_word_ptr", "level_block_ptr", "level_super_ptr", "bits",
        "rank_block", "rank_super", "level_node_ptr", "node_key", "node_start")


def _dt(sigma):
    return np.uint8 if sigma <= 256 else (np.uint16 if sigma <= 65536 else np.uint32)


def _compare(S, sigma):
    import paper_1407_8142_b200 as wt
    t = wt.hwt_build(torch.from_numpy(np.ascontiguousarray(S)).cuda(), sigma)
    got = t.numpy()
    want = oracle.hwt_build(S, sigma)
    assert got["levels"] == want["levels"]
    assert got["total_nodes"] == want["total_nodes"]
    if want["levels"] == 0 and S.size:
        assert got["only_symbol"] == want["only_symbol"]
    for k in KEYS:
        assert got[k].shape == want[k].shape, f"{k} shape {got[k].shape} vs {want[k].shape}"
        if not np.array_equal(got[k], want[k]):
            bad = np.nonzero(got[k] != want[k])[0]
            raise AssertionError(f"{k}: {bad.size} mismatches, first at {bad[:5]}")
    assert got["total_bits"] == int(want["level_len"].sum())
    return t


def _queries(t, S, sigma, k=3000, seed=0):
    rng = np.random.default_rng(seed)
    n = S.size
    pos = rng.integers(0, max(n, 1), k) if n else np.zeros(k, np.int64)
    pos[:3] = [n, n + 5, 0]
    sym = np.where(rng.random(k) < 0.6, S[np.minimum(pos, max(n - 1, 0))] if n else 0,
                   rng.integers(0, sigma + 2, k)).astype(np.uint32)
    with oracle.OracleHWT(S, sigma) as o:
        want_a = o.access(pos)
        want_r = o.rank(sym, pos)
    acc = t.access(torch.from_numpy(pos.astype(np.int64)).cuda()).cpu().numpy()
    rk = t.rank(torch.from_numpy(sym.view(np.int32)).cuda(), torch.from_numpy(pos.astype(np.int64)).cuda()).cpu().numpy()
    assert np.array_equal(acc, want_a)
    assert np.array_equal(rk, want_r)
    # select_c(k): symbols from S and random ones, k in [0, count + 1]
    cs = np.where(rng.random(k) < 0.7, S[rng.integers(0, max(n, 1), k)] if n else 0,
                  rng.integers(0, sigma + 2, k)).astype(np.uint32)
    cnt = np.bincount(S.astype(np.int64), minlength=sigma + 2) if n else np.zeros(sigma + 2, np.int64)
    ks = (rng.random(k) * (cnt[np.minimum(cs, sigma + 1)] + 2)).astype(np.int64)
    # expected: the k'th occurrence from a stable sort of S (brute force, no oracle walk)
    order = np.argsort(S, kind="stable") if n else np.zeros(0, np.int64)
    first = np.searchsorted(S[order], cs) if n else np.zeros(k, np.int64)
    c_ok = (cs < sigma) & (ks >= 1) & (ks <= cnt[np.minimum(cs, sigma + 1)])
    want_s = np.full(k, 2**64 - 1, dtype=np.uint64)
    want_s[c_ok] = order[first[c_ok] + ks[c_ok] - 1]
    sel = t.select(torch.from_numpy(cs.view(np.int32)).cuda(), torch.from_numpy(ks).cuda()).cpu().numpy()
    assert np.array_equal(sel, want_s)
    ok = pos < n
    if n:
        assert np.array_equal(acc[ok], S[pos[ok]].astype(np.uint32))


@pytest.mark.parametrize("sigma", [1, 2, 3, 5, 146, 256, 257, 1000, 8192, 8193, 65536])
@pytest.mark.parametrize("n", [0, 1, 2, 33, 4097, 100000])
def test_hwt_uniform(n, sigma):
    S = gen.uniform_below(n, sigma, seed=17 * n + sigma, dtype=_dt(sigma))
    _compare(S, sigma).free()


@pytest.mark.parametrize("shape", ["zipf", "geometric", "fibonacci", "constant", "two", "sorted", "sparse"])
def test_hwt_shapes(shape):
    rng = np.random.default_rng(5)
    sigma = 256
    if shape == "zipf":
        S = gen.zipf_permuted(300000, 11)
    elif shape == "geometric":
        S = np.minimum(rng.geometric(0.2, 200000) - 1, 255).astype(np.uint8)
    elif shape == "fibonacci":  # path-shaped tree, depth 24 (staged build)
        fib = [1, 1]
        while len(fib) < 25:
            fib.append(fib[-1] + fib[-2])
        S = np.repeat(np.arange(25, dtype=np.uint8), fib)
        rng.shuffle(S)
    elif shape == "constant":
        S = np.full(5000, 77, np.uint8)
    elif shape == "two":
        S = (rng.random(10000) < 0.01).astype(np.uint8) * 200
    elif shape == "sorted":
        S = np.sort(gen.zipf_permuted(100000, 2))
    else:  # few symbols spread over a large alphabet
        S = rng.choice(np.array([3, 900, 40000, 65535], np.uint32), 50000, p=[0.7, 0.2, 0.07, 0.03]).astype(np.uint32)
        sigma = 65536
    t = _compare(S, sigma)
    _queries(t, S, sigma)
    t.free()


def test_hwt_queries_u16():
    S = gen.uniform_below(150000, 3000, seed=8, dtype=np.uint16)
    t = _compare(S, 3000)
    _queries(t, S, 3000, k=5000, seed=3)
    t.free()


def test_hwt_errors():
    import paper_1407_8142_b200 as wt
    with pytest.raises(wt.WtError) as e:
        wt.hwt_build(torch.tensor([0, 1, 5, 2], dtype=torch.uint8).cuda(), 4)
    assert e.value.code == wt.WT_ESYMBOL
    with pytest.raises(wt.WtError) as e:
        wt.hwt_build(torch.tensor([0, 1], dtype=torch.int32).cuda(), 1 << 17)
    assert e.value.code == -1


def test_hwt_too_deep():
    # 34 Fibonacci weights: a 33-bit code (R-20) -> WT_EUNSUPPORTED, nothing leaks
    import paper_1407_8142_b200 as wt
    fib = [1, 1]
    while len(fib) < 34:
        fib.append(fib[-1] + fib[-2])
    S = torch.from_numpy(np.repeat(np.arange(34, dtype=np.uint8), fib)).cuda()
    with pytest.raises(wt.WtError) as e:
        wt.hwt_build(S, 34)
    assert e.value.code == -5


@pytest.mark.parametrize("cfg_idx", [1, 2, 3])
def test_hwt_full_config(cfg_idx):
    cfg = gen.CONFIGS[cfg_idx]
    S = gen.config_input(cfg)
    t = _compare(S, cfg.sigma)
    _queries(t, S, cfg.sigma, k=2000, seed=cfg_idx)
    t.free()


@pytest.mark.parametrize("s,n,sigma,dtype", [(2.0, 300000, 65536, np.uint16), (1.3, 200000, 4096, np.uint16),
                                             (3.0, 100000, 65536, np.uint32), (1.6, 150000, 1000, np.uint16)])
def test_hwt_staged(s, n, sigma, dtype):
    # skewed codes longer than 8 bits: the staged build (8-level stages over the
    # elements still alive), checked array by array and by queries
    S = np.minimum(np.random.default_rng(int(s * 10)).zipf(s, n) - 1, sigma - 1).astype(dtype)
    t = _compare(S, sigma)
    assert t.levels > 8
    if s >= 2.0:
        assert t.stages > 1  # most elements leave within the first 8 levels
    _queries(t, S, sigma, k=1500, seed=1)
    t.free()


@pytest.mark.parametrize("dtype,sigma", [(np.uint8, 200), (np.uint16, 3000), (np.uint32, 70000 - 4465)])
def test_hwt_unaligned_device_pointer(dtype, sigma):
    S = np.minimum(np.random.default_rng(9).zipf(1.5, 50001) - 1, sigma - 1).astype(dtype)
    base = torch.from_numpy(S).cuda()
    for off in (1, 2):
        v = base[off:]
        assert v.data_ptr() % 16 != 0
        import paper_1407_8142_b200 as wt
        t = wt.hwt_build(v, sigma)
        got, want = t.numpy(), oracle.hwt_build(S[off:].copy(), sigma)
        for k in KEYS:
            assert np.array_equal(got[k], want[k]), (off, k)
        t.free()


@pytest.mark.parametrize("sigma,n", [(5, 3000), (256, 5000), (3000, 4000), (1, 100)])
def test_hwt_select_vs_oracle(sigma, n):
    S = np.minimum(np.random.default_rng(n).zipf(1.4, n) - 1, sigma - 1).astype(np.uint16)
    import paper_1407_8142_b200 as wt
    t = wt.hwt_build(torch.from_numpy(S).cuda(), sigma)
    rng = np.random.default_rng(1)
    cs = np.concatenate([S[rng.integers(0, n, 400)], rng.integers(0, sigma + 1, 100)]).astype(np.uint32)
    ks = rng.integers(0, 60, cs.size).astype(np.int64)
    with oracle.OracleHWT(S, sigma) as o:
        want = o.select(cs, ks)
    got = t.select(torch.from_numpy(cs.view(np.int32)).cuda(), torch.from_numpy(ks).cuda()).cpu().numpy()
    assert np.array_equal(got, want)
    t.free()


@pytest.mark.slow
def test_hwt_full_config4():
    """Config 4 (n = 2^28 u32, sigma = 2^16: 16-bit codes, one stage) at full size."""
    cfg = gen.CONFIGS[4]
    S = gen.config_input(cfg)
    t = _compare(S, cfg.sigma)
    _queries(t, S, cfg.sigma, k=1000, seed=4)
    t.free()
