"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact.

Every array of include/wt.h is compared element by element: bitmaps, node
CSR (level_node_ptr, node_key, node_start), rank_block and rank_super.  The
bar is bit-exact (integer work).  Sizes span several warp tiles (4096
elements) and ragged tails; full-size configs use the launch configuration
bench.py times.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import gen
import oracle
from tests import pins

pytestmark = pytest.mark.gpu

KEYS = ("bits", "level_node_ptr", "node_key", "node_start", "rank_block", "rank_super")


def _wt():
    import paper_1407_8142_b200 as wt
    return wt


def _dtype_for(sigma):
    return np.uint8 if sigma <= 256 else (np.uint16 if sigma <= 65536 else np.uint32)


def _compare(S, sigma, tree=None):
    wt = _wt()
    own = tree is None
    if own:
        tree = wt.build(torch.from_numpy(np.ascontiguousarray(S)).cuda(), sigma)
    got = tree.numpy()
    want = oracle.build(S, sigma)
    for k in KEYS:
        assert got[k].shape == want[k].shape, f"{k} shape {got[k].shape} vs {want[k].shape}"
        if not np.array_equal(got[k], want[k]):
            bad = np.nonzero(got[k] != want[k])[0]
            raise AssertionError(f"{k}: {bad.size} mismatches, first at {bad[:5]} "
                                 f"got {got[k][bad[:5]]} want {want[k][bad[:5]]}")
    assert got["total_nodes"] == want["total_nodes"]
    if own:
        tree.free()
    return got


SIZES = [0, 1, 31, 32, 33, 63, 64, 65, 511, 512, 513, 4095, 4096, 4097, 8191, 8192, 8193, 12345,
         65536, 65537, 100000]
SIGMAS = [1, 2, 3, 4, 5, 146, 256, 257, 1000, 4096, 65535, 65536]


@pytest.mark.parametrize("sigma", SIGMAS)
@pytest.mark.parametrize("n", SIZES)
def test_random_small(n, sigma):
    S = gen.uniform_below(n, sigma, seed=1000 * n + sigma, dtype=_dtype_for(sigma))
    _compare(S, sigma)


@pytest.mark.parametrize("dtype", [np.uint16, np.uint32])
@pytest.mark.parametrize("sigma", [256, 300, 65536])
def test_wide_element_types(dtype, sigma):
    S = gen.uniform_below(50000, sigma, seed=7, dtype=dtype)
    _compare(S, sigma)


@pytest.mark.parametrize("n", [1, 4097, 200000])
@pytest.mark.parametrize("sigma", [2, 256, 65536])
def test_adversarial_shapes(n, sigma):
    dt = _dtype_for(sigma)
    _compare(np.full(n, sigma - 1, dtype=dt), sigma)          # all equal (max symbol)
    _compare(np.zeros(n, dtype=dt), sigma)                   # all zero
    S = np.sort(gen.uniform_below(n, sigma, seed=3, dtype=dt))
    _compare(S, sigma)                                       # ascending
    _compare(S[::-1].copy(), sigma)                          # descending
    S = gen.uniform_below(n, sigma, seed=4, dtype=dt)
    S[n // 2] = sigma - 1                                    # a lone max symbol
    _compare(S, sigma)


def test_skewed_zipf():
    S = gen.zipf_permuted(300000, seed=3)
    _compare(S, 256)


def test_upper_bits_nonzero_u32():
    """uint32 symbols whose upper bits are non-zero but < sigma."""
    S = gen.uniform_below(100000, 65536, seed=5, dtype=np.uint32)
    S |= np.uint32(0x8000)
    _compare(S, 65536)


def test_symbol_out_of_range():
    wt = _wt()
    S = np.array([0, 1, 2, 9, 3], dtype=np.uint8)
    with pytest.raises(wt.WtError) as e:
        wt.build(torch.from_numpy(S).cuda(), 5)
    assert e.value.code == -2  # WT_ESYMBOL
    S = gen.uniform_below(100000, 65536, seed=1, dtype=np.uint32)
    S[77777] = 65536
    with pytest.raises(wt.WtError) as e:
        wt.build(torch.from_numpy(S).cuda(), 65536)
    assert e.value.code == -2
    # the library recovers: a valid build right after succeeds
    _compare(S[:77777].copy(), 65536)


def test_unaligned_device_pointer():
    wt = _wt()
    S = gen.uniform_below(70001, 1000, seed=9, dtype=np.uint32)
    buf = torch.from_numpy(np.concatenate([np.zeros(1, np.uint32), S])).cuda()
    tree = wt.build(buf[1:], 1000)
    _compare(S, 1000, tree)
    tree.free()


def test_build_host_matches():
    wt = _wt()
    S = gen.uniform_below(123457, 4096, seed=2, dtype=np.uint16)
    tree = wt.build_host(S, 4096)
    _compare(S, 4096, tree)
    tree.free()


def test_deterministic_repeat():
    wt = _wt()
    S = torch.from_numpy(gen.uniform_below(1 << 20, 65536, seed=8, dtype=np.uint32)).cuda()
    a = wt.build(S, 65536).numpy()
    for _ in range(3):
        b = wt.build(S, 65536).numpy()
        for k in KEYS:
            assert np.array_equal(a[k], b[k])


@pytest.mark.parametrize("n,sigma", [(100000, 1000), (70000, 256), (5000, 65536), (3, 4)])
def test_queries_bruteforce(n, sigma):
    wt = _wt()
    S = gen.uniform_below(n, sigma, seed=n, dtype=_dtype_for(sigma))
    tree = wt.build(torch.from_numpy(S).cuda(), sigma)
    rng = np.random.default_rng(1)
    pos = rng.integers(0, n, 2000)
    got = tree.access(torch.from_numpy(pos).cuda()).cpu().numpy()
    assert np.array_equal(got, S[pos].astype(np.uint32))
    cs = rng.integers(0, sigma, 2000).astype(np.int32)
    cs[:200] = S[pos[:200]]  # present symbols
    r = tree.rank(torch.from_numpy(cs).cuda(), torch.from_numpy(pos).cuda()).cpu().numpy()
    want = np.array([pins.rank_bruteforce(S, c, i) for c, i in zip(cs, pos)], dtype=np.uint64)
    assert np.array_equal(r, want)
    # out-of-range conventions
    bad = tree.access(torch.tensor([n, n + 5], device="cuda")).cpu().numpy()
    assert bad.tolist() == [0xFFFFFFFF] * 2
    rb = tree.rank(torch.tensor([sigma, 0], dtype=torch.int32, device="cuda"),
                   torch.tensor([0, n], device="cuda")).cpu().numpy()
    assert rb.tolist() == [2 ** 64 - 1] * 2
    tree.free()


@pytest.mark.parametrize("cfg_idx", [1, 2, 3, 4])
def test_full_config_vs_oracle(cfg_idx):
    """BASELINE.json configs 1-4 at full size, every array bit-exact."""
    cfg = gen.CONFIGS[cfg_idx]
    S = gen.config_input(cfg)
    _compare(S, cfg.sigma)


# ---- L > 16: four groups, narrowed u32/u16/u8 keys, local mode for small nodes ----
@pytest.mark.parametrize("sigma", [1 << 17, 3 << 18, 1 << 20, 1 << 24, (1 << 31) + 5, 1 << 32])
@pytest.mark.parametrize("n", [1, 4097, 100000, 1 << 20])
def test_large_alphabet(n, sigma):
    S = gen.uniform_below(n, sigma, seed=n + (sigma & 0xFFFF), dtype=np.uint32)
    _compare(S, sigma)


@pytest.mark.parametrize("sigma", [1 << 20, 1 << 32])
def test_large_alphabet_adversarial(sigma):
    n = 60000
    _compare(np.full(n, sigma - 1, dtype=np.uint32), sigma)           # one huge node per level
    S = gen.uniform_below(n, 64, seed=2, dtype=np.uint32) * np.uint32(sigma // 64)
    _compare(S, sigma)                                                # few, large deep nodes
    S = np.sort(gen.uniform_below(n, sigma, seed=4, dtype=np.uint32))
    _compare(S, sigma)


def test_large_alphabet_queries():
    wt = _wt()
    n, sigma = 200000, 1 << 32
    S = gen.uniform_below(n, sigma, seed=77, dtype=np.uint32)
    S[1000:1100] = S[5]  # a repeated symbol
    tree = wt.build(torch.from_numpy(S).cuda(), sigma)
    pos = np.random.default_rng(3).integers(0, n, 3000)
    got = tree.access(torch.from_numpy(pos).cuda()).cpu().numpy()
    assert np.array_equal(got, S[pos])
    cs = S[pos[:500]].astype(np.int64).astype(np.int32)  # u32 symbols through an int32 view
    r = tree.rank(torch.from_numpy(cs).cuda(), torch.from_numpy(pos[:500]).cuda()).cpu().numpy()
    want = [pins.rank_bruteforce(S, np.uint32(c), i) for c, i in zip(S[pos[:500]], pos[:500])]
    assert r.tolist() == want
    tree.free()


@pytest.mark.slow
def test_full_config5_vs_oracle():
    """Config 5 (n = 2^29 u32, sigma = 2^32, 32 levels, ~1.7e9 nodes) at full
    size: every array bit-exact, compared one array at a time (host RAM)."""
    wt = _wt()
    cfg = gen.CONFIGS[5]
    S = gen.config_input(cfg)
    with oracle.OracleTree(S, cfg.sigma) as ot:
        tree = wt.build(torch.from_numpy(S).cuda(), cfg.sigma)
        assert tree.total_nodes == ot.total_nodes
        for k in KEYS:
            want = ot.array(k)
            got = getattr(tree, k).cpu().numpy()
            assert got.shape == want.shape, k
            assert np.array_equal(got, want), f"{k} differs"
            del want, got
        tree.free()


# ---- local mode, rows of 33..64 symbols (two symbols per lane) and their edges ----
@pytest.mark.parametrize("n,sigma", [(12288, 1 << 16), (20000, 1 << 12), (3 << 20, 1 << 24), (9000, 1 << 20)])
def test_local_rows_pair_path(n, sigma):
    S = gen.uniform_below(n, sigma, seed=n ^ sigma, dtype=np.uint32)
    _compare(S, sigma)


@pytest.mark.parametrize("sizes", [(33, 64, 65, 32, 1, 48), (64,) * 40, (40, 63, 33, 2, 64, 31, 64),
                                   (4096, 2000, 1025, 1024, 1100, 70, 65, 64, 33, 1) + (10,) * 200,
                                   (1025,) * 3 + (7,) * 100])
def test_local_rows_exact_sizes(sizes):
    # level-8 nodes of chosen sizes (sigma = 2^16: group 1 runs in local mode)
    rng = np.random.default_rng(len(sizes))
    parts = [(np.uint32(p) << np.uint32(8)) | rng.integers(0, 256, s).astype(np.uint32)
             for p, s in zip(rng.choice(256, len(sizes), replace=False), sizes)]
    S = np.concatenate(parts)
    rng.shuffle(S)
    _compare(S, 1 << 16)


@pytest.mark.parametrize("dtype,sigma", [(np.uint8, 256), (np.uint16, 40000), (np.uint32, 1 << 24)])
@pytest.mark.parametrize("off", [1, 3, 7])
def test_unaligned_narrow_types(dtype, sigma, off):
    wt = _wt()
    S = gen.uniform_below(90001, sigma, seed=off, dtype=dtype)
    v = torch.from_numpy(S).cuda()[off:]
    tree = wt.build(v, sigma)
    _compare(S[off:].copy(), sigma, tree)
    tree.free()


@pytest.mark.parametrize("n,sigma", [(300000, 1 << 16), (1 << 20, 256), (777777, 1 << 12), (5000, 1000)])
def test_no_zero_init_dirty_memory(n, sigma):
    """A5 without a zero-initialised bitmap (put_shared_word): the bitmap words
    are written, never OR-ed into zeros, so a build whose output memory held
    all-ones garbage (the freed bitmap of an earlier build, re-used by the
    stream-ordered pool) is still bit-exact.  Each earlier tree's arrays are
    filled with 0xff before it is freed."""
    wt = _wt()
    S = gen.uniform_below(n, sigma, seed=n % 97, dtype=_dtype_for(sigma))
    St = torch.from_numpy(S).cuda()
    for _ in range(3):
        t = wt.build(St, sigma)
        for k in ("bits", "rank_block", "rank_super", "node_key", "node_start"):
            v = getattr(t, k)
            if v is not None and v.numel():
                v.view(torch.uint8).fill_(0xff)
        torch.cuda.synchronize()
        t.free()
    _compare(S, sigma)


# ---- 8 does not divide L: the first group takes the remainder ----
@pytest.mark.parametrize("dtype,sigma", [(np.uint16, 1 << 9), (np.uint16, 1 << 10), (np.uint32, 1 << 10),
                                         (np.uint16, 1 << 13), (np.uint32, 5000), (np.uint32, 1 << 15),
                                         (np.uint32, 1 << 17), (np.uint32, 1 << 18), (np.uint32, 1 << 21),
                                         (np.uint32, (1 << 23) - 1), (np.uint32, (1 << 26) + 3),
                                         (np.uint32, 1 << 31)])
def test_remainder_first_split(dtype, sigma):
    """Chain mode in every group but the deepest (n is large enough that the
    level-l0 rows of the first full group span many tiles): the first group has
    tau = L mod 8 levels and writes keys narrowed to a multiple of 8 bits."""
    n = 3_000_001
    S = gen.uniform_below(n, sigma, seed=sigma % 1009, dtype=dtype)
    _compare(S, sigma)
    if sigma in (1 << 10, 1 << 18):
        S = np.sort(S)
        S[::7] = S[0]  # skew: one heavy symbol interleaved with ascending runs
        _compare(S, sigma)
