"""GPU parity of the wavelet matrix:
the CUDA path through the C ABI (wm_build / wm_access / wm_rank) against the
CPU oracle (oracle_wm_build), bit-exact on every array."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import gen
import oracle

pytestmark = pytest.mark.gpu
KEYS = ("bits", "zeros", "rank_block", "rank_super")


def _dt(sigma):
    return np.uint8 if sigma <= 256 else (np.uint16 if sigma <= 65536 else np.uint32)


def _compare(S, sigma):
    import paper_1407_8142_b200 as wt
    m = wt.wm_build(torch.from_numpy(np.ascontiguousarray(S)).cuda(), sigma)
    got = m.numpy()
    want = oracle.wm_build(S, sigma)
    for k in KEYS:
        assert got[k].shape == want[k].shape, f"{k} shape"
        if not np.array_equal(got[k], want[k]):
            bad = np.nonzero(got[k] != want[k])[0]
            raise AssertionError(f"{k}: {bad.size} mismatches, first at {bad[:5]}")
    return m


@pytest.mark.parametrize("sigma", [1, 2, 3, 5, 146, 256, 257, 1000, 65536, 1 << 20, 1 << 32])
@pytest.mark.parametrize("n", [0, 1, 33, 4095, 4097, 12345, 100000])
def test_wm_random(n, sigma):
    S = gen.uniform_below(n, sigma, seed=31 * n + sigma, dtype=_dt(sigma))
    _compare(S, sigma).free()


@pytest.mark.parametrize("shape", ["sorted", "descending", "constant", "zipf"])
def test_wm_adversarial(shape):
    S = gen.uniform_below(70000, 256, seed=9, dtype=np.uint8)
    if shape == "zipf":
        S = gen.zipf_permuted(70000, 9, dtype=np.uint8)
    else:
        S = {"sorted": np.sort(S), "descending": np.sort(S)[::-1].copy(), "constant": np.full(70000, 7, np.uint8)}[shape]
    _compare(S, 256).free()


def test_wm_queries():
    S = gen.uniform_below(100000, 3000, seed=4, dtype=np.uint16)
    m = _compare(S, 3000)
    rng = np.random.default_rng(2)
    pos = rng.integers(0, S.size, 2000)
    sym = np.where(rng.random(2000) < 0.5, S[pos], rng.integers(0, 3000, 2000)).astype(np.uint32)
    acc = m.access(torch.from_numpy(pos.astype(np.int64)).cuda()).cpu().numpy()
    assert np.array_equal(acc, S[pos].astype(np.uint32))
    rk = m.rank(torch.from_numpy(sym.view(np.int32)).cuda(), torch.from_numpy(pos.astype(np.int64)).cuda()).cpu().numpy()
    want = np.array([np.count_nonzero(S[:i + 1] == c) for c, i in zip(sym, pos)], dtype=np.uint64)
    assert np.array_equal(rk, want)
    m.free()


def test_wm_symbol_out_of_range():
    import paper_1407_8142_b200 as wt
    S = np.array([0, 1, 5, 2], dtype=np.uint8)
    with pytest.raises(wt.WtError) as e:
        wt.wm_build(torch.from_numpy(S).cuda(), 4)
    assert e.value.code == wt.WT_ESYMBOL


@pytest.mark.parametrize("cfg_idx", [1, 2, 3, 4])
def test_wm_full_config(cfg_idx):
    cfg = gen.CONFIGS[cfg_idx]
    S = gen.config_input(cfg)
    _compare(S, cfg.sigma).free()


@pytest.mark.parametrize("dtype,sigma", [(np.uint8, 200), (np.uint16, 3000), (np.uint32, 1 << 20)])
def test_wm_unaligned_device_pointer(dtype, sigma):
    import paper_1407_8142_b200 as wt
    S = gen.uniform_below(70001, sigma, seed=5, dtype=dtype)
    base = torch.from_numpy(S).cuda()
    for off in (1, 3):
        v = base[off:]
        assert v.data_ptr() % 16 != 0
        m = wt.wm_build(v, sigma)
        want = oracle.wm_build(S[off:], sigma)
        got = m.numpy()
        for k in KEYS:
            assert np.array_equal(got[k], want[k]), (off, k)
        m.free()


@pytest.mark.slow
def test_wm_full_config5():
    """Config 5 (n = 2^29 u32, sigma = 2^32, 32 levels) at full size, every array."""
    cfg = gen.CONFIGS[5]
    S = gen.config_input(cfg)
    _compare(S, cfg.sigma).free()
