"""GPU parity of select: the select
directory and batched select_c through the C ABI against the CPU oracle, for
the tree and the matrix."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import gen
import oracle

pytestmark = pytest.mark.gpu
MAX = 0xFFFFFFFFFFFFFFFF


def _dt(sigma):
    return np.uint8 if sigma <= 256 else (np.uint16 if sigma <= 65536 else np.uint32)


def _queries(S, sigma, rng, q=3000):
    cs, ks = [], []
    vals, counts = np.unique(S, return_counts=True)
    for _ in range(q):
        if vals.size and rng.random() < 0.8:
            i = rng.integers(0, vals.size)
            c, cnt = int(vals[i]), int(counts[i])
            k = int(rng.integers(1, cnt + 2))  # includes k = count + 1 (absent)
        else:
            c, k = int(rng.integers(0, sigma)), int(rng.integers(0, 5))
        cs.append(c)
        ks.append(k)
    return np.array(cs, dtype=np.uint32), np.array(ks, dtype=np.uint64)


def _check(S, sigma, kind):
    import paper_1407_8142_b200 as wt
    dev = torch.from_numpy(np.ascontiguousarray(S)).cuda()
    obj = wt.build(dev, sigma) if kind == "wt" else wt.wm_build(dev, sigma)
    cls = oracle.OracleTree if kind == "wt" else oracle.OracleWM
    rng = np.random.default_rng(S.size + sigma)
    with cls(S, sigma) as o:
        want_dir = o.select_dir()
        got_dir = obj.select_index()
        assert got_dir["select_per_level"] == want_dir["select_per_level"]
        for k in ("select0", "select1"):
            assert np.array_equal(got_dir[k].cpu().numpy(), want_dir[k]), k
        cs, ks = _queries(S, sigma, rng)
        got = obj.select(torch.from_numpy(cs.view(np.int32)).cuda(), torch.from_numpy(ks.view(np.int64)).cuda())
        want = o.select(cs, ks)
        assert np.array_equal(got.cpu().numpy(), want)
    obj.free()


@pytest.mark.parametrize("kind", ["wt", "wm"])
@pytest.mark.parametrize("n,sigma", [(0, 3), (1, 1), (5000, 1), (20000, 2), (70000, 4), (100000, 256), (65537, 1000),
                                     (50000, 65536), (30000, 1 << 32)])
def test_select(kind, n, sigma):
    S = gen.uniform_below(n, sigma, seed=n + sigma, dtype=_dt(sigma))
    _check(S, sigma, kind)


@pytest.mark.parametrize("kind", ["wt", "wm"])
def test_select_zipf(kind):
    _check(gen.zipf_permuted(200000, 5, dtype=np.uint8), 256, kind)


@pytest.mark.parametrize("kind", ["wt", "wm"])
def test_select_config3(kind):
    cfg = gen.CONFIGS[3]
    S = gen.config_input(cfg, 1 << 22)
    _check(S, cfg.sigma, kind)
