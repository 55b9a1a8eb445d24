"""Pin the CPU oracle's wavelet matrix.

The oracle (oracle/wt_oracle.c, oracle_wm_build) follows the paper's
level-by-level construction (stable reorder by the level's bit with the
prefix sum of levelWT).  It is checked here against things other than
itself: hand-derived worked examples (tests/golden_wm/), the paper's sort
characterisation (reverse of the top l bits as the key, :924-925), an
order-independent zero count, a brute-force rank directory, brute-force
access/rank, and an exhaustive sweep of all sequences with n <= 5, sigma <= 4.
"""
from __future__ import annotations

import itertools
import os

import numpy as np
import pytest

import gen
import oracle
from tests import pins

GOLDEN = os.path.join(os.path.dirname(__file__), "golden_wm")


def _parse(path):
    d = {}
    for line in open(path):
        line = line.strip()
        if line and not line.startswith("#"):
            k, v = [x.strip() for x in line.split("=", 1)]
            d[k] = v
    return d


def _check(S, sigma):
    S = np.asarray(S)
    o = oracle.wm_build(S, sigma)
    L = pins.levels_of(sigma)
    assert o["levels"] == L
    bits, zeros = pins.wm_sort(S, sigma)
    assert np.array_equal(o["bits"], bits), "bitmaps differ from the reversed-prefix sort (:924-925)"
    assert np.array_equal(o["zeros"], zeros)
    for l in range(L):  # zeros[l] = symbols whose (l+1)'st highest bit is 0, in any order
        assert int(o["zeros"][l]) == int(np.count_nonzero(((S.astype(np.uint64) >> np.uint64(L - 1 - l)) & 1) == 0))
    blk, sup = pins.rank_directory_bruteforce(o["bits"], S.size, L)
    assert np.array_equal(o["rank_block"], blk)
    assert np.array_equal(o["rank_super"], sup)
    return o


@pytest.mark.parametrize("fname", sorted(os.listdir(GOLDEN)))
def test_wm_golden(fname):
    g = _parse(os.path.join(GOLDEN, fname))
    S = np.array([int(x) for x in g["S"].split()], dtype=np.uint32)
    sigma, L = int(g["sigma"]), int(g["levels"])
    o = oracle.wm_build(S, sigma)
    assert o["levels"] == L
    W = pins.wpl(S.size)
    for l in range(L):
        want = np.array([int(x) for x in g[f"bits_level{l}"].split()], dtype=np.uint8)
        assert np.array_equal(o["bits"][l * W:(l + 1) * W], pins.pack_bits(want, W)), f"level {l}"
    assert [int(z) for z in o["zeros"]] == [int(x) for x in g["zeros"].split()]
    with oracle.OracleWM(S, sigma) as m:
        for item in g["access"].split():
            i, v = item.split(":")
            assert int(m.access([int(i)])[0]) == int(v)
        for item in g["rank"].split():
            ci, v = item.split(":")
            c, i = ci.split("@")
            assert int(m.rank([int(c)], [int(i)])[0]) == int(v)


@pytest.mark.parametrize("n,sigma", [(0, 4), (1, 1), (1, 2), (7, 1), (100, 2), (100, 3), (1000, 5), (4097, 146),
                                     (5000, 256), (3000, 1000), (2000, 65536), (70000, 300)])
def test_wm_closed_forms_random(n, sigma):
    S = gen.uniform_below(n, sigma, seed=7 * n + sigma,
                          dtype=np.uint8 if sigma <= 256 else (np.uint16 if sigma <= 65536 else np.uint32))
    _check(S, sigma)


def test_wm_sigma2_is_the_sequence():
    S = gen.uniform_below(3000, 2, seed=3, dtype=np.uint8)
    o = _check(S, 2)
    assert np.array_equal(o["bits"], pins.pack_bits(S.astype(np.uint8), pins.wpl(S.size)))


@pytest.mark.parametrize("shape", ["sorted", "descending", "constant"])
def test_wm_adversarial(shape):
    S = gen.uniform_below(2000, 256, seed=11, dtype=np.uint8)
    S = {"sorted": np.sort(S), "descending": np.sort(S)[::-1].copy(), "constant": np.full(2000, 77, np.uint8)}[shape]
    _check(S, 256)


def test_wm_queries_bruteforce():
    S = gen.uniform_below(3000, 37, seed=5, dtype=np.uint8)
    acc, rank = pins.wm_access_rank_bruteforce(S)
    rng = np.random.default_rng(1)
    pos = rng.integers(0, S.size, 400)
    sym = rng.integers(0, 37, 400)
    with oracle.OracleWM(S, 37) as m:
        assert list(m.access(pos)) == [acc(i) for i in pos]
        assert list(m.rank(sym, pos)) == [rank(c, i) for c, i in zip(sym, pos)]
        assert int(m.access([S.size])[0]) == 0xFFFFFFFF
        assert int(m.rank([3], [S.size])[0]) == 0xFFFFFFFFFFFFFFFF
        assert int(m.rank([37], [0])[0]) == 0xFFFFFFFFFFFFFFFF


def test_wm_exhaustive_tiny():
    count = 0
    for sigma in (1, 2, 3, 4):
        for n in range(0, 6):
            for seq in itertools.product(range(sigma), repeat=n):
                S = np.array(seq, dtype=np.uint8)
                _check(S, sigma)
                with oracle.OracleWM(S, sigma) as m:
                    if n:
                        assert list(m.access(range(n))) == list(seq)
                        for c in range(sigma):
                            assert list(m.rank([c] * n, range(n))) == [seq[:i + 1].count(c) for i in range(n)]
                count += 1
    assert count > 1000


def test_wm_rejects_out_of_range_symbol():
    with pytest.raises(oracle.OracleError) as e:
        oracle.wm_build(np.array([0, 4, 1], dtype=np.uint8), 4)
    assert e.value.code == oracle.ESYMBOL
