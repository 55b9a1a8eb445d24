"""Pin the oracle's select and sampled select directory
(Clark's first level) for both the tree and
the matrix: brute-force positions of occurrences, brute-force filtered bit
positions, the rank/select identities, and exhaustive tiny inputs."""
from __future__ import annotations

import itertools

import numpy as np
import pytest

import gen
import oracle
from tests import pins

SAMPLE = 4096
MAX = 0xFFFFFFFFFFFFFFFF


def _bits_of(o, l, n):
    W = pins.wpl(n)
    words = o["bits"][l * W:(l + 1) * W]
    return np.array([(int(words[i >> 6]) >> (i & 63)) & 1 for i in range(n)], dtype=np.uint8)


def _dir_bruteforce(o, n, L):
    sps = (n + SAMPLE - 1) // SAMPLE + 1
    s0 = np.full(L * sps, n, dtype=np.uint32)
    s1 = np.full(L * sps, n, dtype=np.uint32)
    for l in range(L):
        b = _bits_of(o, l, n)
        z = np.nonzero(b == 0)[0][::SAMPLE]
        one = np.nonzero(b == 1)[0][::SAMPLE]
        s0[l * sps:l * sps + z.size] = z
        s1[l * sps:l * sps + one.size] = one
    return s0, s1, sps


def _check(S, sigma, kind):
    S = np.asarray(S)
    n, L = S.size, pins.levels_of(sigma)
    cls = oracle.OracleTree if kind == "wt" else oracle.OracleWM
    with cls(S, sigma) as t:
        o = t.arrays()
        d = t.select_dir()
        s0, s1, sps = _dir_bruteforce(o, n, L)
        assert d["select_per_level"] == sps
        assert np.array_equal(d["select0"], s0) and np.array_equal(d["select1"], s1)
        cs, ks, want = [], [], []
        for c in range(min(sigma, 40)):
            occ = np.nonzero(S == c)[0]
            for k in sorted({1, 2, occ.size, occ.size + 1, SAMPLE, SAMPLE + 1, occ.size // 2 + 1}):
                cs.append(c)
                ks.append(k)
                want.append(int(occ[k - 1]) if 1 <= k <= occ.size else MAX)
        cs += [0, sigma]
        ks += [0, 1]
        want += [MAX, MAX]
        got = t.select(cs, ks)
        assert [int(x) for x in got] == want
        # identities: S[select_c(k)] == c and rank_c(select_c(k)) == k
        ok = [(c, k, g) for c, k, g in zip(cs, ks, got) if int(g) != MAX]
        if ok:
            assert all(int(S[int(g)]) == c for c, k, g in ok)
            r = t.rank([c for c, _, _ in ok], [int(g) for _, _, g in ok])
            assert [int(x) for x in r] == [k for _, k, _ in ok]


@pytest.mark.parametrize("kind", ["wt", "wm"])
@pytest.mark.parametrize("n,sigma", [(0, 4), (1, 1), (50, 1), (9000, 2), (20000, 3), (30000, 5), (12345, 256),
                                     (5000, 1000)])
def test_select_random(kind, n, sigma):
    S = gen.uniform_below(n, sigma, seed=n + 13 * sigma, dtype=np.uint8 if sigma <= 256 else np.uint16)
    _check(S, sigma, kind)


@pytest.mark.parametrize("kind", ["wt", "wm"])
def test_select_skewed(kind):
    S = gen.zipf_permuted(40000, 3, dtype=np.uint8)
    _check(S, 256, kind)


@pytest.mark.parametrize("kind", ["wt", "wm"])
def test_select_exhaustive_tiny(kind):
    cls = oracle.OracleTree if kind == "wt" else oracle.OracleWM
    for sigma in (1, 2, 3, 4):
        for n in range(0, 5):
            for seq in itertools.product(range(sigma), repeat=n):
                S = np.array(seq, dtype=np.uint8)
                with cls(S, sigma) as t:
                    for c in range(sigma):
                        occ = [i for i, v in enumerate(seq) if v == c]
                        got = t.select([c] * (len(occ) + 1), list(range(1, len(occ) + 2)))
                        assert [int(x) for x in got] == occ + [MAX]
