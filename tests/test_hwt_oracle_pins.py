"""Pin the CPU oracle's Huffman-shaped wavelet tree (PAPER.md:854-876,
SURVEY §8(f) f3; readings R-17..R-20 in DESIGN.md).

The oracle (oracle/wt_oracle.c, oracle_hwt_build) builds the Huffman tree by
the two-queue method, the canonical codes, the in-order mapping with one
threshold per internal node, and the levels with levelWT's prefix-sum split
(:862-873).  It is checked here against things other than itself:

* hand-derived worked examples and the textbook Huffman example
  (tests/golden_hwt/);
* optimality: the code cost equals the minimum over ALL length vectors that
  satisfy Kraft's inequality (exhaustive enumeration), and Kraft's sum is 1;
* the canonical-code properties (prefix-free, ordered by (length, symbol));
* a sort characterisation of every level (pins.hwt_closed_form) and the
  total-bits identity sum_l n_l = sum_c f_c len_c;
* a running-popcount rank directory per level; brute-force access / rank_c;
* exhaustive tiny inputs, degenerate inputs and the error paths.
"""
from __future__ import annotations

import itertools
import os

import numpy as np
import pytest

import gen
import oracle
from tests import pins

GOLDEN = os.path.join(os.path.dirname(__file__), "golden_hwt")


def _parse(path):
    d = {}
    for line in open(path):
        line = line.strip()
        if line and not line.startswith("#"):
            k, v = [x.strip() for x in line.split("=", 1)]
            d[k] = v
    return d


def _ints(s):
    return [int(x) for x in s.split()]


def _level_bits(o, l):
    lo, hi = int(o["level_word_ptr"][l]), int(o["level_word_ptr"][l + 1])
    n = int(o["level_len"][l])
    return np.unpackbits(o["bits"][lo:hi].view(np.uint8), bitorder="little")[:n]


def check_hwt(S, sigma, o=None):
    """Every independent pin on one input; returns the oracle dict."""
    S = np.asarray(S)
    o = o if o is not None else oracle.hwt_build(S, sigma)
    freq = np.bincount(S.astype(np.int64), minlength=sigma)[:sigma] if S.size else np.zeros(sigma, np.int64)
    ln = o["code_len"].astype(np.int64)
    cd = o["code"].astype(np.int64)
    m = int(np.count_nonzero(freq))
    assert np.array_equal(ln > 0, (freq > 0) & (m >= 2))
    h = int(ln.max()) if m >= 2 else 0
    assert o["levels"] == h
    if m >= 2:
        # Kraft equality (a full binary tree) and monotonicity in (freq, sym) order
        assert sum(2.0 ** -int(x) for x in ln[ln > 0]) == pytest.approx(1.0, abs=1e-12)
        order = sorted(np.nonzero(freq)[0], key=lambda c: (freq[c], c))
        assert all(ln[a] >= ln[b] for a, b in zip(order, order[1:]))
        # canonical: by (len, sym) the left-aligned codes increase by exactly one ulp of the shorter code
        syms = sorted(np.nonzero(ln)[0], key=lambda c: (ln[c], c))
        assert cd[syms[0]] == 0
        for a, b in zip(syms, syms[1:]):
            assert cd[b] == (cd[a] + 1) << (ln[b] - ln[a])
        assert cd[syms[-1]] == (1 << ln[syms[-1]]) - 1
        # prefix-free
        for a, b in itertools.combinations(syms[:64], 2):
            la, lb = ln[a], ln[b]
            if la <= lb:
                assert (cd[b] >> (lb - la)) != cd[a]
            else:
                assert (cd[a] >> (la - lb)) != cd[b]
    # levels by the sort characterisation
    lv, nodes = pins.hwt_closed_form(S, cd, ln) if m >= 2 else ([], [])
    assert len(lv) == h
    assert np.array_equal(o["level_len"], np.array([x.size for x in lv], dtype=np.uint64))
    assert int(o["level_len"].sum()) == int((freq * ln).sum())  # total bits = code cost
    for l in range(h):
        assert np.array_equal(_level_bits(o, l), lv[l]), f"level {l}"
        lo, hi = int(o["level_word_ptr"][l]), int(o["level_word_ptr"][l + 1])
        assert hi - lo == pins.wpl(lv[l].size)
        pad = np.unpackbits(o["bits"][lo:hi].view(np.uint8), bitorder="little")[lv[l].size:]
        assert not pad.any()
        a, b = int(o["level_node_ptr"][l]), int(o["level_node_ptr"][l + 1])
        got = list(zip(o["node_key"][a:b].tolist(), o["node_start"][a:b].tolist()))
        assert got == nodes[l], f"nodes of level {l}"
        blk, sup = pins.rank_directory_one_level(o["bits"][lo:hi], lv[l].size)
        b0, b1 = int(o["level_block_ptr"][l]), int(o["level_block_ptr"][l + 1])
        s0, s1 = int(o["level_super_ptr"][l]), int(o["level_super_ptr"][l + 1])
        assert np.array_equal(o["rank_block"][b0:b1], blk)
        assert np.array_equal(o["rank_super"][s0:s1], sup)
    return o


def _queries(S, sigma, t, k=200, seed=0):
    rng = np.random.default_rng(seed)
    n = len(S)
    if n == 0:
        assert t.access([0])[0] == 0xFFFFFFFF
        return
    pos = rng.integers(0, n, size=k)
    assert np.array_equal(t.access(pos), np.asarray(S)[pos].astype(np.uint32))
    syms = rng.integers(0, sigma, size=k)
    exp = [pins.rank_bruteforce(S, int(c), int(i)) for c, i in zip(syms, pos)]
    assert t.rank(syms, pos).tolist() == exp
    assert t.access([n])[0] == 0xFFFFFFFF
    assert t.rank([0], [n])[0] == 2**64 - 1
    assert t.rank([sigma], [0])[0] == 2**64 - 1
    # select_c(k): the k'th occurrence by brute force; k = 0 / too large / c >= sigma -> UINT64_MAX
    S = np.asarray(S)
    cs = rng.integers(0, sigma, size=k // 4)
    cs[: min(len(cs), 50)] = S[rng.integers(0, n, size=min(len(cs), 50))]
    ks = rng.integers(0, 20, size=cs.size)
    exp = []
    for c, kk in zip(cs, ks):
        occ = np.nonzero(S == c)[0]
        exp.append(int(occ[kk - 1]) if 1 <= kk <= occ.size else 2**64 - 1)
    assert t.select(cs, ks).tolist() == exp
    assert t.select([sigma], [1])[0] == 2**64 - 1


@pytest.mark.parametrize("fname", sorted(os.listdir(GOLDEN)))
def test_hwt_golden(fname):
    g = _parse(os.path.join(GOLDEN, fname))
    sigma = int(g["sigma"])
    if "S" in g:
        S = np.array(_ints(g["S"]), dtype=np.uint8)
    else:
        S = np.repeat(np.arange(sigma, dtype=np.uint8), _ints(g["freq"]))
    o = oracle.hwt_build(S, sigma)
    assert o["code_len"].tolist() == _ints(g["code_len"])
    assert o["code"].tolist() == _ints(g["code"])
    assert o["levels"] == int(g["levels"])
    assert o["level_len"].tolist() == _ints(g["level_len"])
    if "cost" in g:
        freq = np.bincount(S, minlength=sigma)
        assert int((freq * o["code_len"].astype(np.int64)).sum()) == int(g["cost"])
        assert pins.huffman_cost_bruteforce(freq) == int(g["cost"])
    for l in range(o["levels"]):
        if f"bits_level{l}" in g:
            assert _level_bits(o, l).tolist() == _ints(g[f"bits_level{l}"])
        if f"nodes_level{l}" in g:
            a, b = int(o["level_node_ptr"][l]), int(o["level_node_ptr"][l + 1])
            exp = [tuple(int(y) for y in x.split(":")) for x in g[f"nodes_level{l}"].split()]
            assert list(zip(o["node_key"][a:b].tolist(), o["node_start"][a:b].tolist())) == exp
    with oracle.OracleHWT(S, sigma) as t:
        for item in g.get("access", "").split():
            i, v = map(int, item.split(":"))
            assert t.access([i])[0] == v
        for item in g.get("rank", "").split():
            ci, v = item.split(":")
            c, i = map(int, ci.split("@"))
            assert t.rank([c], [i])[0] == int(v)
        for item in g.get("select", "").split():
            ck, v = item.split(":")
            c, kk = map(int, ck.split("#"))
            assert t.select([c], [kk])[0] == int(v)
    check_hwt(S, sigma, o)


@pytest.mark.parametrize("seed", range(40))
def test_hwt_optimal_cost(seed):
    rng = np.random.default_rng(seed)
    m = int(rng.integers(2, 7))
    freq = rng.integers(1, 30, size=m)
    if seed % 4 == 0:
        freq[:] = freq[0]  # all ties
    S = np.repeat(np.arange(m, dtype=np.uint8), freq)
    rng.shuffle(S)
    o = check_hwt(S, m)
    assert int((freq * o["code_len"].astype(np.int64)).sum()) == pins.huffman_cost_bruteforce(freq)


def test_hwt_exhaustive_tiny():
    cnt = 0
    for sigma in (1, 2, 3, 4):
        for n in range(0, 6):
            for S in itertools.product(range(sigma), repeat=n):
                S = np.array(S, dtype=np.uint8)
                check_hwt(S, sigma)
                with oracle.OracleHWT(S, sigma) as t:
                    for i in range(n):
                        assert t.access([i])[0] == S[i]
                        for c in range(sigma):
                            assert t.rank([c], [i])[0] == pins.rank_bruteforce(S, c, i)
                    for c in range(sigma):
                        occ = np.nonzero(S == c)[0]
                        for kk in range(0, n + 2):
                            want = int(occ[kk - 1]) if 1 <= kk <= occ.size else 2**64 - 1
                            assert t.select([c], [kk])[0] == want
                cnt += 1
    assert cnt > 1000


@pytest.mark.parametrize("dist,sigma,n,dtype", [
    ("uniform", 256, 20000, np.uint8),
    ("zipf", 256, 30000, np.uint8),
    ("uniform", 3000, 40000, np.uint16),
    ("geometric", 40, 1 << 16, np.uint8),
    ("uniform", 65536, 70000, np.uint32),
    ("uniform", 7, 1000, np.uint32),
])
def test_hwt_random(dist, sigma, n, dtype):
    rng = np.random.default_rng(sigma + n)
    if dist == "uniform":
        S = rng.integers(0, sigma, size=n).astype(dtype)
    elif dist == "zipf":
        S = gen.zipf_permuted(n, 3)
    else:
        S = np.minimum(rng.geometric(0.3, size=n) - 1, sigma - 1).astype(dtype)
    S = S.astype(dtype)
    check_hwt(S, sigma)
    with oracle.OracleHWT(S, sigma) as t:
        _queries(S, sigma, t)


def test_hwt_degenerate():
    # n = 0
    o = check_hwt(np.zeros(0, np.uint8), 4)
    assert o["levels"] == 0 and o["total_nodes"] == 0
    # one distinct symbol (R-20): 0 levels; queries still answer
    S = np.full(1000, 3, np.uint8)
    o = check_hwt(S, 5)
    assert o["levels"] == 0 and o["only_symbol"] == 3
    with oracle.OracleHWT(S, 5) as t:
        assert t.access([0, 999]).tolist() == [3, 3]
        assert t.rank([3, 0, 4], [10, 10, 999]).tolist() == [11, 0, 0]
        assert t.select([3, 3, 3, 0], [1, 1000, 1001, 1]).tolist() == [0, 999, 2**64 - 1, 2**64 - 1]
    # two symbols: one level, the bitmap is the sequence (0 -> code 0 by R-18)
    S = np.array([1, 0, 1, 1, 0], np.uint8)
    o = check_hwt(S, 2)
    assert o["levels"] == 1 and _level_bits(o, 0).tolist() == [1, 0, 1, 1, 0]
    # absent symbols inside the alphabet get no code; rank answers 0
    S = np.array([0, 5, 5, 9, 0, 0], np.uint8)
    o = check_hwt(S, 10)
    with oracle.OracleHWT(S, 10) as t:
        assert t.rank([3, 5], [5, 5]).tolist() == [0, 2]


def test_hwt_fibonacci_depth():
    # Fibonacci weights force a path-shaped Huffman tree: depth m - 1.
    fib = [1, 1]
    while len(fib) < 20:
        fib.append(fib[-1] + fib[-2])
    S = np.repeat(np.arange(20, dtype=np.uint8), fib)
    o = check_hwt(S, 20)
    assert o["levels"] == 19
    assert sorted(o["code_len"].tolist()) == sorted([19, 19] + list(range(1, 19)))


def test_hwt_errors():
    with pytest.raises(oracle.OracleError) as e:
        oracle.hwt_build(np.array([0, 4], np.uint8), 4)
    assert e.value.code == oracle.ESYMBOL
    with pytest.raises(oracle.OracleError) as e:
        oracle.hwt_build(np.array([0, 1], np.uint32), 1 << 17)
    assert e.value.code == oracle.EINVAL


@pytest.mark.slow
def test_hwt_too_deep():
    # 34 Fibonacci weights: depth 33 > 32 -> unsupported (R-20)
    fib = [1, 1]
    while len(fib) < 34:
        fib.append(fib[-1] + fib[-2])
    S = np.repeat(np.arange(34, dtype=np.uint8), fib)
    with pytest.raises(oracle.OracleError) as e:
        oracle.hwt_build(S, 34)
    assert e.value.code == oracle.EUNSUPPORTED
