"""Pin the CPU oracle to things other than itself (CPU-only).

Every check below compares oracle output with something the paper or the
mathematics fixes: hand-derived worked examples (tests/golden/), the sortWT
closed form (Fig. 2), a prefix-counting form, lower_bound node starts, a
brute-force rank directory, brute-force access/rank, invariants, and an
exhaustive sweep of all sequences with n <= 6, sigma <= 4.
"""
from __future__ import annotations

import itertools
import os

import numpy as np
import pytest

import gen
import oracle
from tests import pins

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _parse_golden(path):
    d = {}
    for line in open(path):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        k, v = [x.strip() for x in line.split("=", 1)]
        d[k] = v
    return d


def _check_against_closed_forms(S, sigma):
    S = np.asarray(S)
    o = oracle.build(S, sigma)
    n = S.size
    L = pins.levels_of(sigma)
    assert o["levels"] == L
    bits_sort, nodes_sort = pins.sortwt(S, sigma)
    assert np.array_equal(o["bits"], bits_sort), "bitmaps differ from sortWT (Fig. 2)"
    got_nodes = pins.nodes_from_csr(o)
    assert got_nodes == nodes_sort, "nodes differ from Fig. 2 boundary filter"
    assert got_nodes == pins.nodes_lower_bound(S, sigma)
    blk, sup = pins.rank_directory_bruteforce(o["bits"], n, L)
    assert np.array_equal(o["rank_block"], blk)
    assert np.array_equal(o["rank_super"], sup)
    return o


@pytest.mark.parametrize("fname", sorted(os.listdir(GOLDEN)))
def test_golden_examples(fname):
    g = _parse_golden(os.path.join(GOLDEN, fname))
    S = np.array([int(x) for x in g["S"].split()], dtype=np.uint32)
    sigma = int(g["sigma"])
    L = int(g["levels"])
    with oracle.OracleTree(S, sigma) as t:
        a = t.arrays()
        assert t.levels == L
        W = t.words_per_level
        for l in range(L):
            want = [int(x) for x in g[f"bits_level{l}"].split()]
            word = int(a["bits"][l * W])
            got = [(word >> i) & 1 for i in range(len(S))]
            assert got == want, f"level {l} bits"
            assert word == int(g[f"word0_level{l}"], 16)
            assert all(int(a["bits"][l * W + w]) == 0 for w in range(1, W)), "padding must be 0"
            nodes = pins.nodes_from_csr(a)[l]
            want_nodes = [tuple(int(y) for y in x.split(":")) for x in g[f"nodes_level{l}"].split()]
            assert nodes == want_nodes, f"level {l} nodes"
            SPL = t.supers_per_level
            sup = a["rank_super"][l * SPL:(l + 1) * SPL].tolist()
            assert sup == [int(x) for x in g[f"rank_super_level{l}"].split()]
            if f"rank_block_level{l}" in g:
                BPL = t.blocks_per_level
                assert a["rank_block"][l * BPL:(l + 1) * BPL].tolist() == \
                    [int(x) for x in g[f"rank_block_level{l}"].split()]
        for item in g["access"].split():
            i, v = map(int, item.split(":"))
            assert int(t.access([i])[0]) == v
        for item in g["rank"].split():
            ci, v = item.split(":")
            c, i = map(int, ci.split("@"))
            assert int(t.rank([c], [i])[0]) == int(v)


def test_spec_node_id_example():
    """SPEC.md:273 [PAPER Fig. 2 l.13]: l=2, L=8, symbol 0b11000001 -> id 6."""
    S = np.array([0b11000001, 3, 77], dtype=np.uint8)
    a = oracle.build(S, 256)
    keys_l2 = pins.nodes_from_csr(a)[2]
    key = 0b11000001 >> (8 - 2)
    assert (key, 2) in keys_l2  # sorted by prefix: 3 (key 0), 77 (key 1), 193 (key 3)
    assert (1 << 2) - 1 + key == 6


def test_exhaustive_tiny():
    """All sequences with n <= 6 over sigma <= 4 (and sigma = 3, 1)."""
    count = 0
    for sigma in (1, 2, 3, 4):
        for n in range(0, 7 if sigma <= 3 else 7):
            for seq in itertools.product(range(sigma), repeat=n):
                S = np.array(seq, dtype=np.uint8)
                o = _check_against_closed_forms(S, sigma)
                with oracle.OracleTree(S, sigma) as t:
                    for i in range(n):
                        assert int(t.access([i])[0]) == seq[i]
                        for c in range(sigma):
                            assert int(t.rank([c], [i])[0]) == pins.rank_bruteforce(S, c, i)
                count += 1
                del o
    assert count == sum(s ** n for s in (1, 2, 3, 4) for n in range(7))


@pytest.mark.parametrize("sigma", [2, 3, 5, 8, 146, 256, 1000, 65536, 1 << 20])
@pytest.mark.parametrize("n", [0, 1, 2, 63, 64, 65, 511, 512, 513, 1000, 4097])
def test_random_vs_closed_forms(n, sigma):
    S = gen.uniform_below(n, sigma, seed=n * 7919 + sigma, dtype=np.uint32)
    o = _check_against_closed_forms(S, sigma)
    if n <= 1200:
        assert np.array_equal(o["bits"], pins.prefix_counting_bits(S, sigma))


def test_prefix_counting_larger():
    S = gen.zipf_permuted(3000, seed=11)
    o = oracle.build(S, 256)
    assert np.array_equal(o["bits"], pins.prefix_counting_bits(S, 256))


def test_directory_across_superblocks():
    """n spans several 2^16-bit superblocks with a ragged tail."""
    n = 3 * 65536 + 1234
    S = gen.uniform_bits(n, 3, seed=9, dtype=np.uint8)
    _check_against_closed_forms(S, 8)


def test_queries_bruteforce_random():
    n, sigma = 5000, 300
    S = gen.uniform_below(n, sigma, seed=5, dtype=np.uint32)
    rng = np.random.default_rng(0)
    with oracle.OracleTree(S, sigma) as t:
        pos = rng.integers(0, n, 500)
        assert np.array_equal(t.access(pos), S[pos])
        cs = rng.integers(0, sigma, 500)
        want = [pins.rank_bruteforce(S, c, i) for c, i in zip(cs, pos)]
        assert t.rank(cs, pos).tolist() == want
        # out-of-range conventions
        assert int(t.access([n])[0]) == 0xFFFFFFFF
        assert int(t.rank([sigma], [0])[0]) == 0xFFFFFFFFFFFFFFFF


def test_invariants_children_sum_and_popcount():
    """Fig. 1 l.18-19: children sizes sum to the parent; the parent's bitmap
    popcount equals the right child's size; level popcount = #{bit set}."""
    n, sigma = 20000, 1000
    S = gen.uniform_below(n, sigma, seed=3, dtype=np.uint32)
    a = oracle.build(S, sigma)
    L = a["levels"]
    W = a["words_per_level"]
    levels = pins.nodes_from_csr(a)
    for l in range(L):
        words = a["bits"][l * W:(l + 1) * W]
        bl = np.unpackbits(words.view(np.uint8), bitorder="little")[:n]
        assert int(bl.sum()) == int(np.count_nonzero((S >> (L - 1 - l)) & 1))
        starts = [s for _, s in levels[l]] + [n]
        for j, (p, s) in enumerate(levels[l]):
            e = starts[j + 1]
            ones = int(bl[s:e].sum())
            if l + 1 < L:
                ch = {k: st for k, st in levels[l + 1]}
                nxt = sorted(levels[l + 1])
                nstarts = dict()
                for jj, (k, st) in enumerate(nxt):
                    nstarts[k] = (st, nxt[jj + 1][1] if jj + 1 < len(nxt) else n)
                lsz = (nstarts[2 * p][1] - nstarts[2 * p][0]) if 2 * p in ch else 0
                rsz = (nstarts[2 * p + 1][1] - nstarts[2 * p + 1][0]) if 2 * p + 1 in ch else 0
                assert lsz + rsz == e - s
                assert rsz == ones


def test_special_cases():
    # sigma = 2: the single bitmap equals S
    S = gen.uniform_bits(777, 1, seed=1, dtype=np.uint8)
    a = oracle.build(S, 2)
    assert np.array_equal(a["bits"], pins.pack_bits(S, pins.wpl(777)))
    # sorted input: S_l = S for every l, so B_l[i] = bit of S[i]
    S = np.sort(gen.uniform_below(3000, 200, seed=2, dtype=np.uint32))
    a = oracle.build(S, 200)
    L, W = 8, pins.wpl(3000)
    for l in range(L):
        assert np.array_equal(a["bits"][l * W:(l + 1) * W],
                              pins.pack_bits((S >> (L - 1 - l)) & 1, W))
    # constant input: one node per level, all words equal in the body
    S = np.full(1000, 173, dtype=np.uint8)
    a = oracle.build(S, 256)
    assert a["total_nodes"] == 8
    # sigma = 1: no levels; n = 0: empty levels with one super entry
    a = oracle.build(np.zeros(5, np.uint8), 1)
    assert a["levels"] == 0 and a["bits"].size == 0
    with oracle.OracleTree(np.zeros(5, np.uint8), 1) as t:
        assert t.access([3]).tolist() == [0]
        assert t.rank([0], [3]).tolist() == [4]
    a = oracle.build(np.zeros(0, np.uint32), 1000)
    assert a["bits"].size == 0 and a["rank_super"].tolist() == [0] * 10
    assert a["level_node_ptr"].tolist() == [0] * 11


def test_errors():
    with pytest.raises(oracle.OracleError) as e:
        oracle.build(np.array([0, 5, 1], np.uint8), 5)
    assert e.value.code == oracle.ESYMBOL
    with pytest.raises(oracle.OracleError) as e:
        oracle.build(np.array([0], np.uint8), 257)
    assert e.value.code == oracle.EINVAL


def test_fault_injection_detected():
    """A single flipped bitmap bit must be caught by the sortWT comparison."""
    S = gen.uniform_below(4096, 256, seed=17, dtype=np.uint8)
    a = oracle.build(S, 256)
    bits, _ = pins.sortwt(S, 256)
    assert np.array_equal(a["bits"], bits)
    bad = a["bits"].copy()
    bad[3 * pins.wpl(4096) + 17] ^= np.uint64(1 << 9)
    assert not np.array_equal(bad, bits)


def test_generators_deterministic():
    a = gen.config_input(gen.CONFIGS[4], 1000)
    b = gen.config_input(gen.CONFIGS[4], 1000)
    assert np.array_equal(a, b) and a.dtype == np.uint32 and int(a.max()) < 65536
    z = gen.config_input(gen.CONFIGS[3], 1 << 18)
    freq = np.bincount(z, minlength=256) / z.size
    assert abs(freq.max() - 0.2065) < 0.005  # H_{256,1.1} p_max
    assert (freq > 0).all()
    # prefix property: a shorter draw is a prefix of the longer one
    assert np.array_equal(gen.config_input(gen.CONFIGS[1], 100), gen.config_input(gen.CONFIGS[1])[:100])
