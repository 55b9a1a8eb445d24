"""Largest supported n (just under 2^32): positions, word and chain indices near
the 32-bit limit.  A periodic sequence makes every check closed-form: S[i] =
P[i mod 2^16] for a seeded pattern P over sigma = 4, so access(i) = P[i mod
2^16], rank_c(i) = (full periods) * count_P(c) + count in the partial period,
and the node table / level totals follow from the symbol counts."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import gen

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_n_near_2_32():
    import paper_1407_8142_b200 as wt
    free, total = torch.cuda.mem_get_info()
    if total < 64 << 30:
        pytest.skip("needs a large-memory GPU")
    P = gen.uniform_below(1 << 16, 4, seed=99, dtype=np.uint8)
    n = (1 << 32) - 4096 - 3
    reps = (n + (1 << 16) - 1) >> 16
    S = torch.from_numpy(P).cuda().repeat(reps)[:n].contiguous()
    t = wt.build(S, 4)
    assert t.n == n and t.levels == 2
    cnt = np.bincount(P, minlength=4).astype(np.int64)
    full, part = n >> 16, n & 0xFFFF
    tot = cnt * full + np.bincount(P[:part], minlength=4)
    # node table (closed form): level 0 root, level 1 the two halves
    ptr = t.level_node_ptr.cpu().numpy().astype(np.int64)
    keys = t.node_key.cpu().numpy().astype(np.int64)
    starts = t.node_start.cpu().numpy().astype(np.int64)
    assert ptr.tolist() == [0, 1, 3]
    assert keys.tolist() == [0, 0, 1] and starts.tolist() == [0, 0, int(tot[0] + tot[1])]
    # level totals (last superblock entries)
    spl = t.supers_per_level
    sup = t.rank_super.cpu().numpy().astype(np.int64)
    assert sup[spl - 1] == tot[2] + tot[3]      # level 0: symbols >= 2
    assert sup[2 * spl - 1] == tot[1] + tot[3]  # level 1: odd symbols
    # sampled access and rank, including the last positions
    rng = np.random.default_rng(5)
    pos = np.concatenate([rng.integers(0, n, 20000), np.arange(n - 70000, n), [0, (1 << 31) - 1, 1 << 31, n - 1]])
    acc = t.access(torch.from_numpy(pos.astype(np.int64)).cuda()).cpu().numpy()
    assert np.array_equal(acc, P[pos & 0xFFFF].astype(np.uint32))
    sym = rng.integers(0, 4, pos.size).astype(np.int32)
    got = t.rank(torch.from_numpy(sym).cuda(), torch.from_numpy(pos.astype(np.int64)).cuda()).cpu().numpy()
    pre = np.zeros((4, (1 << 16) + 1), dtype=np.int64)
    for c in range(4):
        pre[c, 1:] = np.cumsum(P == c)
    want = (pos >> 16) * cnt[sym] + pre[sym, (pos & 0xFFFF) + 1]
    assert np.array_equal(got.astype(np.int64), want)
    # select_c(k) (1-based k): full periods of the pattern plus the r-th occurrence in it
    occ = [np.nonzero(P == c)[0] for c in range(4)]
    ks = np.concatenate([rng.integers(1, tot[s] + 1, 500) for s in range(4)] + [tot[:4]])
    cs = np.concatenate([np.full(500, s) for s in range(4)] + [np.arange(4)]).astype(np.int64)
    sel = t.select(torch.from_numpy(cs.astype(np.int32)).cuda(), torch.from_numpy(ks.astype(np.int64)).cuda())
    q, r = (ks - 1) // cnt[cs], (ks - 1) % cnt[cs]
    want_sel = q * (1 << 16) + np.array([occ[c][i] for c, i in zip(cs, r)])
    assert np.array_equal(sel.cpu().numpy().astype(np.int64), want_sel)
    t.free()


def _closed_form_nodes(tot, L):
    """Node table of a tree whose symbol totals are tot (closed form)."""
    keys, starts, ptr = [], [], [0]
    cum = np.concatenate(([0], np.cumsum(tot)))
    for l in range(L):
        w = L - l
        for p in range(1 << l):
            lo, hi = p << w, (p + 1) << w
            if cum[hi] > cum[lo]:
                keys.append(p)
                starts.append(int(cum[lo]))
        ptr.append(len(keys))
    return ptr, keys, starts


@pytest.mark.parametrize("structure", ["tree", "matrix"])
def test_n_near_2_32_sigma_2_16(structure):
    import paper_1407_8142_b200 as wt
    free, total = torch.cuda.mem_get_info()
    if total < 120 << 30:
        pytest.skip("needs a large-memory GPU")
    sigma, L = 1 << 16, 16
    P = gen.uniform_below(1 << 16, sigma, seed=7, dtype=np.uint16)
    n = (1 << 32) - 12345
    reps = (n + (1 << 16) - 1) >> 16
    S = torch.from_numpy(P.view(np.int16)).cuda().repeat(reps)[:n].contiguous()
    t = wt.build(S, sigma) if structure == "tree" else wt.wm_build(S, sigma)
    cnt = np.bincount(P, minlength=sigma).astype(np.int64)
    full, part = n >> 16, n & 0xFFFF
    tot = cnt * full + np.bincount(P[:part], minlength=sigma)
    if structure == "tree":
        ptr, keys, starts = _closed_form_nodes(tot, L)
        assert t.level_node_ptr.cpu().numpy().astype(np.int64).tolist() == ptr
        assert np.array_equal(t.node_key.cpu().numpy().astype(np.int64), np.array(keys))
        assert np.array_equal(t.node_start.cpu().numpy().astype(np.int64), np.array(starts))
    else:
        sym = np.arange(sigma)
        zeros = [int(tot[((sym >> (L - 1 - l)) & 1) == 0].sum()) for l in range(L)]
        assert t.zeros.cpu().numpy().astype(np.int64).tolist() == zeros
    rng = np.random.default_rng(11)
    pos = np.concatenate([rng.integers(0, n, 20000), np.arange(n - 5000, n), [(1 << 31) - 1, 1 << 31]])
    acc = t.access(torch.from_numpy(pos.astype(np.int64)).cuda()).cpu().numpy()
    assert np.array_equal(acc, P[pos & 0xFFFF].astype(np.uint32))
    sy = P[rng.integers(0, 1 << 16, pos.size)].astype(np.int64)
    got = t.rank(torch.from_numpy(sy.astype(np.int32)).cuda(), torch.from_numpy(pos.astype(np.int64)).cuda()).cpu().numpy()
    # partial-period counts by sorting the pattern positions of each symbol
    order = np.argsort(P, kind="stable")
    first = np.searchsorted(P[order], sy)
    last = np.searchsorted(P[order], sy, side="right")
    inpart = np.array([np.searchsorted(order[a:b], r, side="right") for a, b, r in zip(first, last, pos & 0xFFFF)])
    want = (pos >> 16) * cnt[sy] + inpart
    assert np.array_equal(got.astype(np.int64), want)
    t.free()


def test_hwt_n_near_2_32():
    import paper_1407_8142_b200 as wt
    free, total = torch.cuda.mem_get_info()
    if total < 64 << 30:
        pytest.skip("needs a large-memory GPU")
    # skewed 8-symbol pattern: codes of lengths 1..7
    P = np.minimum(np.random.default_rng(3).geometric(0.5, 1 << 16) - 1, 7).astype(np.uint8)
    n = (1 << 32) - 999
    reps = (n + (1 << 16) - 1) >> 16
    S = torch.from_numpy(P).cuda().repeat(reps)[:n].contiguous()
    t = wt.hwt_build(S, 8)
    cnt = np.bincount(P, minlength=8).astype(np.int64)
    tot = cnt * (n >> 16) + np.bincount(P[:n & 0xFFFF], minlength=8)
    ln = t.code_len.cpu().numpy().astype(np.int64)
    assert t.total_bits == int((tot * ln).sum())
    assert t.level_len.cpu().numpy().astype(np.int64).tolist() == [int(tot[ln > l].sum()) for l in range(t.levels)]
    rng = np.random.default_rng(12)
    pos = np.concatenate([rng.integers(0, n, 20000), np.arange(n - 3000, n)])
    acc = t.access(torch.from_numpy(pos.astype(np.int64)).cuda()).cpu().numpy()
    assert np.array_equal(acc, P[pos & 0xFFFF].astype(np.uint32))
    sy = rng.integers(0, 8, pos.size).astype(np.int64)
    got = t.rank(torch.from_numpy(sy.astype(np.int32)).cuda(), torch.from_numpy(pos.astype(np.int64)).cuda()).cpu().numpy()
    pre = np.zeros((8, (1 << 16) + 1), dtype=np.int64)
    for c in range(8):
        pre[c, 1:] = np.cumsum(P == c)
    assert np.array_equal(got.astype(np.int64), (pos >> 16) * cnt[sy] + pre[sy, (pos & 0xFFFF) + 1])
    t.free()


def test_sigma1_validation_beyond_2_31():
    """sigma = 1 (0 levels): validation alone; a nonzero symbol past position
    2^31 must still give WT_ESYMBOL (tree and matrix)."""
    import paper_1407_8142_b200 as wt
    free, total = torch.cuda.mem_get_info()
    if total < 32 << 30:
        pytest.skip("needs a large-memory GPU")
    n = (1 << 31) + 12345
    S = torch.zeros(n, dtype=torch.uint8, device="cuda")
    t = wt.build(S, 1)
    assert t.n == n and t.levels == 0
    t.free()
    S[(1 << 31) + 777] = 1
    for build in (wt.build, wt.wm_build):
        with pytest.raises(wt.WtError) as e:
            build(S, 1)
        assert e.value.code == -2  # WT_ESYMBOL
    del S
