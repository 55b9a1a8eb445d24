"""Independent closed forms used to pin the oracle (and, transitively, the GPU path).

None of these share code with oracle/ or with the CUDA library.  Each is a
different characterisation of the same result:

* ``sortwt``        -- PAPER.md Fig. 2 (sortWT): level l is S
                       stably sorted by its top l bits;
                       bits from bit L-1-l; node starts by a filter on prefix
                       changes (Fig. 2 l.11).
* ``prefix_counting`` -- position of element x at level l is
                       C_l(p) + #{earlier elements with the same prefix p},
                       C_l(p) = #{y : y >> (L-l) < p}; computed with a
                       per-prefix cursor loop (no sorting at all).
* ``nodes_lower_bound`` -- node starts = lower_bound(sorted(S), p << (L-l)).
* ``rank_directory_bruteforce`` -- a running popcount, sampled per R-9.
* brute-force access / rank_c.
"""
from __future__ import annotations

import numpy as np


def levels_of(sigma: int) -> int:
    return (int(sigma) - 1).bit_length()


def pack_bits(bitarr: np.ndarray, words_per_level: int) -> np.ndarray:
    """LSB-first packing of a 0/1 array into words_per_level u64 words."""
    out = np.zeros(words_per_level, dtype=np.uint64)
    idx = np.nonzero(bitarr)[0]
    np.bitwise_or.at(out, idx >> 6, np.left_shift(np.uint64(1), (idx & 63).astype(np.uint64)))
    return out


def wpl(n: int) -> int:
    return ((n + 511) // 512) * 8


def sortwt(S: np.ndarray, sigma: int):
    """Fig. 2: returns (bits [L*WPL] u64, per-level list of (key, start))."""
    S = np.asarray(S).astype(np.uint64)
    n = S.size
    L = levels_of(sigma)
    W = wpl(n)
    bits = np.zeros(L * W, dtype=np.uint64)
    nodes = []
    for l in range(L):
        prefix = S >> np.uint64(L - l)
        Sl = S[np.argsort(prefix, kind="stable")]  # Fig. 2 l.9
        b = (Sl >> np.uint64(L - 1 - l)) & np.uint64(1)  # Fig. 2 l.10
        bits[l * W:(l + 1) * W] = pack_bits(b, W)
        pl = Sl >> np.uint64(L - l)
        if n:
            O = np.nonzero(np.concatenate(([True], pl[1:] != pl[:-1])))[0]  # Fig. 2 l.11
            nodes.append([(int(pl[o]), int(o)) for o in O])
        else:
            nodes.append([])
    return bits, nodes


def prefix_counting_bits(S, sigma: int) -> np.ndarray:
    """Bits via per-prefix cursors; no sort, no recursion (plain loops)."""
    S = [int(x) for x in S]
    n = len(S)
    L = levels_of(sigma)
    W = wpl(n)
    bits = np.zeros(L * W, dtype=np.uint64)
    for l in range(L):
        cnt = {}
        for x in S:
            p = x >> (L - l)
            cnt[p] = cnt.get(p, 0) + 1
        cursor, acc = {}, 0
        for p in sorted(cnt):
            cursor[p] = acc
            acc += cnt[p]
        for x in S:
            p = x >> (L - l)
            pos = cursor[p]
            cursor[p] += 1
            if (x >> (L - 1 - l)) & 1:
                bits[l * W + (pos >> 6)] |= np.uint64(1) << np.uint64(pos & 63)
    return bits


def nodes_lower_bound(S, sigma: int):
    S = np.sort(np.asarray(S).astype(np.uint64), kind="stable")
    L = levels_of(sigma)
    out = []
    for l in range(L):
        ps = np.unique(S >> np.uint64(L - l))
        out.append([(int(p), int(np.searchsorted(S, np.uint64(p) << np.uint64(L - l), side="left")))
                    for p in ps])
    return out


def rank_directory_bruteforce(bits: np.ndarray, n: int, L: int):
    """R-9: super[s] = ones in [0, min(s*2^16, n)); block[b] = ones in
    [floor(b/128)*2^16, b*512)."""
    W = wpl(n)
    BPL = (n + 511) // 512
    SPL = (n + 65535) // 65536 + 1
    blk = np.zeros(L * BPL, dtype=np.uint16)
    sup = np.zeros(L * SPL, dtype=np.uint64)
    for l in range(L):
        words = bits[l * W:(l + 1) * W]
        b = np.unpackbits(words.view(np.uint8), bitorder="little")[:n].astype(np.int64)
        pre = np.concatenate(([0], np.cumsum(b)))  # pre[i] = ones in [0, i)
        for s in range(SPL):
            sup[l * SPL + s] = pre[min(s * 65536, n)]
        for k in range(BPL):
            blk[l * BPL + k] = pre[k * 512] - pre[(k // 128) * 65536]
    return blk, sup


def access_bruteforce(S, i):
    return int(S[i])


def rank_bruteforce(S, c, i):
    return int(np.count_nonzero(np.asarray(S[: i + 1]) == c))


def nodes_from_csr(arrs) -> list:
    ptr = arrs["level_node_ptr"]
    out = []
    for l in range(len(ptr) - 1):
        lo, hi = int(ptr[l]), int(ptr[l + 1])
        out.append(list(zip(arrs["node_key"][lo:hi].tolist(), arrs["node_start"][lo:hi].tolist())))
    return out


def wm_sort(S: np.ndarray, sigma: int):
    """Wavelet matrix by its sort characterisation ("a strategy
    similar to sortWT, but using the reverse of the top l bits as the key when
    sorting"): level l's sequence is S stably sorted by the bit-reversed top l
    bits; its bitmap holds bit L-1-l; zeros[l] counts its 0 bits.
    Returns (bits [L*WPL] u64, zeros [L] u64)."""
    S = np.asarray(S).astype(np.uint64)
    n = S.size
    L = levels_of(sigma)
    W = wpl(n)
    bits = np.zeros(L * W, dtype=np.uint64)
    zeros = np.zeros(L, dtype=np.uint64)
    for l in range(L):
        top = S >> np.uint64(L - l) if l else np.zeros(n, dtype=np.uint64)
        key = np.zeros(n, dtype=np.uint64)
        for j in range(l):  # reverse the l-bit prefix
            key |= ((top >> np.uint64(j)) & np.uint64(1)) << np.uint64(l - 1 - j)
        order = np.argsort(key, kind="stable")
        Sl = S[order]
        b = ((Sl >> np.uint64(L - 1 - l)) & np.uint64(1)).astype(np.uint8)
        bits[l * W:(l + 1) * W] = pack_bits(b, W)
        zeros[l] = n - int(b.sum())
    return bits, zeros


def wm_access_rank_bruteforce(S: np.ndarray):
    """access(i) = S[i]; rank_c(i) = #{j <= i : S[j] = c}."""
    S = np.asarray(S)

    def rank(c, i):
        return int(np.count_nonzero(S[:i + 1] == c))
    return (lambda i: int(S[i])), rank


# ---------------------------------------------------------------------------
# Huffman-shaped wavelet tree (R-17..R-20)
# ---------------------------------------------------------------------------
def huffman_cost_bruteforce(freqs) -> int:
    """Minimum of sum f_c * len_c over all length vectors (1 <= len <= m-1)
    satisfying Kraft's inequality -- the optimal prefix-code cost, found by
    exhaustive enumeration (no Huffman algorithm involved)."""
    import itertools
    f = [int(x) for x in freqs if x > 0]
    m = len(f)
    if m < 2:
        return 0
    best = None
    for lens in itertools.product(range(1, m), repeat=m):
        if sum(2.0 ** -x for x in lens) <= 1.0 + 1e-12:
            c = sum(a * b for a, b in zip(f, lens))
            best = c if best is None or c < best else best
    return best


def hwt_closed_form(S, code, code_len):
    """Levels of the Huffman-shaped tree by a sort characterisation: level l
    holds the elements with code length > l, in S order stably sorted by
    their l-bit code prefix; each contributes code bit l.  Node starts are
    where the prefix changes.  Returns (per-level bit lists, per-level
    [(key, start)] lists)."""
    S = np.asarray(S).astype(np.int64)
    ln = np.asarray(code_len).astype(np.int64)[S]
    cd = np.asarray(code).astype(np.int64)[S]
    h = int(ln.max()) if S.size else 0
    levels, nodes = [], []
    for l in range(h):
        alive = np.nonzero(ln > l)[0]
        if alive.size == 0:
            break
        pre = cd[alive] >> (ln[alive] - l)
        order = np.argsort(pre, kind="stable")
        el = alive[order]
        bits = (cd[el] >> (ln[el] - 1 - l)) & 1
        pl = pre[order]
        O = np.nonzero(np.concatenate(([True], pl[1:] != pl[:-1])))[0]
        levels.append(bits.astype(np.uint8))
        nodes.append([(int(pl[o]), int(o)) for o in O])
    return levels, nodes


def rank_directory_one_level(words: np.ndarray, n: int):
    """R-9 sampling of one level of n bits (running popcount)."""
    BPL = (n + 511) // 512
    SPL = (n + 65535) // 65536 + 1
    b = np.unpackbits(words.view(np.uint8), bitorder="little")[:n].astype(np.int64)
    pre = np.concatenate(([0], np.cumsum(b)))
    sup = np.array([pre[min(s * 65536, n)] for s in range(SPL)], dtype=np.uint64)
    blk = np.array([pre[k * 512] - pre[(k // 128) * 65536] for k in range(BPL)], dtype=np.uint16)
    return blk, sup
