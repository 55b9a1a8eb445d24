"""Counter-based SplitMix64 generators and the five BASELINE.json configs.

Recipe: r_i = mix64(seed + (i+1) * 0x9E3779B97F4A7C15),
i = 0..n-1, the SplitMix64 finaliser of Steele, Lea & Flood.  Uniform over 2^k
is r_i >> (64-k).  Zipf(s) over m values uses a frozen u64 CDF threshold table
and a Fisher-Yates permutation of the m values (reading R-13).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_CHUNK = 1 << 24


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z.copy()
    z ^= z >> np.uint64(30)
    z *= _M1
    z ^= z >> np.uint64(27)
    z *= _M2
    z ^= z >> np.uint64(31)
    return z


def splitmix64_stream(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """r_i for i in [offset, offset+n) as uint64."""
    with np.errstate(over="ignore"):
        i = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        return _mix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + i * GOLDEN)


def _chunked(n: int, dtype, fn) -> np.ndarray:
    out = np.empty(n, dtype=dtype)
    for lo in range(0, n, _CHUNK):
        hi = min(n, lo + _CHUNK)
        out[lo:hi] = fn(lo, hi - lo)
    return out


def uniform_bits(n: int, k: int, seed: int, dtype=np.uint32) -> np.ndarray:
    """n values uniform over [0, 2^k) (0 <= k <= 32)."""
    if k == 0:
        return np.zeros(n, dtype=dtype)
    sh = np.uint64(64 - k)
    return _chunked(n, dtype, lambda lo, m: (splitmix64_stream(seed, m, lo) >> sh).astype(dtype))


def uniform_below(n: int, bound: int, seed: int, dtype=np.uint32) -> np.ndarray:
    """n values in [0, bound) as ((r >> 32) * bound) >> 32 (bound <= 2^32)."""
    b = np.uint64(bound)
    sh = np.uint64(32)

    def f(lo, m):
        with np.errstate(over="ignore"):
            return (((splitmix64_stream(seed, m, lo) >> sh) * b) >> sh).astype(dtype)
    return _chunked(n, dtype, f)


def zipf_table(m: int = 256, s: float = 1.1) -> np.ndarray:
    """Frozen u64 CDF thresholds T_1..T_{m-1} (T_m = +inf), computed in double."""
    w = np.array([k ** (-s) for k in range(1, m + 1)], dtype=np.float64)
    cdf = np.cumsum(w) / w.sum()
    return np.array([min(int(c * 2.0 ** 64), 2 ** 64 - 1) for c in cdf[:-1]], dtype=np.uint64)


def fisher_yates(m: int, seed: int) -> np.ndarray:
    r = splitmix64_stream(seed ^ 0x5DEECE66D, m)
    perm = np.arange(m, dtype=np.uint32)
    for j, i in enumerate(range(m - 1, 0, -1)):
        k = int(r[j] % np.uint64(i + 1))
        perm[i], perm[k] = perm[k], perm[i]
    return perm


def zipf_permuted(n: int, seed: int, m: int = 256, s: float = 1.1, dtype=np.uint8) -> np.ndarray:
    """Rank k (1..m) with P(k) ~ k^-s, mapped through a seeded permutation."""
    table = zipf_table(m, s)
    perm = fisher_yates(m, seed)

    def f(lo, cnt):
        r = splitmix64_stream(seed, cnt, lo)
        k = np.searchsorted(table, r, side="right")  # rank - 1
        return perm[k].astype(dtype)
    return _chunked(n, dtype, f)


def fnv1a64(a: np.ndarray) -> int:
    """FNV-1a-64 over the little-endian bytes of a (for identity checks)."""
    h = 0xCBF29CE484222325
    for b in np.ascontiguousarray(a).view(np.uint8).tobytes():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


@dataclass(frozen=True)
class Config:
    idx: int
    name: str
    n: int
    elem_bytes: int
    sigma: int
    seed: int
    kind: str  # "uniform" or "zipf"

    @property
    def dtype(self):
        return {1: np.uint8, 2: np.uint16, 4: np.uint32}[self.elem_bytes]

    @property
    def levels(self) -> int:
        return (self.sigma - 1).bit_length()


# BASELINE.json "configs", in order
CONFIGS = {
    1: Config(1, "cfg1_n2^16_u8_uniform256", 1 << 16, 1, 256, 1, "uniform"),
    2: Config(2, "cfg2_n2^26_u8_uniform4", 1 << 26, 1, 4, 2, "uniform"),
    3: Config(3, "cfg3_n2^27_u8_zipf1.1_256", 1 << 27, 1, 256, 3, "zipf"),
    4: Config(4, "cfg4_n2^28_u32_uniform65536", 1 << 28, 4, 1 << 16, 4, "uniform"),
    5: Config(5, "cfg5_n2^29_u32_uniform2^32", 1 << 29, 4, 1 << 32, 5, "uniform"),
}


def config_input(cfg: Config, n: int | None = None) -> np.ndarray:
    """The config's sequence (or its first n elements: same stream prefix)."""
    n = cfg.n if n is None else n
    if cfg.kind == "zipf":
        return zipf_permuted(n, cfg.seed, dtype=cfg.dtype)
    return uniform_bits(n, cfg.levels, cfg.seed, dtype=cfg.dtype)
