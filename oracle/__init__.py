"""CPU oracle for the levelwise wavelet tree -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` and ``--impl reference`` legs) may import this package.
The product package ``paper_1407_8142_b200`` never imports it, and the two
share no code: the oracle is plain C (``wt_oracle.c``) that follows
PAPER.md Fig. 1 (levelWT) step by step, plus this ctypes
marshalling layer.

``build(seq, sigma)`` returns a dict of numpy arrays laid out exactly as the
C-ABI of the CUDA path specifies (``include/wt.h``), so the two can be
compared element by element.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "wt_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK, EINVAL, ESYMBOL, ENOMEM, EUNSUPPORTED = 0, -1, -2, -3, -5


class _Tree(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint64),
        ("sigma", ctypes.c_uint64),
        ("levels", ctypes.c_uint32),
        ("elem_bytes", ctypes.c_uint32),
        ("words_per_level", ctypes.c_uint64),
        ("bits", ctypes.POINTER(ctypes.c_uint64)),
        ("level_node_ptr", ctypes.POINTER(ctypes.c_uint64)),
        ("node_key", ctypes.POINTER(ctypes.c_uint32)),
        ("node_start", ctypes.POINTER(ctypes.c_uint32)),
        ("total_nodes", ctypes.c_uint64),
        ("blocks_per_level", ctypes.c_uint64),
        ("supers_per_level", ctypes.c_uint64),
        ("rank_block", ctypes.POINTER(ctypes.c_uint16)),
        ("rank_super", ctypes.POINTER(ctypes.c_uint64)),
    ]


class _WM(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint64),
        ("sigma", ctypes.c_uint64),
        ("levels", ctypes.c_uint32),
        ("elem_bytes", ctypes.c_uint32),
        ("words_per_level", ctypes.c_uint64),
        ("bits", ctypes.POINTER(ctypes.c_uint64)),
        ("zeros", ctypes.POINTER(ctypes.c_uint64)),
        ("blocks_per_level", ctypes.c_uint64),
        ("supers_per_level", ctypes.c_uint64),
        ("rank_block", ctypes.POINTER(ctypes.c_uint16)),
        ("rank_super", ctypes.POINTER(ctypes.c_uint64)),
    ]


class _HWT(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint64),
        ("sigma", ctypes.c_uint64),
        ("levels", ctypes.c_uint32),
        ("elem_bytes", ctypes.c_uint32),
        ("level_len", ctypes.POINTER(ctypes.c_uint64)),
        ("level_word_ptr", ctypes.POINTER(ctypes.c_uint64)),
        ("level_block_ptr", ctypes.POINTER(ctypes.c_uint64)),
        ("level_super_ptr", ctypes.POINTER(ctypes.c_uint64)),
        ("bits", ctypes.POINTER(ctypes.c_uint64)),
        ("rank_block", ctypes.POINTER(ctypes.c_uint16)),
        ("rank_super", ctypes.POINTER(ctypes.c_uint64)),
        ("level_node_ptr", ctypes.POINTER(ctypes.c_uint64)),
        ("node_key", ctypes.POINTER(ctypes.c_uint32)),
        ("node_start", ctypes.POINTER(ctypes.c_uint32)),
        ("total_nodes", ctypes.c_uint64),
        ("code", ctypes.POINTER(ctypes.c_uint32)),
        ("code_len", ctypes.POINTER(ctypes.c_uint8)),
        ("only_symbol", ctypes.c_uint32),
    ]


def compile_oracle(force: bool = False) -> str:
    """Compile wt_oracle.c with gcc into oracle/liboracle.so (idempotent)."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-Wextra", "-shared",
                           "-fPIC", "-o", tmp, _SRC])
    os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(compile_oracle())
            lib.oracle_build.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32,
                                         ctypes.c_uint64, ctypes.POINTER(ctypes.POINTER(_Tree))]
            lib.oracle_build.restype = ctypes.c_int
            lib.oracle_free.argtypes = [ctypes.POINTER(_Tree)]
            lib.oracle_free.restype = None
            lib.oracle_access.argtypes = [ctypes.POINTER(_Tree), ctypes.c_uint64]
            lib.oracle_access.restype = ctypes.c_uint32
            lib.oracle_rank.argtypes = [ctypes.POINTER(_Tree), ctypes.c_uint32, ctypes.c_uint64]
            lib.oracle_rank.restype = ctypes.c_uint64
            lib.oracle_rank1.argtypes = [ctypes.POINTER(_Tree), ctypes.c_uint32, ctypes.c_uint64]
            lib.oracle_rank1.restype = ctypes.c_uint64
            lib.oracle_levels.argtypes = [ctypes.c_uint64]
            lib.oracle_levels.restype = ctypes.c_uint32
            lib.oracle_wm_build.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32,
                                            ctypes.c_uint64, ctypes.POINTER(ctypes.POINTER(_WM))]
            lib.oracle_wm_build.restype = ctypes.c_int
            lib.oracle_wm_free.argtypes = [ctypes.POINTER(_WM)]
            lib.oracle_wm_free.restype = None
            lib.oracle_wm_access.argtypes = [ctypes.POINTER(_WM), ctypes.c_uint64]
            lib.oracle_wm_access.restype = ctypes.c_uint32
            lib.oracle_wm_rank.argtypes = [ctypes.POINTER(_WM), ctypes.c_uint32, ctypes.c_uint64]
            lib.oracle_wm_rank.restype = ctypes.c_uint64
            PU = ctypes.POINTER(ctypes.POINTER(ctypes.c_uint32))
            lib.oracle_select_dir.argtypes = [ctypes.POINTER(_Tree), PU, PU, ctypes.POINTER(ctypes.c_uint64)]
            lib.oracle_select_dir.restype = ctypes.c_int
            lib.oracle_wm_select_dir.argtypes = [ctypes.POINTER(_WM), PU, PU, ctypes.POINTER(ctypes.c_uint64)]
            lib.oracle_wm_select_dir.restype = ctypes.c_int
            lib.oracle_free_buf.argtypes = [ctypes.c_void_p]
            lib.oracle_free_buf.restype = None
            U32P = ctypes.POINTER(ctypes.c_uint32)
            lib.oracle_select.argtypes = [ctypes.POINTER(_Tree), U32P, U32P, ctypes.c_uint64, ctypes.c_uint32,
                                          ctypes.c_uint64]
            lib.oracle_select.restype = ctypes.c_uint64
            lib.oracle_wm_select.argtypes = [ctypes.POINTER(_WM), U32P, U32P, ctypes.c_uint64, ctypes.c_uint32,
                                             ctypes.c_uint64]
            lib.oracle_wm_select.restype = ctypes.c_uint64
            lib.oracle_hwt_build.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32,
                                             ctypes.c_uint64, ctypes.POINTER(ctypes.POINTER(_HWT))]
            lib.oracle_hwt_build.restype = ctypes.c_int
            lib.oracle_hwt_free.argtypes = [ctypes.POINTER(_HWT)]
            lib.oracle_hwt_free.restype = None
            lib.oracle_hwt_access.argtypes = [ctypes.POINTER(_HWT), ctypes.c_uint64]
            lib.oracle_hwt_access.restype = ctypes.c_uint32
            lib.oracle_hwt_rank.argtypes = [ctypes.POINTER(_HWT), ctypes.c_uint32, ctypes.c_uint64]
            lib.oracle_hwt_rank.restype = ctypes.c_uint64
            lib.oracle_hwt_select.argtypes = [ctypes.POINTER(_HWT), ctypes.c_uint32, ctypes.c_uint64]
            lib.oracle_hwt_select.restype = ctypes.c_uint64
            _lib = lib
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(f"oracle_build failed with code {code}")
        self.code = code


def _copy(ptr, count, dtype):
    if count == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(count,)).astype(dtype, copy=True)




def _select_dir(lib, fn, handle, levels):
    """Run a select-directory builder; returns (sel0, sel1, sps, raw pointers)."""
    s0 = ctypes.POINTER(ctypes.c_uint32)()
    s1 = ctypes.POINTER(ctypes.c_uint32)()
    sps = ctypes.c_uint64()
    rc = fn(handle, ctypes.byref(s0), ctypes.byref(s1), ctypes.byref(sps))
    if rc != OK:
        raise OracleError(rc)
    cnt = levels * sps.value
    a0, a1 = _copy(s0, cnt, np.uint32), _copy(s1, cnt, np.uint32)
    return a0, a1, sps.value, (s0, s1)


class _SelectMixin:
    """select_c and the sampled select directory."""

    def _sel(self):
        if getattr(self, "_seldir", None) is None:
            self._seldir = _select_dir(self._lib, self._sel_dir_fn, self._handle(), self.levels)
        return self._seldir

    def select_dir(self) -> dict:
        a0, a1, sps, _ = self._sel()
        return {"select0": a0, "select1": a1, "select_per_level": sps}

    def select(self, symbols, ks) -> np.ndarray:
        _, _, sps, (p0, p1) = self._sel()
        return np.array([self._sel_fn(self._handle(), p0, p1, sps, int(c), int(k))
                         for c, k in zip(symbols, ks)], dtype=np.uint64)

    def _free_sel(self):
        sd = getattr(self, "_seldir", None)
        if sd is not None:
            self._lib.oracle_free_buf(sd[3][0])
            self._lib.oracle_free_buf(sd[3][1])
            self._seldir = None


class OracleTree(_SelectMixin):
    """Owns one C oracle tree; arrays are copied out into numpy."""

    def __init__(self, seq: np.ndarray, sigma: int):
        lib = _load()
        seq = np.ascontiguousarray(seq)
        if seq.dtype not in (np.uint8, np.uint16, np.uint32):
            raise TypeError("seq must be uint8/uint16/uint32")
        out = ctypes.POINTER(_Tree)()
        rc = lib.oracle_build(seq.ctypes.data if seq.size else None, seq.size,
                              seq.dtype.itemsize, int(sigma), ctypes.byref(out))
        if rc != OK:
            raise OracleError(rc)
        self._lib = lib
        self._t = out
        t = out.contents
        self.n, self.sigma, self.levels = t.n, t.sigma, t.levels
        self.words_per_level = t.words_per_level
        self.blocks_per_level = t.blocks_per_level
        self.supers_per_level = t.supers_per_level
        self.total_nodes = t.total_nodes

    def array(self, name: str) -> np.ndarray:
        """Copy one output array out (keeps peak host memory low for big n)."""
        t = self._t.contents
        L = t.levels
        spec = {
            "bits": (t.bits, L * t.words_per_level, np.uint64),
            "level_node_ptr": (t.level_node_ptr, L + 1, np.uint64),
            "node_key": (t.node_key, t.total_nodes, np.uint32),
            "node_start": (t.node_start, t.total_nodes, np.uint32),
            "rank_block": (t.rank_block, L * t.blocks_per_level, np.uint16),
            "rank_super": (t.rank_super, L * t.supers_per_level, np.uint64),
        }[name]
        return _copy(*spec)

    def arrays(self) -> dict:
        return {k: self.array(k) for k in ("bits", "level_node_ptr", "node_key", "node_start",
                                           "rank_block", "rank_super")}

    def access(self, positions) -> np.ndarray:
        return np.array([self._lib.oracle_access(self._t, int(i)) for i in positions],
                        dtype=np.uint32)

    def rank(self, symbols, positions) -> np.ndarray:
        return np.array([self._lib.oracle_rank(self._t, int(c), int(i))
                         for c, i in zip(symbols, positions)], dtype=np.uint64)

    def rank1(self, level: int, i: int) -> int:
        return int(self._lib.oracle_rank1(self._t, level, i))

    _handle = property(lambda self: (lambda: self._t))
    _sel_dir_fn = property(lambda self: self._lib.oracle_select_dir)
    _sel_fn = property(lambda self: self._lib.oracle_select)

    def close(self):
        self._free_sel()
        if getattr(self, "_t", None):
            self._lib.oracle_free(self._t)
            self._t = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def build(seq: np.ndarray, sigma: int, select: bool = False) -> dict:
    """Oracle construction; returns the §8(b) arrays plus scalar metadata
    (and the select directory when ``select``)."""
    with OracleTree(seq, sigma) as t:
        out = t.arrays()
        if select:
            out.update(t.select_dir())
        out.update(n=t.n, sigma=t.sigma, levels=t.levels,
                   words_per_level=t.words_per_level,
                   blocks_per_level=t.blocks_per_level,
                   supers_per_level=t.supers_per_level, total_nodes=t.total_nodes)
    return out


def levels(sigma: int) -> int:
    return int(_load().oracle_levels(int(sigma)))


class OracleWM(_SelectMixin):
    """Owns one C oracle wavelet matrix; arrays copied out."""

    def __init__(self, seq: np.ndarray, sigma: int):
        lib = _load()
        seq = np.ascontiguousarray(seq)
        if seq.dtype not in (np.uint8, np.uint16, np.uint32):
            raise TypeError("seq must be uint8/uint16/uint32")
        out = ctypes.POINTER(_WM)()
        rc = lib.oracle_wm_build(seq.ctypes.data if seq.size else None, seq.size,
                                 seq.dtype.itemsize, int(sigma), ctypes.byref(out))
        if rc != OK:
            raise OracleError(rc)
        self._lib = lib
        self._m = out
        m = out.contents
        self.n, self.sigma, self.levels = m.n, m.sigma, m.levels
        self.words_per_level = m.words_per_level
        self.blocks_per_level = m.blocks_per_level
        self.supers_per_level = m.supers_per_level

    def arrays(self) -> dict:
        m = self._m.contents
        L = m.levels
        return {
            "bits": _copy(m.bits, L * m.words_per_level, np.uint64),
            "zeros": _copy(m.zeros, L, np.uint64),
            "rank_block": _copy(m.rank_block, L * m.blocks_per_level, np.uint16),
            "rank_super": _copy(m.rank_super, L * m.supers_per_level, np.uint64),
        }

    def access(self, positions) -> np.ndarray:
        return np.array([self._lib.oracle_wm_access(self._m, int(i)) for i in positions], dtype=np.uint32)

    def rank(self, symbols, positions) -> np.ndarray:
        return np.array([self._lib.oracle_wm_rank(self._m, int(c), int(i))
                         for c, i in zip(symbols, positions)], dtype=np.uint64)

    _handle = property(lambda self: (lambda: self._m))
    _sel_dir_fn = property(lambda self: self._lib.oracle_wm_select_dir)
    _sel_fn = property(lambda self: self._lib.oracle_wm_select)

    def close(self):
        self._free_sel()
        if getattr(self, "_m", None):
            self._lib.oracle_wm_free(self._m)
            self._m = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def wm_build(seq: np.ndarray, sigma: int) -> dict:
    """Oracle wavelet matrix; returns bits, zeros, rank_block, rank_super (+ metadata)."""
    with OracleWM(seq, sigma) as m:
        out = m.arrays()
        out.update(m.select_dir())
        out.update(n=m.n, sigma=m.sigma, levels=m.levels, words_per_level=m.words_per_level,
                   blocks_per_level=m.blocks_per_level, supers_per_level=m.supers_per_level)
    return out


class OracleHWT:
    """Owns one C oracle Huffman-shaped wavelet tree."""

    def __init__(self, seq: np.ndarray, sigma: int):
        lib = _load()
        seq = np.ascontiguousarray(seq)
        if seq.dtype not in (np.uint8, np.uint16, np.uint32):
            raise TypeError("seq must be uint8/uint16/uint32")
        out = ctypes.POINTER(_HWT)()
        rc = lib.oracle_hwt_build(seq.ctypes.data if seq.size else None, seq.size,
                                  seq.dtype.itemsize, int(sigma), ctypes.byref(out))
        if rc != OK:
            raise OracleError(rc)
        self._lib = lib
        self._t = out
        t = out.contents
        self.n, self.sigma, self.levels = t.n, t.sigma, t.levels
        self.total_nodes = t.total_nodes
        self.only_symbol = t.only_symbol

    def arrays(self) -> dict:
        t = self._t.contents
        h = t.levels
        wp = _copy(t.level_word_ptr, h + 1, np.uint64)
        bp = _copy(t.level_block_ptr, h + 1, np.uint64)
        sp = _copy(t.level_super_ptr, h + 1, np.uint64)
        return {
            "level_len": _copy(t.level_len, h, np.uint64),
            "level_word_ptr": wp,
            "level_block_ptr": bp,
            "level_super_ptr": sp,
            "bits": _copy(t.bits, int(wp[-1]), np.uint64),
            "rank_block": _copy(t.rank_block, int(bp[-1]), np.uint16),
            "rank_super": _copy(t.rank_super, int(sp[-1]), np.uint64),
            "level_node_ptr": _copy(t.level_node_ptr, h + 1, np.uint64),
            "node_key": _copy(t.node_key, t.total_nodes, np.uint32),
            "node_start": _copy(t.node_start, t.total_nodes, np.uint32),
            "code": _copy(t.code, t.sigma, np.uint32),
            "code_len": _copy(t.code_len, t.sigma, np.uint8),
        }

    def access(self, positions) -> np.ndarray:
        return np.array([self._lib.oracle_hwt_access(self._t, int(i)) for i in positions], dtype=np.uint32)

    def rank(self, symbols, positions) -> np.ndarray:
        return np.array([self._lib.oracle_hwt_rank(self._t, int(c), int(i))
                         for c, i in zip(symbols, positions)], dtype=np.uint64)

    def select(self, symbols, ks) -> np.ndarray:
        return np.array([self._lib.oracle_hwt_select(self._t, int(c), int(k))
                         for c, k in zip(symbols, ks)], dtype=np.uint64)

    def close(self):
        if getattr(self, "_t", None):
            self._lib.oracle_hwt_free(self._t)
            self._t = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def hwt_build(seq: np.ndarray, sigma: int) -> dict:
    """Oracle Huffman-shaped wavelet tree; arrays as include/wt.h's hwt_tree."""
    with OracleHWT(seq, sigma) as t:
        out = t.arrays()
        out.update(n=t.n, sigma=t.sigma, levels=t.levels, total_nodes=t.total_nodes,
                   only_symbol=t.only_symbol)
    return out
