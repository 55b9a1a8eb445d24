"""ctypes binding of include/wt.h (argument marshalling only).

Every step of the build runs in ``libwt_b200.so``; torch is used for device
memory, streams and zero-copy tensor views of the library-owned outputs.
Names follow the C ABI: ``build`` -> ``wt_build``, ``build_host`` ->
``wt_build_host``, ``access`` -> ``wt_access``, ``rank`` -> ``wt_rank``,
``free`` -> ``wt_free``.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# WT_LIB_PATH selects a tuning variant built by tools/tune.py (developer knob)
_LIB_PATH = os.environ.get("WT_LIB_PATH") or os.path.join(_HERE, "libwt_b200.so")

WT_OK, WT_EINVAL, WT_ESYMBOL, WT_ENOMEM, WT_ECUDA, WT_EUNSUPPORTED = 0, -1, -2, -3, -4, -5
_NAMES = {WT_EINVAL: "WT_EINVAL", WT_ESYMBOL: "WT_ESYMBOL", WT_ENOMEM: "WT_ENOMEM",
          WT_ECUDA: "WT_ECUDA", WT_EUNSUPPORTED: "WT_EUNSUPPORTED"}


class WtError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what} failed: {_NAMES.get(code, code)}")
        self.code = code


class _WtTree(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint64), ("sigma", ctypes.c_uint64),
        ("levels", ctypes.c_uint32), ("elem_bytes", ctypes.c_uint32),
        ("words_per_level", ctypes.c_uint64),
        ("bits", ctypes.c_void_p), ("level_node_ptr", ctypes.c_void_p),
        ("node_key", ctypes.c_void_p), ("node_start", ctypes.c_void_p),
        ("total_nodes", ctypes.c_uint64),
        ("blocks_per_level", ctypes.c_uint64), ("supers_per_level", ctypes.c_uint64),
        ("rank_block", ctypes.c_void_p), ("rank_super", ctypes.c_void_p),
        ("select_per_level", ctypes.c_uint64), ("select0", ctypes.c_void_p), ("select1", ctypes.c_void_p),
        ("internal", ctypes.c_void_p),
    ]


class _ProfEntry(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 40), ("ms", ctypes.c_float), ("launches", ctypes.c_uint32),
                ("pad", ctypes.c_uint32), ("algo_bytes", ctypes.c_uint64)]


class _Profile(ctypes.Structure):
    _fields_ = [("count", ctypes.c_uint32), ("total_launches", ctypes.c_uint32),
                ("e", _ProfEntry * 32)]


_lib = None


def lib_path() -> str:
    return _LIB_PATH


class _WmMatrix(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint64),
        ("sigma", ctypes.c_uint64),
        ("levels", ctypes.c_uint32),
        ("elem_bytes", ctypes.c_uint32),
        ("words_per_level", ctypes.c_uint64),
        ("bits", ctypes.c_void_p),
        ("zeros", ctypes.c_void_p),
        ("blocks_per_level", ctypes.c_uint64),
        ("supers_per_level", ctypes.c_uint64),
        ("rank_block", ctypes.c_void_p),
        ("rank_super", ctypes.c_void_p),
        ("select_per_level", ctypes.c_uint64),
        ("select0", ctypes.c_void_p),
        ("select1", ctypes.c_void_p),
        ("internal", ctypes.c_void_p),
    ]


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: run `python __graft_entry__.py build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(_LIB_PATH)
    P = ctypes.POINTER(_WtTree)
    lib.wt_build.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                             ctypes.c_void_p, ctypes.POINTER(P)]
    lib.wt_build.restype = ctypes.c_int
    lib.wt_build_host.argtypes = lib.wt_build.argtypes
    lib.wt_build_host.restype = ctypes.c_int
    lib.wt_free.argtypes = [P]
    lib.wt_free.restype = ctypes.c_int
    lib.wt_access.argtypes = [P, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
    lib.wt_access.restype = ctypes.c_int
    lib.wt_rank.argtypes = [P, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                            ctypes.c_void_p]
    lib.wt_rank.restype = ctypes.c_int
    lib.wt_profile_enable.argtypes = [ctypes.c_int]
    lib.wt_profile_enable.restype = ctypes.c_int
    lib.wt_last_profile.argtypes = [ctypes.POINTER(_Profile)]
    lib.wt_last_profile.restype = ctypes.c_int
    lib.wt_profile_total.argtypes = [ctypes.POINTER(_Profile)]
    lib.wt_profile_total.restype = ctypes.c_int
    lib.wt_version.argtypes = []
    lib.wt_version.restype = ctypes.c_char_p
    PM = ctypes.POINTER(_WmMatrix)
    lib.wm_build.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                             ctypes.c_void_p, ctypes.POINTER(PM)]
    lib.wm_build.restype = ctypes.c_int
    lib.wm_free.argtypes = [PM]
    lib.wm_free.restype = ctypes.c_int
    lib.wm_access.argtypes = [PM, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
    lib.wm_access.restype = ctypes.c_int
    lib.wm_rank.argtypes = [PM, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                            ctypes.c_void_p]
    lib.wm_rank.restype = ctypes.c_int
    for pre, PT in (("wt", P), ("wm", PM)):
        getattr(lib, f"{pre}_select_index").argtypes = [PT, ctypes.c_void_p]
        getattr(lib, f"{pre}_select_index").restype = ctypes.c_int
        getattr(lib, f"{pre}_select").argtypes = [PT, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                                  ctypes.c_void_p, ctypes.c_void_p]
        getattr(lib, f"{pre}_select").restype = ctypes.c_int
    _lib = lib
    return lib


class _CAI:
    """Minimal __cuda_array_interface__ wrapper for a library-owned array.  It
    holds a reference to the owning structure, and torch keeps this object alive
    as long as the tensor view: a view keeps its tree (matrix) from being
    garbage-collected.  An explicit free() still releases the memory and
    invalidates every view (documented on free())."""

    def __init__(self, ptr: int, count: int, typestr: str, owner=None):
        self._owner = owner
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                         "data": (int(ptr or 0), False), "version": 3,
                                         "strides": None}


def _view(ptr, count, typestr, dtype, device, owner=None):
    if count == 0 or not ptr:
        return torch.zeros(0, dtype=dtype, device=device)
    return torch.as_tensor(_CAI(ptr, count, typestr, owner), device=device)


def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


class _SelectOps:
    """select_c through the C ABI; the directory is built on
    first use (``select_index``)."""
    _pre = "wt"

    def select_index(self, stream=None) -> dict:
        lib = _load()
        rc = getattr(lib, f"{self._pre}_select_index")(self.handle, ctypes.c_void_p(_stream_ptr(stream)))
        if rc != WT_OK:
            raise WtError(rc, f"{self._pre}_select_index")
        h = self.handle.contents
        sps = int(h.select_per_level)
        cnt = self.levels * sps
        return {"select_per_level": sps,
                "select0": _view(h.select0, cnt, "<u4", torch.uint32, self.device, self),
                "select1": _view(h.select1, cnt, "<u4", torch.uint32, self.device, self)}

    def select(self, sym: torch.Tensor, k: torch.Tensor, stream=None) -> torch.Tensor:
        lib = _load()
        if not int(self.handle.contents.select_per_level):
            self.select_index(stream)
        sym = sym.contiguous().view(-1)
        k = k.contiguous().view(-1)
        if sym.numel() != k.numel():
            raise ValueError("sym and k must have the same length")
        out = torch.empty(k.numel(), dtype=torch.int64, device=k.device)
        rc = getattr(lib, f"{self._pre}_select")(self.handle, ctypes.c_void_p(sym.data_ptr() if sym.numel() else 0),
                                                 ctypes.c_void_p(k.data_ptr() if k.numel() else 0), k.numel(),
                                                 ctypes.c_void_p(out.data_ptr() if out.numel() else 0),
                                                 ctypes.c_void_p(_stream_ptr(stream)))
        if rc != WT_OK:
            raise WtError(rc, f"{self._pre}_select")
        return out.view(torch.uint64)


class _Lazy:
    """A zero-copy torch view of one library array, made on first access
    (building a tree does not pay for views it never uses)."""

    def __init__(self, field, count, typestr, dtype):
        self.field, self.count, self.typestr, self.dtype = field, count, typestr, dtype

    def __set_name__(self, owner, name):
        self.name = name

    def __get__(self, obj, cls=None):
        if obj is None:
            return self
        v = _view(getattr(obj.handle.contents, self.field), self.count(obj), self.typestr, self.dtype, obj.device,
                  obj)
        obj.__dict__[self.name] = v
        return v


class WaveletTree(_SelectOps):
    """A built tree.  Arrays are zero-copy torch views of library memory and
    stay valid until ``free()`` (called on garbage collection too)."""
    bits = _Lazy("bits", lambda o: o.levels * o.words_per_level, "<u8", torch.uint64)
    level_node_ptr = _Lazy("level_node_ptr", lambda o: o.levels + 1, "<u8", torch.uint64)
    node_key = _Lazy("node_key", lambda o: o.total_nodes, "<u4", torch.uint32)
    node_start = _Lazy("node_start", lambda o: o.total_nodes, "<u4", torch.uint32)
    rank_block = _Lazy("rank_block", lambda o: o.levels * o.blocks_per_level, "<u2", torch.uint16)
    rank_super = _Lazy("rank_super", lambda o: o.levels * o.supers_per_level, "<u8", torch.uint64)

    def __init__(self, handle, device):
        self._h = handle
        t = handle.contents
        self.device = device
        self.n, self.sigma, self.levels = int(t.n), int(t.sigma), int(t.levels)
        self.elem_bytes = int(t.elem_bytes)
        self.words_per_level = int(t.words_per_level)
        self.blocks_per_level = int(t.blocks_per_level)
        self.supers_per_level = int(t.supers_per_level)
        self.total_nodes = int(t.total_nodes)

    @property
    def handle(self):
        if self._h is None:
            raise ValueError("tree already freed")
        return self._h

    def numpy(self) -> dict:
        """Copy every output array to host numpy (for bit-exact comparison)."""
        out = {}
        for k in ("bits", "level_node_ptr", "node_key", "node_start", "rank_block", "rank_super"):
            out[k] = getattr(self, k).cpu().numpy()
        out.update(n=self.n, sigma=self.sigma, levels=self.levels,
                   words_per_level=self.words_per_level, blocks_per_level=self.blocks_per_level,
                   supers_per_level=self.supers_per_level, total_nodes=self.total_nodes)
        return out

    def access(self, pos: torch.Tensor, stream=None) -> torch.Tensor:
        return access(self, pos, stream)

    def rank(self, sym: torch.Tensor, pos: torch.Tensor, stream=None) -> torch.Tensor:
        return rank(self, sym, pos, stream)

    def free(self):
        """Release the tree (wt_free, stream-ordered).  Views of its arrays
        taken earlier become invalid; views keep an unfreed tree alive."""
        if self._h is not None:
            for k in ("bits", "level_node_ptr", "node_key", "node_start", "rank_block", "rank_super"):
                setattr(self, k, None)
            rc = _load().wt_free(self._h)
            self._h = None
            if rc != WT_OK:
                raise WtError(rc, "wt_free")

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _elem_bytes(t: torch.Tensor) -> int:
    eb = t.element_size()
    if eb not in (1, 2, 4) or t.dtype.is_floating_point:
        raise TypeError("sequence must be an 8/16/32-bit integer tensor")
    return eb


def build(seq: torch.Tensor, sigma: int, stream=None) -> WaveletTree:
    """wt_build on a CUDA tensor holding S (any 8/16/32-bit integer dtype,
    read as unsigned)."""
    lib = _load()
    if not seq.is_cuda:
        raise ValueError("build() needs a CUDA tensor; use build_host() for host data")
    seq = seq.contiguous().view(-1)
    out = ctypes.POINTER(_WtTree)()
    rc = lib.wt_build(ctypes.c_void_p(seq.data_ptr() if seq.numel() else 0), seq.numel(),
                      _elem_bytes(seq), int(sigma), ctypes.c_void_p(_stream_ptr(stream)),
                      ctypes.byref(out))
    if rc != WT_OK:
        raise WtError(rc, "wt_build")
    return WaveletTree(out, seq.device)


def build_host(seq, sigma: int, stream=None, device=None) -> WaveletTree:
    """wt_build_host: seq is a host numpy array or CPU tensor (pinned is fastest)."""
    lib = _load()
    if isinstance(seq, torch.Tensor):
        if seq.is_cuda:
            raise ValueError("build_host() needs host memory")
        seq = seq.contiguous().view(-1)
        ptr, cnt, eb = seq.data_ptr(), seq.numel(), _elem_bytes(seq)
    else:
        import numpy as np
        seq = np.ascontiguousarray(seq)
        if seq.dtype not in (np.uint8, np.uint16, np.uint32, np.int8, np.int16, np.int32):
            raise TypeError("sequence must be an 8/16/32-bit integer array")
        ptr, cnt, eb = seq.ctypes.data, seq.size, seq.dtype.itemsize
    out = ctypes.POINTER(_WtTree)()
    rc = lib.wt_build_host(ctypes.c_void_p(ptr if cnt else 0), cnt, eb, int(sigma),
                           ctypes.c_void_p(_stream_ptr(stream)), ctypes.byref(out))
    if rc != WT_OK:
        raise WtError(rc, "wt_build_host")
    return WaveletTree(out, device or torch.device("cuda", torch.cuda.current_device()))


def access(tree: WaveletTree, pos: torch.Tensor, stream=None) -> torch.Tensor:
    """wt_access: pos int64/uint64 CUDA tensor -> uint32 symbols (int64 view returned)."""
    lib = _load()
    pos = pos.contiguous().view(-1)
    out = torch.empty(pos.numel(), dtype=torch.int32, device=pos.device)
    rc = lib.wt_access(tree.handle, ctypes.c_void_p(pos.data_ptr() if pos.numel() else 0), pos.numel(),
                       ctypes.c_void_p(out.data_ptr() if out.numel() else 0),
                       ctypes.c_void_p(_stream_ptr(stream)))
    if rc != WT_OK:
        raise WtError(rc, "wt_access")
    return out.view(torch.uint32)


def rank(tree: WaveletTree, sym: torch.Tensor, pos: torch.Tensor, stream=None) -> torch.Tensor:
    """wt_rank: inclusive rank_c(S, i); sym int32/uint32, pos int64/uint64 CUDA tensors."""
    lib = _load()
    sym = sym.contiguous().view(-1)
    pos = pos.contiguous().view(-1)
    if sym.numel() != pos.numel():
        raise ValueError("sym and pos must have the same length")
    out = torch.empty(pos.numel(), dtype=torch.int64, device=pos.device)
    rc = lib.wt_rank(tree.handle, ctypes.c_void_p(sym.data_ptr() if sym.numel() else 0),
                     ctypes.c_void_p(pos.data_ptr() if pos.numel() else 0), pos.numel(),
                     ctypes.c_void_p(out.data_ptr() if out.numel() else 0),
                     ctypes.c_void_p(_stream_ptr(stream)))
    if rc != WT_OK:
        raise WtError(rc, "wt_rank")
    return out.view(torch.uint64)


def free(tree: WaveletTree) -> None:
    tree.free()


def profile_enable(on: bool = True) -> None:
    _load().wt_profile_enable(1 if on else 0)


def last_profile(total: bool = False) -> dict:
    """Per-kernel record of the last build (or, with total=True, summed over
    every build since profile_enable(True))."""
    p = _Profile()
    (_load().wt_profile_total if total else _load().wt_last_profile)(ctypes.byref(p))
    ents = []
    for i in range(p.count):
        e = p.e[i]
        ents.append({"name": e.name.decode(), "ms": float(e.ms), "launches": int(e.launches),
                     "algo_bytes": int(e.algo_bytes)})
    return {"total_launches": int(p.total_launches), "kernels": ents}


def version() -> str:
    return _load().wt_version().decode()



# ---------------------------------------------------------------- wavelet matrix
class WaveletMatrix(_SelectOps):
    _pre = "wm"
    """A built wavelet matrix (PAPER.md:910-925).  Arrays are zero-copy torch
    views of library memory, valid until ``free()``."""

    def __init__(self, handle, device):
        self._h = handle
        m = handle.contents
        self.device = device
        self.n, self.sigma, self.levels = int(m.n), int(m.sigma), int(m.levels)
        self.words_per_level = int(m.words_per_level)
        self.blocks_per_level = int(m.blocks_per_level)
        self.supers_per_level = int(m.supers_per_level)
        L = self.levels
        self.bits = _view(m.bits, L * self.words_per_level, "<u8", torch.uint64, device, self)
        self.zeros = _view(m.zeros, L, "<u8", torch.uint64, device, self)
        self.rank_block = _view(m.rank_block, L * self.blocks_per_level, "<u2", torch.uint16, device, self)
        self.rank_super = _view(m.rank_super, L * self.supers_per_level, "<u8", torch.uint64, device, self)

    @property
    def handle(self):
        if self._h is None:
            raise ValueError("matrix already freed")
        return self._h

    def numpy(self) -> dict:
        out = {k: getattr(self, k).cpu().numpy() for k in ("bits", "zeros", "rank_block", "rank_super")}
        out.update(n=self.n, sigma=self.sigma, levels=self.levels, words_per_level=self.words_per_level,
                   blocks_per_level=self.blocks_per_level, supers_per_level=self.supers_per_level)
        return out

    def access(self, pos: torch.Tensor, stream=None) -> torch.Tensor:
        lib = _load()
        pos = pos.contiguous().view(-1)
        out = torch.empty(pos.numel(), dtype=torch.int32, device=pos.device)
        rc = lib.wm_access(self.handle, ctypes.c_void_p(pos.data_ptr() if pos.numel() else 0), pos.numel(),
                           ctypes.c_void_p(out.data_ptr() if out.numel() else 0),
                           ctypes.c_void_p(_stream_ptr(stream)))
        if rc != WT_OK:
            raise WtError(rc, "wm_access")
        return out.view(torch.uint32)

    def rank(self, sym: torch.Tensor, pos: torch.Tensor, stream=None) -> torch.Tensor:
        lib = _load()
        sym = sym.contiguous().view(-1)
        pos = pos.contiguous().view(-1)
        if sym.numel() != pos.numel():
            raise ValueError("sym and pos must have the same length")
        out = torch.empty(pos.numel(), dtype=torch.int64, device=pos.device)
        rc = lib.wm_rank(self.handle, ctypes.c_void_p(sym.data_ptr() if sym.numel() else 0),
                         ctypes.c_void_p(pos.data_ptr() if pos.numel() else 0), pos.numel(),
                         ctypes.c_void_p(out.data_ptr() if out.numel() else 0),
                         ctypes.c_void_p(_stream_ptr(stream)))
        if rc != WT_OK:
            raise WtError(rc, "wm_rank")
        return out.view(torch.uint64)

    def free(self):
        if self._h is not None:
            for k in ("bits", "zeros", "rank_block", "rank_super"):
                setattr(self, k, None)
            rc = _load().wm_free(self._h)
            self._h = None
            if rc != WT_OK:
                raise WtError(rc, "wm_free")

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def wm_build(seq: torch.Tensor, sigma: int, stream=None) -> WaveletMatrix:
    """wm_build on a CUDA tensor holding S (8/16/32-bit integers, read as unsigned)."""
    lib = _load()
    if not seq.is_cuda:
        raise ValueError("wm_build() needs a CUDA tensor")
    seq = seq.contiguous().view(-1)
    out = ctypes.POINTER(_WmMatrix)()
    rc = lib.wm_build(ctypes.c_void_p(seq.data_ptr() if seq.numel() else 0), seq.numel(),
                      _elem_bytes(seq), int(sigma), ctypes.c_void_p(_stream_ptr(stream)), ctypes.byref(out))
    if rc != WT_OK:
        raise WtError(rc, "wm_build")
    return WaveletMatrix(out, seq.device)


# ------------------------------------------------------ Huffman-shaped tree
class _HwtTree(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint64), ("sigma", ctypes.c_uint64),
        ("levels", ctypes.c_uint32), ("elem_bytes", ctypes.c_uint32),
        ("level_len", ctypes.c_void_p), ("level_word_ptr", ctypes.c_void_p),
        ("level_block_ptr", ctypes.c_void_p), ("level_super_ptr", ctypes.c_void_p),
        ("bits", ctypes.c_void_p), ("rank_block", ctypes.c_void_p), ("rank_super", ctypes.c_void_p),
        ("level_node_ptr", ctypes.c_void_p), ("node_key", ctypes.c_void_p), ("node_start", ctypes.c_void_p),
        ("total_nodes", ctypes.c_uint64),
        ("code", ctypes.c_void_p), ("code_len", ctypes.c_void_p),
        ("only_symbol", ctypes.c_uint32), ("stages", ctypes.c_uint32),
        ("total_bits", ctypes.c_uint64),
        ("internal", ctypes.c_void_p),
    ]


def _load_hwt():
    lib = _load()
    if getattr(lib, "_hwt_ready", False):
        return lib
    PH = ctypes.POINTER(_HwtTree)
    lib.hwt_build.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                              ctypes.c_void_p, ctypes.POINTER(PH)]
    lib.hwt_build.restype = ctypes.c_int
    lib.hwt_free.argtypes = [PH]
    lib.hwt_free.restype = ctypes.c_int
    lib.hwt_access.argtypes = [PH, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
    lib.hwt_access.restype = ctypes.c_int
    lib.hwt_rank.argtypes = [PH, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                             ctypes.c_void_p]
    lib.hwt_rank.restype = ctypes.c_int
    lib.hwt_select.argtypes = [PH, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                               ctypes.c_void_p]
    lib.hwt_select.restype = ctypes.c_int
    lib._hwt_ready = True
    return lib


class HuffmanWaveletTree:
    """A built Huffman-shaped wavelet tree.  Arrays are
    zero-copy torch views of library memory, valid until ``free()``."""
    _ARRAYS = ("level_len", "level_word_ptr", "level_block_ptr", "level_super_ptr", "bits", "rank_block",
               "rank_super", "level_node_ptr", "node_key", "node_start", "code", "code_len")

    def __init__(self, handle, device):
        self._h = handle
        t = handle.contents
        self.device = device
        self.n, self.sigma, self.levels = int(t.n), int(t.sigma), int(t.levels)
        self.total_nodes, self.total_bits = int(t.total_nodes), int(t.total_bits)
        self.only_symbol = int(t.only_symbol)
        self.stages = int(t.stages)
        h = self.levels
        u8 = lambda p, c: _view(p, c, "<u8", torch.uint64, device, self)  # noqa: E731
        self.level_len = u8(t.level_len, h)
        self.level_word_ptr = u8(t.level_word_ptr, h + 1)
        self.level_block_ptr = u8(t.level_block_ptr, h + 1)
        self.level_super_ptr = u8(t.level_super_ptr, h + 1)
        wp, bp, sp = (int(x[-1]) if h else 0 for x in (self.level_word_ptr.cpu(), self.level_block_ptr.cpu(),
                                                        self.level_super_ptr.cpu()))
        self.bits = u8(t.bits, wp)
        self.rank_block = _view(t.rank_block, bp, "<u2", torch.uint16, device, self)
        self.rank_super = u8(t.rank_super, sp)
        self.level_node_ptr = u8(t.level_node_ptr, h + 1)
        self.node_key = _view(t.node_key, self.total_nodes, "<u4", torch.uint32, device, self)
        self.node_start = _view(t.node_start, self.total_nodes, "<u4", torch.uint32, device, self)
        self.code = _view(t.code, self.sigma, "<u4", torch.uint32, device, self)
        self.code_len = _view(t.code_len, self.sigma, "|u1", torch.uint8, device, self)

    @property
    def handle(self):
        if self._h is None:
            raise ValueError("tree already freed")
        return self._h

    def numpy(self) -> dict:
        out = {k: getattr(self, k).cpu().numpy() for k in self._ARRAYS}
        out.update(n=self.n, sigma=self.sigma, levels=self.levels, total_nodes=self.total_nodes,
                   total_bits=self.total_bits, only_symbol=self.only_symbol)
        return out

    def access(self, pos: torch.Tensor, stream=None) -> torch.Tensor:
        lib = _load_hwt()
        pos = pos.contiguous().view(-1)
        out = torch.empty(pos.numel(), dtype=torch.int32, device=pos.device)
        rc = lib.hwt_access(self.handle, ctypes.c_void_p(pos.data_ptr() if pos.numel() else 0), pos.numel(),
                            ctypes.c_void_p(out.data_ptr() if out.numel() else 0),
                            ctypes.c_void_p(_stream_ptr(stream)))
        if rc != WT_OK:
            raise WtError(rc, "hwt_access")
        return out.view(torch.uint32)

    def rank(self, sym: torch.Tensor, pos: torch.Tensor, stream=None) -> torch.Tensor:
        lib = _load_hwt()
        sym = sym.contiguous().view(-1)
        pos = pos.contiguous().view(-1)
        if sym.numel() != pos.numel():
            raise ValueError("sym and pos must have the same length")
        out = torch.empty(pos.numel(), dtype=torch.int64, device=pos.device)
        rc = lib.hwt_rank(self.handle, ctypes.c_void_p(sym.data_ptr() if sym.numel() else 0),
                          ctypes.c_void_p(pos.data_ptr() if pos.numel() else 0), pos.numel(),
                          ctypes.c_void_p(out.data_ptr() if out.numel() else 0),
                          ctypes.c_void_p(_stream_ptr(stream)))
        if rc != WT_OK:
            raise WtError(rc, "hwt_rank")
        return out.view(torch.uint64)

    def select(self, sym: torch.Tensor, k: torch.Tensor, stream=None) -> torch.Tensor:
        """hwt_select: position of the k'th (1-based) occurrence of each symbol."""
        lib = _load_hwt()
        sym = sym.contiguous().view(-1)
        k = k.contiguous().view(-1)
        if sym.numel() != k.numel():
            raise ValueError("sym and k must have the same length")
        out = torch.empty(k.numel(), dtype=torch.int64, device=k.device)
        rc = lib.hwt_select(self.handle, ctypes.c_void_p(sym.data_ptr() if sym.numel() else 0),
                            ctypes.c_void_p(k.data_ptr() if k.numel() else 0), k.numel(),
                            ctypes.c_void_p(out.data_ptr() if out.numel() else 0),
                            ctypes.c_void_p(_stream_ptr(stream)))
        if rc != WT_OK:
            raise WtError(rc, "hwt_select")
        return out.view(torch.uint64)

    def free(self):
        if self._h is not None:
            for k in self._ARRAYS:
                setattr(self, k, None)
            rc = _load_hwt().hwt_free(self._h)
            self._h = None
            if rc != WT_OK:
                raise WtError(rc, "hwt_free")

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def hwt_build(seq: torch.Tensor, sigma: int, stream=None) -> HuffmanWaveletTree:
    """hwt_build on a CUDA tensor holding S (8/16/32-bit integers, read as unsigned; sigma <= 65536)."""
    lib = _load_hwt()
    if not seq.is_cuda:
        raise ValueError("hwt_build() needs a CUDA tensor")
    seq = seq.contiguous().view(-1)
    out = ctypes.POINTER(_HwtTree)()
    rc = lib.hwt_build(ctypes.c_void_p(seq.data_ptr() if seq.numel() else 0), seq.numel(),
                       _elem_bytes(seq), int(sigma), ctypes.c_void_p(_stream_ptr(stream)), ctypes.byref(out))
    if rc != WT_OK:
        raise WtError(rc, "hwt_build")
    return HuffmanWaveletTree(out, seq.device)


# ------------------------------------------------ sharded-build helpers (C ABI)
def _load_dist():
    lib = _load()
    if getattr(lib, "_dist_ready", False):
        return lib
    V, U64, U32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32
    lib.wt_digit_counts.argtypes = [V, U64, U32, U64, U32, U32, V, V]
    lib.wt_digits.argtypes = [V, U64, U32, U32, U32, V, V]
    lib.wt_partition.argtypes = [V, U64, U32, U32, U32, V, V]
    lib.wt_gather_bits.argtypes = [V, V, U64, V, U64, V]
    lib.wt_create.argtypes = [U64, U64, U32, U64, V, ctypes.POINTER(ctypes.POINTER(_WtTree))]
    lib.wt_finish.argtypes = [ctypes.POINTER(_WtTree), V]
    for f in ("wt_digit_counts", "wt_digits", "wt_partition", "wt_gather_bits", "wt_create", "wt_finish"):
        getattr(lib, f).restype = ctypes.c_int
    lib._dist_ready = True
    return lib


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr() if t.numel() else 0)


def digit_counts(seq: torch.Tensor, sigma: int, shift: int, tau: int, stream=None) -> torch.Tensor:
    """wt_digit_counts: u64 counts of the tau-bit digit (seq >> shift); raises WT_ESYMBOL."""
    lib = _load_dist()
    seq = seq.contiguous().view(-1)
    out = torch.empty(1 << tau, dtype=torch.int64, device=seq.device)
    rc = lib.wt_digit_counts(_ptr(seq), seq.numel(), _elem_bytes(seq), int(sigma), shift, tau, _ptr(out),
                             ctypes.c_void_p(_stream_ptr(stream)))
    if rc != WT_OK:
        raise WtError(rc, "wt_digit_counts")
    return out


def digits(seq: torch.Tensor, shift: int, tau: int, stream=None) -> torch.Tensor:
    """wt_digits: u8 tensor of (seq >> shift) & (2^tau - 1)."""
    lib = _load_dist()
    seq = seq.contiguous().view(-1)
    out = torch.empty(seq.numel(), dtype=torch.uint8, device=seq.device)
    rc = lib.wt_digits(_ptr(seq), seq.numel(), _elem_bytes(seq), shift, tau, _ptr(out),
                       ctypes.c_void_p(_stream_ptr(stream)))
    if rc != WT_OK:
        raise WtError(rc, "wt_digits")
    return out


def partition(seq: torch.Tensor, shift: int, tau: int, stream=None) -> torch.Tensor:
    """wt_partition: seq stably sorted by its tau-bit digit at `shift`."""
    lib = _load_dist()
    seq = seq.contiguous().view(-1)
    out = torch.empty_like(seq)
    rc = lib.wt_partition(_ptr(seq), seq.numel(), _elem_bytes(seq), shift, tau, _ptr(out),
                          ctypes.c_void_p(_stream_ptr(stream)))
    if rc != WT_OK:
        raise WtError(rc, "wt_partition")
    return out


def gather_bits(src: torch.Tensor, segs: torch.Tensor, dst: torch.Tensor, stream=None) -> None:
    """wt_gather_bits: dst (u64 words) <- bit segments (dst_bit, src_bit, len) of src."""
    lib = _load_dist()
    segs = segs.contiguous().view(-1)
    rc = lib.wt_gather_bits(_ptr(src), _ptr(segs), segs.numel() // 3, _ptr(dst), dst.numel(),
                            ctypes.c_void_p(_stream_ptr(stream)))
    if rc != WT_OK:
        raise WtError(rc, "wt_gather_bits")


def create(n: int, sigma: int, elem_bytes: int, total_nodes: int, device, stream=None) -> WaveletTree:
    """wt_create: an empty library-owned tree to be filled, then finish()."""
    lib = _load_dist()
    out = ctypes.POINTER(_WtTree)()
    rc = lib.wt_create(int(n), int(sigma), int(elem_bytes), int(total_nodes), ctypes.c_void_p(_stream_ptr(stream)),
                       ctypes.byref(out))
    if rc != WT_OK:
        raise WtError(rc, "wt_create")
    return WaveletTree(out, device)


def finish(tree: WaveletTree, stream=None) -> None:
    """wt_finish: rank directory from the tree's bits (synchronises)."""
    rc = _load_dist().wt_finish(tree.handle, ctypes.c_void_p(_stream_ptr(stream)))
    if rc != WT_OK:
        raise WtError(rc, "wt_finish")
