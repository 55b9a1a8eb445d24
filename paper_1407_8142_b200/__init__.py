"""B200 (sm_100a) levelwise wavelet-tree construction (arXiv 1407.8142).

The compute path is the C-ABI library ``libwt_b200.so`` (CUDA kernels in
``csrc/``, declared in ``include/wt.h``).  ``wt`` is a thin ctypes binding with
the same names: it only marshals arguments.  There is no CPU fallback: if the
library is missing, importing ``wt`` raises.
"""
from .wt import (WT_ESYMBOL, HuffmanWaveletTree, WaveletMatrix, WaveletTree, WtError, access, build, build_host, free,
                 lib_path, rank, profile_enable, last_profile, version, wm_build, hwt_build)

__all__ = ["WT_ESYMBOL", "HuffmanWaveletTree", "WaveletMatrix", "WaveletTree", "WtError", "access", "build", "build_host",
           "free", "lib_path", "rank", "profile_enable", "last_profile", "version", "wm_build", "hwt_build"]
