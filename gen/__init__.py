"""Seeded synthetic input generators (input plumbing only).

Shared by the oracle tests, the GPU parity tests, smoke() and bench.py.  This
package holds none of the wavelet-tree method's arithmetic: it only produces
the integer sequences S that both sides consume.
"""
from .inputs import (CONFIGS, Config, config_input, splitmix64_stream, uniform_bits,
                     uniform_below, zipf_permuted, fnv1a64)

__all__ = ["CONFIGS", "Config", "config_input", "splitmix64_stream", "uniform_bits",
           "uniform_below", "zipf_permuted", "fnv1a64"]
