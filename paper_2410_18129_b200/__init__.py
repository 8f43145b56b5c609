"""paper_2410_18129_b200 -- B200-native batched constant-time Montgomery modexp.

The hot path of arXiv 2410.18129 (truncated batch Montgomery multiplication and
constant-time fixed-window modular exponentiation) as hand-written sm_100a CUDA
kernels behind a C-ABI library (include/mpb.h, csrc/), with a thin ctypes
binding (``paper_2410_18129_b200.mpb``).  ``inputs`` holds the seeded input
generators shared with the oracle.  The binding is imported lazily so that
CPU-only tooling (tests of the oracle, the input generators) never needs CUDA.
"""
import importlib

__all__ = ["inputs", "mpb"]


def __getattr__(name):
    if name in __all__:
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
