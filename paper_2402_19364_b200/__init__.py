"""B200-native arrow-decomposition SpMM (arXiv 2402.19364): Y = A X through
A = sum_i P_i B_i P_i^T with hand-written sm_100a kernels behind a C ABI (include/arrow.h).

The package holds only the hot path: ``csrc/`` (CUDA kernels, host decomposer, C ABI) and
the ctypes binding ``arrow``.  It never imports ``oracle/`` (test infrastructure).
"""
from .arrow import (ArrowError, Comm, Decomposition, Plan, canonical_sha256, lib, options,  # noqa: F401
                    SYMBOLS, STATUS)

__all__ = ["ArrowError", "Comm", "Decomposition", "Plan", "canonical_sha256", "lib", "options"]
