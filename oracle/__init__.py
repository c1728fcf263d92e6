"""Oracle for the arrow-decomposition SpMM -- TEST INFRASTRUCTURE, NOT THE PRODUCT.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import, call, link or execute anything under
``oracle/``.  The product path (``paper_2402_19364_b200``) never imports it and
shares no code, header, table or constant generator with it; the only common
module is ``datagen`` (seeded inputs, none of the method's arithmetic).

Contents (each function cites the passage it follows):
  * O1 ``spmm`` / ``spmm_rows``  -- plain fp64 CSR SpMM Y = A X (C, OpenMP over rows),
    PAPER.md §2; exact target of Eq. (1) P:359-362 (entries partitioned).
  * O2 ``decompose.la_decompose`` -- LA-Decompose with random-spanning-forest
    arrangement and block-diagonal extraction.
  * O3 ``decompose.spmm_through_decomposition`` -- Eq. (1) / Alg. 2 without ranks.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): brute-force dense A X, closed forms
(identity, path, star), linearity, dyadic exactness, Eq. (1) reconstruction, the
arrow shape, scipy's MST, the smallest-first band lemma, worked examples
(Fig. 3; SPEC extract examples), and the survey's independent golden
hashes (tests/golden/).

Parity unpinned: arrangement *quality* versus the paper's own decompositions (the
paper prints no per-level numbers for graphs we can generate; its RNG stream is
not reproducible).  Only the bounds/invariants above apply.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

from .decompose import (Decomposition, Level, la_decompose, decomposition_sha256,  # noqa: F401
                        prune_head, captured, extract, forest_layout, minimum_spanning_forest,
                        spmm_through_decomposition, reconstruct_entries, splitmix64_int,
                        level0_tile_costs, home_ranges, homes_of)

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.path.join(_HERE, "_lib", "liboracle.so")
_lock = threading.Lock()
_lib = None


def build_lib(force: bool = False) -> str:
    """Compile oracle/spmm_ref.c (gcc -O3 -fopenmp; no -ffast-math)."""
    src = os.path.join(_HERE, "spmm_ref.c")
    if force or not os.path.exists(_LIBPATH) or os.path.getmtime(_LIBPATH) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(_LIBPATH), exist_ok=True)
        tmp = _LIBPATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-fno-fast-math", "-fopenmp",
                               "-shared", "-fPIC", src, "-o", tmp])
        os.replace(tmp, _LIBPATH)
    return _LIBPATH


def _L():
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build_lib())
            p, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
            L.oracle_spmm.argtypes = [i64, p, p, p, p, i32, i64, p, i32]
            L.oracle_spmm.restype = None
            L.oracle_spmm_rows.argtypes = [p, p, p, p, i32, i64, p, i64, p, i32]
            L.oracle_spmm_rows.restype = None
            L.oracle_num_threads.restype = ctypes.c_int
            _lib = L
    return _lib


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def num_threads() -> int:
    return int(_L().oracle_num_threads())


def spmm(n, row_ptr, col, val, X, nthreads: int = 0) -> np.ndarray:
    """O1: Y = A X in fp64 (X fp32 or fp64; fp32 values converted exactly)."""
    rp, cl, vl = _c(row_ptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    X = np.ascontiguousarray(X)
    if X.dtype not in (np.float32, np.float64):
        X = X.astype(np.float64)
    k = X.shape[1] if X.ndim == 2 else 1
    Y = np.empty((n, k), dtype=np.float64)
    _L().oracle_spmm(n, rp.ctypes.data, cl.ctypes.data, vl.ctypes.data, X.ctypes.data,
                     int(X.dtype == np.float32), k, Y.ctypes.data, nthreads)
    return Y


def spmm_rows(row_ptr, col, val, X, rows, nthreads: int = 0) -> np.ndarray:
    """O1 restricted to the sampled output rows `rows` (full-size parity on samples)."""
    rp, cl, vl = _c(row_ptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    X = np.ascontiguousarray(X)
    k = X.shape[1]
    rows = _c(rows, np.int64)
    Y = np.empty((len(rows), k), dtype=np.float64)
    _L().oracle_spmm_rows(rp.ctypes.data, cl.ctypes.data, vl.ctypes.data, X.ctypes.data,
                          int(X.dtype == np.float32), k, rows.ctypes.data, len(rows),
                          Y.ctypes.data, nthreads)
    return Y
