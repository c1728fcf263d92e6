"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

SURVEY.md §8(d) "Concrete inputs": every random choice is a splitmix64 hash, so the
graphs, matrix values and dense X are bit-identical in any implementation.  This
module contains no arithmetic of the arrow method (no decomposition, no product):
it only produces the canonical CSR A (symmetric pattern, no self-loops, no
duplicates; §2 "adjacency matrix of G") and X.

Generators (exact):
  * ``rmat(scale, ef, s)``   R-MAT/Kronecker power-law graph, Graph500 (0.57, 0.19, 0.19)
  * ``grid(side, s)``        2-D road-like planar grid
  * ``path(n, s)``           path graph
  * ``star(m)``              K_{1,m} (centre 0), ``cycle(n)``, ``tree_random(n, s)``
  * ``weblike(logn, s)``     host-block Chung-Lu (numpy RNG; statistics only, not hash-pinned)
all relabelled by ``scramble(n, s)`` where the survey says so.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBDIR = os.path.join(_HERE, "_lib")
_LIBPATH = os.path.join(_LIBDIR, "libdatagen.so")
_lock = threading.Lock()
_lib = None

SEED_GRAPH, SEED_VAL, SEED_X, SEED_DECOMP = 1, 2, 3, 4

M64 = (1 << 64) - 1


def build_lib(force: bool = False) -> str:
    """Compile datagen/gen.c into datagen/_lib/libdatagen.so (gcc, OpenMP)."""
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_LIBPATH) or os.path.getmtime(_LIBPATH) < os.path.getmtime(src):
        os.makedirs(_LIBDIR, exist_ok=True)
        tmp = _LIBPATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-shared", "-fPIC", src, "-o", tmp])
        os.replace(tmp, _LIBPATH)
    return _LIBPATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build_lib())
            p = ctypes.c_void_p
            i64, u64, i32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32
            L.dg_splitmix64.argtypes = [p, p, i64]
            L.dg_scramble_keys.argtypes = [i64, u64, p]
            L.dg_rmat_edges.argtypes = [i32, u64, i64, i64, p, p]
            L.dg_values.argtypes = [p, p, i64, u64, p]
            L.dg_fill_x.argtypes = [i64, i64, i64, u64, p]
            L.dg_fill_x_f32.argtypes = [i64, i64, i64, u64, p]
            L.dg_canonicalize.argtypes = [i64, i64, p, p, p, p]
            L.dg_canonicalize.restype = i64
            for f in (L.dg_splitmix64, L.dg_scramble_keys, L.dg_rmat_edges, L.dg_values,
                      L.dg_fill_x, L.dg_fill_x_f32):
                f.restype = None
            _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


# --------------------------------------------------------------------------- hashing
def splitmix64_py(x: int) -> int:
    """Scalar reference (pure Python ints, mod 2^64); test vectors in SURVEY §8(d)."""
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def splitmix64(x) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(x, dtype=np.uint64))
    out = np.empty_like(x)
    lib().dg_splitmix64(_ptr(x), _ptr(out), x.size)
    return out


def scramble(n: int, s: int) -> np.ndarray:
    """label[v] = rank of v in ascending (key_v, v), key_v = splitmix64(splitmix64(s+1) ^ v)."""
    key = np.empty(n, dtype=np.uint64)
    lib().dg_scramble_keys(n, s, _ptr(key))
    order = np.argsort(key, kind="stable")
    label = np.empty(n, dtype=np.int64)
    label[order] = np.arange(n, dtype=np.int64)
    return label


# --------------------------------------------------------------------------- graphs
def rmat_edges(scale: int, ef: int, s: int, chunk: int = 1 << 24):
    n = 1 << scale
    m = ef * n
    u = np.empty(m, dtype=np.int32)
    v = np.empty(m, dtype=np.int32)
    L = lib()
    for e0 in range(0, m, chunk):
        e1 = min(m, e0 + chunk)
        L.dg_rmat_edges(scale, s, e0, e1, _ptr(u[e0:e1]), _ptr(v[e0:e1]))
    label = scramble(n, s).astype(np.int32)
    return n, label[u], label[v]


def grid_edges(side: int, s: int):
    n = side * side
    ids = np.arange(n, dtype=np.int64).reshape(side, side)
    u1, v1 = ids[:, :-1].ravel(), ids[:, 1:].ravel()
    u2, v2 = ids[:-1, :].ravel(), ids[1:, :].ravel()
    u = np.concatenate([u1, u2])
    v = np.concatenate([v1, v2])
    label = scramble(n, s)
    return n, label[u], label[v]


def path_edges(n: int, s: int | None):
    u = np.arange(n - 1, dtype=np.int64)
    v = u + 1
    if s is None:
        return n, u, v
    label = scramble(n, s)
    return n, label[u], label[v]


def canonicalize(n: int, u, v):
    """Drop self-loops, merge duplicate undirected edges, store both (a,b) and (b,a),
    sort rows and columns.  Returns (row_ptr int64[n+1], col int32[nnz])."""
    u = np.ascontiguousarray(u, dtype=np.int64)
    v = np.ascontiguousarray(v, dtype=np.int64)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    col = np.empty(2 * len(u), dtype=np.int32)
    nnz = lib().dg_canonicalize(n, len(u), _ptr(u), _ptr(v), _ptr(row_ptr), _ptr(col))
    return row_ptr, col[:nnz].copy()


def canonicalize_np(n: int, u, v):
    """numpy rendering of canonicalize (cross-check in tests)."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    keep = u != v
    u, v = u[keep], v[keep]
    lo = np.minimum(u, v).astype(np.uint64)
    hi = np.maximum(u, v).astype(np.uint64)
    und = np.unique((lo << np.uint64(32)) | hi)
    lo = (und >> np.uint64(32)).astype(np.int64)
    hi = (und & np.uint64(0xFFFFFFFF)).astype(np.int64)
    rows = np.concatenate([lo, hi])
    cols = np.concatenate([hi, lo])
    key = np.sort((rows.astype(np.uint64) << np.uint64(32)) | cols.astype(np.uint64))
    rows = (key >> np.uint64(32)).astype(np.int64)
    col = (key & np.uint64(0xFFFFFFFF)).astype(np.int32)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return row_ptr, col


def values(row_ptr, col, s_val: int = SEED_VAL) -> np.ndarray:
    n = len(row_ptr) - 1
    rows = np.repeat(np.arange(n, dtype=np.int32), np.diff(row_ptr))
    col = np.ascontiguousarray(col, dtype=np.int32)
    out = np.empty(len(col), dtype=np.float64)
    lib().dg_values(_ptr(rows), _ptr(col), len(col), s_val, _ptr(out))
    return out


def make_x(n: int, k: int, s_x: int = SEED_X, dtype=np.float64) -> np.ndarray:
    out = np.empty((n, k), dtype=np.float64 if dtype == np.float64 else np.float32)
    if n == 0 or k == 0:
        return out
    if out.dtype == np.float64:
        lib().dg_fill_x(0, n, k, s_x, _ptr(out))
    else:
        lib().dg_fill_x_f32(0, n, k, s_x, _ptr(out))
    return out


class Graph:
    """Canonical CSR A with dyadic symmetric values."""

    def __init__(self, name, n, row_ptr, col, val):
        self.name, self.n = name, int(n)
        self.row_ptr, self.col, self.val = row_ptr, col, val

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def degrees(self):
        return np.diff(self.row_ptr)

    def stats(self):
        d = self.degrees()
        return {"n": self.n, "nnz": self.nnz, "isolated": int((d == 0).sum()),
                "maxdeg": int(d.max()) if self.n else 0}

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col, self.row_ptr), shape=(self.n, self.n))


def _graph(name, n, u, v, s_val):
    rp, col = canonicalize(n, u, v)
    return Graph(name, n, rp, col, values(rp, col, s_val))


def rmat(scale: int, ef: int, s: int = SEED_GRAPH, s_val: int = SEED_VAL) -> Graph:
    n, u, v = rmat_edges(scale, ef, s)
    return _graph(f"RMAT({scale},{ef},{s})", n, u, v, s_val)


def grid(side: int, s: int = SEED_GRAPH, s_val: int = SEED_VAL) -> Graph:
    n, u, v = grid_edges(side, s)
    return _graph(f"GRID({side},{s})", n, u, v, s_val)


def path(n: int, s: int | None = SEED_GRAPH, s_val: int = SEED_VAL) -> Graph:
    n, u, v = path_edges(n, s)
    return _graph(f"PATH({n},{s})", n, u, v, s_val)


def star(m: int, s_val: int = SEED_VAL) -> Graph:
    u = np.zeros(m, dtype=np.int64)
    v = np.arange(1, m + 1, dtype=np.int64)
    return _graph(f"STAR({m})", m + 1, u, v, s_val)


def cycle(n: int, s_val: int = SEED_VAL) -> Graph:
    u = np.arange(n, dtype=np.int64)
    return _graph(f"CYCLE({n})", n, u, (u + 1) % n, s_val)


def tree_random(n: int, s: int, s_val: int = SEED_VAL) -> Graph:
    """Random recursive tree: parent(v) = splitmix64(s ^ v) mod v, v >= 1, then scrambled."""
    v = np.arange(1, n, dtype=np.uint64)
    par = (splitmix64(np.uint64(s) ^ v) % v).astype(np.int64)
    label = scramble(n, s)
    return _graph(f"TREE({n},{s})", n, label[v.astype(np.int64)], label[par], s_val)


def from_edges(name, n, u, v, s_val: int = SEED_VAL) -> Graph:
    return _graph(name, n, u, v, s_val)


def weblike(logn: int, s: int = SEED_GRAPH, s_val: int = SEED_VAL, half_edges: float = 12.0) -> Graph:
    """Host-block Chung-Lu web-like graph (numpy RNG, not hash-pinned).

    Vertices sit in contiguous hidden hosts of Zipf size (mean ~64, max 4096); degree
    weights ~ truncated Zipf(2.2) scaled to `half_edges` half-edges per vertex; 80% of
    edges stay inside the host, 20% go to a Chung-Lu endpoint; labels scrambled."""
    rng = np.random.default_rng(s)
    n = 1 << logn
    sizes = []
    tot = 0
    while tot < n:
        sz = int(min(4096, rng.zipf(1.8) * 16))
        sz = min(sz, n - tot)
        sizes.append(sz)
        tot += sz
    host_start = np.repeat(np.cumsum([0] + sizes[:-1]), sizes)
    host_size = np.repeat(sizes, sizes)
    w = np.minimum(rng.zipf(2.2, size=n).astype(np.float64), n ** 0.5 * 8)
    w *= half_edges / w.mean()
    deg = rng.poisson(w / 2.0)
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    m = len(src)
    local = rng.random(m) < 0.8
    dst = np.empty(m, dtype=np.int64)
    hs, hz = host_start[src[local]], host_size[src[local]]
    dst[local] = hs + (rng.random(local.sum()) * hz).astype(np.int64)
    p = w / w.sum()
    dst[~local] = rng.choice(n, size=int((~local).sum()), p=p)
    label = scramble(n, s)
    return _graph(f"WEB({logn},{s})", n, label[src], label[dst], s_val)


def make_graph(spec: str) -> Graph:
    """Parse 'RMAT(12,4,1)', 'GRID(64,1)', 'PATH(10,1)', 'STAR(8)', 'WEB(18,1)' ..."""
    name, args = spec.split("(")
    a = [int(x) for x in args.rstrip(")").split(",") if x.strip()]
    name = name.upper()
    if name == "RMAT":
        return rmat(*a)
    if name == "GRID":
        return grid(*a)
    if name == "PATH":
        return path(*a)
    if name == "STAR":
        return star(*a)
    if name == "CYCLE":
        return cycle(*a)
    if name == "TREE":
        return tree_random(*a)
    if name == "WEB":
        return weblike(*a)
    raise ValueError(spec)


# Configs of BASELINE.json
CONFIGS = {
    "T": dict(graph="RMAT(12,4,1)", b=256, k=16, dtype="f64"),
    "G": dict(graph="GRID(1024,1)", b=4096, k=32, dtype="f32"),
    "R": dict(graph="RMAT(22,8,1)", b=16384, k=128, dtype="f32"),
    "W": dict(graph="WEB(24,1)", b=65536, k=32, dtype="f32"),
}
