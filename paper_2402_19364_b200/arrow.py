"""Thin ctypes binding of include/arrow.h -- argument marshalling only.

Every step of arrow_spmm runs in libarrow_b200.so's sm_100a kernels; this module only
passes pointers.  There is no fallback: if the library is missing, importing the binding
raises (build it with ``python -m paper_2402_19364_b200.build``), and without a CUDA device
plan creation fails with ARROW_E_CUDA.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
from typing import Optional

import numpy as np

from . import build as _build

_LIB: Optional[ctypes.CDLL] = None

ARROW_F32, ARROW_F64 = 0, 1
ORDER = {"original": 0, "permuted": 1}
RESIDUAL = {"error": 0, "csr": 1}
BAND = {"block": 0, "strict": 1}    # ARROW_BAND_* (step 3 of LA-Decompose; strict = P:253 / Fig. 3)
FLAG_NO_GRAPHS, FLAG_DETERMINISTIC, FLAG_GPU_DECOMPOSE, FLAG_HOME_AWARE = 1, 2, 4, 8   # ARROW_FLAG_*
TRANSPORT = {"auto": 0, "p2p": 1, "nccl": 2}
STATUS = ["ARROW_OK", "ARROW_E_INVALID_ARG", "ARROW_E_BAD_CSR", "ARROW_E_NOT_SYMMETRIC", "ARROW_E_LEVELS",
          "ARROW_E_CUDA", "ARROW_E_NCCL", "ARROW_E_NOMEM", "ARROW_E_STATE", "ARROW_E_UNSUPPORTED"]
KERNELS = ["head_stage", "segments", "head_epilogue", "comm"]

# every symbol declared in include/arrow.h (checked by tests/test_boundary.py)
SYMBOLS = [
    "arrow_options_default", "arrow_plan_create", "arrow_spmm", "arrow_plan_destroy", "arrow_plan_create_ex",
    "arrow_plan_set_stream", "arrow_spmm_ex", "arrow_spmm_host", "arrow_plan_reserve", "arrow_plan_info",
    "arrow_plan_level_info", "arrow_plan_export_level", "arrow_plan_local_rows", "arrow_plan_set_profiling",
    "arrow_plan_kernel_times", "arrow_decompose", "arrow_decomposition_info", "arrow_decomposition_level_info",
    "arrow_decomposition_export_level", "arrow_decomposition_export_residual", "arrow_decomposition_save",
    "arrow_decomposition_load", "arrow_decomposition_destroy", "arrow_plan_create_from", "arrow_comm_unique_id",
    "arrow_comm_create", "arrow_comm_destroy", "arrow_status_string", "arrow_last_error", "arrow_abi_version",
    "arrow_dist_schedule", "arrow_spmm_iterate", "arrow_decompose_ex", "arrow_spmm_host_batch",
    "arrow_decompose_gpu", "arrow_decompose_homes", "arrow_decomposition_homes",
]


class ArrowError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        self.code = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        super().__init__(f"{where}: {self.code}: {detail}")


class CSR(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("row_ptr", ctypes.c_void_p),
                ("col_idx", ctypes.c_void_p), ("values", ctypes.c_void_p), ("dtype", ctypes.c_int)]


class Options(ctypes.Structure):
    _fields_ = [("compute", ctypes.c_int), ("seed", ctypes.c_uint64), ("order", ctypes.c_int32),
                ("residual", ctypes.c_int32), ("window_rows", ctypes.c_int64), ("head_chunk", ctypes.c_int32),
                ("batch_segments", ctypes.c_int32), ("band", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("transport", ctypes.c_int32), ("home_levels", ctypes.c_int32), ("reserved", ctypes.c_int32 * 2)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("b", ctypes.c_int64), ("levels", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("order", ctypes.c_int32), ("distributed", ctypes.c_int32),
                ("residual_nnz", ctypes.c_int64), ("sum_rows", ctypes.c_int64), ("isolated", ctypes.c_int64),
                ("create_seconds", ctypes.c_double), ("bytes_alg_fixed", ctypes.c_int64),
                ("bytes_alg_rows", ctypes.c_int64), ("device_bytes", ctypes.c_int64),
                ("reserved", ctypes.c_int64 * 8)]


class LevelInfo(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("n_i", ctypes.c_int64), ("head", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("head_nnz", ctypes.c_int64), ("tiles", ctypes.c_int64), ("segments", ctypes.c_int64),
                ("reserved", ctypes.c_int64 * 4)]


class KernelTimes(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 4), ("launches", ctypes.c_int64 * 4), ("calls", ctypes.c_int64),
                ("launch_ms", ctypes.c_double * 16)]


def lib() -> ctypes.CDLL:
    """Load the in-tree libarrow_b200.so (building it if the sources are newer)."""
    global _LIB
    if _LIB is None:
        path = _build.LIB
        if not os.path.exists(path) or _build.needs_build():
            try:
                _build.build()
            except Exception as e:  # no toolchain: refuse loudly, never fall back
                if not os.path.exists(path):
                    raise ImportError(f"libarrow_b200.so missing and cannot be built: {e}") from e
        L = ctypes.CDLL(path)
        p, i64, i32, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
        sig = {
            "arrow_options_default": [p],
            "arrow_plan_create": [p, i64, i32, p],
            "arrow_plan_create_ex": [p, i64, i32, p, p, p],
            "arrow_plan_create_from": [p, p, p, p],
            "arrow_spmm": [p, p, p, i64],
            "arrow_spmm_ex": [p, p, p, i64, p],
            "arrow_spmm_host": [p, p, p, i64, p],
            "arrow_spmm_host_batch": [p, p, p, i64, i64, p],
            "arrow_plan_destroy": [p],
            "arrow_plan_set_stream": [p, p],
            "arrow_plan_reserve": [p, i64],
            "arrow_plan_info": [p, p],
            "arrow_plan_level_info": [p, i32, p],
            "arrow_plan_export_level": [p, i32, p, p, p, p],
            "arrow_plan_local_rows": [p, p, p],
            "arrow_plan_set_profiling": [p, i32],
            "arrow_plan_kernel_times": [p, p],
            "arrow_decompose": [p, i64, i32, u64, i32, p],
            "arrow_decompose_ex": [p, i64, i32, u64, i32, i32, p],
            "arrow_decompose_gpu": [p, i64, i32, u64, i32, i32, p],
            "arrow_decompose_homes": [p, i64, i32, u64, i32, i32, i32, i32, i32, p],
            "arrow_decomposition_homes": [p, i32, p, p, p],
            "arrow_decomposition_info": [p, p, p, p, p],
            "arrow_decomposition_level_info": [p, i32, p],
            "arrow_decomposition_export_level": [p, i32, p, p, p, p],
            "arrow_decomposition_export_residual": [p, p, p, p],
            "arrow_decomposition_save": [p, ctypes.c_char_p],
            "arrow_decomposition_load": [ctypes.c_char_p, p],
            "arrow_decomposition_destroy": [p],
            "arrow_comm_unique_id": [p],
            "arrow_comm_create": [i32, i32, p, p],
            "arrow_comm_destroy": [p],
            "arrow_dist_schedule": [p, i32, i32, i64, i32, p, p],
            "arrow_spmm_iterate": [p, p, p, i64, i32, i32, p, p],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.arrow_status_string.argtypes = [ctypes.c_int]
        L.arrow_status_string.restype = ctypes.c_char_p
        L.arrow_last_error.restype = ctypes.c_char_p
        L.arrow_abi_version.restype = ctypes.c_int32
        _LIB = L
    return _LIB


def _check(status: int, where: str):
    if status != 0:
        raise ArrowError(status, where, lib().arrow_last_error().decode(errors="replace"))


def _csr(n, row_ptr, col, val, keep: list) -> CSR:
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(col, dtype=np.int32)
    v = np.ascontiguousarray(val)
    if v.dtype not in (np.float32, np.float64):
        v = v.astype(np.float64)
    keep += [rp, cl, v]
    return CSR(int(n), int(len(cl)), rp.ctypes.data, cl.ctypes.data, v.ctypes.data,
               ARROW_F64 if v.dtype == np.float64 else ARROW_F32)


def _dtype_code(dtype) -> int:
    if dtype is None:
        return -1
    s = str(dtype).replace("torch.", "")
    if s in ("float32", "f32", "fp32"):
        return ARROW_F32
    if s in ("float64", "f64", "fp64", "double"):
        return ARROW_F64
    raise ValueError(f"unsupported dtype {dtype}")


def options(dtype=None, seed: int = 4, order: str = "original", residual: str = "error", window_rows: int = 0,
            head_chunk: int = 0, batch_segments: int = 0, band: str = "block", flags: int = 0,
            transport: str = "auto", home_levels: int = 0) -> Options:
    o = Options()
    _check(lib().arrow_options_default(ctypes.byref(o)), "arrow_options_default")
    o.compute = _dtype_code(dtype)
    o.seed = seed
    o.order = ORDER[order]
    o.residual = RESIDUAL[residual]
    o.window_rows = window_rows
    o.head_chunk = head_chunk
    o.batch_segments = batch_segments
    o.band = BAND[band]
    o.flags = flags
    o.transport = TRANSPORT[transport]
    o.home_levels = home_levels
    return o


def canonical_sha256(levels) -> str:
    """sha256 of (int64 L; per level int64 rows, int32 perm, int64 row_ptr, int32 col, float64 val)."""
    h = hashlib.sha256()
    h.update(np.int64(len(levels)).tobytes())
    for perm, rp, col, val in levels:
        h.update(np.int64(len(perm)).tobytes())
        h.update(perm.astype("<i4").tobytes())
        h.update(rp.astype("<i8").tobytes())
        h.update(col.astype("<i4").tobytes())
        h.update(val.astype("<f8").tobytes())
    return h.hexdigest()


class Decomposition:
    """LA-Decompose result, held on the host.  device="cpu" (no GPU needed) or device="cuda" (the
    current CUDA device; the identical decomposition).  homes = G > 1: home-set-aware levels >= 1 for
    a G-rank plan (arrow_decompose_homes, reading R25)."""

    def __init__(self, n, row_ptr, col, val, b: int, levels: int = 0, seed: int = 4, keep_residual: bool = False,
                 band: str = "block", device: str = "cpu", homes: int = 1, home_levels: int = 0, _handle=None):
        self._h = ctypes.c_void_p()
        if _handle is not None:
            self._h = _handle
            return
        keep: list = []
        A = _csr(n, row_ptr, col, val, keep)
        if device not in ("cpu", "cuda"):
            raise ValueError(f"device must be 'cpu' or 'cuda', not {device!r}")
        if homes != 1:
            _check(lib().arrow_decompose_homes(ctypes.byref(A), b, levels, seed, int(keep_residual), BAND[band], homes,
                                               home_levels, 1 if device == "cuda" else 0, ctypes.byref(self._h)),
                   "arrow_decompose_homes")
            return
        fn = "arrow_decompose_gpu" if device == "cuda" else "arrow_decompose_ex"
        _check(getattr(lib(), fn)(ctypes.byref(A), b, levels, seed, int(keep_residual), BAND[band],
                                  ctypes.byref(self._h)), fn)

    @classmethod
    def load(cls, path: str) -> "Decomposition":
        h = ctypes.c_void_p()
        _check(lib().arrow_decomposition_load(path.encode(), ctypes.byref(h)), "arrow_decomposition_load")
        return cls(0, None, None, None, 2, _handle=h)

    def save(self, path: str):
        _check(lib().arrow_decomposition_save(self._h, path.encode()), "arrow_decomposition_save")

    def info(self) -> dict:
        n, b, r = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        L = ctypes.c_int32()
        _check(lib().arrow_decomposition_info(self._h, ctypes.byref(n), ctypes.byref(b), ctypes.byref(L),
                                              ctypes.byref(r)), "arrow_decomposition_info")
        return {"n": n.value, "b": b.value, "levels": L.value, "residual_nnz": r.value}

    def homes(self, level: int = -1):
        """(G, ranges): level -1 -> the pi_0 home ranges; level in 1..home_levels -> first position of
        each home's trees (G + 1 values); ranges is None when G == 1."""
        G, HL = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().arrow_decomposition_homes(self._h, level, ctypes.byref(G), ctypes.byref(HL), None),
               "arrow_decomposition_homes")
        if G.value == 1:
            return 1, None
        r = np.zeros(G.value + 1, np.int64)
        _check(lib().arrow_decomposition_homes(self._h, level, None, None, r.ctypes.data), "arrow_decomposition_homes")
        return G.value, r

    def home_levels(self) -> int:
        HL = ctypes.c_int32()
        _check(lib().arrow_decomposition_homes(self._h, -1, None, ctypes.byref(HL), None), "arrow_decomposition_homes")
        return HL.value

    def level_info(self, i: int) -> dict:
        li = LevelInfo()
        _check(lib().arrow_decomposition_level_info(self._h, i, ctypes.byref(li)), "arrow_decomposition_level_info")
        return {f: getattr(li, f) for f, _ in LevelInfo._fields_ if f != "reserved"}

    def export_level(self, i: int):
        li = self.level_info(i)
        perm = np.empty(li["rows"], np.int32)
        rp = np.empty(li["rows"] + 1, np.int64)
        col = np.empty(li["nnz"], np.int32)
        val = np.empty(li["nnz"], np.float64)
        _check(lib().arrow_decomposition_export_level(self._h, i, perm.ctypes.data, rp.ctypes.data, col.ctypes.data,
                                                      val.ctypes.data), "arrow_decomposition_export_level")
        return perm, rp, col, val

    def export_residual(self):
        m = self.info()["residual_nnz"]
        u, v, a = np.empty(m, np.int32), np.empty(m, np.int32), np.empty(m, np.float64)
        _check(lib().arrow_decomposition_export_residual(self._h, u.ctypes.data, v.ctypes.data, a.ctypes.data),
               "arrow_decomposition_export_residual")
        return u, v, a

    def sha256(self) -> str:
        return canonical_sha256([self.export_level(i) for i in range(self.info()["levels"])])

    def dist_schedule(self, nranks: int, rank: int, window_rows: int = 0, head_chunk: int = 0) -> dict:
        """Host-only distributed schedule of `rank` (arrow_dist_schedule): pi_0 row range and per-level
        forward/reverse exchange row counts per peer, local entries/segments/heads/zero rows."""
        L = self.info()["levels"]
        lohi = np.zeros(2, np.int64)
        per = 4 * nranks + 4
        counts = np.zeros(max(1, L * per), np.int64)
        _check(lib().arrow_dist_schedule(self._h, nranks, rank, window_rows, head_chunk, lohi.ctypes.data,
                                         counts.ctypes.data), "arrow_dist_schedule")
        levels = []
        for i in range(L):
            c = counts[i * per:(i + 1) * per]
            G = nranks
            levels.append({"send": c[0:G].copy(), "recv": c[G:2 * G].copy(), "out": c[2 * G:3 * G].copy(),
                           "in": c[3 * G:4 * G].copy(), "entries": int(c[4 * G]), "segments": int(c[4 * G + 1]),
                           "heads": int(c[4 * G + 2]), "zero_rows": int(c[4 * G + 3])})
        return {"lo": int(lohi[0]), "hi": int(lohi[1]), "levels": levels}

    def close(self):
        if self._h:
            lib().arrow_decomposition_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _torch_ptr(t, dtype_code: int, rows: int, k: int):
    import torch
    if not t.is_cuda:
        raise ValueError("arrow_spmm needs CUDA tensors (use spmm_host for host buffers)")
    want = torch.float64 if dtype_code == ARROW_F64 else torch.float32
    if t.dtype != want or not t.is_contiguous() or tuple(t.shape) != (rows, k):
        raise ValueError(f"expected contiguous {want} tensor of shape {(rows, k)}, got {t.dtype} {tuple(t.shape)}")
    return t.data_ptr()


class Plan:
    """Device plan (arrow_plan_create_ex / arrow_plan_create_from)."""

    def __init__(self, n=None, row_ptr=None, col=None, val=None, b: int = 2, levels: int = 0, dtype=None,
                 seed: int = 4, order: str = "original", residual: str = "error", window_rows: int = 0,
                 head_chunk: int = 0, batch_segments: int = 0, comm=None,
                 decomposition: Optional[Decomposition] = None, band: str = "block", flags: int = 0,
                 transport: str = "auto", home_levels: int = 0):
        self._h = ctypes.c_void_p()
        opt = options(dtype, seed, order, residual, window_rows, head_chunk, batch_segments, band, flags, transport,
                      home_levels)
        comm_h = comm.handle if comm is not None else None
        if decomposition is not None:
            _check(lib().arrow_plan_create_from(decomposition._h, ctypes.byref(opt), comm_h, ctypes.byref(self._h)),
                   "arrow_plan_create_from")
        else:
            keep: list = []
            A = _csr(n, row_ptr, col, val, keep)
            _check(lib().arrow_plan_create_ex(ctypes.byref(A), b, levels, ctypes.byref(opt), comm_h,
                                              ctypes.byref(self._h)), "arrow_plan_create_ex")
        self._info = self.info()
        self.local_begin, self.local_end = self.local_rows()

    @property
    def handle(self):
        return self._h

    @property
    def dtype_code(self) -> int:
        return self._info["dtype"]

    @property
    def np_dtype(self):
        return np.float64 if self.dtype_code == ARROW_F64 else np.float32

    @property
    def torch_dtype(self):
        import torch
        return torch.float64 if self.dtype_code == ARROW_F64 else torch.float32

    def info(self) -> dict:
        pi = PlanInfo()
        _check(lib().arrow_plan_info(self._h, ctypes.byref(pi)), "arrow_plan_info")
        return {f: getattr(pi, f) for f, _ in PlanInfo._fields_ if f != "reserved"}

    def level_info(self, i: int) -> dict:
        li = LevelInfo()
        _check(lib().arrow_plan_level_info(self._h, i, ctypes.byref(li)), "arrow_plan_level_info")
        return {f: getattr(li, f) for f, _ in LevelInfo._fields_ if f != "reserved"}

    def local_rows(self):
        b, e = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().arrow_plan_local_rows(self._h, ctypes.byref(b), ctypes.byref(e)), "arrow_plan_local_rows")
        return b.value, e.value

    def bytes_alg(self, k: int) -> int:
        """Algorithmic bytes per SpMM: B_alg(k) = fixed + rows * k * sizeof(dtype)."""
        s = 8 if self.dtype_code == ARROW_F64 else 4
        return int(self._info["bytes_alg_fixed"] + self._info["bytes_alg_rows"] * k * s)

    def export_level(self, i: int):
        li = self.level_info(i)
        perm = np.empty(li["rows"], np.int32)
        rp = np.empty(li["rows"] + 1, np.int64)
        col = np.empty(li["nnz"], np.int32)
        val = np.empty(li["nnz"], self.np_dtype)
        _check(lib().arrow_plan_export_level(self._h, i, perm.ctypes.data, rp.ctypes.data, col.ctypes.data,
                                             val.ctypes.data), "arrow_plan_export_level")
        return perm, rp, col, val

    def sha256(self) -> str:
        return canonical_sha256([self.export_level(i) for i in range(self._info["levels"])])

    def reserve(self, k: int):
        _check(lib().arrow_plan_reserve(self._h, k), "arrow_plan_reserve")

    def set_stream(self, stream_ptr: int):
        _check(lib().arrow_plan_set_stream(self._h, stream_ptr), "arrow_plan_set_stream")

    def spmm_ptr(self, x_ptr: int, y_ptr: int, k: int, stream_ptr: int = 0):
        _check(lib().arrow_spmm_ex(self._h, x_ptr, y_ptr, k, stream_ptr), "arrow_spmm_ex")

    def spmm(self, X, Y=None, stream=None):
        """Y = A X for CUDA tensors, on `stream` (default: torch's current stream)."""
        import torch
        rows = self.local_end - self.local_begin
        k = X.shape[1]
        if Y is None:
            Y = torch.empty((rows, k), dtype=X.dtype, device=X.device)
        xp = _torch_ptr(X, self.dtype_code, rows, k)
        yp = _torch_ptr(Y, self.dtype_code, rows, k)
        s = (stream or torch.cuda.current_stream(X.device)).cuda_stream
        self.spmm_ptr(xp, yp, k, s)
        return Y

    def spmm_iterate(self, X, iters: int, activation: str = "relu", Y=None, stream=None):
        """X_{t+1} = act(A X_t) for t < iters (arrow_spmm_iterate).  X (device tensor, n x k) holds
        X_0 and is overwritten, as is Y (allocated if None); returns the tensor that holds X_iters."""
        import torch
        rows = self.local_end - self.local_begin
        k = X.shape[1]
        if Y is None:
            Y = torch.empty((rows, k), dtype=X.dtype, device=X.device)
        xp = _torch_ptr(X, self.dtype_code, rows, k)
        yp = _torch_ptr(Y, self.dtype_code, rows, k)
        act = {"none": 0, "relu": 1}[activation]
        s = (stream or torch.cuda.current_stream(X.device)).cuda_stream
        in_y = ctypes.c_int32()
        _check(lib().arrow_spmm_iterate(self._h, xp, yp, k, iters, act, s, ctypes.byref(in_y)), "arrow_spmm_iterate")
        return Y if in_y.value else X

    def spmm_host(self, X: np.ndarray, Y: Optional[np.ndarray] = None, stream_ptr: int = 0) -> np.ndarray:
        """End-to-end call with host buffers (H2D, kernels, D2H inside arrow_spmm_host)."""
        rows = self.local_end - self.local_begin
        X = np.ascontiguousarray(X, dtype=self.np_dtype)
        k = X.shape[1]
        if X.shape[0] != rows:
            raise ValueError(f"X must have {rows} rows")
        if Y is None:
            Y = np.empty((rows, k), self.np_dtype)
        _check(lib().arrow_spmm_host(self._h, X.ctypes.data, Y.ctypes.data, k, stream_ptr), "arrow_spmm_host")
        return Y

    def spmm_host_batch(self, Xs, Ys=None, stream_ptr: int = 0):
        """Y_c = A X_c for a list of host buffers, copies pipelined with the kernels
        (arrow_spmm_host_batch; pinned buffers give the overlap)."""
        rows = self.local_end - self.local_begin
        Xs = [np.ascontiguousarray(X, dtype=self.np_dtype) for X in Xs]
        if not Xs:
            return []
        k = Xs[0].shape[1]
        for X in Xs:
            if X.shape != (rows, k):
                raise ValueError(f"every X must be {rows} x {k}")
        if Ys is None:
            Ys = [np.empty((rows, k), self.np_dtype) for _ in Xs]
        if len(Ys) != len(Xs) or any(Y.shape != (rows, k) or Y.dtype != self.np_dtype or not Y.flags.c_contiguous
                                     for Y in Ys):
            raise ValueError("Ys must match Xs (shape, dtype, C-contiguous)")
        xp = (ctypes.c_void_p * len(Xs))(*[X.ctypes.data for X in Xs])
        yp = (ctypes.c_void_p * len(Ys))(*[Y.ctypes.data for Y in Ys])
        _check(lib().arrow_spmm_host_batch(self._h, xp, yp, len(Xs), k, stream_ptr), "arrow_spmm_host_batch")
        return Ys

    def set_profiling(self, on: bool):
        _check(lib().arrow_plan_set_profiling(self._h, int(on)), "arrow_plan_set_profiling")

    def kernel_times(self) -> dict:
        kt = KernelTimes()
        _check(lib().arrow_plan_kernel_times(self._h, ctypes.byref(kt)), "arrow_plan_kernel_times")
        c = max(1, kt.calls)
        return {"calls": kt.calls, "launch_ms": [round(kt.launch_ms[i] / c, 4) for i in range(16) if kt.launch_ms[i] > 0],
                **{KERNELS[i]: {"ms": kt.ms[i], "launches": kt.launches[i]} for i in range(4)}}

    def close(self):
        if self._h:
            lib().arrow_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Comm:
    """NCCL communicator for distributed plans (arrow_comm_create)."""

    def __init__(self, nranks: int, rank: int, unique_id: bytes):
        self._h = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(unique_id)
        _check(lib().arrow_comm_create(nranks, rank, buf, ctypes.byref(self._h)), "arrow_comm_create")

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        _check(lib().arrow_comm_unique_id(buf), "arrow_comm_unique_id")
        return bytes(buf)

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib().arrow_comm_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
