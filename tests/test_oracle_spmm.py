"""O1 (plain fp64 CSR SpMM, oracle/spmm_ref.c) pinned to things other than itself.

PAPER.md §2 P:298 (Y = A X).  Pins: dense brute force (numpy triple loop / dot),
closed forms (identity, path, star), linearity,
dyadic exactness, golden Y hashes, row sampling.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

import datagen
import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "a10_golden.json")))


def _dense(g):
    A = np.zeros((g.n, g.n))
    for r in range(g.n):
        for e in range(g.row_ptr[r], g.row_ptr[r + 1]):
            A[r, g.col[e]] += g.val[e]
    return A


@pytest.mark.parametrize("spec,k", [("RMAT(8,4,2)", 5), ("GRID(12,3)", 3), ("PATH(40,1)", 1),
                                    ("TREE(200,4)", 8), ("WEB(9,2)", 4)])
def test_o1_vs_dense_bruteforce(spec, k):
    g = datagen.make_graph(spec)
    rng = np.random.default_rng(0)
    X = rng.standard_normal((g.n, k))
    Y = oracle.spmm(g.n, g.row_ptr, g.col, g.val, X)
    A = _dense(g)
    Yb = np.zeros_like(Y)
    for r in range(g.n):                          # textbook triple loop in a different order
        for c in np.flatnonzero(A[r]):
            Yb[r] += A[r, c] * X[c]
    np.testing.assert_allclose(Y, Yb, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(Y, A @ X, rtol=1e-12, atol=1e-12)


def test_o1_identity_and_closed_forms():
    n, k = 7, 3
    X = datagen.make_x(n, k)
    rp = np.arange(n + 1, dtype=np.int64)
    Y = oracle.spmm(n, rp, np.arange(n, dtype=np.int32), np.ones(n), X)
    assert np.array_equal(Y, X)                                  # A = I -> Y = X
    # path P3, ones, X = 1 -> (1, 2, 1)
    rp = np.array([0, 1, 3, 4]); col = np.array([1, 0, 2, 1], dtype=np.int32)
    Y = oracle.spmm(3, rp, col, np.ones(4), np.ones((3, 1)))
    assert Y.ravel().tolist() == [1.0, 2.0, 1.0]
    # star K_{1,8} with ones: centre 8, leaves 1
    g = datagen.star(8)
    Y = oracle.spmm(g.n, g.row_ptr, g.col, np.ones(g.nnz), np.ones((g.n, 2)))
    assert Y[0].tolist() == [8.0, 8.0] and np.all(Y[1:] == 1.0)
    # empty matrix and k = 0
    Y = oracle.spmm(4, np.zeros(5, np.int64), np.zeros(0, np.int32), np.zeros(0), np.ones((4, 2)))
    assert np.all(Y == 0)


def test_o1_linearity():
    g = datagen.rmat(9, 6, 5)
    rng = np.random.default_rng(1)
    X1, X2 = rng.standard_normal((g.n, 6)), rng.standard_normal((g.n, 6))
    Y = oracle.spmm(g.n, g.row_ptr, g.col, g.val, X1 + X2)
    Ys = oracle.spmm(g.n, g.row_ptr, g.col, g.val, X1) + oracle.spmm(g.n, g.row_ptr, g.col, g.val, X2)
    np.testing.assert_allclose(Y, Ys, rtol=1e-12, atol=1e-12)


def test_o1_dyadic_exact_any_order():
    """P11: dyadic a in 2^-12[2048,6144), X in 2^-16[0,65536): every partial sum exact ->
    the result is independent of summation order (reverse order and fp32 X agree bitwise)."""
    g = datagen.rmat(12, 4, 1)
    X = datagen.make_x(g.n, 16)
    Y = oracle.spmm(g.n, g.row_ptr, g.col, g.val, X)
    rev = np.zeros_like(Y)
    for r in range(g.n):
        for e in range(g.row_ptr[r + 1] - 1, g.row_ptr[r] - 1, -1):
            rev[r] += g.val[e] * X[g.col[e]]
    assert np.array_equal(Y, rev)
    Yf = oracle.spmm(g.n, g.row_ptr, g.col, g.val, X.astype(np.float32))
    assert np.array_equal(Y, Yf)


def test_o1_rows_sample_matches_full():
    g = datagen.rmat(10, 8, 2)
    X = datagen.make_x(g.n, 9)
    Y = oracle.spmm(g.n, g.row_ptr, g.col, g.val, X)
    rows = np.array([0, 5, 17, g.n - 1, 3, 3])
    assert np.array_equal(oracle.spmm_rows(g.row_ptr, g.col, g.val, X, rows), Y[rows])


@pytest.mark.parametrize("inst", [g for g in GOLD["instances"] if not g.get("large")],
                         ids=lambda g: g["graph"])
def test_o1_golden_y(inst):
    g = datagen.make_graph(inst["graph"])
    X = datagen.make_x(g.n, inst["k"])
    Y = oracle.spmm(g.n, g.row_ptr, g.col, g.val, X)
    assert hashlib.sha256(Y.astype("<f8").tobytes()).hexdigest() == inst["sha_y"]
    assert float.hex(math.fsum(Y.ravel())) == inst["fsum"]
