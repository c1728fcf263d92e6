"""Seeded input generators (datagen): determinism, canonical CSR, golden graph stats.

Pins: splitmix64 test vectors; per-graph n / nnz / isolated / Delta from
the survey's independent golden table (tests/golden/a10_golden.json).
"""
import json
import os

import numpy as np
import pytest

import datagen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "a10_golden.json")))


def test_splitmix64_vectors():
    assert datagen.splitmix64_py(0) == 0xE220A8397B1DCDAF
    assert datagen.splitmix64_py(1) == 0x910A2DEC89025CC1
    xs = [0, 1, 2, 12345, (1 << 64) - 1, 0xDEADBEEF]
    got = datagen.splitmix64(np.array(xs, dtype=np.uint64))
    assert [int(g) for g in got] == [datagen.splitmix64_py(x) for x in xs]


def test_scramble_is_permutation():
    for n in (1, 2, 10, 1000):
        lab = datagen.scramble(n, 7)
        assert sorted(lab.tolist()) == list(range(n))


@pytest.mark.parametrize("inst", [g for g in GOLD["instances"] if not g.get("large")],
                         ids=lambda g: g["graph"])
def test_golden_graph_stats(inst):
    g = datagen.make_graph(inst["graph"])
    s = g.stats()
    assert (s["n"], s["nnz"], s["isolated"], s["maxdeg"]) == \
        (inst["n"], inst["nnz"], inst["isolated"], inst["maxdeg"])


@pytest.mark.parametrize("spec", ["RMAT(10,8,3)", "GRID(17,2)", "PATH(50,5)", "TREE(300,9)", "STAR(9)",
                                  "CYCLE(12)", "WEB(12,1)"])
def test_canonical_csr(spec):
    g = datagen.make_graph(spec)
    rp, col, val = g.row_ptr, g.col, g.val
    assert rp[0] == 0 and np.all(np.diff(rp) >= 0) and rp[-1] == len(col)
    rows = np.repeat(np.arange(g.n), np.diff(rp))
    assert np.all(rows != col), "no self-loops"
    for r in range(min(g.n, 200)):
        c = col[rp[r]:rp[r + 1]]
        assert np.all(np.diff(c) > 0), "strictly increasing within a row"
    S = g.to_scipy()
    assert (S != S.T).nnz == 0, "symmetric pattern and values"
    assert np.all((val >= 0.5) & (val < 1.5))
    assert np.all(val * 4096 == np.round(val * 4096)), "dyadic values"


def test_x_dyadic_and_deterministic():
    X = datagen.make_x(100, 7)
    assert np.all((X >= 0) & (X < 1))
    assert np.all(X * 65536 == np.round(X * 65536))
    assert np.array_equal(X, datagen.make_x(100, 7))
    Xf = datagen.make_x(100, 7, dtype=np.float32)
    assert np.array_equal(Xf.astype(np.float64), X)
    # definition: X[i,j] = (splitmix64(s_X ^ (i*k+j)) >> 48) / 65536
    assert X[3, 4] == (datagen.splitmix64_py(3 ^ (3 * 7 + 4)) >> 48) / 65536


def test_rmat_definition_small():
    # first edge of RMAT(4, 1, 1) recomputed from the written definition
    base = datagen.splitmix64_py(1)
    u = v = 0
    for l in range(4):
        r = (datagen.splitmix64_py(base ^ (64 * 0 + l)) >> 11) * 2.0 ** -53
        u |= int(r >= 0.76) << l
        v |= int((0.57 <= r < 0.76) or r >= 0.95) << l
    n, uu, vv = datagen.rmat_edges(4, 1, 1)
    lab = datagen.scramble(16, 1)
    assert (uu[0], vv[0]) == (lab[u], lab[v])
