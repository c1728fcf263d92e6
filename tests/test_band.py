"""NEXT-2: the strict-band variant of LA-Decompose step 3.

Step 3 keeps "the first b rows and columns and a symmetric b-wide band around the
diagonal"; arrow-width b means "for all i>b and j>b ... if A_ij != 0 then |i-j| <= b" (P:253,
1-based).  The default reading R3 captures the diagonal b x b tiles (Alg. 1's block band,
P:467/P:473); band="strict" captures every |p - q| <= b (0-based positions), as Fig. 3 draws it.

Pins (oracle, -m "not gpu"):
  * Fig. 3 worked example (tests/golden/fig3_la_decompose.json): the strict band
    leaves exactly the drawn "outside" edge {(2,5)}; the level-1 rules then capture it (order 2).
  * closed form: a path laid out in its own order has every edge at distance 1, so the strict
    band captures all of it for any b >= 2 (the block band leaves the tile-crossing edges,
    SPEC S:269: {(3,4),(5,6),(7,8)} for P10, b=2).
  * containment: a diagonal b x b tile has |p - q| <= b - 1, so for any arrangement the strict
    capture contains the block capture, and since the level-0 arrangement does not depend on
    the band, level 0 of the strict decomposition leaves a subset of the block remainder.
  * P1-P4 invariants with the strict shape, and O3 == O1 bitwise on dyadic data.
C ABI (-m "not gpu"): the C++ decomposer reproduces the strict oracle bit-exactly, save/load
keeps the band, bad band values are rejected.  GPU parity for the strict band lives in
test_gpu_parity.py::test_strict_band_parity.
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

import datagen
import oracle
import paper_2402_19364_b200 as ab
from paper_2402_19364_b200.arrow import ArrowError

FIG3 = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig3_la_decompose.json")))


def _sym(edges):
    u = [a for a, b in edges] + [b for a, b in edges]
    v = [b for a, b in edges] + [a for a, b in edges]
    return np.array(u, np.int64), np.array(v, np.int64)


def _und(u, v):
    return sorted({(int(min(a, b)), int(max(a, b))) for a, b in zip(u, v)})


def _csr_from_edges(n, u, v, a):
    o = np.lexsort((v, u))
    u, v, a = u[o], v[o], a[o]
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(u, minlength=n), out=rp[1:])
    return rp, v, a


def test_fig3_strict_band():
    edges = FIG3["pruned"] + FIG3["banded"] + FIG3["outside"]
    u, v = _sym(edges)
    a = np.ones(len(u))
    (p, q, _), (ru, rv, ra) = oracle.extract(u, v, a, np.arange(FIG3["n"]), FIG3["b"], band="strict")
    assert [list(e) for e in _und(ru, rv)] == FIG3["expected_strict_band_remainder"]
    # everything the figure draws as pruned or banded is captured
    assert set(_und(p, q)) == {tuple(e) for e in FIG3["pruned"] + FIG3["banded"]}
    # level 1 on the remainder: 2 vertices <= b, both in the head (degree 1 each, id asc)
    rp, col, val = _csr_from_edges(FIG3["n"], ru, rv, ra)
    dec = oracle.la_decompose(FIG3["n"], rp, col, val, FIG3["b"], band="strict")
    assert dec.order == 1 and dec.levels[0].perm[:2].tolist() == [2, 5]
    assert dec.levels[0].nnz == 2


@pytest.mark.parametrize("n,b", [(10, 2), (100, 4), (37, 3)])
def test_path_identity_closed_form(n, b):
    u = np.arange(n - 1, dtype=np.int64)
    uu, vv = np.concatenate([u, u + 1]), np.concatenate([u + 1, u])
    a = np.ones(len(uu))
    _, (ru, _, _) = oracle.extract(uu, vv, a, np.arange(n), b, band="strict")
    assert len(ru) == 0
    _, (bu, bv, _) = oracle.extract(uu, vv, a, np.arange(n), b, band="block")
    # block band: an edge (i, i+1) is lost iff it crosses a tile boundary outside the head
    lost = [(i, i + 1) for i in range(b, n - 1) if (i + 1) % b == 0]
    assert _und(bu, bv) == lost
    if (n, b) == (10, 2):
        assert lost == [(3, 4), (5, 6), (7, 8)]


@pytest.mark.parametrize("spec,b", [("RMAT(10,8,1)", 64), ("GRID(40,2)", 32), ("WEB(10,1)", 64)])
def test_strict_contains_block(spec, b):
    g = datagen.make_graph(spec)
    eu = np.repeat(np.arange(g.n), np.diff(g.row_ptr))
    ev = g.col.astype(np.int64)
    rng = np.random.default_rng(5)
    for _ in range(3):
        order = rng.permutation(g.n)
        pos = np.empty(g.n, np.int64)
        pos[order] = np.arange(g.n)
        blk = oracle.captured(pos[eu], pos[ev], b, "block")
        strict = oracle.captured(pos[eu], pos[ev], b, "strict")
        assert np.all(strict[blk])
    db = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, b)
    ds = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, b, band="strict")
    # same level-0 arrangement (it does not depend on the band), superset capture
    assert np.array_equal(db.levels[0].perm, ds.levels[0].perm)
    assert ds.levels[0].nnz >= db.levels[0].nnz
    assert sum(lv.n_i for lv in ds.levels[1:]) <= sum(lv.n_i for lv in db.levels[1:]) * 1.05 + 8


@pytest.mark.parametrize("spec,b", [("RMAT(10,8,1)", 64), ("RMAT(12,4,1)", 256), ("GRID(40,2)", 32),
                                    ("PATH(300,3)", 4), ("TREE(500,2)", 8), ("WEB(11,3)", 64), ("RMAT(9,8,7)", 3),
                                    ("STAR(20)", 2), ("CYCLE(50)", 2)])
def test_strict_invariants(spec, b):
    g = datagen.make_graph(spec)
    dec = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, b, band="strict")
    # P1: reconstruction (multiset, bit-equal values)
    ru, rv, ra = oracle.reconstruct_entries(dec)
    o = np.lexsort((ra, rv, ru))
    eu = np.repeat(np.arange(g.n), np.diff(g.row_ptr))
    o2 = np.lexsort((g.val, g.col, eu))
    assert np.array_equal(ru[o], eu[o2]) and np.array_equal(rv[o], g.col[o2].astype(np.int64))
    assert np.array_equal(ra[o].view(np.int64), g.val[o2].view(np.int64))
    prev = None
    for i, lv in enumerate(dec.levels):
        p = np.repeat(np.arange(lv.rows), np.diff(lv.row_ptr))
        q = lv.col
        # P2 (strict): head rows/cols or |p - q| <= b -- arrow-width <= b as P:253 defines it
        off = (p >= b) & (q >= b)
        assert np.all(np.abs(p[off] - q[off]) <= b)
        # P3
        assert len(np.unique(lv.perm)) == lv.rows and lv.head == min(b, lv.n_i)
        assert lv.rows == (g.n if i == 0 else lv.n_i)
        assert p.max(initial=-1) < lv.n_i and q.max(initial=-1) < lv.n_i
        B = sp.csr_matrix((np.ones(lv.nnz), lv.col, lv.row_ptr), shape=(lv.rows, lv.rows))
        assert (B != B.T).nnz == 0
        if prev is not None:
            assert lv.n_i <= prev
        prev = lv.n_i
        assert lv.nnz >= 1           # P4
    # O3 == O1 bitwise on dyadic data (P11)
    X = datagen.make_x(g.n, 3)
    assert np.array_equal(oracle.spmm_through_decomposition(dec, X), oracle.spmm(g.n, g.row_ptr, g.col, g.val, X))


def test_strict_depth_gate_paths():
    """Scrambled paths: the strict band never needs more levels than the block band (the
    containment above, level by level, is not guaranteed after level 0; checked empirically
    on the P8 corpus)."""
    for n in (100, 1000, 5000):
        for b in (2, 4, 64):
            g = datagen.path(n, 7)
            ds = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, b, band="strict")
            assert ds.order <= 3


# ------------------------------------------------------------------------------ C ABI (host)
@pytest.mark.parametrize("spec,b", [("RMAT(10,8,1)", 64), ("RMAT(12,4,1)", 256), ("GRID(40,2)", 32),
                                    ("PATH(300,3)", 4), ("TREE(500,2)", 8), ("WEB(11,3)", 64), ("RMAT(9,8,7)", 3),
                                    ("STAR(20)", 2), ("CYCLE(50)", 2), ("RMAT(13,8,2)", 4096), ("RMAT(11,8,5)", 2)])
def test_decomposer_strict_bit_exact_vs_oracle(spec, b):
    g = datagen.make_graph(spec)
    D = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, b, band="strict")
    ref = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, b, band="strict")
    assert D.info()["levels"] == ref.order
    for i, lv in enumerate(ref.levels):
        perm, rp, col, val = D.export_level(i)
        assert np.array_equal(perm, lv.perm) and np.array_equal(rp, lv.row_ptr)
        assert np.array_equal(col, lv.col) and np.array_equal(val.view(np.int64), lv.val.view(np.int64))
    assert D.sha256() == oracle.decomposition_sha256(ref)


def test_strict_save_load_and_errors(tmp_path):
    g = datagen.make_graph("RMAT(10,8,1)")
    D = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 64, band="strict")
    path = str(tmp_path / "strict.adec")
    D.save(path)
    D2 = ab.Decomposition.load(path)
    assert D2.sha256() == D.sha256()
    Db = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 64)
    assert Db.sha256() != D.sha256()
    L = ab.lib()
    from paper_2402_19364_b200.arrow import _csr
    import ctypes
    keep: list = []
    A = _csr(g.n, g.row_ptr, g.col, g.val, keep)
    h = ctypes.c_void_p()
    assert L.arrow_decompose_ex(ctypes.byref(A), 64, 0, 4, 0, 2, ctypes.byref(h)) == ab.STATUS.index("ARROW_E_INVALID_ARG")
    assert not h.value
    with pytest.raises(KeyError):
        ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 64, band="tridiagonal")


# ---------------------------------------------------------------- the band boundary |p - q| = b, b + 1
BOUNDARY = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "band_boundary.json")))


def _boundary_graph():
    """tests/golden/band_boundary.json: hubs joined to each other and to every tree vertex + the tree."""
    n, hubs = BOUNDARY["n"], BOUNDARY["hubs"]
    tree = [v for v in range(n) if v not in hubs]
    edges = [(h1, h2) for i, h1 in enumerate(hubs) for h2 in hubs[i + 1:]]
    edges += [(h, v) for h in hubs for v in tree] + [tuple(e) for e in BOUNDARY["tree_edges"]]
    u, v = _sym(edges)
    a = np.ones(len(u))
    rp, col, val = _csr_from_edges(n, u, v, a)
    return n, rp, col, val


def _level1_edges(levels):
    """undirected original-id edges of level 1 (the level-0 remainder)"""
    perm, rp, col = levels[1][0], levels[1][1], levels[1][2]
    out = set()
    for p in range(len(perm)):
        for e in range(rp[p], rp[p + 1]):
            a, b = int(perm[p]), int(perm[col[e]])
            out.add((min(a, b), max(a, b)))
    return sorted(out)


@pytest.mark.parametrize("band", ["strict", "block"])
def test_band_boundary_worked_example_oracle(band):
    n, rp, col, val = _boundary_graph()
    b = BOUNDARY["b"]
    dec = oracle.la_decompose(n, rp, col, val, b, band=band)
    assert dec.order == BOUNDARY["expected_order"]
    assert dec.levels[0].perm.tolist() == BOUNDARY["expected_level0_perm"]
    levels = [(L.perm, L.row_ptr, L.col) for L in dec.levels]
    assert _level1_edges(levels) == [tuple(e) for e in BOUNDARY[f"expected_{band}_remainder"]]
    assert dec.levels[1].perm[:dec.levels[1].n_i].tolist() == BOUNDARY[f"expected_{band}_level1_perm"]
    # the predicate itself at the boundary (positions >= b): distance b in, b + 1 out (strict)
    p, q = np.array([8, 8, 4]), np.array([12, 13, 8])
    want = {"strict": [True, False, True], "block": [False, False, False]}[band]
    assert oracle.captured(p, q, b, band=band).tolist() == want


@pytest.mark.parametrize("band", ["strict", "block"])
def test_band_boundary_worked_example_decomposer(band):
    """The C++ decomposer (C ABI) on the same hand-derived instance: pins its step-3 rule at the
    boundary independently of the oracle."""
    n, rp, col, val = _boundary_graph()
    d = ab.Decomposition(n, rp, col, val, BOUNDARY["b"], band=band)
    assert d.info()["levels"] == BOUNDARY["expected_order"]
    levels = [d.export_level(i)[:3] for i in range(2)]
    assert levels[0][0].tolist() == BOUNDARY["expected_level0_perm"]
    assert _level1_edges(levels) == [tuple(e) for e in BOUNDARY[f"expected_{band}_remainder"]]
    li = d.level_info(1)
    assert levels[1][0][:li["n_i"]].tolist() == BOUNDARY[f"expected_{band}_level1_perm"]
