"""O2 (LA-Decompose) and O3 (Eq. (1) evaluation) pinned to the paper and mathematics.

Pins: Eq. (1) reconstruction, the arrow shape
(P:253), perm/size invariants, progress, MSF == scipy's MST, the
smallest-first band lemma and contiguity, the complete-binary-tree closed
form and the heavy-light lambda bound, worked examples (Fig. 3
P:595-790), depth gates, O3 == O1 bitwise on dyadic
data (P11) and the survey's independent golden hashes (A.10).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import minimum_spanning_tree

import datagen
import oracle
from oracle.decompose import splitmix64_vec

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "a10_golden.json")))
FIG3 = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig3_la_decompose.json")))


def _entries(g):
    return np.repeat(np.arange(g.n), np.diff(g.row_ptr)), g.col.astype(np.int64), g.val


def _sorted_triples(u, v, a):
    o = np.lexsort((a, v, u))
    return u[o], v[o], a[o]


def check_invariants(g, dec):
    """P1-P4 on a decomposition of graph g."""
    b = dec.b
    # P1: reconstruction, exact multiset equality with bit-equal values
    ru, rv, ra = _sorted_triples(*oracle.reconstruct_entries(dec))
    eu, ev, ea = _sorted_triples(*_entries(g))
    assert np.array_equal(ru, eu) and np.array_equal(rv, ev) and np.array_equal(ra.view(np.int64), ea.view(np.int64))
    prev_n = None
    remaining = g.nnz
    for i, lv in enumerate(dec.levels):
        # P3: perm injective into [0,n), |perm| = rows; rows = n at level 0 else n_i
        assert len(np.unique(lv.perm)) == len(lv.perm) and lv.perm.min() >= 0 and lv.perm.max() < g.n
        assert lv.rows == (g.n if i == 0 else lv.n_i)
        assert lv.head == min(b, lv.n_i)
        if prev_n is not None:
            assert lv.n_i <= prev_n
        prev_n = lv.n_i
        p = np.repeat(np.arange(lv.rows), np.diff(lv.row_ptr))
        q = lv.col
        # P2: shape -- head rows/cols or the same diagonal tile; hence arrow-width <= b
        assert np.all((p < b) | (q < b) | (p // b == q // b))
        off = (p >= b) & (q >= b)
        assert np.all(np.abs(p[off] - q[off]) <= b - 1)
        # rows with entries lie in [0, n_i) (A_i-isolated vertices excluded, R8)
        assert p.max(initial=-1) < lv.n_i and q.max(initial=-1) < lv.n_i
        # symmetric pattern of B_i
        B = sp.csr_matrix((np.ones(lv.nnz), lv.col, lv.row_ptr), shape=(lv.rows, lv.rows))
        assert (B != B.T).nnz == 0
        # canonical CSR: columns strictly increasing per row
        for r in range(min(lv.rows, 64)):
            assert np.all(np.diff(lv.col[lv.row_ptr[r]:lv.row_ptr[r + 1]]) > 0)
        # P4: progress (every level captures >= 1 entry)
        assert lv.nnz >= 1
        remaining -= lv.nnz
    assert remaining == (0 if dec.residual is None else len(dec.residual[0]))


@pytest.mark.parametrize("spec,b", [("RMAT(10,8,1)", 64), ("RMAT(12,4,1)", 256), ("GRID(40,2)", 32),
                                    ("PATH(300,3)", 4), ("TREE(500,2)", 8), ("WEB(11,3)", 64),
                                    ("RMAT(9,8,7)", 3), ("STAR(20)", 2), ("CYCLE(50)", 2)])
def test_invariants(spec, b):
    g = datagen.make_graph(spec)
    dec = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, b)
    check_invariants(g, dec)


def test_level_cap_residual():
    g = datagen.rmat(10, 8, 1)
    full = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, 16)
    assert full.order > 2
    cap = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, 16, levels=2)
    assert cap.order == 2 and cap.residual is not None and len(cap.residual[0]) > 0
    check_invariants(g, cap)
    X = datagen.make_x(g.n, 4)
    assert np.array_equal(oracle.spmm_through_decomposition(cap, X), oracle.spmm(g.n, g.row_ptr, g.col, g.val, X))


def test_closed_form_decompositions():
    # n <= b -> one level, everything captured
    g = datagen.rmat(6, 4, 1)
    dec = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, 64)
    assert dec.order == 1 and dec.levels[0].nnz == g.nnz
    # star K_{1,m}, b >= 2 -> one level
    for m in (1, 5, 100):
        g = datagen.star(m)
        assert oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, 2).order == 1
    # empty matrix -> order 0
    dec = oracle.la_decompose(5, np.zeros(6, np.int64), np.zeros(0, np.int64), np.zeros(0), 2)
    assert dec.order == 0


def _und(u, v):
    return sorted({(min(a, b), max(a, b)) for a, b in zip(u.tolist(), v.tolist())})


def _sym(edges):
    e = np.array(edges, dtype=np.int64).reshape(-1, 2)
    return np.concatenate([e[:, 0], e[:, 1]]), np.concatenate([e[:, 1], e[:, 0]])


def test_extract_spec_examples():
    # path P10 in identity order, b=2 -> remainder {(3,4),(5,6),(7,8)}
    u, v = _sym([(i, i + 1) for i in range(9)])
    _, (ru, rv, _) = oracle.extract(u, v, np.ones(len(u)), np.arange(10), 2)
    assert _und(ru, rv) == [(3, 4), (5, 6), (7, 8)]
    # 4-cycle 0-1-2-3-0, identity, b=2 -> empty remainder
    u, v = _sym([(0, 1), (1, 2), (2, 3), (3, 0)])
    _, (ru, rv, _) = oracle.extract(u, v, np.ones(len(u)), np.arange(4), 2)
    assert len(ru) == 0
    # P100 identity, b=4 -> 23 remainder edges: straddlers (4c-1, 4c) for c >= 2
    u, v = _sym([(i, i + 1) for i in range(99)])
    _, (ru, rv, _) = oracle.extract(u, v, np.ones(len(u)), np.arange(100), 4)
    assert len(_und(ru, rv)) == 23


def test_prune_spec_example():
    # path P6 (identity labels), b=2 -> pruned {1, 2} (two lowest-id degree-2 vertices)
    u, v = _sym([(i, i + 1) for i in range(5)])
    assert oracle.prune_head(u, 6, 2).tolist() == [1, 2]
    # ring n=6, b=2 -> {0, 1}
    u, v = _sym([(i, (i + 1) % 6) for i in range(6)])
    assert oracle.prune_head(u, 6, 2).tolist() == [0, 1]


def test_fig3_worked_example():
    """Fig. 3: 7 vertices, b=2, identity positions.  Block-diagonal reading (R3)
    leaves {(2,5),(3,4),(5,6)}; the strict band of the figure leaves only {(2,5)}; the
    level-1 rules give H_1 = [5, 2], order [5,2,3,4,6], everything captured (order 2)."""
    edges = FIG3["pruned"] + FIG3["banded"] + FIG3["outside"]
    u, v = _sym(edges)
    a = np.ones(len(u))
    (p, q, _), (ru, rv, ra) = oracle.extract(u, v, a, np.arange(FIG3["n"]), FIG3["b"])
    assert [list(e) for e in _und(ru, rv)] == FIG3["expected_block_diagonal_remainder"]
    strict = [e for e in _und(u, v) if not (e[0] < 2 or e[1] < 2 or abs(e[0] - e[1]) <= 2)]
    assert [list(e) for e in strict] == FIG3["expected_strict_band_remainder"]
    # level 1 on the remainder with the decomposer's own rules
    n = FIG3["n"]
    rp = np.zeros(n + 1, np.int64)
    o = np.lexsort((rv, ru))
    ru, rv, ra = ru[o], rv[o], ra[o]
    np.cumsum(np.bincount(ru, minlength=n), out=rp[1:])
    dec = oracle.la_decompose(n, rp, rv, ra, FIG3["b"])
    assert dec.order == 1
    assert dec.levels[0].perm[:2].tolist() == FIG3["expected_level1_head"]
    assert dec.levels[0].perm[:5].tolist() == FIG3["expected_level1_order"]


def test_msf_equals_scipy_mst():
    """P5: the Kruskal forest under (key,u,v) equals scipy's MST with weight 1 + rank."""
    g = datagen.rmat(11, 6, 3)
    u, v, _ = _entries(g)
    m = u < v
    u, v = u[m], v[m]
    key = splitmix64_vec(np.uint64(oracle.splitmix64_int(4)) ^ ((u.astype(np.uint64) << np.uint64(32)) | v.astype(np.uint64)))
    fu, fv = oracle.minimum_spanning_forest(g.n, u, v, key)
    rank = np.empty(len(u), np.int64)
    rank[np.lexsort((v, u, key))] = np.arange(len(u))
    W = sp.csr_matrix(((1 + rank).astype(np.float64), (u, v)), shape=(g.n, g.n))
    T = minimum_spanning_tree(W).tocoo()
    assert _und(fu, fv) == _und(T.row, T.col)


def _prufer_tree(seq, n):
    degree = [1] * n
    for x in seq:
        degree[x] += 1
    edges = []
    for x in seq:
        leaf = min(i for i in range(n) if degree[i] == 1)
        edges.append((leaf, x))
        degree[leaf] -= 1
        degree[x] -= 1
    a, b = [i for i in range(n) if degree[i] == 1]
    edges.append((a, b))
    return edges


def _layout_positions(n, edges):
    e = np.array(edges, dtype=np.int64).reshape(-1, 2)
    order = oracle.forest_layout(np.arange(n), e[:, 0], e[:, 1], n)
    pos = np.empty(n, np.int64)
    pos[order] = np.arange(n)
    return order, pos


def _check_tree_layout(n, edges):
    order, pos = _layout_positions(n, edges)
    assert sorted(order.tolist()) == list(range(n))
    deg = np.bincount(np.array(edges).ravel(), minlength=n)
    D = int(deg.max())
    dist = np.array([abs(pos[a] - pos[b]) for a, b in edges])
    # lem:smallest-first-order: >= min(n-1, ceil((x-1)(n-1)/x) + 1) edges within x*Delta
    for x in (1, 2, 3, 4):
        bound = min(n - 1, math.ceil((x - 1) * (n - 1) / x) + 1)
        assert int((dist <= x * D).sum()) >= bound
    # heavy-light bound (consistent with O(n Delta log n))
    lam = int(dist.sum())
    assert lam <= (n - 1) + (D - 1) * n * math.log2(n)
    # contiguity: every subtree (rooted at min id 0) occupies an interval
    adj = [[] for _ in range(n)]
    for a, b in edges:
        adj[a].append(b); adj[b].append(a)
    par = [-1] * n; stack = [0]; seen = {0}; topo = []
    while stack:
        x = stack.pop(); topo.append(x)
        for y in adj[x]:
            if y not in seen:
                seen.add(y); par[y] = x; stack.append(y)
    lo, hi, sz = pos.copy(), pos.copy(), np.ones(n, np.int64)
    for x in reversed(topo[1:]):
        p = par[x]
        lo[p] = min(lo[p], lo[x]); hi[p] = max(hi[p], hi[x]); sz[p] += sz[x]
    assert np.all(hi - lo + 1 == sz)


def test_smallest_first_lemma_exhaustive_small():
    """Every labeled tree with n <= 6 (all Prufer sequences) -> every shape under every root."""
    for n in range(2, 7):
        for seq in itertools.product(range(n), repeat=n - 2):
            _check_tree_layout(n, _prufer_tree(list(seq), n))


def test_smallest_first_lemma_random_trees():
    rng = np.random.default_rng(11)
    for n in (50, 300, 2000):
        for _ in range(3):
            seq = rng.integers(0, n, size=n - 2).tolist()
            _check_tree_layout(n, _prufer_tree(seq, n) if n <= 300 else
                               [(v, int(rng.integers(0, v))) for v in range(1, n)])


def test_complete_binary_tree_closed_form():
    """Smallest-first on the complete binary tree rooted at 0: lambda = h 2^(h-1) - 1,
    which exceeds Table 1's n*Delta at h=6 (R14) -- so that row is not asserted."""
    for h in range(2, 8):
        n = 2 ** h - 1
        edges = [(i, c) for i in range(n) for c in (2 * i + 1, 2 * i + 2) if c < n]
        _, pos = _layout_positions(n, edges)
        lam = sum(abs(int(pos[a]) - int(pos[b])) for a, b in edges)
        assert lam == h * 2 ** (h - 1) - 1
    assert 6 * 2 ** 5 - 1 > 63 * 3


def test_depth_gates():
    """P8 soft gates: scrambled paths with even b -> order <= 3; random trees with b = x*Delta
    -> order <= ceil(log2 m) + 1 (lem:arrow-tree-decomposition P:947)."""
    for n in (100, 1000, 10000):
        for b in (2, 4, 64):
            g = datagen.path(n, 7)
            assert oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, b).order <= 3
    for s in (1, 2):
        g = datagen.tree_random(3000, s)
        D = int(g.degrees().max())
        for x in (2, 4, 8):
            dec = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, x * D)
            assert dec.order <= math.ceil(math.log2(g.nnz // 2)) + 1


@pytest.mark.parametrize("spec,b,k", [("RMAT(12,4,1)", 256, 16), ("GRID(64,1)", 64, 8),
                                      ("RMAT(10,8,2)", 32, 5), ("WEB(10,1)", 64, 3)])
def test_o3_equals_o1_bitwise_dyadic(spec, b, k):
    """P11: on dyadic data O3 (through the decomposition) equals O1 bitwise."""
    g = datagen.make_graph(spec)
    dec = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, b)
    X = datagen.make_x(g.n, k)
    assert np.array_equal(oracle.spmm_through_decomposition(dec, X), oracle.spmm(g.n, g.row_ptr, g.col, g.val, X))


@pytest.mark.parametrize("inst", [g for g in GOLD["instances"] if not g.get("large")],
                         ids=lambda g: g["graph"])
def test_golden_decomposition(inst):
    """P13: per-level sizes and the canonical sha256 equal the survey's independent values."""
    g = datagen.make_graph(inst["graph"])
    dec = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, inst["b"])
    assert dec.order == inst["levels"]
    assert [lv.n_i for lv in dec.levels] == inst["n_i"]
    assert [lv.nnz for lv in dec.levels] == inst["nnz_i"]
    assert [int(lv.row_ptr[lv.head]) for lv in dec.levels] == inst["head_nnz_i"]
    assert oracle.decomposition_sha256(dec) == inst["sha_dec"]
