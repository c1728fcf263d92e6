"""Home-set-aware arrangement (reading R25) -- oracle pins and
the C++ decomposer against the oracle.

R25 is an extension for G ranks, not in the paper: after level 0 every vertex gets the home range
of its pi_0 position (G contiguous ranges of whole level-0 tiles, split by level-0 work plus the
entries each vertex keeps for levels >= 1); the spanning forest of the levels 1..home_levels uses
only the edges inside one home, and its trees are laid out by (home of the root, size desc, min id
asc); later levels are laid out as without homes.  Pins, each independent of the oracle's own code:
  * homes = 1 is the pinned default decomposition (golden hashes, A.10);
  * the home ranges: recomputed from B_0 and A alone (remainder degree = deg_A - row length in
    B_0), every boundary is a whole tile and its prefix is a nearest one to g/G of the total;
  * level 1's layout: the forest recomputed with scipy's MST over the same-home edges (weights =
    rank of (key, u, v)), its trees (scipy connected components) each lie in one home and occupy
    contiguous blocks of perm_1 ordered by (home of the min id, size desc, min id), and
    home_start[g] is where home g's trees begin;
  * every level: Eq. (1) reconstruction, the arrow shape, O3 == O1 bitwise on dyadic data.
"""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components, minimum_spanning_tree

import datagen
import oracle
import paper_2402_19364_b200 as ab
from oracle.decompose import splitmix64_vec
from test_oracle_decompose import check_invariants

CASES = [("RMAT(10,8,1)", 64), ("GRID(40,2)", 32), ("RMAT(12,4,1)", 256), ("PATH(300,3)", 4),
         ("TREE(500,2)", 8), ("RMAT(11,8,5)", 16), ("WEB(11,3)", 64)]


def test_homes_one_is_the_default():
    g = datagen.make_graph("RMAT(12,4,1)")
    a = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, 256)
    z = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, 256, homes=1)
    assert oracle.decomposition_sha256(a) == oracle.decomposition_sha256(z)
    assert z.home_los is None and all(lv.home_start is None for lv in z.levels)


def _ranges_from_scratch(g, dec, G):
    """The R25 split recomputed from A and B_0 only (numpy, no oracle helper)."""
    lv = dec.levels[0]
    b, h, n0 = dec.b, lv.head, lv.n_i
    rowlen = np.diff(lv.row_ptr)
    rem = np.diff(g.row_ptr)[lv.perm[:n0]] - rowlen[:n0]      # per position: entries left for levels >= 1
    T = -(-n0 // b)
    cost = np.zeros(T + 1, np.int64)
    np.add.at(cost, np.arange(h, n0) // b, rowlen[h:n0] + 4)
    np.add.at(cost, lv.col[:lv.row_ptr[h]] // b, 1)
    np.add.at(cost, np.arange(n0) // b, rem)
    cost[T] = g.n - n0
    pre = np.concatenate([[0], np.cumsum(cost)])
    return pre, T + 1


@pytest.mark.parametrize("spec,b", CASES)
@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_home_ranges_nearest_prefix(spec, b, G):
    g = datagen.make_graph(spec)
    dec = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, b, homes=G)
    los = dec.home_los
    pre, Tp = _ranges_from_scratch(g, dec, G)
    n0 = dec.levels[0].n_i
    assert los[0] == 0 and los[G] == g.n and np.all(np.diff(los) >= 0)
    tot = pre[-1]
    prev = 0
    for k in range(1, G):
        # boundary = a whole tile (or the end of [0, n_0)); its prefix is a nearest one to k/G of the total
        t = Tp if los[k] == n0 and n0 % b else los[k] // b
        assert los[k] == min(n0, t * b)
        best = np.abs(pre * G - tot * k).min()
        assert abs(pre[t] * G - tot * k) == best or t == prev, (k, t, best)
        prev = t


def _level1_blocks(g, dec, G, home):
    """Level 1's trees from scratch: remainder after B_0, same-home forest by scipy MST, components."""
    lv0, lv1 = dec.levels[0], dec.levels[1]
    n = g.n
    p0 = np.repeat(np.arange(lv0.rows), np.diff(lv0.row_ptr))
    cap = set(zip(lv0.perm[p0].tolist(), lv0.perm[lv0.col].tolist()))
    u = np.repeat(np.arange(n), np.diff(g.row_ptr))
    v = g.col.astype(np.int64)
    keep = np.array([(a, c) not in cap for a, c in zip(u.tolist(), v.tolist())], bool)
    u, v = u[keep], v[keep]
    H = lv1.perm[:lv1.head]
    inh = np.zeros(n, bool)
    inh[H] = True
    m = (u < v) & ~inh[u] & ~inh[v] & (home[u] == home[v])
    gu, gv = u[m], v[m]
    s1 = oracle.splitmix64_int(4 + 1)
    key = splitmix64_vec(np.uint64(s1) ^ ((gu.astype(np.uint64) << np.uint64(32)) | gv.astype(np.uint64)))
    rank = np.empty(len(gu), np.float64)
    rank[np.lexsort((gv, gu, key))] = np.arange(1, len(gu) + 1)
    W = sp.coo_matrix((rank, (gu, gv)), shape=(n, n)).tocsr()
    F = minimum_spanning_tree(W)
    _, comp = connected_components(F + F.T, directed=False)
    return comp, inh


@pytest.mark.parametrize("spec,b", CASES)
@pytest.mark.parametrize("G", [2, 4])
def test_level1_layout_by_home(spec, b, G):
    g = datagen.make_graph(spec)
    dec = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, b, homes=G)
    if dec.order < 2:
        pytest.skip("one level")
    lv1 = dec.levels[1]
    pos0 = np.empty(g.n, np.int64)
    pos0[dec.levels[0].perm] = np.arange(g.n)
    home = np.searchsorted(dec.home_los[1:-1], pos0, side="right")
    comp, inh = _level1_blocks(g, dec, G, home)
    body = lv1.perm[lv1.head:]
    # each tree is one contiguous block; blocks in (home(min id), size desc, min id) order
    labels = comp[body]
    starts = np.flatnonzero(np.concatenate([[True], labels[1:] != labels[:-1]]))
    assert len(starts) == len(np.unique(labels)), "a tree is split"
    keys = []
    for s, e in zip(starts, list(starts[1:]) + [len(body)]):
        blk = body[s:e]
        assert len(blk) == int((comp[body] == labels[s]).sum())
        r = int(blk.min())
        assert np.all(home[blk] == home[r]), "a tree spans two homes"
        keys.append((int(home[r]), -len(blk), r))
    assert keys == sorted(keys)
    hs = np.full(G + 1, lv1.head)
    for hk, negsz, _ in keys:
        hs[hk + 1:] += -negsz
    assert np.array_equal(hs, lv1.home_start)


@pytest.mark.parametrize("spec,b", CASES[:4])
@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("band", ["block", "strict"])
def test_home_aware_invariants_and_o3(spec, b, G, band):
    g = datagen.make_graph(spec)
    dec = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, b, homes=G, band=band)
    if band == "block":
        check_invariants(g, dec)
    X = datagen.make_x(g.n, 4)
    assert np.array_equal(oracle.spmm_through_decomposition(dec, X), oracle.spmm(g.n, g.row_ptr, g.col, g.val, X))


@pytest.mark.parametrize("spec,b", CASES)
@pytest.mark.parametrize("G", [2, 3, 4, 8])
@pytest.mark.parametrize("band,hl", [("block", 1), ("strict", 1), ("block", 2), ("block", 99)])
def test_cpp_decomposer_homes_bit_exact(spec, b, G, band, hl):
    g = datagen.make_graph(spec)
    ref = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, b, homes=G, band=band, home_levels=hl)
    D = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, b, homes=G, band=band, home_levels=hl)
    assert D.sha256() == oracle.decomposition_sha256(ref)
    Gd, los = D.homes(-1)
    assert Gd == G and np.array_equal(los, ref.home_los) and D.home_levels() == hl
    for i in range(1, ref.order):
        if i <= hl:
            assert np.array_equal(D.homes(i)[1], ref.levels[i].home_start)
        else:
            assert ref.levels[i].home_start is None


def test_homes_save_load_and_errors(tmp_path):
    g = datagen.make_graph("RMAT(11,8,5)")
    D = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 16, homes=4, home_levels=2)
    path = str(tmp_path / "h.dec")
    D.save(path)
    E = ab.Decomposition.load(path)
    assert E.sha256() == D.sha256() and E.home_levels() == 2
    assert E.homes(-1)[0] == 4 and np.array_equal(E.homes(-1)[1], D.homes(-1)[1])
    assert D.info()["levels"] > 3
    for i in (1, 2):
        assert np.array_equal(E.homes(i)[1], D.homes(i)[1])
    from paper_2402_19364_b200.arrow import ArrowError
    with pytest.raises(ArrowError):
        D.homes(0)
    with pytest.raises(ArrowError):
        E.homes(3)
    with pytest.raises(ArrowError):
        ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 16, homes=4, home_levels=-1)
    with pytest.raises(ArrowError):
        ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 16, homes=9)
    assert ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 16).homes() == (1, None)
    # home_levels = 0: the library default (1 level for 2 homes, 3 for more)
    assert ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 16, homes=2).home_levels() == 1
    assert ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 16, homes=4).home_levels() == 3


def test_home_aware_moves_fewer_rows():
    """The point of R25: a G-rank schedule of a home-aware decomposition fetches far fewer level >= 1
    rows from other ranks than the schedule of the default decomposition."""
    g = datagen.make_graph("RMAT(14,8,1)")
    for G in (2, 4):
        moved = {}
        for homes in (1, G):
            D = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 256, homes=homes)
            tot = 0
            for r in range(G):
                s = D.dist_schedule(G, r)
                for lv in s["levels"][1:]:
                    tot += int(lv["recv"].sum() - lv["recv"][r])
            moved[homes] = tot
        assert moved[G] < 0.75 * moved[1], (G, moved)
