"""O2 -- the arrow matrix decomposition, step by step in the paper's order.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares no code with the CUDA
product path; its own splitmix64 is written out below (the decomposition's
random draws are counter-based).

PAPER.md §5.1 LA-Decompose, pruning, §5.3 random spanning
forest, §5.4 smallest-first order, block-diagonal
extraction (§4.1) and "collect the non-zeros at the top"
(P:369), with every choice the paper leaves open fixed by the readings R3-R12
listed in DESIGN.md §3:

    E_0 := stored entries (u, v, a) of A
    for i = 0, 1, ...:
      stop if E_i empty (R7); if L > 0 and i == L: residual := E_i, stop
      deg_i(v) := #{entries of E_i in row v}                            (R5)
      V_i := {v : deg_i(v) > 0}, n_i := |V_i|                           (R8)
      H_i := first min(b, n_i) of V_i sorted by (deg_i desc, id asc)    (R4, R5)  -- step 1
      G'_i := simple graph on V_i \\ H_i, edges {u,v} of E_i, u != v      -- step 2, P:810
      key(u,v) := splitmix64(splitmix64(s + i) ^ (u << 32 | v)), u < v  (R9)       -- P:892
      F_i := unique minimum spanning forest under (key, u, v)           (R10)      -- P:893
      trees sorted by (size desc, min id asc); singletons included      (R11)      -- P:894
      tree layout: root = min id, preorder, children by (size asc, id asc) (R12)   -- P:900
      order_i := H_i ++ layouts; pos_i(order_i[p]) := p
      (u,v,a) -> B_i at (pos u, pos v) iff p < b or q < b or p//b == q//b (R3)     -- step 3
                 (band="strict": p < b or q < b or |p - q| <= b, P:253 / Fig. 3; NEXT-2)
      otherwise (u,v,a) -> E_{i+1}                                                  -- step 4
    level 0 is presented with n rows: positions n_0..n-1 hold A-isolated vertices in id order.

Home-set-aware arrangement (homes = G > 1, reading R25 in DESIGN.md §3 --
an extension for G GPUs, not in the paper): after level 0, every vertex gets a home
g = home_of(pi_0 position) from the G contiguous pi_0 ranges of home_ranges() (level-0 tiles
split by level-0 work plus the remainder degrees); for the levels 1 <= i <= home_levels the
spanning forest is taken over the edges of G'_i whose endpoints share a home (so every tree lies
in one home) and the trees are sorted by (home of the root, size desc, min id asc) instead of
R11's (size desc, min id asc); home_start[g] records where home g's trees begin.  Edges between
homes wait for a later level (or a head); levels after home_levels are laid out as above.
homes = 1 is the decomposition above.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

_M64 = (1 << 64) - 1


def splitmix64_int(x: int) -> int:
    """splitmix64 on a Python int (SURVEY §8(c) O2 box)."""
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def splitmix64_vec(x: np.ndarray) -> np.ndarray:
    """splitmix64 over a uint64 array (numpy wraps mod 2^64)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


@dataclass
class Level:
    """One arrow matrix B_i in positions, with perm_i[p] = original vertex at position p (pi_i^-1)."""
    n_i: int                 # |V_i|: vertices with an entry in A_i
    perm: np.ndarray         # int64[rows]; rows = n for level 0, n_i otherwise
    row_ptr: np.ndarray      # int64[rows+1]
    col: np.ndarray          # int64[nnz_i] positions, sorted within each row
    val: np.ndarray          # float64[nnz_i]
    head: int                # h_i = min(b, n_i)
    home_start: np.ndarray | None = None   # int64[G+1] (home-aware levels): trees of home g at [hs[g], hs[g+1])

    @property
    def rows(self) -> int:
        return len(self.perm)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])


@dataclass
class Decomposition:
    n: int
    b: int
    levels: list = field(default_factory=list)
    residual: tuple | None = None    # (u, v, a) original-id triples left when the level cap is hit
    band: str = "block"              # step 3's band (captured())
    homes: int = 1                   # G of the home-set-aware arrangement (R25); 1 = R11
    home_los: np.ndarray | None = None   # int64[G+1] pi_0 home ranges (homes > 1)
    home_levels: int = 0             # levels 1..home_levels are home-aware (homes > 1)

    @property
    def order(self) -> int:
        return len(self.levels)


# ---------------------------------------------------------------------------- MSF (Kruskal)
def _find(parent, x):
    root = x
    while parent[root] != root:
        root = parent[root]
    while parent[x] != root:           # path compression
        parent[x], x = root, parent[x]
    return root


def minimum_spanning_forest(n: int, eu: np.ndarray, ev: np.ndarray, key: np.ndarray):
    """Kruskal: scan edges in increasing (key, u, v); keep an edge iff it joins two trees.
    The strict total order makes the forest unique (R10).  Returns kept (u, v) arrays."""
    order = np.lexsort((ev, eu, key))
    parent = list(range(n))
    keep_u, keep_v = [], []
    for idx in order.tolist():
        a, b = int(eu[idx]), int(ev[idx])
        ra, rb = _find(parent, a), _find(parent, b)
        if ra != rb:
            parent[ra] = rb
            keep_u.append(a)
            keep_v.append(b)
    return np.array(keep_u, dtype=np.int64), np.array(keep_v, dtype=np.int64)


# ---------------------------------------------------------------------------- tree layout
def forest_layout(vertices: np.ndarray, fu: np.ndarray, fv: np.ndarray, n: int, home=None, G: int = 1):
    """Linear arrangement of a spanning forest on `vertices`:
    trees in decreasing size (ties: smaller min id), each tree in smallest-first order
    rooted at its min id, children by (subtree size asc, id asc); iterative DFS (R12).
    With `home` (int array over vertex ids, R25): trees sorted by (home[root], size desc, root)
    instead; then also returns home_start (offsets of each home's trees, length G+1)."""
    if len(vertices) == 0:
        empty = np.zeros(0, dtype=np.int64)
        return empty if home is None else (empty, np.zeros(G + 1, dtype=np.int64))
    adj = [[] for _ in range(n)]
    for a, b in zip(fu.tolist(), fv.tolist()):
        adj[a].append(b)
        adj[b].append(a)
    seen = np.zeros(n, dtype=bool)
    trees = []                                   # (size, root, preorder list)
    for r in vertices.tolist():                  # ascending id: first unseen vertex of a tree is its min id
        if seen[r]:
            continue
        # BFS from the root: parent pointers and a top-down order
        order = [r]
        parent = {r: -1}
        seen[r] = True
        h = 0
        while h < len(order):
            x = order[h]
            h += 1
            for y in adj[x]:
                if not seen[y]:
                    seen[y] = True
                    parent[y] = x
                    order.append(y)
        size = {x: 1 for x in order}
        for x in reversed(order[1:]):
            size[parent[x]] += size[x]
        children = {x: [] for x in order}
        for x in order[1:]:
            children[parent[x]].append(x)
        # preorder, children sorted by (subtree size asc, id asc)
        pre = []
        stack = [r]
        while stack:
            x = stack.pop()
            pre.append(x)
            ch = sorted(children[x], key=lambda c: (size[c], c))
            stack.extend(reversed(ch))
        trees.append((len(order), r, pre))
    if home is None:
        trees.sort(key=lambda t: (-t[0], t[1]))
        return np.array([x for t in trees for x in t[2]], dtype=np.int64)
    trees.sort(key=lambda t: (int(home[t[1]]), -t[0], t[1]))
    start = np.zeros(G + 1, dtype=np.int64)
    for size, root, _ in trees:
        start[int(home[root]) + 1:] += size
    return np.array([x for t in trees for x in t[2]], dtype=np.int64), start


# ---------------------------------------------------------------------------- homes (R25)
def level0_tile_costs(lv: Level, b: int, rem_deg: np.ndarray) -> np.ndarray:
    """Work of each level-0 tile t (positions [t b, (t+1) b) of [0, n_0)), R25: every body row
    p >= h costs its entries + 4; every head-row entry costs 1 in the tile of its column; every
    vertex at a position of the tile adds its remainder degree rem_deg (its entries left for
    levels >= 1, which its home computes under the home-aware arrangement)."""
    T = -(-lv.n_i // b)
    cost = np.zeros(T, dtype=np.int64)
    for p in range(lv.head, lv.n_i):
        cost[p // b] += int(lv.row_ptr[p + 1] - lv.row_ptr[p]) + 4
    for j in range(lv.head):
        for q in lv.col[lv.row_ptr[j]:lv.row_ptr[j + 1]]:
            cost[int(q) // b] += 1
    for p in range(lv.n_i):
        cost[p // b] += int(rem_deg[lv.perm[p]])
    return cost


def home_ranges(lv0: Level, n: int, b: int, G: int, rem_deg: np.ndarray) -> np.ndarray:
    """R25: G contiguous pi_0 ranges los[0..G] made of whole level-0 tiles.  The tile costs of
    level0_tile_costs() plus one last pseudo-tile for the A-isolated positions [n_0, n) (cost 1
    each); prefix sums pre[0..T']; boundary g (0 < g < G) is the first t with pre[t] >= g/G of
    the total, moved one tile back if pre[t-1] is strictly nearer to g/G of the total, and never
    before boundary g-1.  los[g] = min(n_0, t_g b); los[0] = 0, los[G] = n."""
    cost = list(level0_tile_costs(lv0, b, rem_deg)) + [n - lv0.n_i]
    Tp = len(cost)
    pre = [0]
    for c in cost:
        pre.append(pre[-1] + c)
    tot = pre[-1]
    tb = [0] * (G + 1)
    tb[G] = Tp
    for g in range(1, G):
        t = next(t for t in range(Tp + 1) if pre[t] * G >= tot * g)
        if t > 0 and tot * g - pre[t - 1] * G < pre[t] * G - tot * g:
            t -= 1
        tb[g] = min(max(t, tb[g - 1]), Tp)
    los = np.array([min(lv0.n_i, t * b) for t in tb], dtype=np.int64)
    los[0], los[G] = 0, n
    return los


def homes_of(lv0: Level, los: np.ndarray, n: int) -> np.ndarray:
    """home[v] = the range g with los[g] <= pi_0(v) < los[g+1] (the last such g if ranges are empty)."""
    pos0 = np.empty(n, dtype=np.int64)
    pos0[lv0.perm] = np.arange(n, dtype=np.int64)
    return np.searchsorted(los[1:-1], pos0, side="right").astype(np.int64)


# ---------------------------------------------------------------------------- steps 1 and 3
def prune_head(eu: np.ndarray, n: int, b: int) -> np.ndarray:
    """Step 1 (R4, R5): the min(b, n_i) vertices of largest remainder degree,
    sorted by (degree desc, id asc)."""
    deg = np.bincount(eu, minlength=n)
    V = np.flatnonzero(deg > 0)
    return V[np.lexsort((V, -deg[V]))][:min(b, len(V))]


BANDS = ("block", "strict")


def captured(p: np.ndarray, q: np.ndarray, b: int, band: str = "block") -> np.ndarray:
    """Step 3: entry at positions (p, q) belongs to B_i iff it lies in the first b rows
    or columns, or in the band around the diagonal:
      band="block"  -- a diagonal b x b tile (the block-diagonal band of §4.1; R3);
      band="strict" -- |p - q| <= b, the arrow-width definition itself ("for all i>b and
                       j>b ... if A_ij != 0 then |i-j| <= b", 1-based) and Fig. 3;
                       NEXT-2 of SURVEY §8(f)."""
    if band == "block":
        return (p < b) | (q < b) | (p // b == q // b)
    if band == "strict":
        return (p < b) | (q < b) | (np.abs(p - q) <= b)
    raise ValueError(f"unknown band {band!r}")


def extract(eu, ev, ea, order, b: int, band: str = "block"):
    """Apply step 3 for a given arrangement `order` (order[p] = vertex at position p).
    Returns ((p, q, a) captured, (u, v, a) remainder)."""
    eu, ev, ea = np.asarray(eu, np.int64), np.asarray(ev, np.int64), np.asarray(ea, np.float64)
    n = int(max(eu.max(initial=-1), ev.max(initial=-1), np.max(order, initial=-1))) + 1
    pos = np.full(n, -1, dtype=np.int64)
    pos[np.asarray(order, np.int64)] = np.arange(len(order), dtype=np.int64)
    p, q = pos[eu], pos[ev]
    if ((p < 0) | (q < 0)).any():
        raise ValueError("arrangement does not cover every endpoint")
    cap = captured(p, q, b, band)
    return (p[cap], q[cap], ea[cap]), (eu[~cap], ev[~cap], ea[~cap])


# ---------------------------------------------------------------------------- LA-Decompose
def la_decompose(n: int, row_ptr, col, val, b: int, levels: int = 0, seed: int = 4,
                 band: str = "block", homes: int = 1, home_levels: int = 1) -> Decomposition:
    if band not in BANDS:
        raise ValueError(f"unknown band {band!r}")
    if not 1 <= homes <= 8:
        raise ValueError("homes must be in [1, 8]")
    if home_levels < 1:
        raise ValueError("home_levels must be >= 1")
    if b < 2:
        raise ValueError("arrow width b must be >= 2 (P:807)")
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    eu = np.repeat(np.arange(n, dtype=np.int64), np.diff(row_ptr))
    ev = np.asarray(col, dtype=np.int64)
    ea = np.asarray(val, dtype=np.float64)
    deg_a = np.diff(row_ptr)
    isolated_a = np.flatnonzero(deg_a == 0)
    dec = Decomposition(n=n, b=b, band=band, homes=homes, home_levels=home_levels if homes > 1 else 0)
    home = None                        # R25: vertex homes, set after level 0 when homes > 1
    i = 0
    while True:
        if len(eu) == 0:
            break
        if levels > 0 and i == levels:
            dec.residual = (eu, ev, ea)
            break
        # step 1: prune the b highest-degree vertices of the current remainder
        V = np.flatnonzero(np.bincount(eu, minlength=n) > 0)
        n_i = len(V)
        H = prune_head(eu, n, b)
        h = len(H)
        in_h = np.zeros(n, dtype=bool)
        in_h[H] = True
        # step 2: arrangement of G'_i = G_i[V_i \ H_i] by a random spanning forest
        aware = home is not None and i <= home_levels
        m = (eu < ev) & ~in_h[eu] & ~in_h[ev]
        if aware:                      # R25: the forest of each home set
            m &= home[eu] == home[ev]
        gu, gv = eu[m], ev[m]
        s_i = splitmix64_int((seed + i) & _M64)
        key = splitmix64_vec(np.uint64(s_i) ^ ((gu.astype(np.uint64) << np.uint64(32)) | gv.astype(np.uint64)))
        fu, fv = minimum_spanning_forest(n, gu, gv, key)
        rest = V[~in_h[V]]
        hs = None
        if not aware:
            order_i = np.concatenate([H, forest_layout(rest, fu, fv, n)])
        else:
            lay, hs = forest_layout(rest, fu, fv, n, home, homes)
            order_i = np.concatenate([H, lay])
            hs = hs + h
        assert len(order_i) == n_i
        pos = np.full(n, -1, dtype=np.int64)
        pos[order_i] = np.arange(n_i, dtype=np.int64)
        # step 3: head rows/columns plus the band: block-diagonal b x b tiles (R3)
        # or, band="strict", |p - q| <= b
        p, q = pos[eu], pos[ev]
        cap = captured(p, q, b, band)
        perm = order_i if i > 0 else np.concatenate([order_i, isolated_a])
        rows = len(perm)
        bp, bq, ba = p[cap], q[cap], ea[cap]
        srt = np.lexsort((bq, bp))
        bp, bq, ba = bp[srt], bq[srt], ba[srt]
        rp = np.zeros(rows + 1, dtype=np.int64)
        np.cumsum(np.bincount(bp, minlength=rows), out=rp[1:])
        dec.levels.append(Level(n_i=n_i, perm=perm, row_ptr=rp, col=bq, val=ba, head=h, home_start=hs))
        # step 4: the remainder A_{i+1} = A_i - P B_i P^T, kept in original ids
        eu, ev, ea = eu[~cap], ev[~cap], ea[~cap]
        if i == 0 and homes > 1:     # R25: homes from level 0 and the remainder's degrees
            dec.home_los = home_ranges(dec.levels[0], n, b, homes, np.bincount(eu, minlength=n))
            home = homes_of(dec.levels[0], dec.home_los, n)
        i += 1
    return dec


# ---------------------------------------------------------------------------- canonical hash
def canonical_bytes(dec: Decomposition):
    """Little-endian serialisation: int64 L; per level int64 rows,
    int32 perm[rows], int64 row_ptr[rows+1], int32 col[nnz], float64 val[nnz]."""
    yield np.int64(dec.order).tobytes()
    for lv in dec.levels:
        yield np.int64(lv.rows).tobytes()
        yield lv.perm.astype("<i4").tobytes()
        yield lv.row_ptr.astype("<i8").tobytes()
        yield lv.col.astype("<i4").tobytes()
        yield lv.val.astype("<f8").tobytes()


def decomposition_sha256(dec: Decomposition) -> str:
    h = hashlib.sha256()
    for chunk in canonical_bytes(dec):
        h.update(chunk)
    return h.hexdigest()


# ---------------------------------------------------------------------------- O3
def spmm_through_decomposition(dec: Decomposition, X: np.ndarray) -> np.ndarray:
    """O3 (Eq. (1); Alg. 2's forward/local/reverse phases without ranks):
    Y := 0; for each level i and position p: Y[perm_i[p]] += sum_{(q,a) in B_i[p]} a X[perm_i[q]];
    then the residual entries.  fp64."""
    import scipy.sparse as sp
    X = np.asarray(X, dtype=np.float64)
    Y = np.zeros((dec.n, X.shape[1]), dtype=np.float64)
    for lv in dec.levels:
        B = sp.csr_matrix((lv.val, lv.col, lv.row_ptr), shape=(lv.rows, lv.rows))
        Xp = X[lv.perm]                    # P_pi^T X  (row p holds X[perm[p]])
        Y[lv.perm] += B @ Xp               # P_pi (B (P_pi^T X)); perm is injective
    if dec.residual is not None:
        u, v, a = dec.residual
        np.add.at(Y, u, a[:, None] * X[v])
    return Y


def reconstruct_entries(dec: Decomposition):
    """Eq. (1) read back: the multiset {(perm_i[p], perm_i[q], a)} over all levels + residual."""
    us, vs, as_ = [], [], []
    for lv in dec.levels:
        p = np.repeat(np.arange(lv.rows, dtype=np.int64), np.diff(lv.row_ptr))
        us.append(lv.perm[p])
        vs.append(lv.perm[lv.col])
        as_.append(lv.val)
    if dec.residual is not None:
        us.append(dec.residual[0])
        vs.append(dec.residual[1])
        as_.append(dec.residual[2])
    if not us:
        return (np.zeros(0, np.int64),) * 2 + (np.zeros(0),)
    return np.concatenate(us), np.concatenate(vs), np.concatenate(as_)
