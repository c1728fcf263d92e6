// decompose.cpp -- host LA-Decompose (arrow_plan_create's preprocessing; not the timed path).
//
// PAPER.md §5.1 LA-Decompose with the evaluation's arrangement, a random
// spanning forest laid out in smallest-first order (§5.3, §5.4),
// and the block-diagonal band of §4.1.  The choices the paper leaves open are the
// readings R3-R12 of DESIGN.md §3; with them the decomposition is a deterministic function
// of (A, b, levels, seed), so every rank of a distributed run builds the same one.
//
//   per level i:  deg_i over the remainder E_i; V_i = {deg_i > 0}; head H_i = first
//   min(b,|V_i|) of V_i by (deg desc, id asc); forest F_i = Kruskal over G'_i = G_i[V_i \ H_i]
//   with edge order (splitmix64(splitmix64(seed+i) ^ (u<<32|v)), u, v); trees by (size desc,
//   min id asc), each rooted at its min id, preorder with children by (subtree size asc, id asc);
//   order_i = H_i ++ trees; entry (u,v) captured iff p<b or q<b or p/b == q/b (p,q positions);
//   band = 1 (strict, NEXT-2): p<b or q<b or |p-q| <= b -- the arrow-width definition of
//   and Fig. 3.
//
// homes = G > 1 (R25): after level 0 every vertex gets the home range of its
// pi_0 position (home_ranges: level-0 tile work plus remainder degrees, split G ways); the forest
// of every level >= 1 takes only edges inside one home and its trees are laid out by (home of the
// root, size desc, min id asc) for the levels 1..home_levels, so that rank g's level-i tiles hold
// rows whose X and Y live on rank g (edges between homes wait for a later level or a head).
//
// Parallel where the work is bulk (degree histograms, edge keys, the edge sort, extraction,
// CSR assembly); union-find and the tree layouts are sequential.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <numeric>
#include <omp.h>
#include <parallel/algorithm>

#include "arrow_internal.h"

namespace arrow {

static inline uint64_t mix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

int validate_csr(int64_t n, int64_t nnz, const int64_t *rp, const int32_t *col, std::string &err) {
    if (rp[0] != 0) { err = "row_ptr[0] != 0"; return 1; }
    if (rp[n] != nnz) { err = "row_ptr[n] != nnz"; return 1; }
    std::atomic<int64_t> bad{-1};
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t r = 0; r < n; ++r) {
        if (bad.load(std::memory_order_relaxed) >= 0) continue;
        if (rp[r + 1] < rp[r]) { bad = r; continue; }
        for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
            if (col[e] < 0 || col[e] >= n || (e > rp[r] && col[e] <= col[e - 1])) { bad = r; break; }
        }
    }
    if (bad >= 0) {
        err = "row " + std::to_string(bad.load()) + ": row_ptr decreasing, column out of range, or columns not strictly increasing";
        return 1;
    }
    return 0;
}

int check_symmetric(int64_t n, const int64_t *rp, const int32_t *col, std::string &err) {
    std::atomic<int64_t> bad{-1};
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t r = 0; r < n; ++r) {
        if (bad.load(std::memory_order_relaxed) >= 0) continue;
        for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
            const int32_t c = col[e];
            if (!std::binary_search(col + rp[c], col + rp[c + 1], (int32_t)r)) { bad = r; break; }
        }
    }
    if (bad >= 0) {
        err = "pattern not symmetric at row " + std::to_string(bad.load());
        return 2;
    }
    return 0;
}

namespace {

struct Edge {
    uint64_t key;
    uint32_t u, v;
};

inline bool edge_less(const Edge &a, const Edge &b) {
    if (a.key != b.key) return a.key < b.key;
    if (a.u != b.u) return a.u < b.u;
    return a.v < b.v;
}

inline int32_t uf_find(std::vector<int32_t> &parent, int32_t x) {
    while (parent[x] != x) {
        parent[x] = parent[parent[x]];  // path halving
        x = parent[x];
    }
    return x;
}

// Stable parallel partition of `in` by predicate into (yes, no), preserving order.
template <class Pred>
void stable_partition_par(const std::vector<uint32_t> &in, Pred pred, std::vector<uint32_t> &yes,
                          std::vector<uint32_t> &no) {
    const int64_t m = (int64_t)in.size();
    const int T = omp_get_max_threads();
    std::vector<int64_t> cy(T + 1, 0), cn(T + 1, 0);
#pragma omp parallel num_threads(T)
    {
        const int t = omp_get_thread_num(), nt = omp_get_num_threads();
        const int64_t lo = m * t / nt, hi = m * (t + 1) / nt;
        int64_t y = 0;
        for (int64_t i = lo; i < hi; ++i) y += pred(in[i]) ? 1 : 0;
        cy[t + 1] = y;
        cn[t + 1] = (hi - lo) - y;
#pragma omp barrier
#pragma omp single
        {
            for (int i = 0; i < nt; ++i) { cy[i + 1] += cy[i]; cn[i + 1] += cn[i]; }
            yes.resize(cy[nt]);
            no.resize(cn[nt]);
        }
        int64_t oy = cy[t], on = cn[t];
        for (int64_t i = lo; i < hi; ++i) {
            if (pred(in[i])) yes[oy++] = in[i];
            else no[on++] = in[i];
        }
    }
}

}  // namespace

std::vector<int64_t> split_prefix(const std::vector<int64_t> &pre, int G) {
    const int64_t T = (int64_t)pre.size() - 1, tot = pre[T];
    std::vector<int64_t> tb(G + 1, T);
    tb[0] = 0;
    for (int g = 1; g < G; ++g) {
        // first t with pre[t] * G >= tot * g (exact), one back if pre[t-1] is strictly nearer
        int64_t lo = 0, hi = T;
        while (lo < hi) {
            const int64_t mid = (lo + hi) / 2;
            if (pre[mid] * G >= tot * g) hi = mid;
            else lo = mid + 1;
        }
        int64_t t = lo;
        if (t > 0 && tot * g - pre[t - 1] * G < pre[t] * G - tot * g) t -= 1;
        tb[g] = std::min(std::max(t, tb[g - 1]), T);
    }
    return tb;
}

std::vector<int64_t> home_ranges(const HostLevel &L0, int64_t n, int64_t b, int G, const int32_t *rem_deg) {
    const int64_t T = (L0.n_i + b - 1) / b, h = L0.head;
    std::vector<int64_t> pre(T + 2, 0);  // T level-0 tiles + the A-isolated pseudo-tile
    for (int64_t p = h; p < L0.n_i; ++p) pre[p / b + 1] += (L0.row_ptr[p + 1] - L0.row_ptr[p]) + 4;
    for (int64_t e = 0; e < L0.row_ptr[h]; ++e) pre[L0.col[e] / b + 1] += 1;
    for (int64_t p = 0; p < L0.n_i; ++p) pre[p / b + 1] += rem_deg[L0.perm[p]];
    pre[T + 1] = n - L0.n_i;
    for (int64_t t = 0; t <= T; ++t) pre[t + 1] += pre[t];
    const std::vector<int64_t> tb = split_prefix(pre, G);
    std::vector<int64_t> los(G + 1);
    for (int g = 0; g <= G; ++g) los[g] = std::min<int64_t>(L0.n_i, tb[g] * b);
    los[0] = 0;
    los[G] = n;
    return los;
}

int la_decompose(int64_t n, const int64_t *rp, const int32_t *col, int64_t b, int32_t max_levels,
                 uint64_t seed, int band, int homes, int home_levels, HostDecomposition &out, std::string &err) {
    out = HostDecomposition{};
    out.n = n;
    out.b = b;
    out.band = band;
    out.homes = homes;
    out.home_levels = homes > 1 ? home_levels : 0;
    std::vector<uint8_t> home;  // homes > 1: home of every vertex (after level 0)
    const int64_t nnz = rp[n];
    if (nnz == 0) return 0;

    std::vector<int32_t> erow(nnz);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t r = 0; r < n; ++r)
        for (int64_t e = rp[r]; e < rp[r + 1]; ++e) erow[e] = (int32_t)r;

    std::vector<int32_t> isolated;
    for (int64_t v = 0; v < n; ++v)
        if (rp[v + 1] == rp[v]) isolated.push_back((int32_t)v);

    std::vector<uint32_t> ent(nnz), captured, rest_ent;
    std::iota(ent.begin(), ent.end(), 0u);

    std::vector<int32_t> deg(n), pos(n), parent(n), sz(n), qbuf, forder;
    std::vector<uint8_t> in_head(n), visited(n);
    std::vector<int64_t> fstart(n + 1);
    std::vector<int32_t> fadj;

    for (int32_t i = 0;; ++i) {
        if (ent.empty()) break;
        if (max_levels > 0 && i == max_levels) {
            out.residual = ent;
            break;
        }
        const int64_t m = (int64_t)ent.size();
        // ---- step 1: degrees of the remainder, V_i, head H_i (R4, R5, R8)
        std::fill(deg.begin(), deg.end(), 0);
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < m; ++t)
            __atomic_fetch_add(&deg[erow[ent[t]]], 1, __ATOMIC_RELAXED);
        std::vector<int32_t> V;
        V.reserve(n);
        for (int64_t v = 0; v < n; ++v)
            if (deg[v] > 0) V.push_back((int32_t)v);
        const int64_t n_i = (int64_t)V.size();
        const int64_t h = std::min<int64_t>(b, n_i);
        std::vector<int32_t> H(V);
        auto by_deg = [&](int32_t a, int32_t c) { return deg[a] != deg[c] ? deg[a] > deg[c] : a < c; };
        std::partial_sort(H.begin(), H.begin() + h, H.end(), by_deg);
        H.resize(h);
        std::fill(in_head.begin(), in_head.end(), 0);
        for (int32_t v : H) in_head[v] = 1;

        const bool aware = !home.empty() && i <= home_levels;  // R25 at this level
        // ---- step 2a: G'_i edges with their random keys (R9)
        const uint64_t s_i = mix64(seed + (uint64_t)i);
        std::vector<uint32_t> gent, dummy;
        stable_partition_par(
            ent,
            [&](uint32_t e) {
                const int32_t u = erow[e], v = col[e];
                return u < v && !in_head[u] && !in_head[v] && (!aware || home[u] == home[v]);
            },
            gent, dummy);
        dummy.clear();
        dummy.shrink_to_fit();
        std::vector<Edge> edges(gent.size());
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < (int64_t)gent.size(); ++t) {
            const uint32_t u = (uint32_t)erow[gent[t]], v = (uint32_t)col[gent[t]];
            edges[t] = Edge{mix64(s_i ^ (((uint64_t)u << 32) | v)), u, v};
        }
        gent.clear();
        gent.shrink_to_fit();
        // ---- step 2b: the unique minimum spanning forest under (key, u, v) (R10)
        __gnu_parallel::sort(edges.begin(), edges.end(), edge_less);
        for (int32_t v : V) parent[v] = v;
        std::vector<std::pair<int32_t, int32_t>> forest;
        forest.reserve(n_i);
        for (const Edge &e : edges) {
            int32_t a = uf_find(parent, (int32_t)e.u), c = uf_find(parent, (int32_t)e.v);
            if (a != c) {
                parent[a] = c;
                forest.emplace_back((int32_t)e.u, (int32_t)e.v);
            }
        }
        edges.clear();
        edges.shrink_to_fit();
        // forest adjacency (CSR over all n; only V_i \ H_i vertices have entries)
        std::fill(fstart.begin(), fstart.end(), 0);
        for (auto &f : forest) { ++fstart[f.first + 1]; ++fstart[f.second + 1]; }
        for (int64_t v = 0; v < n; ++v) fstart[v + 1] += fstart[v];
        fadj.assign(2 * forest.size(), 0);
        {
            std::vector<int64_t> cur(fstart.begin(), fstart.end() - 1);
            for (auto &f : forest) { fadj[cur[f.first]++] = f.second; fadj[cur[f.second]++] = f.first; }
        }
        // ---- step 2c: lay out trees by decreasing size, smallest-first inside (R11, R12)
        struct Tree { int64_t size; int32_t root; int64_t off; };
        std::vector<Tree> trees;
        qbuf.resize(n_i);
        forder.resize(n_i);
        std::fill(visited.begin(), visited.end(), 0);
        int64_t fpos = 0;
        std::vector<int32_t> kids;     // non-root tree vertices sorted by (parent, size, id)
        std::vector<int64_t> kstart;   // per tree-local node: range into kids (indexed via idx map)
        std::vector<int32_t> stack;
        for (int32_t r : V) {
            if (in_head[r] || visited[r]) continue;
            // BFS from the root (min id of its tree: V is scanned in ascending id)
            int64_t qh = 0, qt = 0;
            qbuf[qt++] = r;
            visited[r] = 1;
            parent[r] = -1;
            while (qh < qt) {
                const int32_t x = qbuf[qh++];
                for (int64_t a = fstart[x]; a < fstart[x + 1]; ++a) {
                    const int32_t y = fadj[a];
                    if (!visited[y]) { visited[y] = 1; parent[y] = x; qbuf[qt++] = y; }
                }
            }
            const int64_t tsize = qt;
            for (int64_t t = 0; t < tsize; ++t) sz[qbuf[t]] = 1;
            for (int64_t t = tsize - 1; t > 0; --t) sz[parent[qbuf[t]]] += sz[qbuf[t]];
            const int64_t off = fpos;
            if (tsize == 1) {
                forder[fpos++] = r;
            } else {
                kids.assign(qbuf.begin() + 1, qbuf.begin() + tsize);
                std::sort(kids.begin(), kids.end(), [&](int32_t a, int32_t c) {
                    if (parent[a] != parent[c]) return parent[a] < parent[c];
                    if (sz[a] != sz[c]) return sz[a] < sz[c];
                    return a < c;
                });
                // children of x occupy kids[first[x] .. first[x] + nchild[x]); store first in `pos` (scratch)
                for (int64_t t = 0; t < tsize; ++t) pos[qbuf[t]] = -1;
                for (int64_t t = (int64_t)kids.size() - 1; t >= 0; --t) pos[parent[kids[t]]] = (int32_t)t;
                stack.clear();
                stack.push_back(r);
                while (!stack.empty()) {
                    const int32_t x = stack.back();
                    stack.pop_back();
                    forder[fpos++] = x;
                    const int32_t first = pos[x];
                    if (first < 0) continue;
                    int64_t last = first;
                    while (last < (int64_t)kids.size() && parent[kids[last]] == x) ++last;
                    for (int64_t t = last - 1; t >= first; --t) stack.push_back(kids[t]);
                }
            }
            trees.push_back(Tree{tsize, r, off});
        }
        if (fpos + h != n_i) { err = "internal: forest layout does not cover V_i"; return 1; }
        HostLevel L;
        if (!aware) {
            std::stable_sort(trees.begin(), trees.end(), [](const Tree &a, const Tree &c) {
                return a.size != c.size ? a.size > c.size : a.root < c.root;
            });
        } else {  // R25: by home of the root first
            std::stable_sort(trees.begin(), trees.end(), [&](const Tree &a, const Tree &c) {
                if (home[a.root] != home[c.root]) return home[a.root] < home[c.root];
                return a.size != c.size ? a.size > c.size : a.root < c.root;
            });
            L.home_start.assign(homes + 1, 0);
            for (const Tree &t : trees) L.home_start[home[t.root] + 1] += t.size;
            L.home_start[0] = h;
            for (int g = 0; g < homes; ++g) L.home_start[g + 1] += L.home_start[g];
        }
        L.n_i = n_i;
        L.head = h;
        L.rows = (i == 0) ? n : n_i;
        L.perm.resize(L.rows);
        std::copy(H.begin(), H.end(), L.perm.begin());
        {
            int64_t p = h;
            for (const Tree &t : trees) {
                std::copy(forder.begin() + t.off, forder.begin() + t.off + t.size, L.perm.begin() + p);
                p += t.size;
            }
            if (i == 0) std::copy(isolated.begin(), isolated.end(), L.perm.begin() + p);
        }
        std::fill(pos.begin(), pos.end(), -1);
        for (int64_t p = 0; p < n_i; ++p) pos[L.perm[p]] = (int32_t)p;

        // ---- step 3: capture head rows/columns and diagonal b x b tiles (R3), or the
        // strict band |p - q| <= b (band = 1; Fig. 3)
        stable_partition_par(
            ent,
            [&](uint32_t e) {
                const int64_t p = pos[erow[e]], q = pos[col[e]];
                if (p < b || q < b) return true;
                return band ? (p > q ? p - q : q - p) <= b : (p / b) == (q / b);
            },
            captured, rest_ent);
        // canonical CSR of B_i in positions
        const int64_t cnt = (int64_t)captured.size();
        L.row_ptr.assign(L.rows + 1, 0);
        {
            std::vector<int64_t> rc(L.rows + 1, 0);
#pragma omp parallel for schedule(static)
            for (int64_t t = 0; t < cnt; ++t)
                __atomic_fetch_add(&rc[pos[erow[captured[t]]] + 1], (int64_t)1, __ATOMIC_RELAXED);
            for (int64_t p = 0; p < L.rows; ++p) rc[p + 1] += rc[p];
            L.row_ptr = rc;
        }
        std::vector<uint64_t> packed(cnt);
        {
            std::vector<int64_t> cursor(L.row_ptr.begin(), L.row_ptr.end() - 1);
#pragma omp parallel for schedule(static)
            for (int64_t t = 0; t < cnt; ++t) {
                const uint32_t e = captured[t];
                const int64_t p = pos[erow[e]];
                const int64_t at = __atomic_fetch_add(&cursor[p], (int64_t)1, __ATOMIC_RELAXED);
                packed[at] = ((uint64_t)(uint32_t)pos[col[e]] << 32) | e;
            }
        }
#pragma omp parallel for schedule(dynamic, 1024)
        for (int64_t p = 0; p < L.rows; ++p) std::sort(packed.begin() + L.row_ptr[p], packed.begin() + L.row_ptr[p + 1]);
        L.col.resize(cnt);
        L.src.resize(cnt);
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < cnt; ++t) {
            L.col[t] = (int32_t)(packed[t] >> 32);
            L.src[t] = (uint32_t)(packed[t] & 0xFFFFFFFFu);
        }
        out.levels.push_back(std::move(L));
        if (i == 0 && homes > 1) {  // R25: homes from level 0's tile work and the remainder degrees
            std::vector<int32_t> rem(n, 0);
            for (uint32_t e : rest_ent) rem[erow[e]]++;
            out.home_los = home_ranges(out.levels[0], n, b, homes, rem.data());
            home.assign(n, 0);
            for (int64_t p = 0; p < n; ++p) {
                const int64_t g = std::upper_bound(out.home_los.begin() + 1, out.home_los.end() - 1, p) -
                                  (out.home_los.begin() + 1);
                home[out.levels[0].perm[p]] = (uint8_t)g;
            }
        }
        // ---- step 4: remainder A_{i+1}, kept as original entries
        ent.swap(rest_ent);
        rest_ent.clear();
    }
    return 0;
}

}  // namespace arrow
