// gdecompose.cu -- LA-Decompose on the GPU: the rules of decompose.cpp and of
// the oracle O2 (DESIGN.md §3 readings R3-R12), bit-exact, with the sequential parts of the host
// decomposer replaced by data-parallel ones.
//
// PAPER.md §5.1 LA-Decompose, the random spanning forest arrangement (§5.3)
// and smallest-first order (§5.4).  Per level i:
//   1. degrees of the remainder E_i (atomics), V_i = {deg > 0}, head H_i = the first min(b, n_i) of
//      V_i by (deg desc, id asc): one radix sort of 64-bit keys (~deg << 32 | id).
//   2. G'_i = edges u < v of E_i outside the head; key(u,v) = splitmix64(splitmix64(seed+i) ^ (u<<32|v)).
//   3. the unique minimum spanning forest under (key, u, v) by Boruvka: every component takes its
//      lightest outgoing edge (64-bit atomicMin on the key, then on (u<<32|v) among equal keys), the
//      components hook along them (a mutual pair keeps the smaller id as root), pointer jumping
//      flattens the labels; O(log n) rounds.  (Kruskal and Boruvka give the same forest: the order
//      is strict.)
//   4. trees by (size desc, min id asc) -- one radix sort; each rooted at its min id.
//   5. smallest-first preorder by two Euler tours: the first (any child order) gives parents and
//      subtree sizes, the adjacency is then re-sorted to (children by (size, id), parent last) and the
//      second tour gives the preorder.  Tours are ranked by pointer jumping (list ranking).
//   6. capture (block tiles R3 or the strict band) and the canonical CSR of B_i by one radix
//      sort of (pos(u) << 32 | pos(v)) keys; the rest is E_{i+1}.
// Host preprocessing, not the timed path; CUB (CUDA toolkit) provides sorts, scans and selections.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "arrow_internal.h"

namespace arrow {
namespace {

#define GD_TRY(expr)                                                                            \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess) {                                                                \
            err = std::string(#expr) + ": " + cudaGetErrorString(_e);                           \
            return 1;                                                                           \
        }                                                                                       \
    } while (0)

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// device buffer with growth
template <typename T> struct Buf {
    T *p = nullptr;
    size_t cap = 0;
    cudaError_t need(size_t n) {
        if (n <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T));
        if (e == cudaSuccess) cap = std::max<size_t>(n, 1);
        return e;
    }
    ~Buf() {
        if (p) cudaFree(p);
    }
};

template <typename T> void swap_buf(Buf<T> &a, Buf<T> &b) {
    std::swap(a.p, b.p);
    std::swap(a.cap, b.cap);
}

inline unsigned blocks_for(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 1 << 20)); }
#define GRID_LOOP(i, n) for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

__global__ void k_rows_of_entries(const int64_t *rp, int64_t n, int32_t *erow) {
    GRID_LOOP(r, n) for (int64_t e = rp[r]; e < rp[r + 1]; ++e) erow[e] = (int32_t)r;
}
__global__ void k_iota(uint32_t *a, int64_t m) { GRID_LOOP(t, m) a[t] = (uint32_t)t; }
// symmetric pattern: entry (r, c) needs (c, r) -- a binary search in row c (rows sorted, validated);
// the smallest offending row lands in *bad
__global__ void k_check_symmetric(const int64_t *rp, const int32_t *col, const int32_t *erow, int64_t nnz,
                                  unsigned long long *bad) {
    GRID_LOOP(e, nnz) {
        const int32_t r = erow[e], c = col[e];
        int64_t lo = rp[c], hi = rp[c + 1];
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (col[mid] < r) lo = mid + 1;
            else hi = mid;
        }
        if (lo == rp[c + 1] || col[lo] != r) atomicMin(bad, (unsigned long long)r);
    }
}
__global__ void k_degree(const uint32_t *ent, int64_t m, const int32_t *erow, int32_t *deg) {
    GRID_LOOP(t, m) atomicAdd(&deg[erow[ent[t]]], 1);
}
__global__ void k_head_keys(const int32_t *deg, int64_t n, uint64_t *key, int32_t *vflag) {
    GRID_LOOP(v, n) {
        vflag[v] = deg[v] > 0;
        key[v] = ((uint64_t)(0xFFFFFFFFu - (uint32_t)deg[v]) << 32) | (uint64_t)v;
    }
}
__global__ void k_mark_head(const uint64_t *sorted, int64_t h, uint8_t *in_head, int32_t *head) {
    GRID_LOOP(j, h) {
        const uint32_t v = (uint32_t)(sorted[j] & 0xFFFFFFFFu);
        in_head[v] = 1;
        head[j] = (int32_t)v;
    }
}
// home != nullptr (R25, levels >= 1): only edges inside one home
__global__ void k_gprime_flags(const uint32_t *ent, int64_t m, const int32_t *erow, const int32_t *col,
                               const uint8_t *in_head, const uint8_t *home, uint8_t *flag) {
    GRID_LOOP(t, m) {
        const uint32_t e = ent[t];
        const int32_t u = erow[e], v = col[e];
        flag[t] = (u < v && !in_head[u] && !in_head[v] && (!home || home[u] == home[v])) ? 1 : 0;
    }
}
__global__ void k_edge_keys(const uint32_t *gent, int64_t me, const int32_t *erow, const int32_t *col, uint64_t s_i,
                            uint32_t *eu, uint32_t *ev, uint64_t *ek) {
    GRID_LOOP(t, me) {
        const uint32_t e = gent[t];
        const uint32_t u = (uint32_t)erow[e], v = (uint32_t)col[e];
        eu[t] = u;
        ev[t] = v;
        ek[t] = mix64(s_i ^ (((uint64_t)u << 32) | v));
    }
}
__global__ void k_fill_u64(uint64_t *a, int64_t n, uint64_t v) { GRID_LOOP(i, n) a[i] = v; }
__global__ void k_comp_init(int32_t *comp, int64_t n) { GRID_LOOP(v, n) comp[v] = (int32_t)v; }
// Boruvka step A: lightest key per component (and mark edges whose endpoints already share one)
__global__ void k_bv_min_key(const uint32_t *eu, const uint32_t *ev, const uint64_t *ek, int64_t me, const int32_t *comp,
                             uint64_t *best, uint8_t *alive) {
    GRID_LOOP(t, me) {
        const int32_t cu = comp[eu[t]], cv = comp[ev[t]];
        if (cu == cv) {
            alive[t] = 0;
            continue;
        }
        alive[t] = 1;
        atomicMin((unsigned long long *)&best[cu], (unsigned long long)ek[t]);
        atomicMin((unsigned long long *)&best[cv], (unsigned long long)ek[t]);
    }
}
// step B: among edges with the component's lightest key, the smallest (u, v)
__global__ void k_bv_min_uv(const uint32_t *eu, const uint32_t *ev, const uint64_t *ek, int64_t me, const int32_t *comp,
                            const uint64_t *best, uint64_t *bestuv) {
    GRID_LOOP(t, me) {
        const int32_t cu = comp[eu[t]], cv = comp[ev[t]];
        if (cu == cv) continue;
        const uint64_t uv = ((uint64_t)eu[t] << 32) | ev[t];
        if (ek[t] == best[cu]) atomicMin((unsigned long long *)&bestuv[cu], (unsigned long long)uv);
        if (ek[t] == best[cv]) atomicMin((unsigned long long *)&bestuv[cv], (unsigned long long)uv);
    }
}
// step C: hook every component along its edge; a mutual pair (both chose the same edge) keeps the
// smaller id as the root; the hooking side records the forest edge
__global__ void k_bv_hook(const int32_t *roots, int64_t nr, const int32_t *comp, const uint64_t *best,
                          const uint64_t *bestuv, int32_t *par, uint32_t *fu, uint32_t *fv, unsigned *nf,
                          unsigned *hooked) {
    GRID_LOOP(j, nr) {
        const int32_t c = roots[j];
        if (best[c] == ~0ull) continue;
        const uint64_t uv = bestuv[c];
        const uint32_t u = (uint32_t)(uv >> 32), v = (uint32_t)(uv & 0xFFFFFFFFu);
        const int32_t o = comp[u] == c ? comp[v] : comp[u];
        if (bestuv[o] == uv && c < o) continue;  // mutual: o hooks onto c
        par[c] = o;
        const unsigned at = atomicAdd(nf, 1u);
        fu[at] = u;
        fv[at] = v;
        *hooked = 1u;
    }
}
__global__ void k_jump(int32_t *par, const int32_t *roots, int64_t nr, unsigned *changed) {
    GRID_LOOP(j, nr) {
        const int32_t c = roots[j];
        const int32_t p = par[c], pp = par[p];
        if (pp != p) {
            par[c] = pp;
            *changed = 1u;
        }
    }
}
__global__ void k_relabel(const int32_t *verts, int64_t nv, const int32_t *par, int32_t *comp) {
    GRID_LOOP(j, nv) {
        const int32_t v = verts[j];
        comp[v] = par[comp[v]];
    }
}
__global__ void k_root_flags(const int32_t *roots, int64_t nr, const int32_t *par, uint8_t *keep) {
    GRID_LOOP(j, nr) keep[j] = par[roots[j]] == roots[j] ? 1 : 0;
}
// tree statistics: size and min id per component root
__global__ void k_tree_stats(const int32_t *verts, int64_t nv, const int32_t *comp, int32_t *tsize, int32_t *tmin) {
    GRID_LOOP(j, nv) {
        const int32_t v = verts[j];
        atomicAdd(&tsize[comp[v]], 1);
        atomicMin(&tmin[comp[v]], v);
    }
}
__global__ void k_tree_keys(const int32_t *roots, int64_t nt, const int32_t *tsize, const int32_t *tmin, uint64_t *key,
                            int32_t *val) {
    GRID_LOOP(j, nt) {
        const int32_t r = roots[j];
        key[j] = ((uint64_t)(0xFFFFFFFFu - (uint32_t)tsize[r]) << 32) | (uint32_t)tmin[r];
        val[j] = r;
    }
}
// per tree (in tree order t): vertex offset toff (exclusive scan of sizes), index; per root: both
__global__ void k_tree_place(const int32_t *troot, int64_t nt, const int32_t *tsize, const int64_t *toff_scan,
                             int64_t *toff_of_root, int32_t *tidx_of_root) {
    GRID_LOOP(t, nt) {
        const int32_t r = troot[t];
        toff_of_root[r] = toff_scan[t];
        tidx_of_root[r] = (int32_t)t;
    }
}
__global__ void k_tree_sizes_ordered(const int32_t *troot, int64_t nt, const int32_t *tsize, int64_t *sz) {
    GRID_LOOP(t, nt) sz[t] = tsize[troot[t]];
}
// forest arcs (both directions), keyed (src << 32 | dst)
__global__ void k_arcs(const uint32_t *fu, const uint32_t *fv, int64_t nf, uint64_t *akey) {
    GRID_LOOP(t, nf) {
        akey[2 * t] = ((uint64_t)fu[t] << 32) | fv[t];
        akey[2 * t + 1] = ((uint64_t)fv[t] << 32) | fu[t];
    }
}
__global__ void k_arc_src_dst(const uint64_t *akey, int64_t na, int32_t *asrc, int32_t *adst) {
    GRID_LOOP(a, na) {
        asrc[a] = (int32_t)(akey[a] >> 32);
        adst[a] = (int32_t)(akey[a] & 0xFFFFFFFFu);
    }
}
// reverse arc: position of (dst -> src) in dst's range (ranges sorted by dst of the key: binary search)
__global__ void k_rev_sorted(const uint64_t *akey, int64_t na, const int64_t *astart, int64_t *rev) {
    GRID_LOOP(a, na) {
        const uint32_t u = (uint32_t)(akey[a] >> 32), v = (uint32_t)(akey[a] & 0xFFFFFFFFu);
        const uint64_t want = ((uint64_t)v << 32) | u;
        int64_t lo = astart[v], hi = astart[v + 1];
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (akey[mid] < want) lo = mid + 1;
            else hi = mid;
        }
        rev[a] = lo;
    }
}
// Euler-tour successor: the arc after rev(a) in the circular adjacency of dst(a); the tour of a tree
// starts at the first arc of its root, so the arc returning to that start ends the list (-1)
__global__ void k_succ(const int32_t *asrc, const int32_t *adst, int64_t na, const int64_t *rev, const int64_t *astart,
                       const int32_t *comp, const int32_t *tmin, int64_t *succ) {
    GRID_LOOP(a, na) {
        const int32_t v = adst[a];
        int64_t nx = rev[a] + 1;
        if (nx == astart[v + 1]) nx = astart[v];
        const int32_t root = tmin[comp[asrc[a]]];
        succ[a] = (nx == astart[root]) ? -1 : nx;
    }
}
// list ranking by pointer jumping: dist[a] = number of arcs after a in its tour
__global__ void k_rank_init(const int64_t *succ, int64_t na, int64_t *dist, int64_t *nxt) {
    GRID_LOOP(a, na) {
        dist[a] = succ[a] < 0 ? 0 : 1;
        nxt[a] = succ[a];
    }
}
__global__ void k_rank_step(const int64_t *dist_in, const int64_t *nxt_in, int64_t na, int64_t *dist_out,
                            int64_t *nxt_out, unsigned *more) {
    GRID_LOOP(a, na) {
        const int64_t x = nxt_in[a];
        if (x < 0) {
            dist_out[a] = dist_in[a];
            nxt_out[a] = -1;
        } else {
            dist_out[a] = dist_in[a] + dist_in[x];
            nxt_out[a] = nxt_in[x];
            if (nxt_in[x] >= 0) *more = 1u;
        }
    }
}
// first tour: forward arcs (u -> child w) have dist(a) > dist(rev a); size(w) = (dist(a) - dist(rev)+1)/2
__global__ void k_child_keys(const int32_t *asrc, const int32_t *adst, int64_t na, const int64_t *rev,
                             const int64_t *dist, uint64_t *k2, int32_t *wsize) {
    GRID_LOOP(a, na) {
        const int64_t r = rev[a];
        if (dist[a] > dist[r]) {  // forward: adst[a] is a child of asrc[a]
            const int64_t s = (dist[a] - dist[r] + 1) / 2;
            wsize[adst[a]] = (int32_t)s;
            k2[a] = ((uint64_t)s << 32) | (uint32_t)adst[a];
        } else {
            k2[a] = ~0ull;  // the parent arc goes last
        }
    }
}
__global__ void k_inverse(const int32_t *perm, int64_t na, int32_t *inv) { GRID_LOOP(a, na) inv[perm[a]] = (int32_t)a; }
__global__ void k_rev2(const int32_t *perm, const int32_t *inv, const int64_t *rev1, int64_t na, int64_t *rev2) {
    GRID_LOOP(a, na) rev2[a] = inv[rev1[perm[a]]];
}
__global__ void k_gather_i32(const int32_t *src, const int32_t *idx, int64_t n, int32_t *dst) {
    GRID_LOOP(i, n) dst[i] = src[idx[i]];
}
// second tour: preorder.  tour position of arc a = arcoff(tree) + rank; forward flag per position
__global__ void k_tour_positions(const int32_t *asrc, int64_t na, const int64_t *dist, const int64_t *rev,
                                 const int32_t *comp, const int32_t *tsize, const int64_t *toff_of_root,
                                 const int32_t *tidx_of_root, int64_t *tpos, uint8_t *fwd_at) {
    GRID_LOOP(a, na) {
        const int32_t root = comp[asrc[a]];
        const int64_t L = 2 * (int64_t)(tsize[root] - 1);
        const int64_t arcoff = 2 * (toff_of_root[root] - tidx_of_root[root]);
        const int64_t p = arcoff + (L - 1 - dist[a]);
        tpos[a] = p;
        fwd_at[p] = dist[a] > dist[rev[a]] ? 1 : 0;
    }
}
__global__ void k_preorder(const int32_t *asrc, const int32_t *adst, int64_t na, const int64_t *dist,
                           const int64_t *rev, const int64_t *tpos, const int64_t *fscan, const int32_t *comp,
                           const int64_t *toff_of_root, const int32_t *tidx_of_root, int64_t h, int32_t *perm) {
    GRID_LOOP(a, na) {
        if (!(dist[a] > dist[rev[a]])) continue;
        const int32_t root = comp[asrc[a]];
        const int64_t base = toff_of_root[root] - tidx_of_root[root];  // forward arcs of earlier trees
        const int64_t pre = 1 + fscan[tpos[a]] - base;
        perm[h + toff_of_root[root] + pre] = adst[a];
    }
}
__global__ void k_place_roots(const int32_t *troot, int64_t nt, const int32_t *tmin, const int64_t *toff_of_root,
                              int64_t h, int32_t *perm) {
    GRID_LOOP(t, nt) {
        const int32_t r = troot[t];
        perm[h + toff_of_root[r]] = tmin[r];
    }
}
__global__ void k_positions(const int32_t *perm, int64_t ni, int32_t *pos) { GRID_LOOP(p, ni) pos[perm[p]] = (int32_t)p; }
__global__ void k_capture(const uint32_t *ent, int64_t m, const int32_t *erow, const int32_t *col, const int32_t *pos,
                          int64_t b, int band, uint8_t *cap, uint8_t *rest) {
    GRID_LOOP(t, m) {
        const uint32_t e = ent[t];
        const int64_t p = pos[erow[e]], q = pos[col[e]];
        bool c = p < b || q < b;
        if (!c) c = band ? ((p > q ? p - q : q - p) <= b) : (p / b == q / b);
        cap[t] = c ? 1 : 0;
        rest[t] = c ? 0 : 1;
    }
}
__global__ void k_csr_keys(const uint32_t *capt, int64_t mc, const int32_t *erow, const int32_t *col, const int32_t *pos,
                           uint64_t *key) {
    GRID_LOOP(t, mc) {
        const uint32_t e = capt[t];
        key[t] = ((uint64_t)(uint32_t)pos[erow[e]] << 32) | (uint32_t)pos[col[e]];
    }
}
__global__ void k_row_counts(const uint64_t *key, int64_t mc, int64_t *cnt) {
    GRID_LOOP(t, mc) atomicAdd((unsigned long long *)&cnt[(key[t] >> 32) + 1], 1ull);
}
__global__ void k_low32(const uint64_t *key, int64_t mc, int32_t *out) { GRID_LOOP(t, mc) out[t] = (int32_t)(key[t] & 0xFFFFFFFFu); }

struct NotHead {
    const uint8_t *ih;
    __device__ bool operator()(const int32_t &v) const { return !ih[v]; }
};
__global__ void k_iota_i32(int32_t *a, int64_t m) { GRID_LOOP(t, m) a[t] = (int32_t)t; }
__global__ void k_count_src64(const int32_t *asrc, int64_t na, unsigned long long *cnt) {
    GRID_LOOP(a, na) atomicAdd(&cnt[asrc[a]], 1ull);
}
__global__ void k_u8_to_i64(const uint8_t *x, int64_t n, int64_t *y) { GRID_LOOP(i, n) y[i] = x[i]; }
// R25: home of each tree's root (its min id; troot holds component labels) and the vertices per home
__global__ void k_root_homes(const int32_t *troot, int64_t nt, const int32_t *tmin, const uint8_t *home, uint8_t *key) {
    GRID_LOOP(t, nt) key[t] = home[tmin[troot[t]]];
}
__global__ void k_home_sizes(const int32_t *troot, int64_t nt, const int32_t *tmin, const uint8_t *home,
                             const int32_t *tsize, unsigned long long *cnt) {
    GRID_LOOP(t, nt) atomicAdd(&cnt[home[tmin[troot[t]]]], (unsigned long long)tsize[troot[t]]);
}

// ARROW_DECOMPOSE_TRACE=1: per-phase wall times (device synchronised at each mark) on stderr
struct Trace {
    bool on = std::getenv("ARROW_DECOMPOSE_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    double acc[8] = {};
    void mark(int phase) {
        if (!on) return;
        cudaDeviceSynchronize();
        const auto now = std::chrono::steady_clock::now();
        acc[phase] += std::chrono::duration<double, std::milli>(now - t).count();
        t = now;
    }
    void print(int levels) const {
        if (!on) return;
        fprintf(stderr, "[arrow decompose gpu] levels %d  ms: upload %.1f heads %.1f edges %.1f msf %.1f trees %.1f "
                        "tours %.1f capture+csr %.1f download %.1f\n",
                levels, acc[0], acc[1], acc[2], acc[3], acc[4], acc[5], acc[6], acc[7]);
    }
};

// CUB temp storage, grown on demand
struct Cub {
    Buf<uint8_t> tmp;
    template <class F> cudaError_t run(F f) {
        size_t bytes = 0;
        cudaError_t e = f(nullptr, bytes);
        if (e != cudaSuccess) return e;
        e = tmp.need(bytes);
        if (e != cudaSuccess) return e;
        return f(tmp.p, bytes);
    }
};

}  // namespace

int la_decompose_gpu(int64_t n, const int64_t *rp, const int32_t *col_h, int64_t b, int32_t max_levels, uint64_t seed,
                     int band, int homes, int home_levels, HostDecomposition &out, std::string &err) {
    out = HostDecomposition{};
    out.n = n;
    out.b = b;
    out.band = band;
    out.homes = homes;
    out.home_levels = homes > 1 ? home_levels : 0;
    const int64_t nnz = rp[n];
    if (nnz == 0) return 0;
    if (n >= ((int64_t)1 << 30) || nnz >= ((int64_t)1 << 31) - 1) {  // CUB item counts (2 n arcs) are int
        err = "GPU decomposer: n or nnz beyond 32-bit indices";
        return 1;
    }
    Cub cub;
    Trace tr;
    Buf<int64_t> d_rp;
    Buf<int32_t> d_col, d_erow, d_deg, d_vflag_i, d_head, d_comp, d_par, d_roots, d_roots2, d_verts, d_tsize, d_tmin,
        d_troot, d_asrc, d_adst, d_asrc2, d_adst2, d_aperm, d_ainv, d_wsize, d_perm, d_pos, d_tidx, d_i32tmp;
    Buf<uint32_t> d_ent, d_ent2, d_rest, d_gent, d_eu, d_ev, d_eu2, d_ev2, d_fu, d_fv, d_capt;
    Buf<uint64_t> d_key, d_key2, d_ek, d_ek2, d_best, d_bestuv, d_akey, d_akey2, d_k2, d_k2b;
    Buf<uint8_t> d_inhead, d_flag, d_alive, d_fwd, d_cap, d_restf;
    Buf<int64_t> d_astart, d_rev, d_rev2, d_succ, d_dist, d_dist2, d_nxt, d_nxt2, d_tpos, d_fscan, d_toff_scan,
        d_toff_root, d_tsz, d_rowcnt;
    Buf<unsigned> d_flags;  // [0] nf, [1] hooked, [2] changed / more
    Buf<int64_t> d_cnt;     // selection counts
    // scratch reused by every level / round (no allocation inside the loops)
    Buf<int32_t> ids, vals, idx, idx2, cols;
    Buf<uint8_t> keep;
    Buf<int64_t> cnt, dist1, dist2, f64;
    Buf<uint64_t> k1, k1s;
    Buf<uint32_t> srcs;
    Buf<uint8_t> d_home, hk, hk2;  // R25: vertex homes (after level 0), root-home sort keys
    Buf<int32_t> troot2;
    Buf<unsigned long long> hcnt;
    GD_TRY(d_rp.need(n + 1));
    GD_TRY(d_col.need(nnz));
    GD_TRY(d_erow.need(nnz));
    GD_TRY(cudaMemcpy(d_rp.p, rp, (n + 1) * 8, cudaMemcpyHostToDevice));
    GD_TRY(cudaMemcpy(d_col.p, col_h, nnz * 4, cudaMemcpyHostToDevice));
    k_rows_of_entries<<<blocks_for(n), 256>>>(d_rp.p, n, d_erow.p);
    {  // the pattern must be symmetric (what the host path's check_symmetric tests, here on the device)
        Buf<unsigned long long> bad;
        GD_TRY(bad.need(1));
        GD_TRY(cudaMemset(bad.p, 0xff, 8));
        k_check_symmetric<<<blocks_for(nnz), 256>>>(d_rp.p, d_col.p, d_erow.p, nnz, bad.p);
        unsigned long long hb = 0;
        GD_TRY(cudaMemcpy(&hb, bad.p, 8, cudaMemcpyDeviceToHost));
        if (hb != ~0ull) {
            err = "pattern not symmetric at row " + std::to_string(hb);
            return 2;
        }
    }
    GD_TRY(d_ent.need(nnz));
    k_iota<<<blocks_for(nnz), 256>>>(d_ent.p, nnz);
    GD_TRY(d_flags.need(4));
    GD_TRY(d_cnt.need(4));
    std::vector<int32_t> isolated;
    for (int64_t v = 0; v < n; ++v)
        if (rp[v + 1] == rp[v]) isolated.push_back((int32_t)v);
    GD_TRY(d_deg.need(n));
    GD_TRY(d_vflag_i.need(n));
    GD_TRY(d_key.need(n));
    GD_TRY(d_key2.need(n));
    GD_TRY(d_inhead.need(n));
    GD_TRY(d_comp.need(n));
    GD_TRY(d_par.need(n));
    GD_TRY(d_best.need(n));
    GD_TRY(d_bestuv.need(n));
    GD_TRY(d_tsize.need(n));
    GD_TRY(d_tmin.need(n));
    GD_TRY(d_wsize.need(n));
    GD_TRY(d_pos.need(n));
    GD_TRY(d_toff_root.need(n));
    GD_TRY(d_tidx.need(n));
    GD_TRY(d_verts.need(n));
    GD_TRY(d_roots.need(n));
    GD_TRY(d_roots2.need(n));
    int64_t m = nnz;
    auto count = [&](int64_t *dst) -> cudaError_t {
        int64_t c = 0;
        cudaError_t e = cudaMemcpy(&c, d_cnt.p, 8, cudaMemcpyDeviceToHost);
        *dst = c;
        return e;
    };
    tr.mark(0);
    for (int32_t i = 0;; ++i) {
        if (m == 0) break;
        if (max_levels > 0 && i == max_levels) {
            out.residual.resize(m);
            GD_TRY(cudaMemcpy(out.residual.data(), d_ent.p, m * 4, cudaMemcpyDeviceToHost));
            std::sort(out.residual.begin(), out.residual.end());
            break;
        }
        // ---- step 1: degrees, V_i, head
        GD_TRY(cudaMemset(d_deg.p, 0, n * 4));
        k_degree<<<blocks_for(m), 256>>>(d_ent.p, m, d_erow.p, d_deg.p);
        k_head_keys<<<blocks_for(n), 256>>>(d_deg.p, n, d_key.p, d_vflag_i.p);
        // V_i (ascending ids) and its head keys
        {
            GD_TRY(ids.need(n));
            k_iota_i32<<<blocks_for(n), 256>>>(ids.p, n);
            GD_TRY(cub.run([&](void *t, size_t &s) {
                return cub::DeviceSelect::Flagged(t, s, ids.p, d_vflag_i.p, d_verts.p, d_cnt.p, (int)n);
            }));
        }
        int64_t n_i = 0;
        GD_TRY(count(&n_i));
        const int64_t h = std::min<int64_t>(b, n_i);
        GD_TRY(cub.run([&](void *t, size_t &s) {
            return cub::DeviceSelect::Flagged(t, s, d_key.p, d_vflag_i.p, d_key2.p, d_cnt.p, (int)n);
        }));
        GD_TRY(cub.run([&](void *t, size_t &s) { return cub::DeviceRadixSort::SortKeys(t, s, d_key2.p, d_key.p, (int)n_i); }));
        GD_TRY(cudaMemset(d_inhead.p, 0, n));
        GD_TRY(d_head.need(std::max<int64_t>(h, 1)));
        k_mark_head<<<blocks_for(h), 256>>>(d_key.p, h, d_inhead.p, d_head.p);
        tr.mark(1);
        const bool aware = i > 0 && homes > 1 && i <= home_levels;  // R25 at this level
        // ---- step 2: G'_i edges with their keys
        GD_TRY(d_flag.need(m));
        GD_TRY(d_gent.need(m));
        k_gprime_flags<<<blocks_for(m), 256>>>(d_ent.p, m, d_erow.p, d_col.p, d_inhead.p,
                                               aware ? d_home.p : nullptr, d_flag.p);
        GD_TRY(cub.run([&](void *t, size_t &s) {
            return cub::DeviceSelect::Flagged(t, s, d_ent.p, d_flag.p, d_gent.p, d_cnt.p, (int)m);
        }));
        int64_t me = 0;
        GD_TRY(count(&me));
        GD_TRY(d_eu.need(me));
        GD_TRY(d_ev.need(me));
        GD_TRY(d_ek.need(me));
        GD_TRY(d_eu2.need(me));
        GD_TRY(d_ev2.need(me));
        GD_TRY(d_ek2.need(me));
        GD_TRY(d_alive.need(me));
        const uint64_t s_i = mix64(seed + (uint64_t)i);
        k_edge_keys<<<blocks_for(me), 256>>>(d_gent.p, me, d_erow.p, d_col.p, s_i, d_eu.p, d_ev.p, d_ek.p);
        tr.mark(2);
        // ---- step 3: Boruvka
        k_comp_init<<<blocks_for(n), 256>>>(d_comp.p, n);
        k_comp_init<<<blocks_for(n), 256>>>(d_par.p, n);
        // forest vertices list: V_i minus head (select from d_verts with not-in-head)
        int64_t nfv = 0;
        {
            GD_TRY(cub.run([&](void *t, size_t &s) {
                return cub::DeviceSelect::If(t, s, d_verts.p, d_roots.p, d_cnt.p, (int)n_i, NotHead{d_inhead.p});
            }));
            GD_TRY(count(&nfv));
            GD_TRY(d_i32tmp.need(std::max<int64_t>(nfv, 1)));
            GD_TRY(cudaMemcpy(d_i32tmp.p, d_roots.p, nfv * 4, cudaMemcpyDeviceToDevice));  // forest vertices
        }
        int32_t *fverts = d_i32tmp.p;
        int64_t nr = nfv;  // live component roots, initially every forest vertex
        GD_TRY(d_fu.need(std::max<int64_t>(nfv, 1)));
        GD_TRY(d_fv.need(std::max<int64_t>(nfv, 1)));
        GD_TRY(cudaMemset(d_flags.p, 0, 16));
        int64_t live_e = me;
        uint32_t *eu = d_eu.p, *ev = d_ev.p, *eu2 = d_eu2.p, *ev2 = d_ev2.p;
        uint64_t *ek = d_ek.p, *ek2 = d_ek2.p;
        for (int round = 0; round < 64 && live_e > 0 && nr > 1; ++round) {
            k_fill_u64<<<blocks_for(n), 256>>>(d_best.p, n, ~0ull);
            k_fill_u64<<<blocks_for(n), 256>>>(d_bestuv.p, n, ~0ull);
            k_bv_min_key<<<blocks_for(live_e), 256>>>(eu, ev, ek, live_e, d_comp.p, d_best.p, d_alive.p);
            k_bv_min_uv<<<blocks_for(live_e), 256>>>(eu, ev, ek, live_e, d_comp.p, d_best.p, d_bestuv.p);
            GD_TRY(cudaMemset(d_flags.p + 1, 0, 4));
            k_bv_hook<<<blocks_for(nr), 256>>>(d_roots.p, nr, d_comp.p, d_best.p, d_bestuv.p, d_par.p, d_fu.p, d_fv.p,
                                               d_flags.p, d_flags.p + 1);
            unsigned hooked = 0;
            GD_TRY(cudaMemcpy(&hooked, d_flags.p + 1, 4, cudaMemcpyDeviceToHost));
            if (!hooked) break;
            for (;;) {  // pointer jumping over the component roots
                GD_TRY(cudaMemset(d_flags.p + 2, 0, 4));
                k_jump<<<blocks_for(nr), 256>>>(d_par.p, d_roots.p, nr, d_flags.p + 2);
                unsigned ch = 0;
                GD_TRY(cudaMemcpy(&ch, d_flags.p + 2, 4, cudaMemcpyDeviceToHost));
                if (!ch) break;
            }
            k_relabel<<<blocks_for(nfv), 256>>>(fverts, nfv, d_par.p, d_comp.p);
            // live roots: par[c] == c
            GD_TRY(keep.need(nr));
            k_root_flags<<<blocks_for(nr), 256>>>(d_roots.p, nr, d_par.p, keep.p);
            GD_TRY(cub.run([&](void *t, size_t &s) {
                return cub::DeviceSelect::Flagged(t, s, d_roots.p, keep.p, d_roots2.p, d_cnt.p, (int)nr);
            }));
            GD_TRY(count(&nr));
            swap_buf(d_roots, d_roots2);
            // drop edges inside one component (k_bv_min_key marked them with the pre-hook labels; the
            // survivors are re-tested next round)
            GD_TRY(cub.run([&](void *t, size_t &s) {
                return cub::DeviceSelect::Flagged(t, s, eu, d_alive.p, eu2, d_cnt.p, (int)live_e);
            }));
            GD_TRY(cub.run([&](void *t, size_t &s) {
                return cub::DeviceSelect::Flagged(t, s, ev, d_alive.p, ev2, d_cnt.p, (int)live_e);
            }));
            GD_TRY(cub.run([&](void *t, size_t &s) {
                return cub::DeviceSelect::Flagged(t, s, ek, d_alive.p, ek2, d_cnt.p, (int)live_e);
            }));
            GD_TRY(count(&live_e));
            std::swap(eu, eu2);
            std::swap(ev, ev2);
            std::swap(ek, ek2);
        }
        unsigned nf_u = 0;
        GD_TRY(cudaMemcpy(&nf_u, d_flags.p, 4, cudaMemcpyDeviceToHost));
        const int64_t nf = nf_u;
        tr.mark(3);
        // ---- step 4: trees (components incl. singletons) by (size desc, min id asc)
        GD_TRY(cudaMemset(d_tsize.p, 0, n * 4));
        // tmin[c] = c, then atomicMin over the component's vertices (the root c is one of them)
        k_comp_init<<<blocks_for(n), 256>>>(d_tmin.p, n);
        k_tree_stats<<<blocks_for(nfv), 256>>>(fverts, nfv, d_comp.p, d_tsize.p, d_tmin.p);
        // tree roots = live roots: d_roots[0..nr)  (every forest vertex's component root)
        // recount roots: components are exactly the distinct comp[] values == live roots
        const int64_t nt = nr;
        GD_TRY(d_troot.need(std::max<int64_t>(nt, 1)));
        GD_TRY(d_k2.need(std::max<int64_t>(nt, 1)));
        GD_TRY(d_k2b.need(std::max<int64_t>(nt, 1)));
        {
            GD_TRY(vals.need(std::max<int64_t>(nt, 1)));
            k_tree_keys<<<blocks_for(nt), 256>>>(d_roots.p, nt, d_tsize.p, d_tmin.p, d_k2.p, vals.p);
            GD_TRY(cub.run([&](void *t, size_t &s) {
                return cub::DeviceRadixSort::SortPairs(t, s, d_k2.p, d_k2b.p, vals.p, d_troot.p, (int)nt);
            }));
        }
        std::vector<int64_t> home_start;
        if (aware) {  // R25: stable re-sort by the home of the root, home starts
            GD_TRY(hk.need(std::max<int64_t>(nt, 1)));
            GD_TRY(hk2.need(std::max<int64_t>(nt, 1)));
            GD_TRY(troot2.need(std::max<int64_t>(nt, 1)));
            GD_TRY(hcnt.need(homes));
            k_root_homes<<<blocks_for(nt), 256>>>(d_troot.p, nt, d_tmin.p, d_home.p, hk.p);
            GD_TRY(cub.run([&](void *t, size_t &s) {
                return cub::DeviceRadixSort::SortPairs(t, s, hk.p, hk2.p, d_troot.p, troot2.p, (int)nt, 0, 8);
            }));
            GD_TRY(cudaMemcpy(d_troot.p, troot2.p, nt * 4, cudaMemcpyDeviceToDevice));
            GD_TRY(cudaMemset(hcnt.p, 0, homes * 8));
            k_home_sizes<<<blocks_for(nt), 256>>>(d_troot.p, nt, d_tmin.p, d_home.p, d_tsize.p, hcnt.p);
            std::vector<unsigned long long> hc(homes);
            GD_TRY(cudaMemcpy(hc.data(), hcnt.p, homes * 8, cudaMemcpyDeviceToHost));
            home_start.assign(homes + 1, h);
            for (int g = 0; g < homes; ++g) home_start[g + 1] = home_start[g] + (int64_t)hc[g];
        }
        GD_TRY(d_tsz.need(std::max<int64_t>(nt, 1)));
        GD_TRY(d_toff_scan.need(std::max<int64_t>(nt, 1)));
        k_tree_sizes_ordered<<<blocks_for(nt), 256>>>(d_troot.p, nt, d_tsize.p, d_tsz.p);
        GD_TRY(cub.run([&](void *t, size_t &s) {
            return cub::DeviceScan::ExclusiveSum(t, s, d_tsz.p, d_toff_scan.p, (int)nt);
        }));
        k_tree_place<<<blocks_for(nt), 256>>>(d_troot.p, nt, d_tsize.p, d_toff_scan.p, d_toff_root.p, d_tidx.p);
        tr.mark(4);
        // ---- step 5: Euler tours over the forest arcs
        const int64_t rows = (i == 0) ? n : n_i;
        GD_TRY(d_perm.need(std::max<int64_t>(rows, 1)));
        GD_TRY(cudaMemcpy(d_perm.p, d_head.p, h * 4, cudaMemcpyDeviceToDevice));
        k_place_roots<<<blocks_for(nt), 256>>>(d_troot.p, nt, d_tmin.p, d_toff_root.p, h, d_perm.p);
        const int64_t na = 2 * nf;
        if (na > 0) {
            GD_TRY(d_akey.need(na));
            GD_TRY(d_akey2.need(na));
            GD_TRY(d_asrc.need(na));
            GD_TRY(d_adst.need(na));
            GD_TRY(d_asrc2.need(na));
            GD_TRY(d_adst2.need(na));
            GD_TRY(d_aperm.need(na));
            GD_TRY(d_ainv.need(na));
            GD_TRY(d_rev.need(na));
            GD_TRY(d_rev2.need(na));
            GD_TRY(d_succ.need(na));
            GD_TRY(d_dist.need(na));
            GD_TRY(d_dist2.need(na));
            GD_TRY(d_nxt.need(na));
            GD_TRY(d_nxt2.need(na));
            GD_TRY(d_tpos.need(na));
            GD_TRY(d_fscan.need(na));
            GD_TRY(d_fwd.need(na));
            GD_TRY(d_astart.need(n + 1));
            GD_TRY(d_k2.need(na));
            GD_TRY(d_k2b.need(na));
            k_arcs<<<blocks_for(nf), 256>>>(d_fu.p, d_fv.p, nf, d_akey.p);
            GD_TRY(cub.run([&](void *t, size_t &s) { return cub::DeviceRadixSort::SortKeys(t, s, d_akey.p, d_akey2.p, (int)na); }));
            k_arc_src_dst<<<blocks_for(na), 256>>>(d_akey2.p, na, d_asrc.p, d_adst.p);
            // astart: exclusive scan of per-vertex arc counts
            GD_TRY(cnt.need(n + 1));
            GD_TRY(cudaMemset(cnt.p, 0, (n + 1) * 8));
            k_count_src64<<<blocks_for(na), 256>>>(d_asrc.p, na, reinterpret_cast<unsigned long long *>(cnt.p));
            GD_TRY(cub.run([&](void *t, size_t &s) { return cub::DeviceScan::ExclusiveSum(t, s, cnt.p, d_astart.p, (int)(n + 1)); }));
            // a pass over sorted (src, dst) adjacency: reverse arcs, successors, ranks
            auto euler_rank = [&](const int64_t *rev, int64_t *dist_out) -> int {
                k_succ<<<blocks_for(na), 256>>>(d_asrc.p, d_adst.p, na, rev, d_astart.p, d_comp.p, d_tmin.p, d_succ.p);
                k_rank_init<<<blocks_for(na), 256>>>(d_succ.p, na, d_dist.p, d_nxt.p);
                int64_t *di = d_dist.p, *ni = d_nxt.p, *dout = d_dist2.p, *nout = d_nxt2.p;
                for (int it2 = 0; it2 < 64; ++it2) {
                    GD_TRY(cudaMemset(d_flags.p + 2, 0, 4));
                    k_rank_step<<<blocks_for(na), 256>>>(di, ni, na, dout, nout, d_flags.p + 2);
                    std::swap(di, dout);
                    std::swap(ni, nout);
                    unsigned more = 0;
                    GD_TRY(cudaMemcpy(&more, d_flags.p + 2, 4, cudaMemcpyDeviceToHost));
                    if (!more) break;
                }
                GD_TRY(cudaMemcpy(dist_out, di, na * 8, cudaMemcpyDeviceToDevice));
                return 0;
            };
            k_rev_sorted<<<blocks_for(na), 256>>>(d_akey2.p, na, d_astart.p, d_rev.p);
            GD_TRY(dist1.need(na));
            if (euler_rank(d_rev.p, dist1.p)) return 1;
            // children by (subtree size, id), parent arc last: stable sort by k2, then by src
            k_child_keys<<<blocks_for(na), 256>>>(d_asrc.p, d_adst.p, na, d_rev.p, dist1.p, d_k2.p, d_wsize.p);
            {
                    GD_TRY(idx.need(na));
                GD_TRY(idx2.need(na));
                k_iota<<<blocks_for(na), 256>>>(reinterpret_cast<uint32_t *>(idx.p), na);
                GD_TRY(cub.run([&](void *t, size_t &s) {
                    return cub::DeviceRadixSort::SortPairs(t, s, d_k2.p, d_k2b.p, idx.p, idx2.p, (int)na);
                }));
                // stable by src: key = src of arc idx2[j]
                k_gather_i32<<<blocks_for(na), 256>>>(d_asrc.p, idx2.p, na, d_asrc2.p);
                GD_TRY(cub.run([&](void *t, size_t &s) {
                    return cub::DeviceRadixSort::SortPairs(t, s, d_asrc2.p, d_adst2.p, idx2.p, d_aperm.p, (int)na);
                }));
                // d_aperm[newpos] = old arc; rebuild src/dst and reverse indices in the new order
                k_gather_i32<<<blocks_for(na), 256>>>(d_asrc.p, d_aperm.p, na, d_asrc2.p);
                k_gather_i32<<<blocks_for(na), 256>>>(d_adst.p, d_aperm.p, na, d_adst2.p);
                k_inverse<<<blocks_for(na), 256>>>(d_aperm.p, na, d_ainv.p);
                k_rev2<<<blocks_for(na), 256>>>(d_aperm.p, d_ainv.p, d_rev.p, na, d_rev2.p);
                swap_buf(d_asrc, d_asrc2);
                swap_buf(d_adst, d_adst2);
            }
            GD_TRY(dist2.need(na));
            if (euler_rank(d_rev2.p, dist2.p)) return 1;
            // preorder positions from the second tour
            GD_TRY(cudaMemset(d_fwd.p, 0, na));
            k_tour_positions<<<blocks_for(na), 256>>>(d_asrc.p, na, dist2.p, d_rev2.p, d_comp.p, d_tsize.p, d_toff_root.p,
                                                     d_tidx.p, d_tpos.p, d_fwd.p);
            {
                    GD_TRY(f64.need(na));
                k_u8_to_i64<<<blocks_for(na), 256>>>(d_fwd.p, na, f64.p);
                GD_TRY(cub.run([&](void *t, size_t &s) { return cub::DeviceScan::ExclusiveSum(t, s, f64.p, d_fscan.p, (int)na); }));
            }
            k_preorder<<<blocks_for(na), 256>>>(d_asrc.p, d_adst.p, na, dist2.p, d_rev2.p, d_tpos.p, d_fscan.p, d_comp.p,
                                                d_toff_root.p, d_tidx.p, h, d_perm.p);
        }
        GD_TRY(cudaGetLastError());
        tr.mark(5);
        HostLevel L;
        L.n_i = n_i;
        L.head = h;
        L.rows = rows;
        L.home_start = std::move(home_start);
        L.perm.resize(rows);
        GD_TRY(cudaMemcpy(L.perm.data(), d_perm.p, n_i * 4, cudaMemcpyDeviceToHost));
        if (i == 0) std::copy(isolated.begin(), isolated.end(), L.perm.begin() + n_i);
        // ---- step 6: capture and the canonical CSR of B_i
        GD_TRY(cudaMemset(d_pos.p, 0xff, n * 4));
        k_positions<<<blocks_for(n_i), 256>>>(d_perm.p, n_i, d_pos.p);
        GD_TRY(d_cap.need(m));
        GD_TRY(d_restf.need(m));
        GD_TRY(d_capt.need(m));
        GD_TRY(d_rest.need(m));
        k_capture<<<blocks_for(m), 256>>>(d_ent.p, m, d_erow.p, d_col.p, d_pos.p, b, band, d_cap.p, d_restf.p);
        GD_TRY(cub.run([&](void *t, size_t &s) {
            return cub::DeviceSelect::Flagged(t, s, d_ent.p, d_cap.p, d_capt.p, d_cnt.p, (int)m);
        }));
        int64_t mc = 0;
        GD_TRY(count(&mc));
        GD_TRY(cub.run([&](void *t, size_t &s) {
            return cub::DeviceSelect::Flagged(t, s, d_ent.p, d_restf.p, d_rest.p, d_cnt.p, (int)m);
        }));
        int64_t mr = 0;
        GD_TRY(count(&mr));
        if (mc + mr != m || mc == 0) {
            err = "internal: GPU level " + std::to_string(i) + " captured nothing or lost entries";
            return 1;
        }
        {
            GD_TRY(k1.need(mc));
            GD_TRY(k1s.need(mc));
            GD_TRY(srcs.need(mc));
            k_csr_keys<<<blocks_for(mc), 256>>>(d_capt.p, mc, d_erow.p, d_col.p, d_pos.p, k1.p);
            GD_TRY(cub.run([&](void *t, size_t &s) {
                return cub::DeviceRadixSort::SortPairs(t, s, k1.p, k1s.p, d_capt.p, srcs.p, (int)mc);
            }));
            GD_TRY(d_rowcnt.need(rows + 1));
            GD_TRY(cudaMemset(d_rowcnt.p, 0, (rows + 1) * 8));
            k_row_counts<<<blocks_for(mc), 256>>>(k1s.p, mc, d_rowcnt.p);
            std::vector<int64_t> rc(rows + 1);
            GD_TRY(cudaMemcpy(rc.data(), d_rowcnt.p, (rows + 1) * 8, cudaMemcpyDeviceToHost));
            for (int64_t p = 0; p < rows; ++p) rc[p + 1] += rc[p];
            L.row_ptr = std::move(rc);
            GD_TRY(cols.need(mc));
            k_low32<<<blocks_for(mc), 256>>>(k1s.p, mc, cols.p);
            L.col.resize(mc);
            L.src.resize(mc);
            tr.mark(6);
            GD_TRY(cudaMemcpy(L.col.data(), cols.p, mc * 4, cudaMemcpyDeviceToHost));
            GD_TRY(cudaMemcpy(L.src.data(), srcs.p, mc * 4, cudaMemcpyDeviceToHost));
            tr.mark(7);
        }
        out.levels.push_back(std::move(L));
        if (i == 0 && homes > 1) {  // R25: homes from level 0's tile work and the remainder degrees
            GD_TRY(cudaMemset(d_deg.p, 0, n * 4));
            k_degree<<<blocks_for(mr), 256>>>(d_rest.p, mr, d_erow.p, d_deg.p);
            std::vector<int32_t> rem(n);
            GD_TRY(cudaMemcpy(rem.data(), d_deg.p, n * 4, cudaMemcpyDeviceToHost));
            out.home_los = home_ranges(out.levels[0], n, b, homes, rem.data());
            std::vector<uint8_t> hv(n, 0);
            for (int64_t p = 0; p < n; ++p) {
                const int64_t g = std::upper_bound(out.home_los.begin() + 1, out.home_los.end() - 1, p) -
                                  (out.home_los.begin() + 1);
                hv[out.levels[0].perm[p]] = (uint8_t)g;
            }
            GD_TRY(d_home.need(n));
            GD_TRY(cudaMemcpy(d_home.p, hv.data(), n, cudaMemcpyHostToDevice));
        }
        swap_buf(d_ent, d_rest);
        m = mr;
    }
    GD_TRY(cudaDeviceSynchronize());
    tr.print((int)out.levels.size());
    return 0;
}

}  // namespace arrow
