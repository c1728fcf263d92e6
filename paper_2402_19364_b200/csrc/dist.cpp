// dist.cpp -- distributed arrow SpMM: one process per GPU, NCCL over NVLink/NVSwitch.
//
// PAPER.md §4.1 / §6: Alg. 1 distributes the tiles of an arrow matrix over ranks with
// one broadcast of the head block D^(0) and one reduction of the head partial C^(0); Alg. 2
// moves X rows forward to the ranks of the next matrix (permutation pi_{j+1} o pi_j^-1)
// and the partial results back ("aggregated in reverse order").  Lemma 6.1 / Thm 6.2
// give the costs; their sorting network is unnecessary here (routes are static and NVSwitch is
// one hop), so each exchange is one grouped NCCL send/recv with routes computed at plan time.
//
// Layout (ARROW_ORDER_PERMUTED, R18): rank g owns the contiguous pi_0 row range [lo_g, hi_g) of X
// and Y, made of whole level-0 tiles balanced by cost (A-isolated rows go to the last rank).  For
// every level i the tiles are split contiguously by cost as well; rank g computes the body rows
// and the head-row slices B^(0,t) X_t of its level-i tiles (Alg. 1's co-location, R17).
// Per arrow_spmm call:
//   1. D0_i = X[head_i] assembled on every rank (owners fill their rows, one all-reduce for all
//      levels) -- Alg. 1 line 1; the level>=1 rows a rank's tiles need are packed by their home
//      ranks and exchanged (grouped send/recv) -- Alg. 2 forward propagation.
//   2. local K-A per level (the descriptor kernel in distributed mode: head columns read D0,
//      head partials add into C0, body rows are stored locally (level 0) or into a staging buffer
//      grouped by home rank (levels >= 1)).
//   3. staging rows go home (grouped send/recv) and all C0 are all-reduced -- Alg. 1 line 3 and
//      Alg. 2 reverse aggregation; homes add them into Y.
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "comm.h"
#include "plan.h"

namespace arrow {

struct DistLevel {
    int64_t h = 0;
    SegLevel seg;
    // forward exchange (levels >= 1)
    int64_t halo_rows = 0, send_rows = 0;
    std::vector<int64_t> recv_cnt, recv_off, send_cnt, send_off;
    int32_t *send_idx = nullptr;
    // reverse exchange (levels >= 1)
    int64_t out_rows = 0, in_rows_n = 0;
    std::vector<int64_t> out_cnt, out_off, in_cnt, in_off;
    int32_t *in_rows = nullptr;
    // heads whose home is this rank
    int64_t nhead_own = 0;
    int32_t *head_j = nullptr, *head_row = nullptr;
    // level 0: rows written as zero (entry-less rows of the home range)
    int64_t nzero = 0;
    int32_t *zero_rows = nullptr;
    // row offsets inside the k-dependent workspace
    int64_t o_d0 = 0, o_c0 = 0, o_halo = 0, o_send = 0, o_out = 0, o_in = 0;
};

// host side of one rank's part of one level (computed without a GPU; uploaded by dist_build)
struct DistHostLevel {
    int64_t h = 0;
    std::vector<int64_t> recv_cnt, send_cnt, out_cnt, in_cnt;
    std::vector<int32_t> send_idx, in_rows, head_j, head_row, zero_rows;
    std::vector<int32_t> seg_out, ent_col;
    std::vector<uint32_t> seg_end;
    std::vector<uint8_t> ent_val;
};

struct DistHost {
    int G = 1, me = 0;
    int64_t lo = 0, hi = 0;
    std::vector<DistHostLevel> L;
};

struct DistState {
    ncclComm_t comm = nullptr;
    int G = 1, me = 0;
    int64_t lo = 0, hi = 0;
    std::vector<DistLevel> L;
    std::vector<void *> allocs;
    unsigned *counters = nullptr;
    int64_t d0_rows = 0, c0_rows = 0, ws_rows = 0;
    void *ws = nullptr;
    int64_t ws_k = 0;
    int bseg = 16;
};

void dist_free(DistState *d) {
    if (!d) return;
    for (void *p : d->allocs) cudaFree(p);
    if (d->ws) cudaFree(d->ws);
    delete d;
}

namespace {

template <typename V>
int32_t *upload(DistState *S, const std::vector<V> &v, bool &ok) {
    void *d = nullptr;
    const size_t bytes = std::max<size_t>(v.size() * sizeof(V), 16);
    if (cudaMalloc(&d, bytes) != cudaSuccess) { ok = false; return nullptr; }
    S->allocs.push_back(d);
    if (!v.empty() && cudaMemcpy(d, v.data(), v.size() * sizeof(V), cudaMemcpyHostToDevice) != cudaSuccess) ok = false;
    return reinterpret_cast<int32_t *>(d);
}

// contiguous split of tiles [0, T) into G ranges of ~equal cost; returns G+1 tile boundaries
std::vector<int64_t> split_tiles(const std::vector<int64_t> &cost, int G) {
    const int64_t T = (int64_t)cost.size();
    std::vector<int64_t> pre(T + 1, 0);
    for (int64_t t = 0; t < T; ++t) pre[t + 1] = pre[t] + cost[t];
    std::vector<int64_t> tb(G + 1, T);
    tb[0] = 0;
    for (int g = 1; g < G; ++g) {
        const double target = (double)pre[T] * g / G;
        tb[g] = std::lower_bound(pre.begin(), pre.end(), (int64_t)target) - pre.begin();
        tb[g] = std::max(tb[g], tb[g - 1]);
        tb[g] = std::min(tb[g], T);
    }
    return tb;
}

std::vector<int64_t> tile_costs(const HostLevel &L, int64_t b) {
    const int64_t T = (L.n_i + b - 1) / b, h = L.head;
    std::vector<int64_t> cost(T, 0);
    for (int64_t p = h; p < L.n_i; ++p) cost[p / b] += (L.row_ptr[p + 1] - L.row_ptr[p]) + 4;
    for (int64_t j = 0; j < h; ++j)
        for (int64_t e = L.row_ptr[j]; e < L.row_ptr[j + 1]; ++e) cost[L.col[e] / b] += 1;
    return cost;
}

}  // namespace

arrow_status dist_schedule(const arrow_decomposition_s &D, int G, int me, int64_t window_rows, int32_t head_chunk,
                           size_t es, DistHost &H) {
    if (!D.res_u.empty()) return set_error(ARROW_E_UNSUPPORTED, "distributed mode does not support a residual level");
    if (G < 1 || me < 0 || me >= G) return set_error(ARROW_E_INVALID_ARG, "bad nranks/rank");
    H.G = G;
    H.me = me;
    const int64_t n = D.n, b = D.b;
    const int nl = (int)D.levels.size();

    // ---- home ranges from the level-0 tile split
    std::vector<int64_t> los(G + 1, 0);
    std::vector<int32_t> pos0(n, 0);
    if (nl > 0) {
        const HostLevel &L0 = D.levels[0];
        for (int64_t p = 0; p < n; ++p) pos0[L0.perm[p]] = (int32_t)p;
        const std::vector<int64_t> tb = split_tiles(tile_costs(L0, b), G);
        for (int g = 0; g <= G; ++g) los[g] = std::min<int64_t>(L0.n_i, tb[g] * b);
        los[G] = n;
    } else {
        for (int g = 0; g <= G; ++g) los[g] = n * g / G;
    }
    H.lo = los[me];
    H.hi = los[me + 1];
    const int64_t lo = H.lo, hi = H.hi;
    auto owner = [&](int64_t P0) -> int { return (int)(std::upper_bound(los.begin() + 1, los.end() - 1, P0) - (los.begin() + 1)); };

    H.L.resize(nl);
    for (int i = 0; i < nl; ++i) {
        const HostLevel &L = D.levels[i];
        DistHostLevel &DL = H.L[i];
        const int64_t h = L.head, n_i = L.n_i;
        DL.h = h;
        const std::vector<int64_t> tb = (i == 0) ? std::vector<int64_t>() : split_tiles(tile_costs(L, b), G);
        auto tile_owner = [&](int64_t q) -> int {
            if (i == 0) return owner(q);
            return (int)(std::upper_bound(tb.begin() + 1, tb.end() - 1, q / b) - (tb.begin() + 1));
        };
        const int64_t qa = (i == 0) ? std::min(lo, n_i) : std::min<int64_t>(n_i, tb[me] * b);
        const int64_t qb = (i == 0) ? std::min(hi, n_i) : std::min<int64_t>(n_i, tb[me + 1] * b);
        const int64_t ha = std::max(h, qa);

        // ---- forward exchange: halo slots of the vertices of my tiles, grouped by home rank
        std::vector<int32_t> halo_slot;
        if (i > 0) {
            DL.recv_cnt.assign(G, 0);
            for (int64_t q = ha; q < qb; ++q) DL.recv_cnt[owner(pos0[L.perm[q]])]++;
            std::vector<int64_t> cur(G, 0);
            for (int g = 1; g < G; ++g) cur[g] = cur[g - 1] + DL.recv_cnt[g - 1];
            halo_slot.resize(std::max<int64_t>(0, qb - ha));
            for (int64_t q = ha; q < qb; ++q) halo_slot[q - ha] = (int32_t)(cur[owner(pos0[L.perm[q]])]++);
            // what I send: rows I own that other ranks' tiles need, in their slot order
            std::vector<std::vector<int32_t>> sl(G);
            for (int64_t q = h; q < n_i; ++q) {
                const int64_t P0 = pos0[L.perm[q]];
                if (owner(P0) == me) sl[tile_owner(q)].push_back((int32_t)(P0 - lo));
            }
            DL.send_cnt.assign(G, 0);
            for (int g = 0; g < G; ++g) {
                DL.send_cnt[g] = (int64_t)sl[g].size();
                DL.send_idx.insert(DL.send_idx.end(), sl[g].begin(), sl[g].end());
            }
        }
        // ---- reverse exchange: staging slots of my level>=1 body rows, grouped by home rank
        std::vector<int32_t> out_slot;
        if (i > 0) {
            DL.out_cnt.assign(G, 0);
            for (int64_t p = ha; p < qb; ++p)
                if (L.row_ptr[p + 1] > L.row_ptr[p]) DL.out_cnt[owner(pos0[L.perm[p]])]++;
            std::vector<int64_t> cur(G, 0);
            for (int g = 1; g < G; ++g) cur[g] = cur[g - 1] + DL.out_cnt[g - 1];
            out_slot.assign(std::max<int64_t>(0, qb - ha), -1);
            for (int64_t p = ha; p < qb; ++p)
                if (L.row_ptr[p + 1] > L.row_ptr[p]) out_slot[p - ha] = (int32_t)(cur[owner(pos0[L.perm[p]])]++);
            // what I receive: rows of all ranks' tiles whose home is me, by source rank, in p order
            std::vector<std::vector<int32_t>> il(G);
            for (int64_t p = h; p < n_i; ++p) {
                if (L.row_ptr[p + 1] == L.row_ptr[p]) continue;
                const int64_t P0 = pos0[L.perm[p]];
                if (owner(P0) == me) il[tile_owner(p)].push_back((int32_t)(P0 - lo));
            }
            DL.in_cnt.assign(G, 0);
            for (int g = 0; g < G; ++g) {
                DL.in_cnt[g] = (int64_t)il[g].size();
                DL.in_rows.insert(DL.in_rows.end(), il[g].begin(), il[g].end());
            }
        }
        // ---- heads whose home is me
        for (int64_t j = 0; j < h; ++j) {
            const int64_t P0 = pos0[L.perm[j]];
            if (owner(P0) == me) { DL.head_j.push_back((int32_t)j); DL.head_row.push_back((int32_t)(P0 - lo)); }
        }
        // ---- level 0: entry-less rows of my home range (incl. A-isolated vertices) start at zero
        if (i == 0)
            for (int64_t p = std::max(lo, h); p < hi; ++p)
                if (L.row_ptr[p + 1] == L.row_ptr[p]) DL.zero_rows.push_back((int32_t)(p - lo));
        // ---- descriptor layout of my tiles, window-ordered
        auto colmap = [&](int32_t q) -> int32_t {
            if (q < h) return (int32_t)(kFlag | (uint32_t)q);
            return (i == 0) ? (int32_t)(q - lo) : halo_slot[q - ha];
        };
        auto push_val = [&](double v) {
            const size_t at = DL.ent_val.size();
            DL.ent_val.resize(at + es);
            if (es == 8) std::memcpy(DL.ent_val.data() + at, &v, 8);
            else { const float f = (float)v; std::memcpy(DL.ent_val.data() + at, &f, 4); }
        };
        const int64_t W = std::max<int64_t>(1, window_rows / b) * b;
        for (int64_t lo_w = qa; lo_w < qb; lo_w += W) {
            const int64_t hi_w = std::min(qb, lo_w + W);
            for (int64_t p = std::max(h, lo_w); p < hi_w; ++p) {
                if (L.row_ptr[p + 1] == L.row_ptr[p]) continue;
                for (int64_t e = L.row_ptr[p]; e < L.row_ptr[p + 1]; ++e) { DL.ent_col.push_back(colmap(L.col[e])); push_val(L.val[e]); }
                DL.seg_out.push_back(i == 0 ? (int32_t)(p - lo) : out_slot[p - ha]);
                DL.seg_end.push_back((uint32_t)DL.ent_col.size());
            }
            for (int64_t j = 0; j < h; ++j) {
                const int32_t *a = L.col.data() + L.row_ptr[j], *z = L.col.data() + L.row_ptr[j + 1];
                int64_t x0 = L.row_ptr[j] + (std::lower_bound(a, z, (int32_t)lo_w) - a);
                const int64_t x1 = L.row_ptr[j] + (std::lower_bound(a, z, (int32_t)hi_w) - a);
                while (x0 < x1) {
                    const int64_t x2 = std::min<int64_t>(x1, x0 + head_chunk);
                    for (int64_t e = x0; e < x2; ++e) { DL.ent_col.push_back(colmap(L.col[e])); push_val(L.val[e]); }
                    DL.seg_out.push_back((int32_t)(kFlag | (uint32_t)j));
                    DL.seg_end.push_back((uint32_t)DL.ent_col.size());
                    x0 = x2;
                }
            }
        }
    }
    return ARROW_OK;
}

static void offsets(const std::vector<int64_t> &cnt, std::vector<int64_t> &off) {
    off.assign(cnt.size() + 1, 0);
    for (size_t g = 0; g < cnt.size(); ++g) off[g + 1] = off[g] + cnt[g];
}

arrow_status dist_build(arrow_plan P, const arrow_decomposition_s &D, arrow_comm comm, int64_t window_rows,
                        int32_t head_chunk) {
    DistHost H;
    arrow_status st = dist_schedule(D, comm->nranks, comm->rank, window_rows, head_chunk, P->esize(), H);
    if (st != ARROW_OK) return st;
    auto *S = new DistState();
    P->dist = S;
    S->comm = (ncclComm_t)comm->comm;
    S->G = H.G;
    S->me = H.me;
    S->lo = H.lo;
    S->hi = H.hi;
    if (const char *e = std::getenv("ARROW_SEG_BS")) S->bseg = std::atoi(e);
    const int nl = (int)H.L.size();
    bool ok = true;
    S->L.resize(nl);
    for (int i = 0; i < nl; ++i) {
        DistHostLevel &HL = H.L[i];
        DistLevel &DL = S->L[i];
        DL.h = HL.h;
        DL.recv_cnt = HL.recv_cnt;
        DL.send_cnt = HL.send_cnt;
        DL.out_cnt = HL.out_cnt;
        DL.in_cnt = HL.in_cnt;
        if (i > 0) {
            offsets(DL.recv_cnt, DL.recv_off);
            offsets(DL.send_cnt, DL.send_off);
            offsets(DL.out_cnt, DL.out_off);
            offsets(DL.in_cnt, DL.in_off);
            DL.halo_rows = DL.recv_off.back();
            DL.send_rows = DL.send_off.back();
            DL.out_rows = DL.out_off.back();
            DL.in_rows_n = DL.in_off.back();
        }
        DL.send_idx = upload(S, HL.send_idx, ok);
        DL.in_rows = upload(S, HL.in_rows, ok);
        DL.nhead_own = (int64_t)HL.head_j.size();
        DL.head_j = upload(S, HL.head_j, ok);
        DL.head_row = upload(S, HL.head_row, ok);
        DL.nzero = (int64_t)HL.zero_rows.size();
        DL.zero_rows = upload(S, HL.zero_rows, ok);
        DL.seg.nseg = (int64_t)HL.seg_out.size();
        DL.seg.mode = 0;  // every output row is written exactly once (local Y at level 0, staging otherwise)
        DL.seg.seg_out = upload(S, HL.seg_out, ok);
        DL.seg.seg_end = reinterpret_cast<uint32_t *>(upload(S, HL.seg_end, ok));
        DL.seg.ent_col = upload(S, HL.ent_col, ok);
        DL.seg.ent_val = upload(S, HL.ent_val, ok);
    }
    if (!ok) return set_error(ARROW_E_CUDA, "cudaMalloc/cudaMemcpy of the distributed layout failed");
    // workspace row offsets: [D0 | C0 | halo | send | out | in]
    int64_t r = 0;
    for (auto &DL : S->L) { DL.o_d0 = r; r += DL.h; }
    S->d0_rows = r;
    for (auto &DL : S->L) { DL.o_c0 = r; r += DL.h; }
    S->c0_rows = r - S->d0_rows;
    for (auto &DL : S->L) { DL.o_halo = r; r += DL.halo_rows; }
    for (auto &DL : S->L) { DL.o_send = r; r += DL.send_rows; }
    for (auto &DL : S->L) { DL.o_out = r; r += DL.out_rows; }
    for (auto &DL : S->L) { DL.o_in = r; r += DL.in_rows_n; }
    S->ws_rows = r;
    if (cudaMalloc(&S->counters, (nl + 1) * sizeof(unsigned)) != cudaSuccess)
        return set_error(ARROW_E_CUDA, "cudaMalloc(counters)");
    S->allocs.push_back(S->counters);
    P->local_begin = S->lo;
    P->local_end = S->hi;
    return ARROW_OK;
}

#define DCUDA(expr)                                                                                 \
    do {                                                                                            \
        cudaError_t _e = (expr);                                                                    \
        if (_e != cudaSuccess) return set_error(ARROW_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)
#define DNCCL(expr)                                                                                 \
    do {                                                                                            \
        arrow_status _s = comm_status((int)(expr), #expr);                                          \
        if (_s != ARROW_OK) return _s;                                                              \
    } while (0)
#define DK(expr)                                                                                    \
    do {                                                                                            \
        int _e = (expr);                                                                            \
        if (_e) return set_error(ARROW_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString((cudaError_t)_e)); \
    } while (0)

arrow_status dist_spmm(arrow_plan P, const void *X, void *Y, int64_t k, cudaStream_t st) {
    DistState *S = P->dist;
    const int dt = P->dtype == ARROW_F64 ? 1 : 0;
    const size_t es = P->esize();
    const ncclDataType_t nt = dt ? ncclDouble : ncclFloat;
    const int G = S->G, me = S->me, nl = (int)S->L.size();
    if (nl == 0) {
        DCUDA(cudaMemsetAsync(Y, 0, (size_t)(S->hi - S->lo) * k * es, st));
        return ARROW_OK;
    }
    if (k > S->ws_k) {
        DCUDA(cudaStreamSynchronize(st));
        if (S->ws) cudaFree(S->ws);
        S->ws = nullptr;
        S->ws_k = 0;
        DCUDA(cudaMalloc(&S->ws, (size_t)std::max<int64_t>(S->ws_rows, 1) * k * es));
        S->ws_k = k;
    }
    char *ws = reinterpret_cast<char *>(S->ws);
    auto row = [&](int64_t r) { return ws + (size_t)r * k * es; };
    const char *Xc = reinterpret_cast<const char *>(X);
    char *Yc = reinterpret_cast<char *>(Y);
    // profiling: three intervals (pre-exchange, compute, post-exchange), each with its own event pair
    cudaEvent_t pe[6] = {};
    auto mark = [&](int i) {
        if (!P->profiling) return;
        cudaEventCreate(&pe[i]);
        cudaEventRecord(pe[i], st);
    };
    mark(0);
    static const bool trace = std::getenv("ARROW_DIST_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto tmark = [&]() {
        if (!trace) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        tev.push_back(e);
    };
    tmark();
    // 1. D0 (owners fill their head rows), C0 = 0, pack the forward rows
    DCUDA(cudaMemsetAsync(S->counters, 0, (nl + 1) * sizeof(unsigned), st));
    DCUDA(cudaMemsetAsync(row(0), 0, (size_t)(S->d0_rows + S->c0_rows) * k * es, st));
    for (auto &DL : S->L) {
        DK(launch_rows(dt, X, DL.head_row, DL.head_j, DL.nhead_own, k, 0, row(DL.o_d0), st));
        if (DL.send_rows) DK(launch_rows(dt, X, DL.send_idx, nullptr, DL.send_rows, k, 0, row(DL.o_send), st));
    }
    tmark();  // after memsets, D0 fill, pack
    DNCCL(ncclGroupStart());
    for (auto &DL : S->L) {
        if (DL.recv_cnt.empty()) continue;
        for (int g = 0; g < G; ++g) {
            if (g == me) continue;
            if (DL.send_cnt[g]) DNCCL(ncclSend(row(DL.o_send + DL.send_off[g]), DL.send_cnt[g] * k, nt, g, S->comm, st));
            if (DL.recv_cnt[g]) DNCCL(ncclRecv(row(DL.o_halo + DL.recv_off[g]), DL.recv_cnt[g] * k, nt, g, S->comm, st));
        }
    }
    DNCCL(ncclAllReduce(row(0), row(0), S->d0_rows * k, nt, ncclSum, S->comm, st));
    DNCCL(ncclGroupEnd());
    tmark();  // after forward exchange + D0 all-reduce
    for (auto &DL : S->L)
        if (!DL.recv_cnt.empty() && DL.send_cnt[me])
            DCUDA(cudaMemcpyAsync(row(DL.o_halo + DL.recv_off[me]), row(DL.o_send + DL.send_off[me]),
                                  (size_t)DL.send_cnt[me] * k * es, cudaMemcpyDeviceToDevice, st));
    tmark();  // after self copies
    mark(1);
    mark(2);

    // 2. local compute per level
    for (int i = 0; i < nl; ++i) {
        DistLevel &DL = S->L[i];
        if (i == 0 && DL.nzero) DK(launch_zero_rows(dt, DL.zero_rows, DL.nzero, k, Y, st));
        const void *src = (i == 0) ? X : (const void *)row(DL.o_halo);
        void *dst = (i == 0) ? Y : (void *)row(DL.o_out);
        DK(launch_seg(dt, 1, DL.seg, src, row(DL.o_d0), dst, row(DL.o_c0), k, P->num_sms, S->counters + i, S->bseg, st));
    }
    mark(3);
    mark(4);
    tmark();  // after compute

    // 3. reverse exchange + head reduction
    DNCCL(ncclGroupStart());
    for (auto &DL : S->L) {
        if (DL.out_cnt.empty()) continue;
        for (int g = 0; g < G; ++g) {
            if (g == me) continue;
            if (DL.out_cnt[g]) DNCCL(ncclSend(row(DL.o_out + DL.out_off[g]), DL.out_cnt[g] * k, nt, g, S->comm, st));
            if (DL.in_cnt[g]) DNCCL(ncclRecv(row(DL.o_in + DL.in_off[g]), DL.in_cnt[g] * k, nt, g, S->comm, st));
        }
    }
    DNCCL(ncclAllReduce(row(S->d0_rows), row(S->d0_rows), S->c0_rows * k, nt, ncclSum, S->comm, st));
    DNCCL(ncclGroupEnd());
    tmark();  // after reverse exchange + C0 all-reduce
    for (auto &DL : S->L)
        if (!DL.out_cnt.empty() && DL.out_cnt[me])
            DCUDA(cudaMemcpyAsync(row(DL.o_in + DL.in_off[me]), row(DL.o_out + DL.out_off[me]),
                                  (size_t)DL.out_cnt[me] * k * es, cudaMemcpyDeviceToDevice, st));
    // 4. Y[level-0 heads] = C0_0 (home rank 0), then every level >= 1 adds its rows and head partials
    DK(launch_rows(dt, row(S->L[0].o_c0), S->L[0].head_j, S->L[0].head_row, S->L[0].nhead_own, k, 0, Y, st));
    for (int i = 1; i < nl; ++i) {
        DistLevel &DL = S->L[i];
        if (DL.in_rows_n) DK(launch_rows(dt, row(DL.o_in), nullptr, DL.in_rows, DL.in_rows_n, k, 1, Y, st));
        DK(launch_rows(dt, row(DL.o_c0), DL.head_j, DL.head_row, DL.nhead_own, k, 1, Y, st));
    }
    mark(5);
    tmark();  // after adds
    if (trace && !tev.empty()) {
        cudaEventSynchronize(tev.back());
        std::string line = "[arrow dist rank " + std::to_string(me) + "] phases ms:";
        for (size_t i = 1; i < tev.size(); ++i) {
            float ms = 0;
            cudaEventElapsedTime(&ms, tev[i - 1], tev[i]);
            line += " " + std::to_string(ms);
        }
        int64_t fs = 0, fr = 0, rs = 0, rr = 0;
        for (auto &DL : S->L) {
            for (int g = 0; g < G && !DL.recv_cnt.empty(); ++g) {
                if (g == me) continue;
                fs += DL.send_cnt[g]; fr += DL.recv_cnt[g]; rs += DL.out_cnt[g]; rr += DL.in_cnt[g];
            }
        }
        line += " | rows fwd send " + std::to_string(fs) + " recv " + std::to_string(fr) + ", rev send " +
                std::to_string(rs) + " recv " + std::to_string(rr) + ", d0/c0 rows " + std::to_string(S->d0_rows);
        fprintf(stderr, "%s\n", line.c_str());
        for (auto e : tev) cudaEventDestroy(e);
    }
    if (P->profiling) {
        P->prof.push_back(ProfRec{ARROW_K_COMM, P->prof_pos++, pe[0], pe[1]});
        P->prof.push_back(ProfRec{ARROW_K_SEGMENTS, P->prof_pos++, pe[2], pe[3]});
        P->prof.push_back(ProfRec{ARROW_K_COMM, P->prof_pos++, pe[4], pe[5]});
        P->prof_acc.calls += 1;
    }
    (void)Xc;
    (void)Yc;
    return ARROW_OK;
}

}  // namespace arrow

extern "C" arrow_status arrow_dist_schedule(arrow_decomposition d, int32_t nranks, int32_t rank, int64_t window_rows,
                                            int32_t head_chunk, int64_t *lohi, int64_t *counts) {
    if (!d || !lohi) return arrow::set_error(ARROW_E_INVALID_ARG, "NULL argument");
    arrow::DistHost H;
    arrow_status st = arrow::dist_schedule(*d, nranks, rank, window_rows > 0 ? window_rows : arrow::kDefaultWindowRows,
                                           head_chunk > 0 ? head_chunk : arrow::kDefaultHeadChunk, 8, H);
    if (st != ARROW_OK) return st;
    lohi[0] = H.lo;
    lohi[1] = H.hi;
    if (counts) {
        // per level: [send_cnt[G], recv_cnt[G], out_cnt[G], in_cnt[G], entries, segments, heads_owned, zero_rows]
        const int G = nranks;
        int64_t *c = counts;
        for (auto &L : H.L) {
            for (int g = 0; g < G; ++g) c[g] = L.send_cnt.empty() ? 0 : L.send_cnt[g];
            for (int g = 0; g < G; ++g) c[G + g] = L.recv_cnt.empty() ? 0 : L.recv_cnt[g];
            for (int g = 0; g < G; ++g) c[2 * G + g] = L.out_cnt.empty() ? 0 : L.out_cnt[g];
            for (int g = 0; g < G; ++g) c[3 * G + g] = L.in_cnt.empty() ? 0 : L.in_cnt[g];
            c[4 * G + 0] = (int64_t)L.ent_col.size();
            c[4 * G + 1] = (int64_t)L.seg_out.size();
            c[4 * G + 2] = (int64_t)L.head_j.size();
            c[4 * G + 3] = (int64_t)L.zero_rows.size();
            c += 4 * G + 4;
        }
    }
    return ARROW_OK;
}
