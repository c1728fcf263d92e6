// dist.cpp -- distributed arrow SpMM: one process per GPU, NCCL over NVLink/NVSwitch.
//
// PAPER.md §4.1 / §6: Alg. 1 distributes the tiles of an arrow matrix over ranks with
// one broadcast of the head block D^(0) and one reduction of the head partial C^(0); Alg. 2
// moves X rows forward to the ranks of the next matrix (permutation pi_{j+1} o pi_j^-1)
// and the partial results back ("aggregated in reverse order").  Lemma 6.1 / Thm 6.2
// give the costs; their sorting network is unnecessary here (routes are static and NVSwitch is
// one hop), so each exchange is ONE grouped NCCL send/recv per peer, routes computed at plan time.
//
// Layout (ARROW_ORDER_PERMUTED, R18): rank g owns the contiguous pi_0 row range [lo_g, hi_g) of X
// and Y, made of whole level-0 tiles balanced by cost (A-isolated rows go to the last rank).  For
// every level i the tiles are split contiguously by cost as well; rank g computes the body rows
// and the head-row slices B^(0,t) X_t of its level-i tiles (Alg. 1's co-location, R17).
// Communication buffers are peer-major (for peer g: level 1, level 2, ...), so every exchange is
// one contiguous send and one contiguous receive per peer; a rank's own rows never leave the GPU
// (packed straight into its halo, added straight from its staging buffer).
//
// Per arrow_spmm call, NCCL transport (compute stream S = the caller's, communication stream C):
//   S: one row-mover launch: my owned head rows into D0, C0 = 0, X rows packed for the peers and
//      for this rank's own halo (and the strict-band H0 rows); zero Y rows no K-A launch writes -> e0
//   C: Alg. 1 line 1, Broadcast(D^(0)): one ncclBroadcast per owner of level 0's head block (+ the
//      strict-band H0 send/recv) -> e1; grouped send/recv of the forward rows + the broadcasts of
//      the other levels' head blocks -> e2                 (Alg. 2 forward propagation)
//   S: wait e1; K-A level 0 (overlaps the forward exchange); wait e2; K-A levels >= 1 into the
//      peer-major staging buffer -> e3
//   C: wait e3; grouped send/recv of the staging rows to their homes + Alg. 1 line 3, Reduce(C^(0)):
//      one ncclReduce per owner of each head block -> e4    (Alg. 2 reverse aggregation)
//   S: add this rank's own staging rows (overlaps the reverse exchange); wait e4; add received
//      rows and owned head partials -- both as CSR gather-adds, contributions in level order.
// K-A leaves a few SMs' worth of blocks out (DistState::reserve_sms) so that the NCCL kernels can
// run next to it.  The P2P transport (dist_spmm_p2p) replaces the collectives by stores into the
// peers' memory and flag barriers.
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "comm.h"
#include "plan.h"

namespace arrow {

// host side of one rank's part of one level (computed without a GPU; uploaded by dist_build)
struct DistHostLevel {
    int64_t h = 0;
    std::vector<int64_t> recv_cnt, send_cnt, out_cnt, in_cnt;  // per peer (levels >= 1)
    std::vector<int32_t> head_j, head_row, zero_rows;
    HostSegs segs;  // K-A work of this rank (layout.cpp pads and uploads it)
};

struct DistHost {
    int G = 1, me = 0;
    // D0 / C0 row of head j of level i: NCCL transport = owner-major (level 0's heads first, then the
    // heads of levels >= 1, each block ordered by owning rank), so Alg. 1's broadcast of D^(0) and
    // reduction of C^(0) are one ncclBroadcast / ncclReduce per owner (rows [blk[r], blk[r+1]) of a
    // block); P2P transport = level-major (d0_off[i] + j)
    std::vector<std::vector<int32_t>> d0_index;
    std::vector<int64_t> blk0, blk1;  // [G + 1] owner ranges of the level-0 block / levels >= 1 block
    int64_t lo = 0, hi = 0;
    std::vector<DistHostLevel> L;
    // peer-major, levels >= 1 concatenated per peer:
    std::vector<int32_t> send_idx_peers;  // local X rows packed for the peers (peer order, me skipped)
    std::vector<int32_t> send_idx_self;   // local X rows packed into my own halo chunk
    std::vector<int32_t> in_rows_peers;   // local Y rows of the received rows (peer order, me skipped)
    std::vector<int32_t> in_rows_self;    // local Y rows of my own staging chunk
    std::vector<int64_t> send_peer, recv_peer, out_peer, in_peer;  // per-peer totals (rows)
    int64_t halo_rows = 0, out_rows = 0;                             // incl. my own chunks
    int64_t halo_self_off = 0, out_self_off = 0;                     // my own chunks' offsets
    // P2P transport (p2p != 0): workspace of rank t = [D0 | C0 x 2 | halo_t | stage_t]; rows
    // are encoded (rank << kPeerShift | workspace row)
    int p2p = 0;
    int64_t d0_rows = 0;
    int64_t zero_tail_lo = 0, zero_tail_n = 0;  // local Y rows of the A-isolated tail (written as 0)
    std::vector<int64_t> halo_all, stage_all;           // per rank
    std::vector<int32_t> d0push_src, d0push_dst;        // my heads -> every rank's D0
    std::vector<int32_t> pack_src, pack_dst;            // my X rows -> my send chunks / my own halo (DMA)
    std::vector<int64_t> send_row, halo_dst_row;        // per peer: my send chunk, its place in the peer's halo
    int64_t send_rows = 0;
    std::vector<std::pair<int32_t, int32_t>> post;      // (local Y row, encoded source row)
    // strict band, level 0: H0 = the outside rows my level-0 body rows read (ascending q, grouped by
    // home), at workspace row o_h0 of every rank (P2P: [D0 | C0 x 2 | H0 | halo ...], NCCL:
    // [D0 | C0 | H0 | halo ...]), h0_max rows reserved on every rank
    int64_t h0_max = 0, o_h0 = 0;
    std::vector<int32_t> h0_slot_q;
    std::vector<int32_t> send0_idx;                     // NCCL: my local X rows for the peers' H0 (peer order)
};

struct DistState {
    ncclComm_t comm = nullptr;
    int G = 1, me = 0;
    int64_t lo = 0, hi = 0;
    int nl = 0;
    int p2p = 0;
    std::vector<int64_t> h, d0_off;  // head rows per level, offset of the level inside D0 / C0
    std::vector<int64_t> blk0, blk1; // NCCL: owner ranges of the level-0 / levels >= 1 head blocks
    int64_t d0_rows = 0;
    std::vector<SegLevel> seg;
    std::vector<int64_t> send_peer, recv_peer, out_peer, in_peer;
    // k-dependent workspace (rows).  NCCL: [D0 | C0 | halo | send | staging | recv];
    // P2P: [D0 | C0 (call parity 0) | C0 (parity 1) | halo | stage], shared with the peers
    int64_t o_d0 = 0, o_c0 = 0, o_halo = 0, o_send = 0, o_out = 0, o_in = 0, ws_rows = 0;
    // strict band: level-0 outside rows (H0) and, NCCL, my packed rows for the peers' H0 (S0)
    int64_t o_h0 = 0, o_s0 = 0;
    std::vector<int64_t> send0_peer, recv0_peer;
    // NCCL: pre-exchange row mover (src X, dst workspace)
    int32_t *pre_src = nullptr, *pre_dst = nullptr;
    int64_t n_pre = 0;
    // P2P: pushes of my head rows into every D0 and of my X rows into every halo (encoded rows)
    int32_t *d0push_src = nullptr, *d0push_dst = nullptr;
    int64_t n_d0push = 0;
    // P2P halo: X rows packed per peer, then one copy-engine transfer per peer into its halo
    int32_t *pack_src = nullptr, *pack_dst = nullptr;
    int64_t n_pack = 0;
    std::vector<int64_t> send_row, halo_dst_row;
    int32_t *zero_rows = nullptr;  // Y rows no K-A launch writes (+ owned level-0 heads)
    int64_t n_zero = 0;
    int64_t zero_tail_lo = 0, zero_tail_n = 0;
    // CSR gather-adds into Y (NCCL: own staging rows / received rows + head partials; P2P: post only)
    int32_t *self_ptr = nullptr, *self_src = nullptr, *self_dst = nullptr;
    int32_t *post_ptr = nullptr, *post_src = nullptr, *post_dst = nullptr;
    int64_t n_self = 0, n_post = 0;
    void *ws = nullptr;
    int64_t ws_k = 0;
    PeerPtrs ws_peer{}, flags_peer{};  // P2P: every rank's workspace / flag array (mine included)
    unsigned *flags = nullptr;
    unsigned epoch[3] = {0, 0, 0};
    uint64_t calls = 0;
    std::vector<void *> allocs;
    unsigned *counters = nullptr;
    cudaStream_t cs = nullptr;
    cudaEvent_t ev[6] = {};
    // P2P DMA halo: one copy stream per peer, so the transfers to different peers run on
    // different copy engines concurrently
    std::vector<cudaStream_t> ds;
    std::vector<cudaEvent_t> ds_ev;
    int reserve_sms = 16;  // NCCL transport: SMs' worth of K-A blocks left free for the NCCL kernels
    int64_t fwd_rows = 0, rev_rows = 0;  // rows exchanged with peers (trace)
    bool ready = false;                  // dist_build completed on this rank (teardown is collective)
};

namespace {
void close_peers(DistState *d, PeerPtrs &pp) {
    for (int g = 0; g < d->G && g < kMaxPeers; ++g)
        if (g != d->me && pp.p[g]) cudaIpcCloseMemHandle(pp.p[g]);
    pp = PeerPtrs{};
}
}  // namespace

namespace {

template <typename V>
int32_t *upload(DistState *S, const V *data, size_t count, bool &ok) {
    void *d = nullptr;
    const size_t bytes = std::max<size_t>(count * sizeof(V), 16);
    if (cudaMalloc(&d, bytes) != cudaSuccess) { ok = false; return nullptr; }
    S->allocs.push_back(d);
    if (count && cudaMemcpy(d, data, count * sizeof(V), cudaMemcpyHostToDevice) != cudaSuccess) ok = false;
    return reinterpret_cast<int32_t *>(d);
}
template <typename V>
int32_t *upload(DistState *S, const std::vector<V> &v, bool &ok) { return upload(S, v.data(), v.size(), ok); }

// contiguous split of tiles [0, T) into G ranges of ~equal cost; returns G+1 tile boundaries
std::vector<int64_t> split_tiles(const std::vector<int64_t> &cost, int G) {
    std::vector<int64_t> pre(cost.size() + 1, 0);
    for (size_t t = 0; t < cost.size(); ++t) pre[t + 1] = pre[t] + cost[t];
    return split_prefix(pre, G);
}

std::vector<int64_t> tile_costs(const HostLevel &L, int64_t b) {
    const int64_t T = (L.n_i + b - 1) / b, h = L.head;
    std::vector<int64_t> cost(T, 0);
    for (int64_t p = h; p < L.n_i; ++p) cost[p / b] += (L.row_ptr[p + 1] - L.row_ptr[p]) + 4;
    for (int64_t j = 0; j < h; ++j)
        for (int64_t e = L.row_ptr[j]; e < L.row_ptr[j + 1]; ++e) cost[L.col[e] / b] += 1;
    return cost;
}

// CSR of (dst, src) contributions grouped by dst, contributions of one dst kept in list order
void build_csr(const std::vector<std::pair<int32_t, int32_t>> &c, std::vector<int32_t> &ptr, std::vector<int32_t> &src,
               std::vector<int32_t> &dst) {
    std::vector<int32_t> ord(c.size());
    for (size_t i = 0; i < c.size(); ++i) ord[i] = (int32_t)i;
    std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return c[a].first < c[b].first; });
    ptr.assign(1, 0);
    src.clear();
    dst.clear();
    for (size_t i = 0; i < ord.size(); ++i) {
        const auto &e = c[ord[i]];
        if (dst.empty() || dst.back() != e.first) {
            if (!dst.empty()) ptr.push_back((int32_t)src.size());
            dst.push_back(e.first);
        }
        src.push_back(e.second);
    }
    if (!dst.empty()) ptr.push_back((int32_t)src.size());
}

}  // namespace

arrow_status dist_schedule(const arrow_decomposition_s &D, int G, int me, int64_t window_rows, int64_t window_rows0,
                           int32_t head_chunk, size_t es, int p2p, DistHost &H) {
    if (!D.res_u.empty()) return set_error(ARROW_E_UNSUPPORTED, "distributed mode does not support a residual level");
    if (G < 1 || me < 0 || me >= G) return set_error(ARROW_E_INVALID_ARG, "bad nranks/rank");
    if (p2p && G > kMaxPeers) return set_error(ARROW_E_UNSUPPORTED, "P2P transport supports at most 8 ranks");
    H.G = G;
    H.me = me;
    const int64_t n = D.n, b = D.b;
    const int nl = (int)D.levels.size();

    // ---- home ranges from the level-0 tile split (home-aware decompositions for G ranks: the ranges
    // the arrangement was made for, R25)
    std::vector<int64_t> los(G + 1, 0);
    std::vector<int32_t> pos0(n, 0);
    const bool aware = G > 1 && D.homes == G && nl > 0;
    if (aware) {
        const HostLevel &L0 = D.levels[0];
        for (int64_t p = 0; p < n; ++p) pos0[L0.perm[p]] = (int32_t)p;
        los = D.home_los;
    } else if (nl > 0) {
        const HostLevel &L0 = D.levels[0];
        for (int64_t p = 0; p < n; ++p) pos0[L0.perm[p]] = (int32_t)p;
        // A-isolated rows (positions >= n_0, R8) go to the last rank: one pseudo tile costing a
        // row write each, so that rank takes correspondingly fewer level-0 tiles
        std::vector<int64_t> cost = tile_costs(L0, b);
        cost.push_back(n - L0.n_i);
        const std::vector<int64_t> tb = split_tiles(cost, G);
        for (int g = 0; g <= G; ++g) los[g] = std::min<int64_t>(L0.n_i, tb[g] * b);
        los[G] = n;
    } else {
        for (int g = 0; g <= G; ++g) los[g] = n * g / G;
    }
    H.lo = los[me];
    H.hi = los[me + 1];
    const int64_t lo = H.lo, hi = H.hi;
    auto owner = [&](int64_t P0) -> int {
        return (int)(std::upper_bound(los.begin() + 1, los.end() - 1, P0) - (los.begin() + 1));
    };

    // ---- pass 1: tile split and per-peer counts of every level
    // level i >= 1: contiguous chunks c of tiles [tbs[i][c], tbs[i][c+1]); chunk c goes to rank
    // rk[i][c] (cr[i][g] = chunk of rank g): per level the heaviest chunk goes to the rank with the
    // least work so far over the previous levels (LPT), so per-level rounding does not pile up
    std::vector<std::vector<int64_t>> tbs(nl);
    std::vector<std::vector<int>> rk(nl), cr(nl);
    std::vector<int64_t> load(G, 0);
    auto range = [&](int i, int g, int64_t &qa, int64_t &qb) {
        const int64_t n_i = D.levels[i].n_i;
        if (i == 0) { qa = std::min(los[g], n_i); qb = std::min(los[g + 1], n_i); }
        else {
            const int c = cr[i][g];
            qa = std::min<int64_t>(n_i, tbs[i][c] * b);
            qb = std::min<int64_t>(n_i, tbs[i][c + 1] * b);
        }
    };
    H.L.resize(nl);
    // strict band: a body row p also reads the columns q with |p - q| <= b that lie outside its
    // rank's tile range [qa, qb) -- only rows within b of the range ends can.  outside(i, t): those
    // columns of rank t's level-i body rows, heads excluded (D0 serves them), ascending, unique.
    const bool strict = D.band == ARROW_BAND_STRICT;
    auto outside = [&](int i, int t) {
        std::vector<int32_t> o;
        if (!strict) return o;
        const HostLevel &L = D.levels[i];
        int64_t qa, qb;
        range(i, t, qa, qb);
        const int64_t ha = std::max(L.head, qa);
        if (ha >= qb) return o;
        auto scan = [&](int64_t p0, int64_t p1) {
            for (int64_t p = p0; p < p1; ++p)
                for (int64_t e = L.row_ptr[p]; e < L.row_ptr[p + 1]; ++e) {
                    const int32_t q = L.col[e];
                    if (q >= L.head && (q < qa || q >= qb)) o.push_back(q);
                }
        };
        const int64_t m1 = std::min(qb, qa + b);
        scan(ha, m1);
        scan(std::max(m1, qb - b), qb);
        std::sort(o.begin(), o.end());
        o.erase(std::unique(o.begin(), o.end()), o.end());
        return o;
    };
    // RC / OC[i][t * G + h]: halo rows (all) / body rows with entries of rank t's level-i tiles whose home is h
    std::vector<std::vector<int64_t>> RC(nl, std::vector<int64_t>((size_t)G * G, 0)), OC = RC;
    // sl[i][g]: local X rows I own that g's level-i tiles need (g's halo slot order);
    // il[i][g]: local Y rows of g's level-i body rows whose home is me (g's staging order)
    std::vector<std::vector<std::vector<int32_t>>> sl(nl), il(nl);
    for (int i = 0; i < nl; ++i) {
        const HostLevel &L = D.levels[i];
        DistHostLevel &DL = H.L[i];
        DL.h = L.head;
        if (i == 0) continue;
        if (aware && (int)L.home_start.size() == G + 1) {
            // R25: rank g takes the tiles of home g's trees (boundaries at the nearest tile edge)
            const std::vector<int64_t> cost = tile_costs(L, b);
            const int64_t T = (int64_t)cost.size();
            tbs[i].assign(G + 1, T);
            tbs[i][0] = 0;
            for (int g = 1; g < G; ++g)
                tbs[i][g] = std::min(std::max((L.home_start[g] + b / 2) / b, tbs[i][g - 1]), T);
            rk[i].resize(G);
            cr[i].resize(G);
            for (int g = 0; g < G; ++g) {
                rk[i][g] = cr[i][g] = g;
                for (int64_t t = tbs[i][g]; t < tbs[i][g + 1]; ++t) load[g] += cost[t];
            }
        } else {
            const std::vector<int64_t> cost = tile_costs(L, b);
            tbs[i] = split_tiles(cost, G);
            std::vector<int64_t> cc(G, 0);
            for (int c = 0; c < G; ++c)
                for (int64_t t = tbs[i][c]; t < tbs[i][c + 1]; ++t) cc[c] += cost[t];
            std::vector<int> co(G), ro(G);
            for (int c = 0; c < G; ++c) co[c] = ro[c] = c;
            std::stable_sort(co.begin(), co.end(), [&](int a, int z) { return cc[a] > cc[z]; });
            std::stable_sort(ro.begin(), ro.end(), [&](int a, int z) { return load[a] < load[z]; });
            rk[i].assign(G, 0);
            cr[i].assign(G, 0);
            for (int j = 0; j < G; ++j) {
                rk[i][co[j]] = ro[j];
                cr[i][ro[j]] = co[j];
                load[ro[j]] += cc[co[j]];
            }
        }
        const int64_t h = L.head;
        DL.recv_cnt.assign(G, 0);
        DL.out_cnt.assign(G, 0);
        sl[i].assign(G, {});
        il[i].assign(G, {});
        // halo of rank t = its body rows [max(h, qa), qb) merged with outside(i, t), ascending
        for (int t = 0; t < G; ++t) {
            int64_t qa, qb;
            range(i, t, qa, qb);
            const int64_t ha = std::max(h, qa);
            const std::vector<int32_t> ext = outside(i, t);
            size_t x = 0;
            auto visit = [&](int64_t q) {
                const int64_t P0 = pos0[L.perm[q]];
                const int home = owner(P0);
                RC[i][(size_t)t * G + home]++;
                if (t == me) DL.recv_cnt[home]++;
                if (home == me) sl[i][t].push_back((int32_t)(P0 - lo));
            };
            for (int64_t q = ha; q < qb; ++q) {
                for (; x < ext.size() && ext[x] < q; ++x) visit(ext[x]);
                visit(q);
                const int64_t P0 = pos0[L.perm[q]];
                const int home = owner(P0);
                if (L.row_ptr[q + 1] == L.row_ptr[q]) continue;
                OC[i][(size_t)t * G + home]++;
                if (t == me) DL.out_cnt[home]++;
                if (home == me) il[i][t].push_back((int32_t)(P0 - lo));
            }
            for (; x < ext.size(); ++x) visit(ext[x]);
        }
        DL.send_cnt.assign(G, 0);
        DL.in_cnt.assign(G, 0);
        for (int g = 0; g < G; ++g) {
            DL.send_cnt[g] = (int64_t)sl[i][g].size();
            DL.in_cnt[g] = (int64_t)il[i][g].size();
        }
    }
    // strict band, level 0: rank t's outside rows (H0 of t, ascending = grouped by home) are sent by
    // their homes before level 0 runs, next to D0
    std::vector<std::vector<int32_t>> ext0(G);
    if (nl > 0 && strict) {
        DistHostLevel &DL = H.L[0];
        DL.send_cnt.assign(G, 0);
        DL.recv_cnt.assign(G, 0);
        for (int t = 0; t < G; ++t) {
            ext0[t] = outside(0, t);
            H.h0_max = std::max<int64_t>(H.h0_max, (int64_t)ext0[t].size());
            for (int32_t q : ext0[t]) {
                const int home = owner(q);
                if (t == me) DL.recv_cnt[home]++;
                if (home == me) DL.send_cnt[t]++;
            }
        }
        H.h0_slot_q = ext0[me];
    }
    // ---- peer-major buffer layout: HB / OB = halo / staging offset of (home g, level i)
    std::vector<std::vector<int64_t>> HB(G, std::vector<int64_t>(nl, 0)), OB(G, std::vector<int64_t>(nl, 0));
    H.send_peer.assign(G, 0);
    H.recv_peer.assign(G, 0);
    H.out_peer.assign(G, 0);
    H.in_peer.assign(G, 0);
    int64_t hb = 0, ob = 0;
    for (int g = 0; g < G; ++g) {
        if (g == me) { H.halo_self_off = hb; H.out_self_off = ob; }
        for (int i = 1; i < nl; ++i) {
            const DistHostLevel &DL = H.L[i];
            HB[g][i] = hb;
            OB[g][i] = ob;
            hb += DL.recv_cnt[g];
            ob += DL.out_cnt[g];
            H.send_peer[g] += DL.send_cnt[g];
            H.recv_peer[g] += DL.recv_cnt[g];
            H.out_peer[g] += DL.out_cnt[g];
            H.in_peer[g] += DL.in_cnt[g];
            auto &s = (g == me) ? H.send_idx_self : H.send_idx_peers;
            s.insert(s.end(), sl[i][g].begin(), sl[i][g].end());
            auto &r = (g == me) ? H.in_rows_self : H.in_rows_peers;
            r.insert(r.end(), il[i][g].begin(), il[i][g].end());
        }
    }
    H.halo_rows = hb;
    H.out_rows = ob;
    // P2P layout of every rank: HBt[t][h][i] = halo offset (home-major), SBt[t][s][i] = staging
    // offset (source-major) inside rank t's buffers
    H.p2p = p2p;
    for (int i = 0; i < nl; ++i) H.d0_rows += D.levels[i].head;
    H.d0_index.assign(nl, {});
    H.blk0.assign(G + 1, 0);
    H.blk1.assign(G + 1, 0);
    {
        int64_t off = 0;
        if (p2p) {
            for (int i = 0; i < nl; ++i) {
                H.d0_index[i].resize(D.levels[i].head);
                for (int64_t j = 0; j < D.levels[i].head; ++j) H.d0_index[i][j] = (int32_t)(off + j);
                off += D.levels[i].head;
            }
        } else {
            // two blocks (level 0 | levels >= 1), each owner-major; heads keep level, then j order
            for (int blk = 0; blk < 2; ++blk) {
                std::vector<int64_t> &bnd = blk == 0 ? H.blk0 : H.blk1;
                const int i0 = blk == 0 ? 0 : 1, i1 = blk == 0 ? std::min(nl, 1) : nl;
                const int64_t base = off;
                for (int r = 0; r < G; ++r) {
                    bnd[r] = off - base;
                    for (int i = i0; i < i1; ++i) {
                        const HostLevel &L = D.levels[i];
                        H.d0_index[i].resize(L.head, -1);
                        for (int64_t j = 0; j < L.head; ++j)
                            if (owner(pos0[L.perm[j]]) == r) H.d0_index[i][j] = (int32_t)(off++);
                    }
                }
                bnd[G] = off - base;
            }
        }
    }
    std::vector<std::vector<std::vector<int64_t>>> HBt, SBt;
    if (p2p) {
        HBt.assign(G, std::vector<std::vector<int64_t>>(G, std::vector<int64_t>(nl, 0)));
        SBt = HBt;
        H.halo_all.assign(G, 0);
        H.stage_all.assign(G, 0);
        for (int t = 0; t < G; ++t)
            for (int g = 0; g < G; ++g)
                for (int i = 1; i < nl; ++i) {
                    HBt[t][g][i] = H.halo_all[t];
                    H.halo_all[t] += RC[i][(size_t)t * G + g];
                    SBt[t][g][i] = H.stage_all[t];
                    if (g != t) H.stage_all[t] += OC[i][(size_t)g * G + t];  // own rows: RMW into Y
                }
        const int64_t o_halo = 3 * H.d0_rows + H.h0_max;
        for (int t = 0; t < G; ++t) {
            if (o_halo + H.halo_all[t] + H.stage_all[t] > (int64_t)kPeerRowMask)
                return set_error(ARROW_E_UNSUPPORTED, "P2P workspace exceeds 2^27 rows");
        }
        const int64_t o_stage = o_halo + H.halo_all[me];
        // DMA variant: pack every peer's rows contiguously ([D0 | C0 x 2 | halo | stage | send]),
        // the rows of my own tiles straight into my halo; the copy engines move the chunks
        const int64_t o_send = o_stage + H.stage_all[me];
        H.send_row.assign(G, 0);
        H.halo_dst_row.assign(G, 0);
        for (int t = 0; t < G; ++t) {
            H.send_row[t] = o_send + H.send_rows;
            H.halo_dst_row[t] = o_halo + (nl > 1 ? HBt[t][me][1] : 0);
            int64_t m2 = 0;
            for (int i = 1; i < nl; ++i)
                for (size_t m = 0; m < sl[i][t].size(); ++m, ++m2) {
                    H.pack_src.push_back(sl[i][t][m]);
                    H.pack_dst.push_back((int32_t)(t == me ? o_halo + HBt[me][me][i] + (int64_t)m : o_send + H.send_rows + m2));
                }
            if (t != me) H.send_rows += m2;
        }
        if (o_send + H.send_rows > (int64_t)kPeerRowMask) return set_error(ARROW_E_UNSUPPORTED, "P2P workspace exceeds 2^27 rows");
        if (hi - lo > (int64_t)kPeerRowMask) return set_error(ARROW_E_UNSUPPORTED, "P2P transport: more than 2^27 rows per rank");
        for (int s = 0; s < G; ++s)
            for (int i = 1; s != me && i < nl; ++i)
                for (size_t m = 0; m < il[i][s].size(); ++m)
                    H.post.emplace_back(il[i][s][m], (int32_t)(((uint32_t)me << kPeerShift) | (uint32_t)(o_stage + SBt[me][s][i] + (int64_t)m)));
    }

    // strict band, level 0: H0 offset; my rows for every peer's H0 (P2P: pushed with D0; NCCL: packed
    // peer-major and sent before level 0)
    H.o_h0 = (p2p ? 3 : 2) * H.d0_rows;
    if (strict)
        for (int t = 0; t < G; ++t) {
            if (t == me) continue;
            for (size_t m = 0; m < ext0[t].size(); ++m) {
                const int32_t q = ext0[t][m];
                if (owner(q) != me) continue;
                if (p2p) {
                    H.d0push_src.push_back((int32_t)(q - lo));
                    H.d0push_dst.push_back((int32_t)(((uint32_t)t << kPeerShift) | (uint32_t)(H.o_h0 + (int64_t)m)));
                } else {
                    H.send0_idx.push_back((int32_t)(q - lo));
                }
            }
        }

    // ---- pass 2: heads, zero rows and descriptor layout of my tiles, per level
    for (int i = 0; i < nl; ++i) {
        const HostLevel &L = D.levels[i];
        DistHostLevel &DL = H.L[i];
        const int64_t h = L.head;
        int64_t qa, qb;
        range(i, me, qa, qb);
        const int64_t ha = std::max(h, qa);
        std::vector<int32_t> halo_slot, out_slot, ext, ext_slot;
        if (i > 0) {
            std::vector<int64_t> hcur(G), ocur(G);
            for (int g = 0; g < G; ++g) {
                hcur[g] = HB[g][i];
                // P2P: staging rows are stored straight into the home rank's buffer
                ocur[g] = p2p ? 3 * H.d0_rows + H.h0_max + H.halo_all[g] + SBt[g][me][i] : OB[g][i];
            }
            halo_slot.resize(std::max<int64_t>(0, qb - ha));
            out_slot.assign(std::max<int64_t>(0, qb - ha), -1);
            // halo slots in the order of pass 1 (body rows merged with the outside rows, ascending)
            ext = outside(i, me);
            ext_slot.resize(ext.size());
            size_t x = 0;
            auto slot_of = [&](int64_t q) { return (int32_t)(hcur[owner(pos0[L.perm[q]])]++); };
            for (int64_t q = ha; q < qb; ++q) {
                for (; x < ext.size() && ext[x] < q; ++x) ext_slot[x] = slot_of(ext[x]);
                halo_slot[q - ha] = slot_of(q);
            }
            for (; x < ext.size(); ++x) ext_slot[x] = slot_of(ext[x]);
            for (int64_t q = ha; q < qb; ++q) {
                if (L.row_ptr[q + 1] == L.row_ptr[q]) continue;
                const int home = owner(pos0[L.perm[q]]);
                if (p2p && home == me)  // P2P: my own rows are read-modify-written into Y directly
                    out_slot[q - ha] = (int32_t)(kLocalRmwBit | (uint32_t)(pos0[L.perm[q]] - lo));
                else
                    out_slot[q - ha] = (int32_t)((p2p ? ((uint32_t)home << kPeerShift) : 0u) | (uint32_t)(ocur[home]++));
            }
        } else {
            ext = H.h0_slot_q;
            ext_slot.resize(ext.size());
            for (size_t m = 0; m < ext.size(); ++m) ext_slot[m] = (int32_t)(kFlag | (uint32_t)(H.o_h0 + (int64_t)m));
        }
        for (int64_t j = 0; j < h; ++j) {
            const int64_t P0 = pos0[L.perm[j]];
            if (owner(P0) != me) continue;
            DL.head_j.push_back((int32_t)j);
            DL.head_row.push_back((int32_t)(P0 - lo));
            if (p2p)
                for (int t = 0; t < G; ++t) {
                    H.d0push_src.push_back((int32_t)(P0 - lo));
                    H.d0push_dst.push_back((int32_t)(((uint32_t)t << kPeerShift) | (uint32_t)H.d0_index[i][j]));
                    H.post.emplace_back((int32_t)(P0 - lo), (int32_t)(((uint32_t)t << kPeerShift) | kParityBit |
                                                                       (uint32_t)(H.d0_rows + H.d0_index[i][j])));
                }
        }
        if (i == 0) {  // level 0: entry-less body rows of my home range; the A-isolated tail is a range
            for (int64_t p = std::max(lo, h); p < std::min(hi, L.n_i); ++p)
                if (L.row_ptr[p + 1] == L.row_ptr[p]) DL.zero_rows.push_back((int32_t)(p - lo));
            H.zero_tail_lo = std::max(lo, L.n_i) - lo;
            H.zero_tail_n = std::max<int64_t>(0, hi - std::max(lo, L.n_i));
        }
        auto colmap = [&](int32_t q) -> int32_t {
            if (q < h) return (int32_t)(kFlag | (uint32_t)H.d0_index[i][q]);
            if (q < qa || q >= qb) return ext_slot[std::lower_bound(ext.begin(), ext.end(), q) - ext.begin()];
            return (i == 0) ? (int32_t)(q - lo) : halo_slot[q - ha];
        };
        auto push_val = [&](double v) {
            const size_t at = DL.segs.ent_val.size();
            DL.segs.ent_val.resize(at + es);
            if (es == 8) std::memcpy(DL.segs.ent_val.data() + at, &v, 8);
            else { const float f = (float)v; std::memcpy(DL.segs.ent_val.data() + at, &f, 4); }
        };
        const int64_t W = std::max<int64_t>(1, (i == 0 ? window_rows0 : window_rows) / b) * b;
        for (int64_t lo_w = qa; lo_w < qb; lo_w += W) {
            const int64_t hi_w = std::min(qb, lo_w + W);
            for (int64_t p = std::max(h, lo_w); p < hi_w; ++p) {
                if (L.row_ptr[p + 1] == L.row_ptr[p]) continue;
                for (int64_t e = L.row_ptr[p]; e < L.row_ptr[p + 1]; ++e) { DL.segs.ent_col.push_back(colmap(L.col[e])); push_val(L.val[e]); }
                DL.segs.seg_out.push_back(i == 0 ? (int32_t)(p - lo) : out_slot[p - ha]);
                DL.segs.seg_end.push_back((uint32_t)DL.segs.ent_col.size());
            }
            for (int64_t j = 0; j < h; ++j) {
                const int32_t *a = L.col.data() + L.row_ptr[j], *z = L.col.data() + L.row_ptr[j + 1];
                int64_t x0 = L.row_ptr[j] + (std::lower_bound(a, z, (int32_t)lo_w) - a);
                const int64_t x1 = L.row_ptr[j] + (std::lower_bound(a, z, (int32_t)hi_w) - a);
                while (x0 < x1) {
                    const int64_t x2 = std::min<int64_t>(x1, x0 + head_chunk);
                    for (int64_t e = x0; e < x2; ++e) { DL.segs.ent_col.push_back(colmap(L.col[e])); push_val(L.val[e]); }
                    DL.segs.seg_out.push_back((int32_t)(kFlag | (uint32_t)H.d0_index[i][j]));
                    DL.segs.seg_end.push_back((uint32_t)DL.segs.ent_col.size());
                    x0 = x2;
                }
            }
        }
    }
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

namespace {

// all ranks: every rank's mapping of `local` (a cudaMalloc base) via CUDA IPC; `ok` = this rank
// could open every peer's handle (callers agree collectively before using the mappings)
arrow_status share_ptr(DistState *S, void *local, PeerPtrs &out, bool &ok) {
    out = PeerPtrs{};
    ok = true;
    cudaIpcMemHandle_t mine;
    std::memset(&mine, 0, sizeof(mine));
    if (cudaIpcGetMemHandle(&mine, local) != cudaSuccess) {
        cudaGetLastError();
        ok = false;
    }
    const size_t hs = sizeof(cudaIpcMemHandle_t);
    char *dbuf = nullptr;
    DCUDA(cudaMalloc(&dbuf, hs * S->G));
    DCUDA(cudaMemcpy(dbuf + hs * S->me, &mine, hs, cudaMemcpyHostToDevice));
    DNCCL(ncclAllGather(dbuf + hs * S->me, dbuf, hs, ncclUint8, S->comm, S->cs));
    DCUDA(cudaStreamSynchronize(S->cs));
    std::vector<cudaIpcMemHandle_t> all(S->G);
    DCUDA(cudaMemcpy(all.data(), dbuf, hs * S->G, cudaMemcpyDeviceToHost));
    cudaFree(dbuf);
    for (int g = 0; g < S->G; ++g) {
        if (g == S->me) { out.p[g] = local; continue; }
        if (!ok) continue;
        if (cudaIpcOpenMemHandle(&out.p[g], all[g], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            out.p[g] = nullptr;
            ok = false;
        }
    }
    return ARROW_OK;
}

// all ranks: logical AND of `v` over the ranks
arrow_status all_true(DistState *S, bool &v) {
    int *d = nullptr;
    DCUDA(cudaMalloc(&d, sizeof(int)));
    const int h = v ? 1 : 0;
    DCUDA(cudaMemcpy(d, &h, sizeof(int), cudaMemcpyHostToDevice));
    DNCCL(ncclAllReduce(d, d, 1, ncclInt32, ncclMin, S->comm, S->cs));
    DCUDA(cudaStreamSynchronize(S->cs));
    int r = 0;
    DCUDA(cudaMemcpy(&r, d, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(d);
    v = r != 0;
    return ARROW_OK;
}

}  // namespace

// Collective for P2P plans: every rank's last gather-add still reads its peers' workspaces over
// NVLink, so no rank unmaps or frees its workspace before all ranks have drained their streams
// (one NCCL all-reduce after a device synchronise).  arrow_plan_destroy is therefore collective for
// distributed plans (include/arrow.h).
void dist_free(DistState *d) {
    if (!d) return;
    if (d->ready && d->p2p && d->comm) {
        cudaDeviceSynchronize();
        bool dummy = true;
        all_true(d, dummy);
    }
    if (d->cs) cudaStreamSynchronize(d->cs);
    close_peers(d, d->ws_peer);
    close_peers(d, d->flags_peer);
    for (void *p : d->allocs) cudaFree(p);
    if (d->ws) cudaFree(d->ws);
    for (auto e : d->ev)
        if (e) cudaEventDestroy(e);
    for (auto e : d->ds_ev) cudaEventDestroy(e);
    for (auto s : d->ds) cudaStreamDestroy(s);
    if (d->cs) cudaStreamDestroy(d->cs);
    delete d;
}


arrow_status dist_build(arrow_plan P, const arrow_decomposition_s &D, arrow_comm comm, int64_t window_rows,
                        int64_t window_rows0, int32_t head_chunk, int bs) {
    auto *S = new DistState();
    P->dist = S;
    S->comm = (ncclComm_t)comm->comm;
    S->G = comm->nranks;
    S->me = comm->rank;
    if (cudaStreamCreateWithFlags(&S->cs, cudaStreamNonBlocking) != cudaSuccess)
        return set_error(ARROW_E_CUDA, "cudaStreamCreate(comm stream)");
    for (auto &e : S->ev)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
            return set_error(ARROW_E_CUDA, "cudaEventCreate");
    // transport: P2P (peer memory over NVLink, fused with the kernels) unless options.transport is
    // NCCL, a single rank, or some rank cannot map its peers' memory (decided collectively)
    bool p2p = S->G > 1 && S->G <= kMaxPeers && P->transport != ARROW_TRANSPORT_NCCL;
    if (p2p) {
        DCUDA(cudaMalloc(&S->flags, 3 * kMaxPeers * sizeof(unsigned)));
        DCUDA(cudaMemset(S->flags, 0, 3 * kMaxPeers * sizeof(unsigned)));
        DCUDA(cudaDeviceSynchronize());
        bool ok = true;
        arrow_status st = share_ptr(S, S->flags, S->flags_peer, ok);
        if (st != ARROW_OK) return st;
        st = all_true(S, ok);
        if (st != ARROW_OK) return st;
        if (!ok) {
            close_peers(S, S->flags_peer);
            if (P->transport == ARROW_TRANSPORT_P2P)
                return set_error(ARROW_E_UNSUPPORTED, "P2P transport requested but a peer's memory cannot be mapped");
            p2p = false;
        }
        if (std::getenv("ARROW_DIST_TRACE"))
            fprintf(stderr, "[arrow dist rank %d] transport %s\n", S->me, p2p ? "p2p" : "nccl (peer mapping failed)");
    }
    S->p2p = p2p ? 1 : 0;
    if (S->flags) S->allocs.push_back(S->flags);

    DistHost H;
    arrow_status st = dist_schedule(D, S->G, S->me, window_rows, window_rows0, head_chunk, P->esize(), S->p2p, H);
    if (st != ARROW_OK) return st;
    S->lo = H.lo;
    S->hi = H.hi;
    S->nl = (int)H.L.size();
    const int nl = S->nl, G = S->G, me = S->me;
    for (int i = 0; i < nl; ++i) {
        S->h.push_back(H.L[i].h);
        S->d0_off.push_back(S->d0_rows);
        S->d0_rows += H.L[i].h;
    }
    S->blk0 = H.blk0;
    S->blk1 = H.blk1;
    S->send_peer = H.send_peer;
    S->recv_peer = H.recv_peer;
    S->out_peer = H.out_peer;
    S->in_peer = H.in_peer;
    for (int g = 0; g < G; ++g)
        if (g != me) { S->fwd_rows += H.recv_peer[g]; S->rev_rows += H.out_peer[g]; }
    std::vector<int32_t> zero = H.L.empty() ? std::vector<int32_t>() : H.L[0].zero_rows;
    // level-0 heads owned here: Y starts at zero, every level adds its head partial afterwards
    if (nl > 0) zero.insert(zero.end(), H.L[0].head_row.begin(), H.L[0].head_row.end());
    std::vector<int32_t> pre_src, pre_dst, sp, ss, sd, pp, ps, pd;
    if (S->p2p) {
        S->o_d0 = 0;
        S->o_c0 = S->d0_rows;
        S->o_h0 = H.o_h0;
        S->o_halo = 3 * S->d0_rows + H.h0_max;
        S->o_out = S->o_halo + H.halo_all[me];
        S->ws_rows = S->o_out + H.stage_all[me] + H.send_rows;
        S->send_row = H.send_row;
        S->halo_dst_row = H.halo_dst_row;
        for (int g = 0; g < G; ++g) {
            if (g == me) continue;
            cudaStream_t q;
            cudaEvent_t e;
            if (cudaStreamCreateWithFlags(&q, cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
                return set_error(ARROW_E_CUDA, "cudaStreamCreate/cudaEventCreate (copy streams)");
            S->ds.push_back(q);
            S->ds_ev.push_back(e);
        }
        build_csr(H.post, pp, ps, pd);
    } else {
        // workspace rows: [D0 | C0 | H0 | halo | send | S0 | staging | recv]
        const int64_t n_send = (int64_t)H.send_idx_peers.size(), n_in = (int64_t)H.in_rows_peers.size();
        const int64_t n_s0 = (int64_t)H.send0_idx.size();
        S->o_d0 = 0;
        S->o_c0 = S->d0_rows;
        S->o_h0 = H.o_h0;
        S->o_halo = 2 * S->d0_rows + H.h0_max;
        S->o_send = S->o_halo + H.halo_rows;
        S->o_s0 = S->o_send + n_send;
        S->o_out = S->o_s0 + n_s0;
        if (nl > 0 && !H.L[0].send_cnt.empty()) {
            S->send0_peer = H.L[0].send_cnt;
            S->recv0_peer = H.L[0].recv_cnt;
        }
        S->o_in = S->o_out + H.out_rows;
        S->ws_rows = S->o_in + n_in;
        if (S->ws_rows >= ((int64_t)1 << 31))
            return set_error(ARROW_E_UNSUPPORTED, "distributed workspace exceeds 2^31 rows");
        // pre-exchange row mover: D0 (owned heads from X, the rest zero), C0 = 0, pack for peers and self
        for (int i = 0; i < nl; ++i)
            for (size_t m = 0; m < H.L[i].head_j.size(); ++m) {
                pre_src.push_back(H.L[i].head_row[m]);
                pre_dst.push_back((int32_t)(S->o_d0 + H.d0_index[i][H.L[i].head_j[m]]));
            }
        for (int64_t r = 0; r < S->d0_rows; ++r) { pre_src.push_back(-1); pre_dst.push_back((int32_t)(S->o_c0 + r)); }
        for (int64_t m = 0; m < n_send; ++m) { pre_src.push_back(H.send_idx_peers[m]); pre_dst.push_back((int32_t)(S->o_send + m)); }
        for (int64_t m = 0; m < n_s0; ++m) { pre_src.push_back(H.send0_idx[m]); pre_dst.push_back((int32_t)(S->o_s0 + m)); }
        for (size_t m = 0; m < H.send_idx_self.size(); ++m) {
            pre_src.push_back(H.send_idx_self[m]);
            pre_dst.push_back((int32_t)(S->o_halo + H.halo_self_off + (int64_t)m));
        }
        // gather-adds: own staging rows (before the reverse exchange completes), then received rows
        // and the head partials of every level (after)
        std::vector<std::pair<int32_t, int32_t>> cself, cpost;
        for (size_t m = 0; m < H.in_rows_self.size(); ++m)
            cself.emplace_back(H.in_rows_self[m], (int32_t)(S->o_out + H.out_self_off + (int64_t)m));
        for (int64_t m = 0; m < n_in; ++m) cpost.emplace_back(H.in_rows_peers[m], (int32_t)(S->o_in + m));
        for (int i = 0; i < nl; ++i)
            for (size_t m = 0; m < H.L[i].head_j.size(); ++m)
                cpost.emplace_back(H.L[i].head_row[m], (int32_t)(S->o_c0 + H.d0_index[i][H.L[i].head_j[m]]));
        build_csr(cself, sp, ss, sd);
        build_csr(cpost, pp, ps, pd);
    }

    bool ok = true;
    for (int i = 0; i < nl; ++i) {
        // every output row is written once (mode 0): local Y (level 0) or a staging buffer
        SegLevel sg;
        std::string err;
        // level 0 reads the local X rows (and D0), levels >= 1 the halo inside the workspace
        const int64_t xr = (i == 0) ? std::max<int64_t>(S->hi - S->lo, S->o_halo) : S->ws_rows;
        const int e = upload_seg_level(H.L[i].segs, (int)P->esize(), bs, 0, xr, S->allocs, sg, err);
        if (e) return set_error(e == -1 ? ARROW_E_UNSUPPORTED : ARROW_E_CUDA, err);
        H.L[i].segs = HostSegs();
        S->seg.push_back(sg);
    }
    S->n_pre = (int64_t)pre_src.size();
    S->pre_src = upload(S, pre_src, ok);
    S->pre_dst = upload(S, pre_dst, ok);
    S->n_d0push = (int64_t)H.d0push_src.size();
    S->d0push_src = upload(S, H.d0push_src, ok);
    S->d0push_dst = upload(S, H.d0push_dst, ok);
    S->n_pack = (int64_t)H.pack_src.size();
    S->pack_src = upload(S, H.pack_src, ok);
    S->pack_dst = upload(S, H.pack_dst, ok);
    S->n_zero = (int64_t)zero.size();
    S->zero_rows = upload(S, zero, ok);
    S->zero_tail_lo = H.zero_tail_lo;
    S->zero_tail_n = H.zero_tail_n;
    S->n_self = (int64_t)sd.size();
    S->self_ptr = upload(S, sp, ok);
    S->self_src = upload(S, ss, ok);
    S->self_dst = upload(S, sd, ok);
    S->n_post = (int64_t)pd.size();
    S->post_ptr = upload(S, pp, ok);
    S->post_src = upload(S, ps, ok);
    S->post_dst = upload(S, pd, ok);
    if (!ok) return set_error(ARROW_E_CUDA, "cudaMalloc/cudaMemcpy of the distributed layout failed");
    if (cudaMalloc(&S->counters, (nl + 1) * sizeof(unsigned)) != cudaSuccess)
        return set_error(ARROW_E_CUDA, "cudaMalloc(counters)");
    S->allocs.push_back(S->counters);
    P->local_begin = S->lo;
    P->local_end = S->hi;
    S->ready = true;
    return ARROW_OK;
}

namespace {

// (re)allocate the k-dependent workspace; P2P: collectively, then map every peer's workspace
arrow_status ensure_ws(arrow_plan P, DistState *S, int64_t k, cudaStream_t st) {
    if (k <= S->ws_k) return ARROW_OK;
    const size_t es = P->esize();
    DCUDA(cudaStreamSynchronize(st));
    DCUDA(cudaStreamSynchronize(S->cs));
    if (S->p2p) {
        close_peers(S, S->ws_peer);
        bool dummy = true;  // every rank has unmapped the old workspaces before any is freed
        arrow_status s = all_true(S, dummy);
        if (s != ARROW_OK) return s;
    }
    if (S->ws) cudaFree(S->ws);
    S->ws = nullptr;
    S->ws_k = 0;
    DCUDA(cudaMalloc(&S->ws, (size_t)std::max<int64_t>(S->ws_rows, 1) * k * es));
    S->ws_k = k;
    if (S->p2p) {
        bool ok = true;
        arrow_status s = share_ptr(S, S->ws, S->ws_peer, ok);
        if (s != ARROW_OK) return s;
        s = all_true(S, ok);
        if (s != ARROW_OK) return s;
        if (!ok) return set_error(ARROW_E_CUDA, "mapping a peer's workspace (CUDA IPC) failed");
    }
    return ARROW_OK;
}

struct Marks {
    bool on = false;
    std::vector<cudaEvent_t> ev;
    int operator()(cudaStream_t s) {
        if (!on) return -1;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        ev.push_back(e);
        return (int)ev.size() - 1;
    }
    std::string el(int a, int b) const {
        float ms = 0;
        cudaEventElapsedTime(&ms, ev[a], ev[b]);
        return std::to_string(ms);
    }
};

// hand interval [a, b] to the profiling counters (the record owns both events)
void prof_rec(arrow_plan P, Marks &M, int kid, int a, int b) {
    P->prof.push_back(ProfRec{kid, P->prof_pos++, M.ev[a], M.ev[b]});
    M.ev[a] = M.ev[b] = nullptr;
}
void marks_done(Marks &M) {
    for (auto e : M.ev)
        if (e) cudaEventDestroy(e);
}

// P2P transport: pushes and staging stores go straight into the peers' memory over NVLink;
// three cross-GPU flag barriers order them (slot 0: every D0 complete; slot 1: every halo complete;
// slot 2: every staging row and head partial complete).
arrow_status dist_spmm_p2p(arrow_plan P, DistState *S, const void *X, void *Y, int64_t k, cudaStream_t st) {
    const int dt = P->dtype == ARROW_F64 ? 1 : 0;
    const size_t es = P->esize();
    const int G = S->G, me = S->me, nl = S->nl;
    char *ws = reinterpret_cast<char *>(S->ws);
    auto row = [&](int64_t r) { return ws + (size_t)r * k * es; };
    const int par = (int)(S->calls & 1);
    S->calls++;
    const int64_t c0 = S->o_c0 + par * S->d0_rows;  // this call's C0
    const int sms = P->num_sms;
    static const bool trace = std::getenv("ARROW_DIST_TRACE") != nullptr;
    Marks M;
    M.on = P->profiling || trace;

    // S: the previous call (and the caller's writes of X) precede everything.  My head rows go into
    // every rank's D0 first (level 0 needs only them), then C0 = 0 and the zero rows; the rows for
    // the peers are packed, and C moves one chunk per peer with the copy engines while the SMs run
    // level 0.
    const int m0 = M(st);
    DK(launch_push_rows(dt, X, S->d0push_src, S->d0push_dst, S->n_d0push, k, S->ws_peer, 0, st));
    DCUDA(cudaMemsetAsync(S->counters, 0, (nl + 1) * sizeof(unsigned), st));
    DCUDA(cudaMemsetAsync(row(c0), 0, (size_t)S->d0_rows * k * es, st));
    DK(launch_zero_rows(dt, S->zero_rows, S->n_zero, k, Y, st));
    DK(launch_rows(dt, X, S->pack_src, S->pack_dst, S->n_pack, k, 0, ws, st));
    const int m0p = M(st);
    DCUDA(cudaEventRecord(S->ev[0], st));
    DCUDA(cudaStreamWaitEvent(S->cs, S->ev[0], 0));
    const int m0c = M(S->cs);
    {
        DCUDA(cudaEventRecord(S->ev[5], S->cs));
        for (int g = 0, q = 0; g < G; ++g) {
            if (g == me) continue;
            cudaStream_t d = S->ds[q];
            DCUDA(cudaStreamWaitEvent(d, S->ev[5], 0));
            if (S->send_peer[g])
                DCUDA(cudaMemcpyAsync(reinterpret_cast<char *>(S->ws_peer.p[g]) + (size_t)S->halo_dst_row[g] * k * es,
                                      row(S->send_row[g]), (size_t)S->send_peer[g] * k * es, cudaMemcpyDeviceToDevice,
                                      d));
            DCUDA(cudaEventRecord(S->ds_ev[q], d));
            DCUDA(cudaStreamWaitEvent(S->cs, S->ds_ev[q], 0));
            ++q;
        }
    }
    const int m1c = M(S->cs);
    DK(launch_barrier(S->flags_peer, S->flags, 1, ++S->epoch[1], me, G, S->cs));
    const int m2c = M(S->cs);
    DCUDA(cudaEventRecord(S->ev[1], S->cs));
    // S: every D0 complete -> level 0
    DK(launch_barrier(S->flags_peer, S->flags, 0, ++S->epoch[0], me, G, st));
    const int m1 = M(st), m1b = M(st);
    DK(launch_seg(dt, 1, S->seg[0], X, row(S->o_d0), Y, row(c0), k, sms, S->counters, st, P->launch));
    const int m2 = M(st);
    // levels >= 1 once every halo is complete; body rows are stored into their home rank's stage
    DCUDA(cudaStreamWaitEvent(st, S->ev[1], 0));
    const int m3 = M(st);
    for (int i = 1; i < nl; ++i)
        DK(launch_seg(dt, 2, S->seg[i], row(S->o_halo), row(S->o_d0), Y, row(c0),
                      k, sms, S->counters + i, st, P->launch, &S->ws_peer));
    const int m4 = M(st), m4b = M(st);
    // the A-isolated tail of Y (no level writes it) is zeroed while the other ranks finish
    if (S->zero_tail_n)
        DCUDA(cudaMemsetAsync(reinterpret_cast<char *>(Y) + (size_t)S->zero_tail_lo * k * es, 0,
                              (size_t)S->zero_tail_n * k * es, st));
    DK(launch_barrier(S->flags_peer, S->flags, 2, ++S->epoch[2], me, G, st));
    const int m5 = M(st);
    DK(launch_gather_add_peers(dt, S->ws_peer, S->d0_rows * par, S->post_ptr, S->post_src, S->post_dst, S->n_post, k,
                               Y, st));
    const int m6 = M(st);
    if (trace) {
        cudaEventSynchronize(M.ev[m6]);
        std::string line = "[arrow dist rank " + std::to_string(me) + " p2p] ms: halo " +
                           std::string("D0+zero+pack " + M.el(m0, m0p) + " dma ") + M.el(m0c, m1c) +
                           " + barrier " + M.el(m1c, m2c) + " (done at " + M.el(m0, m2c) + ") | barrier0 " +
                           M.el(m0p, m1) + " | K-A L0 " + M.el(m1, m2) + " | wait " + M.el(m2, m3) + " | K-A L>=1 " +
                           M.el(m3, m4) + " | barrier " + M.el(m4, m5) + " | gather-add " + M.el(m5, m6) +
                           " | total " + M.el(m0, m6) + " | rows fwd " + std::to_string(S->fwd_rows) + " rev " +
                           std::to_string(S->rev_rows) + " d0 " + std::to_string(S->d0_rows);
        fprintf(stderr, "%s\n", line.c_str());
    }
    if (P->profiling) {
        prof_rec(P, M, ARROW_K_COMM, m0c, m2c);
        prof_rec(P, M, ARROW_K_COMM, m0, m1);
        prof_rec(P, M, ARROW_K_SEGMENTS, m1b, m2);
        prof_rec(P, M, ARROW_K_SEGMENTS, m3, m4);
        prof_rec(P, M, ARROW_K_COMM, m4b, m6);
        P->prof_acc.calls += 1;
    }
    marks_done(M);
    return ARROW_OK;
}

}  // namespace

arrow_status dist_spmm(arrow_plan P, const void *X, void *Y, int64_t k, cudaStream_t st) {
    DistState *S = P->dist;
    const int dt = P->dtype == ARROW_F64 ? 1 : 0;
    const size_t es = P->esize();
    const ncclDataType_t nt = dt ? ncclDouble : ncclFloat;
    const int G = S->G, me = S->me, nl = S->nl;
    if (nl == 0) {
        if (S->hi > S->lo) DCUDA(cudaMemsetAsync(Y, 0, (size_t)(S->hi - S->lo) * k * es, st));
        return ARROW_OK;
    }
    arrow_status wst = ensure_ws(P, S, k, st);
    if (wst != ARROW_OK) return wst;
    if (S->p2p) return dist_spmm_p2p(P, S, X, Y, k, st);
    char *ws = reinterpret_cast<char *>(S->ws);
    auto row = [&](int64_t r) { return ws + (size_t)r * k * es; };
    const int sms = std::max(1, P->num_sms - (G > 1 ? S->reserve_sms : 0));
    static const bool trace = std::getenv("ARROW_DIST_TRACE") != nullptr;
    Marks M;
    M.on = P->profiling || trace;

    // 1. (S) D0 / C0 / packing, zero rows
    const int m0 = M(st);
    DCUDA(cudaMemsetAsync(S->counters, 0, (nl + 1) * sizeof(unsigned), st));
    DK(launch_rows(dt, X, S->pre_src, S->pre_dst, S->n_pre, k, 0, ws, st));
    DK(launch_zero_rows(dt, S->zero_rows, S->n_zero, k, Y, st));
    if (S->zero_tail_n)
        DCUDA(cudaMemsetAsync(reinterpret_cast<char *>(Y) + (size_t)S->zero_tail_lo * k * es, 0,
                              (size_t)S->zero_tail_n * k * es, st));
    const int m1 = M(st);
    DCUDA(cudaEventRecord(S->ev[0], st));
    // 2. (C) D0 of level 0; forward rows + D0 of the other levels
    DCUDA(cudaStreamWaitEvent(S->cs, S->ev[0], 0));
    const int m2 = M(S->cs);
    // Alg. 1 line 1, Broadcast(D^(0)): every owner broadcasts its head rows of level 0 (owner-major block)
    DNCCL(ncclGroupStart());
    for (int r = 0; r < G; ++r)
        if (S->blk0[r + 1] > S->blk0[r])
            DNCCL(ncclBroadcast(row(S->o_d0 + S->blk0[r]), row(S->o_d0 + S->blk0[r]), (S->blk0[r + 1] - S->blk0[r]) * k,
                                nt, r, S->comm, S->cs));
    DNCCL(ncclGroupEnd());
    if (!S->send0_peer.empty()) {  // strict band: level 0's outside rows from their homes (H0)
        DNCCL(ncclGroupStart());
        int64_t s0 = 0, r0 = 0;
        for (int g = 0; g < G; ++g) {
            if (g != me && S->send0_peer[g])
                DNCCL(ncclSend(row(S->o_s0 + s0), S->send0_peer[g] * k, nt, g, S->comm, S->cs));
            if (g != me && S->recv0_peer[g])
                DNCCL(ncclRecv(row(S->o_h0 + r0), S->recv0_peer[g] * k, nt, g, S->comm, S->cs));
            s0 += S->send0_peer[g];
            r0 += S->recv0_peer[g];
        }
        DNCCL(ncclGroupEnd());
    }
    DCUDA(cudaEventRecord(S->ev[1], S->cs));
    DNCCL(ncclGroupStart());
    int64_t so = 0, ro = 0;
    for (int g = 0; g < G; ++g) {
        if (g == me) { ro += S->recv_peer[g]; continue; }
        if (S->send_peer[g]) DNCCL(ncclSend(row(S->o_send + so), S->send_peer[g] * k, nt, g, S->comm, S->cs));
        if (S->recv_peer[g]) DNCCL(ncclRecv(row(S->o_halo + ro), S->recv_peer[g] * k, nt, g, S->comm, S->cs));
        so += S->send_peer[g];
        ro += S->recv_peer[g];
    }
    for (int r = 0; r < G; ++r)  // the other levels' head blocks, by owner
        if (S->blk1[r + 1] > S->blk1[r])
            DNCCL(ncclBroadcast(row(S->o_d0 + S->blk0[G] + S->blk1[r]), row(S->o_d0 + S->blk0[G] + S->blk1[r]),
                                (S->blk1[r + 1] - S->blk1[r]) * k, nt, r, S->comm, S->cs));
    DNCCL(ncclGroupEnd());
    const int m3 = M(S->cs);
    DCUDA(cudaEventRecord(S->ev[2], S->cs));
    // 3. (S) level 0 overlaps the forward exchange; levels >= 1 after it
    DCUDA(cudaStreamWaitEvent(st, S->ev[1], 0));
    const int m4 = M(st);
    DK(launch_seg(dt, 1, S->seg[0], X, row(S->o_d0), Y, row(S->o_c0), k, sms, S->counters, st, P->launch));
    const int m5 = M(st);
    DCUDA(cudaStreamWaitEvent(st, S->ev[2], 0));
    const int m6 = M(st);
    for (int i = 1; i < nl; ++i)
        DK(launch_seg(dt, 1, S->seg[i], row(S->o_halo), row(S->o_d0), row(S->o_out), row(S->o_c0), k, sms,
                      S->counters + i, st, P->launch));
    const int m7 = M(st), m7b = M(st);
    DCUDA(cudaEventRecord(S->ev[3], st));
    // 4. (C) staging rows go home, head partials are reduced
    DCUDA(cudaStreamWaitEvent(S->cs, S->ev[3], 0));
    const int m8 = M(S->cs);
    DNCCL(ncclGroupStart());
    so = 0;
    ro = 0;
    for (int g = 0; g < G; ++g) {
        if (g == me) { so += S->out_peer[g]; continue; }
        if (S->out_peer[g]) DNCCL(ncclSend(row(S->o_out + so), S->out_peer[g] * k, nt, g, S->comm, S->cs));
        if (S->in_peer[g]) DNCCL(ncclRecv(row(S->o_in + ro), S->in_peer[g] * k, nt, g, S->comm, S->cs));
        so += S->out_peer[g];
        ro += S->in_peer[g];
    }
    // Alg. 1 line 3, Reduce(C^(0)): each head block's partials are reduced onto the rank that owns it
    for (int r = 0; r < G; ++r) {
        if (S->blk0[r + 1] > S->blk0[r])
            DNCCL(ncclReduce(row(S->o_c0 + S->blk0[r]), row(S->o_c0 + S->blk0[r]), (S->blk0[r + 1] - S->blk0[r]) * k, nt,
                             ncclSum, r, S->comm, S->cs));
        if (S->blk1[r + 1] > S->blk1[r])
            DNCCL(ncclReduce(row(S->o_c0 + S->blk0[G] + S->blk1[r]), row(S->o_c0 + S->blk0[G] + S->blk1[r]),
                             (S->blk1[r + 1] - S->blk1[r]) * k, nt, ncclSum, r, S->comm, S->cs));
    }
    DNCCL(ncclGroupEnd());
    const int m9 = M(S->cs);
    DCUDA(cudaEventRecord(S->ev[4], S->cs));
    // 5. (S) own staging rows (overlaps the exchange), then received rows and owned head partials
    DK(launch_gather_add(dt, ws, S->self_ptr, S->self_src, S->self_dst, S->n_self, k, Y, st));
    const int m10 = M(st);
    DCUDA(cudaStreamWaitEvent(st, S->ev[4], 0));
    const int m11 = M(st);
    DK(launch_gather_add(dt, ws, S->post_ptr, S->post_src, S->post_dst, S->n_post, k, Y, st));
    const int m12 = M(st);
    if (trace) {
        cudaEventSynchronize(M.ev[m12]);
        std::string line = "[arrow dist rank " + std::to_string(me) + " nccl] ms: pre " + M.el(m0, m1) + " | fwd " +
                           M.el(m2, m3) + " (ends at " + M.el(m0, m3) + ") | K-A L0 " + M.el(m4, m5) + " (starts at " +
                           M.el(m0, m4) + ") | wait " + M.el(m5, m6) + " | K-A L>=1 " + M.el(m6, m7) + " | rev " +
                           M.el(m8, m9) + " | self-add " + M.el(m7, m10) + " | wait " + M.el(m10, m11) +
                           " | post-add " + M.el(m11, m12) + " | total " + M.el(m0, m12) + " | rows fwd " +
                           std::to_string(S->fwd_rows) + " rev " + std::to_string(S->rev_rows) + " d0 " +
                           std::to_string(S->d0_rows);
        fprintf(stderr, "%s\n", line.c_str());
    }
    if (P->profiling) {
        // compute: both K-A phases; communication: pre-exchange work, the two exchanges, the adds
        prof_rec(P, M, ARROW_K_COMM, m0, m1);
        prof_rec(P, M, ARROW_K_COMM, m2, m3);
        prof_rec(P, M, ARROW_K_SEGMENTS, m4, m5);
        prof_rec(P, M, ARROW_K_SEGMENTS, m6, m7);
        prof_rec(P, M, ARROW_K_COMM, m8, m9);
        prof_rec(P, M, ARROW_K_COMM, m7b, m12);
        P->prof_acc.calls += 1;
    }
    marks_done(M);
    return ARROW_OK;
}

}  // namespace arrow

extern "C" arrow_status arrow_dist_schedule(arrow_decomposition d, int32_t nranks, int32_t rank, int64_t window_rows,
                                            int32_t head_chunk, int64_t *lohi, int64_t *counts) {
    if (!d || !lohi) return arrow::set_error(ARROW_E_INVALID_ARG, "NULL argument");
    if (nranks < 1 || nranks > arrow::kMaxPeers || rank < 0 || rank >= nranks)
        return arrow::set_error(ARROW_E_INVALID_ARG, "nranks must be in [1, 8] and rank in [0, nranks)");
    arrow::DistHost H;
    arrow_status st = arrow::dist_schedule(
        *d, nranks, rank, window_rows > 0 ? window_rows : arrow::kDefaultWindowRows,
        window_rows > 0 ? window_rows : arrow::kDefaultWindowRows,
        head_chunk > 0 ? head_chunk : arrow::kDefaultHeadChunk, 8, 0, H);
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
            c[4 * G + 0] = (int64_t)L.segs.ent_col.size();
            c[4 * G + 1] = (int64_t)L.segs.seg_out.size();
            c[4 * G + 2] = (int64_t)L.head_j.size();
            c[4 * G + 3] = (int64_t)L.zero_rows.size() + (&L == &H.L[0] ? H.zero_tail_n : 0);
            c += 4 * G + 4;
        }
    }
    return ARROW_OK;
}
