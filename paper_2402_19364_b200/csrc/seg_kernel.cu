// seg_kernel.cu -- K-A, the segment-stream SpMM kernels of one arrow level (S1, S2, S4, S5).
//
// PAPER.md Alg. 1 per level i: body rows C^(r) = B^(r,0) D^(0) + B^(r,r) D^(r) and
// head-row slices C^(0) += B^(0,t) D^(t) one tile window t at a time; the permutations of
// Alg. 2 are folded into the column and output indices (S4), and levels >= 1 add into the
// Y rows written by level 0 (reverse aggregation; S5).
//
// Device layout of a level (arrow_internal.h SegLevel, built by layout.cpp): a list of non-empty
// segments (an output row, or one window's chunk of a head row) in tile-window order, cut into
// batches of `bs` consecutive segments.  Each batch's (col, val) entries are contiguous and start at
// a multiple of 8 entries (the gap before it is padding), so that a warp reads 4 columns or values
// with one 16-byte load that every lane issues on the same address (one L1 wavefront, no shuffles),
// and `gmask[e / 8]` marks which of the 8 entries of a group close a segment.
//   seg_out >= 0            : store (MODE 0, level 0) or read-modify-write (MODE 1) Y[out]
//   seg_out <  0, DIST == 0 : red.global.add into Y[out & 0x7fffffff] (head-row slice of one window)
//   seg_out <  0, DIST == 1 : red.global.add into C0[out & 0x7fffffff] (head partial, reduced over ranks)
//   col     <  0 (DIST only): the row comes from the head block D0 (broadcast), else from X
//   DIST == 2               : seg_out >= 0 encodes (rank << kPeerShift | row): the row is stored into
//                             rank's staging buffer outs.p[rank] -- over NVLink for a peer rank; with
//                             kLocalRmwBit it is added into Y[row] (a row homed on this GPU)
// Warps grab batches dynamically from a per-level counter, so all resident warps work on a narrow
// front of the window-ordered list and the X rows of the current window stay L2-resident while all
// their users run (the IO lemma's "tiles stay resident").
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>

#include "arrow_internal.h"
#include "dev_common.cuh"

namespace arrow {
namespace kseg {
namespace {

using dev::Frag;
using dev::VecT;
using dev::atomic_add_frag;
using dev::ld_plain;
using dev::ld_x;
using dev::st_plain;
using dev::st_stream;

template <typename T, int VEC>
__device__ __forceinline__ void apply_act(Frag<T, VEC> &f, int act) {
    if (act == 1) {
#pragma unroll
        for (int i = 0; i < VEC; ++i) f.v[i] = f.v[i] > T(0) ? f.v[i] : T(0);
    }
}

// Folded K-Z: grab g of ngrab zeroes its share of outs.zrows (streaming stores of zero rows, no
// dependence on anything the warp computes, so they drain while the warp gathers).  Lanes fetch
// up to 32 row ids at once; the whole warp then stores row by row (lanes with col < k).
template <typename T, int VEC>
__device__ __forceinline__ void zero_share(const PeerPtrs &outs, int64_t g, int64_t ngrab, T *Y, int64_t k, int lane) {
    if (outs.nzero == 0) return;
    const int64_t per = (outs.nzero + ngrab - 1) / ngrab;
    const int64_t z0 = g * per, z1 = (z0 + per < outs.nzero) ? z0 + per : outs.nzero;
    if (z0 >= z1) return;
    Frag<T, VEC> z;
    z.zero();
    const uint32_t kv = (uint32_t)(k / VEC);  // VEC-wide chunks per row (k % VEC == 0)
    if (kv <= 32u && (32u % kv) == 0u) {
        // rows of <= 32 chunks: RP = 32 / kv rows per warp store, lane -> (row lane / kv, chunk lane % kv)
        const uint32_t rp = 32u / kv, sub = (uint32_t)lane / kv, ch = (uint32_t)lane % kv;
        for (int64_t r0 = z0; r0 < z1; r0 += 32) {
            const int cnt = (z1 - r0 < 32) ? (int)(z1 - r0) : 32;
            const int32_t myrow = lane < cnt ? __ldg(outs.zrows + r0 + lane) : 0;
            for (uint32_t t = 0; t < (uint32_t)cnt; t += rp) {
                const int32_t row = __shfl_sync(0xffffffffu, myrow, (int)((t + sub) & 31u));
                if (t + sub < (uint32_t)cnt) st_stream<T, VEC>(Y + (int64_t)row * k + ch * VEC, z);
            }
        }
        return;
    }
    for (int64_t r0 = z0; r0 < z1; r0 += 32) {
        const int cnt = (z1 - r0 < 32) ? (int)(z1 - r0) : 32;
        const int32_t myrow = lane < cnt ? __ldg(outs.zrows + r0 + lane) : 0;
        for (int t = 0; t < cnt; ++t) {
            T *row = Y + (int64_t)__shfl_sync(0xffffffffu, myrow, t) * k;
            for (uint32_t c = (uint32_t)lane; c < kv; c += 32u) st_stream<T, VEC>(row + c * VEC, z);
        }
    }
}

template <typename T, int VEC, int MODE, int DIST>
__device__ __forceinline__ void flush_row(int32_t o, const Frag<T, VEC> &acc, T *Y, T *C0, int64_t k, int64_t col0,
                                          const PeerPtrs &outs) {
    if (o == (int32_t)kDiscard) return;  // a padding segment
    if (o < 0) {
        if (DIST == 0 && C0 != nullptr) {  // deterministic head partial: its own slot, plain store
            st_plain<T, VEC>(C0 + (int64_t)(o & 0x7fffffff) * k + col0, acc);
            return;
        }
        T *dst = DIST ? C0 + (int64_t)(o & 0x7fffffff) * k : Y + (int64_t)(o & 0x7fffffff) * k;
        atomic_add_frag<T, VEC>(dst + col0, acc);
    } else if (DIST == 2 && (o & kLocalRmwBit)) {
        T *py = Y + (int64_t)(o & kPeerRowMask) * k + col0;
        Frag<T, VEC> y = ld_plain<T, VEC>(py);
#pragma unroll
        for (int i = 0; i < VEC; ++i) y.v[i] += acc.v[i];
        st_plain<T, VEC>(py, y);
    } else if (DIST == 2) {
        T *base = reinterpret_cast<T *>(outs.p[(uint32_t)o >> kPeerShift]);
        st_stream<T, VEC>(base + (int64_t)(o & kPeerRowMask) * k + col0, acc);
    } else {
        // single GPU: bit 30 marks the row's final segment (iterate mode applies the activation)
        const bool fin = DIST == 0 && (o & kFinalBit) && outs.act;
        T *py = Y + (int64_t)(DIST == 0 ? (o & kRowMask30) : o) * k + col0;
        Frag<T, VEC> y = acc;
        if (MODE != 0) {
            y = ld_plain<T, VEC>(py);
#pragma unroll
            for (int i = 0; i < VEC; ++i) y.v[i] += acc.v[i];
        }
        if (fin) apply_act<T, VEC>(y, outs.act);
        if (MODE == 0) st_stream<T, VEC>(py, y);
        else st_plain<T, VEC>(py, y);
    }
}

// ------------------------------------------------------------------------------------ K-A (full warp)
// One warp per output row slab of 32*VEC elements (k = 128 fp32 / 64 fp64: the whole 512-byte row,
// one 16-byte load per lane per entry).  A group of 8 entries costs two broadcast 16-byte loads of
// columns, two (fp64: four) of values and one byte of end mask, then per entry one address IMAD.WIDE,
// one 16-byte gather and VEC/2 packed fp32 FMAs (FFMA2; fp64: VEC DFMAs).  The 8 gathers of a group
// are issued before their first use.  A group with no segment end runs without per-entry tests.
__device__ __forceinline__ void fma_x2(float &a0, float &a1, float s, float x0, float x1) {
    uint64_t acc, xv;
    asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(xv) : "f"(x0), "f"(x1));
    uint64_t sv;
    asm("mov.b64 %0, {%1, %1};" : "=l"(sv) : "f"(s));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(sv), "l"(xv));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(acc));
}

template <typename T, int VEC>
__device__ __forceinline__ void fma_frag(Frag<T, VEC> &acc, T a, const Frag<T, VEC> &x) {
    if constexpr (sizeof(T) == 4 && VEC % 2 == 0) {
#pragma unroll
        for (int i = 0; i < VEC; i += 2) fma_x2(acc.v[i], acc.v[i + 1], a, x.v[i], x.v[i + 1]);
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) acc.v[i] = fma(a, x.v[i], acc.v[i]);
    }
}

// the 8 values of a group: two float4 / four double2 broadcast loads
template <typename T> struct Vals8;
template <> struct Vals8<float> {
    float v[8];
    __device__ __forceinline__ void load(const float *p) {
        const float4 a = __ldg(reinterpret_cast<const float4 *>(p));
        const float4 b = __ldg(reinterpret_cast<const float4 *>(p) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
};
template <> struct Vals8<double> {
    double v[8];
    __device__ __forceinline__ void load(const double *p) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double2 a = __ldg(reinterpret_cast<const double2 *>(p) + i);
            v[2 * i] = a.x;
            v[2 * i + 1] = a.y;
        }
    }
};

template <typename T, int VEC, int DIST>
__device__ __forceinline__ const char *row_addr(int32_t c, const char *Xl, const char *Dl, uint32_t rb) {
    if (DIST && c < 0) return Dl + (uint64_t)((uint32_t)c & 0x7fffffffu) * rb;
    return Xl + (uint64_t)(uint32_t)c * rb;
}

// One group of 8 entries starting at e (a multiple of 8); the first n are this warp's; m = end mask.
template <typename T, int VEC, int MODE, int DIST, bool FULL>
__device__ __forceinline__ void ka_group(const int32_t *__restrict__ ent_col, const T *__restrict__ ent_val,
                                         uint32_t e, int n, unsigned m, const char *Xl, const char *Dl, uint32_t rb,
                                         Frag<T, VEC> &acc, int &cur, int32_t my_out, T *Y, T *C0, int64_t k,
                                         int64_t col0, const PeerPtrs &outs) {
    const int4 ca = __ldg(reinterpret_cast<const int4 *>(ent_col + e));
    const int4 cb = __ldg(reinterpret_cast<const int4 *>(ent_col + e) + 1);
    const int32_t c[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
    Frag<T, VEC> x[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        if (FULL || t < n) x[t] = ld_x<T, VEC>(reinterpret_cast<const T *>(row_addr<T, VEC, DIST>(c[t], Xl, Dl, rb)));
        else x[t].zero();
    }
    Vals8<T> a;
    a.load(ent_val + e);
    if (FULL && m == 0u) {  // warp-uniform: no segment ends in this group
#pragma unroll
        for (int t = 0; t < 8; ++t) fma_frag<T, VEC>(acc, a.v[t], x[t]);
        return;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        if (FULL || t < n) fma_frag<T, VEC>(acc, a.v[t], x[t]);
        if ((m >> t) & 1u) {  // (only set for t < n)
            const int32_t o = __shfl_sync(0xffffffffu, my_out, cur & 31);
            flush_row<T, VEC, MODE, DIST>(o, acc, Y, C0, k, col0, outs);
            acc.zero();
            ++cur;
        }
    }
}

// A warp takes one work batch of (up to) 16 segments at a time (measured: 16 better than 32 at
// k = 128); a batch starts at a multiple of 8 entries and usually ends inside a group of 8.
template <typename T, int VEC, int MODE, int DIST>
__global__ void __launch_bounds__(256, sizeof(T) == 8 ? 3 : 4) k_ka(const int32_t *__restrict__ seg_out,
                                               const uint32_t *__restrict__ seg_end, int64_t nseg,
                                               const int32_t *__restrict__ ent_col, const T *__restrict__ ent_val,
                                               const uint8_t *__restrict__ gmask, const uint2 *__restrict__ bat,
                                               int64_t nbatch, const T *__restrict__ X, const T *__restrict__ D0,
                                               T *__restrict__ Y, T *__restrict__ C0, int64_t k, uint32_t rb,
                                               unsigned *__restrict__ counter, const PeerPtrs outs) {
    // rb = k * sizeof(T), a 32-bit parameter: every gather address is then ONE IMAD.WIDE.U32
    const int lane = threadIdx.x & 31;
    (void)seg_end;
    for (;;) {
        unsigned wb = 0;
        if (lane == 0) wb = atomicAdd(counter, 1u);
        wb = __shfl_sync(0xffffffffu, wb, 0);
        if ((int64_t)wb >= nbatch) break;
        // batch wb: segments [wb * 17, wb * 17 + 16) (the last batch may be shorter), entries be
        const int64_t s0 = (int64_t)wb * 17;
        const int32_t my_out = (lane < 16 && s0 + lane < nseg) ? __ldg(seg_out + s0 + lane) : 0;
        const uint2 be = __ldg(bat + wb);
        const uint32_t e_lo = be.x, e_hi = be.y;
        if (MODE == 0 && DIST == 0) zero_share<T, VEC>(outs, wb, nbatch, Y, k, lane);

        for (int64_t c0 = 0; c0 < k; c0 += 32 * VEC) {
            const int64_t col0 = c0 + (int64_t)lane * VEC;
            // per-lane row bases, opaque to the compiler so that every gather address is one
            // IMAD.WIDE.U32 (col * row bytes + base)
            const char *Xl, *Dl;
            asm("mov.b64 %0, %1;" : "=l"(Xl) : "l"(reinterpret_cast<const char *>(X + col0)));
            asm("mov.b64 %0, %1;" : "=l"(Dl) : "l"(reinterpret_cast<const char *>(DIST ? D0 + col0 : X + col0)));
            Frag<T, VEC> acc;
            acc.zero();
            int cur = 0;
            uint32_t e = e_lo;  // (a multiple of 8)
#pragma unroll 1
            for (; e + 8u <= e_hi; e += 8u) {
                const unsigned m = __ldg(gmask + (e >> 3));
                ka_group<T, VEC, MODE, DIST, true>(ent_col, ent_val, e, 8, m, Xl, Dl, rb, acc, cur, my_out, Y, C0, k,
                                                    col0, outs);
            }
            if (e < e_hi) {  // the last group: the padding segment's end bit beyond it is masked off
                const int n = (int)(e_hi - e);
                const unsigned m = __ldg(gmask + (e >> 3)) & ((1u << n) - 1u);
                ka_group<T, VEC, MODE, DIST, false>(ent_col, ent_val, e, n, m, Xl, Dl, rb, acc, cur, my_out, Y, C0, k,
                                                     col0, outs);
            }
        }
    }
}

template <typename T, int VEC, int MODE, int DIST>
int run_ka(const SegLevel &L, const void *X, const void *D0, void *Y, void *C0, int64_t k, int num_sms,
           unsigned *counter, const PeerPtrs &outs, cudaStream_t st) {
    auto kern = k_ka<T, VEC, MODE, DIST>;
    static int b = 0;  // resident blocks per SM, per instantiation
    if (b == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 256, 0);
        if (b <= 0) b = 1;
    }
    int64_t blocks = std::min<int64_t>((int64_t)num_sms * b, (L.nbatch + 7) / 8);
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, 256, 0, st>>>(L.seg_out, L.seg_end, L.nseg, L.ent_col, reinterpret_cast<const T *>(L.ent_val),
                                           L.gmask, reinterpret_cast<const uint2 *>(L.bat), L.nbatch,
                                           reinterpret_cast<const T *>(X), reinterpret_cast<const T *>(D0),
                                           reinterpret_cast<T *>(Y), reinterpret_cast<T *>(C0), k,
                                           (uint32_t)(k * (int64_t)sizeof(T)), counter, outs);
    return (int)cudaGetLastError();
}

template <typename T, int VEC>
int run_ka_mode(int dist, const SegLevel &L, const void *X, const void *D0, void *Y, void *C0, int64_t k, int num_sms,
                unsigned *counter, const PeerPtrs &outs, cudaStream_t st) {
    if (dist == 2) return run_ka<T, VEC, 0, 2>(L, X, D0, Y, C0, k, num_sms, counter, outs, st);
    if (dist) return run_ka<T, VEC, 0, 1>(L, X, D0, Y, C0, k, num_sms, counter, outs, st);
    return L.mode == 0 ? run_ka<T, VEC, 0, 0>(L, X, D0, Y, C0, k, num_sms, counter, outs, st)
                       : run_ka<T, VEC, 1, 0>(L, X, D0, Y, C0, k, num_sms, counter, outs, st);
}

// ------------------------------------------------------------------------------------ K-A
// Segment stream.  A sub-warp of LPE lanes owns a row slab of LPE*VEC elements.  Work is a list
// of non-empty segments in tile-window order, cut into batches of LPE consecutive segments.
// Warps grab batches dynamically from a per-launch counter (one atomic per warp per grab), so
// all resident warps work on a narrow, advancing front of the window-ordered list and the X rows
// of the current window stay L2-resident while every user of them runs (the IO lemma's "tiles
// stay resident").  Lane s of a sub-warp holds the output row and end offset of
// segment s of its batch; the batch's entries are contiguous and are streamed in chunks of LPE
// (one coalesced load of col and val per lane).  A per-chunk bit mask of segment ends
// (__reduce_or_sync) tells the accumulate loop where to flush; UNROLL row loads are issued
// before their FMAs so short rows do not serialise on latency.
//   out >= 0             : store (MODE 0, level 0) or read-modify-write (MODE 1) Y[out]
//   out <  0, DIST == 0  : atomic add into Y[out & 0x7fffffff]  (head-row slice of one window)
//   out <  0, DIST == 1  : atomic add into C0[out & 0x7fffffff] (head partial, reduced over ranks)
//   col <  0 (DIST only) : the row comes from the head block D0 (broadcast), else from X
//   DIST == 2            : out >= 0 encodes (rank << kPeerShift | row): the row is stored into
//                          rank's staging buffer outs.p[rank] -- over NVLink for a peer rank;
//                          with kLocalRmwBit it is added into Y[row] (a row homed on this GPU)
template <typename T, int VEC, int LPE, int MODE, int DIST>
__global__ void __launch_bounds__(256, 4) k_segments(const int32_t *__restrict__ seg_out,
                                                     const uint32_t *__restrict__ seg_end, int64_t nseg,
                                                     const int32_t *__restrict__ ent_col,
                                                     const T *__restrict__ ent_val, const T *__restrict__ X,
                                                     const T *__restrict__ D0, T *__restrict__ Y,
                                                     T *__restrict__ C0, int64_t k, unsigned *__restrict__ counter,
                                                     int bseg, const PeerPtrs outs) {
    constexpr int UNROLL = (LPE == 32) ? 8 : 4;
    constexpr int SLAB = LPE * VEC;
    constexpr int SUBS = 32 / LPE;
    const int lane = threadIdx.x & 31;
    const int sl = lane % LPE;
    const int sub = lane / LPE;
    const unsigned mask = (LPE == 32) ? 0xffffffffu : (((1u << LPE) - 1u) << (sub * LPE));
    const int64_t nbatch = (nseg + bseg - 1) / bseg;
    const uint32_t rowbytes = (uint32_t)(k * (int64_t)sizeof(T));

    for (;;) {
        unsigned wb = 0;
        if (lane == 0) wb = atomicAdd(counter, 1u);
        wb = __shfl_sync(0xffffffffu, wb, 0);
        const int64_t bt = (int64_t)wb * SUBS + sub;
        if ((int64_t)wb * SUBS >= nbatch) break;       // warp-uniform exit
        if (MODE == 0 && DIST == 0) zero_share<T, VEC>(outs, wb, (nbatch + SUBS - 1) / SUBS, Y, k, lane);
        if (bt >= nbatch) continue;                    // sub-warp idle this round
        const int64_t s0 = bt * bseg;
        const int nb = (nseg - s0 < bseg) ? (int)(nseg - s0) : bseg;
        const int32_t my_out = (sl < nb) ? __ldg(seg_out + s0 + sl) : 0;
        const uint32_t my_end = (sl < nb) ? __ldg(seg_end + s0 + sl) : 0xffffffffu;
        const uint32_t e_begin = (s0 == 0) ? 0u : __ldg(seg_end + s0 - 1);
        const uint32_t e_end = __shfl_sync(mask, my_end, nb - 1, LPE);

        for (int64_t c0 = 0; c0 < k; c0 += SLAB) {
            const int64_t col0 = c0 + (int64_t)sl * VEC;
            const bool active = col0 < k;
            const char *xlane = reinterpret_cast<const char *>(X + (active ? col0 : 0));
            const char *dlane = reinterpret_cast<const char *>(D0 + (active ? col0 : 0));
            Frag<T, VEC> acc;
            acc.zero();
            int cur = 0;
            for (uint32_t cb = e_begin; cb < e_end; cb += LPE) {
                const int cnt = (e_end - cb < (uint32_t)LPE) ? (int)(e_end - cb) : LPE;
                int32_t mycol = 0;
                T myval = T(0);
                if (sl < cnt) {
                    mycol = __ldcs(ent_col + cb + sl);
                    myval = __ldcs(ent_val + cb + sl);
                }
                const uint32_t rel = my_end - 1u - cb;  // position of my segment's last entry in this chunk
                const unsigned endmask = __reduce_or_sync(mask, (rel < (uint32_t)LPE) ? (1u << rel) : 0u);
#pragma unroll 1
                for (int u0 = 0; u0 < cnt; u0 += UNROLL) {
                    Frag<T, VEC> xv[UNROLL];
                    T av[UNROLL];
#pragma unroll
                    for (int t = 0; t < UNROLL; ++t) {
                        const int idx = u0 + t;
                        const uint32_t cc = (uint32_t)__shfl_sync(mask, mycol, idx & (LPE - 1), LPE);
                        const T a = __shfl_sync(mask, myval, idx & (LPE - 1), LPE);
                        const bool ok = idx < cnt;
                        av[t] = ok ? a : T(0);
                        const char *p;
                        if (DIST && (int32_t)cc < 0) p = dlane + (uint64_t)(cc & 0x7fffffffu) * rowbytes;
                        else p = xlane + (uint64_t)cc * rowbytes;
                        if (ok && active) xv[t] = ld_x<T, VEC>(reinterpret_cast<const T *>(p));
                        else xv[t].zero();
                    }
#pragma unroll
                    for (int t = 0; t < UNROLL; ++t) {
#pragma unroll
                        for (int i = 0; i < VEC; ++i) acc.v[i] = fma(av[t], xv[t].v[i], acc.v[i]);
                        if ((u0 + t < cnt) && ((endmask >> ((u0 + t) & 31)) & 1u)) {   // sub-warp uniform
                            const int32_t o = __shfl_sync(mask, my_out, cur, LPE);
                            if (active && o != (int32_t)kDiscard) {
                                if (o < 0 && DIST == 0 && C0 != nullptr) {  // deterministic head partial
                                    st_plain<T, VEC>(C0 + (int64_t)(o & 0x7fffffff) * k + col0, acc);
                                } else if (o < 0) {
                                    T *dst = DIST ? C0 + (int64_t)(o & 0x7fffffff) * k : Y + (int64_t)(o & 0x7fffffff) * k;
                                    atomic_add_frag<T, VEC>(dst + col0, acc);
                                } else if (DIST == 2 && (o & kLocalRmwBit)) {
                                    T *py = Y + (int64_t)(o & kPeerRowMask) * k + col0;
                                    Frag<T, VEC> y = ld_plain<T, VEC>(py);
#pragma unroll
                                    for (int i = 0; i < VEC; ++i) y.v[i] += acc.v[i];
                                    st_plain<T, VEC>(py, y);
                                } else if (DIST == 2) {
                                    T *base = reinterpret_cast<T *>(outs.p[(uint32_t)o >> kPeerShift]);
                                    st_stream<T, VEC>(base + (int64_t)(o & kPeerRowMask) * k + col0, acc);
                                } else {
                                    const bool fin = DIST == 0 && (o & kFinalBit) && outs.act;
                                    T *py = Y + (int64_t)(DIST == 0 ? (o & kRowMask30) : o) * k + col0;
                                    Frag<T, VEC> y = acc;
                                    if (MODE != 0) {
                                        y = ld_plain<T, VEC>(py);
#pragma unroll
                                        for (int i = 0; i < VEC; ++i) y.v[i] += acc.v[i];
                                    }
                                    if (fin) apply_act<T, VEC>(y, outs.act);
                                    if (MODE == 0) st_stream<T, VEC>(py, y);
                                    else st_plain<T, VEC>(py, y);
                                }
                            }
                            acc.zero();
                            ++cur;
                        }
                    }
                }
            }
        }
    }
}

// ------------------------------------------------------------------------------------ K-A (short rows)
// Rows of LPE < 32 lanes (k = 8/16/32 fp32 with 16-byte lanes): the warp still works on ONE batch,
// and each step hands G = 32/LPE consecutive entries to its G sub-warps (one entry each), so a
// warp instruction gathers G rows.  Sub-warps keep private partial sums while no segment ends in
// a step; in a step with ends, the partials are folded (butterfly over the sub-warps), the step's
// products are combined by a segmented inclusive scan across the sub-warps, and every sub-warp
// whose entry closes a segment flushes that row -- several rows per step, in parallel.
template <typename T, int VEC>
__device__ __forceinline__ Frag<T, VEC> shfl_frag(const Frag<T, VEC> &f, int src_or_delta, int mode) {
    Frag<T, VEC> r;
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
        if (mode == 0) r.v[i] = __shfl_xor_sync(0xffffffffu, f.v[i], src_or_delta);
        else r.v[i] = __shfl_up_sync(0xffffffffu, f.v[i], src_or_delta);
    }
    return r;
}

template <typename T, int VEC, int LPE, int MODE, int DIST, bool OFF32, bool PF>
__global__ void __launch_bounds__(256, 4) k_segsmall(const int32_t *__restrict__ seg_out,
                                                     const uint32_t *__restrict__ seg_end, int64_t nseg,
                                                     const int32_t *__restrict__ ent_col,
                                                     const T *__restrict__ ent_val, const T *__restrict__ X,
                                                     const T *__restrict__ D0, T *__restrict__ Y, T *__restrict__ C0,
                                                     int64_t k, unsigned *__restrict__ counter, int bseg,
                                                     const PeerPtrs outs) {
    constexpr int G = 32 / LPE;
    // steps whose rows are loaded together (PF: a whole 32-entry chunk when it fits in 8 steps)
    constexpr int UMAX = PF ? 8 : 4;
    constexpr int U = (32 / G) < UMAX ? (32 / G) : UMAX;
    const int lane = threadIdx.x & 31;
    const int q = lane / LPE;   // sub-warp: entry slot within a step
    const int sl = lane % LPE;  // 16-byte slice of the row
    const int64_t col0 = (int64_t)sl * VEC;
    const uint32_t lane_off = (uint32_t)(col0 * (int64_t)sizeof(T));
    const int64_t nbatch = (nseg + bseg - 1) / bseg;
    const uint32_t rowbytes = (uint32_t)(k * (int64_t)sizeof(T));
    const char *Xc = reinterpret_cast<const char *>(X);
    const char *Dc = reinterpret_cast<const char *>(D0);

    for (;;) {
        unsigned wb = 0;
        if (lane == 0) wb = atomicAdd(counter, 1u);
        wb = __shfl_sync(0xffffffffu, wb, 0);
        if ((int64_t)wb >= nbatch) break;
        const int64_t s0 = (int64_t)wb * bseg;
        const int nb = (nseg - s0 < bseg) ? (int)(nseg - s0) : bseg;
        const int32_t my_out = (lane < nb) ? __ldg(seg_out + s0 + lane) : 0;
        const uint32_t my_end = (lane < nb) ? __ldg(seg_end + s0 + lane) : 0xffffffffu;
        const uint32_t e_begin = (s0 == 0) ? 0u : __ldg(seg_end + s0 - 1);
        const uint32_t e_end = __shfl_sync(0xffffffffu, my_end, nb - 1);
        if (MODE == 0 && DIST == 0) zero_share<T, VEC>(outs, wb, nbatch, Y, k, lane);
        if (MODE == 1 && DIST == 0 && lane < nb && my_out >= 0 && my_out != (int32_t)kDiscard)  // RMW: Y rows into L2
            asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(reinterpret_cast<const char *>(Y) +
                                                                  (uint64_t)(uint32_t)(my_out & kRowMask30) * rowbytes));

        Frag<T, VEC> acc;
        acc.zero();
        int cur = 0;  // segments of the batch closed so far
        // PF: the next chunk's (col, val) are requested before this chunk's rows are gathered, so a
        // chunk costs one memory latency (its gathers) instead of two
        int32_t pcol = 0;
        T pval = T(0);
        if (PF && e_begin + lane < e_end) {
            pcol = __ldcs(ent_col + e_begin + lane);
            pval = __ldcs(ent_val + e_begin + lane);
        }
        for (uint32_t cb = e_begin; cb < e_end; cb += 32) {
            const int cnt = (e_end - cb < 32u) ? (int)(e_end - cb) : 32;
            int32_t mycol = 0;
            T myval = T(0);
            if (PF) {
                mycol = pcol;
                myval = pval;
                if (cb + 32 + lane < e_end) {
                    pcol = __ldcs(ent_col + cb + 32 + lane);
                    pval = __ldcs(ent_val + cb + 32 + lane);
                }
            } else if (lane < cnt) {
                mycol = __ldcs(ent_col + cb + lane);
                myval = __ldcs(ent_val + cb + lane);
            }
            const uint32_t rel = my_end - 1u - cb;
            const unsigned endmask = __reduce_or_sync(0xffffffffu, (rel < 32u) ? (1u << rel) : 0u);
#pragma unroll 1
            for (int g0 = 0; g0 < cnt; g0 += G * U) {
                // U steps' rows are requested before the first is used (memory-level parallelism)
                Frag<T, VEC> xs[U];
                T vals[U];
#pragma unroll
                for (int t = 0; t < U; ++t) {
                    const int e = g0 + t * G + q;
                    const int32_t col = __shfl_sync(0xffffffffu, mycol, e & 31);
                    vals[t] = __shfl_sync(0xffffffffu, myval, e & 31);
                    const char *p;
                    if (DIST && col < 0) p = Dc + (uint64_t)((uint32_t)col & 0x7fffffffu) * rowbytes + lane_off;
                    else if (OFF32) p = Xc + (uint32_t)((uint32_t)col * rowbytes + lane_off);
                    else p = Xc + (uint64_t)(uint32_t)col * rowbytes + lane_off;
                    if (e < cnt) xs[t] = ld_x<T, VEC>(reinterpret_cast<const T *>(p));
                    else xs[t].zero();
                }
#pragma unroll
                for (int t = 0; t < U; ++t) {
                    const int u0 = g0 + t * G;
                    if (u0 >= cnt) break;  // warp-uniform
                    const unsigned ends = (endmask >> u0) & ((G == 32) ? 0xffffffffu : ((1u << G) - 1u));
                    if (ends == 0u) {  // warp-uniform: every entry of the step continues the open segment
#pragma unroll
                        for (int i = 0; i < VEC; ++i) acc.v[i] = fma(vals[t], xs[t].v[i], acc.v[i]);
                        continue;
                    }
                    Frag<T, VEC> v;
#pragma unroll
                    for (int i = 0; i < VEC; ++i) v.v[i] = vals[t] * xs[t].v[i];
                    if (__popc(ends) == 1) {  // warp-uniform, the common case: one segment closes at slot e
                        const int e = __ffs(ends) - 1;
                        // total = every partial + the products of slots <= e; slots > e open the next one
                        Frag<T, VEC> w = acc;
                        if (q <= e) {
#pragma unroll
                            for (int i = 0; i < VEC; ++i) w.v[i] += v.v[i];
                        }
#pragma unroll
                        for (int o = LPE; o < 32; o <<= 1) {
                            const Frag<T, VEC> tt = shfl_frag<T, VEC>(w, o, 0);
#pragma unroll
                            for (int i = 0; i < VEC; ++i) w.v[i] += tt.v[i];
                        }
                        const int32_t o1 = __shfl_sync(0xffffffffu, my_out, cur & 31);
                        if (q == 0) flush_row<T, VEC, MODE, DIST>(o1, w, Y, C0, k, col0, outs);
                        cur += 1;
                        if (q > e) acc = v;
                        else acc.zero();
                        continue;
                    }
                    // fold the sub-warps' partials of the open segment into slot 0's product
#pragma unroll
                    for (int o = LPE; o < 32; o <<= 1) {
                        const Frag<T, VEC> tt = shfl_frag<T, VEC>(acc, o, 0);
#pragma unroll
                        for (int i = 0; i < VEC; ++i) acc.v[i] += tt.v[i];
                    }
                    if (q == 0) {
#pragma unroll
                        for (int i = 0; i < VEC; ++i) v.v[i] += acc.v[i];
                    }
                    // segmented inclusive scan over the G slots; slot q starts a segment if q-1 ended one
                    bool f = q > 0 && ((ends >> (q - 1)) & 1u);
#pragma unroll
                    for (int d = 1; d < G; d <<= 1) {
                        const Frag<T, VEC> tt = shfl_frag<T, VEC>(v, d * LPE, 1);
                        const bool tf = __shfl_up_sync(0xffffffffu, f, d * LPE);
                        if (q >= d && !f) {
#pragma unroll
                            for (int i = 0; i < VEC; ++i) v.v[i] += tt.v[i];
                            f = tf;
                        }
                    }
                    // slots that close a segment flush it (segment index cur + closed ends before them)
                    const bool closes = (ends >> q) & 1u;
                    const int sidx = cur + __popc(ends & ((1u << q) - 1u));
                    const int32_t o = __shfl_sync(0xffffffffu, my_out, sidx & 31);
                    if (closes) flush_row<T, VEC, MODE, DIST>(o, v, Y, C0, k, col0, outs);
                    cur += __popc(ends);
                    // the open segment continues with the scanned value of the last valid slot
                    const int last = min(G, cnt - u0) - 1;
                    acc.zero();
                    if (q == last && !closes) acc = v;
                }
            }
        }
    }
}

template <typename T, int VEC, int LPE, int MODE, int DIST>
int run_segsmall(const SegLevel &L, const void *X, const void *D0, void *Y, void *C0, int64_t k, int num_sms,
                 unsigned *counter, const PeerPtrs &outs, bool off32, cudaStream_t st) {
    const int bseg = 32;
    // the next chunk's entries requested one chunk ahead, whole-chunk row loads (PF)
    auto kern = off32 ? k_segsmall<T, VEC, LPE, MODE, DIST, true, true> : k_segsmall<T, VEC, LPE, MODE, DIST, false, true>;
    static int bps[2] = {0, 0};
    int &b = bps[off32 ? 1 : 0];
    if (b == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 256, 0);
        if (b <= 0) b = 1;
    }
    const int64_t nbatch = (L.nseg + bseg - 1) / bseg;
    int64_t blocks = std::min<int64_t>((int64_t)num_sms * b, (nbatch + 7) / 8);
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, 256, 0, st>>>(L.seg_out, L.seg_end, L.nseg, L.ent_col,
                                           reinterpret_cast<const T *>(L.ent_val), reinterpret_cast<const T *>(X),
                                           reinterpret_cast<const T *>(D0), reinterpret_cast<T *>(Y),
                                           reinterpret_cast<T *>(C0), k, counter, bseg, outs);
    return (int)cudaGetLastError();
}

template <typename T, int VEC, int LPE>
int run_segsmall_mode(int dist, const SegLevel &L, const void *X, const void *D0, void *Y, void *C0, int64_t k,
                      int num_sms, unsigned *counter, const PeerPtrs &outs, bool off32, cudaStream_t st) {
    if (dist == 2) return run_segsmall<T, VEC, LPE, 0, 2>(L, X, D0, Y, C0, k, num_sms, counter, outs, off32, st);
    if (dist) return L.mode == 0 ? run_segsmall<T, VEC, LPE, 0, 1>(L, X, D0, Y, C0, k, num_sms, counter, outs, off32, st)
                                 : run_segsmall<T, VEC, LPE, 1, 1>(L, X, D0, Y, C0, k, num_sms, counter, outs, off32, st);
    return L.mode == 0 ? run_segsmall<T, VEC, LPE, 0, 0>(L, X, D0, Y, C0, k, num_sms, counter, outs, off32, st)
                       : run_segsmall<T, VEC, LPE, 1, 0>(L, X, D0, Y, C0, k, num_sms, counter, outs, off32, st);
}

template <typename T, int VEC, int LPE, int MODE, int DIST>
int run_segments(const SegLevel &L, const void *X, const void *D0, void *Y, void *C0, int64_t k, int num_sms,
                 unsigned *counter, int bseg, const PeerPtrs &outs, cudaStream_t st) {
    if (bseg <= 0 || bseg > LPE) bseg = LPE;
    auto kern = k_segments<T, VEC, LPE, MODE, DIST>;
    static int bps = 0;
    if (bps == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 256, 0);
        if (bps <= 0) bps = 1;
    }
    const int64_t nbatch = (L.nseg + bseg - 1) / bseg;
    const int64_t batches_per_block = 8 * (32 / LPE);
    int64_t blocks = std::min<int64_t>((int64_t)num_sms * bps, (nbatch + batches_per_block - 1) / batches_per_block);
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, 256, 0, st>>>(L.seg_out, L.seg_end, L.nseg, L.ent_col,
                                            reinterpret_cast<const T *>(L.ent_val), reinterpret_cast<const T *>(X),
                                            reinterpret_cast<const T *>(D0), reinterpret_cast<T *>(Y),
                                            reinterpret_cast<T *>(C0), k, counter, bseg, outs);
    return (int)cudaGetLastError();
}

template <typename T, int VEC, int MODE, int DIST>
int run_segments_lpe(int lpe, const SegLevel &L, const void *X, const void *D0, void *Y, void *C0, int64_t k,
                     int num_sms, unsigned *counter, int bseg, const PeerPtrs &outs, cudaStream_t st) {
    switch (lpe) {
        case 32: return run_segments<T, VEC, 32, MODE, DIST>(L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, st);
        case 16: return run_segments<T, VEC, 16, MODE, DIST>(L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, st);
        case 8: return run_segments<T, VEC, 8, MODE, DIST>(L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, st);
        case 4: return run_segments<T, VEC, 4, MODE, DIST>(L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, st);
        case 2: return run_segments<T, VEC, 2, MODE, DIST>(L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, st);
        default: return run_segments<T, VEC, 1, MODE, DIST>(L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, st);
    }
}

template <typename T, int VEC>
int run_segments_mode(int lpe, int dist, const SegLevel &L, const void *X, const void *D0, void *Y, void *C0,
                      int64_t k, int num_sms, unsigned *counter, int bseg, const PeerPtrs &outs, cudaStream_t st) {
    if (dist == 2) return run_segments_lpe<T, VEC, 0, 2>(lpe, L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, st);
    if (dist) {
        return L.mode == 0 ? run_segments_lpe<T, VEC, 0, 1>(lpe, L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, st)
                           : run_segments_lpe<T, VEC, 1, 1>(lpe, L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, st);
    }
    return L.mode == 0 ? run_segments_lpe<T, VEC, 0, 0>(lpe, L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, st)
                       : run_segments_lpe<T, VEC, 1, 0>(lpe, L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, st);
}


}  // namespace
}  // namespace kseg

int launch_seg(int dtype, int dist, const SegLevel &L, const void *X, const void *D0, void *Y, void *C0, int64_t k,
               int num_sms, unsigned *counter, void *stream, const SegLaunch &opt, const PeerPtrs *outs, int act,
               const int32_t *zrows, int64_t nzero) {
    using namespace kseg;
    if (k == 0) return 0;
    if (L.nseg == 0) return nzero > 0 ? launch_zero_rows(dtype, zrows, nzero, k, Y, stream) : 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    PeerPtrs po{};
    if (outs) po = *outs;
    po.act = act;
    (void)opt;
    if (dist == 0 && nzero > 0) {
        po.zrows = zrows;
        po.nzero = nzero;
    }
    if (dist == 2 && !outs) return (int)cudaErrorInvalidValue;
    int vec = dist ? pick_vec(dtype, k, {X, Y, D0, C0}) : pick_vec(dtype, k, {X, Y});
    if (dist == 2)
        for (const void *p : po.p) vec = std::min(vec, pick_vec(dtype, k, {p}));
    const int lpe = pick_lpe(k, vec);
    // 32-bit X offsets when every X (and D0) row offset fits
    const bool off32 = (uint64_t)L.max_x_row * (uint64_t)k * (dtype == 1 ? 8u : 4u) < (1ull << 32) - (1ull << 20);
    const int bseg = 16;
    // full-warp rows (k = 128 fp32 / 64 fp64 and multiples): the broadcast-entry kernel
    if (lpe == 32 && k % (32 * vec) == 0) {
        if (dtype == 0 && vec == 4) return run_ka_mode<float, 4>(dist, L, X, D0, Y, C0, k, num_sms, counter, po, st);
        if (dtype == 1 && vec == 2) return run_ka_mode<double, 2>(dist, L, X, D0, Y, C0, k, num_sms, counter, po, st);
    }
    // short rows (k = 8/16/32 fp32, 4/8/16/32 fp64 with 16-byte lanes): G entries per warp step,
    // segmented scan across the sub-warps
    if (lpe < 32 && lpe >= 2 && k == (int64_t)lpe * vec && vec == 16 / (dtype == 1 ? 8 : 4)) {
        if (dtype == 0) {
            if (lpe == 16) return run_segsmall_mode<float, 4, 16>(dist, L, X, D0, Y, C0, k, num_sms, counter, po, off32, st);
            if (lpe == 8) return run_segsmall_mode<float, 4, 8>(dist, L, X, D0, Y, C0, k, num_sms, counter, po, off32, st);
            if (lpe == 4) return run_segsmall_mode<float, 4, 4>(dist, L, X, D0, Y, C0, k, num_sms, counter, po, off32, st);
            return run_segsmall_mode<float, 4, 2>(dist, L, X, D0, Y, C0, k, num_sms, counter, po, off32, st);
        } else {
            if (lpe == 16) return run_segsmall_mode<double, 2, 16>(dist, L, X, D0, Y, C0, k, num_sms, counter, po, off32, st);
            if (lpe == 8) return run_segsmall_mode<double, 2, 8>(dist, L, X, D0, Y, C0, k, num_sms, counter, po, off32, st);
            if (lpe == 4) return run_segsmall_mode<double, 2, 4>(dist, L, X, D0, Y, C0, k, num_sms, counter, po, off32, st);
            return run_segsmall_mode<double, 2, 2>(dist, L, X, D0, Y, C0, k, num_sms, counter, po, off32, st);
        }
    }
    // fp32 rows of 64 elements: one row per warp with 8-byte lanes (one 256-byte request per entry)
    // instead of 16-lane sub-warps that run different batches in lockstep
    if (dtype == 0 && k == 64 && vec >= 2)
        return run_ka_mode<float, 2>(dist, L, X, D0, Y, C0, k, num_sms, counter, po, st);
    if (dtype == 0) {
        if (vec == 4) return run_segments_mode<float, 4>(lpe, dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, po, st);
        if (vec == 2) return run_segments_mode<float, 2>(lpe, dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, po, st);
        return run_segments_mode<float, 1>(lpe, dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, po, st);
    }
    if (vec == 2) return run_segments_mode<double, 2>(lpe, dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, po, st);
    return run_segments_mode<double, 1>(lpe, dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, po, st);
}

}  // namespace arrow
