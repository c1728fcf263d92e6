// seg_kernel.cu -- the earlier descriptor-based K-A ("v2"): per-segment (out, end) descriptors +
// (col, val) entries, sub-warp batches of LPE segments, end-of-segment bit masks.  Kept as an
// alternative path (ARROW_SEG=1 at plan creation) for A/B measurements against k_rec; layout is
// derived from the record stream (arrow_api.cpp::derive_seg).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "arrow_internal.h"

namespace arrow {
namespace kseg {
namespace {

template <typename T, int VEC> struct VecT;
template <> struct VecT<float, 4> { using type = float4; };
template <> struct VecT<float, 2> { using type = float2; };
template <> struct VecT<float, 1> { using type = float; };
template <> struct VecT<double, 2> { using type = double2; };
template <> struct VecT<double, 1> { using type = double; };

template <typename T, int VEC> struct Frag {
    T v[VEC];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < VEC; ++i) v[i] = T(0);
    }
};

template <typename T, int VEC>
__device__ __forceinline__ Frag<T, VEC> ld_x(const T *p) {  // read-only path, 16 B per lane at VEC*sizeof(T)=16
    using V = typename VecT<T, VEC>::type;
    V r = __ldg(reinterpret_cast<const V *>(p));
    Frag<T, VEC> f;
    static_assert(sizeof(V) == sizeof(f), "frag size");
    memcpy(&f, &r, sizeof(V));
    return f;
}

template <typename T, int VEC>
__device__ __forceinline__ Frag<T, VEC> ld_plain(const T *p) {
    using V = typename VecT<T, VEC>::type;
    V r = *reinterpret_cast<const V *>(p);
    Frag<T, VEC> f;
    memcpy(&f, &r, sizeof(V));
    return f;
}

template <typename T, int VEC>
__device__ __forceinline__ void st_stream(T *p, const Frag<T, VEC> &f) {  // evict-first: Y is write-once
    using V = typename VecT<T, VEC>::type;
    V r;
    memcpy(&r, &f, sizeof(V));
    __stcs(reinterpret_cast<V *>(p), r);
}

template <typename T, int VEC>
__device__ __forceinline__ void st_plain(T *p, const Frag<T, VEC> &f) {
    using V = typename VecT<T, VEC>::type;
    V r;
    memcpy(&r, &f, sizeof(V));
    *reinterpret_cast<V *>(p) = r;
}

template <typename T, int VEC>
__device__ __forceinline__ void atomic_add_frag(T *p, const Frag<T, VEC> &f) {
    if constexpr (sizeof(T) == 4 && VEC == 4) {
        atomicAdd(reinterpret_cast<float4 *>(p), make_float4(f.v[0], f.v[1], f.v[2], f.v[3]));
    } else if constexpr (sizeof(T) == 4 && VEC == 2) {
        atomicAdd(reinterpret_cast<float2 *>(p), make_float2(f.v[0], f.v[1]));
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) atomicAdd(p + i, f.v[i]);
    }
}

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
    const uint32_t kv = (uint32_t)(k / VEC);           // VEC-wide chunks per row (pick_vec: k % VEC == 0)
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

// Levels >= 1 (read-modify-write): every lane holding one of the batch's segments asks L2 for that
// segment's Y row at batch start, so the flush's load hits L2 instead of waiting on DRAM.
template <typename T>
__device__ __forceinline__ void prefetch_y_rows(int ypf, int32_t my_out, bool valid, const T *Y, int64_t k) {
    if (!ypf || !valid || my_out < 0) return;
    const char *row = reinterpret_cast<const char *>(Y) + (uint64_t)(uint32_t)(my_out & kRowMask30) * (uint64_t)(k * sizeof(T));
    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(row));  // first 128-byte line (k <= 32 fp32: the row)
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
                            if (active) {
                                if (o < 0) {
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


inline int pick_vec(int dtype, int64_t k, std::initializer_list<const void *> ptrs) {
    const int es = dtype == 1 ? 8 : 4;
    int vec = 16 / es;
    while (vec > 1) {
        bool ok = (k % vec) == 0;
        for (const void *p : ptrs) ok = ok && ((reinterpret_cast<uintptr_t>(p) % (vec * es)) == 0);
        if (ok) break;
        vec >>= 1;
    }
    return vec;
}

inline int pick_lpe(int64_t k, int vec) {
    const int64_t need = (k + vec - 1) / vec;
    int lpe = 1;
    while (lpe < 32 && lpe < need) lpe <<= 1;
    return lpe;
}

// ------------------------------------------------------------------------------------ K-A (full warp)
// The same segment stream as k_segments, specialised for full-warp rows (LPE = 32, k a multiple
// of 32*VEC -- k = 128 fp32 / 64 fp64 and up): per 32-entry chunk every lane stages one (col, val)
// pair into a warp-private shared-memory slot, after which an entry costs one broadcast LDS, one
// address IMAD, one 16-byte LDG and VEC FFMAs.  Groups of 8 entries with no segment end (long rows,
// head-row chunks) run without per-entry end tests; only a batch's last group is predicated.
template <typename T> struct StagedEnt;
template <> struct alignas(8) StagedEnt<float> { int32_t col; float val; };
template <> struct alignas(16) StagedEnt<double> { int32_t col; int32_t pad; double val; };

template <typename T, int VEC, int MODE, int DIST>
__device__ __forceinline__ void flush_row(int32_t o, const Frag<T, VEC> &acc, T *Y, T *C0, int64_t k, int64_t col0,
                                          const PeerPtrs &outs) {
    if (o < 0) {
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

template <typename T> struct Seg32Unroll { static constexpr int value = sizeof(T) == 4 ? 8 : 4; };

template <typename T, int VEC, int MODE, int DIST, bool OFF32>
__device__ __forceinline__ void seg32_group(int32_t mycol, T myval, int u0, int n, unsigned grp, const char *Xc,
                                            const char *Dc, uint32_t rowbytes, uint32_t lane_off, Frag<T, VEC> &acc,
                                            int &cur, int32_t my_out, T *Y, T *C0, int64_t k, int64_t col0,
                                            const PeerPtrs &outs) {
    constexpr int UNROLL = Seg32Unroll<T>::value;
    Frag<T, VEC> xv[UNROLL];
    T av[UNROLL];
#pragma unroll
    for (int t = 0; t < UNROLL; ++t) {
        const int32_t col = __shfl_sync(0xffffffffu, mycol, (u0 + t) & 31);
        av[t] = __shfl_sync(0xffffffffu, myval, (u0 + t) & 31);
        const char *p;
        if (DIST && col < 0) p = Dc + (uint64_t)((uint32_t)col & 0x7fffffffu) * rowbytes + lane_off;
        else if (OFF32) p = Xc + (uint32_t)((uint32_t)col * rowbytes + lane_off);
        else p = Xc + (uint64_t)(uint32_t)col * rowbytes + lane_off;
        if (t < n) xv[t] = ld_x<T, VEC>(reinterpret_cast<const T *>(p));
    }
    if (n == UNROLL && grp == 0u) {  // warp-uniform: no segment ends in this group
#pragma unroll
        for (int t = 0; t < UNROLL; ++t)
#pragma unroll
            for (int i = 0; i < VEC; ++i) acc.v[i] = fma(av[t], xv[t].v[i], acc.v[i]);
        return;
    }
#pragma unroll
    for (int t = 0; t < UNROLL; ++t) {
        if (t < n) {
#pragma unroll
            for (int i = 0; i < VEC; ++i) acc.v[i] = fma(av[t], xv[t].v[i], acc.v[i]);
        }
        if ((grp >> t) & 1u) {  // (only set for t < n)
            const int32_t o = __shfl_sync(0xffffffffu, my_out, cur);
            flush_row<T, VEC, MODE, DIST>(o, acc, Y, C0, k, col0, outs);
            acc.zero();
            ++cur;
        }
    }
}

template <typename T, int VEC, int MODE, int DIST, bool OFF32, bool PF>
__global__ void __launch_bounds__(256, 4) k_seg32(const int32_t *__restrict__ seg_out,
                                                  const uint32_t *__restrict__ seg_end, int64_t nseg,
                                                  const int32_t *__restrict__ ent_col, const T *__restrict__ ent_val,
                                                  const T *__restrict__ X, const T *__restrict__ D0,
                                                  T *__restrict__ Y, T *__restrict__ C0, int64_t k,
                                                  unsigned *__restrict__ counter, int bseg, const PeerPtrs outs) {
    constexpr int UNROLL = Seg32Unroll<T>::value;
    const int lane = threadIdx.x & 31;
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

        for (int64_t c0 = 0; c0 < k; c0 += 32 * VEC) {
            const int64_t col0 = c0 + (int64_t)lane * VEC;
            const uint32_t lane_off = (uint32_t)(col0 * (int64_t)sizeof(T));
            Frag<T, VEC> acc;
            acc.zero();
            int cur = 0;
            // PF: the next chunk's (col, val) are requested one chunk ahead
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
                for (int u0 = 0; u0 < cnt; u0 += UNROLL) {
                    const unsigned grp = (endmask >> u0) & ((1u << UNROLL) - 1u);
                    seg32_group<T, VEC, MODE, DIST, OFF32>(mycol, myval, u0, min(cnt - u0, UNROLL), grp, Xc,
                                                                  Dc, rowbytes, lane_off, acc, cur, my_out, Y, C0, k,
                                                                  col0, outs);
                }
            }
        }
    }
}

template <typename T, int VEC, int MODE, int DIST>
int run_seg32(const SegLevel &L, const void *X, const void *D0, void *Y, void *C0, int64_t k, int num_sms,
              unsigned *counter, int bseg, const PeerPtrs &outs, bool off32, cudaStream_t st) {
    if (bseg <= 0 || bseg > 32) bseg = 32;
    // (a deferred read-modify-write of level >= 1 rows -- the Y load issued when a segment closes and
    // completed at the next close -- measured no gain on config R, 2.84 vs 2.82 ms K-A; removed.
    // Preloading the Y rows of every segment ending in an 8-entry group together with its gathers
    // needs 80 registers (3 blocks/SM): level 1 0.66 vs 0.50 ms, step 3.17 vs 2.88 ms; removed,
    // profiles/r01/ab_yp/.  An L2 evict-first policy (createpolicy + .L2::cache_hint) on those Y
    // loads/stores: 2.85/2.85/2.92 vs 2.86/2.87/2.87 ms, neutral; removed, profiles/r01/yef/)
    // entry prefetch one chunk ahead (ARROW_SEG32_PF=1; measured neutral-to-worse at k = 128 -- the
    // full-warp kernel's chunk has four 8-row gather groups, so the entry load was 1 of 5 latencies)
    static const bool pf = std::getenv("ARROW_SEG32_PF") && std::getenv("ARROW_SEG32_PF")[0] == '1';
    auto kern = pf ? (off32 ? k_seg32<T, VEC, MODE, DIST, true, true> : k_seg32<T, VEC, MODE, DIST, false, true>)
                   : (off32 ? k_seg32<T, VEC, MODE, DIST, true, false> : k_seg32<T, VEC, MODE, DIST, false, false>);
    static int bps[4] = {0, 0, 0, 0};
    int &b = bps[(off32 ? 1 : 0) + (pf ? 2 : 0)];
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

template <typename T, int VEC>
int run_seg32_mode(int dist, const SegLevel &L, const void *X, const void *D0, void *Y, void *C0, int64_t k,
                   int num_sms, unsigned *counter, int bseg, const PeerPtrs &outs, bool off32, cudaStream_t st) {
    if (dist == 2) return run_seg32<T, VEC, 0, 2>(L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, off32, st);
    if (dist) return L.mode == 0 ? run_seg32<T, VEC, 0, 1>(L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, off32, st)
                                 : run_seg32<T, VEC, 1, 1>(L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, off32, st);
    return L.mode == 0 ? run_seg32<T, VEC, 0, 0>(L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, off32, st)
                       : run_seg32<T, VEC, 1, 0>(L, X, D0, Y, C0, k, num_sms, counter, bseg, outs, off32, st);
}

// ------------------------------------------------------------------------------------ K-A (levels >= 1)
// Levels >= 1 of a single-GPU plan read-modify-write scattered Y rows.  In k_seg32 the read of a
// row is issued when its segment closes and the warp waits for it before going on (one DRAM
// latency per segment, ~6 entries).  Here a warp takes STAGE segments at a time and, before
// gathering their entries, starts asynchronous copies (cp.async, 16 B per lane) of all their Y
// slabs into a warp-private shared-memory stage; the flush then reads the row from shared memory.
// The Y reads overlap the gathers as in a plain RMW stream (profiles/rmw_bw.cu: 6.2 TB/s).
template <typename T, int VEC, bool OFF32, int STAGE>
__global__ void __launch_bounds__(256, 4) k_tail32(const int32_t *__restrict__ seg_out,
                                                   const uint32_t *__restrict__ seg_end, int64_t nseg,
                                                   const int32_t *__restrict__ ent_col, const T *__restrict__ ent_val,
                                                   const T *__restrict__ X, T *__restrict__ Y, int64_t k,
                                                   unsigned *__restrict__ counter, const PeerPtrs outs) {
    constexpr int UNROLL = Seg32Unroll<T>::value;
    using V = typename VecT<T, VEC>::type;
    __shared__ V stage[8][STAGE][32];  // 8 warps x STAGE rows x 512 B
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int64_t nbatch = (nseg + STAGE - 1) / STAGE;
    const uint32_t rowbytes = (uint32_t)(k * (int64_t)sizeof(T));
    const char *Xc = reinterpret_cast<const char *>(X);
    for (;;) {
        unsigned wb = 0;
        if (lane == 0) wb = atomicAdd(counter, 1u);
        wb = __shfl_sync(0xffffffffu, wb, 0);
        if ((int64_t)wb >= nbatch) break;
        const int64_t s0 = (int64_t)wb * STAGE;
        const int nb = (nseg - s0 < STAGE) ? (int)(nseg - s0) : STAGE;
        const int32_t my_out = (lane < nb) ? __ldg(seg_out + s0 + lane) : 0;
        const uint32_t my_end = (lane < nb) ? __ldg(seg_end + s0 + lane) : 0xffffffffu;
        const uint32_t e_begin = (s0 == 0) ? 0u : __ldg(seg_end + s0 - 1);
        const uint32_t e_end = __shfl_sync(0xffffffffu, my_end, nb - 1);
        for (int64_t c0 = 0; c0 < k; c0 += 32 * VEC) {
            const int64_t col0 = c0 + (int64_t)lane * VEC;
            const uint32_t lane_off = (uint32_t)(col0 * (int64_t)sizeof(T));
            // stage the Y slabs of the body segments (head partials are L2 atomics, not staged)
#pragma unroll
            for (int s = 0; s < STAGE; ++s) {
                const int32_t o = __shfl_sync(0xffffffffu, my_out, s);
                if (s < nb && o >= 0) {
                    const T *src = Y + (int64_t)(o & kRowMask30) * k + col0;
                    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&stage[wid][s][lane]);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            Frag<T, VEC> acc;
            acc.zero();
            int cur = 0;
            bool waited = false;
            for (uint32_t cb = e_begin; cb < e_end; cb += 32) {
                const int cnt = (e_end - cb < 32u) ? (int)(e_end - cb) : 32;
                int32_t mycol = 0;
                T myval = T(0);
                if (lane < cnt) {
                    mycol = __ldcs(ent_col + cb + lane);
                    myval = __ldcs(ent_val + cb + lane);
                }
                const uint32_t rel = my_end - 1u - cb;
                const unsigned endmask = __reduce_or_sync(0xffffffffu, (rel < 32u) ? (1u << rel) : 0u);
#pragma unroll 1
                for (int u0 = 0; u0 < cnt; u0 += UNROLL) {
                    const int n = min(cnt - u0, UNROLL);
                    const unsigned grp = (endmask >> u0) & ((1u << UNROLL) - 1u);
                    Frag<T, VEC> xv[UNROLL];
                    T av[UNROLL];
#pragma unroll
                    for (int t = 0; t < UNROLL; ++t) {
                        const int32_t col = __shfl_sync(0xffffffffu, mycol, (u0 + t) & 31);
                        av[t] = __shfl_sync(0xffffffffu, myval, (u0 + t) & 31);
                        const char *p;
                        if (OFF32) p = Xc + (uint32_t)((uint32_t)col * rowbytes + lane_off);
                        else p = Xc + (uint64_t)(uint32_t)col * rowbytes + lane_off;
                        if (t < n) xv[t] = ld_x<T, VEC>(reinterpret_cast<const T *>(p));
                    }
                    if (n == UNROLL && grp == 0u) {
#pragma unroll
                        for (int t = 0; t < UNROLL; ++t)
#pragma unroll
                            for (int i = 0; i < VEC; ++i) acc.v[i] = fma(av[t], xv[t].v[i], acc.v[i]);
                        continue;
                    }
#pragma unroll
                    for (int t = 0; t < UNROLL; ++t) {
                        if (t < n) {
#pragma unroll
                            for (int i = 0; i < VEC; ++i) acc.v[i] = fma(av[t], xv[t].v[i], acc.v[i]);
                        }
                        if ((grp >> t) & 1u) {
                            const int32_t o = __shfl_sync(0xffffffffu, my_out, cur);
                            if (o < 0) {
                                atomic_add_frag<T, VEC>(Y + (int64_t)(o & 0x7fffffff) * k + col0, acc);
                            } else {
                                if (!waited) {
                                    asm volatile("cp.async.wait_all;" ::: "memory");
                                    waited = true;
                                }
                                Frag<T, VEC> y;
                                const V sv = stage[wid][cur][lane];
                                memcpy(&y, &sv, sizeof(V));
#pragma unroll
                                for (int i = 0; i < VEC; ++i) y.v[i] += acc.v[i];
                                if ((o & kFinalBit) && outs.act) apply_act<T, VEC>(y, outs.act);
                                st_plain<T, VEC>(Y + (int64_t)(o & kRowMask30) * k + col0, y);
                            }
                            acc.zero();
                            ++cur;
                        }
                    }
                }
            }
            if (!waited) asm volatile("cp.async.wait_all;" ::: "memory");  // never leave copies in flight
            __syncwarp();
        }
    }
}

template <typename T, int VEC>
int run_tail32(const SegLevel &L, const void *X, void *Y, int64_t k, int num_sms, unsigned *counter,
               const PeerPtrs &outs, bool off32, cudaStream_t st) {
    constexpr int STAGE = 8;
    auto kern = off32 ? k_tail32<T, VEC, true, STAGE> : k_tail32<T, VEC, false, STAGE>;
    static int bps[2] = {0, 0};
    int &b = bps[off32 ? 1 : 0];
    if (b == 0) {
        // 4 blocks x 32 KB of stage per SM: ask for the shared-memory carveout that holds them
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 256, 0);
        if (std::getenv("ARROW_TAIL_STAGE_VERBOSE")) fprintf(stderr, "k_tail32: %d blocks/SM\n", b);
        if (b <= 0) b = 1;
    }
    const int64_t nbatch = (L.nseg + STAGE - 1) / STAGE;
    int64_t blocks = std::min<int64_t>((int64_t)num_sms * b, (nbatch + 7) / 8);
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, 256, 0, st>>>(L.seg_out, L.seg_end, L.nseg, L.ent_col,
                                           reinterpret_cast<const T *>(L.ent_val), reinterpret_cast<const T *>(X),
                                           reinterpret_cast<T *>(Y), k, counter, outs);
    return (int)cudaGetLastError();
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
        if (MODE == 1 && DIST == 0) prefetch_y_rows<T>(outs.ypf, my_out, lane < nb, Y, k);

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
    // entry prefetch + whole-chunk row loads (ARROW_SEG_PF=0: the earlier 4-step groups)
    static const bool pf = !(std::getenv("ARROW_SEG_PF") && std::getenv("ARROW_SEG_PF")[0] == '0');
    auto kern = pf ? (off32 ? k_segsmall<T, VEC, LPE, MODE, DIST, true, true> : k_segsmall<T, VEC, LPE, MODE, DIST, false, true>)
                   : (off32 ? k_segsmall<T, VEC, LPE, MODE, DIST, true, false> : k_segsmall<T, VEC, LPE, MODE, DIST, false, false>);
    static int bps[4] = {0, 0, 0, 0};
    int &b = bps[(off32 ? 1 : 0) + (pf ? 2 : 0)];
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

static bool narrow_k32() {
    static const bool v = std::getenv("ARROW_SEG_K32") && std::string(std::getenv("ARROW_SEG_K32")) == "narrow";
    return v;
}

int launch_seg(int dtype, int dist, const SegLevel &L, const void *X, const void *D0, void *Y, void *C0, int64_t k,
               int num_sms, unsigned *counter, int bseg, void *stream, const PeerPtrs *outs, int act,
               const int32_t *zrows, int64_t nzero) {
    using namespace kseg;
    if (k == 0) return 0;
    if (L.nseg == 0) return nzero > 0 ? launch_zero_rows(dtype, zrows, nzero, k, Y, stream) : 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    PeerPtrs po{};
    if (outs) po = *outs;
    po.act = act;
    if (!dist && nzero > 0) {
        po.zrows = zrows;
        po.nzero = nzero;
    }
    // L2 prefetch of the batch's Y rows in the levels >= 1 of the short-row kernel (measured 1-2 %
    // faster at k = 8/32 and on G; ARROW_SEG_YPF=0 disables)
    static const bool ypf = !(std::getenv("ARROW_SEG_YPF") && std::getenv("ARROW_SEG_YPF")[0] == '0');
    po.ypf = (!dist && ypf) ? 1 : 0;
    if (dist == 2 && !outs) return (int)cudaErrorInvalidValue;
    int vec = dist ? pick_vec(dtype, k, {X, Y, D0, C0}) : pick_vec(dtype, k, {X, Y});
    if (dist == 2)
        for (const void *p : po.p) vec = std::min(vec, pick_vec(dtype, k, {p}));
    const int lpe = pick_lpe(k, vec);
    // full-warp rows: the staged-entry kernel (ARROW_SEG32=0 keeps the generic one)
    static const bool seg32 = !(std::getenv("ARROW_SEG32") && std::getenv("ARROW_SEG32")[0] == '0');
    // 32-bit X offsets when every X row offset (and D0's) fits
    const bool off32 = (uint64_t)L.max_x_row * (uint64_t)k * (dtype == 1 ? 8u : 4u) < (1ull << 32) - (1ull << 20);
    // levels >= 1, single GPU, full-warp rows: Y slabs staged by cp.async (ARROW_TAIL_STAGE=1; measured
    // slower on config R, 3.58 vs 2.86 ms: level 1 757 vs 506 us at 2.4 TB/s -- off by default)
    static const bool tail_stage = std::getenv("ARROW_TAIL_STAGE") && std::getenv("ARROW_TAIL_STAGE")[0] == '1';
    if (seg32 && tail_stage && dist == 0 && L.mode == 1 && lpe == 32 && k % (32 * vec) == 0) {
        if (dtype == 0 && vec == 4) return run_tail32<float, 4>(L, X, Y, k, num_sms, counter, po, off32, st);
        if (dtype == 1 && vec == 2) return run_tail32<double, 2>(L, X, Y, k, num_sms, counter, po, off32, st);
    }
    if (seg32 && lpe == 32 && k % (32 * vec) == 0) {
        if (dtype == 0 && vec == 4)
            return run_seg32_mode<float, 4>(dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, po, off32, st);
        if (dtype == 1 && vec == 2)
            return run_seg32_mode<double, 2>(dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, po, off32, st);
    }
    // short rows (k = 8/16/32 fp32 -- 32 one row per warp with ARROW_SEG_K32=narrow --, 4/8/16/32
    // fp64 with 16-byte lanes): G entries per warp step,
    // segmented scan across the sub-warps (ARROW_SEG_SMALL=0 disables)
    static const bool small = !(std::getenv("ARROW_SEG_SMALL") && std::getenv("ARROW_SEG_SMALL")[0] == '0');
    if (seg32 && small && lpe < 32 && lpe >= 2 && k == (int64_t)lpe * vec && vec == 16 / (dtype == 1 ? 8 : 4) &&
        !(dtype == 0 && lpe == 8 && narrow_k32())) {
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
    // fp32 rows of 32 or 64 elements: one row per warp with 4- or 8-byte lanes (one 128/256-byte
    // request per entry) instead of 8/16-lane sub-warps that run different batches in lockstep
    static const bool narrow = !(std::getenv("ARROW_SEG_NARROW") && std::getenv("ARROW_SEG_NARROW")[0] == '0');
    if (seg32 && narrow && dtype == 0 && (k == 32 || k == 64) && vec >= k / 32)
        return k == 64 ? run_seg32_mode<float, 2>(dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, po, off32, st)
                       : run_seg32_mode<float, 1>(dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, po, off32, st);
    if (dtype == 0) {
        if (vec == 4) return run_segments_mode<float, 4>(lpe, dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, po, st);
        if (vec == 2) return run_segments_mode<float, 2>(lpe, dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, po, st);
        return run_segments_mode<float, 1>(lpe, dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, po, st);
    }
    if (vec == 2) return run_segments_mode<double, 2>(lpe, dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, po, st);
    return run_segments_mode<double, 1>(lpe, dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, po, st);
}

}  // namespace arrow
