// stream_kernel.cuh -- K-A, the per-level SpMM of the arrow path (S1 body rows, S2 head slices,
// S4 folded permutations, S5 store/RMW), as one "record stream" kernel for sm_100a.
//
// PAPER.md Alg. 1: C^(r) = B^(r,0) D^(0) + B^(r,r) D^(r) for body tiles and
// C^(0) = sum_t B^(0,t) D^(t) for the head rows; Alg. 2 / Eq. (1): Y = sum_i P_i B_i P_i^T X.
//
// Encoding (built by arrow_api.cpp, see arrow_internal.h): a level is one array of records
// (key, val) in tile-window order.  A plain record (bit 31 clear) is a nonzero: key's low 30 bits
// are the X row to read (the permutation is folded in), bit 30 selects the staged head block D0
// instead (distributed mode).  A pseudo record (bit 31 set) closes the current output segment:
// low 30 bits = output row, bit 30 = "add atomically" (head-row partial of one window: into Y on
// one GPU, into C0 in distributed mode); otherwise store (level 0) or read-modify-write (>= 1).
// The stream is cut into batches at pseudo records; warps grab batches from a per-launch counter,
// so all resident warps work on a narrow front of the window-ordered stream and the window's X
// rows stay L2-resident while all their users run (IO lemma).
//
// Mapping: a sub-warp of LPE lanes owns one stream; each lane holds NV vectors of VB bytes of the
// output row, interleaved so that every load instruction covers LPE*VB contiguous bytes of a row.
// k=128 fp32: LPE=8, NV=4, VB=16 -> 4 independent streams per warp, one warp instruction serves 4
// nonzeros.  Loads are software-pipelined through a ring of D register slots: record r is issued
// D records before it is consumed, across segment boundaries, so each stream keeps D rows in
// flight continuously.  fp32 FMAs use the packed FFMA2 (fma.rn.f32x2).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace arrow {
namespace ks {

constexpr uint32_t kPseudo = 0x80000000u;
constexpr uint32_t kAux = 0x40000000u;
constexpr uint32_t kRowMask = 0x3fffffffu;

template <int VB> struct Raw;
template <> struct Raw<16> { using type = uint4; };
template <> struct Raw<8> { using type = uint2; };
template <> struct Raw<4> { using type = uint32_t; };

template <typename T, int VB> struct Vec {
    static constexpr int N = VB / (int)sizeof(T);
    T v[N];
};

template <typename T, int VB>
__device__ __forceinline__ Vec<T, VB> ldg_vec(const char *p) {
    using R = typename Raw<VB>::type;
    R r = __ldg(reinterpret_cast<const R *>(p));
    Vec<T, VB> out;
    memcpy(&out, &r, VB);
    return out;
}

// Predicated read-only load into `dst` (unchanged when !pred).  Written as one PTX instruction
// with read-write operands so that every pipeline slot keeps its own registers: a C++
// "if (pred) dst = load" makes the compiler merge through a temporary and wait on the load.
template <typename T, int VB>
__device__ __forceinline__ void ldg_vec_pred(bool pred, const char *p, Vec<T, VB> &dst) {
    if constexpr (VB == 16) {
        uint32_t *r = reinterpret_cast<uint32_t *>(&dst);
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
                     "@q ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}"
                     : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3])
                     : "l"(p), "r"((int)pred));
    } else if constexpr (VB == 8) {
        uint32_t *r = reinterpret_cast<uint32_t *>(&dst);
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t"
                     "@q ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];\n\t}"
                     : "+r"(r[0]), "+r"(r[1])
                     : "l"(p), "r"((int)pred));
    } else {
        uint32_t *r = reinterpret_cast<uint32_t *>(&dst);
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
                     "@q ld.global.nc.L1::no_allocate.u32 %0, [%1];\n\t}"
                     : "+r"(r[0])
                     : "l"(p), "r"((int)pred));
    }
}

// Predicated coherent streaming load (evict-first) of a Y row that this warp will rewrite.
template <typename T, int VB>
__device__ __forceinline__ void ld_vec_pred_cs(bool pred, const char *p, Vec<T, VB> &dst) {
    static_assert(VB == 16, "16-byte rows only");
    uint32_t *r = reinterpret_cast<uint32_t *>(&dst);
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
                 "@q ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3])
                 : "l"(p), "r"((int)pred));
}

template <typename T, int VB>
__device__ __forceinline__ Vec<T, VB> ld_vec(const char *p) {
    using R = typename Raw<VB>::type;
    R r = *reinterpret_cast<const R *>(p);
    Vec<T, VB> out;
    memcpy(&out, &r, VB);
    return out;
}

// streaming (evict-first) load of a Y row that is read once and rewritten (levels >= 1)
template <typename T, int VB>
__device__ __forceinline__ Vec<T, VB> ld_vec_stream(const char *p) {
    using R = typename Raw<VB>::type;
    R r = __ldcs(reinterpret_cast<const R *>(p));
    Vec<T, VB> out;
    memcpy(&out, &r, VB);
    return out;
}

template <typename T, int VB>
__device__ __forceinline__ void st_vec(char *p, const Vec<T, VB> &v) {
    using R = typename Raw<VB>::type;
    R r;
    memcpy(&r, &v, VB);
    *reinterpret_cast<R *>(p) = r;
}

template <typename T, int VB>
__device__ __forceinline__ void st_vec_stream(char *p, const Vec<T, VB> &v) {
    using R = typename Raw<VB>::type;
    R r;
    memcpy(&r, &v, VB);
    __stcs(reinterpret_cast<R *>(p), r);
}

template <typename T, int VB>
__device__ __forceinline__ void zero(Vec<T, VB> &a) {
#pragma unroll
    for (int i = 0; i < Vec<T, VB>::N; ++i) a.v[i] = T(0);
}

// acc += a * x.  The packed FFMA2 (fma.rn.f32x2) halves the FMA instructions but makes ptxas
// allocate the row registers as 64-bit pairs, which breaks the aligned quads LDG.128 writes and
// serialises the load pipeline; plain FFMA keeps the loads landing in their slots.
constexpr bool kUseFfma2 = false;
template <typename T, int VB>
__device__ __forceinline__ void fma_vec(Vec<T, VB> &acc, T a, const Vec<T, VB> &x) {
    constexpr int N = Vec<T, VB>::N;
    if constexpr (kUseFfma2 && sizeof(T) == 4 && (N % 2) == 0) {
#pragma unroll
        for (int i = 0; i < N; i += 2) {
            uint64_t c, xb;
            memcpy(&c, &acc.v[i], 8);
            memcpy(&xb, &x.v[i], 8);
            const float2 aa = make_float2(a, a);
            uint64_t ab;
            memcpy(&ab, &aa, 8);
            asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(ab), "l"(xb));
            memcpy(&acc.v[i], &c, 8);
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) acc.v[i] = fma(a, x.v[i], acc.v[i]);
    }
}

template <typename T, int VB>
__device__ __forceinline__ void red_vec(char *p, const Vec<T, VB> &v) {
    constexpr int N = Vec<T, VB>::N;
    if constexpr (sizeof(T) == 4 && N == 4) {
        atomicAdd(reinterpret_cast<float4 *>(p), make_float4(v.v[0], v.v[1], v.v[2], v.v[3]));
    } else if constexpr (sizeof(T) == 4 && N == 2) {
        atomicAdd(reinterpret_cast<float2 *>(p), make_float2(v.v[0], v.v[1]));
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) atomicAdd(reinterpret_cast<T *>(p) + i, v.v[i]);
    }
}

template <typename T, int LPE, int NV, int VB, int D, int MODE, int DIST>
__global__ void __launch_bounds__(256, (NV * D * VB / 4 > 48) ? 2 : 3)
k_stream(const uint32_t *__restrict__ keys, const T *__restrict__ vals, const uint32_t *__restrict__ bstart,
         int64_t nbatch, const T *__restrict__ X, const T *__restrict__ D0, T *__restrict__ Y, T *__restrict__ C0,
         int64_t k, unsigned *__restrict__ counter) {
    using V = Vec<T, VB>;
    constexpr int SUBS = 32 / LPE;
    constexpr int EPV = V::N;                  // elements per vector
    constexpr int SLAB = LPE * NV * EPV;       // elements per slab
    const int lane = threadIdx.x & 31;
    const int sl = lane % LPE;
    const int sub = lane / LPE;
    const unsigned mask = (LPE == 32) ? 0xffffffffu : (((1u << LPE) - 1u) << (sub * LPE));
    const uint32_t rowbytes = (uint32_t)(k * (int64_t)sizeof(T));   // < 2^32 (checked on the host)

    for (;;) {
        unsigned wb = 0;
        if (lane == 0) wb = atomicAdd(counter, 1u);
        wb = __shfl_sync(0xffffffffu, wb, 0);
        if ((int64_t)wb * SUBS >= nbatch) break;            // warp-uniform exit
        // The SUBS sub-warps of a warp run their streams in lockstep: the same relative record
        // index every step, so chunk refills and shuffles are warp-uniform and per-stream
        // differences are lane predicates, not divergent branches.
        const int64_t bt = (int64_t)wb * SUBS + sub;
        uint32_t r0 = 0, r1 = 0;
        if (bt < nbatch) { r0 = __ldg(bstart + bt); r1 = __ldg(bstart + bt + 1); }
        const int len = (int)(r1 - r0);
        const int maxlen = (SUBS == 1) ? len : (int)__reduce_max_sync(0xffffffffu, (unsigned)len);

        for (int64_t c0 = 0; c0 < k; c0 += SLAB) {
            bool act[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) act[v] = c0 + (int64_t)(v * LPE + sl) * EPV < k;
            const int64_t lane_off = (c0 + (int64_t)sl * EPV) * (int64_t)sizeof(T);  // bytes
            const char *xl = reinterpret_cast<const char *>(X) + lane_off;
            const char *dl = reinterpret_cast<const char *>(D0) + lane_off;
            V acc[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) zero<T, VB>(acc[v]);

            // record chunks: lane sl holds record cb + sl (cur) and cb + LPE + sl (nxt) of its stream
            int cb = 0;
            uint32_t ckey = kPseudo, nkey = kPseudo;
            T cval = T(0), nval = T(0);
            if (sl < len) { ckey = __ldcs(keys + r0 + sl); cval = __ldcs(vals + r0 + sl); }
            if (LPE + sl < len) { nkey = __ldcs(keys + r0 + LPE + sl); nval = __ldcs(vals + r0 + LPE + sl); }

            uint32_t skey[D];
            T sval[D];
            V xs[D][NV];
#pragma unroll
            for (int d = 0; d < D; ++d) skey[d] = 0;

            // Two ping-pong groups of G = D/2 slots: consume a whole group (its loads were issued
            // together, so one scoreboard wait covers them), then refill it D records ahead while
            // the other group's loads stay in flight.
            constexpr int G = D / 2;
            for (int base = 0; base < maxlen + D; base += D) {
#pragma unroll
                for (int half = 0; half < 2; ++half) {
#pragma unroll
                    for (int t = 0; t < G; ++t) {
                        const int d = half * G + t;
                        const int r = base + d;
                        // ---- consume record r - D of this stream from slot d
                        const bool live = (r >= D) && (r - D < len);
                        const uint32_t key = skey[d];
                        if (live && !(key & kPseudo)) {
#pragma unroll
                            for (int v = 0; v < NV; ++v) fma_vec<T, VB>(acc[v], sval[d], xs[d][v]);
                        }
                        if (live && (key & kPseudo)) {
                            const uint32_t row = key & kRowMask;
                            if (key & kAux) {
                                char *dst = reinterpret_cast<char *>(DIST ? C0 : Y) + (uint64_t)row * rowbytes + lane_off;
#pragma unroll
                                for (int v = 0; v < NV; ++v)
                                    if (act[v]) red_vec<T, VB>(dst + v * LPE * VB, acc[v]);
                            } else {
                                char *dst = reinterpret_cast<char *>(Y) + (uint64_t)row * rowbytes + lane_off;
#pragma unroll
                                for (int v = 0; v < NV; ++v) {
                                    if (!act[v]) continue;
                                    if (MODE == 0) {
                                        st_vec_stream<T, VB>(dst + v * LPE * VB, acc[v]);
                                    } else {
                                        V y = ld_vec<T, VB>(dst + v * LPE * VB);
#pragma unroll
                                        for (int i = 0; i < EPV; ++i) y.v[i] += acc[v].v[i];
                                        st_vec<T, VB>(dst + v * LPE * VB, y);
                                    }
                                }
                            }
#pragma unroll
                            for (int v = 0; v < NV; ++v) zero<T, VB>(acc[v]);
                        }
                    }
#pragma unroll
                    for (int t = 0; t < G; ++t) {
                        const int d = half * G + t;
                        const int r = base + d;
                        // ---- issue record r into slot d
                        if (r < maxlen) {                          // warp-uniform
                            if (r - cb == LPE) {                   // advance the record chunk (warp-uniform)
                                cb += LPE;
                                ckey = nkey;
                                cval = nval;
                                nkey = kPseudo;
                                nval = T(0);
                                if (cb + LPE + sl < len) {
                                    nkey = __ldcs(keys + r0 + cb + LPE + sl);
                                    nval = __ldcs(vals + r0 + cb + LPE + sl);
                                }
                            }
                            const uint32_t kk = __shfl_sync(0xffffffffu, ckey, r - cb, LPE);
                            const T vv = __shfl_sync(0xffffffffu, cval, r - cb, LPE);
                            skey[d] = kk;
                            sval[d] = vv;
                            const bool ld = r < len && !(kk & kPseudo);
                            const char *p = ((DIST && (kk & kAux)) ? dl : xl) + (uint64_t)(kk & kRowMask) * (uint64_t)rowbytes;
#pragma unroll
                            for (int v = 0; v < NV; ++v) ldg_vec_pred<T, VB>(ld && act[v], p + v * LPE * VB, xs[d][v]);
                        }
                    }
                }
            }
        }
    }
}

}  // namespace ks
}  // namespace arrow
