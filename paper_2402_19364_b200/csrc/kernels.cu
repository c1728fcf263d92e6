// kernels.cu -- the hot path of arrow_spmm on sm_100a (B200).
//
// Per level i of the decomposition A X = sum_i P_{pi_i} (B_i (P_{pi_i}^T X))  (Eq. (1)):
//   K-H  head stage      D0 = X[head_i] (Alg. 1 line 1 "Broadcast(D^(0))"), C0 = 0
//   K-A  segment stream  body rows  y_p = B^(p,0) D0 + B^(p,p) X_p  -> Y[perm_i[p]] (store at level 0,
//                        read-modify-write at levels >= 1: Alg. 2's reverse aggregation)
//                        head rows  C0[j] += B^(0,t) X_t, one tile window t at a time (Alg. 1 line 2,
//                        P:464), combined with fp atomics in L2 (C0 is L2-resident)
//   K-C  head epilogue   Y[head_i] (= or +=) C0 (Alg. 1 line 3 "Reduce(C^(0))")
// The permutations P_pi^T X / P_pi Y are folded into the column and output indices at plan
// time (S4): no permuted copy of X or Y ever exists.
//
// The path is HBM-bound (<= 2 FLOP/B), so there are no tensor cores: the design
// goal is that every X row of a tile is fetched from DRAM once (window-ordered work keeps the
// tile's rows L2-hot while all its users run) and that each warp keeps many 16-byte loads in
// flight.  A "sub-warp" of LPE lanes owns one row slab of LPE*VEC elements: LPE=32 lanes x float4
// covers a 512-byte row (k=128 fp32) with one coalesced request per entry.
#include <cuda_runtime.h>
#include <cstdint>

#include "arrow_internal.h"

namespace arrow {
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
template <typename T, int VEC, int LPE, int MODE, int DIST>
__global__ void __launch_bounds__(256, 4) k_segments(const int32_t *__restrict__ seg_out,
                                                     const uint32_t *__restrict__ seg_end, int64_t nseg,
                                                     const int32_t *__restrict__ ent_col,
                                                     const T *__restrict__ ent_val, const T *__restrict__ X,
                                                     const T *__restrict__ D0, T *__restrict__ Y,
                                                     T *__restrict__ C0, int64_t k, unsigned *__restrict__ counter,
                                                     int bseg) {
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
                                } else if (MODE == 0) {
                                    st_stream<T, VEC>(Y + (int64_t)o * k + col0, acc);
                                } else {
                                    T *py = Y + (int64_t)o * k + col0;
                                    Frag<T, VEC> y = ld_plain<T, VEC>(py);
#pragma unroll
                                    for (int i = 0; i < VEC; ++i) y.v[i] += acc.v[i];
                                    st_plain<T, VEC>(py, y);
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

// K-Z: zero the listed Y rows (level 0: head rows, which then accumulate head slices atomically,
// and rows with no entry in B_0, incl. A-isolated vertices).
template <typename T, int VEC>
__global__ void __launch_bounds__(256) k_zero_rows(const int32_t *__restrict__ rows, int64_t nrows, int64_t k,
                                                   T *__restrict__ Y) {
    const int64_t kv = k / VEC, total = nrows * kv;
    Frag<T, VEC> z;
    z.zero();
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / kv, c = (t - j * kv) * VEC;
        st_stream<T, VEC>(Y + (int64_t)__ldg(rows + j) * k + c, z);
    }
}

// ------------------------------------------------------------------------------------ K-H / K-C
template <typename T, int VEC>
__global__ void __launch_bounds__(256) k_head_stage(const T *__restrict__ X, const int32_t *__restrict__ head,
                                                    int64_t h, int64_t k, T *__restrict__ D0, T *__restrict__ C0) {
    const int64_t kv = k / VEC, total = h * kv;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / kv, c = (t - j * kv) * VEC;
        const Frag<T, VEC> x = ld_x<T, VEC>(X + (int64_t)__ldg(head + j) * k + c);
        st_plain<T, VEC>(D0 + j * k + c, x);
        Frag<T, VEC> z;
        z.zero();
        st_plain<T, VEC>(C0 + j * k + c, z);
    }
}

template <typename T, int VEC>
__global__ void __launch_bounds__(256) k_head_epilogue(const T *__restrict__ C0, const int32_t *__restrict__ head,
                                                       int64_t h, int64_t k, int add, T *__restrict__ Y) {
    const int64_t kv = k / VEC, total = h * kv;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / kv, c = (t - j * kv) * VEC;
        Frag<T, VEC> a = ld_plain<T, VEC>(C0 + j * k + c);
        T *p = Y + (int64_t)__ldg(head + j) * k + c;
        if (add) {
            Frag<T, VEC> y = ld_plain<T, VEC>(p);
#pragma unroll
            for (int i = 0; i < VEC; ++i) a.v[i] += y.v[i];
        }
        st_plain<T, VEC>(p, a);
    }
}

// ------------------------------------------------------------------------------------ dispatch
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

template <typename T, int VEC, int LPE, int MODE, int DIST>
int run_segments(const DeviceLevel &L, const void *X, const void *D0, void *Y, void *C0, int64_t k, int num_sms,
                 unsigned *counter, int bseg, cudaStream_t st) {
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
                                            reinterpret_cast<T *>(C0), k, counter, bseg);
    return (int)cudaGetLastError();
}

template <typename T, int VEC, int MODE, int DIST>
int run_segments_lpe(int lpe, const DeviceLevel &L, const void *X, const void *D0, void *Y, void *C0, int64_t k,
                     int num_sms, unsigned *counter, int bseg, cudaStream_t st) {
    switch (lpe) {
        case 32: return run_segments<T, VEC, 32, MODE, DIST>(L, X, D0, Y, C0, k, num_sms, counter, bseg, st);
        case 16: return run_segments<T, VEC, 16, MODE, DIST>(L, X, D0, Y, C0, k, num_sms, counter, bseg, st);
        case 8: return run_segments<T, VEC, 8, MODE, DIST>(L, X, D0, Y, C0, k, num_sms, counter, bseg, st);
        case 4: return run_segments<T, VEC, 4, MODE, DIST>(L, X, D0, Y, C0, k, num_sms, counter, bseg, st);
        case 2: return run_segments<T, VEC, 2, MODE, DIST>(L, X, D0, Y, C0, k, num_sms, counter, bseg, st);
        default: return run_segments<T, VEC, 1, MODE, DIST>(L, X, D0, Y, C0, k, num_sms, counter, bseg, st);
    }
}

template <typename T, int VEC>
int run_segments_mode(int lpe, int dist, const DeviceLevel &L, const void *X, const void *D0, void *Y, void *C0,
                      int64_t k, int num_sms, unsigned *counter, int bseg, cudaStream_t st) {
    if (dist) {
        return L.mode == 0 ? run_segments_lpe<T, VEC, 0, 1>(lpe, L, X, D0, Y, C0, k, num_sms, counter, bseg, st)
                           : run_segments_lpe<T, VEC, 1, 1>(lpe, L, X, D0, Y, C0, k, num_sms, counter, bseg, st);
    }
    return L.mode == 0 ? run_segments_lpe<T, VEC, 0, 0>(lpe, L, X, D0, Y, C0, k, num_sms, counter, bseg, st)
                       : run_segments_lpe<T, VEC, 1, 0>(lpe, L, X, D0, Y, C0, k, num_sms, counter, bseg, st);
}

inline unsigned grid_for(int64_t total) {
    int64_t g = (total + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    return (unsigned)g;
}

}  // namespace

int launch_segments(int dtype, int dist, const DeviceLevel &L, const void *X, const void *D0, void *Y, void *C0,
                    int64_t k, int num_sms, unsigned *counter, int bseg, void *stream) {
    if (L.nseg == 0 || k == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int vec = dist ? pick_vec(dtype, k, {X, Y, D0, C0}) : pick_vec(dtype, k, {X, Y});
    const int lpe = pick_lpe(k, vec);
    if (dtype == 0) {
        if (vec == 4) return run_segments_mode<float, 4>(lpe, dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, st);
        if (vec == 2) return run_segments_mode<float, 2>(lpe, dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, st);
        return run_segments_mode<float, 1>(lpe, dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, st);
    }
    if (vec == 2) return run_segments_mode<double, 2>(lpe, dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, st);
    return run_segments_mode<double, 1>(lpe, dist, L, X, D0, Y, C0, k, num_sms, counter, bseg, st);
}

int launch_zero_rows(int dtype, const int32_t *rows, int64_t nrows, int64_t k, void *Y, void *stream) {
    if (nrows == 0 || k == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int vec = pick_vec(dtype, k, {Y});
    const unsigned g = grid_for(nrows * (k / vec));
    if (dtype == 0) {
        if (vec == 4) k_zero_rows<float, 4><<<g, 256, 0, st>>>(rows, nrows, k, (float *)Y);
        else if (vec == 2) k_zero_rows<float, 2><<<g, 256, 0, st>>>(rows, nrows, k, (float *)Y);
        else k_zero_rows<float, 1><<<g, 256, 0, st>>>(rows, nrows, k, (float *)Y);
    } else {
        if (vec == 2) k_zero_rows<double, 2><<<g, 256, 0, st>>>(rows, nrows, k, (double *)Y);
        else k_zero_rows<double, 1><<<g, 256, 0, st>>>(rows, nrows, k, (double *)Y);
    }
    return (int)cudaGetLastError();
}

int launch_head_stage(int dtype, const void *X, const int32_t *head_rows, int64_t h, int64_t k, void *D0, void *C0,
                      void *stream) {
    if (h == 0 || k == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int vec = pick_vec(dtype, k, {X, D0, C0});
    const unsigned g = grid_for(h * (k / vec));
    if (dtype == 0) {
        if (vec == 4) k_head_stage<float, 4><<<g, 256, 0, st>>>((const float *)X, head_rows, h, k, (float *)D0, (float *)C0);
        else if (vec == 2) k_head_stage<float, 2><<<g, 256, 0, st>>>((const float *)X, head_rows, h, k, (float *)D0, (float *)C0);
        else k_head_stage<float, 1><<<g, 256, 0, st>>>((const float *)X, head_rows, h, k, (float *)D0, (float *)C0);
    } else {
        if (vec == 2) k_head_stage<double, 2><<<g, 256, 0, st>>>((const double *)X, head_rows, h, k, (double *)D0, (double *)C0);
        else k_head_stage<double, 1><<<g, 256, 0, st>>>((const double *)X, head_rows, h, k, (double *)D0, (double *)C0);
    }
    return (int)cudaGetLastError();
}

int launch_head_epilogue(int dtype, const void *C0, const int32_t *head_rows, int64_t h, int64_t k, int add, void *Y,
                         void *stream) {
    if (h == 0 || k == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int vec = pick_vec(dtype, k, {C0, Y});
    const unsigned g = grid_for(h * (k / vec));
    if (dtype == 0) {
        if (vec == 4) k_head_epilogue<float, 4><<<g, 256, 0, st>>>((const float *)C0, head_rows, h, k, add, (float *)Y);
        else if (vec == 2) k_head_epilogue<float, 2><<<g, 256, 0, st>>>((const float *)C0, head_rows, h, k, add, (float *)Y);
        else k_head_epilogue<float, 1><<<g, 256, 0, st>>>((const float *)C0, head_rows, h, k, add, (float *)Y);
    } else {
        if (vec == 2) k_head_epilogue<double, 2><<<g, 256, 0, st>>>((const double *)C0, head_rows, h, k, add, (double *)Y);
        else k_head_epilogue<double, 1><<<g, 256, 0, st>>>((const double *)C0, head_rows, h, k, add, (double *)Y);
    }
    return (int)cudaGetLastError();
}

int launch_zero(void *Y, int64_t bytes, void *stream) {
    if (bytes == 0) return 0;
    return (int)cudaMemsetAsync(Y, 0, (size_t)bytes, reinterpret_cast<cudaStream_t>(stream));
}

}  // namespace arrow
