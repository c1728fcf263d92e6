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
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

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

// K-Z: zero the listed Y rows (level 0: head rows, which then accumulate head slices atomically,
// and rows with no entry in B_0, incl. A-isolated vertices).
template <typename T, int VEC>
__global__ void __launch_bounds__(256) k_zero_rows(const int32_t *__restrict__ rows, int64_t nrows, int64_t k,
                                                   T *__restrict__ Y) {
    // one warp per row, 4 rows per warp pass (streaming stores)
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    Frag<T, VEC> z;
    z.zero();
    for (int64_t r0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 4; r0 < nrows; r0 += nw * 4) {
        int64_t row[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) row[t] = (r0 + t < nrows) ? (int64_t)__ldg(rows + r0 + t) : -1;
        for (int64_t c = (int64_t)lane * VEC; c < k; c += 32 * VEC)
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (row[t] >= 0) st_stream<T, VEC>(Y + row[t] * k + c, z);
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

inline unsigned grid_for(int64_t total) {
    int64_t g = (total + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    return (unsigned)g;
}

}  // namespace

StreamCfg pick_stream_cfg(int dtype, int64_t k, const void *X, const void *Y, const void *D0, const void *C0) {
    const int es = dtype == 1 ? 8 : 4;
    const int64_t rb = k * es;
    auto aligned = [&](int a) {
        for (const void *p : {X, Y, D0, C0})
            if (p && (reinterpret_cast<uintptr_t>(p) % a) != 0) return false;
        return true;
    };
    int vb = 4;
    if (rb % 16 == 0 && aligned(16)) vb = 16;
    else if (rb % 8 == 0 && aligned(8)) vb = 8;
    if (vb < es) vb = es;
    const int64_t rv = rb / vb;  // vectors per row
    StreamCfg c{vb, 1, 1, 8};
    if (vb == 16) {
        if (rv >= 17) c = {16, 8, 4, 4};
        else if (rv >= 9) c = {16, 4, 4, 4};
        else if (rv >= 5) c = {16, 2, 4, 4};
        else if (rv >= 3) c = {16, 1, 4, 4};
        else c = {16, 1, 1, 8};
    } else {
        if (rv >= 17) c = {vb, 32, 1, 8};
        else if (rv >= 3) c = {vb, 8, 1, 8};
        else c = {vb, 1, 1, 8};
    }
    // experiment hook: ARROW_KA_CFG="lpe,nv,d" for 16-byte rows (must be an instantiated config)
    if (vb == 16) {
        if (const char *e = std::getenv("ARROW_KA_CFG")) {
            int l = 0, nv = 0, d = 0;
            if (std::sscanf(e, "%d,%d,%d", &l, &nv, &d) == 3) c = {16, l, nv, d};
        }
    }
    return c;
}

int launch_stream(int dtype, int dist, const DeviceLevel &L, const void *X, const void *D0, void *Y, void *C0,
                  int64_t k, int num_sms, unsigned *counter, void *stream) {
    if (L.nbatch == 0 || k == 0) return 0;
    StreamArgs a{L.keys, L.vals, L.bstart, L.nbatch, X, D0, Y, C0, k, counter, num_sms, L.mode, dist};
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    // TMA bulk-gather kernel when rows are 16-byte multiples of at most 1 KiB on 16-byte aligned
    // buffers; otherwise the register-pipelined record-stream kernel.
    const int es = dtype == 1 ? 8 : 4;
    const int64_t rb = k * es;
    bool tma = rb % 16 == 0 && rb <= 1024;
    for (const void *p : {X, (const void *)Y, D0, (const void *)C0})
        if (p && (reinterpret_cast<uintptr_t>(p) % 16) != 0) tma = false;
    // kernel choice: ARROW_KA=rec (default for 16-byte rows <= 1 KiB), tma, stream
    const char *ka = std::getenv("ARROW_KA");
    const std::string kas = ka ? ka : "seg";
    StreamCfg c = pick_stream_cfg(dtype, k, X, Y, dist ? D0 : nullptr, dist ? C0 : nullptr);
    if (tma && kas == "rec") c = StreamCfg{16, -1, 0, 0};
    else if (tma && kas == "tma") c = StreamCfg{16, 0, 0, 0};
    return dtype == 1 ? launch_stream_f64(a, c, st) : launch_stream_f32(a, c, st);
}

int launch_zero_rows(int dtype, const int32_t *rows, int64_t nrows, int64_t k, void *Y, void *stream, int blocks) {
    if (nrows == 0 || k == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int vec = pick_vec(dtype, k, {Y});
    int64_t gw = (nrows + 31) / 32;  // 8 warps x 4 rows per block pass
    if (gw > 148 * 8) gw = 148 * 8;
    unsigned g = (unsigned)std::max<int64_t>(gw, 1);
    if (blocks > 0 && (unsigned)blocks < g) g = (unsigned)blocks;
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

// generic row mover for the distributed path: dst[didx ? didx[i] : i] (= | +=) src[sidx ? sidx[i] : i]
namespace {
constexpr int kRowsInFlight = 4;
inline unsigned warp_row_grid(int64_t n) {  // 8 warps per block, kRowsInFlight rows per warp pass
    int64_t g = (n + 8 * kRowsInFlight - 1) / (8 * kRowsInFlight);
    if (g > 148 * 8) g = 148 * 8;
    if (g < 1) g = 1;
    return (unsigned)g;
}
template <typename T, int VEC>
__global__ void __launch_bounds__(256) k_rows(const T *__restrict__ src, const int32_t *__restrict__ sidx,
                                              const int32_t *__restrict__ didx, int64_t n, int64_t k, int add,
                                              T *__restrict__ dst) {
    // one warp per row, kRowsInFlight rows per warp iteration (all loads issued before the stores)
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kRowsInFlight; r0 < n;
         r0 += nw * kRowsInFlight) {
        int64_t si[kRowsInFlight], di[kRowsInFlight];
#pragma unroll
        for (int t = 0; t < kRowsInFlight; ++t) {
            const int64_t i = r0 + t;
            const bool v = i < n;
            si[t] = !v ? -1 : sidx ? (int64_t)__ldg(sidx + i) : i;  // sidx < 0: the row is zeroed
            di[t] = !v ? -1 : didx ? (int64_t)__ldg(didx + i) : i;
        }
        for (int64_t c = (int64_t)lane * VEC; c < k; c += 32 * VEC) {
            Frag<T, VEC> a[kRowsInFlight];
#pragma unroll
            for (int t = 0; t < kRowsInFlight; ++t) {
                if (si[t] >= 0) a[t] = ld_plain<T, VEC>(src + si[t] * k + c);
                else a[t].zero();
            }
#pragma unroll
            for (int t = 0; t < kRowsInFlight; ++t) {
                if (di[t] < 0) continue;
                T *p = dst + di[t] * k + c;
                if (add) {
                    Frag<T, VEC> y = ld_plain<T, VEC>(p);
#pragma unroll
                    for (int q = 0; q < VEC; ++q) a[t].v[q] += y.v[q];
                }
                st_plain<T, VEC>(p, a[t]);
            }
        }
    }
}

// dst[drow[r]] += sum_{e in [ptr[r], ptr[r+1])} src[sidx[e]], contributions summed in list order
// (deterministic; every destination row appears once, so rows need no atomics).
template <typename T, int VEC>
__global__ void __launch_bounds__(256) k_gather_add(const T *__restrict__ src, const int32_t *__restrict__ ptr,
                                                    const int32_t *__restrict__ sidx, const int32_t *__restrict__ drow,
                                                    int64_t n, int64_t k, T *__restrict__ dst) {
    const int64_t kv = k / VEC, total = n * kv;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / kv, c = (t - r * kv) * VEC;
        T *p = dst + (int64_t)__ldg(drow + r) * k + c;
        Frag<T, VEC> a = ld_plain<T, VEC>(p);
        const int e1 = __ldg(ptr + r + 1);
        for (int e = __ldg(ptr + r); e < e1; ++e) {
            const Frag<T, VEC> s = ld_plain<T, VEC>(src + (int64_t)__ldg(sidx + e) * k + c);
#pragma unroll
            for (int q = 0; q < VEC; ++q) a.v[q] += s.v[q];
        }
        st_plain<T, VEC>(p, a);
    }
}
// ---------------------------------------------------------- P2P transport (peer memory over NVLink)
// push: row enc(didx[i]) of bases (this GPU's or a peer's workspace) = src[sidx[i]] (or zero).
// Remote stores are posted writes over NVLink, so a modest grid saturates the link.
template <typename T, int VEC>
__global__ void __launch_bounds__(256) k_push_rows(const T *__restrict__ src, const int32_t *__restrict__ sidx,
                                                   const int32_t *__restrict__ didx, int64_t n, int64_t k,
                                                   const PeerPtrs bases) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kRowsInFlight; r0 < n;
         r0 += nw * kRowsInFlight) {
        int64_t si[kRowsInFlight];
        T *dp[kRowsInFlight];
#pragma unroll
        for (int t = 0; t < kRowsInFlight; ++t) {
            const int64_t i = r0 + t;
            si[t] = -1;
            dp[t] = nullptr;
            if (i < n) {
                si[t] = __ldg(sidx + i);
                const uint32_t d = (uint32_t)__ldg(didx + i);
                dp[t] = reinterpret_cast<T *>(bases.p[d >> kPeerShift]) + (int64_t)(d & kPeerRowMask) * k;
            }
        }
        for (int64_t c = (int64_t)lane * VEC; c < k; c += 32 * VEC) {
            Frag<T, VEC> a[kRowsInFlight];
#pragma unroll
            for (int t = 0; t < kRowsInFlight; ++t) {
                if (si[t] >= 0) a[t] = ld_x<T, VEC>(src + si[t] * k + c);
                else a[t].zero();
            }
#pragma unroll
            for (int t = 0; t < kRowsInFlight; ++t)
                if (dp[t]) st_stream<T, VEC>(dp[t] + c, a[t]);
        }
    }
}

// Y[drow[r]] += sum of encoded rows (local staging rows, head partials of every rank's C0)
template <typename T, int VEC>
__global__ void __launch_bounds__(256) k_gather_add_peers(const PeerPtrs bases, int64_t par_shift,
                                                          const int32_t *__restrict__ ptr,
                                                          const int32_t *__restrict__ sidx,
                                                          const int32_t *__restrict__ drow, int64_t n, int64_t k,
                                                          T *__restrict__ Y) {
    const int64_t kv = k / VEC, total = n * kv;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / kv, c = (t - r * kv) * VEC;
        T *p = Y + (int64_t)__ldg(drow + r) * k + c;
        Frag<T, VEC> a = ld_plain<T, VEC>(p);
        const int e1 = __ldg(ptr + r + 1);
        for (int e = __ldg(ptr + r); e < e1; ++e) {
            const uint32_t s = (uint32_t)__ldg(sidx + e);
            const int64_t row = (int64_t)(s & kPeerRowMask) + ((s & kParityBit) ? par_shift : 0);
            const T *q = reinterpret_cast<const T *>(bases.p[(s & ~kParityBit) >> kPeerShift]) + row * k + c;
            const Frag<T, VEC> v = ld_plain<T, VEC>(q);
#pragma unroll
            for (int u = 0; u < VEC; ++u) a.v[u] += v.v[u];
        }
        st_plain<T, VEC>(p, a);
    }
}

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_barrier(const PeerPtrs flags, const unsigned *mine, int slot, unsigned epoch, int me, int G) {
    const int g = threadIdx.x;
    if (g >= G) return;
    unsigned *dst = reinterpret_cast<unsigned *>(flags.p[g]) + slot * kMaxPeers + me;
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(dst), "r"(epoch) : "memory");
    const unsigned *src = mine + slot * kMaxPeers + g;
    const uint64_t t0 = global_ns();
    for (;;) {
        unsigned v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(src) : "memory");
        if ((int)(v - epoch) >= 0) break;
        if (global_ns() - t0 > 60ull * 1000000000ull) {
            printf("arrow: cross-GPU barrier timed out (rank %d waiting for rank %d, slot %d, epoch %u)\n", me, g,
                   slot, epoch);
            __trap();
        }
        __nanosleep(100);
    }
}
}  // namespace

int launch_push_rows(int dtype, const void *src, const int32_t *sidx, const int32_t *didx, int64_t n, int64_t k,
                     const PeerPtrs &bases, int blocks, void *stream) {
    if (n == 0 || k == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int vec = pick_vec(dtype, k, {src});
    for (const void *p : bases.p) vec = std::min(vec, pick_vec(dtype, k, {p}));
    unsigned g = warp_row_grid(n);
    if (blocks > 0 && (unsigned)blocks < g) g = (unsigned)blocks;
    if (dtype == 0) {
        if (vec == 4) k_push_rows<float, 4><<<g, 256, 0, st>>>((const float *)src, sidx, didx, n, k, bases);
        else if (vec == 2) k_push_rows<float, 2><<<g, 256, 0, st>>>((const float *)src, sidx, didx, n, k, bases);
        else k_push_rows<float, 1><<<g, 256, 0, st>>>((const float *)src, sidx, didx, n, k, bases);
    } else {
        if (vec == 2) k_push_rows<double, 2><<<g, 256, 0, st>>>((const double *)src, sidx, didx, n, k, bases);
        else k_push_rows<double, 1><<<g, 256, 0, st>>>((const double *)src, sidx, didx, n, k, bases);
    }
    return (int)cudaGetLastError();
}

int launch_gather_add_peers(int dtype, const PeerPtrs &bases, int64_t par_shift, const int32_t *ptr,
                            const int32_t *src, const int32_t *drow, int64_t n, int64_t k, void *Y, void *stream) {
    if (n == 0 || k == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int vec = pick_vec(dtype, k, {Y});
    for (const void *p : bases.p) vec = std::min(vec, pick_vec(dtype, k, {p}));
    const unsigned g = grid_for(n * (k / vec));
    if (dtype == 0) {
        if (vec == 4) k_gather_add_peers<float, 4><<<g, 256, 0, st>>>(bases, par_shift, ptr, src, drow, n, k, (float *)Y);
        else if (vec == 2) k_gather_add_peers<float, 2><<<g, 256, 0, st>>>(bases, par_shift, ptr, src, drow, n, k, (float *)Y);
        else k_gather_add_peers<float, 1><<<g, 256, 0, st>>>(bases, par_shift, ptr, src, drow, n, k, (float *)Y);
    } else {
        if (vec == 2) k_gather_add_peers<double, 2><<<g, 256, 0, st>>>(bases, par_shift, ptr, src, drow, n, k, (double *)Y);
        else k_gather_add_peers<double, 1><<<g, 256, 0, st>>>(bases, par_shift, ptr, src, drow, n, k, (double *)Y);
    }
    return (int)cudaGetLastError();
}

int launch_barrier(const PeerPtrs &flags, const unsigned *mine, int slot, unsigned epoch, int me, int G,
                   void *stream) {
    k_barrier<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(flags, mine, slot, epoch, me, G);
    return (int)cudaGetLastError();
}

namespace {
template <typename T, int VEC>
__global__ void __launch_bounds__(256) k_act_rows(const int32_t *__restrict__ rows, int64_t nrows, int64_t k, int act,
                                                  T *__restrict__ Y) {
    const int64_t kv = k / VEC, total = nrows * kv;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / kv, c = (t - j * kv) * VEC;
        T *p = Y + (int64_t)__ldg(rows + j) * k + c;
        Frag<T, VEC> y = ld_plain<T, VEC>(p);
        if (act == 1) {
#pragma unroll
            for (int i = 0; i < VEC; ++i) y.v[i] = y.v[i] > T(0) ? y.v[i] : T(0);
        }
        st_plain<T, VEC>(p, y);
    }
}
}  // namespace

int launch_act_rows(int dtype, const int32_t *rows, int64_t nrows, int64_t k, int act, void *Y, void *stream) {
    if (nrows == 0 || k == 0 || act == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int vec = pick_vec(dtype, k, {Y});
    const unsigned g = grid_for(nrows * (k / vec));
    if (dtype == 0) {
        if (vec == 4) k_act_rows<float, 4><<<g, 256, 0, st>>>(rows, nrows, k, act, (float *)Y);
        else if (vec == 2) k_act_rows<float, 2><<<g, 256, 0, st>>>(rows, nrows, k, act, (float *)Y);
        else k_act_rows<float, 1><<<g, 256, 0, st>>>(rows, nrows, k, act, (float *)Y);
    } else {
        if (vec == 2) k_act_rows<double, 2><<<g, 256, 0, st>>>(rows, nrows, k, act, (double *)Y);
        else k_act_rows<double, 1><<<g, 256, 0, st>>>(rows, nrows, k, act, (double *)Y);
    }
    return (int)cudaGetLastError();
}

int launch_gather_add(int dtype, const void *src, const int32_t *ptr, const int32_t *sidx, const int32_t *drow,
                      int64_t n, int64_t k, void *dst, void *stream) {
    if (n == 0 || k == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int vec = pick_vec(dtype, k, {src, dst});
    const unsigned g = grid_for(n * (k / vec));
    if (dtype == 0) {
        if (vec == 4) k_gather_add<float, 4><<<g, 256, 0, st>>>((const float *)src, ptr, sidx, drow, n, k, (float *)dst);
        else if (vec == 2) k_gather_add<float, 2><<<g, 256, 0, st>>>((const float *)src, ptr, sidx, drow, n, k, (float *)dst);
        else k_gather_add<float, 1><<<g, 256, 0, st>>>((const float *)src, ptr, sidx, drow, n, k, (float *)dst);
    } else {
        if (vec == 2) k_gather_add<double, 2><<<g, 256, 0, st>>>((const double *)src, ptr, sidx, drow, n, k, (double *)dst);
        else k_gather_add<double, 1><<<g, 256, 0, st>>>((const double *)src, ptr, sidx, drow, n, k, (double *)dst);
    }
    return (int)cudaGetLastError();
}

int launch_rows(int dtype, const void *src, const int32_t *sidx, const int32_t *didx, int64_t n, int64_t k, int add,
                void *dst, void *stream) {
    if (n == 0 || k == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int vec = pick_vec(dtype, k, {src, dst});
    const unsigned g = warp_row_grid(n);
    if (dtype == 0) {
        if (vec == 4) k_rows<float, 4><<<g, 256, 0, st>>>((const float *)src, sidx, didx, n, k, add, (float *)dst);
        else if (vec == 2) k_rows<float, 2><<<g, 256, 0, st>>>((const float *)src, sidx, didx, n, k, add, (float *)dst);
        else k_rows<float, 1><<<g, 256, 0, st>>>((const float *)src, sidx, didx, n, k, add, (float *)dst);
    } else {
        if (vec == 2) k_rows<double, 2><<<g, 256, 0, st>>>((const double *)src, sidx, didx, n, k, add, (double *)dst);
        else k_rows<double, 1><<<g, 256, 0, st>>>((const double *)src, sidx, didx, n, k, add, (double *)dst);
    }
    return (int)cudaGetLastError();
}

int launch_zero(void *Y, int64_t bytes, void *stream) {
    if (bytes == 0) return 0;
    return (int)cudaMemsetAsync(Y, 0, (size_t)bytes, reinterpret_cast<cudaStream_t>(stream));
}

}  // namespace arrow
