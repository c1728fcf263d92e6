// kernels.cu -- the small sm_100a kernels around K-A (seg_kernel.cu): zero rows (K-Z), the
// iterate-mode activation pass, and the row movers / gather-adds / cross-GPU barrier of the
// distributed transports (S6).
//
// Per level i of the decomposition A X = sum_i P_{pi_i} (B_i (P_{pi_i}^T X))  (Eq. (1))
// the work is done by K-A; on one GPU the head block of Alg. 1 line 1 is read straight from
// X (columns are folded to X rows) and the head-row partials of line 2 are added into
// Y[head] by K-A's L2 reductions, so the stage (K-H) and epilogue (K-C) of Alg. 1 are folded away;
// in distributed mode D0 is pushed to every rank (k_push_rows) and C0 is combined by the transport.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>

#include "arrow_internal.h"
#include "dev_common.cuh"

namespace arrow {

// SM count of the current device (cached per device)
int device_sms() {
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (cache[dev] == 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cache[dev] = v;
    }
    return cache[dev];
}

namespace {

using dev::Frag;
using dev::ld_plain;
using dev::ld_x;
using dev::st_plain;
using dev::st_stream;

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

}  // namespace

int launch_zero_rows(int dtype, const int32_t *rows, int64_t nrows, int64_t k, void *Y, void *stream, int blocks) {
    if (nrows == 0 || k == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int vec = pick_vec(dtype, k, {Y});
    int64_t gw = (nrows + 31) / 32;  // 8 warps x 4 rows per block pass
    if (gw > (int64_t)device_sms() * 8) gw = (int64_t)device_sms() * 8;
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

// generic row mover for the distributed path: dst[didx ? didx[i] : i] (= | +=) src[sidx ? sidx[i] : i]
namespace {
constexpr int kRowsInFlight = 4;
inline unsigned warp_row_grid(int64_t n) {  // 8 warps per block, kRowsInFlight rows per warp pass
    int64_t g = (n + 8 * kRowsInFlight - 1) / (8 * kRowsInFlight);
    if (g > (int64_t)device_sms() * 8) g = (int64_t)device_sms() * 8;
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
        int e = __ldg(ptr + r);
        // 8 source rows in flight, added in list order (the order fixes the fp result: deterministic
        // head combine, fixed-order distributed adds); long lists (hub head rows) are latency-bound
        for (; e + 8 <= e1; e += 8) {
            Frag<T, VEC> s[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) s[u] = ld_plain<T, VEC>(src + (int64_t)__ldg(sidx + e + u) * k + c);
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int q = 0; q < VEC; ++q) a.v[q] += s[u].v[q];
        }
        for (; e < e1; ++e) {
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
    const unsigned g = grid_for(n * (k / vec), device_sms());
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
    const unsigned g = grid_for(nrows * (k / vec), device_sms());
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
    const unsigned g = grid_for(n * (k / vec), device_sms());
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
