// tma_kernel.cuh -- K-A on sm_100a with the Tensor Memory Accelerator as a row-gather engine.
//
// Same record stream and semantics as stream_kernel.cuh (Alg. 1, Eq. (1)
// P:359-362; encoding in arrow_internal.h), different data movement:
//   * each warp is one stream; it grabs record batches from the per-launch counter;
//   * PRODUCE: lane l of the warp takes record l of the next chunk (C = 32 records) and, if it is
//     a nonzero, issues one 1-D bulk copy (cp.async.bulk, TMA) of its X row (row bytes RB) into
//     a shared-memory ring slot; one mbarrier per chunk collects the bytes (expect_tx = nreal*RB);
//   * CONSUME: the warp waits on the chunk's mbarrier once, then walks the chunk's records: a
//     nonzero is one LDS.128 per lane + FMAs, a pseudo record flushes the accumulator (store,
//     read-modify-write, or L2 atomics for head-row partials);
//   * the ring holds NCH chunks, so NCH*32 rows per warp are in flight while the warp computes,
//     and the keys/values of the chunk after next are prefetched into registers.
// Per nonzero the SM executes ~10 instructions (shuffles, LDS, FMAs); address generation and
// the 512-byte transfers run on the TMA engine.  No registers are tied up by loads in flight.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "stream_kernel.cuh"

namespace arrow {
namespace kt {

using ks::kAux;
using ks::kPseudo;
using ks::kRowMask;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <typename T> struct V16 {
    static constexpr int N = 16 / (int)sizeof(T);
    T v[N];
};

template <typename T>
__device__ __forceinline__ V16<T> lds16(const char *p) {
    uint4 r = *reinterpret_cast<const uint4 *>(p);
    V16<T> o;
    memcpy(&o, &r, 16);
    return o;
}

// C = 32 records per chunk, NCH chunks in the ring, NV 16-byte vectors per lane (RB <= NV * 512).
template <typename T, int NV, int NCH, int MODE, int DIST>
__global__ void __launch_bounds__(256, 1)
k_tma(const uint32_t *__restrict__ keys, const T *__restrict__ vals, const uint32_t *__restrict__ bstart,
      int64_t nbatch, const T *__restrict__ X, const T *__restrict__ D0, T *__restrict__ Y, T *__restrict__ C0,
      int64_t k, unsigned *__restrict__ counter) {
    constexpr int C = 32;
    constexpr int N = V16<T>::N;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t RB = (uint32_t)(k * (int64_t)sizeof(T));
    const uint32_t warp_bytes = (NCH * C * RB + NCH * 8 + 127) / 128 * 128;
    unsigned char *ring = smem + (size_t)warp * warp_bytes;
    uint64_t *bars = reinterpret_cast<uint64_t *>(ring + NCH * C * RB);
    if (lane < NCH) mbar_init(bars + lane, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();

    bool act[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) act[v] = (uint32_t)(lane * 16 + v * 512) < RB;

    // ---- producer cursor (warp-uniform): current batch [p_r, p_end)
    uint32_t p_r = 0, p_end = 0;
    bool exhausted = false;
    auto next_batch = [&]() {
        unsigned wb = 0;
        if (lane == 0) wb = atomicAdd(counter, 1u);
        wb = __shfl_sync(0xffffffffu, wb, 0);
        if ((int64_t)wb >= nbatch) {
            exhausted = true;
            p_r = p_end = 0;
        } else {
            p_r = __ldg(bstart + wb);
            p_end = __ldg(bstart + wb + 1);
        }
    };
    // prefetched descriptor of the next chunk to produce
    uint32_t n_key = kPseudo;
    T n_val = T(0);
    int n_cnt = 0;
    auto prefetch = [&]() {
        if (!exhausted && p_r >= p_end) next_batch();
        n_cnt = exhausted ? 0 : (int)min((uint32_t)C, p_end - p_r);
        n_key = kPseudo;
        n_val = T(0);
        if (lane < n_cnt) {
            n_key = __ldcs(keys + p_r + lane);
            n_val = __ldcs(vals + p_r + lane);
        }
        p_r += (uint32_t)n_cnt;
    };

    uint32_t qkey[NCH];
    T qval[NCH];
    int qcnt[NCH];
    uint32_t phase = 0;  // bit q: parity of chunk slot q
    const char *xbase = reinterpret_cast<const char *>(X);
    const char *dbase = reinterpret_cast<const char *>(D0);

    auto produce = [&](int q) {
        const int cnt = n_cnt;
        const uint32_t key = n_key;
        const bool real = lane < cnt && !(key & kPseudo);
        const unsigned rm = __ballot_sync(0xffffffffu, real);
        fence_proxy_async();  // generic reads of this slot range happen-before the async writes
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(bars + q, (uint32_t)__popc(rm) * RB);
        __syncwarp();
        if (real) {
            const char *src = ((DIST && (key & kAux)) ? dbase : xbase) + (uint64_t)(key & kRowMask) * RB;
            bulk_g2s(ring + (size_t)(q * C + lane) * RB, src, RB, bars + q);
        }
        qkey[q] = key;
        qval[q] = n_val;
        qcnt[q] = cnt;
        prefetch();
    };

    V16<T> acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int i = 0; i < N; ++i) acc[v].v[i] = T(0);

    auto flush = [&](uint32_t key) {
        const uint32_t row = key & kRowMask;
        const uint64_t off = (uint64_t)row * RB + (uint64_t)lane * 16;
        if (key & kAux) {
            char *dst = reinterpret_cast<char *>(DIST ? C0 : Y) + off;
#pragma unroll
            for (int v = 0; v < NV; ++v)
                if (act[v]) ks::red_vec<T, 16>(dst + v * 512, *reinterpret_cast<ks::Vec<T, 16> *>(&acc[v]));
        } else {
            char *dst = reinterpret_cast<char *>(Y) + off;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                if (!act[v]) continue;
                if (MODE == 0) {
                    ks::st_vec_stream<T, 16>(dst + v * 512, *reinterpret_cast<ks::Vec<T, 16> *>(&acc[v]));
                } else {
                    ks::Vec<T, 16> y = ks::ld_vec<T, 16>(dst + v * 512);
#pragma unroll
                    for (int i = 0; i < N; ++i) y.v[i] += acc[v].v[i];
                    ks::st_vec<T, 16>(dst + v * 512, y);
                }
            }
        }
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int i = 0; i < N; ++i) acc[v].v[i] = T(0);
    };

    // prologue: fill the ring
    prefetch();
#pragma unroll
    for (int q = 0; q < NCH; ++q) produce(q);

    for (;;) {
        bool any = false;
#pragma unroll
        for (int q = 0; q < NCH; ++q) {
            const int cnt = qcnt[q];
            any |= cnt > 0;
            mbar_wait(bars + q, (phase >> q) & 1u);
            phase ^= 1u << q;
            const unsigned char *slot0 = ring + (size_t)(q * C) * RB + lane * 16;
            int t = 0;
#pragma unroll 1
            for (; t + 4 <= cnt; t += 4) {
                uint32_t kk[4];
                T aa[4];
                V16<T> xx[4][NV];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    kk[u] = __shfl_sync(0xffffffffu, qkey[q], t + u);
                    aa[u] = __shfl_sync(0xffffffffu, qval[q], t + u);
#pragma unroll
                    for (int v = 0; v < NV; ++v)
                        if (act[v] && !(kk[u] & kPseudo))
                            xx[u][v] = lds16<T>(reinterpret_cast<const char *>(slot0) + (size_t)(t + u) * RB + v * 512);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (kk[u] & kPseudo) {
                        flush(kk[u]);
                    } else {
#pragma unroll
                        for (int v = 0; v < NV; ++v)
#pragma unroll
                            for (int i = 0; i < N; ++i) acc[v].v[i] = fma(aa[u], xx[u][v].v[i], acc[v].v[i]);
                    }
                }
            }
#pragma unroll 1
            for (; t < cnt; ++t) {
                const uint32_t kk = __shfl_sync(0xffffffffu, qkey[q], t);
                const T aa = __shfl_sync(0xffffffffu, qval[q], t);
                if (kk & kPseudo) {
                    flush(kk);
                } else {
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        if (!act[v]) continue;
                        const V16<T> x = lds16<T>(reinterpret_cast<const char *>(slot0) + (size_t)t * RB + v * 512);
#pragma unroll
                        for (int i = 0; i < N; ++i) acc[v].v[i] = fma(aa, x.v[i], acc[v].v[i]);
                    }
                }
            }
            __syncwarp();
            produce(q);
        }
        if (!any) break;
    }
}

}  // namespace kt
}  // namespace arrow
