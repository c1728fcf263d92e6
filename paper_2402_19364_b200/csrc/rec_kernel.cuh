// rec_kernel.cuh -- K-A for rows of 16-byte multiples: the record stream consumed by whole warps.
//
// PAPER.md Alg. 1 / Eq. (1); record encoding in arrow_internal.h.
// A warp owns one record batch at a time (dynamic grab, window order).  Records are streamed in
// chunks of 32 (one coalesced key/value load per lane, prefetched a chunk ahead) and consumed
// in four groups of 8 with two register buffers: the 8 row loads of group g+1 are issued before
// group g is consumed, so 8-16 rows per warp are always in flight.  Lane l holds bytes
// [16 l + 512 v, +16) of the row (NV vectors), i.e. each load instruction moves 512 contiguous
// bytes of one X row.  Every slot is loaded with a predicated PTX load into its own registers
// (a C++ conditional assignment makes ptxas stage through a temporary and wait on each load).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>

#include "stream_kernel.cuh"

namespace arrow {
namespace kr {

using ks::kAux;
using ks::kPseudo;
using ks::kRowMask;
using ks::Vec;

template <typename T, int NV>
struct Rows {
    Vec<T, 16> x[8][NV];
    uint32_t key[8];
    T val[8];
};

template <typename T, int NV, int MODE, int DIST>
__global__ void __launch_bounds__(256, 2)
k_rec(const uint32_t *__restrict__ keys, const T *__restrict__ vals, const uint32_t *__restrict__ bstart,
      int64_t nbatch, const T *__restrict__ X, const T *__restrict__ D0, T *__restrict__ Y, T *__restrict__ C0,
      int64_t k, unsigned *__restrict__ counter) {
    constexpr int N = Vec<T, 16>::N;
    const int lane = threadIdx.x & 31;
    const uint32_t RB = (uint32_t)(k * (int64_t)sizeof(T));
    bool act[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) act[v] = (uint32_t)(lane * 16 + v * 512) < RB;
    const char *xl = reinterpret_cast<const char *>(X) + lane * 16;
    const char *dl = reinterpret_cast<const char *>(D0) + lane * 16;

    Vec<T, 16> acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) ks::zero<T, 16>(acc[v]);

    auto flush = [&](uint32_t key) {
        const uint64_t off = (uint64_t)(key & kRowMask) * RB + (uint64_t)lane * 16;
        if (key & kAux) {
            char *dst = reinterpret_cast<char *>(DIST ? C0 : Y) + off;
#pragma unroll
            for (int v = 0; v < NV; ++v)
                if (act[v]) ks::red_vec<T, 16>(dst + v * 512, acc[v]);
        } else {
            char *dst = reinterpret_cast<char *>(Y) + off;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                if (!act[v]) continue;
                if (MODE == 0) {
                    ks::st_vec_stream<T, 16>(dst + v * 512, acc[v]);
                } else {
                    Vec<T, 16> y = ks::ld_vec_stream<T, 16>(dst + v * 512);
#pragma unroll
                    for (int i = 0; i < N; ++i) y.v[i] += acc[v].v[i];
                    ks::st_vec_stream<T, 16>(dst + v * 512, y);
                }
            }
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) ks::zero<T, 16>(acc[v]);
    };

    // issue the 8 records [base, base+8) of the current chunk into buffer B
    auto issue = [&](Rows<T, NV> &B, uint32_t ck, T cv, int base, int cnt, auto full) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const uint32_t key = __shfl_sync(0xffffffffu, ck, base + t);
            B.key[t] = key;
            B.val[t] = __shfl_sync(0xffffffffu, cv, base + t);
            const bool ld = (decltype(full)::value || base + t < cnt) && !(key & kPseudo);
            const char *p = ((DIST && (key & kAux)) ? dl : xl) + (uint64_t)(key & kRowMask) * RB;
#pragma unroll
            for (int v = 0; v < NV; ++v) ks::ldg_vec_pred<T, 16>(ld && act[v], p + v * 512, B.x[t][v]);
        }
    };
    auto consume = [&](Rows<T, NV> &B, int base, int cnt, auto full) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            if (decltype(full)::value || base + t < cnt) {
                const uint32_t key = B.key[t];
                if (key & kPseudo) {
                    flush(key);
                } else {
#pragma unroll
                    for (int v = 0; v < NV; ++v)
#pragma unroll
                        for (int i = 0; i < N; ++i) acc[v].v[i] = fma(B.val[t], B.x[t][v].v[i], acc[v].v[i]);
                }
            }
        }
    };

    Rows<T, NV> A, B;
    for (;;) {
        unsigned wb = 0;
        if (lane == 0) wb = atomicAdd(counter, 1u);
        wb = __shfl_sync(0xffffffffu, wb, 0);
        if ((int64_t)wb >= nbatch) break;
        const uint32_t r0 = __ldg(bstart + wb), r1 = __ldg(bstart + wb + 1);
        uint32_t ck = kPseudo, nk = kPseudo;
        T cv = T(0), nv = T(0);
        if (r0 + lane < r1) { ck = __ldcs(keys + r0 + lane); cv = __ldcs(vals + r0 + lane); }
        if (r0 + 32 + lane < r1) { nk = __ldcs(keys + r0 + 32 + lane); nv = __ldcs(vals + r0 + 32 + lane); }
        int cnt = (r1 - r0 < 32u) ? (int)(r1 - r0) : 32;
        const std::true_type F{};
        const std::false_type P{};
        issue(A, ck, cv, 0, cnt, P);
        issue(B, ck, cv, 8, cnt, P);
        for (uint32_t c = r0; c < r1; c += 32) {
            // next chunk: its first two groups are issued before this chunk's last two are consumed
            const int ncnt = (c + 32 < r1) ? ((r1 - c - 32 < 32u) ? (int)(r1 - c - 32) : 32) : 0;
            if (cnt == 32 && ncnt == 32) {   // fast path: no bounds checks
                consume(A, 0, 32, F);
                issue(A, ck, cv, 16, 32, F);
                consume(B, 8, 32, F);
                issue(B, ck, cv, 24, 32, F);
                consume(A, 16, 32, F);
                issue(A, nk, nv, 0, 32, F);
                consume(B, 24, 32, F);
                issue(B, nk, nv, 8, 32, F);
            } else {
                consume(A, 0, cnt, P);
                issue(A, ck, cv, 16, cnt, P);
                consume(B, 8, cnt, P);
                issue(B, ck, cv, 24, cnt, P);
                consume(A, 16, cnt, P);
                issue(A, nk, nv, 0, ncnt, P);
                consume(B, 24, cnt, P);
                issue(B, nk, nv, 8, ncnt, P);
            }
            ck = nk;
            cv = nv;
            cnt = ncnt;
            nk = kPseudo;
            nv = T(0);
            if (c + 64 + lane < r1) { nk = __ldcs(keys + c + 64 + lane); nv = __ldcs(vals + c + 64 + lane); }
        }
    }
}

}  // namespace kr
}  // namespace arrow
