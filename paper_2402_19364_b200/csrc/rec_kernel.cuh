// rec_kernel.cuh -- K-A for rows of 16-byte multiples: the record stream consumed by whole warps.
//
// PAPER.md Alg. 1 / Eq. (1); record encoding in arrow_internal.h.
// A warp owns one record batch at a time (dynamic grab, window order).  Lane l holds bytes
// [16 l + 512 v, +16) of a row (NV vectors), so each load instruction moves 512 contiguous bytes
// of one X row.  Records are consumed in groups of 8 through two register buffers A and B: the
// group two ahead is issued right after a group is consumed, so 8-16 rows per warp are always in
// flight.  Keys/values come from two 32-record chunk registers (lane l holds record cb + l and
// cb + 32 + l), refilled a chunk ahead.  Every slot is loaded with a predicated PTX load into its
// own registers (a C++ conditional assignment makes ptxas stage through a temporary and wait).
// The code is kept small on purpose (16 record bodies): a version with 64 unrolled bodies lost
// 11% of its issue slots to instruction-cache misses.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "stream_kernel.cuh"

namespace arrow {
namespace kr {

using ks::kAux;
using ks::kPseudo;
using ks::kRowMask;
using ks::Vec;

// acc += a * x with the accumulator as a read-write PTX operand: keeps it in one register set
// (otherwise ptxas writes the result into the dead slot registers and copies it back at every
// segment-flush join: 4 MOVs per record).
__device__ __forceinline__ void fma_inplace(float &acc, float a, float x) {
    asm("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc) : "f"(a), "f"(x));
}
__device__ __forceinline__ void fma_inplace(double &acc, double a, double x) {
    asm("fma.rn.f64 %0, %1, %2, %0;" : "+d"(acc) : "d"(a), "d"(x));
}

template <typename T, int NV, int G>
struct Rows {
    Vec<T, 16> x[G][NV];
};

template <typename T, int NV, int MODE, int DIST, int PIPE, int G>
__global__ void __launch_bounds__(128, (PIPE * G * NV <= 4) ? 10 : ((PIPE * G * NV <= 8) ? 8 : 4))
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
    char *yl = reinterpret_cast<char *>(Y) + lane * 16;
    char *al = reinterpret_cast<char *>(DIST ? C0 : Y) + lane * 16;  // atomic target

    Vec<T, 16> acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) ks::zero<T, 16>(acc[v]);

    Rows<T, NV, G> A, B;
    uint32_t k0 = kPseudo, k1 = kPseudo;  // chunk registers: records cb + lane, cb + 32 + lane
    T v0 = T(0), v1 = T(0);
    int len = 0, cb = 0;
    uint32_t r0 = 0;

    // issue group g (records [g, g+G) of the batch) into buffer R.  Slots that load nothing (pseudo
    // records, records past the batch) are zeroed so the FMA below can be unconditional.
    auto issue = [&](Rows<T, NV, G> &R, int g) {
        const bool second = (g - cb) >= 32;          // warp-uniform: which chunk register holds it
        const uint32_t kc = second ? k1 : k0;
        const int lb = (g - cb) & 31;
#pragma unroll
        for (int t = 0; t < G; ++t) {
            const uint32_t key = __shfl_sync(0xffffffffu, kc, lb + t);
            const bool ld = (g + t < len) && !(key & kPseudo);
            const char *p = ((DIST && (key & kAux)) ? dl : xl) + (uint64_t)(key & kRowMask) * RB;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                ks::zero<T, 16>(R.x[t][v]);
                ks::ldg_vec_pred<T, 16>(ld && act[v], p + v * 512, R.x[t][v]);
            }
        }
    };
    // consume group g from buffer R (g always lies in the first chunk register here).  Pseudo
    // records carry value 0 and a zero slot, so every record does the same FMA; only the flush
    // at a segment end is a (warp-uniform) branch.
    auto consume = [&](Rows<T, NV, G> &R, int g) {
        const int lb = (g - cb) & 31;
        const bool full = g + G <= len;
#pragma unroll
        for (int t = 0; t < G; ++t) {
            const uint32_t key = __shfl_sync(0xffffffffu, k0, lb + t);
            const T a = __shfl_sync(0xffffffffu, v0, lb + t);
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
                for (int i = 0; i < N; ++i) fma_inplace(acc[v].v[i], a, R.x[t][v].v[i]);
            if ((key & kPseudo) && (full || g + t < len)) {
                const uint64_t off = (uint64_t)(key & kRowMask) * RB;
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    if (!act[v]) continue;
                    if (key & kAux) {
                        ks::red_vec<T, 16>(al + off + v * 512, acc[v]);
                    } else if (MODE == 0) {
                        ks::st_vec_stream<T, 16>(yl + off + v * 512, acc[v]);
                    } else {
                        Vec<T, 16> y = ks::ld_vec_stream<T, 16>(yl + off + v * 512);
#pragma unroll
                        for (int i = 0; i < N; ++i) y.v[i] += acc[v].v[i];
                        ks::st_vec_stream<T, 16>(yl + off + v * 512, y);
                    }
                }
#pragma unroll
                for (int v = 0; v < NV; ++v) ks::zero<T, 16>(acc[v]);
            }
        }
    };
    // after consuming group g: retire the first chunk register when it is exhausted
    auto advance = [&](int g) {
        if (g + G - cb == 32) {
            cb += 32;
            k0 = k1;
            v0 = v1;
            k1 = kPseudo;
            v1 = T(0);
            if (cb + 32 + lane < len) {
                k1 = __ldcs(keys + r0 + cb + 32 + lane);
                v1 = __ldcs(vals + r0 + cb + 32 + lane);
            }
        }
    };

    for (;;) {
        unsigned wb = 0;
        if (lane == 0) wb = atomicAdd(counter, 1u);
        wb = __shfl_sync(0xffffffffu, wb, 0);
        if ((int64_t)wb >= nbatch) break;
        r0 = __ldg(bstart + wb);
        len = (int)(__ldg(bstart + wb + 1) - r0);
        cb = 0;
        k0 = k1 = kPseudo;
        v0 = v1 = T(0);
        if (lane < len) { k0 = __ldcs(keys + r0 + lane); v0 = __ldcs(vals + r0 + lane); }
        if (32 + lane < len) { k1 = __ldcs(keys + r0 + 32 + lane); v1 = __ldcs(vals + r0 + 32 + lane); }
        if (PIPE == 2) {
            issue(A, 0);
            issue(B, G);
            for (int g = 0; g < len; g += 2 * G) {
                consume(A, g);
                issue(A, g + 2 * G);
                advance(g);
                if (g + G >= len) break;
                consume(B, g + G);
                issue(B, g + 3 * G);
                advance(g + G);
            }
        } else {  // one buffer: issue 8, consume 8 (more warps per SM instead of a deeper pipeline)
            for (int g = 0; g < len; g += G) {
                issue(A, g);
                consume(A, g);
                advance(g);
            }
        }
    }
}

}  // namespace kr
}  // namespace arrow
