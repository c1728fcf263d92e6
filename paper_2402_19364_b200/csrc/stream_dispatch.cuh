// stream_dispatch.cuh -- host-side launch of k_stream for one dtype (included by kernels_f32.cu /
// kernels_f64.cu so the instantiations compile in parallel).
#pragma once
#include <algorithm>

#include "arrow_internal.h"
#include "stream_kernel.cuh"
#include "tma_kernel.cuh"
#include "rec_kernel.cuh"
#include <cstdlib>

namespace arrow {
namespace ks {

template <typename T, int LPE, int NV, int VB, int D, int MODE, int DIST>
int run_one(const StreamArgs &a, cudaStream_t st) {
    auto kern = k_stream<T, LPE, NV, VB, D, MODE, DIST>;
    static int bps = 0;
    if (bps == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 256, 0);
        if (bps <= 0) bps = 1;
    }
    constexpr int64_t batches_per_block = 8 * (32 / LPE);
    int64_t blocks = std::min<int64_t>((int64_t)a.num_sms * bps, (a.nbatch + batches_per_block - 1) / batches_per_block);
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, 256, 0, st>>>(a.keys, reinterpret_cast<const T *>(a.vals), a.bstart, a.nbatch,
                                            reinterpret_cast<const T *>(a.X), reinterpret_cast<const T *>(a.D0),
                                            reinterpret_cast<T *>(a.Y), reinterpret_cast<T *>(a.C0), a.k, a.counter);
    return (int)cudaGetLastError();
}

template <typename T, int LPE, int NV, int VB, int D>
int run_cfg(const StreamArgs &a, cudaStream_t st) {
    if (a.dist) return a.mode == 0 ? run_one<T, LPE, NV, VB, D, 0, 1>(a, st) : run_one<T, LPE, NV, VB, D, 1, 1>(a, st);
    return a.mode == 0 ? run_one<T, LPE, NV, VB, D, 0, 0>(a, st) : run_one<T, LPE, NV, VB, D, 1, 0>(a, st);
}

}  // namespace ks

namespace kt {

inline int env_int(const char *name, int dflt) {
    const char *e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

template <typename T, int NV, int NCH, int MODE, int DIST>
int run_tma_one(const StreamArgs &a, int warps, cudaStream_t st) {
    auto kern = k_tma<T, NV, NCH, MODE, DIST>;
    const uint32_t RB = (uint32_t)(a.k * (int64_t)sizeof(T));
    const size_t warp_bytes = ((size_t)NCH * 32 * RB + NCH * 8 + 127) / 128 * 128;
    const size_t smem = warp_bytes * (size_t)warps;
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        configured = smem;
    }
    int bps = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, warps * 32, smem);
    if (bps <= 0) bps = 1;
    int64_t blocks = std::min<int64_t>((int64_t)a.num_sms * bps, (a.nbatch + warps - 1) / warps);
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, warps * 32, smem, st>>>(a.keys, reinterpret_cast<const T *>(a.vals), a.bstart, a.nbatch,
                                                      reinterpret_cast<const T *>(a.X),
                                                      reinterpret_cast<const T *>(a.D0), reinterpret_cast<T *>(a.Y),
                                                      reinterpret_cast<T *>(a.C0), a.k, a.counter);
    return (int)cudaGetLastError();
}

template <typename T, int NV, int NCH>
int run_tma_cfg(const StreamArgs &a, int warps, cudaStream_t st) {
    if (a.dist) return a.mode == 0 ? run_tma_one<T, NV, NCH, 0, 1>(a, warps, st) : run_tma_one<T, NV, NCH, 1, 1>(a, warps, st);
    return a.mode == 0 ? run_tma_one<T, NV, NCH, 0, 0>(a, warps, st) : run_tma_one<T, NV, NCH, 1, 0>(a, warps, st);
}

// TMA path for rows of 16..1024 bytes (multiple of 16).  Returns -1 if not applicable.
template <typename T>
int run_tma(const StreamArgs &a, cudaStream_t st) {
    const int64_t RB = a.k * (int64_t)sizeof(T);
    if (RB % 16 != 0 || RB > 1024 || env_int("ARROW_KA_STREAM", 0)) return -1;
    const int nv = RB <= 512 ? 1 : 2;
    int nch = env_int("ARROW_TMA_NCH", RB <= 512 ? 3 : 2);
    if (nch < 2) nch = 2;
    if (nch > 4) nch = 4;
    const size_t warp_bytes = ((size_t)nch * 32 * RB + nch * 8 + 127) / 128 * 128;
    int warps = env_int("ARROW_TMA_WARPS", (int)std::min<size_t>(8, (200 * 1024) / warp_bytes));
    if (warps < 1) warps = 1;
    if (warps > 8) warps = 8;
    if (nv == 1) {
        if (nch == 2) return run_tma_cfg<T, 1, 2>(a, warps, st);
        if (nch == 3) return run_tma_cfg<T, 1, 3>(a, warps, st);
        return run_tma_cfg<T, 1, 4>(a, warps, st);
    }
    return run_tma_cfg<T, 2, 2>(a, warps, st);
}

}  // namespace kt

namespace kr {

template <typename T, int NV, int MODE, int DIST, int PIPE, int G>
int run_rec_one(const StreamArgs &a, cudaStream_t st) {
    auto kern = k_rec<T, NV, MODE, DIST, PIPE, G>;
    constexpr int threads = 128;
    static int bps = 0;
    if (bps == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, threads, 0);
        if (bps <= 0) bps = 1;
    }
    int64_t blocks = std::min<int64_t>((int64_t)a.num_sms * bps, (a.nbatch + threads / 32 - 1) / (threads / 32));
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, threads, 0, st>>>(a.keys, reinterpret_cast<const T *>(a.vals), a.bstart, a.nbatch,
                                                reinterpret_cast<const T *>(a.X), reinterpret_cast<const T *>(a.D0),
                                                reinterpret_cast<T *>(a.Y), reinterpret_cast<T *>(a.C0), a.k, a.counter);
    return (int)cudaGetLastError();
}

template <typename T, int NV, int PIPE, int G>
int run_rec_pipe(const StreamArgs &a, cudaStream_t st) {
    if (a.dist) return a.mode == 0 ? run_rec_one<T, NV, 0, 1, PIPE, G>(a, st) : run_rec_one<T, NV, 1, 1, PIPE, G>(a, st);
    return a.mode == 0 ? run_rec_one<T, NV, 0, 0, PIPE, G>(a, st) : run_rec_one<T, NV, 1, 0, PIPE, G>(a, st);
}

// variants: ARROW_REC=<pipe><group>, e.g. 18 (default: one buffer of 8 rows), 14, 24, 28
template <typename T, int NV>
int run_rec_cfg(const StreamArgs &a, cudaStream_t st) {
    static const int v = kt::env_int("ARROW_REC", 18);
    switch (v) {
        case 14: return run_rec_pipe<T, NV, 1, 4>(a, st);
        case 24: return run_rec_pipe<T, NV, 2, 4>(a, st);
        case 28: return run_rec_pipe<T, NV, 2, 8>(a, st);
        default: return run_rec_pipe<T, NV, 1, 8>(a, st);
    }
}

// Whole-warp record kernel for rows of 16-byte multiples up to 1 KiB.  Returns -1 otherwise.
template <typename T>
int run_rec(const StreamArgs &a, cudaStream_t st) {
    const int64_t RB = a.k * (int64_t)sizeof(T);
    if (RB % 16 != 0 || RB > 1024) return -1;
    return RB <= 512 ? run_rec_cfg<T, 1>(a, st) : run_rec_cfg<T, 2>(a, st);
}

}  // namespace kr
}  // namespace arrow
