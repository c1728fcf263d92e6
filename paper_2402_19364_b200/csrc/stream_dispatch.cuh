// stream_dispatch.cuh -- host-side launch of k_stream for one dtype (included by kernels_f32.cu /
// kernels_f64.cu so the instantiations compile in parallel).
#pragma once
#include <algorithm>

#include "arrow_internal.h"
#include "stream_kernel.cuh"

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
}  // namespace arrow
