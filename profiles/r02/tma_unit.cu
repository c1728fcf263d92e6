// tma_unit.cu -- smallest TMA checks on sm_100a: one CTA, one thread issues ONE tensor copy of a
// 2D fp32 tensor (rows of 128 floats) into shared memory and waits (bounded) on its mbarrier.
//   variant 0: 1D bulk copy  cp.async.bulk.shared::cluster.global            (no tensor map)
//   variant 1: 2D tile       cp.async.bulk.tensor.2d.shared::cluster ... tile (box {BOXC, 1})
//   variant 2: 2D tile       same with .shared::cta destination
//   variant 3: 2D gather4    cp.async.bulk.tensor.2d.shared::cta ... tile::gather4
// Prints the copied values' checksum and the bounded-wait outcome.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tu profiles/r02/tma_unit.cu -lcuda && /tmp/tu 1 128
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_unit(const __grid_constant__ CUtensorMap tm, const float *X, int variant, int boxc, float *out,
                       unsigned *status) {
    __shared__ __align__(1024) float buf[4 * 128];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x != 0) return;
    for (int i = 0; i < 4 * 128; ++i) buf[i] = -1.f;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const unsigned bytes = variant == 3 ? 4u * boxc * 4u : (unsigned)boxc * 4u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes) : "memory");
    const int r0 = 5, r1 = 9, r2 = 100, r3 = 4000;
    if (variant == 0) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(buf)),
                     "l"(X + (size_t)r0 * 128), "r"(bytes), "r"(sa(&bar))
                     : "memory");
    } else if (variant == 1) {
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                         sa(buf)),
                     "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(r0), "r"(sa(&bar))
                     : "memory");
    } else if (variant == 2) {
        asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                         sa(buf)),
                     "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(r0), "r"(sa(&bar))
                     : "memory");
    } else {
        asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
                         sa(buf)),
                     "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sa(&bar))
                     : "memory");
    }
    unsigned ok = 0;
    long long t0 = clock64();
    while (!ok && clock64() - t0 < 2000000000ll) {  // ~1 s
        asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(sa(&bar)) : "memory");
    }
    status[0] = ok;
    float s = 0;
    for (int i = 0; i < 4 * 128; ++i) s += buf[i];
    out[0] = s;
    out[1] = buf[0];
    out[2] = buf[boxc - 1];
    out[3] = buf[boxc];
}

int main(int argc, char **argv) {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const int variant = argc > 1 ? atoi(argv[1]) : 1;
    const int boxc = argc > 2 ? atoi(argv[2]) : 128;
    const long rows = 8192;
    float *hX = (float *)malloc(rows * 128 * 4);
    for (long i = 0; i < rows * 128; ++i) hX[i] = (float)(i / 128) + (float)(i % 128) / 1024.f;
    float *X, *out;
    unsigned *st;
    cudaMalloc(&X, rows * 128 * 4);
    cudaMemcpy(X, hX, rows * 128 * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&out, 64);
    cudaMalloc(&st, 16);
    cudaMemset(st, 0, 16);
    CUtensorMap tm;
    cuuint64_t gdim[2] = {128, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {512};
    cuuint32_t box[2] = {(cuuint32_t)boxc, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, gdim, gstride, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("variant %d box %d: encode %d  &tm %% 64 = %d\n", variant, boxc, (int)cr, (int)((uintptr_t)&tm % 64));
    k_unit<<<1, 32>>>(tm, X, variant, boxc, out, st);
    cudaError_t e = cudaDeviceSynchronize();
    float ho[4] = {0, 0, 0, 0};
    unsigned hs = 0;
    cudaMemcpy(ho, out, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hs, st, 4, cudaMemcpyDeviceToHost);
    printf("  cuda %s  completed %u  sum %.3f  buf[0] %.4f buf[box-1] %.4f buf[box] %.4f\n", cudaGetErrorString(e), hs,
           ho[0], ho[1], ho[2], ho[3]);
    return e == cudaSuccess ? 0 : 2;
}
