// tma_gather.cu -- can TMA gather4 (cp.async.bulk.tensor.2d ... tile::gather4, sm_100a) add gather
// bandwidth on top of the LSU path?  K-A's level-0 gathers are limited by the L1TEX data pipe
// (ncu: ~64 B/clk/SM of global-load data, 83 % busy at 14.5 TB/s); TMA writes shared memory through
// the async proxy.  Random 512-byte rows (k = 128 fp32) from 16,384-row windows, like gather_bw.cu:
//   lsu   : one warp per row, ld.global.nc.v4 (the K-A pattern), 8 rows in flight per warp
//   tma   : per warp, lane 0 issues gather4 (4 rows = 2 KB) into an R-stage shared-memory ring, one
//           mbarrier per stage; the warp sums the rows from shared memory (LDS.128)
//   mix   : warps 0..L-1 of each block run lsu, the others tma (same kernel, same grid)
// Build + run on the GPU box (bounded waits: a wrong expect_tx count reports an error, never hangs):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tg profiles/r02/tma_gather.cu -lcuda && /tmp/tg
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

constexpr int K = 128;            // fp32 columns per row (512 B)
constexpr int RB = K * 4;         // row bytes
constexpr int STAGES = 6;         // gather4 stages per tma warp
constexpr int STAGE_BYTES = 4 * RB;
__constant__ int c_boxc;          // columns per TMA op (box inner dimension)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// bounded wait: returns false after ~2^26 polls (reported, never hangs)
__device__ __forceinline__ bool mbar_wait(uint64_t *b, unsigned phase) {
    for (unsigned it = 0; it < (1u << 26); ++it) {
        unsigned ok;
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(smem_u32(b)), "r"(phase) : "memory");
        if (ok) return true;
    }
    return false;
}
__device__ __forceinline__ void tma_gather4(const CUtensorMap *tm, uint64_t *bar, void *dst, int c0, int r0, int r1, int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}
__device__ __forceinline__ void tma_tile(const CUtensorMap *tm, uint64_t *bar, void *dst, int c0, int r0) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(r0)
        : "memory");
}

// MODE 0: all warps lsu; 1: all warps tma; 2: the first LSUW warps of a block lsu, the rest tma
template <int MODE, int LSUW>
__global__ void __launch_bounds__(256, 2) k_gather(const __grid_constant__ CUtensorMap tm, const float *__restrict__ X,
                                                  const int *__restrict__ idx, long n, unsigned *counter, float4 *out,
                                                  unsigned *err) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool tma = MODE == 1 || MODE == 3 || (MODE == 2 && wid >= LSUW);
    float4 acc = make_float4(0, 0, 0, 0);
    __shared__ uint64_t bars[8][STAGES];
    // TMA destinations must be 128-byte aligned: align the dynamic region by hand (1 KB slack)
    unsigned char *base_al = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~(uintptr_t)1023);
    unsigned char *ring = base_al + (size_t)wid * STAGES * STAGE_BYTES;
    if (tma && lane == 0)
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[wid][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    unsigned phase_bits = 0;  // bit s: parity of the phase stage s completes next (persists across blocks)
    for (;;) {
        unsigned c = 0;
        if (lane == 0) c = atomicAdd(counter, 1u);
        c = __shfl_sync(0xffffffffu, c, 0);
        const long base = (long)c * 256;
        if (base >= n) break;
        if (!tma) {
            for (int u = 0; u < 256; u += 32) {
                const int blk = __ldg(idx + base + u + lane);
#pragma unroll
                for (int t0 = 0; t0 < 32; t0 += 8) {
                    float4 v[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        const int r = __shfl_sync(0xffffffffu, blk, t0 + t);
                        v[t] = __ldg(reinterpret_cast<const float4 *>(X + (long)r * K) + lane);
                    }
#pragma unroll
                    for (int t = 0; t < 8; ++t) { acc.x += v[t].x; acc.y += v[t].y; acc.z += v[t].z; acc.w += v[t].w; }
                }
            }
        } else {
            // 64 gather4 ops per 256-row block, STAGES in flight
            const int ngroups = 64;
            int issued = 0;
            auto issue = [&](int g) {
                const int s = g % STAGES;
                if (lane == 0) {
                    const int4 r = __ldg(reinterpret_cast<const int4 *>(idx + base) + g);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect(&bars[wid][s], STAGE_BYTES);
                    unsigned char *d = ring + s * STAGE_BYTES;
                    const int bc = c_boxc;
                    if (MODE == 3) {  // plain tiles: one op per row slab
                        const int rr[4] = {r.x, r.y, r.z, r.w};
                        for (int t = 0; t < 4; ++t)
                            for (int c0 = 0; c0 < K; c0 += bc) tma_tile(&tm, &bars[wid][s], d + t * RB + c0 * 4, c0, rr[t]);
                    } else {
                        // gather4 of a column slab: 4 rows x bc columns, slabs stacked [slab][row][col]
                        for (int c0 = 0; c0 < K; c0 += bc) tma_gather4(&tm, &bars[wid][s], d + c0 * 16, c0, r.x, r.y, r.z, r.w);
                    }
                }
            };
            for (; issued < STAGES && issued < ngroups; ++issued) issue(issued);
            for (int g = 0; g < ngroups; ++g) {
                const int s = g % STAGES;
                if (!mbar_wait(&bars[wid][s], (phase_bits >> s) & 1u)) {
                    if (lane == 0) atomicAdd(err, 1u);
                    return;
                }
                phase_bits ^= 1u << s;
                const float4 *rows = reinterpret_cast<const float4 *>(ring + s * STAGE_BYTES);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float4 v = rows[t * 32 + lane];
                    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
                }
                __syncwarp();
                if (issued < ngroups) issue(issued++);
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE, int LSUW>
float run(const CUtensorMap &tm, const float *X, const int *idx, long n, unsigned *cnt, float4 *out, unsigned *err,
          int grid) {
    const size_t sm = MODE == 0 ? 0 : (size_t)8 * STAGES * STAGE_BYTES + 1024;
    cudaFuncSetAttribute(k_gather<MODE, LSUW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaMemset(cnt, 0, 4);
        cudaEventRecord(a);
        k_gather<MODE, LSUW><<<grid, 256, sm>>>(tm, X, idx, n, cnt, out, err);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)
int main(int argc, char **argv) {
    const int variant = argc > 1 ? atoi(argv[1]) : 0;
    const int boxc = argc > 2 ? atoi(argv[2]) : 128;
    const int swz = argc > 3 ? atoi(argv[3]) : 0;
    setvbuf(stdout, nullptr, _IONBF, 0);
    printf("start\n");
    const long rows = 1 << 22, window = 16384, n = 64l << 20;  // 64 M gathers
    std::vector<int> h(n);
    std::mt19937 rng(1);
    for (long i = 0; i < n; ++i) {
        const long w = (i / (1 << 20)) % (rows / window);
        h[i] = (int)(w * window + rng() % window);
    }
    float *X;
    float4 *out;
    int *idx;
    unsigned *cnt, *err;
    CK(cudaMalloc(&X, rows * RB));
    CK(cudaMemset(X, 0, rows * RB));
    CK(cudaMalloc(&idx, n * 4));
    CK(cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&out, 148 * 4 * 256 * 16));
    CK(cudaMalloc(&cnt, 4));
    CK(cudaMalloc(&err, 4));
    CK(cudaMemset(err, 0, 4));
    printf("allocated\n");
    CUtensorMap tm;
    cuuint64_t gdim[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {(cuuint64_t)RB};
    cuuint32_t box[2] = {(cuuint32_t)boxc, 1};
    cudaMemcpyToSymbol(c_boxc, &boxc, 4);
    cuuint32_t es[2] = {1, 1};
    CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, gdim, gstride, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("tensor map: %d\n", (int)cr);
    if (cr != CUDA_SUCCESS) return 1;
    const double bytes = (double)n * RB;
    auto rep = [&](const char *name, float ms) {
        unsigned e = 0;
        cudaMemcpy(&e, err, 4, cudaMemcpyDeviceToHost);
        const cudaError_t ce = cudaGetLastError();
        printf("%-28s %8.3f ms  %6.2f TB/s  wait-timeouts %u  cuda: %s\n", name, ms, bytes / (ms * 1e-3) / 1e12, e,
               cudaGetErrorString(ce));
        if (ce != cudaSuccess) exit(2);
    };
    printf("variant %d box %d swizzle %d\n", variant, boxc, swz);
    if (variant == 0) {
        rep("lsu 32 warps/SM", run<0, 8>(tm, X, idx, n, cnt, out, err, 148 * 4));
        rep("lsu 16 warps/SM", run<0, 8>(tm, X, idx, n, cnt, out, err, 148 * 2));
    } else if (variant == 1) {
        rep("tma gather4 16 warps/SM", run<1, 0>(tm, X, idx, n, cnt, out, err, 148 * 2));
        rep("tma gather4 8 warps/SM", run<1, 0>(tm, X, idx, n, cnt, out, err, 148));
        rep("mix 6 lsu + 2 tma (x2/SM)", run<2, 6>(tm, X, idx, n, cnt, out, err, 148 * 2));
        rep("mix 4 lsu + 4 tma (x2/SM)", run<2, 4>(tm, X, idx, n, cnt, out, err, 148 * 2));
    } else {
        rep("tma tiles 16 warps/SM", run<3, 0>(tm, X, idx, n, cnt, out, err, 148 * 2));
    }
    return 0;
}
