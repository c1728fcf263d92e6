// gather_bw2.cu -- which load form moves random L2-resident 512-byte rows (k = 128 fp32) into the SM
// fastest?  Same access pattern as gather_bw.cu (random rows from a 16,384-row window that advances
// every 1 M gathers), one variant per load form:
//   0 ld.global.nc.v4.f32                      (K-A today: __ldg, L1-allocating)
//   1 ld.global.nc.L1::no_allocate.v4.f32
//   2 ld.global.cg.v4.f32                      (L2 only)
//   3 ld.global.nc.v8.f32  (256-bit, sm_100+)  half-warp per row, 2 rows per warp instruction
//   4 ld.global.cg.v8.f32 ... (L2 only, 256-bit)
// Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gbw2 profiles/gather_bw2.cu && /tmp/gbw2
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

struct F8 { float v[8]; };

template <int MODE>
__device__ __forceinline__ float4 ld4(const float4 *p) {
    float4 r;
    if (MODE == 0) asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    else if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    else asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}

template <int MODE>
__device__ __forceinline__ F8 ld8(const float *p) {
    F8 r;
    if (MODE == 3)
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7]) : "l"(p));
    else
        asm volatile("ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7]) : "l"(p));
    return r;
}

template <int MODE, int UNROLL>
__global__ void __launch_bounds__(256) gather(const float *__restrict__ X, const int *__restrict__ idx, long n,
                                             float4 *__restrict__ out, unsigned *counter) {
    const int lane = threadIdx.x & 31;
    float a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (;;) {
        unsigned c = 0;
        if (lane == 0) c = atomicAdd(counter, 1u);
        c = __shfl_sync(0xffffffffu, c, 0);
        long base = (long)c * 256;
        if (base >= n) break;
        const int myidx = __ldg(idx + base + (lane & 31));
        for (int u = 0; u < 256; u += 32) {
            const int blk = __ldg(idx + base + u + lane);
            if (MODE <= 2) {
#pragma unroll
                for (int t0 = 0; t0 < 32; t0 += UNROLL) {
                    float4 v[UNROLL];
#pragma unroll
                    for (int t = 0; t < UNROLL; ++t) {
                        const int r = __shfl_sync(0xffffffffu, blk, t0 + t);
                        v[t] = ld4<MODE>(reinterpret_cast<const float4 *>(X) + (long)r * 32 + lane);
                    }
#pragma unroll
                    for (int t = 0; t < UNROLL; ++t) { a0 += v[t].x; a1 += v[t].y; a2 += v[t].z; a3 += v[t].w; }
                }
            } else {
                // half-warp per row, 32 B per lane: rows 2t (lanes 0-15) and 2t+1 (lanes 16-31)
                const int half = lane >> 4, hl = lane & 15;
#pragma unroll
                for (int t0 = 0; t0 < 32; t0 += 2 * UNROLL) {
                    F8 v[UNROLL];
#pragma unroll
                    for (int t = 0; t < UNROLL; ++t) {
                        const int r = __shfl_sync(0xffffffffu, blk, t0 + 2 * t + half);
                        v[t] = ld8<MODE>(X + (long)r * 128 + hl * 8);
                    }
#pragma unroll
                    for (int t = 0; t < UNROLL; ++t) {
                        a0 += v[t].v[0] + v[t].v[4]; a1 += v[t].v[1] + v[t].v[5];
                        a2 += v[t].v[2] + v[t].v[6]; a3 += v[t].v[3] + v[t].v[7];
                    }
                }
            }
        }
        a0 += (float)myidx * 0.f;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = make_float4(a0, a1, a2, a3);
}

template <int MODE>
float run(const float *X, const int *idx, long n, float4 *out, unsigned *cnt, int grid) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(cnt, 0, 4);
        cudaEventRecord(a);
        gather<MODE, 8><<<grid, 256>>>(X, idx, n, out, cnt);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    const long rows = 1 << 22, window = 16384, n = 64l << 20;  // 64 M gathers
    std::vector<int> h(n);
    std::mt19937 rng(1);
    for (long i = 0; i < n; ++i) {
        long w = (i / (1 << 20)) % (rows / window);
        h[i] = (int)(w * window + rng() % window);
    }
    float *X;
    float4 *out;
    int *idx;
    unsigned *cnt;
    cudaMalloc(&X, rows * 512);
    cudaMemset(X, 0, rows * 512);
    cudaMalloc(&idx, n * 4);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&out, 148 * 8 * 256 * 16);
    cudaMalloc(&cnt, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char *names[5] = {"nc.v4", "nc.L1::no_allocate.v4", "cg.v4", "nc.v8 (half-warp rows)", "cg.v8 (half-warp rows)"};
    for (int bps : {4, 8}) {
        const int grid = sms * bps;
        float t[5];
        t[0] = run<0>(X, idx, n, out, cnt, grid);
        t[1] = run<1>(X, idx, n, out, cnt, grid);
        t[2] = run<2>(X, idx, n, out, cnt, grid);
        t[3] = run<3>(X, idx, n, out, cnt, grid);
        t[4] = run<4>(X, idx, n, out, cnt, grid);
        for (int m = 0; m < 5; ++m)
            printf("blocks/SM %d %-24s %.3f ms  %.2f TB/s  %.1f Mrows/ms\n", bps, names[m], t[m], n * 512.0 / t[m] / 1e9,
                   n / t[m] / 1e6);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
