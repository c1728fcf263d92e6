// gather_bw.cu -- ceiling of the K-A access pattern on this GPU: warps gather random 512-byte rows
// (k = 128 fp32) from an L2-resident window and accumulate them (no segments, no flushes).
// Build + run on the GPU box:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gbw profiles/gather_bw.cu && /tmp/gbw
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int UNROLL>
__global__ void __launch_bounds__(256) gather(const float4 *__restrict__ X, const int *__restrict__ idx, long n,
                                             float4 *__restrict__ out, unsigned *counter) {
    const int lane = threadIdx.x & 31;
    float4 acc = make_float4(0, 0, 0, 0);
    for (;;) {
        unsigned c = 0;
        if (lane == 0) c = atomicAdd(counter, 1u);
        c = __shfl_sync(0xffffffffu, c, 0);
        long base = (long)c * 256;
        if (base >= n) break;
        for (int u = 0; u < 256; u += UNROLL) {
            float4 v[UNROLL];
#pragma unroll
            for (int t = 0; t < UNROLL; ++t) v[t] = __ldg(X + (long)__ldg(idx + base + u + t) * 32 + lane);
#pragma unroll
            for (int t = 0; t < UNROLL; ++t) { acc.x += v[t].x; acc.y += v[t].y; acc.z += v[t].z; acc.w += v[t].w; }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    const long rows = 1 << 22, window = 16384, n = 64l << 20;  // 64 M gathers
    std::vector<int> h(n);
    std::mt19937 rng(1);
    for (long i = 0; i < n; ++i) {
        long w = (i / (1 << 20)) % (rows / window);  // windows advance every 1 M gathers
        h[i] = (int)(w * window + rng() % window);
    }
    float4 *X, *out;
    int *idx;
    unsigned *cnt;
    cudaMalloc(&X, rows * 512);
    cudaMemset(X, 0, rows * 512);
    cudaMalloc(&idx, n * 4);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&out, 148 * 2048 * 16);
    cudaMalloc(&cnt, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int bps : {2, 4, 6, 8}) {
        for (int un : {4, 8}) {
            float best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                cudaMemset(cnt, 0, 4);
                cudaEventRecord(a);
                if (un == 4) gather<4><<<sms * bps, 256>>>(X, idx, n, out, cnt);
                else gather<8><<<sms * bps, 256>>>(X, idx, n, out, cnt);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("blocks/SM %d unroll %d: %.3f ms  %.2f TB/s gathered (%.1f Mrows/ms)\n", bps, un, best,
                   n * 512.0 / best / 1e9, n / best / 1e6);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
