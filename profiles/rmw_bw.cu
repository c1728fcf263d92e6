// rmw_bw.cu -- HBM ceiling of the level >= 1 access pattern: warps read-modify-write random 512-byte
// rows (k = 128 fp32) of a 2 GiB Y, optionally gathering a random 512-byte X row per update too.
// Reports DRAM-side bytes (a row read + a row write per RMW, + a row read per gather) per second.
// Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rmw profiles/rmw_bw.cu && /tmp/rmw
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int UNROLL, bool GATHER, bool RMW>
__global__ void __launch_bounds__(256) kern(float4 *__restrict__ Y, const float4 *__restrict__ X,
                                           const int *__restrict__ yi, const int *__restrict__ xi, long n,
                                           unsigned *counter) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned c = 0;
        if (lane == 0) c = atomicAdd(counter, 1u);
        c = __shfl_sync(0xffffffffu, c, 0);
        const long base = (long)c * 32;
        if (base >= n) break;
        const int my_y = __ldg(yi + base + lane);
        const int my_x = GATHER ? __ldg(xi + base + lane) : 0;
        for (int u = 0; u < 32; u += UNROLL) {
            float4 a[UNROLL], y[UNROLL];
#pragma unroll
            for (int t = 0; t < UNROLL; ++t) {
                const int r = __shfl_sync(0xffffffffu, my_y, u + t);
                if (GATHER) a[t] = __ldg(X + (long)__shfl_sync(0xffffffffu, my_x, u + t) * 32 + lane);
                else a[t] = make_float4(1, 1, 1, 1);
                if (RMW) y[t] = Y[(long)r * 32 + lane];
            }
#pragma unroll
            for (int t = 0; t < UNROLL; ++t) {
                const int r = __shfl_sync(0xffffffffu, my_y, u + t);
                float4 o = a[t];
                if (RMW) { o.x += y[t].x; o.y += y[t].y; o.z += y[t].z; o.w += y[t].w; }
                Y[(long)r * 32 + lane] = o;
            }
        }
    }
}

int main() {
    const long rows = 1l << 22, n = 4l << 20;  // 4 M updates of distinct random rows
    std::vector<int> hy(rows), hx(n);
    for (long i = 0; i < rows; ++i) hy[i] = (int)i;
    std::mt19937 rng(3);
    for (long i = rows - 1; i > 0; --i) std::swap(hy[i], hy[rng() % (i + 1)]);  // a permutation: rows unique
    for (long i = 0; i < n; ++i) hx[i] = (int)(rng() % rows);
    float4 *Y, *X;
    int *yi, *xi;
    unsigned *cnt;
    cudaMalloc(&Y, rows * 512);
    cudaMalloc(&X, rows * 512);
    cudaMemset(Y, 0, rows * 512);
    cudaMemset(X, 0, rows * 512);
    cudaMalloc(&yi, n * 4);
    cudaMalloc(&xi, n * 4);
    cudaMemcpy(yi, hy.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(xi, hx.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&cnt, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    char *flush;
    cudaMalloc(&flush, 512l << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char *name, int mode, int bps, double bytes_per_update) {
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
            cudaMemset(flush, rep, 512l << 20);  // evict Y and X from L2
            cudaMemset(cnt, 0, 4);
            cudaEventRecord(a);
            const int g = sms * bps;
            if (mode == 0) kern<8, false, false><<<g, 256>>>(Y, X, yi, xi, n, cnt);
            if (mode == 1) kern<8, false, true><<<g, 256>>>(Y, X, yi, xi, n, cnt);
            if (mode == 2) kern<8, true, true><<<g, 256>>>(Y, X, yi, xi, n, cnt);
            if (mode == 3) kern<4, true, true><<<g, 256>>>(Y, X, yi, xi, n, cnt);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-34s blocks/SM %d: %.3f ms  %.2f TB/s DRAM-side  %.1f M updates/ms\n", name, bps, best,
               n * bytes_per_update / best / 1e9, n / best / 1e6);
    };
    for (int bps : {4, 8}) {
        run("random row store", 0, bps, 512);
        run("random row RMW", 1, bps, 1024);
        run("random row RMW + random X gather", 2, bps, 1536);
        run("  (unroll 4)", 3, bps, 1536);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
