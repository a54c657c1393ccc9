// Microbenchmark: FP64 DMMA (mma.sync m8n8k4 f64) vs DFMA throughput on sm_100a.
// Decides whether the per-cell outer-product contraction belongs on the FP64
// tensor pipe (north_star part 2: "DMMA only if it beats the smem/DFMA path").
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 1.2345) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
    double r[8];
    for (int i = 0; i < 8; ++i) r[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) r[i] = fma(r[i], 0.999, 1e-3);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += r[i];
    if (s == 1.2345) out[0] = s;
}

// Mixed: DMMA and DFMA interleaved in the same warp (do the pipes overlap?)
__global__ void mixed_loop(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
    double c[4][2];
    double r[8];
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
    for (int i = 0; i < 8; ++i) r[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) r[i] = fma(r[i], 0.999, 1e-3);
    }
    double s = 0;
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
    for (int i = 0; i < 8; ++i) s += r[i];
    if (s == 1.2345) out[0] = s;
}

template <class K>
float timeit(K kernel, int blocks, int threads, int iters, double* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kernel<<<blocks, threads>>>(out, 16);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 64);
    const int iters = 2048;
    for (int warps : {4, 8, 16, 32}) {
        const int blocks = sms * 2, threads = warps * 32 / 2;
        float ms = timeit(dmma_loop, blocks, threads, iters, out);
        double macs = 256.0 * 8 * iters * (blocks * threads / 32.0);
        printf("DMMA  warps/SM=%2d  %.2f TFLOP/s (%.1f MAC/clk/SM @1965)\n", warps, 2 * macs / ms / 1e9,
               macs / (ms * 1e-3) / sms / 1.965e9);
        ms = timeit(dfma_loop, blocks, threads, iters, out);
        double fmas = 64.0 * iters * blocks * threads;
        printf("DFMA  warps/SM=%2d  %.2f TFLOP/s (%.1f FMA/clk/SM)\n", warps, 2 * fmas / ms / 1e9,
               fmas / (ms * 1e-3) / sms / 1.965e9);
        ms = timeit(mixed_loop, blocks, threads, iters, out);
        double mix = (256.0 * 4 + 32.0 * 32) * iters * (blocks * threads / 32.0);
        printf("MIXED warps/SM=%2d  %.2f TFLOP/s (%.1f MAC/clk/SM)\n", warps, 2 * mix / ms / 1e9,
               mix / (ms * 1e-3) / sms / 1.965e9);
    }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
