// HBM behaviour of the 64-byte record store access patterns (tools/, not the product):
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_probe hbm_probe.cu && ./hbm_probe [records]
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct Rec { double x, y, z, vx, vy, vz, w, id; };

template <int MODE, int UNR>
__global__ void __launch_bounds__(256) k(Rec* A, Rec* B, uint64_t n, double dt, int* sink) {
    const uint64_t base = ((uint64_t)blockIdx.x * blockDim.x * UNR) + threadIdx.x;
    double2 a[UNR], b[UNR], c[UNR], d[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
        const uint64_t i = base + (uint64_t)u * blockDim.x;
        if (i >= n) continue;
        if (MODE != 5) {
            const double2* r = reinterpret_cast<const double2*>(A + i);
            a[u] = r[0]; b[u] = r[1]; c[u] = r[2];
            if (MODE == 0 || MODE == 4 || MODE == 6) d[u] = r[3];
        }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
        const uint64_t i = base + (uint64_t)u * blockDim.x;
        if (i >= n) continue;
        double2* o = reinterpret_cast<double2*>(A + i);
        switch (MODE) {
            case 0: if (a[u].x + b[u].x + c[u].x + d[u].x == 12345.0) atomicAdd(sink, 1); break;   // read 64
            case 1: o[0] = make_double2(a[u].x + b[u].y * dt, a[u].y + c[u].x * dt);                  // read 48, write x y z
                    A[i].z = b[u].x + c[u].y * dt; break;
            case 2: o[0] = make_double2(a[u].x + b[u].y * dt, a[u].y + c[u].x * dt);                  // write sector 0 whole
                    o[1] = make_double2(b[u].x + c[u].y * dt, b[u].y); break;
            case 3: { double* p = reinterpret_cast<double*>(A + i);                                    // x y z via separate stores
                    p[0] = a[u].x + b[u].y * dt; p[1] = a[u].y + c[u].x * dt; p[2] = b[u].x + c[u].y * dt; } break;
            case 4: o[0] = make_double2(a[u].x + b[u].y * dt, a[u].y + c[u].x * dt);                  // read 64, write whole record
                    o[1] = make_double2(b[u].x + c[u].y * dt, b[u].y); o[2] = c[u]; o[3] = d[u]; break;
            case 5: { double2* q = reinterpret_cast<double2*>(B + i); const double2 v = make_double2(1.0, 2.0);  // write 64 only
                    q[0] = v; q[1] = v; q[2] = v; q[3] = v; } break;
            case 6: { double2* q = reinterpret_cast<double2*>(B + i); q[0] = a[u]; q[1] = b[u]; q[2] = c[u]; q[3] = d[u]; } break;  // copy
        }
    }
}

static size_t g_smem = 0;  // dynamic shared memory per CTA: limits CTAs (warps) per SM

template <int MODE, int UNR>
void run(const char* name, Rec* A, Rec* B, uint64_t n, double bytes_per, int* sink) {
    const unsigned blocks = (unsigned)((n + 256ull * UNR - 1) / (256ull * UNR));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaFuncSetAttribute(k<MODE, UNR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    k<MODE, UNR><<<blocks, 256, g_smem>>>(A, B, n, 0.0, sink);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) k<MODE, UNR><<<blocks, 256, g_smem>>>(A, B, n, 0.0, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    ms /= 3;
    printf("%-28s UNR %d smem %6zu  %8.3f ms  %7.1f GB/s\n", name, UNR, g_smem, ms, n * bytes_per / (ms * 1e-3) / 1e9);
}

int main(int argc, char** argv) {
    uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 400000000ull;
    Rec *A, *B; int* sink;
    if (cudaMalloc(&A, n * 64) || cudaMalloc(&B, n * 64) || cudaMalloc(&sink, 4)) { printf("alloc failed\n"); return 1; }
    cudaMemset(A, 0, n * 64); cudaMemset(B, 0, n * 64);
    printf("records %llu (%.1f GB each array)\n", (unsigned long long)n, n * 64 / 1e9);
    for (size_t sm : {(size_t)0, (size_t)50000, (size_t)70000, (size_t)100000}) {  // 8 / 4 / 3 / 2 CTAs of 256 per SM
        g_smem = sm;
        run<1, 1>("read 48 + write xyz in place", A, B, n, 48 + 24, sink);
        run<1, 2>("read 48 + write xyz in place", A, B, n, 48 + 24, sink);
    }
    g_smem = 0;
    run<0, 1>("read 64", A, B, n, 64, sink);
    run<0, 2>("read 64", A, B, n, 64, sink);
    run<1, 1>("read 48 + write xyz in place", A, B, n, 48 + 24, sink);
    run<1, 2>("read 48 + write xyz in place", A, B, n, 48 + 24, sink);
    run<2, 1>("read 48 + write sector 0", A, B, n, 48 + 32, sink);
    run<3, 1>("read 48 + 3 x STG.64", A, B, n, 48 + 24, sink);
    run<4, 1>("read 64 + write 64 in place", A, B, n, 128, sink);
    run<5, 1>("write 64", A, B, n, 64, sink);
    run<6, 1>("copy 64 A->B", A, B, n, 128, sink);
    run<6, 2>("copy 64 A->B", A, B, n, 128, sink);
    return 0;
}
