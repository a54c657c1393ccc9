// esirkepov.cu -- charge-conserving current deposition (Esirkepov 2001) on the
// staggered Yee grid, shape orders 1/2/3.  An EXTENSION of the reference:
// pic:: deposits J collocated on the nodes (proj/include/pic/deposit.hpp:60-73)
// and SPEC.md:8 lists charge-conserving schemes as future work, so there is
// no reference oracle.  The checker is this project's C restatement
// (oracle/picoracle.c po_deposit_esirkepov) and the discrete continuity
// equation (tests/test_esirkepov.py): with rho = q*w*S on the nodes (the
// reference-pinned deposit_density),
//   (rho(x1) - rho(x0)) / dt + div J = 0   to round-off.
//
// Per particle and axis the shape windows of the old and the new position
// (Shape<ORDER>: W nodes from cell + OFF, the reference's B-spline weights)
// are merged into one of L = W + 1 nodes (a step of less than one cell moves
// the base by at most one); DS = S1 - S0 there, and
//   Wx(i,j,k) = DSx(i) (S0y S0z + DSy S0z / 2 + S0y DSz / 2 + DSy DSz / 3)  (cyclic).
// J on the faces is the running sum of W along its axis times -q w h / dt;
// Jx(i + 1/2, j, k) is stored at node (i, j, k) of jx (likewise y, z).
//
// One thread per particle; the (L-1) L^2 face sums per component are flushed
// with RED.ADD.F64 (L2 atomics): QSP 3 x 100 reductions per particle.  This is
// a correctness-first kernel for the extension, not the measured hot path.
#include "common.cuh"
#include "kernels.hpp"

namespace picgpu {

namespace {

// Merged old/new window on one periodic axis; false if the cell step is not -1/0/+1.
template <int ORDER>
__device__ __forceinline__ bool axis_window(double x0, double x1, double o, double h, double inv, int pow2, int n,
                                            double (&S0)[Shape<ORDER>::W + 1], double (&D)[Shape<ORDER>::W + 1],
                                            int (&node)[Shape<ORDER>::W + 1]) {
    constexpr int W = Shape<ORDER>::W, L = W + 1, OFF = Shape<ORDER>::OFF;
    double f0, f1;
    const int c0 = locate_axis(x0, o, h, inv, pow2, n, f0);
    const int c1 = locate_axis(x1, o, h, inv, pow2, n, f1);
    int dc = c1 - c0;
    if (dc == n - 1) dc = -1;  // periodic: the step across the seam
    else if (dc == 1 - n) dc = 1;
    if (dc < -1 || dc > 1) return false;
    double a[W], b[W];
    int up;
    Shape<ORDER>::weights(f0, a, up);
    Shape<ORDER>::weights(f1, b, up);
    const int sh0 = dc < 0 ? 1 : 0, sh1 = dc > 0 ? 1 : 0;  // offsets of the two windows in the merged one
    const int lo = c0 + OFF - sh0;
#pragma unroll
    for (int t = 0; t < L; ++t) {
        const double s0 = (t - sh0 >= 0 && t - sh0 < W) ? a[t - sh0] : 0.0;
        const double s1 = (t - sh1 >= 0 && t - sh1 < W) ? b[t - sh1] : 0.0;
        S0[t] = s0;
        D[t] = s1 - s0;
        node[t] = wrap_index(lo + t, n);
    }
    return true;
}

template <int ORDER>
__global__ void __launch_bounds__(128) k_esirkepov(const GridD g, const double* __restrict__ x0,
                                                   const double* __restrict__ y0, const double* __restrict__ z0,
                                                   const double* __restrict__ x1, const double* __restrict__ y1,
                                                   const double* __restrict__ z1, const double* __restrict__ w,
                                                   double q, double dt, uint64_t n, double* __restrict__ jx,
                                                   double* __restrict__ jy, double* __restrict__ jz, int* err) {
    constexpr int L = Shape<ORDER>::W + 1;
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const double ax = x0[p], ay = y0[p], az = z0[p], bx = x1[p], by = y1[p], bz = z1[p];
    if (!finite3(ax, ay, az) || !finite3(bx, by, bz)) {
        raise_error(err, PICGPU_EINVAL);
        return;
    }
    double S0[3][L], D[3][L];
    int nd[3][L];
    if (!axis_window<ORDER>(ax, bx, g.ox, g.dx, g.inv_dx, g.pow2x, g.nx, S0[0], D[0], nd[0]) ||
        !axis_window<ORDER>(ay, by, g.oy, g.dy, g.inv_dy, g.pow2y, g.ny, S0[1], D[1], nd[1]) ||
        !axis_window<ORDER>(az, bz, g.oz, g.dz, g.inv_dz, g.pow2z, g.nz, S0[2], D[2], nd[2])) {
        raise_error(err, PICGPU_EDOMAIN);
        return;
    }
    const double qw = q * w[p];
    const double c[3] = {-qw * g.dx / dt, -qw * g.dy / dt, -qw * g.dz / dt};
    double* J[3] = {jx, jy, jz};
    const size_t sy = (size_t)g.nx, sz = (size_t)g.nx * (size_t)g.ny;
    // component a runs along axis a; (b, e) are the two transverse axes
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int b = a == 0 ? 1 : 0, e = a == 2 ? 1 : 2;
        const size_t st[3] = {1, sy, sz};
#pragma unroll
        for (int ke = 0; ke < L; ++ke)
#pragma unroll
            for (int kb = 0; kb < L; ++kb) {
                const double t = S0[b][kb] * S0[e][ke] + 0.5 * D[b][kb] * S0[e][ke] + 0.5 * S0[b][kb] * D[e][ke] +
                                 (1.0 / 3.0) * D[b][kb] * D[e][ke];
                if (t == 0.0) continue;
                const size_t base = (size_t)nd[b][kb] * st[b] + (size_t)nd[e][ke] * st[e];
                double run = 0.0;
#pragma unroll
                for (int i = 0; i < L - 1; ++i) {
                    run += D[a][i] * t;
                    if (run != 0.0) atomicAdd(J[a] + base + (size_t)nd[a][i] * st[a], c[a] * run);
                }
            }
    }
}

}  // namespace

void launch_deposit_esirkepov(int order, const GridD& g, const double* x0, const double* y0, const double* z0,
                              const double* x1, const double* y1, const double* z1, const double* w, double q,
                              double dt, uint64_t n, double* jx, double* jy, double* jz, int* err, cudaStream_t st) {
    if (!n) return;
    const unsigned blocks = (unsigned)((n + 127) / 128);
    switch (order) {
        case 1: k_esirkepov<1><<<blocks, 128, 0, st>>>(g, x0, y0, z0, x1, y1, z1, w, q, dt, n, jx, jy, jz, err); break;
        case 2: k_esirkepov<2><<<blocks, 128, 0, st>>>(g, x0, y0, z0, x1, y1, z1, w, q, dt, n, jx, jy, jz, err); break;
        default: k_esirkepov<3><<<blocks, 128, 0, st>>>(g, x0, y0, z0, x1, y1, z1, w, q, dt, n, jx, jy, jz, err); break;
    }
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

}  // namespace picgpu
