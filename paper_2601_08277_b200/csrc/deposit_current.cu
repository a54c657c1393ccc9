// deposit_current.cu -- sm_100a current deposition J = sum_p q W_p v_p S(x_i - x_p)
// at shape orders 1 (CIC), 2 (TSC, padded into a 4-tap window) and 3 (QSP).
//
// Replaces pic::deposit_scalar (proj/include/pic/deposit.hpp:62-73) and its
// MPU-tiled variants (deposit_tiled :284-334, rhocell :87-119).  The paper's
// block outer-product form J_cell = sum_p (wq_p*Sx_p) (x) (Sy_p (x) Sz_p)
// (tile.hpp:57-108) is kept, but recast for Blackwell:
//
//  * A CTA owns a PX x PY tile of cell "pencils" (x-y) and walks a z-chunk of
//    cells.  Particles are read from the cell bins maintained by the sorter
//    (sorter.cu), i.e. cell-local and coalesced.
//  * A group of G lanes owns one pencil.  Each lane owns a fixed sub-block of
//    the per-cell outer product (its ix/jy subset x 3 components) for a
//    sliding window of W z-planes held in REGISTERS: after the pencil's cell k
//    is done, plane k+OFF can receive nothing more from this pencil, so it is
//    emitted and the window slides.  The contraction over the cell's particles
//    therefore never touches shared or global memory (FP64 FMA in registers).
//  * Emitted planes of all pencils meet in a shared-memory patch buffer
//    (double-buffered, one __syncthreads per z-step); a gather pass sums the
//    overlapping W x W patches per node (no shared-memory atomics -- FP64
//    shared atomics are CAS loops on sm_100a) and flushes each node ONCE:
//    a plain store for nodes whose every contributing cell lies in this CTA,
//    a global FP64 reduction (RED.ADD.F64, native in L2) for halo nodes.
//
// J is compared with the reference at 1e-12 peak-normalised; it
// uses FMA and its own summation order.  Cell location and shape weights are
// bit-identical to the reference so the particle always belongs to its bin.
#include <algorithm>

#include "common.cuh"
#include "kernels.hpp"

namespace picgpu {

namespace {

template <int ORDER>
struct JCfg;
// CIC: one lane per pencil owns the whole 2x2x2x3 block (24 accumulators); no staging.
template <>
struct JCfg<1> {
    static constexpr int G = 1, NJ = 2, NI = 2, PX = 32, PY = 4, MINB = 4;
};
// TSC / QSP: 8 lanes per pencil, lane = (jy, ix-half): 1 jy x 2 ix x 3 comps x 4 planes = 24 acc.
template <>
struct JCfg<2> {
    static constexpr int G = 8, NJ = 1, NI = 2, PX = 8, PY = 4, MINB = 2;
};
template <>
struct JCfg<3> {
    static constexpr int G = 8, NJ = 1, NI = 2, PX = 8, PY = 4, MINB = 2;
};

template <int ORDER>
struct JLayout {
    using C = JCfg<ORDER>;
    static constexpr int W = Shape<ORDER>::W;
    static constexpr int NP = C::PX * C::PY;
    static constexpr int NT = NP * C::G;
    static constexpr int REC = 5 * W;                         // a[3][W] | sy[W] | sz[W]
    static constexpr int GSTRIDE = C::G * REC + 4;            // +32 B: de-alias groups across banks
    static constexpr int PATCH = NP * 3 * W * W;              // one buffer
    static constexpr int STAGE = C::G > 1 ? NP * GSTRIDE : 0;
    static constexpr size_t SMEM = (size_t)(2 * PATCH + STAGE) * sizeof(double);
};

// Per-particle prologue (shape.hpp:64-85 + particle_weights :46-50): the
// window weights and the x-weights pre-multiplied by wq_c = (q*W)*v_c.
template <int ORDER>
__device__ __forceinline__ void particle_window(const GridD& g, const CSoa& p, uint32_t s, double q,
                                                double (&a)[3][Shape<ORDER>::W], double (&sy)[Shape<ORDER>::W],
                                                double (&sz)[Shape<ORDER>::W]) {
    constexpr int W = Shape<ORDER>::W;
    const double x = p.x[s], y = p.y[s], z = p.z[s];
    const double qw = q * p.w[s];
    const double wq0 = qw * p.vx[s], wq1 = qw * p.vy[s], wq2 = qw * p.vz[s];
    double fx, fy, fz;
    int up;
    locate_axis(x, g.ox, g.dx, g.inv_dx, g.pow2x, g.nx, fx);
    locate_axis(y, g.oy, g.dy, g.inv_dy, g.pow2y, g.ny, fy);
    locate_axis(z, g.oz, g.dz, g.inv_dz, g.pow2z, g.nz, fz);
    double sx[W];
    Shape<ORDER>::weights(fx, sx, up);
    Shape<ORDER>::weights(fy, sy, up);
    Shape<ORDER>::weights(fz, sz, up);
#pragma unroll
    for (int t = 0; t < W; ++t) {
        a[0][t] = wq0 * sx[t];
        a[1][t] = wq1 * sx[t];
        a[2][t] = wq2 * sx[t];
    }
}

template <int ORDER>
__global__ void __launch_bounds__(JLayout<ORDER>::NT, JCfg<ORDER>::MINB)
    deposit_current_kernel(const GridD g, const CSoa p, const uint32_t* __restrict__ off,
                           const uint32_t* __restrict__ cnt, const double q, double* __restrict__ jx,
                           double* __restrict__ jy, double* __restrict__ jz, const int zlen) {
    using C = JCfg<ORDER>;
    using L = JLayout<ORDER>;
    constexpr int W = L::W, OFF = Shape<ORDER>::OFF;
    constexpr int G = C::G, NJ = C::NJ, NI = C::NI, PX = C::PX, PY = C::PY;
    constexpr int JS = W / NJ;  // lanes splitting jy
    constexpr int FX = PX + W - 1, FY = PY + W - 1;

    extern __shared__ __align__(16) double smem[];
    double* patch = smem;                 // [2][NP][3][W(jy)][W(ix)]
    double* stage = smem + 2 * L::PATCH;  // [NP][GSTRIDE]

    const int tid = threadIdx.x;
    const int grp = tid / G, lg = tid % G;
    const int px = grp % PX, py = grp / PX;
    const int i0 = blockIdx.x * PX, j0 = blockIdx.y * PY;
    const int k0 = blockIdx.z * zlen;
    const int k1 = min(k0 + zlen, g.nz);
    const int i = i0 + px, j = j0 + py;
    const bool pv = (i < g.nx) && (j < g.ny);
    const int jsub = lg % JS, isub = lg / JS;
    const int pxv = min(PX, g.nx - i0), pyv = min(PY, g.ny - j0);
    const bool alias_xy = (pxv + W - 1 > g.nx) || (pyv + W - 1 > g.ny);

    double acc[W][NJ][NI][3];
#pragma unroll
    for (int kz = 0; kz < W; ++kz)
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
            for (int ii = 0; ii < NI; ++ii)
#pragma unroll
                for (int c = 0; c < 3; ++c) acc[kz][jj][ii][c] = 0.0;

    int buf = 0;
    for (int k = k0; k < k1 + W - 1; ++k) {
        if (k < k1) {
            uint32_t c_off = 0;
            int n_c = 0;
            if (pv) {
                const uint32_t c = (uint32_t)i + (uint32_t)g.nx * ((uint32_t)j + (uint32_t)g.ny * (uint32_t)k);
                c_off = off[c];
                n_c = (int)cnt[c];
            }
            if constexpr (G == 1) {
                for (int t = 0; t < n_c; ++t) {
                    double a[3][W], sy[W], sz[W];
                    particle_window<ORDER>(g, p, c_off + t, q, a, sy, sz);
#pragma unroll
                    for (int kz = 0; kz < W; ++kz)
#pragma unroll
                        for (int jj = 0; jj < NJ; ++jj) {
                            const double b = sy[jsub * NJ + jj] * sz[kz];
#pragma unroll
                            for (int ii = 0; ii < NI; ++ii)
#pragma unroll
                                for (int c = 0; c < 3; ++c)
                                    acc[kz][jj][ii][c] = fma(a[c][isub * NI + ii], b, acc[kz][jj][ii][c]);
                        }
                }
            } else {
                const int m = (int)__reduce_max_sync(0xffffffffu, (unsigned)n_c);
                double* gstage = stage + grp * L::GSTRIDE;
                for (int base = 0; base < m; base += G) {
                    {
                        double* rec = gstage + lg * L::REC;
                        const int idx = base + lg;
                        double a[3][W], sy[W], sz[W];
                        if (idx < n_c) {
                            particle_window<ORDER>(g, p, c_off + idx, q, a, sy, sz);
                        } else {
#pragma unroll
                            for (int t = 0; t < W; ++t) {
                                a[0][t] = a[1][t] = a[2][t] = 0.0;
                                sy[t] = sz[t] = 0.0;
                            }
                        }
                        // a grouped by ix-subset so a lane reads its 3*NI values contiguously
#pragma unroll
                        for (int is = 0; is < W / NI; ++is)
#pragma unroll
                            for (int c = 0; c < 3; ++c)
#pragma unroll
                                for (int ii = 0; ii < NI; ++ii) rec[is * 3 * NI + c * NI + ii] = a[c][is * NI + ii];
#pragma unroll
                        for (int t = 0; t < W; ++t) {
                            rec[3 * W + t] = sy[t];
                            rec[4 * W + t] = sz[t];
                        }
                    }
                    __syncwarp();
                    const int nn = min(G, m - base);
                    for (int jj0 = 0; jj0 < nn; ++jj0) {
                        const double* r = gstage + jj0 * L::REC;
                        double av[3 * NI];
                        const double2* ap = reinterpret_cast<const double2*>(r + isub * 3 * NI);
#pragma unroll
                        for (int u = 0; u < 3 * NI / 2; ++u) {
                            const double2 v = ap[u];
                            av[2 * u] = v.x;
                            av[2 * u + 1] = v.y;
                        }
                        double syv[NJ];
#pragma unroll
                        for (int jj = 0; jj < NJ; ++jj) syv[jj] = r[3 * W + jsub * NJ + jj];
                        double szv[W];
                        const double2* zp = reinterpret_cast<const double2*>(r + 4 * W);
#pragma unroll
                        for (int u = 0; u < W / 2; ++u) {
                            const double2 v = zp[u];
                            szv[2 * u] = v.x;
                            szv[2 * u + 1] = v.y;
                        }
#pragma unroll
                        for (int kz = 0; kz < W; ++kz)
#pragma unroll
                            for (int jj = 0; jj < NJ; ++jj) {
                                const double b = syv[jj] * szv[kz];
#pragma unroll
                                for (int ii = 0; ii < NI; ++ii)
#pragma unroll
                                    for (int c = 0; c < 3; ++c)
                                        acc[kz][jj][ii][c] = fma(av[c * NI + ii], b, acc[kz][jj][ii][c]);
                            }
                    }
                    __syncwarp();
                }
            }
        }

        // Plane k+OFF is final for this pencil: emit it, slide the window.
        {
            double* pp = patch + (buf * L::NP + grp) * (3 * W * W);
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
                    for (int ii = 0; ii < NI; ++ii)
                        pp[(c * W + jsub * NJ + jj) * W + isub * NI + ii] = acc[0][jj][ii][c];
#pragma unroll
            for (int kz = 0; kz < W - 1; ++kz)
#pragma unroll
                for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
                    for (int ii = 0; ii < NI; ++ii)
#pragma unroll
                        for (int c = 0; c < 3; ++c) acc[kz][jj][ii][c] = acc[kz + 1][jj][ii][c];
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
                for (int ii = 0; ii < NI; ++ii)
#pragma unroll
                    for (int c = 0; c < 3; ++c) acc[W - 1][jj][ii][c] = 0.0;
        }
        __syncthreads();

        // Gather the overlapping pencil patches of plane Z and flush each node once.
        {
            const double* pb = patch + buf * L::NP * (3 * W * W);
            const int Z = wrap_index(k + OFF, g.nz);
            const bool zc = (k >= k0 + W - 1) && (k < k1);  // every contributing cell is in [k0, k1)
            const size_t zrow = (size_t)g.ny * (size_t)Z;
            for (int it = tid; it < 3 * FX * FY; it += L::NT) {
                const int c = it / (FX * FY);
                const int r = it - c * (FX * FY);
                const int uy = r / FX, ux = r - uy * FX;
                if (ux >= pxv + W - 1 || uy >= pyv + W - 1) continue;
                double s = 0.0;
#pragma unroll
                for (int dy = 0; dy < W; ++dy) {
                    const int qy = uy - dy;
                    if (qy < 0 || qy >= pyv) continue;
#pragma unroll
                    for (int dx = 0; dx < W; ++dx) {
                        const int qx = ux - dx;
                        if (qx < 0 || qx >= pxv) continue;
                        s += pb[((qy * PX + qx) * 3 + c) * W * W + dy * W + dx];
                    }
                }
                const int X = wrap_index(i0 + OFF + ux, g.nx);
                const int Y = wrap_index(j0 + OFF + uy, g.ny);
                const size_t node = (size_t)X + (size_t)g.nx * ((size_t)Y + zrow);
                double* f = c == 0 ? jx : (c == 1 ? jy : jz);
                const bool interior = zc && !alias_xy && ux >= W - 1 && ux <= pxv - 1 && uy >= W - 1 && uy <= pyv - 1;
                if (interior)
                    f[node] = s;
                else if (s != 0.0)
                    atomicAdd(f + node, s);
            }
        }
        buf ^= 1;
    }
}

template <int ORDER>
void launch_order(const GridD& g, const CSoa& p, const uint32_t* off, const uint32_t* cnt, double q, double* j,
                  int num_sms, cudaStream_t st) {
    using C = JCfg<ORDER>;
    using L = JLayout<ORDER>;
    constexpr int W = L::W;
    static bool configured = false;
    if (!configured) {
        PICGPU_CUDA_TRY(cudaFuncSetAttribute(deposit_current_kernel<ORDER>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM));
        configured = true;
    }
    const int tx = div_up(g.nx, C::PX), ty = div_up(g.ny, C::PY);
    // z-chunks: enough CTAs for several waves on every SM, but chunks of at
    // least 4*W cells so most planes are complete (plain stores, no RED).
    const long long tiles = (long long)tx * ty;
    const long long target = (long long)num_sms * C::MINB * 4;
    int zch = (int)std::max<long long>(1, (target + tiles - 1) / tiles);
    zch = std::min(zch, std::max(1, g.nz / (4 * W)));
    const int zlen = div_up(g.nz, zch);
    zch = div_up(g.nz, zlen);
    dim3 grid(tx, ty, zch);
    deposit_current_kernel<ORDER><<<grid, L::NT, L::SMEM, st>>>(g, p, off, cnt, q, j, j + g.ncells,
                                                                j + 2 * (size_t)g.ncells, zlen);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

}  // namespace

// J must be zeroed by the caller (halo nodes are reduced into it).
void launch_deposit_current(int order, const GridD& g, const CSoa& p, const uint32_t* off, const uint32_t* cnt,
                            double q, double* j, int num_sms, cudaStream_t st) {
    switch (order) {
        case 1: launch_order<1>(g, p, off, cnt, q, j, num_sms, st); break;
        case 2: launch_order<2>(g, p, off, cnt, q, j, num_sms, st); break;
        case 3: launch_order<3>(g, p, off, cnt, q, j, num_sms, st); break;
        default: throw Status{PICGPU_EINVAL, "deposit: shape order must be 1, 2 or 3"};
    }
}

}  // namespace picgpu
