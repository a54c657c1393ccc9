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
//  * G lanes own one pencil.  Lane l owns the jy-slice(s) of the per-cell outer
//    product for ALL ix, all 3 components and a sliding window of W z-planes,
//    held in REGISTERS (QSP: 4 ix x 3 c x 4 kz = 48 accumulators).  After the
//    pencil's cell k is done, plane k+OFF can receive nothing more from it, so
//    it is emitted and the window slides.  The contraction over a cell's
//    particles never touches shared or global memory: per particle a lane
//    reads 12+1+4 staged weights (conflict-free LDS.128) and issues 4 DMUL +
//    48 DFMA.  (FP64 DMMA was measured at the same 64 MAC/clk/SM as DFMA on
//    B200 -- tools/fp64_pipes.cu -- and would pad the 12x16 block to 16x16,
//    so the register-blocked DFMA form is the faster one.)
//  * Emitted planes of all pencils meet in a shared-memory patch buffer
//    (double-buffered, one __syncthreads per z-step); a gather pass sums the
//    overlapping W x W patches per node (no shared-memory atomics -- FP64
//    shared atomics are CAS loops on sm_100a) and flushes each node ONCE:
//    a plain store for nodes whose every contributing cell lies in this CTA,
//    a global FP64 reduction (RED.ADD.F64, native in L2) for halo nodes.
//  * The fused form (launch_deposit_current_push, the default session step)
//    runs pic::advance (deposit.hpp / simulation.hpp) inside the same pass:
//    each staged particle is pushed bit-exactly in registers and written back;
//    a particle that stays in its cell deposits on the register window as
//    above, a particle that moved one cell has its taps shifted into the old
//    cell's window where they fit, and is listed in its CTA's mover segment
//    (shared-memory reservation) for k_movers, which moves its record, leaves
//    a hole, and deposits the taps outside the window with RED.ADD.F64.
//
// J is compared with the reference at 1e-12 peak-normalised; it
// uses FMA and its own summation order.  Cell location and shape weights are
// bit-identical to the reference so the particle always belongs to its bin.
#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "kernels.hpp"

namespace picgpu {

namespace {

template <int ORDER>
struct JCfg;
// CIC: one lane per pencil owns the whole 2x2x2x3 block (24 accumulators) and
// reads its own particles (no staging; the order is HBM-bound).
template <>
struct JCfg<1> {
    static constexpr int G = 1, PX = 32, PY = 4, MINB = 4, CH = 1;
};
// QSP/TSC with 8 lanes per pencil (lane = jy x x-half, 24 accumulators each):
// fewer registers per thread, more warps per SM, more shared loads per FMA.
#ifndef PICGPU_G8_PX
#define PICGPU_G8_PX 4
#endif
#ifndef PICGPU_G8_PY
#define PICGPU_G8_PY 4
#endif
#ifndef PICGPU_G8_MINB
#define PICGPU_G8_MINB 4
#endif
struct JCfgG8 {
    static constexpr int G = 8, PX = PICGPU_G8_PX, PY = PICGPU_G8_PY, MINB = PICGPU_G8_MINB, CH = 8;
};
// CIC on the v3 kernel: 2 lanes per pencil (lane = jy), 12 accumulators each.
#ifndef PICGPU_CIC_PX
#define PICGPU_CIC_PX 16
#endif
#ifndef PICGPU_CIC_PY
#define PICGPU_CIC_PY 4
#endif
#ifndef PICGPU_CIC_MINB
#define PICGPU_CIC_MINB 4
#endif
struct JCfgCic3 {
    static constexpr int G = 2, PX = PICGPU_CIC_PX, PY = PICGPU_CIC_PY, MINB = PICGPU_CIC_MINB, CH = 2;
};
// TSC / QSP, "lane" variant: 4 lanes per pencil (lane = jy), 8 pencils per
// warp, 48 accumulators per lane (4 ix x 3 c x 4 kz).
#ifndef PICGPU_LANE_MINB
#define PICGPU_LANE_MINB 3
#endif
#ifndef PICGPU_LANE_PX
#define PICGPU_LANE_PX 8
#endif
#ifndef PICGPU_LANE_UNROLL
#define PICGPU_LANE_UNROLL 1
#endif
constexpr int kLaneUnroll = PICGPU_LANE_UNROLL;
#ifndef PICGPU_LANE_PY
#define PICGPU_LANE_PY 4
#endif
template <>
struct JCfg<2> {
    static constexpr int G = 4, PX = PICGPU_LANE_PX, PY = PICGPU_LANE_PY, MINB = PICGPU_LANE_MINB, CH = 4;
};
template <>
struct JCfg<3> {
    static constexpr int G = 4, PX = PICGPU_LANE_PX, PY = PICGPU_LANE_PY, MINB = PICGPU_LANE_MINB, CH = 4;
};

template <int ORDER, class CF = JCfg<ORDER>>
struct JLayout {
    using C = CF;
    static constexpr int W = Shape<ORDER>::W;
    static constexpr int NJ = W / C::G;                 // jy values per lane
    static constexpr int NP = C::PX * C::PY;            // pencils per CTA
    static constexpr int NT = NP * C::G;                // threads per CTA
    // Field-major staging: field f (a[c][ix] = c*W+ix, sy[t] = 3W+t, sz[t] =
    // 4W+t) of chunk position l of pencil grp at [f*FSS + l*SS + grp].  SS =
    // NP + 4 makes the writes of a half-warp (4 pencils x 4 positions) hit 16
    // distinct banks and the reads (8 pencils, same position) contiguous.
    static constexpr int NF = 5 * W;
    static constexpr int SS = NP + 4;
    static constexpr int FSS = C::CH * SS;
    static constexpr int STAGE = C::G > 1 ? NF * FSS : 0;
    // v3 stages fields in PAIRS (16 bytes: one LDS.128 reads two taps): pair
    // f/2 of chunk position l of pencil grp at 16-byte unit (f/2)*PFS + l*PSS +
    // grp.  PSS = NP + 2 (2 mod 8 units) keeps a quarter-warp's writes (2
    // pencils x 4 positions) in distinct banks; a warp's reads (8 pencils, one
    // position) are 128 contiguous bytes.
    static constexpr int PSS = NP + 2;
    static constexpr int PFS = C::CH * PSS;
    static_assert(NF % 2 == 0 && (NF / 2) * PFS * 2 <= NF * FSS, "paired staging fits the v1 staging area");
    // v3: PPB emitted planes per CTA barrier (double-buffered), paired staging.
    // C2 QSP: PPB 1 / 2 / 4 -> J 1.177 / 1.171 / 2.03 ms (4: 2 CTAs/SM), fused
    // step kernel 1.681 / 1.698 / 3.29 ms: one plane per barrier
#ifdef PICGPU_V3_PPB
    static constexpr int PPB = PICGPU_V3_PPB;
#else
    static constexpr int PPB = 1;
#endif
    static constexpr int STAGE3 = C::G > 1 ? (NF / 2) * PFS * 2 : 0;

    // One emitted plane of every pencil, offset-major: [jy][ix][c][PY][PX] with
    // a 2-double skew per (jy,ix,c) row so the 4 jy-lanes of a pencil write
    // to distinct banks and the gather reads consecutive pencils contiguously.
    static constexpr int PSTRIDE = NP + 2;
    static constexpr int PATCH = W * W * 3 * PSTRIDE;
    static constexpr size_t SMEM = (size_t)(2 * PATCH + STAGE) * sizeof(double);
    static constexpr size_t SMEM3 = (size_t)(2 * PPB * PATCH + STAGE3) * sizeof(double);
};

struct PData {  // one particle as read from the bins
    double x, y, z, vx, vy, vz, w;
};

// One particle record: x y | z vx | vy vz | w as three 16-byte loads and one
// 8-byte load (id is not needed).  RW: the kernel writes the positions back
// (fused step): coherent loads, not the read-only path.
template <bool RW = false>
__device__ __forceinline__ void load_particle(const CAos& p, uint32_t s, PData& d) {
    const double2* r = reinterpret_cast<const double2*>(p.p + s);
    double2 a, b, c;
    if constexpr (RW) {
        a = r[0];
        b = r[1];
        c = r[2];
        d.w = p.p[s].w;
    } else {
        a = __ldg(r);
        b = __ldg(r + 1);
        c = __ldg(r + 2);
        d.w = __ldg(&p.p[s].w);
    }
    d.x = a.x;
    d.y = a.y;
    d.z = b.x;
    d.vx = b.y;
    d.vy = c.x;
    d.vz = c.y;
}

// Per-particle prologue (shape.hpp:64-85 + particle_weights :46-50): the
// window weights and the x-weights pre-multiplied by wq_c = (q*W)*v_c.
template <int ORDER>
__device__ __forceinline__ void particle_window(const GridD& g, const PData& d, double q,
                                                double (&a)[3][Shape<ORDER>::W], double (&sy)[Shape<ORDER>::W],
                                                double (&sz)[Shape<ORDER>::W]) {
    constexpr int W = Shape<ORDER>::W;
    const double qw = q * d.w;
    const double wq0 = qw * d.vx, wq1 = qw * d.vy, wq2 = qw * d.vz;
    double fx, fy, fz;
    int up;
    locate_x(g, d.x, fx);
    locate_axis(d.y, g.oy, g.dy, g.inv_dy, g.pow2y, g.ny, fy);
    locate_axis(d.z, g.oz, g.dz, g.inv_dz, g.pow2z, g.nz, fz);
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

// J-only prologue: same cell location (bit-identical locate_axis, so the
// particle is in its bin's cell), weights evaluated with FMA-contracted
// polynomials (J is compared at 1e-12; rho keeps the exact forms).
template <int ORDER>
__device__ __forceinline__ void weights_fast(double d, double (&s)[4]) {
    if constexpr (ORDER == 3) {
        const double t2 = d * d, t3 = t2 * d, u = 1.0 - d;
        s[0] = u * u * u * (1.0 / 6.0);
        s[1] = fma(0.5, t3, fma(-1.0, t2, 2.0 / 3.0));
        s[2] = fma(-0.5, t3, fma(0.5, t2, fma(0.5, d, 1.0 / 6.0)));
        s[3] = t3 * (1.0 / 6.0);
    } else {
        const bool up = d >= 0.5;
        const double dl = up ? d - 1.0 : d;
        const double a = 0.5 - dl, b = 0.5 + dl;
        const double w0 = 0.5 * a * a, w1 = fma(-dl, dl, 0.75), w2 = 0.5 * b * b;
        s[0] = up ? 0.0 : w0;
        s[1] = up ? w0 : w1;
        s[2] = up ? w1 : w2;
        s[3] = up ? w2 : 0.0;
    }
}

template <int ORDER>
__device__ __forceinline__ void particle_window_fast(const GridD& g, const PData& d, double q, double (&a)[3][4],
                                                     double (&sy)[4], double (&sz)[4]) {
    const double qw = q * d.w;
    const double wq0 = qw * d.vx, wq1 = qw * d.vy, wq2 = qw * d.vz;
    double fx, fy, fz;
    locate_x(g, d.x, fx);
    locate_axis(d.y, g.oy, g.dy, g.inv_dy, g.pow2y, g.ny, fy);
    locate_axis(d.z, g.oz, g.dz, g.inv_dz, g.pow2z, g.nz, fz);
    double sx[4];
    weights_fast<ORDER>(fx, sx);
    weights_fast<ORDER>(fy, sy);
    weights_fast<ORDER>(fz, sz);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        a[0][t] = wq0 * sx[t];
        a[1][t] = wq1 * sx[t];
        a[2][t] = wq2 * sx[t];
    }
}

// Fractional coordinate of a binned particle relative to its bin's cell
// index `ci` (one FMA-free sub/mul per axis instead of floor/convert/branches).
// Exact when the spacing is a power of two; otherwise within an ulp, which
// only perturbs J at the 1e-16 level.  A position that is not inside its bin's
// cell (periodic image after an upload of unwrapped positions) takes the exact
// locate_axis path.
__device__ __forceinline__ double frac_in_cell(double x, double origin, double spacing, double inv, int pow2, int n,
                                               int ci) {
    const double u = (x - origin) * inv;
    const double f = u - (double)ci;
    if (f >= -0.5 && f <= 1.5) return f;
    double fr;
    locate_axis(x, origin, spacing, inv, pow2, n, fr);
    return fr;
}

// J prologue for a particle binned in cell (ci, cj, ck): window weights with
// FMA polynomials and x-weights pre-multiplied by wq_c = (q*W)*v_c.
template <int ORDER>
__device__ __forceinline__ void particle_window_cell(const GridD& g, const PData& d, double q, int ci, int cj, int ck,
                                                     double (&a)[3][Shape<ORDER>::W], double (&sy)[Shape<ORDER>::W],
                                                     double (&sz)[Shape<ORDER>::W]) {
    constexpr int W = Shape<ORDER>::W;
    const double qw = q * d.w;
    const double wq0 = qw * d.vx, wq1 = qw * d.vy, wq2 = qw * d.vz;
    const double fx = frac_in_cell(d.x, g.gox, g.dx, g.inv_dx, g.pow2x, g.gnx, ci + g.sx_shift);
    const double fy = frac_in_cell(d.y, g.oy, g.dy, g.inv_dy, g.pow2y, g.ny, cj);
    const double fz = frac_in_cell(d.z, g.oz, g.dz, g.inv_dz, g.pow2z, g.nz, ck);
    double sx[W];
    if constexpr (ORDER == 1) {
        sx[0] = 1.0 - fx; sx[1] = fx;
        sy[0] = 1.0 - fy; sy[1] = fy;
        sz[0] = 1.0 - fz; sz[1] = fz;
    } else {
        weights_fast<ORDER>(fx, sx);
        weights_fast<ORDER>(fy, sy);
        weights_fast<ORDER>(fz, sz);
    }
#pragma unroll
    for (int t = 0; t < W; ++t) {
        a[0][t] = wq0 * sx[t];
        a[1][t] = wq1 * sx[t];
        a[2][t] = wq2 * sx[t];
    }
}

template <int W, int NJ>
__device__ __forceinline__ void accumulate(double (&acc)[W][NJ][W][3], const double (&a)[3][W], const double (&syv)[NJ],
                                           const double (&sz)[W]) {
#pragma unroll
    for (int kz = 0; kz < W; ++kz)
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) {
            const double b = syv[jj] * sz[kz];
#pragma unroll
            for (int ix = 0; ix < W; ++ix)
#pragma unroll
                for (int c = 0; c < 3; ++c) acc[kz][jj][ix][c] = fma(a[c][ix], b, acc[kz][jj][ix][c]);
        }
}

template <int ORDER>
__global__ void __launch_bounds__(JLayout<ORDER>::NT, JCfg<ORDER>::MINB)
    deposit_current_kernel(const GridD g, const CAos p, const uint32_t* __restrict__ off,
                           const uint32_t* __restrict__ cnt, const double q, double* __restrict__ jx,
                           double* __restrict__ jy, double* __restrict__ jz, const int zlen) {
    using C = JCfg<ORDER>;
    using L = JLayout<ORDER>;
    constexpr int W = L::W, OFF = Shape<ORDER>::OFF, NJ = L::NJ;
    constexpr int G = C::G, PX = C::PX, PY = C::PY, CH = C::CH;
    constexpr int FX = PX + W - 1, FY = PY + W - 1;

    extern __shared__ __align__(16) double smem[];
    double* patch = smem;                 // [2][W(jy)][W(ix)][3][PSTRIDE]
    double* stage = smem + 2 * L::PATCH;  // [NF][CH][SS]

    const int tid = threadIdx.x;
    const int grp = tid / G, lg = tid % G;
    const int px = grp % PX, py = grp / PX;
    const int i0 = blockIdx.x * PX, j0 = blockIdx.y * PY;
    const int k0 = blockIdx.z * zlen;
    const int k1 = min(k0 + zlen, g.nz);
    const int i = i0 + px, j = j0 + py;
    const bool pv = (i < g.nx) && (j < g.ny);
    const int pxv = min(PX, g.nx - i0), pyv = min(PY, g.ny - j0);
    const bool alias_xy = (pxv + W - 1 > g.nx) || (pyv + W - 1 > g.ny);
    const uint32_t col = (uint32_t)i + (uint32_t)g.nx * (uint32_t)j;
    const uint32_t plane_cells = (uint32_t)g.nx * (uint32_t)g.ny;

    double acc[W][NJ][W][3];
#pragma unroll
    for (int kz = 0; kz < W; ++kz)
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
            for (int ix = 0; ix < W; ++ix)
#pragma unroll
                for (int c = 0; c < 3; ++c) acc[kz][jj][ix][c] = 0.0;

    // bin of this pencil's current cell, and a prefetched particle for the
    // next chunk (loads of chunk n+1 are in flight while chunk n is consumed)
    uint32_t c_off = 0;
    int n_c = 0;
    if (pv && k0 < k1) {
        c_off = off[col + plane_cells * k0];
        n_c = (int)cnt[col + plane_cells * k0];
    }
    PData nxt{};
    if constexpr (G > 1) {
        if (lg < n_c) load_particle(p, c_off + lg, nxt);
    }

    int buf = 0;
    for (int k = k0; k < k1 + W - 1; ++k) {
        if (k < k1) {
            // bin of the next cell (for the cross-cell prefetch)
            uint32_t n_off = 0;
            int n_n = 0;
            if (pv && k + 1 < k1) {
                n_off = off[col + plane_cells * (k + 1)];
                n_n = (int)cnt[col + plane_cells * (k + 1)];
            }
            if constexpr (G == 1) {
                for (int t = 0; t < n_c; ++t) {
                    PData d;
                    load_particle(p, c_off + t, d);
                    if (is_gap(d.x)) continue;  // a hole of the bin (GPMA gap)
                    double a[3][W], sy[W], sz[W];
                    particle_window_cell<ORDER>(g, d, q, i, j, k, a, sy, sz);
                    double syv[NJ];
#pragma unroll
                    for (int jj = 0; jj < NJ; ++jj) syv[jj] = sy[jj];
                    accumulate<W, NJ>(acc, a, syv, sz);
                }
            } else {
                const int m = (int)__reduce_max_sync(0xffffffffu, (unsigned)n_c);
                if (m == 0 && lg < n_n) load_particle(p, n_off + lg, nxt);  // empty cells: still prefetch
                for (int base = 0; base < m; base += CH) {
                    // prologue of this lane's particle -> staging slot (lg, grp)
                    {
                        const PData cur = nxt;
                        const bool valid = base + lg < n_c && !is_gap(cur.x);  // holes count as padding
                        // prefetch the next chunk: same cell, or the next cell's first chunk
                        if (base + CH < m) {
                            if (base + CH + lg < n_c) load_particle(p, c_off + base + CH + lg, nxt);
                        } else if (lg < n_n) {
                            load_particle(p, n_off + lg, nxt);
                        }
                        double a[3][W], sy[W], sz[W];
                        if (valid) {
                            particle_window_cell<ORDER>(g, cur, q, i, j, k, a, sy, sz);
                        } else {
#pragma unroll
                            for (int t = 0; t < W; ++t) a[0][t] = a[1][t] = a[2][t] = sy[t] = sz[t] = 0.0;
                        }
                        double* rec = stage + lg * L::SS + grp;
#pragma unroll
                        for (int c = 0; c < 3; ++c)
#pragma unroll
                            for (int t = 0; t < W; ++t) rec[(c * W + t) * L::FSS] = a[c][t];
#pragma unroll
                        for (int t = 0; t < W; ++t) {
                            rec[(3 * W + t) * L::FSS] = sy[t];
                            rec[(4 * W + t) * L::FSS] = sz[t];
                        }
                    }
                    __syncwarp();
                    const int nn = min(CH, m - base);
#pragma unroll kLaneUnroll
                    for (int jj0 = 0; jj0 < nn; ++jj0) {
                        const double* r = stage + jj0 * L::SS + grp;
                        double b[W][NJ];
#pragma unroll
                        for (int kz = 0; kz < W; ++kz) {
                            const double z = r[(4 * W + kz) * L::FSS];
#pragma unroll
                            for (int jj = 0; jj < NJ; ++jj) b[kz][jj] = r[(3 * W + lg * NJ + jj) * L::FSS] * z;
                        }
#pragma unroll
                        for (int c = 0; c < 3; ++c)
#pragma unroll
                            for (int ix = 0; ix < W; ++ix) {
                                const double av = r[(c * W + ix) * L::FSS];
#pragma unroll
                                for (int kz = 0; kz < W; ++kz)
#pragma unroll
                                    for (int jj = 0; jj < NJ; ++jj)
                                        acc[kz][jj][ix][c] = fma(av, b[kz][jj], acc[kz][jj][ix][c]);
                            }
                    }
                    __syncwarp();
                }
            }
            c_off = n_off;
            n_c = n_n;
        }

        // Plane k+OFF is final for this pencil: emit it, slide the window.
        {
            double* pp = patch + buf * L::PATCH + grp;
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
                    for (int ix = 0; ix < W; ++ix)
                        pp[(((lg * NJ + jj) * W + ix) * 3 + c) * L::PSTRIDE] = acc[0][jj][ix][c];
#pragma unroll
            for (int kz = 0; kz < W - 1; ++kz)
#pragma unroll
                for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
                    for (int ix = 0; ix < W; ++ix)
#pragma unroll
                        for (int c = 0; c < 3; ++c) acc[kz][jj][ix][c] = acc[kz + 1][jj][ix][c];
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
                for (int ix = 0; ix < W; ++ix)
#pragma unroll
                    for (int c = 0; c < 3; ++c) acc[W - 1][jj][ix][c] = 0.0;
        }
        __syncthreads();

        // Gather the overlapping pencil patches of plane Z and flush each node once.
        {
            const double* pb = patch + buf * L::PATCH;
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
                        s += pb[((dy * W + dx) * 3 + c) * L::PSTRIDE + qy * PX + qx];
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

// ---------------------------------------------------------------------------
// Orders 2 and 3, "lane" kernel v3 (default): the same decomposition as
// deposit_current_kernel (8x4 pencils per CTA, lane = jy, 48 accumulators per
// lane), with the per-z-step overheads taken out:
//  * the z loop is unrolled by W = 4 and the window slides by static register
//    rotation (logical plane kz lives in physical slot (kz + R) & 3 at step R),
//    so no accumulator is moved when a plane is emitted;
//  * padding slots of a chunk run the prologue branch-free on a zero-weight
//    particle at the cell origin (finite weights, zero contribution);
//  * the gather's node list (plane offset, which of the W*W pencil offsets
//    contribute, interior flag) is computed once per CTA, not per plane.
// Scaled J weights: QSP 6*S(d), TSC 2*S(d) (the constant 1/216 or 1/8 is
// folded into q*W once per particle; fewer multiplies per axis).
template <int ORDER>
__device__ __forceinline__ void weights_scaled(double d, double (&s)[Shape<ORDER>::W]) {
    if constexpr (ORDER == 1) {
        s[0] = 1.0 - d;
        s[1] = d;
    } else if constexpr (ORDER == 3) {
        const double t2 = d * d, t3 = t2 * d, u = 1.0 - d;
        s[0] = u * u * u;
        s[1] = fma(3.0, t3, fma(-6.0, t2, 4.0));
        s[2] = fma(-3.0, t3, fma(3.0, t2, fma(3.0, d, 1.0)));
        s[3] = t3;
    } else {
        const bool up = d >= 0.5;
        const double dl = up ? d - 1.0 : d;
        const double a = 0.5 - dl, b = 0.5 + dl;
        const double w0 = a * a, w1 = fma(-2.0 * dl, dl, 1.5), w2 = b * b;
        s[0] = up ? 0.0 : w0;
        s[1] = up ? w0 : w1;
        s[2] = up ? w1 : w2;
        s[3] = up ? w2 : 0.0;
    }
}

// Fractions of a binned particle relative to its cell (dci, dcj, dck as
// doubles), one combined range check; the exact locate only for a position
// outside [-0.5, 1.5] of its cell (periodic image of an unwrapped upload).
// Padding slots (valid = false) get d = 0 and zero charge: finite weights,
// no contribution, whatever the slot's registers hold.
template <int ORDER>
__device__ __forceinline__ void particle_window_sel(const GridD& g, const PData& d, double qs, bool valid,
                                                    double dci, double dcj, double dck,
                                                    double (&a)[3][Shape<ORDER>::W], double (&sy)[Shape<ORDER>::W],
                                                    double (&sz)[Shape<ORDER>::W]) {
    constexpr int W = Shape<ORDER>::W;
    const double qw = qs * d.w;
    const double wq0 = valid ? qw * d.vx : 0.0, wq1 = valid ? qw * d.vy : 0.0, wq2 = valid ? qw * d.vz : 0.0;
    double fx = (d.x - g.gox) * g.inv_dx - dci;
    double fy = (d.y - g.oy) * g.inv_dy - dcj;
    double fz = (d.z - g.oz) * g.inv_dz - dck;
    const bool in = fx >= -0.5 && fx <= 1.5 && fy >= -0.5 && fy <= 1.5 && fz >= -0.5 && fz <= 1.5;
    if (valid && !in) {
        if (!(fx >= -0.5 && fx <= 1.5)) locate_axis(d.x, g.gox, g.dx, g.inv_dx, g.pow2x, g.gnx, fx);
        if (!(fy >= -0.5 && fy <= 1.5)) locate_axis(d.y, g.oy, g.dy, g.inv_dy, g.pow2y, g.ny, fy);
        if (!(fz >= -0.5 && fz <= 1.5)) locate_axis(d.z, g.oz, g.dz, g.inv_dz, g.pow2z, g.nz, fz);
    }
    fx = valid ? fx : 0.0;
    fy = valid ? fy : 0.0;
    fz = valid ? fz : 0.0;
    double sx[W];
    weights_scaled<ORDER>(fx, sx);
    weights_scaled<ORDER>(fy, sy);
    weights_scaled<ORDER>(fz, sz);
#pragma unroll
    for (int t = 0; t < W; ++t) {
        a[0][t] = wq0 * sx[t];
        a[1][t] = wq1 * sx[t];
        a[2][t] = wq2 * sx[t];
    }
}

// Paired staging (JLayout PSS/PFS): address of field f of chunk position l of pencil grp.
template <class L>
__device__ __forceinline__ double* pfield(double* stage, int f, int l, int grp) {
    return stage + ((((f >> 1) * L::PFS + l * L::PSS + grp) << 1) | (f & 1));
}
template <class L>
__device__ __forceinline__ const double* pfield(const double* stage, int f, int l, int grp) {
    return stage + ((((f >> 1) * L::PFS + l * L::PSS + grp) << 1) | (f & 1));
}

// Stage one particle's window: a[c][t] and sy[t] as tap pairs; sz[t] at its
// physical z slot (t + R) & (W-1) (the accumulators' rotated window).
template <class L, int W>
__device__ __forceinline__ void stage_record(double* stage, int l, int grp, int R, const double (&a)[3][W],
                                             const double (&sy)[W], const double (&sz)[W]) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int t = 0; t < W; t += 2)
            *reinterpret_cast<double2*>(pfield<L>(stage, c * W + t, l, grp)) = make_double2(a[c][t], a[c][t + 1]);
#pragma unroll
    for (int t = 0; t < W; t += 2)
        *reinterpret_cast<double2*>(pfield<L>(stage, 3 * W + t, l, grp)) = make_double2(sy[t], sy[t + 1]);
#pragma unroll
    for (int t = 0; t < W; ++t) *pfield<L>(stage, 4 * W + ((t + R) & (W - 1)), l, grp) = sz[t];
}

// Shift one staged W-tap array (fields f0 .. f0+W-1, logical tap t stored at
// f0 + ((t + rot) & (W-1))) by sh (-1, 0, +1) taps, zero-filling the vacated one.
template <class L, int W>
__device__ __forceinline__ void restage_shifted(double* stage, int l, int grp, int f0, int sh, int rot) {
    if (sh == 0) return;
    double v[W];
#pragma unroll
    for (int t = 0; t < W; ++t) {
        const int u = t - sh;
        v[t] = (u >= 0 && u < W) ? *pfield<L>(stage, f0 + ((u + rot) & (W - 1)), l, grp) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < W; ++t) *pfield<L>(stage, f0 + ((t + rot) & (W - 1)), l, grp) = v[t];
}

// Cell step of a mover on one periodic axis, folded into {-1, 0, +1}.
__device__ __forceinline__ int cell_step(int d, int n) {
    return d == 0 ? 0 : (d == 1 || d == 1 - n) ? 1 : -1;
}

// Window weights from the particle's cell fractions (the J forms:
// weights_scaled, x-weights pre-multiplied by wq_c); zero charge when invalid.
template <int ORDER>
__device__ __forceinline__ void window_from_fractions(const PData& d, double qs, bool valid, double fx, double fy,
                                                      double fz, double (&a)[3][Shape<ORDER>::W],
                                                      double (&sy)[Shape<ORDER>::W], double (&sz)[Shape<ORDER>::W]) {
    constexpr int W = Shape<ORDER>::W;
    const double qw = qs * d.w;
    const double wq0 = valid ? qw * d.vx : 0.0, wq1 = valid ? qw * d.vy : 0.0, wq2 = valid ? qw * d.vz : 0.0;
    double sx[W];
    weights_scaled<ORDER>(valid ? fx : 0.0, sx);
    weights_scaled<ORDER>(valid ? fy : 0.0, sy);
    weights_scaled<ORDER>(valid ? fz : 0.0, sz);
#pragma unroll
    for (int t = 0; t < W; ++t) {
        a[0][t] = wq0 * sx[t];
        a[1][t] = wq1 * sx[t];
        a[2][t] = wq2 * sx[t];
    }
}

// wrap_position (workload.hpp:128-132) with its common case first: a pushed
// coordinate inside [origin, origin + length) is returned unchanged, which is
// exactly what the full form computes there (floor((x-o)/L) = 0, x - L*0 = x,
// and x - o < L); otherwise the full form.
template <bool P2>
__device__ __forceinline__ double wrap_fast(double x, double origin, double length, double inv, int pow2) {
    const double t = __dsub_rn(x, origin);
    if (t >= 0.0 && t < length) return x;
    return wrap_position(x, origin, length, inv, P2 || pow2);
}

// Fused step, one binned particle of bin b (cell i, j, k; dci/dcj/dck the
// same as doubles): the bit-exact push written back to its slot
// (pic::advance, workload.hpp:139-155), the move test of detect_moves
// (gpma.hpp:162-177) and the particle's fractions for the deposit -- relative
// to its bin's cell, or for a mover to its new cell, with the cell step
// (shx, shy, shz) that places its taps in the bin's window.  Positions are
// finite on entry (the store only holds located particles).  Returns false
// on an error (the reference would throw; the device flag is raised).
template <bool P2, bool SLAB = false>
__device__ __forceinline__ bool push_fused(const GridD& g, const PushCtx& pc, PData& d, uint32_t s, uint32_t b,
                                           int i, int j, int k, double dci, double dcj, double dck, double& fx,
                                           double& fy, double& fz, bool& mv, uint32_t& mv_cell, int& shx,
                                           int& shy, int& shz) {
    const double v2 = __dadd_rn(__dadd_rn(__dmul_rn(d.vx, d.vx), __dmul_rn(d.vy, d.vy)), __dmul_rn(d.vz, d.vz));
    if (!(v2 <= pc.cap2)) {
        // v^2 > cap^2: domain_error; NaN velocity: the reference's position
        // becomes NaN and cell_of throws invalid_argument
        raise_error(&pc.ctr->err, v2 > pc.cap2 ? PICGPU_EDOMAIN : PICGPU_EINVAL);
        return false;
    }
    d.x = wrap_fast<P2>(__dadd_rn(d.x, __dmul_rn(d.vx, pc.dt)), g.gox, g.gLx, g.ginv_Lx, g.gpow2Lx);
    d.y = wrap_fast<P2>(__dadd_rn(d.y, __dmul_rn(d.vy, pc.dt)), g.oy, g.Ly, g.inv_Ly, g.pow2Ly);
    d.z = wrap_fast<P2>(__dadd_rn(d.z, __dmul_rn(d.vz, pc.dt)), g.oz, g.Lz, g.inv_Lz, g.pow2Lz);
    reinterpret_cast<double2*>(pc.A.p + s)[0] = make_double2(d.x, d.y);
    pc.A.p[s].z = d.z;
    // fractions relative to the bin's cell; with power-of-two spacings u =
    // (x-o)*inv is locate_axis's exact u, so 0 <= u - c < 1 on every axis is
    // exactly "same cell"; otherwise compare the exact floors
    fx = __dmul_rn(__dsub_rn(d.x, g.gox), g.inv_dx) - dci;
    fy = __dmul_rn(__dsub_rn(d.y, g.oy), g.inv_dy) - dcj;
    fz = __dmul_rn(__dsub_rn(d.z, g.oz), g.inv_dz) - dck;
    bool same;
    if constexpr (P2)
        same = fx >= 0.0 && fx < 1.0 && fy >= 0.0 && fy < 1.0 && fz >= 0.0 && fz < 1.0;
    else
        same = axis_floor(d.x, g.gox, g.dx, g.inv_dx, g.pow2x) == dci &&
               axis_floor(d.y, g.oy, g.dy, g.inv_dy, g.pow2y) == dcj &&
               axis_floor(d.z, g.oz, g.dz, g.inv_dz, g.pow2z) == dck;
    if (same) return true;
    if constexpr (P2) {
        // Pushed positions are wrapped into [o, o + L), so u = (x-o)*inv lies in
        // [0, n) and locate_axis's cell is floor(u) = c + floor(f) exactly; a
        // one-cell step leaves f in [-1, 2) (otherwise: wrapped around the box)
        if (fx >= -1.0 && fx < 2.0 && fy >= -1.0 && fy < 2.0 && fz >= -1.0 && fz < 2.0) {
            shx = fx < 0.0 ? -1 : (fx >= 1.0 ? 1 : 0);
            shy = fy < 0.0 ? -1 : (fy >= 1.0 ? 1 : 0);
            shz = fz < 0.0 ? -1 : (fz >= 1.0 ? 1 : 0);
            if constexpr (SLAB) {
                if (i + shx < g.sx_lo || i + shx >= g.sx_hi) {  // left the slab: k_movers exports it
                    mv = true;
                    mv_cell = i + shx < g.sx_lo ? kLeaveLeft : kLeaveRight;
                    return false;
                }
            }
            fx -= (double)shx;
            fy -= (double)shy;
            fz -= (double)shz;
            mv = true;
            mv_cell = (uint32_t)(i + shx) + (uint32_t)g.nx * ((uint32_t)(j + shy) + (uint32_t)g.ny * (uint32_t)(k + shz));
            return true;
        }
    }
    int ni, nj, nk;
    const uint32_t nc = cell_linear<P2>(g, d.x, d.y, d.z, ni, nj, nk, fx, fy, fz);  // exact (pic::cell_of)
    if constexpr (SLAB) {
        const uint32_t code = store_cell<P2>(g, d.x, d.y, d.z);  // kLeaveLeft / kLeaveRight off the slab
        if (code >= kLeaveRight) {  // left the slab: k_movers exports it, nothing deposited here
            mv = true;
            mv_cell = code;
            return false;
        }
    }
    if (nc == b) return true;  // a periodic image of the bin's cell
    mv = true;
    mv_cell = nc;
    // the step on the GLOBAL periodic x axis: a one-slab store (P = 1) wraps
    // through its ghost layers, where the local index difference is not +-1
    shx = cell_step(ni - i, g.gnx);
    shy = cell_step(nj - j, g.ny);
    shz = cell_step(nk - k, g.nz);
    return true;
}

// PM (fused step, PushCtx): 0 = deposit only; 1 = push + move detection + deposit of the
// particles that stay in their cell (launch_deposit_current_push); 2 = the same
// with every spacing and box length a power of two (compile-time reciprocals).
template <int ORDER, class CF = JCfg<ORDER>, int PM = 0, bool SLAB = false>
__global__ void __launch_bounds__(JLayout<ORDER, CF>::NT, CF::MINB)
    deposit_current_kernel_v3(const GridD g, const CAos p, const uint32_t* __restrict__ off,
                              const uint32_t* __restrict__ cnt, const double q, double* __restrict__ jx,
                              double* __restrict__ jy, double* __restrict__ jz, const int zlen,
                              const PushCtx pc) {
    using C = CF;
    using L = JLayout<ORDER, CF>;
    constexpr int W = L::W, OFF = Shape<ORDER>::OFF, NJ = L::NJ;
    constexpr int G = C::G, PX = C::PX, PY = C::PY, CH = C::CH;
    constexpr int FX = PX + W - 1, FY = PY + W - 1;
    constexpr int NODES = 3 * FX * FY;
    constexpr int NIT = (NODES + L::NT - 1) / L::NT;
    // lane = ly + W * xh (ly = jy): G = W * XS lanes per pencil, each owning IX = W / XS x-taps
    constexpr int XS = G / W, IX = W / XS;
    static_assert(G == W * XS && W % XS == 0 && (W & (W - 1)) == 0, "v3: lanes = jy x x-halves");
    (void)NJ;
    // 1/6^3 (QSP) or 1/2^3 (TSC) of the scaled weights, folded into q
    const double qs = q * (ORDER == 3 ? 1.0 / 216.0 : ORDER == 2 ? 0.125 : 1.0);

    extern __shared__ __align__(16) double smem[];
    constexpr int PPB = L::PPB;
    double* patch = smem;                       // [2][PPB][W(jy)][W(ix)][3][PSTRIDE]
    double* stage = smem + 2 * PPB * L::PATCH;  // paired fields (JLayout PSS/PFS)

    const int tid = threadIdx.x;
    const int grp = tid / G, lg = tid % G;
    const int ly = lg % W, xh = lg / W;  // this lane's jy and x-half
    const int px = grp % PX, py = grp / PX;
    const int i0 = blockIdx.x * PX, j0 = blockIdx.y * PY;
    const int k0 = blockIdx.z * zlen;
    const int k1 = min(k0 + zlen, g.nz);
    const int i = i0 + px, j = j0 + py;
    const bool pv = (i < g.nx) && (j < g.ny);
    const int pxv = min(PX, g.nx - i0), pyv = min(PY, g.ny - j0);
    const bool alias_xy = (pxv + W - 1 > g.nx) || (pyv + W - 1 > g.ny);
    const uint32_t col = (uint32_t)i + (uint32_t)g.nx * (uint32_t)j;
    const uint32_t plane_cells = (uint32_t)g.nx * (uint32_t)g.ny;
    const double dci = (double)(i + g.sx_shift), dcj = (double)j;
    // this CTA's segment of the mover arrays (reserved with shared-memory atomics)
    [[maybe_unused]] const uint32_t seg = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    __shared__ unsigned s_movers;
    if (PM != 0 && threadIdx.x == 0) s_movers = 0;

    // gather plan of this thread's nodes (constant over z)
    int gn_base[NIT], gn_node[NIT];
    unsigned gn_mask[NIT];
    bool gn_inner[NIT];
#pragma unroll
    for (int t = 0; t < NIT; ++t) {
        const int it = tid + t * L::NT;
        gn_mask[t] = 0u;
        gn_base[t] = 0;
        gn_node[t] = 0;
        gn_inner[t] = false;
        if (it < NODES) {
            const int c = it / (FX * FY);
            const int r = it - c * (FX * FY);
            const int uy = r / FX, ux = r - uy * FX;
            if (ux < pxv + W - 1 && uy < pyv + W - 1) {
#pragma unroll
                for (int dy = 0; dy < W; ++dy)
#pragma unroll
                    for (int dx = 0; dx < W; ++dx) {
                        const int qy = uy - dy, qx = ux - dx;
                        if (qy >= 0 && qy < pyv && qx >= 0 && qx < pxv) gn_mask[t] |= 1u << (dy * W + dx);
                    }
                // patch offset of pencil (0,0)'s contribution, component in the top bits
                gn_base[t] = (c << 28) | (c * L::PSTRIDE + uy * PX + ux);
                const int X = wrap_index(i0 + OFF + ux, g.nx);
                const int Y = wrap_index(j0 + OFF + uy, g.ny);
                gn_node[t] = X + g.nx * Y;
                gn_inner[t] = !alias_xy && ux >= W - 1 && ux <= pxv - 1 && uy >= W - 1 && uy <= pyv - 1;
            }
        }
    }

    // acc[s]: physical slot s of the sliding z window; at step k the slot s
    // holds logical plane (s - R) mod W of the window, R = (k - k0) mod W
    double acc[W][IX][3];
#pragma unroll
    for (int sl = 0; sl < W; ++sl)
#pragma unroll
        for (int ix = 0; ix < IX; ++ix)
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[sl][ix][c] = 0.0;

    // an entirely empty tile (vacuum) writes nothing: J was zeroed by the caller
    {
        bool any = false;
        if (pv)
            for (int kk = k0 + lg; kk < k1; kk += G) any |= cnt[col + plane_cells * kk] != 0;
        if (!__syncthreads_or(any)) {
            if (PM != 0 && threadIdx.x == 0) pc.seg_cnt[seg] = 0;
            return;
        }
    }
    uint32_t c_off = 0;
    int n_c = 0;
    if (pv && k0 < k1) {
        c_off = off[col + plane_cells * k0];
        n_c = (int)cnt[col + plane_cells * k0];
    }
    int last_busy = k0 - W;  // last z-step in which any pencil of the CTA deposited (CTA-uniform)
    PData nxt{};
    if (lg < n_c) load_particle<PM != 0>(p, c_off + lg, nxt);

    int phase = 0;
    bool busy_acc = false;  // any deposit in this barrier's batch of planes
    const int kend = k1 + W - 1;
    for (int k = k0; k < kend; ++k) {
        const int R = (k - k0) & (W - 1);
        const int sub = (k - k0) % PPB;
        const bool busy = k < k1 && n_c > 0;
        if (k < k1) {
            uint32_t n_off = 0;
            int n_n = 0;
            if (pv && k + 1 < k1) {
                n_off = off[col + plane_cells * (k + 1)];
                n_n = (int)cnt[col + plane_cells * (k + 1)];
            }
            const double dck = (double)k;
            const int m = (int)__reduce_max_sync(0xffffffffu, (unsigned)n_c);
            if (m == 0 && lg < n_n) load_particle<PM != 0>(p, n_off + lg, nxt);  // empty cells: still prefetch
            for (int base = 0; base < m; base += CH) {
                [[maybe_unused]] bool mv = false;  // fused step: this lane's particle changed cell
                [[maybe_unused]] uint32_t mv_cell = 0;
                [[maybe_unused]] unsigned mv_bal = 0, mv_b0 = 0;
                {
                    PData cur = nxt;
                    bool valid = base + lg < n_c && !is_gap(cur.x);  // holes count as padding
                    if (base + CH < m) {
                        if (base + CH + lg < n_c) load_particle<PM != 0>(p, c_off + base + CH + lg, nxt);
                    } else if (lg < n_n) {
                        load_particle<PM != 0>(p, n_off + lg, nxt);
                    }
                    double a[3][W], sy[W], sz[W];
                    if constexpr (PM != 0) {
                        // pic::advance (workload.hpp:139-155) + Gpma::detect_moves (gpma.hpp:162-177):
                        // fractions of the pushed particle, relative to its new cell for a mover
                        double fx = 0.0, fy = 0.0, fz = 0.0;
                        int shx = 0, shy = 0, shz = 0;
                        if (valid)
                            valid = push_fused<PM == 2, SLAB>(g, pc, cur, c_off + (uint32_t)(base + lg),
                                                              col + plane_cells * (uint32_t)k, i, j, k, dci, dcj, dck,
                                                              fx, fy, fz, mv, mv_cell, shx, shy, shz);
                        // one mover-list reservation per warp; its result is only
                        // needed after the contraction below
                        mv_bal = __ballot_sync(0xffffffffu, mv);
                        if (mv_bal && (tid & 31) == __ffs(mv_bal) - 1)
                            mv_b0 = atomicAdd(&s_movers, (unsigned)__popc(mv_bal));
                        window_from_fractions<ORDER>(cur, qs, valid, fx, fy, fz, a, sy, sz);
                        stage_record<L, W>(stage, lg, grp, R, a, sy, sz);
                        if (mv && valid) {
                            // a mover's taps, shifted into this cell's window by its cell
                            // step (read back from its staged record: runtime offsets stay
                            // in shared memory); taps that leave the window are k_movers'
                            restage_shifted<L, W>(stage, lg, grp, 0, shx, 0);
                            restage_shifted<L, W>(stage, lg, grp, W, shx, 0);
                            restage_shifted<L, W>(stage, lg, grp, 2 * W, shx, 0);
                            restage_shifted<L, W>(stage, lg, grp, 3 * W, shy, 0);
                            restage_shifted<L, W>(stage, lg, grp, 4 * W, shz, R);
                        }
                    } else {
                        particle_window_sel<ORDER>(g, cur, qs, valid, dci, dcj, dck, a, sy, sz);
                        stage_record<L, W>(stage, lg, grp, R, a, sy, sz);
                    }
                }
                __syncwarp();
                const int nn = min(CH, m - base);
#pragma unroll
                for (int jj0 = 0; jj0 < CH; ++jj0) {
                    if (jj0 >= nn) break;
                    const double yv = *pfield<L>(stage, 3 * W + ly, jj0, grp);
                    double b[W];
#pragma unroll
                    for (int sl = 0; sl < W; sl += 2) {  // sz of physical slots sl, sl+1
                        const double2 zz = *reinterpret_cast<const double2*>(pfield<L>(stage, 4 * W + sl, jj0, grp));
                        b[sl] = yv * zz.x;
                        b[sl + 1] = yv * zz.y;
                    }
#pragma unroll
                    for (int c = 0; c < 3; ++c)
#pragma unroll
                        for (int ix = 0; ix < IX; ix += 2) {
                            const double2 av =
                                *reinterpret_cast<const double2*>(pfield<L>(stage, c * W + xh * IX + ix, jj0, grp));
#pragma unroll
                            for (int sl = 0; sl < W; ++sl) {
                                acc[sl][ix][c] = fma(av.x, b[sl], acc[sl][ix][c]);
                                acc[sl][ix + 1][c] = fma(av.y, b[sl], acc[sl][ix + 1][c]);
                            }
                        }
                }
                if constexpr (PM != 0) {
                    if (mv_bal) {
                        const unsigned b0 = __shfl_sync(0xffffffffu, mv_b0, __ffs(mv_bal) - 1);
                        if (mv) {
                            const unsigned idx = b0 + (unsigned)__popc(mv_bal & ((1u << (tid & 31)) - 1u));
                            size_t e = (size_t)seg * pc.segcap + idx;
                            if (idx >= pc.segcap) {  // segment full: the shared overflow segment
                                const unsigned o = atomicAdd(&pc.ctr->ovf_movers, 1u);
                                e = o < pc.ovcap ? (size_t)pc.nseg * pc.segcap + o : ~(size_t)0;
                            }
                            if (e != ~(size_t)0) {
                                pc.mslot[e] = c_off + (uint32_t)(base + lg);
                                pc.mbin[e] = col + plane_cells * (uint32_t)k;
                                pc.mcellseg[e] = mv_cell;
                            }
                        }
                    }
                }
                __syncwarp();
            }
            c_off = n_off;
            n_c = n_n;
        }
        // logical plane 0 (physical slot R) is final: emit it and zero the slot,
        // which becomes the window's top plane at the next step
        {
            double* pp = patch + (phase * PPB + sub) * L::PATCH + grp;
            auto emit = [&](auto Sc) {
                constexpr int S = decltype(Sc)::value;
#pragma unroll
                for (int c = 0; c < 3; ++c)
#pragma unroll
                    for (int ix = 0; ix < IX; ++ix) {
                        pp[((ly * W + xh * IX + ix) * 3 + c) * L::PSTRIDE] = acc[S][ix][c];
                        acc[S][ix][c] = 0.0;
                    }
            };
            if constexpr (W == 2) {
                if (R == 0)
                    emit(std::integral_constant<int, 0>{});
                else
                    emit(std::integral_constant<int, 1>{});
            } else {
                switch (R) {
                    case 0: emit(std::integral_constant<int, 0>{}); break;
                    case 1: emit(std::integral_constant<int, 1>{}); break;
                    case 2: emit(std::integral_constant<int, 2>{}); break;
                    default: emit(std::integral_constant<int, 3>{}); break;
                }
            }
        }
        // PPB planes per CTA barrier: the batch's planes are gathered together
        busy_acc |= busy;
        if (sub != PPB - 1 && k + 1 < kend) continue;
        // a plane emitted at step kk gathers cells kk-W+1..kk: if none of them
        // held a particle anywhere in the CTA, every node sum is zero -- skip it
        if (__syncthreads_or(busy_acc)) last_busy = k;
        busy_acc = false;
        for (int sl = 0; sl <= sub; ++sl) {
            const int kk = k - sub + sl;
            if (last_busy < kk - (W - 1)) continue;
            const double* pb = patch + (phase * PPB + sl) * L::PATCH;
            const int Z = wrap_index(kk + OFF, g.nz);
            const bool zc = (kk >= k0 + W - 1) && (kk < k1);
            const size_t zrow = (size_t)plane_cells * (size_t)Z;
#pragma unroll
            for (int t = 0; t < NIT; ++t) {
                const unsigned msk = gn_mask[t];
                if (!msk) continue;
                const int c = gn_base[t] >> 28;
                const double* src = pb + (gn_base[t] & 0x0fffffff);
                double v[W * W];
#pragma unroll
                for (int dy = 0; dy < W; ++dy)
#pragma unroll
                    for (int dx = 0; dx < W; ++dx)
                        v[dy * W + dx] = (msk & (1u << (dy * W + dx)))
                                             ? src[(dy * W + dx) * 3 * L::PSTRIDE - dy * PX - dx]
                                             : 0.0;
#pragma unroll
                for (int h = W * W / 2; h >= 1; h /= 2)  // pairwise sum: 4 dependent adds, not 16
#pragma unroll
                    for (int e = 0; e < h; ++e) v[e] += v[e + h];
                const double s = v[0];
                double* f = c == 0 ? jx : (c == 1 ? jy : jz);
                const size_t node = (size_t)gn_node[t] + zrow;
                if (zc && gn_inner[t])
                    f[node] = s;
                else if (s != 0.0)
                    atomicAdd(f + node, s);
            }
        }
        phase ^= 1;
    }
    if constexpr (PM != 0) {  // this CTA's mover count (every reservation precedes the last barrier)
        __syncthreads();
        if (threadIdx.x == 0) pc.seg_cnt[seg] = s_movers;
    }
}

// ---------------------------------------------------------------------------
// Orders 2 and 3 (4-tap window): ONE WARP PER PENCIL.
//
// The warp streams its pencil's particles (cells k0..k1-1 concatenated) in
// chunks of 32: lane l loads and pre-processes the l-th particle of the chunk
// (all lanes busy whatever the cell counts), writes a 30-double record
// {a[ix][c] = wq_c*sx[ix] (12), b[jy][kz] = sy[jy]*sz[kz] (16)} to the warp's
// staging area, and the next chunk's loads are already in flight.  Then the
// four quarter-warps consume the staged particles four at a time (same
// cell): lane = (quarter, jy, ix pair) owns 4 kz x 2 ix x 3 comps = 24
// accumulators, reads 10 operands with LDS.64 (1 wavefront each; LDS.128
// costs 4) and issues 24 DFMA.  The z window slides by register rotation
// (the z loop is unrolled 4x); the quarters' partial sums meet with two
// shuffles when a plane is emitted.
#ifndef PICGPU_WARP_MINB
#define PICGPU_WARP_MINB 2
#endif
struct WCfg {
    static constexpr int PX = 4, PY = 2, NW = PX * PY, NT = NW * 32, MINB = PICGPU_WARP_MINB;
    // Staging is field-major: field f of chunk particle l at [f*FS + l].  The
    // 36-double field stride makes the staging writes conflict-free and puts
    // the four quarter-warps' operands (particles l..l+3) in disjoint banks;
    // the operands of one lane sit FS doubles apart, so ptxas cannot fuse them
    // into LDS.128 (4 wavefronts) -- every operand load is a 1-wavefront LDS.64.
    static constexpr int NF = 28, FS = 36, REC = NF * FS;  // per-warp staging block (doubles)
    static constexpr int R = 2;                         // planes emitted per CTA barrier
    static constexpr int PS = 49;                       // per-pencil patch stride (3*16 + 1 skew)
    static constexpr int PATCH = NW * PS;               // one plane slot: [pencil][c][jy][ix]
    static constexpr int STAGE = NW * REC;
    static constexpr size_t SMEM = (size_t)(2 * R * PATCH + STAGE) * sizeof(double);
};

template <int ORDER>
__global__ void __launch_bounds__(WCfg::NT, WCfg::MINB)
    deposit_current_warp_kernel(const GridD g, const CAos p, const uint32_t* __restrict__ off,
                                const uint32_t* __restrict__ cnt, const double q, double* __restrict__ jx,
                                double* __restrict__ jy, double* __restrict__ jz, const int zlen) {
    constexpr int W = 4, OFF = Shape<ORDER>::OFF;
    static_assert(Shape<ORDER>::W == 4, "warp kernel is for the 4-tap window");
    constexpr int PX = WCfg::PX, PY = WCfg::PY, FS = WCfg::FS, PS = WCfg::PS;
    constexpr int FX = PX + W - 1, FY = PY + W - 1, NITEM = 3 * FX * FY;
    static_assert(NITEM <= WCfg::NT, "one gather item per thread");
    constexpr int SY = W - PX * PS, SX = 1 - PS;  // patch offset of tap (dy, dx) from tap (0, 0)
    constexpr unsigned FULL = 0xffffffffu;

    extern __shared__ __align__(16) double smem[];
    double* patch = smem;  // [2 phases][R planes][pencil][c][jy][ix]
    double* stage = smem + 2 * WCfg::R * WCfg::PATCH;

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int px = wid % PX, py = wid / PX;
    const int jyl = lane & 3, ixp = (lane >> 2) & 1, qq = lane >> 3;  // (jy, ix pair, quarter)
    const int i0 = blockIdx.x * PX, j0 = blockIdx.y * PY;
    const int k0 = blockIdx.z * zlen;
    const int k1 = min(k0 + zlen, g.nz);
    const int i = i0 + px, j = j0 + py;
    const bool pv = (i < g.nx) && (j < g.ny);
    const int pxv = min(PX, g.nx - i0), pyv = min(PY, g.ny - j0);
    const bool alias_xy = (pxv + W - 1 > g.nx) || (pyv + W - 1 > g.ny);
    const uint32_t col = (uint32_t)i + (uint32_t)g.nx * (uint32_t)j;
    const uint32_t plane_cells = (uint32_t)g.nx * (uint32_t)g.ny;
    double* recs = stage + wid * WCfg::REC;

    // ---- this thread's gather item (fixed for all planes) ----
    bool g_active = false, g_inxy = false;
    uint32_t g_taps = 0;
    int g_base = 0;
    double* g_field = jx;
    size_t g_xy = 0;
    {
        const int it = threadIdx.x;
        if (it < NITEM) {
            const int c = it / (FX * FY);
            const int r = it - c * (FX * FY);
            const int uy = r / FX, ux = r - uy * FX;
            if (ux < pxv + W - 1 && uy < pyv + W - 1) {
                g_active = true;
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                    const int qy = uy - (t >> 2), qx = ux - (t & 3);
                    if (qy >= 0 && qy < pyv && qx >= 0 && qx < pxv) g_taps |= 1u << t;
                }
                g_base = (uy * PX + ux) * PS + c * 16;  // pencil (ux, uy), tap (0, 0)
                g_field = c == 0 ? jx : (c == 1 ? jy : jz);
                g_xy = (size_t)wrap_index(i0 + OFF + ux, g.nx) +
                       (size_t)g.nx * (size_t)wrap_index(j0 + OFF + uy, g.ny);
                g_inxy = !alias_xy && ux >= W - 1 && ux <= pxv - 1 && uy >= W - 1 && uy <= pyv - 1;
            }
        }
    }

    // ---- stream planner: lane l gets the l-th particle from (sk, spos) ----
    int sk = k0;
    uint32_t spos = 0;
    auto plan = [&](uint32_t& slot, int& cz, bool& valid) {
        uint32_t wcnt = 0, woff = 0;
        const int kk = sk + lane;
        if (pv && kk < k1) {
            const uint32_t c = col + plane_cells * (uint32_t)kk;
            woff = off[c];
            wcnt = cnt[c];
        }
        uint32_t incl = wcnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t v = __shfl_up_sync(FULL, incl, d);
            if (lane >= d) incl += v;
        }
        const uint32_t total = __shfl_sync(FULL, incl, 31);
        const uint32_t t = spos + (uint32_t)lane;
        valid = t < total;
        int pos = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const uint32_t v = __shfl_sync(FULL, incl, pos + step - 1);
            if (v <= t) pos += step;
        }
        const int jw = pos < 31 ? pos : 31;
        const uint32_t excl_j = __shfl_sync(FULL, incl - wcnt, jw);
        const uint32_t off_j = __shfl_sync(FULL, woff, jw);
        slot = off_j + (t - excl_j);
        cz = sk + jw;
        const uint32_t tend = total > spos ? min(spos + 32u, total) : spos;
        if (tend >= total) {
            sk = min(sk + 32, k1);
            spos = 0;
        } else {
            const int pe = __popc(__ballot_sync(FULL, incl <= tend));
            spos = tend - __shfl_sync(FULL, incl - wcnt, pe);
            sk = sk + pe;
        }
    };

    PData nxt{};
    uint32_t nslot = 0;
    int ncz = 0;
    bool nvalid = false;
    plan(nslot, ncz, nvalid);
    if (nvalid) load_particle(p, nslot, nxt);
    bool pending = __any_sync(FULL, nvalid);

    double acc[W][2][3];  // [kz slot][ix in pair][c]
#pragma unroll
    for (int kz = 0; kz < W; ++kz)
#pragma unroll
        for (int e = 0; e < 2; ++e) acc[kz][e][0] = acc[kz][e][1] = acc[kz][e][2] = 0.0;
    int navail = 0, nidx = 0, cz_reg = 0x7fffffff;
    const int T = k1 + W - 1 - k0;  // planes emitted by every warp (CTA-uniform)

    // One z-step at register rotation RT (slot (kz+RT)&3 holds local plane kz),
    // unrolled 4x so the sliding window never moves registers.
    auto step = [&](auto rot, int kb) {
        constexpr int RT = decltype(rot)::value;
        const int k = k0 + kb + RT;
        if (kb + RT >= T) return;
        if (k < k1) {
            for (;;) {
                if (nidx == navail) {
                    if (!pending) break;
                    __syncwarp();  // the previous chunk's records are no longer read
                    if (nvalid) {  // prologue: shape.hpp:64-85 + particle_weights :46-50
                        double a[3][W], sy[W], sz[W];
                        particle_window_fast<ORDER>(g, nxt, q, a, sy, sz);
                        if (is_gap(nxt.x)) {  // a hole of the bin (GPMA gap): zero charge
#pragma unroll
                            for (int t = 0; t < W; ++t) a[0][t] = a[1][t] = a[2][t] = sy[t] = sz[t] = 0.0;
                        }
                        // fields: a[c][ix] at f = c*4 + ix; b[kz][jy] = sy*sz at f = 12 + kz*4 + jy
                        double* rr = recs + lane;
#pragma unroll
                        for (int c = 0; c < 3; ++c)
#pragma unroll
                            for (int xx = 0; xx < W; ++xx) rr[(c * 4 + xx) * FS] = a[c][xx];
#pragma unroll
                        for (int zz = 0; zz < W; ++zz)
#pragma unroll
                            for (int yy = 0; yy < W; ++yy) rr[(12 + zz * 4 + yy) * FS] = sy[yy] * sz[zz];
                    }
                    cz_reg = nvalid ? ncz : 0x7fffffff;
                    navail = __popc(__ballot_sync(FULL, nvalid));
                    nidx = 0;
                    __syncwarp();
                    plan(nslot, ncz, nvalid);  // prefetch the following chunk
                    if (nvalid) load_particle(p, nslot, nxt);
                    pending = __any_sync(FULL, nvalid);
                    continue;
                }
                // staged particles nidx.. of cell k (contiguous): the four
                // quarter-warps take them four at a time
                const unsigned mk = __ballot_sync(FULL, cz_reg == k) & (FULL << nidx);
                const int cntk = __popc(mk);
                const double* ra = recs + (2 * ixp) * FS + nidx + qq;
                const double* rb = recs + (12 + jyl) * FS + nidx + qq;
                for (int t = 0; t < cntk; t += 4) {
                    if (t + qq < cntk) {
                        double av[3][2], bv[W];
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            av[c][0] = ra[(c * 4) * FS];
                            av[c][1] = ra[(c * 4 + 1) * FS];
                        }
#pragma unroll
                        for (int kz = 0; kz < W; ++kz) bv[kz] = rb[kz * 4 * FS];
#pragma unroll
                        for (int kz = 0; kz < W; ++kz)
#pragma unroll
                            for (int e = 0; e < 2; ++e)
#pragma unroll
                                for (int c = 0; c < 3; ++c)
                                    acc[(kz + RT) & 3][e][c] = fma(av[c][e], bv[kz], acc[(kz + RT) & 3][e][c]);
                    }
                    ra += 4;
                    rb += 4;
                }
                nidx += cntk;
                if (nidx < navail || cntk == 0) break;  // the rest of the chunk is in later cells
            }
        }
        // Plane k+OFF is final for this pencil: add the halves, emit, recycle the slot.
        constexpr int SL = RT & 1, PH = (RT >> 1) & 1;  // ring slot and phase (R = 2 planes per barrier)
        {
            double* pp = patch + (PH * WCfg::R + SL) * WCfg::PATCH + wid * PS + jyl * W + 2 * ixp;
#pragma unroll
            for (int e = 0; e < 2; ++e)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    double v = acc[RT & 3][e][c];
                    v += __shfl_xor_sync(FULL, v, 8);
                    v += __shfl_xor_sync(FULL, v, 16);
                    if (qq == 0) pp[c * 16 + e] = v;
                    acc[RT & 3][e][c] = 0.0;
                }
        }
        if (SL == 0 && kb + RT + 1 < T) return;  // flush every 2 planes (and after the last)
        __syncthreads();
        if (g_active) {
#pragma unroll
            for (int sl = 0; sl <= SL; ++sl) {
                const int kk = k - SL + sl;
                const double* pb = patch + (PH * WCfg::R + sl) * WCfg::PATCH + g_base;
                double s = 0.0;
#pragma unroll
                for (int tp = 0; tp < 16; ++tp)
                    if (g_taps & (1u << tp)) s += pb[(tp >> 2) * SY + (tp & 3) * SX];
                const int Z = wrap_index(kk + OFF, g.nz);
                const size_t node = g_xy + (size_t)plane_cells * (size_t)Z;
                const bool zc = (kk >= k0 + W - 1) && (kk < k1);
                if (g_inxy && zc)
                    g_field[node] = s;
                else if (s != 0.0)
                    atomicAdd(g_field + node, s);
            }
        }
    };

    for (int kb = 0; kb < T; kb += 4) {
        step(std::integral_constant<int, 0>{}, kb);
        step(std::integral_constant<int, 1>{}, kb);
        step(std::integral_constant<int, 2>{}, kb);
        step(std::integral_constant<int, 3>{}, kb);
    }
}

// ---------------------------------------------------------------------------
// Orders 2 and 3, FP64 tensor-core variant: ONE WARP PER PENCIL, the per-cell
// outer-product contraction J_cell[(c,ix)][(kz,jy)] = sum_p a_p (x) b_p issued
// as DMMA m8n8k4 (mma.sync ... f64): K = 4 particles per MMA, M = 12 (c,ix)
// rows padded to 16, N = 16 (kz,jy) columns.  Each lane holds only the 8
// accumulator doubles of the 2x2 fragment tiles; per 4 particles it issues 4
// LDS.64 (2 wavefronts each) and 4 DMMA.  This is the paper's MPU
// outer-product form (tile.hpp:23-29, pack_qsp :83-92) on Blackwell's FP64
// matrix pipe.  The pipe's rate equals DFMA's (64 MAC/clk/SM, measured by
// tools/fp64_pipes.cu) and the row padding costs 25%, but the instruction
// count per particle drops ~4x, which is what bounded the DFMA kernels.
struct MCfg {
    static constexpr int PX = 4, PY = 2, NW = PX * PY, NT = NW * 32, MINB = 3;
    static constexpr int NF = 28, FS = 36;               // staging fields: a[(c,ix)] 12 | b[(kz,jy)] 16
    static constexpr int REC = NF * FS;                  // per-warp staging block (doubles)
    static constexpr int R = 2;                          // planes emitted per CTA barrier
    static constexpr int PS = 49;                        // per-pencil patch stride
    static constexpr int PATCH = NW * PS;
    static constexpr int STAGE = NW * REC;
    static constexpr size_t SMEM = (size_t)(2 * R * PATCH + STAGE) * sizeof(double);
};

__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <int ORDER>
__global__ void __launch_bounds__(MCfg::NT, MCfg::MINB)
    deposit_current_dmma_kernel(const GridD g, const CAos p, const uint32_t* __restrict__ off,
                                const uint32_t* __restrict__ cnt, const double q, double* __restrict__ jx,
                                double* __restrict__ jy, double* __restrict__ jz, const int zlen) {
    constexpr int W = 4, OFF = Shape<ORDER>::OFF;
    static_assert(Shape<ORDER>::W == 4, "DMMA kernel is for the 4-tap window");
    constexpr int PX = MCfg::PX, PY = MCfg::PY, FS = MCfg::FS, PS = MCfg::PS;
    constexpr int FX = PX + W - 1, FY = PY + W - 1, NITEM = 3 * FX * FY;
    static_assert(NITEM <= MCfg::NT, "one gather item per thread");
    constexpr int SY = W - PX * PS, SX = 1 - PS;
    constexpr unsigned FULL = 0xffffffffu;

    extern __shared__ __align__(16) double smem[];
    double* patch = smem;  // [2 phases][R planes][pencil][c][jy][ix]
    double* stage = smem + 2 * MCfg::R * MCfg::PATCH;

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int gq = lane >> 2, tq = lane & 3;  // mma fragment coordinates
    const int px = wid % PX, py = wid / PX;
    const int i0 = blockIdx.x * PX, j0 = blockIdx.y * PY;
    const int k0 = blockIdx.z * zlen;
    const int k1 = min(k0 + zlen, g.nz);
    const int i = i0 + px, j = j0 + py;
    const bool pv = (i < g.nx) && (j < g.ny);
    const int pxv = min(PX, g.nx - i0), pyv = min(PY, g.ny - j0);
    const bool alias_xy = (pxv + W - 1 > g.nx) || (pyv + W - 1 > g.ny);
    const uint32_t col = (uint32_t)i + (uint32_t)g.nx * (uint32_t)j;
    const uint32_t plane_cells = (uint32_t)g.nx * (uint32_t)g.ny;
    double* recs = stage + wid * MCfg::REC;

    // ---- this thread's gather item ----
    bool g_active = false, g_inxy = false;
    uint32_t g_taps = 0;
    int g_base = 0;
    double* g_field = jx;
    size_t g_xy = 0;
    {
        const int it = threadIdx.x;
        if (it < NITEM) {
            const int c = it / (FX * FY);
            const int r = it - c * (FX * FY);
            const int uy = r / FX, ux = r - uy * FX;
            if (ux < pxv + W - 1 && uy < pyv + W - 1) {
                g_active = true;
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                    const int qy = uy - (t >> 2), qx = ux - (t & 3);
                    if (qy >= 0 && qy < pyv && qx >= 0 && qx < pxv) g_taps |= 1u << t;
                }
                g_base = (uy * PX + ux) * PS + c * 16;
                g_field = c == 0 ? jx : (c == 1 ? jy : jz);
                g_xy = (size_t)wrap_index(i0 + OFF + ux, g.nx) +
                       (size_t)g.nx * (size_t)wrap_index(j0 + OFF + uy, g.ny);
                g_inxy = !alias_xy && ux >= W - 1 && ux <= pxv - 1 && uy >= W - 1 && uy <= pyv - 1;
            }
        }
    }

    // ---- stream planner (as in the DFMA warp kernel) ----
    int sk = k0;
    uint32_t spos = 0;
    auto plan = [&](uint32_t& slot, int& cz, bool& valid) {
        uint32_t wcnt = 0, woff = 0;
        const int kk = sk + lane;
        if (pv && kk < k1) {
            const uint32_t c = col + plane_cells * (uint32_t)kk;
            woff = off[c];
            wcnt = cnt[c];
        }
        uint32_t incl = wcnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t v = __shfl_up_sync(FULL, incl, d);
            if (lane >= d) incl += v;
        }
        const uint32_t total = __shfl_sync(FULL, incl, 31);
        const uint32_t t = spos + (uint32_t)lane;
        valid = t < total;
        int pos = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const uint32_t v = __shfl_sync(FULL, incl, pos + step - 1);
            if (v <= t) pos += step;
        }
        const int jw = pos < 31 ? pos : 31;
        const uint32_t excl_j = __shfl_sync(FULL, incl - wcnt, jw);
        const uint32_t off_j = __shfl_sync(FULL, woff, jw);
        slot = off_j + (t - excl_j);
        cz = sk + jw;
        const uint32_t tend = total > spos ? min(spos + 32u, total) : spos;
        if (tend >= total) {
            sk = min(sk + 32, k1);
            spos = 0;
        } else {
            const int pe = __popc(__ballot_sync(FULL, incl <= tend));
            spos = tend - __shfl_sync(FULL, incl - wcnt, pe);
            sk = sk + pe;
        }
    };

    PData nxt{};
    uint32_t nslot = 0;
    int ncz = 0;
    bool nvalid = false;
    plan(nslot, ncz, nvalid);
    if (nvalid) load_particle(p, nslot, nxt);
    bool pending = __any_sync(FULL, nvalid);

    // D[mt][nt][2]: rows m = mt*8 + gq = (c, ix) = (m/4, m%4); cols n = nt*8 + 2tq + e = (kz, jy) = (n/4, n%4)
    double D[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
    int navail = 0, nidx = 0, cz_reg = 0x7fffffff;
    int phase = 0;
    const int T = k1 + W - 1 - k0;
    const bool a_hi = gq < 4;  // rows 8..11 of the second m-tile are c = 2; 12..15 are padding
    for (int st = 0; st < T; ++st) {
        const int k = k0 + st;
        if (k < k1) {
            for (;;) {
                if (nidx == navail) {
                    if (!pending) break;
                    __syncwarp();
                    if (nvalid) {  // prologue: shape.hpp:64-85 + particle_weights :46-50
                        double a[3][W], sy[W], sz[W];
                        particle_window<ORDER>(g, nxt, q, a, sy, sz);
                        if (is_gap(nxt.x)) {  // a hole of the bin (GPMA gap): zero charge
#pragma unroll
                            for (int t = 0; t < W; ++t) a[0][t] = a[1][t] = a[2][t] = sy[t] = sz[t] = 0.0;
                        }
                        double* rr = recs + lane;
#pragma unroll
                        for (int c = 0; c < 3; ++c)
#pragma unroll
                            for (int xx = 0; xx < W; ++xx) rr[(c * 4 + xx) * FS] = a[c][xx];
#pragma unroll
                        for (int zz = 0; zz < W; ++zz)
#pragma unroll
                            for (int yy = 0; yy < W; ++yy) rr[(12 + zz * 4 + yy) * FS] = sy[yy] * sz[zz];
                    }
                    cz_reg = nvalid ? ncz : 0x7fffffff;
                    navail = __popc(__ballot_sync(FULL, nvalid));
                    nidx = 0;
                    __syncwarp();
                    plan(nslot, ncz, nvalid);
                    if (nvalid) load_particle(p, nslot, nxt);
                    pending = __any_sync(FULL, nvalid);
                    continue;
                }
                const unsigned mk = __ballot_sync(FULL, cz_reg == k) & (FULL << nidx);
                const int cntk = __popc(mk);
                for (int kb = 0; kb < cntk; kb += 4) {
                    const bool v = kb + tq < cntk;
                    const int pidx = nidx + kb + tq;
                    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
                    if (v) {
                        const double* r = recs + pidx;
                        a0 = r[gq * FS];                       // a row m = gq
                        if (a_hi) a1 = r[(8 + gq) * FS];       // a row m = 8 + gq (c = 2)
                        b0 = r[(12 + gq) * FS];                // b col n = gq
                        b1 = r[(20 + gq) * FS];                // b col n = 8 + gq
                    }
                    dmma_8x8x4(D[0][0], a0, b0);
                    dmma_8x8x4(D[0][1], a0, b1);
                    dmma_8x8x4(D[1][0], a1, b0);
                    dmma_8x8x4(D[1][1], a1, b1);
                }
                nidx += cntk;
                if (nidx < navail || cntk == 0) break;
            }
        }
        // Emit local plane kz = 0 (tile nt = 0, lanes tq < 2), then slide:
        // kz <- kz + 1 is a swap between lanes tq and tq ^ 2 and tiles.
        const int SL = st % MCfg::R, PH = phase;
        {
            double* pp = patch + (PH * MCfg::R + SL) * MCfg::PATCH + wid * PS;
            if (tq < 2) {
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    const int m = mt * 8 + gq;
                    if (m < 12) {
                        const int c = m >> 2, ix = m & 3;
                        pp[c * 16 + (2 * tq) * W + ix] = D[mt][0][0];
                        pp[c * 16 + (2 * tq + 1) * W + ix] = D[mt][0][1];
                    }
                }
            }
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const double x0 = __shfl_xor_sync(FULL, D[mt][0][e], 2);
                    const double x1 = __shfl_xor_sync(FULL, D[mt][1][e], 2);
                    D[mt][0][e] = (tq & 2) ? x1 : x0;
                    D[mt][1][e] = (tq & 2) ? 0.0 : x1;
                }
        }
        if (SL != MCfg::R - 1 && st + 1 < T) continue;
        __syncthreads();
        if (g_active) {
            for (int sl = 0; sl <= SL; ++sl) {
                const int kk = k - SL + sl;
                const double* pb = patch + (PH * MCfg::R + sl) * MCfg::PATCH + g_base;
                double s = 0.0;
#pragma unroll
                for (int tp = 0; tp < 16; ++tp)
                    if (g_taps & (1u << tp)) s += pb[(tp >> 2) * SY + (tp & 3) * SX];
                const int Z = wrap_index(kk + OFF, g.nz);
                const size_t node = g_xy + (size_t)plane_cells * (size_t)Z;
                const bool zc = (kk >= k0 + W - 1) && (kk < k1);
                if (g_inxy && zc)
                    g_field[node] = s;
                else if (s != 0.0)
                    atomicAdd(g_field + node, s);
            }
        }
        phase ^= 1;
    }
}

template <int ORDER>
void launch_dmma(const GridD& g, const CAos& p, const uint32_t* off, const uint32_t* cnt, double q, double* j,
                 int num_sms, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        PICGPU_CUDA_TRY(cudaFuncSetAttribute(deposit_current_dmma_kernel<ORDER>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)MCfg::SMEM));
        configured = true;
    }
    const int tx = div_up(g.nx, MCfg::PX), ty = div_up(g.ny, MCfg::PY);
    const long long tiles = (long long)tx * ty;
    const long long target = (long long)num_sms * MCfg::MINB * 8;
    int zch = (int)std::max<long long>(1, (target + tiles - 1) / tiles);
    zch = std::min(zch, std::max(1, g.nz / 16));
    const int zlen = div_up(g.nz, zch);
    zch = div_up(g.nz, zlen);
    dim3 grid(tx, ty, zch);
    deposit_current_dmma_kernel<ORDER><<<grid, MCfg::NT, MCfg::SMEM, st>>>(g, p, off, cnt, q, j, j + g.ncells,
                                                                          j + 2 * (size_t)g.ncells, zlen);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Orders 2 and 3, "mma" kernel v4: v3's decomposition (a CTA of 8x4 cell
// pencils walks a z-chunk; every lane runs one particle's prologue -- the
// fused push included -- and stages it; emitted planes meet in the shared
// patch and a gather flushes each node once) with the per-cell contraction
// J_cell += sum_p a_p (x) b_p on the FP64 tensor cores: mma.sync m8n8k4 f64,
// M = (c, ix) 12 rows padded to 16, N = (kz, jy) 16 columns, K = 4 particles.
// A warp serves 4 pencils (8 particles of each per chunk); its accumulators
// are 4 pencils x 2 x 2 m8n8 tiles = 32 doubles per lane (v3: 48 per lane for
// 8 pencils).  One DMMA replaces 8 DFMA instructions: the contraction drops
// from ~9 to ~3 warp-instructions per particle; the FP64 pipe is the same one
// (tools/fp64_pipes.cu), so the padding costs pipe time, not issue slots.
// The z window slides by index rotation: at z-step R the staged b puts
// logical plane kz in column block (kz + R) & 3, so the plane to emit is the
// column block R -- no accumulator moves.
struct V4Cfg {
    static constexpr int W = 4, PX = 8, PY = 4, NP = PX * PY, NW = 8, NT = NW * 32;
    static constexpr int PPW = 4, CH = 8;  // pencils per warp, particles per pencil per chunk
#ifdef PICGPU_V4_MINB
    static constexpr int MINB = PICGPU_V4_MINB;
#else
    static constexpr int MINB = 2;
#endif
    static constexpr int NF = 28, FS = 36;  // staged fields a[(c,ix)] 12 | b[(kz,jy)] 16; per-warp stride
    static constexpr int REC = NF * FS;
    static constexpr int PSTRIDE = NP + 2;
    static constexpr int PATCH = W * W * 3 * PSTRIDE;
    static constexpr size_t SMEM = (size_t)(2 * PATCH + NW * REC) * sizeof(double);
};

template <int W>
__device__ __forceinline__ double shifted_tap(const double (&v)[W], int t, int sh) {
    const double up = t >= 1 ? v[t >= 1 ? t - 1 : 0] : 0.0;
    const double dn = t + 1 < W ? v[t + 1 < W ? t + 1 : 0] : 0.0;
    return sh == 0 ? v[t] : (sh > 0 ? up : dn);
}

template <int ORDER, int PM = 0>
__global__ void __launch_bounds__(V4Cfg::NT, V4Cfg::MINB)
    deposit_current_kernel_v4(const GridD g, const CAos p, const uint32_t* __restrict__ off,
                              const uint32_t* __restrict__ cnt, const double q, double* __restrict__ jx,
                              double* __restrict__ jy, double* __restrict__ jz, const int zlen,
                              const PushCtx pc) {
    using C = V4Cfg;
    constexpr int W = 4, OFF = Shape<ORDER>::OFF, PX = C::PX, PY = C::PY, CH = C::CH, FS = C::FS;
    static_assert(Shape<ORDER>::W == 4, "v4 is the 4-tap kernel");
    constexpr int FX = PX + W - 1, FY = PY + W - 1;
    constexpr int NODES = 3 * FX * FY;
    constexpr int NIT = (NODES + C::NT - 1) / C::NT;
    constexpr unsigned FULL = 0xffffffffu;
    const double qs = q * (ORDER == 3 ? 1.0 / 216.0 : 0.125);

    extern __shared__ __align__(16) double smem[];
    double* patch = smem;  // [2][jy][ix][c][PSTRIDE]

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    double* recs = smem + 2 * C::PATCH + wid * C::REC;  // [NF][FS], particle = pq * CH + lg
    const int pq = lane >> 3, lg = lane & 7;            // prologue: pencil of the warp, chunk position
    const int gq = lane >> 2, tq = lane & 3;            // mma fragment coordinates
    const int grp = wid * C::PPW + pq;
    const int px = grp % PX, py = grp / PX;
    const int i0 = blockIdx.x * PX, j0 = blockIdx.y * PY;
    const int k0 = blockIdx.z * zlen;
    const int k1 = min(k0 + zlen, g.nz);
    const int i = i0 + px, j = j0 + py;
    const bool pv = (i < g.nx) && (j < g.ny);
    const int pxv = min(PX, g.nx - i0), pyv = min(PY, g.ny - j0);
    const bool alias_xy = (pxv + W - 1 > g.nx) || (pyv + W - 1 > g.ny);
    const uint32_t col = (uint32_t)i + (uint32_t)g.nx * (uint32_t)j;
    const uint32_t plane_cells = (uint32_t)g.nx * (uint32_t)g.ny;
    const double dci = (double)(i + g.sx_shift), dcj = (double)j;
    // this CTA's segment of the mover arrays (reserved with shared-memory atomics)
    [[maybe_unused]] const uint32_t seg = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    __shared__ unsigned s_movers;
    if (PM != 0 && threadIdx.x == 0) s_movers = 0;

    // gather plan (as v3)
    int gn_base[NIT], gn_node[NIT];
    unsigned gn_mask[NIT];
    bool gn_inner[NIT];
#pragma unroll
    for (int t = 0; t < NIT; ++t) {
        const int it = tid + t * C::NT;
        gn_mask[t] = 0u;
        gn_base[t] = 0;
        gn_node[t] = 0;
        gn_inner[t] = false;
        if (it < NODES) {
            const int c = it / (FX * FY);
            const int r = it - c * (FX * FY);
            const int uy = r / FX, ux = r - uy * FX;
            if (ux < pxv + W - 1 && uy < pyv + W - 1) {
#pragma unroll
                for (int dy = 0; dy < W; ++dy)
#pragma unroll
                    for (int dx = 0; dx < W; ++dx) {
                        const int qy = uy - dy, qx = ux - dx;
                        if (qy >= 0 && qy < pyv && qx >= 0 && qx < pxv) gn_mask[t] |= 1u << (dy * W + dx);
                    }
                gn_base[t] = (c << 28) | (c * C::PSTRIDE + uy * PX + ux);
                const int X = wrap_index(i0 + OFF + ux, g.nx);
                const int Y = wrap_index(j0 + OFF + uy, g.ny);
                gn_node[t] = X + g.nx * Y;
                gn_inner[t] = !alias_xy && ux >= W - 1 && ux <= pxv - 1 && uy >= W - 1 && uy <= pyv - 1;
            }
        }
    }

    // D[pp][mt][nt][e]: pencil pp of the warp; row m = mt*8 + gq = (c, ix); column
    // n = nt*8 + 2*tq + e = (kz block, jy) = (n >> 2, n & 3)
    double D[C::PPW][2][2][2];
#pragma unroll
    for (int a = 0; a < C::PPW; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int c = 0; c < 2; ++c) D[a][b][c][0] = D[a][b][c][1] = 0.0;

    {
        bool any = false;
        if (pv)
            for (int kk = k0 + lg; kk < k1; kk += CH) any |= cnt[col + plane_cells * kk] != 0;
        if (!__syncthreads_or(any)) {
            if (PM != 0 && threadIdx.x == 0) pc.seg_cnt[seg] = 0;
            return;
        }
    }
    uint32_t c_off = 0;
    int n_c = 0;
    if (pv && k0 < k1) {
        c_off = off[col + plane_cells * k0];
        n_c = (int)cnt[col + plane_cells * k0];
    }
    int last_busy = k0 - W;
    PData nxt{};
    if (lg < n_c) load_particle<PM != 0>(p, c_off + lg, nxt);
    const bool a_hi = gq < 4;  // rows 8..11 of m-tile 1 are c = 2; 12..15 are padding

    int buf = 0;
    const int kend = k1 + W - 1;
    for (int k = k0; k < kend; ++k) {
        const int R = (k - k0) & (W - 1);
        const bool busy = k < k1 && n_c > 0;
        if (k < k1) {
            uint32_t n_off = 0;
            int n_n = 0;
            if (pv && k + 1 < k1) {
                n_off = off[col + plane_cells * (k + 1)];
                n_n = (int)cnt[col + plane_cells * (k + 1)];
            }
            const double dck = (double)k;
            const int m = (int)__reduce_max_sync(FULL, (unsigned)n_c);
            if (m == 0 && lg < n_n) load_particle<PM != 0>(p, n_off + lg, nxt);
            for (int base = 0; base < m; base += CH) {
                [[maybe_unused]] bool mv = false;
                [[maybe_unused]] uint32_t mv_cell = 0;
                [[maybe_unused]] unsigned mv_bal = 0, mv_b0 = 0;
                {
                    PData cur = nxt;
                    bool valid = base + lg < n_c && !is_gap(cur.x);
                    if (base + CH < m) {
                        if (base + CH + lg < n_c) load_particle<PM != 0>(p, c_off + base + CH + lg, nxt);
                    } else if (lg < n_n) {
                        load_particle<PM != 0>(p, n_off + lg, nxt);
                    }
                    double a[3][W], sy[W], sz[W];
                    if constexpr (PM != 0) {
                        double fx = 0.0, fy = 0.0, fz = 0.0;
                        int shx = 0, shy = 0, shz = 0;
                        if (valid)
                            valid = push_fused<PM == 2>(g, pc, cur, c_off + (uint32_t)(base + lg),
                                                        col + plane_cells * (uint32_t)k, i, j, k, dci, dcj, dck,
                                                        fx, fy, fz, mv, mv_cell, shx, shy, shz);
                        mv_bal = __ballot_sync(FULL, mv);
                        if (mv_bal && lane == __ffs(mv_bal) - 1)
                            mv_b0 = atomicAdd(&s_movers, (unsigned)__popc(mv_bal));
                        window_from_fractions<ORDER>(cur, qs, valid, fx, fy, fz, a, sy, sz);
                        if (mv) {  // a mover's taps, shifted into this cell's window by its cell step
                            double t0[3][W], t1[W], t2[W];
#pragma unroll
                            for (int t = 0; t < W; ++t) {
#pragma unroll
                                for (int c = 0; c < 3; ++c) t0[c][t] = shifted_tap<W>(a[c], t, shx);
                                t1[t] = shifted_tap<W>(sy, t, shy);
                                t2[t] = shifted_tap<W>(sz, t, shz);
                            }
#pragma unroll
                            for (int t = 0; t < W; ++t) {
#pragma unroll
                                for (int c = 0; c < 3; ++c) a[c][t] = t0[c][t];
                                sy[t] = t1[t];
                                sz[t] = t2[t];
                            }
                        }
                    } else {
                        particle_window_sel<ORDER>(g, cur, qs, valid, dci, dcj, dck, a, sy, sz);
                    }
                    double* rr = recs + pq * CH + lg;
#pragma unroll
                    for (int c = 0; c < 3; ++c)
#pragma unroll
                        for (int t = 0; t < W; ++t) rr[(c * W + t) * FS] = a[c][t];
                    // b in rotated column blocks: logical plane kz at block (kz + R) & 3
#pragma unroll
                    for (int kz = 0; kz < W; ++kz) {
                        double* rb = rr + (12 + ((kz + R) & (W - 1)) * W) * FS;
#pragma unroll
                        for (int t = 0; t < W; ++t) rb[t * FS] = sy[t] * sz[kz];
                    }
                }
                __syncwarp();
                // contraction: per pencil of the warp, groups of 4 particles
#pragma unroll
                for (int pp = 0; pp < C::PPW; ++pp) {
                    const int np = __shfl_sync(FULL, n_c, pp * CH) - base;  // this pencil's particles left
#pragma unroll
                    for (int kg = 0; kg < CH / 4; ++kg) {
                        if (kg * 4 >= np) break;
                        const double* r = recs + pp * CH + kg * 4 + tq;
                        const double a0 = r[gq * FS];
                        const double a1 = a_hi ? r[(8 + gq) * FS] : 0.0;
                        const double b0 = r[(12 + gq) * FS];
                        const double b1 = r[(20 + gq) * FS];
                        dmma_8x8x4(D[pp][0][0], a0, b0);
                        dmma_8x8x4(D[pp][0][1], a0, b1);
                        dmma_8x8x4(D[pp][1][0], a1, b0);
                        dmma_8x8x4(D[pp][1][1], a1, b1);
                    }
                }
                if constexpr (PM != 0) {
                    if (mv_bal) {
                        const unsigned b0 = __shfl_sync(FULL, mv_b0, __ffs(mv_bal) - 1);
                        if (mv) {
                            const unsigned idx = b0 + (unsigned)__popc(mv_bal & ((1u << lane) - 1u));
                            size_t e = (size_t)seg * pc.segcap + idx;
                            if (idx >= pc.segcap) {  // segment full: the shared overflow segment
                                const unsigned o = atomicAdd(&pc.ctr->ovf_movers, 1u);
                                e = o < pc.ovcap ? (size_t)pc.nseg * pc.segcap + o : ~(size_t)0;
                            }
                            if (e != ~(size_t)0) {
                                pc.mslot[e] = c_off + (uint32_t)(base + lg);
                                pc.mbin[e] = col + plane_cells * (uint32_t)k;
                                pc.mcellseg[e] = mv_cell;
                            }
                        }
                    }
                }
                __syncwarp();
            }
            c_off = n_off;
            n_c = n_n;
        }
        // logical plane 0 sits in column block R (tile R >> 1, lanes with tq >> 1 == R & 1):
        // emit it into the patch and zero it (it becomes the window's top plane)
        {
            double* pb = patch + buf * C::PATCH + wid * C::PPW;
            const bool mine = (tq >> 1) == (R & 1);
            auto emit = [&](auto NTc) {
                constexpr int NT_ = decltype(NTc)::value;
#pragma unroll
                for (int pp = 0; pp < C::PPW; ++pp)
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int mrow = mt * 8 + gq;
                            const int jyv = (2 * tq + e) & 3;
                            if (mine && mrow < 12)
                                pb[((jyv * W + (mrow & 3)) * 3 + (mrow >> 2)) * C::PSTRIDE + pp] = D[pp][mt][NT_][e];
                            if (mine) D[pp][mt][NT_][e] = 0.0;
                        }
            };
            if (R < 2)
                emit(std::integral_constant<int, 0>{});
            else
                emit(std::integral_constant<int, 1>{});
        }
        if (__syncthreads_or(busy)) last_busy = k;
        if (last_busy >= k - (W - 1)) {
            const double* pb = patch + buf * C::PATCH;
            const int Z = wrap_index(k + OFF, g.nz);
            const bool zc = (k >= k0 + W - 1) && (k < k1);
            const size_t zrow = (size_t)plane_cells * (size_t)Z;
#pragma unroll
            for (int t = 0; t < NIT; ++t) {
                const unsigned msk = gn_mask[t];
                if (!msk) continue;
                const int c = gn_base[t] >> 28;
                const double* src = pb + (gn_base[t] & 0x0fffffff);
                double v[W * W];
#pragma unroll
                for (int dy = 0; dy < W; ++dy)
#pragma unroll
                    for (int dx = 0; dx < W; ++dx)
                        v[dy * W + dx] = (msk & (1u << (dy * W + dx)))
                                             ? src[(dy * W + dx) * 3 * C::PSTRIDE - dy * PX - dx]
                                             : 0.0;
#pragma unroll
                for (int h = W * W / 2; h >= 1; h /= 2)
#pragma unroll
                    for (int e = 0; e < h; ++e) v[e] += v[e + h];
                const double s = v[0];
                double* f = c == 0 ? jx : (c == 1 ? jy : jz);
                const size_t node = (size_t)gn_node[t] + zrow;
                if (zc && gn_inner[t])
                    f[node] = s;
                else if (s != 0.0)
                    atomicAdd(f + node, s);
            }
        }
        buf ^= 1;
    }
    if constexpr (PM != 0) {  // this CTA's mover count (every reservation precedes the last barrier)
        __syncthreads();
        if (threadIdx.x == 0) pc.seg_cnt[seg] = s_movers;
    }
}

// One mover segment per CTA of the fused kernel: its size and count.
inline void set_segments(PushCtx& pc, const dim3& grid, PushCtx* used) {
    const uint64_t nseg = (uint64_t)grid.x * grid.y * grid.z;
    if (nseg > kMaxFusedCtas) throw Status{PICGPU_ELENGTH, "fused step: too many CTAs for the mover segments"};
    pc.nseg = (uint32_t)nseg;
    pc.segcap = (uint32_t)(pc.mcap / 2 / nseg);
    pc.ovcap = pc.mcap - pc.nseg * pc.segcap;
    if (used) *used = pc;
}

template <int ORDER, int PM>
void launch_v4(const GridD& g, const CAos& p, const uint32_t* off, const uint32_t* cnt, double q, double* j,
               int num_sms, cudaStream_t st, PushCtx pc, PushCtx* used = nullptr) {
    using C = V4Cfg;
    static bool configured = false;
    if (!configured) {
        PICGPU_CUDA_TRY(cudaFuncSetAttribute(deposit_current_kernel_v4<ORDER, PM>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
        configured = true;
    }
    const int tx = div_up(g.nx, C::PX), ty = div_up(g.ny, C::PY);
    const long long tiles = (long long)tx * ty;
    const long long target = (long long)num_sms * C::MINB * 4;
    int zch = (int)std::max<long long>(1, (target + tiles - 1) / tiles);
    zch = std::min(zch, std::max(1, g.nz / (4 * C::W)));
    const int zlen = div_up(g.nz, zch);
    zch = div_up(g.nz, zlen);
    dim3 grid(tx, ty, zch);
    if constexpr (PM != 0) set_segments(pc, grid, used);
    deposit_current_kernel_v4<ORDER, PM><<<grid, C::NT, C::SMEM, st>>>(g, p, off, cnt, q, j, j + g.ncells,
                                                                      j + 2 * (size_t)g.ncells, zlen, pc);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

static bool use_v4() {
    static const bool v = [] {
        const char* e = std::getenv("PICGPU_J_V4");
        return e && e[0] == '1';
    }();
    return v;
}

template <int ORDER>
void launch_warp(const GridD& g, const CAos& p, const uint32_t* off, const uint32_t* cnt, double q, double* j,
                 int num_sms, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        PICGPU_CUDA_TRY(cudaFuncSetAttribute(deposit_current_warp_kernel<ORDER>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WCfg::SMEM));
        configured = true;
    }
    const int tx = div_up(g.nx, WCfg::PX), ty = div_up(g.ny, WCfg::PY);
    const long long tiles = (long long)tx * ty;
    const long long target = (long long)num_sms * WCfg::MINB * 8;
    int zch = (int)std::max<long long>(1, (target + tiles - 1) / tiles);
    zch = std::min(zch, std::max(1, g.nz / 16));
    const int zlen = div_up(g.nz, zch);
    zch = div_up(g.nz, zlen);
    dim3 grid(tx, ty, zch);
    deposit_current_warp_kernel<ORDER><<<grid, WCfg::NT, WCfg::SMEM, st>>>(g, p, off, cnt, q, j, j + g.ncells,
                                                                          j + 2 * (size_t)g.ncells, zlen);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

// z-chunked grid of one of the pencil kernels (v3 or the original v1); PM > 0:
// the fused push + detect + deposit form of v3.
template <int ORDER, class C, bool V3, int PM = 0, bool SLAB = false>
void launch_kernel(const GridD& g, const CAos& p, const uint32_t* off, const uint32_t* cnt, double q, double* j,
                   int num_sms, cudaStream_t st, PushCtx pc = PushCtx{}, PushCtx* used = nullptr) {
    static_assert(V3 || PM == 0, "the fused step runs on the v3 kernel");
    using L = JLayout<ORDER, C>;
    constexpr int W = L::W;
    constexpr size_t smem = V3 ? L::SMEM3 : JLayout<ORDER>::SMEM;
    static bool configured = false;
    if (!configured) {
        if constexpr (V3)
            PICGPU_CUDA_TRY(cudaFuncSetAttribute(deposit_current_kernel_v3<ORDER, C, PM, SLAB>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        else
            PICGPU_CUDA_TRY(cudaFuncSetAttribute(deposit_current_kernel<ORDER>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
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
    if constexpr (PM != 0) set_segments(pc, grid, used);
    if constexpr (V3)
        deposit_current_kernel_v3<ORDER, C, PM, SLAB><<<grid, L::NT, smem, st>>>(g, p, off, cnt, q, j, j + g.ncells,
                                                                                j + 2 * (size_t)g.ncells, zlen, pc);
    else
        deposit_current_kernel<ORDER><<<grid, L::NT, smem, st>>>(g, p, off, cnt, q, j, j + g.ncells,
                                                                 j + 2 * (size_t)g.ncells, zlen);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

template <int ORDER>
void launch_order(const GridD& g, const CAos& p, const uint32_t* off, const uint32_t* cnt, double q, double* j,
                  int num_sms, cudaStream_t st) {
    static const bool v1 = [] {
        const char* e = std::getenv("PICGPU_J_LANE");
        return e && std::string(e) == "v1";
    }();
    // v3 (default): orders 2/3 with JCfg<ORDER>, CIC with 2 lanes per pencil
#ifdef PICGPU_J_G8
    using C3 = std::conditional_t<ORDER == 1, JCfgCic3, JCfgG8>;
#else
    using C3 = std::conditional_t<ORDER == 1, JCfgCic3, JCfg<ORDER>>;
#endif
    if constexpr (ORDER != 1) {
        if (use_v4()) return launch_v4<ORDER, 0>(g, p, off, cnt, q, j, num_sms, st, PushCtx{});
    }
    if (v1)
        launch_kernel<ORDER, JCfg<ORDER>, false>(g, p, off, cnt, q, j, num_sms, st);
    else
        launch_kernel<ORDER, C3, true>(g, p, off, cnt, q, j, num_sms, st);
}

}  // namespace

// Order-2/3 kernel variant (ablation / profiling; PICGPU_J_VARIANT):
//   lane (default) -- 8 pencils per warp, 48 DFMA accumulators per lane
//   dfma           -- one warp per pencil, streamed chunks, 24 accumulators per lane
//   dmma           -- one warp per pencil, FP64 tensor-core contraction
static int j_variant() {
    static const int v = [] {
        const char* e = std::getenv("PICGPU_J_VARIANT");
        if (!e) return 0;
        const std::string s(e);
        return s == "dfma" ? 1 : s == "dmma" ? 2 : 0;
    }();
    return v;
}

// J must be zeroed by the caller (halo nodes are reduced into it).
void launch_deposit_current(int order, const GridD& g, const CAos& p, const uint32_t* off, const uint32_t* cnt,
                            double q, double* j, int num_sms, cudaStream_t st, int kernel) {
    const int k = kernel == kJDefault ? j_variant() : kernel;
    switch (order) {
        case 1: launch_order<1>(g, p, off, cnt, q, j, num_sms, st); break;
        case 2:
            if (k == kJVector) launch_warp<2>(g, p, off, cnt, q, j, num_sms, st);
            else if (k == kJMatrix) launch_dmma<2>(g, p, off, cnt, q, j, num_sms, st);
            else launch_order<2>(g, p, off, cnt, q, j, num_sms, st);
            break;
        case 3:
            if (k == kJVector) launch_warp<3>(g, p, off, cnt, q, j, num_sms, st);
            else if (k == kJMatrix) launch_dmma<3>(g, p, off, cnt, q, j, num_sms, st);
            else launch_order<3>(g, p, off, cnt, q, j, num_sms, st);
            break;
        default: throw Status{PICGPU_EINVAL, "deposit: shape order must be 1, 2 or 3"};
    }
}

namespace {

template <int ORDER>
void launch_push_order(const GridD& g, PushCtx& pc, const uint32_t* off, const uint32_t* cnt, double q,
                       double* j, int num_sms, cudaStream_t st) {
#ifdef PICGPU_J_G8
    using C3 = std::conditional_t<ORDER == 1, JCfgCic3, JCfgG8>;
#else
    using C3 = std::conditional_t<ORDER == 1, JCfgCic3, JCfg<ORDER>>;
#endif
    const bool p2 = g.pow2x && g.pow2y && g.pow2z && g.gpow2Lx && g.pow2Ly && g.pow2Lz;
    const CAos p(pc.A);
    if constexpr (ORDER != 1) {
        if (use_v4() && !g.slab) {
            if (p2)
                return launch_v4<ORDER, 2>(g, p, off, cnt, q, j, num_sms, st, pc, &pc);
            return launch_v4<ORDER, 1>(g, p, off, cnt, q, j, num_sms, st, pc, &pc);
        }
    }
    if (g.slab) {
        if (p2)
            launch_kernel<ORDER, C3, true, 2, true>(g, p, off, cnt, q, j, num_sms, st, pc, &pc);
        else
            launch_kernel<ORDER, C3, true, 1, true>(g, p, off, cnt, q, j, num_sms, st, pc, &pc);
    } else if (p2) {
        launch_kernel<ORDER, C3, true, 2>(g, p, off, cnt, q, j, num_sms, st, pc, &pc);
    } else {
        launch_kernel<ORDER, C3, true, 1>(g, p, off, cnt, q, j, num_sms, st, pc, &pc);
    }
}

// Movers of the fused step, W threads per mover (one z-plane of its window
// each): thread 0 copies the particle from its slot into the mover record and
// turns the slot into a hole of its old bin (delete_in_bin, gpma.hpp:328-335).
// The fused kernel deposited the mover's taps that fall inside its old cell's
// window (a mover steps at most one cell per axis); each thread reduces the
// rest of its plane -- the nodes outside that window -- into J (RED.ADD.F64):
// 16 of 64 nodes for a one-axis QSP mover.
template <int ORDER>
__global__ void __launch_bounds__(256) k_movers(const GridD g, const PushCtx pc, const Soa M,
                                                const uint32_t* __restrict__ off, uint32_t* __restrict__ holes,
                                                uint32_t* __restrict__ hl, const double qs, double* __restrict__ jx,
                                                double* __restrict__ jy, double* __restrict__ jz) {
    constexpr int W = Shape<ORDER>::W, OFF = Shape<ORDER>::OFF;
    // one CTA per mover segment (the last: the shared overflow segment); its
    // movers take a block of the compact mover list (any order of blocks: the
    // list is a set, as the reference's pending moves are applied one by one)
    // (the overflow segment is split over the CTAs past the last segment)
    __shared__ uint32_t s_base, s_n, s_first;
    const uint32_t sg = min(blockIdx.x, pc.nseg);
    if (threadIdx.x == 0) {
        uint32_t c, n, first = 0;
        if (blockIdx.x < pc.nseg) {
            c = pc.seg_cnt[sg];
            n = min(c, pc.segcap);  // the rest went to the overflow segment
            c = n;
        } else {
            const uint32_t part = blockIdx.x - pc.nseg, parts = gridDim.x - pc.nseg;
            const uint32_t o = pc.ctr->ovf_movers;
            const uint32_t total = min(o, pc.ovcap);
            const uint32_t chunk = (total + parts - 1) / parts;
            first = min(part * chunk, total);
            n = min(total - first, chunk);
            c = n;
            if (part == 0) {
                if (o > total) atomicAdd(&pc.ctr->mover_drop, o - total);
                c += o - total;  // dropped movers moved too
            }
        }
        s_n = n;
        s_first = first;
        s_base = n ? atomicAdd(&pc.ctr->nmovers, n) : 0u;
        if (c) atomicAdd(&pc.ctr->moved, (unsigned long long)c);
    }
    __syncthreads();
    const uint32_t nm = s_n;
    const int lane = threadIdx.x & 31;
    const unsigned grp = ((1u << W) - 1u) << (lane & ~(W - 1));  // the W lanes of one mover
    for (uint32_t t = threadIdx.x; t < nm * W; t += blockDim.x) {
        const uint32_t local = t / W;
        const uint64_t i = (uint64_t)s_base + local;  // compact index
        const int kz = (int)(t % W);
        const size_t e = (size_t)sg * pc.segcap + s_first + local;
        const uint32_t s = pc.mslot[e], b = pc.mbin[e];
        const double2* rec = reinterpret_cast<const double2*>(pc.A.p + s);
        const double2 r0 = rec[0], r1 = rec[1], r2 = rec[2], r3 = rec[3];
        const double x = r0.x, y = r0.y, z = r1.x, vx = r1.y, vy = r2.x, vz = r2.y, w = r3.x;
        __syncwarp(grp);  // every lane of the mover has read the slot before it becomes a hole
        const uint32_t mc = pc.mcellseg[e];
        if (mc >= kLeaveRight) {  // left the slab: an exchange record for the neighbour, no deposit
            if (kz == 0) {
                pc.mcell[i] = kNoCell;  // k_insert skips the entry
                const int dir = mc == kLeaveLeft ? 0 : 1;
                const unsigned li = atomicAdd(&pc.ctr->nleave[dir], 1u);
                if (li < pc.lcap) {
                    double* rr = pc.L + ((size_t)dir * pc.lcap + li) * 8;
                    rr[0] = x; rr[1] = y; rr[2] = z;
                    rr[3] = vx; rr[4] = vy; rr[5] = vz;
                    rr[6] = w;
                    rr[7] = r3.y;
                    push_hole(pc.A, s, b, off, holes, hl);
                } else {
                    raise_error(&pc.ctr->err, PICGPU_ELENGTH);
                }
            }
            continue;
        }
        if (kz == 0) {
            M.x[i] = x;
            M.y[i] = y;
            M.z[i] = z;
            M.vx[i] = vx;
            M.vy[i] = vy;
            M.vz[i] = vz;
            M.w[i] = w;
            M.id[i] = (uint64_t)__double_as_longlong(r3.y);
            pc.mcell[i] = mc;
            push_hole(pc.A, s, b, off, holes, hl);
        }
        int ci, cj, ck;
        double fx, fy, fz;
        cell_linear(g, x, y, z, ci, cj, ck, fx, fy, fz);
        const uint32_t bi = b % (uint32_t)g.nx, bj = (b / (uint32_t)g.nx) % (uint32_t)g.ny,
                       bk = b / ((uint32_t)g.nx * (uint32_t)g.ny);
        const int shx = cell_step(ci - (int)bi, g.gnx), shy = cell_step(cj - (int)bj, g.ny),
                  shz = cell_step(ck - (int)bk, g.nz);
        double sx[W], sy[W], sz[W];
        weights_scaled<ORDER>(fx, sx);
        weights_scaled<ORDER>(fy, sy);
        weights_scaled<ORDER>(fz, sz);
        const double qw = qs * w;
        const double wq0 = qw * vx, wq1 = qw * vy, wq2 = qw * vz;
        const bool zin = kz + shz >= 0 && kz + shz < W;
        const size_t Z = (size_t)wrap_index(ck + OFF + kz, g.nz);
        double szk = sz[0];  // sz[kz] without a local-memory array
#pragma unroll
        for (int t = 1; t < W; ++t) szk = kz == t ? sz[t] : szk;
#pragma unroll
        for (int jj = 0; jj < W; ++jj) {
            const bool yin = zin && jj + shy >= 0 && jj + shy < W;
            const double bb = sy[jj] * szk;
            const size_t row = ((size_t)wrap_index(cj + OFF + jj, g.ny) + (size_t)g.ny * Z) * (size_t)g.nx;
#pragma unroll
            for (int ix = 0; ix < W; ++ix) {
                if (yin && ix + shx >= 0 && ix + shx < W) continue;  // deposited by the fused kernel
                const double v = sx[ix] * bb;
                if (v == 0.0) continue;
                const size_t node = row + (size_t)wrap_index(ci + OFF + ix, g.nx);
                atomicAdd(jx + node, wq0 * v);
                atomicAdd(jy + node, wq1 * v);
                atomicAdd(jz + node, wq2 * v);
            }
        }
    }
}

}  // namespace

bool fused_step_available(int order, int kernel) {
    static const bool v1 = [] {
        const char* e = std::getenv("PICGPU_J_LANE");
        return e && std::string(e) == "v1";
    }();
    const int k = kernel == kJDefault ? j_variant() : kernel;
    return !v1 && (order == 1 || k == kJLane);
}

void launch_deposit_current_push(int order, const GridD& g, PushCtx& pc, const uint32_t* off,
                                 const uint32_t* cnt, double q, double* j, int num_sms, cudaStream_t st) {
    switch (order) {
        case 1: launch_push_order<1>(g, pc, off, cnt, q, j, num_sms, st); break;
        case 2: launch_push_order<2>(g, pc, off, cnt, q, j, num_sms, st); break;
        case 3: launch_push_order<3>(g, pc, off, cnt, q, j, num_sms, st); break;
        default: throw Status{PICGPU_EINVAL, "deposit: shape order must be 1, 2 or 3"};
    }
}

namespace {
// Slab arrivals of a fused step over their full window, W threads per record
// (one z-plane each).  The records sit after the local movers in M; their
// cells are owned by this slab, so the window stays on the slab grid.
template <int ORDER>
__global__ void __launch_bounds__(256) k_deposit_records(const GridD g, const Soa M, const StepCounters* ctr,
                                                         uint32_t base, const double qs, double* __restrict__ jx,
                                                         double* __restrict__ jy, double* __restrict__ jz) {
    constexpr int W = Shape<ORDER>::W, OFF = Shape<ORDER>::OFF;
    const uint64_t n = ctr->nimport;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * W;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = base + t / W;
        const int kz = (int)(t % W);
        const double x = M.x[i], y = M.y[i], z = M.z[i];
        int ci, cj, ck;
        double fx, fy, fz;
        cell_linear(g, x, y, z, ci, cj, ck, fx, fy, fz);
        double sx[W], sy[W], sz[W];
        weights_scaled<ORDER>(fx, sx);
        weights_scaled<ORDER>(fy, sy);
        weights_scaled<ORDER>(fz, sz);
        double szk = sz[0];
#pragma unroll
        for (int u = 1; u < W; ++u) szk = kz == u ? sz[u] : szk;
        const double qw = qs * M.w[i];
        const double wq0 = qw * M.vx[i], wq1 = qw * M.vy[i], wq2 = qw * M.vz[i];
        const size_t Z = (size_t)wrap_index(ck + OFF + kz, g.nz);
#pragma unroll
        for (int jj = 0; jj < W; ++jj) {
            const double bb = sy[jj] * szk;
            const size_t row = ((size_t)wrap_index(cj + OFF + jj, g.ny) + (size_t)g.ny * Z) * (size_t)g.nx;
#pragma unroll
            for (int ix = 0; ix < W; ++ix) {
                const double v = sx[ix] * bb;
                if (v == 0.0) continue;
                const size_t node = row + (size_t)wrap_index(ci + OFF + ix, g.nx);
                atomicAdd(jx + node, wq0 * v);
                atomicAdd(jy + node, wq1 * v);
                atomicAdd(jz + node, wq2 * v);
            }
        }
    }
}
}  // namespace

void launch_deposit_records(int order, const GridD& g, const Soa& M, const StepCounters* ctr, uint32_t base,
                            double q, double* j, int num_sms, cudaStream_t st) {
    const double qs = q * (order == 3 ? 1.0 / 216.0 : order == 2 ? 0.125 : 1.0);
    auto* kern = order == 1 ? k_deposit_records<1> : order == 2 ? k_deposit_records<2> : k_deposit_records<3>;
    kern<<<num_sms * 4, 256, 0, st>>>(g, M, ctr, base, qs, j, j + g.ncells, j + 2 * (size_t)g.ncells);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

void launch_movers(int order, const GridD& g, const PushCtx& pc, const Soa& M, const uint32_t* off,
                   uint32_t* holes, uint32_t* hl, double q, double* j, int num_sms, cudaStream_t st) {
    const double qs = q * (order == 3 ? 1.0 / 216.0 : order == 2 ? 0.125 : 1.0);
    auto* kern = order == 1 ? k_movers<1> : order == 2 ? k_movers<2> : k_movers<3>;
#ifndef PICGPU_MOVERS_NT
#define PICGPU_MOVERS_NT 256  // C2: 256 0.242 ms, 128 0.247, 64 0.264 (movers + insert + borrow)
#endif
    kern<<<pc.nseg + (uint32_t)num_sms * 4, PICGPU_MOVERS_NT, 0, st>>>(g, pc, M, off, holes, hl, qs, j, j + g.ncells, j + 2 * (size_t)g.ncells);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

}  // namespace picgpu
