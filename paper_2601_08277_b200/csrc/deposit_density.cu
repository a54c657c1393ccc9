// deposit_density.cu -- bit-exact charge density (pic::deposit_density,
// proj/include/pic/deposit.hpp:76-83).
//
// The reference scatters quantity[p]*S in STORAGE order, so node n's value is
// the left-to-right sum of its contributions ordered by storage index.  A GPU
// scatter (atomics or per-cell partials) reorders that sum (SURVEY Appendix
// A.3: 507/756 and 650/756 nodes differ).  This file is an ordered GATHER: a
// thread owns one node and visits exactly the particles that touch it, in
// storage order, with round-to-nearest intrinsics (no FMA contraction):
//
//  * sorted storage (the session's bins, or any cell-sorted store): the
//    contributions of node n come from its W^3 source cells; storage order is
//    then "source cells by ascending linear id, then slot order".  Per axis
//    the W wrapped source indices are sorted once; nested k->j->i loops over
//    the sorted lists visit cells in ascending linear id (grid.hpp:50-54).
//  * unsorted storage (stateless calls on arbitrary arrays): a k-way merge of
//    the W^3 per-cell lists by storage rank.
//
// Value order per contribution: wq * (sx[ix] * (sy[jy] * sz[kz])), exactly
// scatter_deposit's (deposit.hpp:41-48).
#include <cstdlib>

#include "common.cuh"
#include "kernels.hpp"

namespace picgpu {

namespace {

template <int ORDER>
__global__ void density_prologue(const GridD g, const CAos p, const double* __restrict__ quantity, double qscale,
                                 uint64_t slots, double* __restrict__ S, uint8_t* __restrict__ upb) {
    constexpr int W = Shape<ORDER>::W;
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= slots) return;
    const double x = p.p[s].x, y = p.p[s].y, z = p.p[s].z;
    if (is_gap(x)) {  // slack or a hole: a NaN quantity marks it for the gathers
        S[(size_t)(3 * Shape<ORDER>::W) * slots + s] = __longlong_as_double(0x7ff8000000000000LL);
        return;
    }
    double f[3];
    locate_x(g, x, f[0]);
    locate_axis(y, g.oy, g.dy, g.inv_dy, g.pow2y, g.ny, f[1]);
    locate_axis(z, g.oz, g.dz, g.inv_dz, g.pow2z, g.nz, f[2]);
    int bits = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double w[W];
        int up;
        Shape<ORDER>::weights(f[a], w, up);
        bits |= up << a;
#pragma unroll
        for (int t = 0; t < W; ++t) S[(size_t)(a * W + t) * slots + s] = w[t];
    }
    S[(size_t)(3 * W) * slots + s] = quantity ? quantity[s] : qscale * p.p[s].w;
    if (ORDER == 2) upb[s] = (uint8_t)bits;
}

// Sorted list of the W wrapped source indices of node coordinate X along one
// axis: src = wrap(X - OFF - t), tap t (node = cell + OFF + t).
template <int W, int OFF>
__device__ __forceinline__ void sources(int X, int n, int (&src)[W], int (&tap)[W]) {
#pragma unroll
    for (int t = 0; t < W; ++t) {
        src[t] = wrap_index(X - OFF - t, n);
        tap[t] = t;
    }
    // tiny insertion sort (W <= 4), ascending by src
#pragma unroll
    for (int a = 1; a < W; ++a)
#pragma unroll
        for (int b = a; b > 0; --b)
            if (src[b] < src[b - 1]) {
                const int ts = src[b]; src[b] = src[b - 1]; src[b - 1] = ts;
                const int tt = tap[b]; tap[b] = tap[b - 1]; tap[b - 1] = tt;
            }
}

// TSC pads 3 taps into the 4-wide window; the padded tap must be skipped, not
// added as zero (keeps -0.0 / +0.0 identical to the 27-tap reference loop).
template <int ORDER>
__device__ __forceinline__ bool tap_valid(int up, int t) {
    if (ORDER != 2) return true;
    return up ? t != 0 : t != 3;
}

// Box of nodes whose W source cells never wrap on any axis (sorted sources =
// ascending, contiguous): those go through density_rows.  Empty on an axis
// shorter than the stencil.
struct Interior {
    int lo[3], hi[3];  // inclusive node ranges per axis
    __host__ __device__ bool contains(int X, int Y, int Z) const {
        return X >= lo[0] && X <= hi[0] && Y >= lo[1] && Y <= hi[1] && Z >= lo[2] && Z <= hi[2];
    }
    __host__ __device__ bool empty() const { return lo[0] > hi[0] || lo[1] > hi[1] || lo[2] > hi[2]; }
};

template <int ORDER>
Interior interior_of(const GridD& g) {
    constexpr int W = Shape<ORDER>::W, OFF = Shape<ORDER>::OFF;
    // node X gathers cells X-OFF-(W-1) .. X-OFF
    const int n[3] = {g.nx, g.ny, g.nz};
    Interior in{};
    for (int a = 0; a < 3; ++a) {
        in.lo[a] = OFF + W - 1;
        in.hi[a] = n[a] - 1 + OFF;
    }
    return in;
}

template <int ORDER>
__global__ void density_gather_sorted(const GridD g, const uint32_t* __restrict__ off,
                                      const uint32_t* __restrict__ cnt, const double* __restrict__ S, uint64_t slots,
                                      const uint8_t* __restrict__ upb, double* __restrict__ rho, Interior skip) {
    constexpr int W = Shape<ORDER>::W, OFF = Shape<ORDER>::OFF;
    const uint64_t node = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= g.ncells) return;
    const int X = (int)(node % (uint32_t)g.nx);
    const int Y = (int)((node / (uint32_t)g.nx) % (uint32_t)g.ny);
    const int Z = (int)(node / ((uint64_t)g.nx * (uint32_t)g.ny));
    if (skip.contains(X, Y, Z)) return;
    int xs[W], xt[W], ys[W], yt[W], zs[W], zt[W];
    sources<W, OFF>(X, g.nx, xs, xt);
    sources<W, OFF>(Y, g.ny, ys, yt);
    sources<W, OFF>(Z, g.nz, zs, zt);
    const double* SQ = S + (size_t)(3 * W) * slots;
    double acc = 0.0;
    for (int zi = 0; zi < W; ++zi) {
        const double* Sz = S + (size_t)(2 * W + zt[zi]) * slots;
        for (int yi = 0; yi < W; ++yi) {
            const double* Sy = S + (size_t)(W + yt[yi]) * slots;
            const uint32_t row = (uint32_t)g.nx * ((uint32_t)ys[yi] + (uint32_t)g.ny * (uint32_t)zs[zi]);
            for (int xi = 0; xi < W; ++xi) {
                const double* Sx = S + (size_t)xt[xi] * slots;
                const uint32_t c = (uint32_t)xs[xi] + row;
                const uint32_t o = off[c], n = cnt[c];
                for (uint32_t u = 0; u < n; ++u) {
                    const uint32_t s = o + u;
                    const double qv = SQ[s];
                    if (qv != qv) continue;  // a hole of the bin (GPMA gap)
                    if (ORDER == 2) {
                        const int b = upb[s];
                        if (!tap_valid<ORDER>(b & 1, xt[xi]) || !tap_valid<ORDER>((b >> 1) & 1, yt[yi]) ||
                            !tap_valid<ORDER>((b >> 2) & 1, zt[zi]))
                            continue;
                    }
                    const double syz = __dmul_rn(Sy[s], Sz[s]);
                    const double sv = __dmul_rn(Sx[s], syz);
                    acc = __dadd_rn(acc, __dmul_rn(qv, sv));
                }
            }
        }
    }
    rho[node] = acc;
}

// The boundary shell of the sorted path, without the prologue: the exact
// weights of each visited slot are evaluated on the fly (the same
// locate_axis + Shape<ORDER>::weights as the prologue, so bit-identical), and
// only the shell's nodes pay for them.
template <int ORDER>
__global__ void density_gather_shell(const GridD g, const CAos p, const double* __restrict__ quantity, double qscale,
                                     const uint32_t* __restrict__ off, const uint32_t* __restrict__ cnt,
                                     double* __restrict__ rho, Interior skip) {
    constexpr int W = Shape<ORDER>::W, OFF = Shape<ORDER>::OFF;
    const uint64_t node = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= g.ncells) return;
    const int X = (int)(node % (uint32_t)g.nx);
    const int Y = (int)((node / (uint32_t)g.nx) % (uint32_t)g.ny);
    const int Z = (int)(node / ((uint64_t)g.nx * (uint32_t)g.ny));
    if (skip.contains(X, Y, Z)) return;
    int xs[W], xt[W], ys[W], yt[W], zs[W], zt[W];
    sources<W, OFF>(X, g.nx, xs, xt);
    sources<W, OFF>(Y, g.ny, ys, yt);
    sources<W, OFF>(Z, g.nz, zs, zt);
    double acc = 0.0;
    for (int zi = 0; zi < W; ++zi) {
        for (int yi = 0; yi < W; ++yi) {
            const uint32_t row = (uint32_t)g.nx * ((uint32_t)ys[yi] + (uint32_t)g.ny * (uint32_t)zs[zi]);
            for (int xi = 0; xi < W; ++xi) {
                const uint32_t c = (uint32_t)xs[xi] + row;
                const uint32_t o = off[c], n = cnt[c];
                for (uint32_t u = 0; u < n; ++u) {
                    const uint32_t sl = o + u;
                    const double xv = p.p[sl].x;
                    if (is_gap(xv)) continue;  // a hole of the bin (GPMA gap)
                    double f[3], w[3][W];
                    int up[3];
                    locate_x(g, xv, f[0]);
                    locate_axis(p.p[sl].y, g.oy, g.dy, g.inv_dy, g.pow2y, g.ny, f[1]);
                    locate_axis(p.p[sl].z, g.oz, g.dz, g.inv_dz, g.pow2z, g.nz, f[2]);
#pragma unroll
                    for (int a = 0; a < 3; ++a) Shape<ORDER>::weights(f[a], w[a], up[a]);
                    if (ORDER == 2 && (!tap_valid<ORDER>(up[0], xt[xi]) || !tap_valid<ORDER>(up[1], yt[yi]) ||
                                       !tap_valid<ORDER>(up[2], zt[zi])))
                        continue;
                    double sx = 0, sy = 0, sz = 0;
#pragma unroll
                    for (int t = 0; t < W; ++t) {
                        sx = t == xt[xi] ? w[0][t] : sx;
                        sy = t == yt[yi] ? w[1][t] : sy;
                        sz = t == zt[zi] ? w[2][t] : sz;
                    }
                    const double q = quantity ? quantity[sl] : qscale * p.p[sl].w;
                    const double syz = __dmul_rn(sy, sz);
                    const double sv = __dmul_rn(sx, syz);
                    acc = __dadd_rn(acc, __dmul_rn(q, sv));
                }
            }
        }
    }
    rho[node] = acc;
}

template <int ORDER>
__global__ void density_gather_merge(const GridD g, const uint32_t* __restrict__ off, const uint32_t* __restrict__ cnt,
                                     const uint32_t* __restrict__ rank, const double* __restrict__ S, uint64_t slots,
                                     const uint8_t* __restrict__ upb, double* __restrict__ rho) {
    constexpr int W = Shape<ORDER>::W, OFF = Shape<ORDER>::OFF;
    constexpr int NC = W * W * W;
    const uint64_t node = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= g.ncells) return;
    const int X = (int)(node % (uint32_t)g.nx);
    const int Y = (int)((node / (uint32_t)g.nx) % (uint32_t)g.ny);
    const int Z = (int)(node / ((uint64_t)g.nx * (uint32_t)g.ny));
    int xs[W], xt[W], ys[W], yt[W], zs[W], zt[W];
    sources<W, OFF>(X, g.nx, xs, xt);
    sources<W, OFF>(Y, g.ny, ys, yt);
    sources<W, OFF>(Z, g.nz, zs, zt);
    uint32_t head[NC], end[NC];
    int taps[NC];
#pragma unroll
    for (int zi = 0; zi < W; ++zi)
#pragma unroll
        for (int yi = 0; yi < W; ++yi)
#pragma unroll
            for (int xi = 0; xi < W; ++xi) {
                const int l = (zi * W + yi) * W + xi;
                const uint32_t c =
                    (uint32_t)xs[xi] + (uint32_t)g.nx * ((uint32_t)ys[yi] + (uint32_t)g.ny * (uint32_t)zs[zi]);
                head[l] = off[c];
                end[l] = off[c] + cnt[c];
                taps[l] = xt[xi] | (yt[yi] << 4) | (zt[zi] << 8);
            }
    const double* SQ = S + (size_t)(3 * W) * slots;
    double acc = 0.0;
    for (;;) {
        int best = -1;
        uint32_t br = 0xffffffffu;
        for (int l = 0; l < NC; ++l)
            if (head[l] < end[l]) {
                const uint32_t r = rank[head[l]];
                if (r < br) {
                    br = r;
                    best = l;
                }
            }
        if (best < 0) break;
        const uint32_t s = head[best]++;
        const int tx = taps[best] & 15, ty = (taps[best] >> 4) & 15, tz = taps[best] >> 8;
        if (ORDER == 2) {
            const int b = upb[s];
            if (!tap_valid<ORDER>(b & 1, tx) || !tap_valid<ORDER>((b >> 1) & 1, ty) ||
                !tap_valid<ORDER>((b >> 2) & 1, tz))
                continue;
        }
        const double syz = __dmul_rn(S[(size_t)(W + ty) * slots + s], S[(size_t)(2 * W + tz) * slots + s]);
        const double sv = __dmul_rn(S[(size_t)tx * slots + s], syz);
        acc = __dadd_rn(acc, __dmul_rn(SQ[s], sv));
    }
    rho[node] = acc;
}

// Row-staged ordered gather for the interior nodes.  CTA = RX x RY node
// columns (one warp per node row) over a z-chunk [Za, Zb) of nodes.  Source
// planes zs stream in ascending order, and within a plane the source rows ys
// in ascending order; each row's contiguous slot range (cells X0-OFF-(W-1) ..
// X0+RX-1-OFF, slack slots included) is staged into shared memory in pieces,
// with the exact weights (locate_axis + Shape<ORDER>::weights, as the
// prologue computes them) evaluated once per staged slot.  A node thread then
// adds, for each of its z-window nodes, the terms of its own W cells' slots in
// slot order.  Per node this is the reference's order -- source planes, rows,
// cells ascending (= ascending linear id), then slots -- with the same value
// expression q*(sx*(sy*sz)) and round-to-nearest intrinsics: bit-identical to
// density_gather_sorted (and to pic::deposit_density on this storage order).
#ifndef PICGPU_RHO_RX
#define PICGPU_RHO_RX 16
#endif
#ifndef PICGPU_RHO_RY
#define PICGPU_RHO_RY 16
#endif
#ifndef PICGPU_RHO_ZLEN
#define PICGPU_RHO_ZLEN 16
#endif
#ifndef PICGPU_RHO_CAP
#define PICGPU_RHO_CAP 512
#endif
constexpr int kRowX = PICGPU_RHO_RX, kRowY = PICGPU_RHO_RY, kRowCap = PICGPU_RHO_CAP;

template <int ORDER>
__global__ void __launch_bounds__(kRowX * kRowY)
    density_rows(const GridD g, const CAos p, const double* __restrict__ quantity, double qscale,
                 const uint32_t* __restrict__ off, const uint32_t* __restrict__ cnt, Interior in, int zlen,
                 double* __restrict__ rho) {
    constexpr int W = Shape<ORDER>::W, OFF = Shape<ORDER>::OFF;
    constexpr int NT = kRowX * kRowY;
    extern __shared__ __align__(16) double dsm[];
    double* s_q = dsm;                                     // [kRowCap]
    double (*s_w)[W][kRowCap] = reinterpret_cast<double (*)[W][kRowCap]>(dsm + kRowCap);  // sx, sy, sz taps
    int* s_xs = reinterpret_cast<int*>(dsm + (1 + 3 * W) * kRowCap);  // source x-cell, -1 for slack
    unsigned char* s_up = reinterpret_cast<unsigned char*>(s_xs + kRowCap);

    const int tid = threadIdx.x;
    const int X0 = in.lo[0] + blockIdx.x * kRowX, Y0 = in.lo[1] + blockIdx.y * kRowY;
    const int X = X0 + (tid % kRowX), Y = Y0 + (tid / kRowX);
    const int Za = in.lo[2] + blockIdx.z * zlen;
    const int Zb = min(Za + zlen, in.hi[2] + 1);
    const bool nv = X <= in.hi[0] && Y <= in.hi[1];
    const int Xl = min(X0 + kRowX - 1, in.hi[0]), Yl = min(Y0 + kRowY - 1, in.hi[1]);
    const int cx0 = X0 - OFF - (W - 1), cx1 = Xl - OFF;  // source x-cells of the CTA
    double acc[W];  // logical window: acc[t] is node zs + OFF + t at plane zs
#pragma unroll
    for (int t = 0; t < W; ++t) acc[t] = 0.0;

    for (int zs = Za - OFF - (W - 1); zs <= Zb - 1 - OFF; ++zs) {
        for (int ys = Y0 - OFF - (W - 1); ys <= Yl - OFF; ++ys) {
            const uint32_t rowc = (uint32_t)g.nx * ((uint32_t)ys + (uint32_t)g.ny * (uint32_t)zs);
            const uint32_t sbeg = off[rowc + cx0];
            const uint32_t send = off[rowc + cx1] + cnt[rowc + cx1];
            // this thread's cells X-OFF-(W-1) .. X-OFF in this row, if the row is in its y-window
            const int ty = Y - ys - OFF;
            const bool uses = nv && ty >= 0 && ty < W;
            uint32_t mbeg = 0, mend = 0;
            if (uses) {
                const uint32_t c_lo = rowc + (uint32_t)(X - OFF - (W - 1)), c_hi = rowc + (uint32_t)(X - OFF);
                mbeg = off[c_lo];
                mend = off[c_hi] + cnt[c_hi];
            }
            for (uint32_t piece = sbeg; piece < send; piece += kRowCap) {
                const uint32_t pn = min((uint32_t)kRowCap, send - piece);
                __syncthreads();  // the previous piece is consumed
                for (uint32_t i = tid; i < pn; i += NT) {
                    const uint32_t sl = piece + i;
                    const double x = p.p[sl].x;
                    if (__double_as_longlong(x) == -1LL) {  // slack sentinel
                        s_xs[i] = -1;
                        continue;
                    }
                    const double y = p.p[sl].y, z = p.p[sl].z;
                    double f[3];
                    s_xs[i] = locate_x(g, x, f[0]);
                    locate_axis(y, g.oy, g.dy, g.inv_dy, g.pow2y, g.ny, f[1]);
                    locate_axis(z, g.oz, g.dz, g.inv_dz, g.pow2z, g.nz, f[2]);
                    int bits = 0;
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        double w[W];
                        int up;
                        Shape<ORDER>::weights(f[a], w, up);
                        bits |= up << a;
#pragma unroll
                        for (int t = 0; t < W; ++t) s_w[a][t][i] = w[t];
                    }
                    if (ORDER == 2) s_up[i] = (unsigned char)bits;
                    s_q[i] = quantity ? quantity[sl] : qscale * p.p[sl].w;
                }
                __syncthreads();
                if (!uses || mend <= piece || mbeg >= piece + pn) continue;
                const uint32_t ib = max(mbeg, piece) - piece, ie = min(mend, piece + pn) - piece;
                for (uint32_t i = ib; i < ie; ++i) {
                    const int xs = s_xs[i];
                    if (xs < 0) continue;
                    const int tx = X - xs - OFF;
                    const double q = s_q[i];
                    const double sxv = s_w[0][tx][i];
                    const double syv = s_w[1][ty][i];
                    const int ub = ORDER == 2 ? s_up[i] : 0;
                    if (ORDER == 2 && (!tap_valid<ORDER>(ub & 1, tx) || !tap_valid<ORDER>((ub >> 1) & 1, ty)))
                        continue;
#pragma unroll
                    for (int t = 0; t < W; ++t) {
                        if (ORDER == 2 && !tap_valid<ORDER>((ub >> 2) & 1, t)) continue;
                        const double syz = __dmul_rn(syv, s_w[2][t][i]);
                        const double sv = __dmul_rn(sxv, syz);
                        acc[t] = __dadd_rn(acc[t], __dmul_rn(q, sv));
                    }
                }
            }
        }
        // node zs + OFF has seen its last source plane
        const int Zd = zs + OFF;
        if (nv && Zd >= Za && Zd < Zb)
            rho[(size_t)X + (size_t)g.nx * ((size_t)Y + (size_t)g.ny * (size_t)Zd)] = acc[0];
#pragma unroll
        for (int t = 0; t < W - 1; ++t) acc[t] = acc[t + 1];
        acc[W - 1] = 0.0;
    }
}

// ---------------------------------------------------------------------------
// Block-staged ordered gather, every node (wrapped sources included).
//
// A CTA owns a block of RX x RY x ZL nodes and keeps their sums in shared
// memory.  Per axis the block's source cells form one ascending run, or two
// when they wrap ([0, hi] then [lo, n-1]); streaming planes, then rows, then
// the cells of a row in ascending order visits every node's own source cells
// in ascending linear id -- the reference's storage order on a cell-sorted
// store (bins ascending, slots in order), wrapped or not.  Each source row's
// slot range is staged in pieces with the exact weights evaluated once per
// slot (locate_axis + Shape<ORDER>::weights); then thread (X, ty, tz) adds,
// for the one node (X, Y = ys+OFF+ty, Z = zs+OFF+tz) of its block that the row
// feeds, the terms of its W cells' slots in slot order: q*(sx*(sy*sz)) with
// round-to-nearest intrinsics, bit-identical to pic::deposit_density.  The
// (ty, tz) pairs are the fast thread index, so the 16 lanes sharing X read
// the same slots (broadcast).  Replaces the interior row kernel + the
// prologue-based shell gather (C2 QSP: 11.2 ms).
// L2 prefetch of the next source row's records while the current row is summed
// (C2: QSP 4.314 -> 4.287 ms, CIC 1.482 -> 1.466, TSC 5.977 -> 5.91: the loads are
// not what bounds this kernel).
#ifndef PICGPU_RHO_L2PF
#define PICGPU_RHO_L2PF 1
#endif

template <int ORDER>
struct DBCfg {
    static constexpr int W = Shape<ORDER>::W;
#ifndef PICGPU_RHO_CIC_RX
#define PICGPU_RHO_CIC_RX 32  // C2 CIC: 1.65 ms (64: 1.76-1.80, 16: 2.40)
#endif
#ifndef PICGPU_RHO_CIC_CAP
#define PICGPU_RHO_CIC_CAP 512
#endif
    static constexpr int RX = ORDER == 1 ? PICGPU_RHO_CIC_RX : 16, RY = ORDER == 1 ? 256 / PICGPU_RHO_CIC_RX : 16;
#ifdef PICGPU_RHO_ZL
    static constexpr int ZL = PICGPU_RHO_ZL;
#else
    static constexpr int ZL = 8;
#endif
    static constexpr int NT = RX * W * W;
#ifdef PICGPU_RHO_MINB
    static constexpr int MINB = PICGPU_RHO_MINB;
#else
    static constexpr int MINB = 3;  // C2 QSP: 4.35 ms at 3 CTAs/SM vs 5.05 at 2 (ZL 8)
#endif
    // SYZ: the staging also evaluates the W*W products sy*sz per slot (the
    // reference's inner product, deposit.hpp:41-48), so a term is
    // q*(sx*syz) from 3 broadcast-or-conflict-free loads: every one of the 16
    // (ty, tz) lanes of an x read its own syz array (odd stride), instead of
    // each lane recomputing sy*sz.  TSC keeps the explicit tap test.
    // C2 (128^3 x 16): CIC 1.58 ms with SYZ vs 1.64 without; QSP 4.90 vs 4.34 --
    // the term loop drops from ~11 to 8.25 warp-instructions per term, but the
    // heavier staging (16 more products and stores per slot) at half the piece
    // size doubles the row barriers (40% of the stall samples) -- so QSP keeps
    // the three weight arrays (profiles/r02/ncu_rho_syz.txt).
#ifndef PICGPU_RHO_SYZ
#define PICGPU_RHO_SYZ 1
#endif
    static constexpr bool SYZ = PICGPU_RHO_SYZ && ORDER == 1;
    static constexpr int CAP = SYZ ? (ORDER == 1 ? PICGPU_RHO_CIC_CAP : 256)
                                   : (ORDER == 1 ? PICGPU_RHO_CIC_CAP : 512);  // slots per staged piece
    static constexpr int WS = SYZ ? CAP + 1 : CAP + 2;  // staged array stride (bank skew)
    static constexpr int NA = SYZ ? W + W * W : 3 * W;  // staged weight arrays
    static constexpr int MAXC = RX + W + 1;  // cells per staged row
    static constexpr size_t SMEM = (size_t)(ZL * RY * RX + CAP + NA * WS) * 8 + (size_t)2 * MAXC * 4 + CAP;
};

struct Runs {  // ascending source cells along one axis: [a0, a1] then [b0, b1] (b0 > b1: none)
    int a0, a1, b0, b1;
    __device__ int len_a() const { return a1 - a0 + 1; }
    __device__ int len() const { return a1 - a0 + 1 + (b1 >= b0 ? b1 - b0 + 1 : 0); }
    __device__ int at(int k) const { return k < len_a() ? a0 + k : b0 + (k - len_a()); }
};

template <int W, int OFF>
__device__ __forceinline__ Runs source_runs(int B0, int Bn, int n) {
    const int lo = B0 - OFF - (W - 1), hi = B0 + Bn - 1 - OFF;
    if (hi - lo + 1 >= n) return Runs{0, n - 1, 1, 0};
    const int lw = wrap_index(lo, n), hw = wrap_index(hi, n);
    if (lw <= hw) return Runs{lw, hw, 1, 0};
    return Runs{0, hw, lw, n - 1};
}

// P2: every spacing is a power of two (the locate is a multiply by the exact
// reciprocal, no division code: the same correctly rounded value).
template <int ORDER, bool P2>
__global__ void __launch_bounds__(DBCfg<ORDER>::NT, DBCfg<ORDER>::MINB)
    density_blocks(const GridD g, const CAos p, const double* __restrict__ quantity, double qscale,
                   const uint32_t* __restrict__ off, const uint32_t* __restrict__ cnt, double* __restrict__ rho) {
    using C = DBCfg<ORDER>;
    constexpr int W = C::W, OFF = Shape<ORDER>::OFF, RX = C::RX, RY = C::RY, ZL = C::ZL, NT = C::NT, CAP = C::CAP;
    extern __shared__ __align__(16) double dsm[];
    double* s_acc = dsm;                        // [ZL][RY][RX]
    double* s_q = s_acc + ZL * RY * RX;         // [CAP]
    double* s_w = s_q + CAP;                    // [3][W][WS] (SYZ: sx [W][WS], then syz [W*W][WS])
    uint32_t* s_cb = reinterpret_cast<uint32_t*>(s_w + C::NA * C::WS);  // [MAXC] first slot of each row cell
    uint32_t* s_ce = s_cb + C::MAXC;                                     // [MAXC] end of its extent
    unsigned char* s_up = reinterpret_cast<unsigned char*>(s_ce + C::MAXC);  // [CAP] 0x80 valid | up bits
#if PICGPU_RHO_L2PF
    __shared__ uint32_t s_nx[2];
#endif

    const int tid = threadIdx.x;
    const int X0 = blockIdx.x * RX, Y0 = blockIdx.y * RY, Z0 = blockIdx.z * ZL;
    const int Bx = min(RX, g.nx - X0), By = min(RY, g.ny - Y0), Bz = min(ZL, g.nz - Z0);
    const int tyz = tid % (W * W), ty = tyz % W, tz = tyz / W, xl = tid / (W * W);
    const int X = X0 + xl;
    const bool xv = xl < Bx;
    for (int i = tid; i < ZL * RY * RX; i += NT) s_acc[i] = 0.0;

    const Runs rx = source_runs<W, OFF>(X0, Bx, g.nx);
    const Runs ry = source_runs<W, OFF>(Y0, By, g.ny);
    const Runs rz = source_runs<W, OFF>(Z0, Bz, g.nz);
    const int ncx = rx.len(), la = rx.len_a();
    // this thread's x source cells (ascending) as indices into the row's cell list
    int ck[W], ct[W];
    {
        int xs[W];
        sources<W, OFF>(xv ? X : 0, g.nx, xs, ct);
#pragma unroll
        for (int c = 0; c < W; ++c) ck[c] = xs[c] >= rx.a0 && xs[c] <= rx.a1 ? xs[c] - rx.a0 : la + xs[c] - rx.b0;
    }

    const int nzs = rz.len(), nys = ry.len();
    for (int zi = 0; zi < nzs; ++zi) {
        const int zs = rz.at(zi);
        const int zl = wrap_index(zs + OFF + tz, g.nz) - Z0;
        for (int yi = 0; yi < nys; ++yi) {
            const int ys = ry.at(yi);
            const int yl = wrap_index(ys + OFF + ty, g.ny) - Y0;
            const bool mine = xv && zl >= 0 && zl < Bz && yl >= 0 && yl < By;
            const uint32_t rowc = (uint32_t)g.nx * ((uint32_t)ys + (uint32_t)g.ny * (uint32_t)zs);
            __syncthreads();  // the previous row is consumed
            for (int k = tid; k < ncx; k += NT) {
                const uint32_t c = rowc + (uint32_t)rx.at(k);
                const uint32_t o = off[c];
                s_cb[k] = o;
                s_ce[k] = o + cnt[c];
            }
#if PICGPU_RHO_L2PF
            // the NEXT source row's run-A slot range (its bins are contiguous), for the L2 prefetch below
            if (tid >= NT - 2) {
                int ny2 = yi + 1, nz2 = zi;
                if (ny2 >= nys) {
                    ny2 = 0;
                    ++nz2;
                }
                uint32_t v = 0;
                if (nz2 < nzs) {
                    const uint32_t rc2 =
                        (uint32_t)g.nx * ((uint32_t)ry.at(ny2) + (uint32_t)g.ny * (uint32_t)rz.at(nz2));
                    v = off[rc2 + (uint32_t)(tid == NT - 2 ? rx.a0 : rx.a1 + 1)];
                }
                s_nx[tid - (NT - 2)] = v;
            }
#endif
            __syncthreads();
#if PICGPU_RHO_L2PF
            {   // one 128-byte line per thread: the next row's records land in L2 while this row is summed
                const char* pb = reinterpret_cast<const char*>(p.p);
                const size_t b1 = (size_t)s_nx[1] * 64;
                for (size_t b = (size_t)s_nx[0] * 64 + (size_t)tid * 128; b < b1; b += (size_t)NT * 128)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(pb + b));
            }
#endif
            // the row's stream: run A's slots [cb[0], ce[la-1]), then run B's
            const uint32_t lena = s_ce[la - 1] - s_cb[0];
            const uint32_t total = lena + (ncx > la ? s_ce[ncx - 1] - s_cb[la] : 0u);
            uint32_t mb[W], me[W];
#pragma unroll
            for (int c = 0; c < W; ++c) {
                const int k = ck[c];
                const uint32_t base = k < la ? s_cb[k] - s_cb[0] : lena + (s_cb[k] - s_cb[la]);
                mb[c] = base;
                me[c] = base + (s_ce[k] - s_cb[k]);
            }
            for (uint32_t piece = 0; piece < total; piece += CAP) {
                const uint32_t pn = min((uint32_t)CAP, total - piece);
                if (piece) __syncthreads();  // the previous piece is consumed
                for (uint32_t i = tid; i < pn; i += NT) {
                    const uint32_t pos = piece + i;
                    const uint32_t sl = pos < lena ? s_cb[0] + pos : s_cb[la] + (pos - lena);
                    const double2 r0 = reinterpret_cast<const double2*>(p.p + sl)[0];
                    if (is_gap(r0.x)) {  // slack or a hole
                        s_up[i] = 0;
                        if (ORDER != 2) {
                            // a zero term: adding +-0 never changes a node sum, which starts
                            // at +0.0 and so can never be -0.0 (x + -x rounds to +0.0)
                            s_q[i] = 0.0;
#pragma unroll
                            for (int a = 0; a < C::NA; ++a) s_w[a * C::WS + i] = 0.0;
                        }
                        continue;
                    }
                    double f[3];
                    locate_x<P2>(g, r0.x, f[0]);
                    locate_axis<P2>(r0.y, g.oy, g.dy, g.inv_dy, g.pow2y, g.ny, f[1]);
                    locate_axis<P2>(p.p[sl].z, g.oz, g.dz, g.inv_dz, g.pow2z, g.nz, f[2]);
                    int bits = 0;
                    if constexpr (C::SYZ) {
                        double wx[W], wy[W], wz[W];
                        int up;
                        Shape<ORDER>::weights(f[0], wx, up);
                        Shape<ORDER>::weights(f[1], wy, up);
                        Shape<ORDER>::weights(f[2], wz, up);
#pragma unroll
                        for (int t = 0; t < W; ++t) s_w[t * C::WS + i] = wx[t];
#pragma unroll
                        for (int a = 0; a < W; ++a)
#pragma unroll
                            for (int b = 0; b < W; ++b) s_w[(W + a * W + b) * C::WS + i] = __dmul_rn(wy[a], wz[b]);
                    } else {
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            double w[W];
                            int up;
                            Shape<ORDER>::weights(f[a], w, up);
                            bits |= up << a;
#pragma unroll
                            for (int t = 0; t < W; ++t) s_w[(a * W + t) * C::WS + i] = w[t];
                        }
                    }
                    s_up[i] = (unsigned char)(0x80 | bits);
                    s_q[i] = quantity ? quantity[sl] : qscale * p.p[sl].w;
                }
                __syncthreads();
                if (!mine) continue;
                double* ap = s_acc + ((size_t)zl * RY + yl) * RX + xl;
                double acc = *ap;
                if constexpr (C::SYZ) {
                    const double* syz = s_w + (W + ty * W + tz) * C::WS;
#pragma unroll
                    for (int c = 0; c < W; ++c) {
                        const uint32_t b = max(mb[c], piece), e = min(me[c], piece + pn);
                        const double* wx = s_w + ct[c] * C::WS;
#pragma unroll 4
                        for (uint32_t u = b; u < e; ++u) {
                            const uint32_t i = u - piece;
                            acc = __dadd_rn(acc, __dmul_rn(s_q[i], __dmul_rn(wx[i], syz[i])));
                        }
                    }
                    *ap = acc;
                    continue;
                }
                const double* wy = s_w + (W + ty) * C::WS;
                const double* wz = s_w + (2 * W + tz) * C::WS;
#pragma unroll
                for (int c = 0; c < W; ++c) {
                    const uint32_t b = max(mb[c], piece), e = min(me[c], piece + pn);
                    const double* wx = s_w + ct[c] * C::WS;
                    for (uint32_t u = b; u < e; ++u) {
                        const uint32_t i = u - piece;
                        if (ORDER == 2) {  // TSC: skip gaps and the padded tap
                            const int ub = s_up[i];
                            if (!(ub & 0x80) || !tap_valid<ORDER>(ub & 1, ct[c]) ||
                                !tap_valid<ORDER>((ub >> 1) & 1, ty) || !tap_valid<ORDER>((ub >> 2) & 1, tz))
                                continue;
                        }
                        const double syz = __dmul_rn(wy[i], wz[i]);
                        const double sv = __dmul_rn(wx[i], syz);
                        acc = __dadd_rn(acc, __dmul_rn(s_q[i], sv));
                    }
                }
                *ap = acc;
            }
        }
    }
    __syncthreads();
    for (int i = tid; i < ZL * RY * RX; i += NT) {
        const int xl2 = i % RX, yl2 = (i / RX) % RY, zl2 = i / (RX * RY);
        if (xl2 < Bx && yl2 < By && zl2 < Bz)
            rho[(size_t)(X0 + xl2) + (size_t)g.nx * ((size_t)(Y0 + yl2) + (size_t)g.ny * (size_t)(Z0 + zl2))] =
                s_acc[i];
    }
}

template <int ORDER>
void prologue(const GridD& g, const CAos& p, const double* quantity, double qscale, uint64_t slots, void* scratch,
              cudaStream_t st, double*& S, uint8_t*& upb) {
    constexpr int W = Shape<ORDER>::W;
    S = static_cast<double*>(scratch);
    upb = reinterpret_cast<uint8_t*>(S + (size_t)(3 * W + 1) * slots);
    if (slots == 0) return;
    density_prologue<ORDER><<<div_up((long long)slots, 256), 256, 0, st>>>(g, p, quantity, qscale, slots, S, upb);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

template <int ORDER>
void run_rows_and_shell(const GridD& g, const CAos& p, const double* quantity, double qscale, const uint32_t* off,
                        const uint32_t* cnt, uint64_t slots, void* scratch, double* rho, cudaStream_t st);

template <int ORDER>
void run_sorted(const GridD& g, const CAos& p, const double* quantity, double qscale, const uint32_t* off, const uint32_t* cnt,
                uint64_t slots, void* scratch, double* rho, cudaStream_t st) {
    static const bool rows = [] {
        const char* e = std::getenv("PICGPU_RHO_ROWS");
        return e && e[0] == '1';
    }();
    if (rows) return run_rows_and_shell<ORDER>(g, p, quantity, qscale, off, cnt, slots, scratch, rho, st);
    // (a v2 with thread = (X, jy) and CTA-uniform z chains measured slower:
    // QSP 6.64 vs 4.34 ms -- its 8 x-lanes per warp walk 8 cells' slot ranges;
    // removed, profiles/r02/ncu_rho_v2.txt)
    using C = DBCfg<ORDER>;
    int dev = 0;
    PICGPU_CUDA_TRY(cudaGetDevice(&dev));
    static int configured_dev = -1;
    if (configured_dev != dev) {  // per device (one process may drive several GPUs)
        PICGPU_CUDA_TRY(cudaFuncSetAttribute(density_blocks<ORDER, false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
        PICGPU_CUDA_TRY(cudaFuncSetAttribute(density_blocks<ORDER, true>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
        configured_dev = dev;
    }
    const dim3 grid(div_up(g.nx, C::RX), div_up(g.ny, C::RY), div_up(g.nz, C::ZL));
    if (g.pow2x && g.pow2y && g.pow2z)
        density_blocks<ORDER, true><<<grid, C::NT, C::SMEM, st>>>(g, p, quantity, qscale, off, cnt, rho);
    else
        density_blocks<ORDER, false><<<grid, C::NT, C::SMEM, st>>>(g, p, quantity, qscale, off, cnt, rho);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

// The previous path (PICGPU_RHO_ROWS=1): interior row kernel + prologue-based shell gather.
template <int ORDER>
void run_rows_and_shell(const GridD& g, const CAos& p, const double* quantity, double qscale, const uint32_t* off,
                        const uint32_t* cnt, uint64_t slots, void* scratch, double* rho, cudaStream_t st) {
    const Interior in = interior_of<ORDER>(g);
    Interior skip = in;
    if (!in.empty()) {
        const int zlen = PICGPU_RHO_ZLEN;
        const dim3 grid(div_up(in.hi[0] - in.lo[0] + 1, kRowX), div_up(in.hi[1] - in.lo[1] + 1, kRowY),
                        div_up(in.hi[2] - in.lo[2] + 1, zlen));
        constexpr size_t smem = (size_t)(1 + 3 * Shape<ORDER>::W) * kRowCap * 8 + (size_t)kRowCap * 5;
        static int configured_dev = -1;
        int dev = 0;
        PICGPU_CUDA_TRY(cudaGetDevice(&dev));
        if (configured_dev != dev) {  // per device (one process may drive several GPUs)
            PICGPU_CUDA_TRY(cudaFuncSetAttribute(density_rows<ORDER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem));
            configured_dev = dev;
        }
        density_rows<ORDER><<<grid, kRowX * kRowY, smem, st>>>(g, p, quantity, qscale, off, cnt, in, zlen, rho);
        note_launch();
        PICGPU_CUDA_TRY(cudaGetLastError());
    } else {
        skip.lo[0] = 1;  // nothing is interior
        skip.hi[0] = 0;
    }
    // the boundary shell (wrapped, re-sorted sources): prologue + per-node gather
    const bool shell = in.empty() || (uint64_t)(in.hi[0] - in.lo[0] + 1) * (in.hi[1] - in.lo[1] + 1) *
                                             (in.hi[2] - in.lo[2] + 1) < g.ncells;
    if (!shell) return;
    if (ORDER == 1) {  // 8 taps per node: evaluating the weights on the fly beats a full prologue
        density_gather_shell<ORDER><<<div_up(g.ncells, 128), 128, 0, st>>>(g, p, quantity, qscale, off, cnt, rho,
                                                                           skip);
    } else {  // 64 taps per node: weights once per slot (prologue), then the shell gather
        double* S;
        uint8_t* upb;
        prologue<ORDER>(g, p, quantity, qscale, slots, scratch, st, S, upb);
        density_gather_sorted<ORDER><<<div_up(g.ncells, 128), 128, 0, st>>>(g, off, cnt, S, slots, upb, rho, skip);
    }
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

template <int ORDER>
void run_merge(const GridD& g, const CAos& p, const double* quantity, double qscale, const uint32_t* rank, const uint32_t* off,
               const uint32_t* cnt, uint64_t slots, void* scratch, double* rho, cudaStream_t st) {
    double* S;
    uint8_t* upb;
    prologue<ORDER>(g, p, quantity, qscale, slots, scratch, st, S, upb);
    density_gather_merge<ORDER><<<div_up(g.ncells, 128), 128, 0, st>>>(g, off, cnt, rank, S, slots, upb, rho);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

}  // namespace

size_t density_scratch_bytes(int order, uint64_t slots) {
    const int W = order == 1 ? 2 : 4;
    return (size_t)(3 * W + 1) * slots * sizeof(double) + slots + 16;
}

void launch_deposit_density(int order, const GridD& g, const CAos& p, const double* quantity, double qscale,
                            const uint32_t* off,
                            const uint32_t* cnt, uint64_t slots, void* scratch, double* rho, cudaStream_t st) {
    switch (order) {
        case 1: run_sorted<1>(g, p, quantity, qscale, off, cnt, slots, scratch, rho, st); break;
        case 2: run_sorted<2>(g, p, quantity, qscale, off, cnt, slots, scratch, rho, st); break;
        case 3: run_sorted<3>(g, p, quantity, qscale, off, cnt, slots, scratch, rho, st); break;
        default: throw Status{PICGPU_EINVAL, "deposit_density: shape order must be 1, 2 or 3"};
    }
}

void launch_deposit_density_merge(int order, const GridD& g, const CAos& p, const double* quantity, double qscale,
                                  const uint32_t* rank, const uint32_t* off, const uint32_t* cnt, uint64_t slots,
                                  void* scratch, double* rho, cudaStream_t st) {
    switch (order) {
        case 1: run_merge<1>(g, p, quantity, qscale, rank, off, cnt, slots, scratch, rho, st); break;
        case 2: run_merge<2>(g, p, quantity, qscale, rank, off, cnt, slots, scratch, rho, st); break;
        case 3: run_merge<3>(g, p, quantity, qscale, rank, off, cnt, slots, scratch, rho, st); break;
        default: throw Status{PICGPU_EINVAL, "deposit_density: shape order must be 1, 2 or 3"};
    }
}

}  // namespace picgpu
