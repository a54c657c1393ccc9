// deposit_current.cu -- the register-blocked DFMA J kernels (the default
// "lane" family and the "vector" family; the "matrix" family is the DMMA
// pencil kernel in deposit_pencil.cu), the movers' kernel of the fused step
// and the slab arrivals' deposit.  J = sum_p q W_p v_p S(x_i - x_p) at shape orders 1 (CIC),
// 2 (TSC, padded into a 4-tap window) and 3 (QSP).
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

#include "jcommon.cuh"

namespace picgpu {

namespace {

using namespace jdev;

// z-chunks of the lane kernel: enough CTAs for this many waves on every SM.  C2 fused
// kernel, 2 / 4 / 6 / 8 waves: QSP 1.664 / 1.554 / 1.546 / 1.559 ms, CIC 1.415 / 1.252 /
// 1.224 / 1.225, TSC 1.809 / 1.673 / 1.657 / 1.673 (profiles/r02/lane_memory_ab.txt)
#ifndef PICGPU_ZCH_WAVES
#define PICGPU_ZCH_WAVES 6
#endif

// Record prefetch of the lane kernel: 1 = after the window is staged, into the
// record's own registers (no copy, 14 fewer registers live; the fused kernels
// do not spill); 0 = before the prologue into a second record of registers.
// C2 fused kernel: QSP 1.612 vs 1.617 ms, CIC 1.352 vs 1.403; TSC alone was
// 1.703 vs 1.669, but with the L2 prefetch of the next cell 1.603 vs 1.656 (no
// spills) -- so every order prefetches late (profiles/r02/lane_memory_ab.txt).
#ifndef PICGPU_LATE_PREFETCH
#define PICGPU_LATE_PREFETCH 1
#endif
// L2 prefetch of the next cell's records one cell step ahead (prefetch.global.L2),
// fused QSP and TSC kernels.  C2 fused kernel: QSP 1.612 -> 1.568 ms, TSC (with the
// late record prefetch) 1.656 -> 1.603; CIC 1.356 -> 1.402 (1.225 -> 1.337 at 5 CTAs/SM) and the J-only QSP kernel
// 1.132 -> 1.187 (slower: left off) -- profiles/r02/lane_memory_ab.txt.
#ifndef PICGPU_L2_PREFETCH
#define PICGPU_L2_PREFETCH 1
#endif

template <int ORDER>
struct JCfg;
// CIC on the v3 kernel: 2 lanes per pencil (lane = jy), 12 accumulators each.
#ifndef PICGPU_CIC_PX
#define PICGPU_CIC_PX 16
#endif
#ifndef PICGPU_CIC_PY
#define PICGPU_CIC_PY 4
#endif
// 5 CTAs/SM (96 registers, no spills): the CIC pass is bound by the latency of its
// record loads, so warps count -- C2 fused 1.308 -> 1.252 ms, J only 0.632 -> 0.599;
// 6 (80 registers, spills) 1.230 but C1 0.089 -> 0.096 (profiles/r02/lane_memory_ab.txt)
#ifndef PICGPU_CIC_MINB
#define PICGPU_CIC_MINB 5
#endif
// (A per-lane cp.async record ring instead of the one-record register
// prefetch measured slower -- CIC fused 1.466 vs 1.403 ms, QSP 1.751 vs 1.615:
// fewer long-scoreboard stalls, more shared-memory pressure; removed,
// profiles/r02/ncu_fused_cic_ring.txt.)
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
    static constexpr size_t SMEM3 = (size_t)(2 * PPB * PATCH + STAGE3) * sizeof(double);
};




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
    // tiles cover x-cells [xb, xe): a slab's owned cells (its ghost cells hold no particles)
    const int xb = g.slab ? g.sx_lo : 0, xe = g.slab ? g.sx_hi : g.nx;
    const int i0 = xb + blockIdx.x * PX, j0 = blockIdx.y * PY;
    const int k0 = blockIdx.z * zlen;
    const int k1 = min(k0 + zlen, g.nz);
    const int i = i0 + px, j = j0 + py;
    const bool pv = (i < xe) && (j < g.ny);
    const int pxv = min(PX, xe - i0), pyv = min(PY, g.ny - j0);
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
            // empty cells: still prefetch -- behind a (warp-uniform) branch, so that the
            // next bin's count, just requested, is not waited for at every cell step
            if (m == 0) {
                asm volatile("" ::: "memory");
                if (lg < n_n) load_particle<PM != 0>(p, n_off + lg, nxt);
            }
            for (int base = 0; base < m; base += CH) {
                [[maybe_unused]] bool mv = false;  // fused step: this lane's particle changed cell
                [[maybe_unused]] uint32_t mv_cell = 0;
                [[maybe_unused]] unsigned mv_bal = 0, mv_b0 = 0;
                {
                    // LATE: the record is used in place and its registers take the
                    // next record once the window is staged (the load has the whole
                    // contraction to land): no copy, one record of registers
                    constexpr bool LATE = PICGPU_LATE_PREFETCH;
                    PData early;
                    if constexpr (!LATE) early = nxt;
                    PData& cur = LATE ? nxt : early;
                    bool valid = base + lg < n_c && !is_gap(cur.x);  // holes count as padding
                    auto prefetch = [&] {
                        if (base + CH < m) {
                            if (base + CH + lg < n_c) load_particle<PM != 0>(p, c_off + base + CH + lg, nxt);
                        } else if (lg < n_n) {
                            load_particle<PM != 0>(p, n_off + lg, nxt);
                        }
                    };
                    if constexpr (!LATE) prefetch();
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
                    if constexpr (LATE) prefetch();
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
                            if (idx >= pc.segcap) {  // segment full
                                if constexpr (SLAB) {
                                    if (mv_cell >= kLeaveRight) {  // a leaver: exported here
                                        export_leaver_now(pc, c_off + (uint32_t)(base + lg),
                                                          col + plane_cells * (uint32_t)k, mv_cell);
                                        e = ~(size_t)1;
                                    }
                                }
                                if (e != ~(size_t)1) {  // the shared overflow segment
                                    const unsigned o = atomicAdd(&pc.ctr->ovf_movers, 1u);
                                    e = o < pc.ovcap ? (size_t)pc.nseg * pc.segcap + o : ~(size_t)0;
                                }
                            }
                            if (e < ~(size_t)1) {
                                pc.mslot[e] = c_off + (uint32_t)(base + lg);
                                pc.mbin[e] = col + plane_cells * (uint32_t)k;
                                pc.mcellseg[e] = mv_cell;
                            }
                        }
                    }
                }
                __syncwarp();
                // After the cell's first chunk (the next bin's offset and count,
                // loaded at the top of the step, have landed): the next cell's
                // records are prefetched into L2, one 128-byte line per request, the
                // pencil's G lanes interleaved -- the rest of this cell's chunks to land.
                if constexpr (PICGPU_L2_PREFETCH && ORDER >= 2 && PM != 0) {
                    if (base == 0) {
                        const char* pb = reinterpret_cast<const char*>(p.p + n_off);
                        for (int b = lg * 128; b < n_n * 64 + 64; b += G * 128)
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(pb + b));
                    }
                }
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

template <int ORDER>
void launch_warp(const GridD& g, const CAos& p, const uint32_t* off, const uint32_t* cnt, double q, double* j,
                 int num_sms, cudaStream_t st) {
    static int configured_dev = -1;
    int dev = 0;
    PICGPU_CUDA_TRY(cudaGetDevice(&dev));
    if (configured_dev != dev) {  // per device (one process may drive several GPUs)
        PICGPU_CUDA_TRY(cudaFuncSetAttribute(deposit_current_warp_kernel<ORDER>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WCfg::SMEM));
        configured_dev = dev;
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

// z-chunked grid of the lane kernel (v3); PM > 0: its fused push + detect +
// deposit form.
template <int ORDER, class C, int PM = 0, bool SLAB = false>
void launch_kernel(const GridD& g, const CAos& p, const uint32_t* off, const uint32_t* cnt, double q, double* j,
                   int num_sms, cudaStream_t st, PushCtx pc = PushCtx{}, PushCtx* used = nullptr) {
    using L = JLayout<ORDER, C>;
    constexpr int W = L::W;
    constexpr size_t smem = L::SMEM3;
    static int configured_dev = -1;
    int dev = 0;
    PICGPU_CUDA_TRY(cudaGetDevice(&dev));
    if (configured_dev != dev) {  // per device (one process may drive several GPUs)
        PICGPU_CUDA_TRY(cudaFuncSetAttribute(deposit_current_kernel_v3<ORDER, C, PM, SLAB>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured_dev = dev;
    }
    const int tx = div_up(g.slab ? g.sx_hi - g.sx_lo : g.nx, C::PX), ty = div_up(g.ny, C::PY);
    // z-chunks: enough CTAs for several waves on every SM, but chunks of at
    // least 4*W cells so most planes are complete (plain stores, no RED).
    const long long tiles = (long long)tx * ty;
    const long long target = (long long)num_sms * C::MINB * PICGPU_ZCH_WAVES;
    int zch = (int)std::max<long long>(1, (target + tiles - 1) / tiles);
    zch = std::min(zch, std::max(1, g.nz / (4 * W)));
    const int zlen = div_up(g.nz, zch);
    zch = div_up(g.nz, zlen);
    dim3 grid(tx, ty, zch);
    if constexpr (PM != 0) set_segments(pc, grid, used);
    deposit_current_kernel_v3<ORDER, C, PM, SLAB><<<grid, L::NT, smem, st>>>(g, p, off, cnt, q, j, j + g.ncells,
                                                                            j + 2 * (size_t)g.ncells, zlen, pc);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

// The lane family's kernel.  (A warp-specialised form -- producer warps for the
// push + prologue feeding consumer warps through an mbarrier ring, setmaxnreg
// split -- was measured and removed: C2 QSP fused 1.63 vs 1.61 ms, J only 1.31
// vs 1.18; the producers' dependent FP64 chains cannot feed the consumers,
// profiles/r02/ncu_fused_ws.txt, ncu_fused_ws2.txt.)
template <int ORDER, class C, int PM = 0, bool SLAB = false>
void launch_lane(const GridD& g, const CAos& p, const uint32_t* off, const uint32_t* cnt, double q, double* j,
                 int num_sms, cudaStream_t st, PushCtx pc = PushCtx{}, PushCtx* used = nullptr) {
    launch_kernel<ORDER, C, PM, SLAB>(g, p, off, cnt, q, j, num_sms, st, pc, used);
}

template <int ORDER>
using LaneCfg = std::conditional_t<ORDER == 1, JCfgCic3, JCfg<ORDER>>;

}  // namespace

// Kernel family of a call: an explicit family, else PICGPU_J_VARIANT
// (profiling / ablation: "dmma", "dfma"), else the register-lane DFMA kernel.
// C2 QSP, J only (B200): lane 1.18 ms, DMMA pencil 1.54 ms, warp DFMA 1.8-2.7 ms.
static int resolve_family(int kernel) {
    if (kernel != kJDefault) return kernel;
    static const int v = [] {
        const char* e = std::getenv("PICGPU_J_VARIANT");
        if (!e) return (int)kJLane;
        const std::string s(e);
        return s == "dmma" ? (int)kJMatrix : s == "dfma" ? (int)kJVector : (int)kJLane;
    }();
    return v;
}

// J must be zeroed by the caller (halo nodes are reduced into it).
void launch_deposit_current(int order, const GridD& g, const CAos& p, const uint32_t* off, const uint32_t* cnt,
                            double q, double* j, int num_sms, cudaStream_t st, int kernel) {
    if (order < 1 || order > 3) throw Status{PICGPU_EINVAL, "deposit: shape order must be 1, 2 or 3"};
    const int k = resolve_family(kernel);
    if (k == kJMatrix) return launch_pencil_current(order, g, p, off, cnt, q, j, num_sms, st);
    switch (order) {
        case 1: launch_lane<1, LaneCfg<1>>(g, p, off, cnt, q, j, num_sms, st); break;
        case 2:
            if (k == kJVector) launch_warp<2>(g, p, off, cnt, q, j, num_sms, st);
            else launch_lane<2, LaneCfg<2>>(g, p, off, cnt, q, j, num_sms, st);
            break;
        default:
            if (k == kJVector) launch_warp<3>(g, p, off, cnt, q, j, num_sms, st);
            else launch_lane<3, LaneCfg<3>>(g, p, off, cnt, q, j, num_sms, st);
            break;
    }
}

namespace {

template <int ORDER>
void launch_push_order(const GridD& g, PushCtx& pc, const uint32_t* off, const uint32_t* cnt, double q,
                       double* j, int num_sms, cudaStream_t st) {
    using C3 = LaneCfg<ORDER>;
    const bool p2 = g.pow2x && g.pow2y && g.pow2z && g.gpow2Lx && g.pow2Ly && g.pow2Lz;
    const CAos p(pc.A);
    if (g.slab) {
        if (p2)
            launch_kernel<ORDER, C3, 2, true>(g, p, off, cnt, q, j, num_sms, st, pc, &pc);
        else
            launch_kernel<ORDER, C3, 1, true>(g, p, off, cnt, q, j, num_sms, st, pc, &pc);
    } else if (p2) {
        launch_lane<ORDER, C3, 2>(g, p, off, cnt, q, j, num_sms, st, pc, &pc);
    } else {
        launch_lane<ORDER, C3, 1>(g, p, off, cnt, q, j, num_sms, st, pc, &pc);
    }
}

// Node index on a periodic axis for i within a window of [0, n): the common
// case without the integer modulo.
__device__ __forceinline__ int wrap_near(int i, int n) {
    return (unsigned)i < (unsigned)n ? i : wrap_index(i, n);
}

// One mover's deposit descriptor (shared memory): its scaled window weights,
// charge x velocity, wrapped node indices per axis and packed cell steps.
template <int W>
struct MoverDesc {
    double sx[W], sy[W], sz[W], wq[3];
    int X[W], Y[W], Z[W];
    int sh;  // (shx + 1) | (shy + 1) << 2 | (shz + 1) << 4; -1: nothing to deposit (a slab leaver)
    int pad;
};

// Movers of the fused step, one CTA per mover segment (= per CTA of the fused
// kernel; the shared overflow segment is split over the CTAs past the last
// segment), in batches of MB movers and two phases:
//  1. one thread per mover copies the particle from its slot into the mover
//     record (k_insert's input), turns the slot into a hole of its old bin
//     (delete_in_bin, gpma.hpp:328-335) and writes the mover's window (cell,
//     weights, wrapped node indices, cell steps) as a descriptor -- the
//     records' dependent loads of a whole batch are in flight together;
//  2. W*W threads per mover, one (ix, jy) column of its window each, reduce the
//     taps the fused kernel could NOT deposit into J (RED.ADD.F64): the fused
//     kernel deposited the taps inside the old cell's window (a mover steps at
//     most one cell per axis), the rest -- 16 of 64 nodes for a one-axis QSP
//     mover -- lie outside it.
// A slab leaver becomes an exchange record for the neighbour, no deposit.
// A segment's movers take a block of the compact mover list (any order of
// blocks: the list is a set, as the reference's pending moves are applied one
// by one).
// Measured at C2 (movers + insert + borrow): 0.210 ms; the first form (W threads
// per mover, each repeating the window evaluation and testing 16 taps: 161
// warp-instructions per mover) 0.239; this kernel flat over a compact entry
// list that the fused CTAs fill at their ends 0.217 plus 0.03 ms in the fused
// kernel; the movers processed in the fused kernel's own tail: fused kernel
// +0.20 ms (profiles/r02/kmovers_ab.txt).  With the REDs removed the phase
// drops by 0.05 ms: the rest is the latency of the dependent entry -> record
// loads and the hole-list atomics.
#ifndef PICGPU_MOVERS_MB
#define PICGPU_MOVERS_MB 128
#endif
#ifndef PICGPU_MOVERS_NT
#define PICGPU_MOVERS_NT 256
#endif
template <int ORDER, bool P2>
__global__ void __launch_bounds__(PICGPU_MOVERS_NT) k_movers(const GridD g, const PushCtx pc, const Soa M,
                                                const uint32_t* __restrict__ off, uint32_t* __restrict__ holes,
                                                uint32_t* __restrict__ hl, const double qs, double* __restrict__ jx,
                                                double* __restrict__ jy, double* __restrict__ jz) {
    constexpr int W = Shape<ORDER>::W, OFF = Shape<ORDER>::OFF;
    constexpr int MB = PICGPU_MOVERS_MB;  // movers per batch
    constexpr int LPM = W * W;  // deposit threads per mover
    __shared__ MoverDesc<W> s_d[MB];
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
    for (uint32_t batch = 0; batch < nm; batch += MB) {
        const uint32_t nb = min((uint32_t)MB, nm - batch);
        if (threadIdx.x < nb) {
            MoverDesc<W>& d = s_d[threadIdx.x];
            const uint32_t local = batch + threadIdx.x;
            const uint64_t i = (uint64_t)s_base + local;  // compact index
            const size_t e = (size_t)sg * pc.segcap + s_first + local;
            const uint32_t s = pc.mslot[e], b = pc.mbin[e];
            const uint32_t mc = pc.mcellseg[e];
            const double2* rec = reinterpret_cast<const double2*>(pc.A.p + s);
            const double2 r0 = rec[0], r1 = rec[1], r2 = rec[2], r3 = rec[3];
            const double x = r0.x, y = r0.y, z = r1.x, vx = r1.y, vy = r2.x, vz = r2.y, w = r3.x;
            if (mc >= kLeaveRight) {  // left the slab: an exchange record for the neighbour
                d.sh = -1;
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
            } else {
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
                int ci, cj, ck;
                double fx, fy, fz;
                cell_linear<P2>(g, x, y, z, ci, cj, ck, fx, fy, fz);
                const uint32_t bi = b % (uint32_t)g.nx, bj = (b / (uint32_t)g.nx) % (uint32_t)g.ny,
                               bk = b / ((uint32_t)g.nx * (uint32_t)g.ny);
                const int shx = cell_step(ci - (int)bi, g.gnx), shy = cell_step(cj - (int)bj, g.ny),
                          shz = cell_step(ck - (int)bk, g.nz);
                d.sh = (shx + 1) | ((shy + 1) << 2) | ((shz + 1) << 4);
                weights_scaled<ORDER>(fx, d.sx);
                weights_scaled<ORDER>(fy, d.sy);
                weights_scaled<ORDER>(fz, d.sz);
                const double qw = qs * w;
                d.wq[0] = qw * vx;
                d.wq[1] = qw * vy;
                d.wq[2] = qw * vz;
#pragma unroll
                for (int t = 0; t < W; ++t) {
                    d.X[t] = wrap_near(ci + OFF + t, g.nx);
                    d.Y[t] = wrap_near(cj + OFF + t, g.ny);
                    d.Z[t] = wrap_near(ck + OFF + t, g.nz);
                }
            }
        }
        __syncthreads();
        for (uint32_t t = threadIdx.x; t < nb * LPM; t += blockDim.x) {
            const MoverDesc<W>& d = s_d[t / LPM];
            const int sh = d.sh;
            if (sh < 0) continue;
            const int l = (int)(t % LPM), ix = l % W, jj = l / W;
            const int shx = (sh & 3) - 1, shy = ((sh >> 2) & 3) - 1, shz = ((sh >> 4) & 3) - 1;
            const bool xyin = ix + shx >= 0 && ix + shx < W && jj + shy >= 0 && jj + shy < W;
            const double sxv = d.sx[ix], syv = d.sy[jj];
            const double wq0 = d.wq[0], wq1 = d.wq[1], wq2 = d.wq[2];
            const size_t X = (size_t)d.X[ix], Y = (size_t)d.Y[jj];
#pragma unroll
            for (int kz = 0; kz < W; ++kz) {
                if (xyin && kz + shz >= 0 && kz + shz < W) continue;  // deposited by the fused kernel
                const double v = sxv * (syv * d.sz[kz]);
                if (v == 0.0) continue;
                const size_t node = (Y + (size_t)g.ny * (size_t)d.Z[kz]) * (size_t)g.nx + X;
                atomicAdd(jx + node, wq0 * v);
                atomicAdd(jy + node, wq1 * v);
                atomicAdd(jz + node, wq2 * v);
            }
        }
        __syncthreads();
    }
}

}  // namespace

bool fused_step_available(int order, int kernel) {
    (void)order;
    const int k = resolve_family(kernel);
    return k == kJMatrix || k == kJLane;
}

void launch_deposit_current_push(int order, const GridD& g, PushCtx& pc, const uint32_t* off,
                                 const uint32_t* cnt, double q, double* j, int num_sms, cudaStream_t st,
                                 int kernel) {
    if (order < 1 || order > 3) throw Status{PICGPU_EINVAL, "deposit: shape order must be 1, 2 or 3"};
    if (resolve_family(kernel) == kJMatrix) return launch_pencil_current_push(order, g, pc, off, cnt, q, j, num_sms, st);
    switch (order) {
        case 1: launch_push_order<1>(g, pc, off, cnt, q, j, num_sms, st); break;
        case 2: launch_push_order<2>(g, pc, off, cnt, q, j, num_sms, st); break;
        default: launch_push_order<3>(g, pc, off, cnt, q, j, num_sms, st); break;
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
    if (base == kBaseFromCounters) base = ctr->nmovers;  // device-resident exchange: base set by k_import_plan
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
    const bool p2 = g.pow2x && g.pow2y && g.pow2z;
    auto* kern = order == 1   ? (p2 ? k_movers<1, true> : k_movers<1, false>)
                 : order == 2 ? (p2 ? k_movers<2, true> : k_movers<2, false>)
                              : (p2 ? k_movers<3, true> : k_movers<3, false>);
    kern<<<pc.nseg + (uint32_t)num_sms * 4, PICGPU_MOVERS_NT, 0, st>>>(g, pc, M, off, holes, hl, qs, j, j + g.ncells,
                                                         j + 2 * (size_t)g.ncells);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

}  // namespace picgpu
