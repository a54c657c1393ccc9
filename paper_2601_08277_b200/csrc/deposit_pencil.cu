// deposit_pencil.cu -- the "matrix" J kernel family: one warp per cell
// pencil, the per-cell outer-product contraction on the FP64 tensor cores
// (DMMA), warp-specialised plane reduction behind an mbarrier ring.
//
// Replaces pic::deposit_scalar (proj/include/pic/deposit.hpp:62-73) and is the
// matrix-unit form of deposit_tiled (deposit.hpp:284-334): the paper's block
// outer product J_cell = sum_p (wq_p Sx_p) (x) (Sy_p (x) Sz_p) (tile.hpp:57-108,
// PAPER.md "MOPA") is issued as mma.sync m8n8k4.f64 (SASS DMMA.884):
//
//   D[(c, ix)][(slot, jy)] += sum_{p in 4 particles} A[(c, ix)][p] * B[p][(slot, jy)]
//   A[(c, ix)][p] = wq_c(p) * Sx_ix(p)          (3W rows: 12 at W = 4, 6 at W = 2)
//   B[p][(slot, jy)] = Sy_jy(p) * Sz_kz(p)      (W*W columns; kz's z-plane slot)
//
// Decomposition (B200: 148 SMs, one CTA per SM; 14 warps, so each SM
// sub-partition holds at most 4 and a thread may use 128 registers):
//  * A CTA owns a PX x PY tile of cell pencils (x-y columns) and a z-chunk.
//    Each PENCIL WARP streams its pencil's bins (cells k0 .. k1-1 in z order,
//    the sorter's cell-sorted records) in passes of 32 particles -- lane = one
//    particle, whatever the cell boundaries, so no lane idles on a light cell
//    and no pencil waits for a heavier neighbour (the old 8-pencils-per-warp
//    kernel ran every pencil as long as the fullest one).
//  * Per pass each lane runs one particle's prologue (the fused bit-exact push
//    and move detection when PM > 0, cell fractions, scaled shape weights),
//    stages its A column and B row in the warp's shared staging block, and the
//    warp contracts the pass cell by cell: 4 particles per DMMA k-step, tiles
//    (row m8, col n8) = 2 x 2 at W = 4, 1 x 1 at W = 2.  The accumulators are
//    8 doubles per lane.
//  * z window: logical plane kz of a particle in cell k sits in column block
//    slot = (kz + k - k0) mod W, so when cell k is done its lowest plane
//    (k + OFF) is final in block (k - k0) mod W: it is written to the shared
//    plane ring and zeroed (it becomes the top plane of the next cell) -- no
//    accumulator moves.
//  * Plane ring: NB slots of one emitted plane per pencil; mbarriers full[s]
//    (arrive: every pencil warp) and empty[s] (arrive: every gather warp).
//    GATHER WARPS sum the W x W overlapping pencil patches of each node and
//    flush it once: plain store when every contributing cell is in this CTA,
//    RED.ADD.F64 otherwise.  Pencil warps run up to NB planes ahead of the
//    gather and of each other; no __syncthreads inside the z loop.
//
// Roofline: the FP64 pipe is shared by DMMA and DFMA on B200
// (tools/fp64_pipes.cu: 63.6 vs 63.3 MAC/clk/SM); DMMA spends 16 MAC-slots per
// particle per tile (QSP: 256 per particle for 192 useful) but issues one
// instruction per 256 MACs: the contraction costs ~3 warp-instructions per
// particle against ~10 in the register DFMA (lane) kernel.  Measured (C2 QSP,
// J only, ncu): 1.54 ms, 24.6 warp-instructions per particle, issue 48%, DMMA
// sub-pipe 29% -- latency-bound: each pencil warp runs one serial chain
// (prologue, then 8 dependent k-steps, then the plane hand-off) at 14 warps
// per SM, where the lane kernel's 8-pencil warps have far more independent
// FMAs in flight (1.18 ms); so the lane kernel stays the default.
//
// J is compared with the reference at 1e-12 peak-normalised.
#include <algorithm>
#include <type_traits>

#include "jcommon.cuh"

namespace picgpu {

namespace {

using namespace jdev;

constexpr unsigned kFull = 0xffffffffu;

template <int ORDER>
struct PCfg {
    static constexpr int W = Shape<ORDER>::W;
    static constexpr int MT = W == 4 ? 2 : 1;   // m8 row tiles over (c, ix): 3W rows
    static constexpr int NTL = W == 4 ? 2 : 1;  // n8 column tiles over (slot, jy): W*W columns
    static constexpr int NA = 3 * W, NBF = W * W, NF = NA + NBF;
    static constexpr int PX = 4, PY = 3, NP = PX * PY;  // pencil warps
    static constexpr int NGW = 2;                        // gather warps
    static constexpr int NT = (NP + NGW) * 32;           // 14 warps: <= 4 per SM sub-partition
    static constexpr int NB = 4;                         // plane ring slots
    // staging: field f of pass position l at [f*FS + l]; FS = 36 puts the
    // fragment reads (8 rows x 4 particles per LDS.64) in distinct banks
    static constexpr int FS = 36;
    static constexpr int STAGE = NF * FS;
    // one emitted plane of every pencil: [jy][ix][c][pencil] (v3's patch layout)
    static constexpr int PSTRIDE = NP + 2;
    static constexpr int PATCH = W * W * 3 * PSTRIDE;
    // per-warp record ring: 2 passes x 4 chunks x 32 lanes x 16 bytes (cp.async,
    // chunk-major so each lane's 16-byte reads are conflict-free)
    static constexpr int RING = 2 * 4 * 32 * 2;  // doubles
    static constexpr int NODES = 3 * (PX + W - 1) * (PY + W - 1);  // nodes of one plane of the CTA
    static constexpr size_t SMEM = (size_t)(NP * (STAGE + RING) + NB * PATCH) * sizeof(double) +
                                   2 * NB * sizeof(uint64_t);
};

// Shift a W-tap array by sh in {-1, 0, +1} taps, zero-filling (mover taps in
// the old cell's window; those that fall out are k_movers').
template <int W>
__device__ __forceinline__ void shift_taps(double (&v)[W], int sh) {
    double o[W];
#pragma unroll
    for (int t = 0; t < W; ++t) {
        const double up = t >= 1 ? v[t >= 1 ? t - 1 : 0] : 0.0;
        const double dn = t + 1 < W ? v[t + 1 < W ? t + 1 : 0] : 0.0;
        o[t] = sh == 0 ? v[t] : (sh > 0 ? up : dn);
    }
#pragma unroll
    for (int t = 0; t < W; ++t) v[t] = o[t];
}

// PM: 0 = deposit only; 1 = fused push + move detection + deposit; 2 = the
// same with power-of-two spacings and lengths.  SLAB: x-slab store (leavers).
template <int ORDER, int PM, bool SLAB>
__global__ void __launch_bounds__(PCfg<ORDER>::NT, 1)
    k_pencil(const GridD g, const CAos p, const uint32_t* __restrict__ off, const uint32_t* __restrict__ cnt,
             const double q, double* __restrict__ jx, double* __restrict__ jy, double* __restrict__ jz,
             const int zlen, const PushCtx pc) {
    using C = PCfg<ORDER>;
    constexpr int W = C::W, OFF = Shape<ORDER>::OFF, PX = C::PX, PY = C::PY, NP = C::NP, FS = C::FS, NB = C::NB;
    constexpr int NA = C::NA, NBF = C::NBF, MT = C::MT, NTL = C::NTL;
    constexpr int FX = PX + W - 1, FY = PY + W - 1, NODES = C::NODES;
    // 1/6^3 (QSP) or 1/2^3 (TSC) of the scaled weights, folded into q
    const double qs = q * (ORDER == 3 ? 1.0 / 216.0 : ORDER == 2 ? 0.125 : 1.0);

    extern __shared__ __align__(16) double smem[];
    double* patch = smem + NP * (C::STAGE + C::RING);
    uint64_t* full = reinterpret_cast<uint64_t*>(patch + NB * C::PATCH);
    uint64_t* empty = full + NB;
    __shared__ unsigned s_movers;

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int i0 = blockIdx.x * PX, j0 = blockIdx.y * PY;
    const int k0 = blockIdx.z * zlen;
    const int k1 = min(k0 + zlen, g.nz);
    const int T = k1 - k0 + W - 1;  // planes emitted by this CTA
    const int pxv = min(PX, g.nx - i0), pyv = min(PY, g.ny - j0);
    const bool alias_xy = (pxv + W - 1 > g.nx) || (pyv + W - 1 > g.ny);
    const uint32_t plane_cells = (uint32_t)g.nx * (uint32_t)g.ny;
    [[maybe_unused]] const uint32_t seg = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);

    if (tid == 0) {
        for (int s = 0; s < NB; ++s) {
            mbar_init(full + s, NP);
            mbar_init(empty + s, C::NGW);
        }
        mbar_fence_init();
        s_movers = 0;
    }
    // this warp's pencil
    const int pw = wid < NP ? wid : 0;
    const int px = pw % PX, py = pw / PX;
    const int i = i0 + px, j = j0 + py;
    const bool pv = wid < NP && i < g.nx && j < g.ny;
    const uint32_t col = (uint32_t)i + (uint32_t)g.nx * (uint32_t)j;
    {
        // an entirely empty tile (vacuum) writes nothing: J was zeroed by the caller
        bool any = false;
        if (pv)
            for (int kk = k0 + lane; kk < k1; kk += 32) any |= cnt[col + plane_cells * (uint32_t)kk] != 0;
        if (!__syncthreads_or(any)) {
            if (PM != 0 && tid == 0) pc.seg_cnt[seg] = 0;
            return;
        }
    }

    if (wid >= NP) {
        // ---------------- gather warps ----------------
        // plane t: sum every node's W x W pencil contributions from ring slot
        // t mod NB, flush it once, free the slot
        constexpr int NGT = C::NGW * 32, NIT = (NODES + NGT - 1) / NGT;
        const int gt = tid - NP * 32;
        int gn_base[NIT], gn_node[NIT];
        unsigned gn_mask[NIT];
        bool gn_inner[NIT];
#pragma unroll
        for (int u = 0; u < NIT; ++u) {
            const int it = gt + u * NGT;
            gn_mask[u] = 0u;
            gn_base[u] = 0;
            gn_node[u] = 0;
            gn_inner[u] = false;
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
                            if (qy >= 0 && qy < pyv && qx >= 0 && qx < pxv) gn_mask[u] |= 1u << (dy * W + dx);
                        }
                    // patch offset of tap (jy = 0, ix = 0) from pencil (0, 0); component on top
                    gn_base[u] = (c << 28) | (c * C::PSTRIDE + uy * PX + ux);
                    gn_node[u] = wrap_index(i0 + OFF + ux, g.nx) + g.nx * wrap_index(j0 + OFF + uy, g.ny);
                    gn_inner[u] = !alias_xy && ux >= W - 1 && ux <= pxv - 1 && uy >= W - 1 && uy <= pyv - 1;
                }
            }
        }
        for (int t = 0; t < T; ++t) {
            const int s = t % NB;
            mbar_wait(full + s, (unsigned)(t / NB) & 1u);
            const double* pb = patch + s * C::PATCH;
            const int kk = k0 + t;
            const size_t zrow = (size_t)plane_cells * (size_t)wrap_index(kk + OFF, g.nz);
            const bool zc = t >= W - 1 && kk < k1;  // every cell feeding this plane is in the chunk
#pragma unroll
            for (int u = 0; u < NIT; ++u) {
                const unsigned msk = gn_mask[u];
                if (!msk) continue;
                const int c = gn_base[u] >> 28;
                const double* src = pb + (gn_base[u] & 0x0fffffff);
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
                    for (int q = 0; q < h; ++q) v[q] += v[q + h];
                const double sum = v[0];
                if (sum != 0.0) {
                    double* f = c == 0 ? jx : (c == 1 ? jy : jz);
                    const size_t node = (size_t)gn_node[u] + zrow;
                    if (zc && gn_inner[u])
                        f[node] = sum;
                    else
                        atomicAdd(f + node, sum);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
        }
    } else {
        // ---------------- pencil warps ----------------
        const int gq = lane >> 2, tq = lane & 3;  // DMMA fragment coordinates
        double* S = smem + pw * C::STAGE;
        double* ring = smem + NP * C::STAGE + pw * C::RING;
        double D[MT][NTL][2];
#pragma unroll
        for (int a = 0; a < MT; ++a)
#pragma unroll
            for (int b = 0; b < NTL; ++b) D[a][b][0] = D[a][b][1] = 0.0;
        const double dci = (double)(i + g.sx_shift), dcj = (double)j;
        int t_next = 0;  // next plane step to emit

        // Emit step t: block (t mod W) holds plane k0 + t + OFF; write it to ring
        // slot t mod NB and zero it.
        // Emit step t: block (t mod W) holds plane k0 + t + OFF; write it to ring
        // slot t mod NB and zero it.
        auto emit = [&]() {
            const int t = t_next++;
            const int s = t % NB;
            if (t >= NB) mbar_wait(empty + s, (unsigned)(t / NB - 1) & 1u);
            double* P = patch + s * C::PATCH + pw;
            const int R = t & (W - 1);
            auto tile = [&](auto NTc) {
                constexpr int NT_ = decltype(NTc)::value;
                const bool mine = W == 4 ? ((tq >> 1) == (R & 1)) : (tq == R);
                if (mine) {
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int row = mt * 8 + gq;
                            const int jyv = W == 4 ? ((2 * tq + e) & 3) : e;
                            if (row < NA) P[((jyv * W + row % W) * 3 + row / W) * C::PSTRIDE] = D[mt][NT_][e];
                            D[mt][NT_][e] = 0.0;
                        }
                }
            };
            if constexpr (NTL == 2) {
                if (R >> 1)
                    tile(std::integral_constant<int, 1>{});
                else
                    tile(std::integral_constant<int, 0>{});
            } else {
                tile(std::integral_constant<int, 0>{});
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(full + s);
        };

        if (!pv) {  // a pencil outside the grid: arrive for every plane
            while (t_next < T) emit();
        } else {
            // The pencil's cells are taken 32 at a time (a WINDOW: lane j holds
            // cell kw + j's bin extent and offset).  Each cell's particles get a
            // 4-aligned run of the window's stream (inclusive scan of the rounded
            // counts), so a DMMA k-group never straddles two cells; a PASS is 32
            // consecutive stream positions, one per lane (padding lanes stage zero
            // charge).  em: cells that end after k-group gi of the pass, in byte gi;
            // em0: empty cells emitted before group 0.
            struct Pass {
                int kc;  // this lane's cell
                uint32_t ms;
                bool has;
                bool live;
                int ng, em0;
                unsigned long long em;
            };
            int kw = k0 - 32;        // window start
            uint32_t wc = 0, wo = 0;  // lane j: extent / offset of cell kw + j
            int wP = 0, wtot = 0, wX = 0, wpre = 0;
            bool wdone = false;
            auto load_window = [&](int kb) {
                kw = kb;
                const bool cell = kb + lane < k1;
                wc = cell ? cnt[col + plane_cells * (uint32_t)(kb + lane)] : 0u;
                wo = cell ? off[col + plane_cells * (uint32_t)(kb + lane)] : 0u;
                int v = (int)((wc + 3u) & ~3u);
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int u = __shfl_up_sync(kFull, v, d);
                    if (lane >= d) v += u;
                }
                wP = v;
                wtot = __shfl_sync(kFull, v, 31);
                wX = 0;
                wpre = __popc(__ballot_sync(kFull, cell && v == 0));  // leading empty cells
            };
            auto next_pass = [&](Pass& d) {
                d.live = !wdone;
                d.has = false;
                d.kc = k0;
                d.ms = 0;
                d.ng = 0;
                d.em = 0;
                d.em0 = 0;
                if (wdone) return;
                d.em0 = wX == 0 ? wpre : 0;
                const int X = wX;
                if (X < wtot) {
                    const int x = X + lane;
                    int jj = 0;  // first cell of the window whose run ends after x
#pragma unroll
                    for (int st = 16; st >= 1; st >>= 1) {
                        const int pv = __shfl_sync(kFull, wP, jj + st - 1);
                        if (pv <= x) jj += st;
                    }
                    const int jc = min(jj, 31);
                    const int pe = __shfl_sync(kFull, wP, jc);
                    const uint32_t c = __shfl_sync(kFull, wc, jc), o = __shfl_sync(kFull, wo, jc);
                    const int r = x - (pe - (int)((c + 3u) & ~3u));
                    d.has = jj < 32 && r < (int)c;
                    d.kc = kw + jc;
                    d.ms = o + (uint32_t)r;
                    d.ng = min(8, (wtot - X) >> 2);
                    // a nonempty cell (or an empty one after it) ends in this pass
                    const bool endh = kw + lane < k1 && wP > X && wP <= X + 32;
                    const int gi = (wP - X) / 4 - 1;
                    const uint32_t lo = __reduce_add_sync(kFull, endh && gi < 4 ? 1u << (8 * gi) : 0u);
                    const uint32_t hi = __reduce_add_sync(kFull, endh && gi >= 4 ? 1u << (8 * (gi - 4)) : 0u);
                    d.em = (unsigned long long)lo | ((unsigned long long)hi << 32);
                }
                wX += 32;
                if (wX >= wtot) {
                    if (kw + 32 >= k1)
                        wdone = true;
                    else
                        load_window(kw + 32);
                }
            };

            // One pass: prologue of this lane's particle (rec), staging, contraction
            // group by group, the planes of the cells that end.
            auto process = [&](const Pass& cur, const PData& rec0) {
                PData rec = rec0;
                const int kc = cur.kc;
                const uint32_t ms = cur.ms;
                const bool has = cur.has;
                const int R = (kc - k0) & (W - 1);
                double a[3][W], sy[W], sz[W];
                bool valid = has && !is_gap(rec.x);  // holes and padding lanes stage zero charge
                [[maybe_unused]] bool mv = false;
                [[maybe_unused]] int shx = 0, shy = 0, shz = 0;
                if constexpr (PM != 0) {
                    // pic::advance (workload.hpp:139-155) + Gpma::detect_moves (gpma.hpp:162-177)
                    double fx = 0.0, fy = 0.0, fz = 0.0;
                    uint32_t mv_cell = 0;
                    const uint32_t bin = col + plane_cells * (uint32_t)kc;
                    if (valid)
                        valid = push_fused<PM == 2, SLAB>(g, pc, rec, ms, bin, i, j, kc, dci, dcj, (double)kc, fx,
                                                          fy, fz, mv, mv_cell, shx, shy, shz);
                    window_from_fractions<ORDER>(rec, qs, valid, fx, fy, fz, a, sy, sz);
                    // mover list: one shared-memory reservation per warp and pass
                    const unsigned bal = __ballot_sync(kFull, mv);
                    if (bal) {
                        unsigned b0 = 0;
                        const int leader = __ffs(bal) - 1;
                        if (lane == leader) b0 = atomicAdd(&s_movers, (unsigned)__popc(bal));
                        b0 = __shfl_sync(kFull, b0, leader);
                        if (mv) {
                            const unsigned idx = b0 + (unsigned)__popc(bal & ((1u << lane) - 1u));
                            size_t e = (size_t)seg * pc.segcap + idx;
                            if (idx >= pc.segcap) {  // segment full
                                if constexpr (SLAB) {
                                    if (mv_cell >= kLeaveRight) {  // a leaver: exported here
                                        export_leaver_now(pc, ms, bin, mv_cell);
                                        e = ~(size_t)1;
                                    }
                                }
                                if (e != ~(size_t)1) {  // the shared overflow segment
                                    const unsigned o = atomicAdd(&pc.ctr->ovf_movers, 1u);
                                    e = o < pc.ovcap ? (size_t)pc.nseg * pc.segcap + o : ~(size_t)0;
                                }
                            }
                            if (e < ~(size_t)1) {
                                pc.mslot[e] = ms;
                                pc.mbin[e] = bin;
                                pc.mcellseg[e] = mv_cell;
                            }
                        }
                    }
                } else {
                    particle_window_sel<ORDER>(g, rec, qs, valid, dci, dcj, (double)kc, a, sy, sz);
                }
                // stage: A column (c, ix) and B row (slot, jy), slot = (kz + R) mod W
#pragma unroll
                for (int c = 0; c < 3; ++c)
#pragma unroll
                    for (int ix = 0; ix < W; ++ix) S[(c * W + ix) * FS + lane] = a[c][ix];
#pragma unroll
                for (int kz = 0; kz < W; ++kz) {
                    double* b = S + (NA + ((kz + R) & (W - 1)) * W) * FS + lane;
#pragma unroll
                    for (int jj = 0; jj < W; ++jj) b[jj * FS] = sy[jj] * sz[kz];
                }
                if constexpr (PM != 0) {
                    if (mv && valid) {
                        // a mover's taps, shifted into its old cell's window by its cell
                        // step; the taps that fall out are k_movers'
#pragma unroll
                        for (int f = 0; f < NA + NBF; ++f) S[f * FS + lane] = 0.0;
#pragma unroll
                        for (int c = 0; c < 3; ++c)
#pragma unroll
                            for (int ix = 0; ix < W; ++ix) {
                                const int tx = ix + shx;
                                if (tx >= 0 && tx < W) S[(c * W + tx) * FS + lane] = a[c][ix];
                            }
#pragma unroll
                        for (int kz = 0; kz < W; ++kz) {
                            const int tz = kz + shz;
                            if (tz < 0 || tz >= W) continue;
                            double* b = S + (NA + ((tz + R) & (W - 1)) * W) * FS + lane;
#pragma unroll
                            for (int jj = 0; jj < W; ++jj) {
                                const int ty = jj + shy;
                                if (ty >= 0 && ty < W) b[ty * FS] = sy[jj] * sz[kz];
                            }
                        }
                    }
                }
                __syncwarp();

                // ---- contraction: k-group gi = pass lanes 4gi .. 4gi+3, one cell ----
                for (int e = cur.em0; e; --e) emit();
#pragma unroll 1
                for (int gi = 0; gi < cur.ng; ++gi) {
                    const double* sp = S + tq + 4 * gi;
                    const double a0 = gq < NA ? sp[gq * FS] : 0.0;
                    const double a1 = MT > 1 && gq < NA - 8 ? sp[(8 + gq) * FS] : 0.0;
                    const double b0 = gq < NBF ? sp[(NA + gq) * FS] : 0.0;
                    const double b1 = NTL > 1 ? sp[(NA + 8 + gq) * FS] : 0.0;
                    dmma_8x8x4(D[0][0], a0, b0);
                    if constexpr (NTL > 1) dmma_8x8x4(D[0][NTL - 1], a0, b1);
                    if constexpr (MT > 1) {
                        dmma_8x8x4(D[MT - 1][0], a1, b0);
                        dmma_8x8x4(D[MT - 1][NTL - 1], a1, b1);
                    }
                    for (uint32_t e = (uint32_t)(cur.em >> (8 * gi)) & 255u; e; --e) emit();
                }
                __syncwarp();
            };

            // The records of a pass go HBM -> shared memory with cp.async (one
            // 64-byte record per lane as four 16-byte chunks), so the next pass's
            // loads are in flight during this one without holding registers.
            auto prefetch = [&](int buf, bool has, uint32_t ms) {
                if (has) {
                    const char* src = reinterpret_cast<const char*>(p.p + ms);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        cp_async16(ring + ((buf * 4 + k) * 32 + lane) * 2, src + 16 * k);
                }
                cp_async_commit();
            };
            auto fetch = [&](int buf, PData& d) {
                cp_async_wait_1();  // all but the most recent group (the other buffer's)
                const double2* r = reinterpret_cast<const double2*>(ring) + buf * 4 * 32 + lane;
                const double2 c0 = r[0], c1 = r[32], c2 = r[64], c3 = r[96];
                d.x = c0.x;
                d.y = c0.y;
                d.z = c1.x;
                d.vx = c1.y;
                d.vy = c2.x;
                d.vz = c2.y;
                d.w = c3.x;
            };
            // the next pass's records load (cp.async) while this one is processed
            load_window(k0);
            Pass cur, nxt;
            next_pass(cur);
            prefetch(0, cur.has, cur.ms);
            int buf = 0;
            while (cur.live) {
                next_pass(nxt);
                prefetch(buf ^ 1, nxt.has, nxt.ms);
                PData r;
                fetch(buf, r);
                process(cur, r);
                cur = nxt;
                buf ^= 1;
            }
            cp_async_wait_0();
            // the last W - 1 planes
            while (t_next < T) emit();
        }
    }
    if constexpr (PM != 0) {  // this CTA's mover count (every reservation precedes this barrier)
        __syncthreads();
        if (tid == 0) pc.seg_cnt[seg] = s_movers;
    }
}

template <int ORDER, int PM, bool SLAB>
void launch_pencil(const GridD& g, const CAos& p, const uint32_t* off, const uint32_t* cnt, double q, double* j,
                   int num_sms, cudaStream_t st, PushCtx pc, PushCtx* used) {
    using C = PCfg<ORDER>;
    constexpr int W = C::W;
    static int configured_dev = -1;
    int dev = 0;
    PICGPU_CUDA_TRY(cudaGetDevice(&dev));
    if (configured_dev != dev) {  // per device (one process may drive several GPUs)
        PICGPU_CUDA_TRY(cudaFuncSetAttribute(k_pencil<ORDER, PM, SLAB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)C::SMEM));
        configured_dev = dev;
    }
    const int tx = div_up(g.nx, C::PX), ty = div_up(g.ny, C::PY);
    // one CTA per SM: z-chunks give >= 4 waves, chunks of at least 4*W cells
    const long long tiles = (long long)tx * ty;
    const long long target = (long long)num_sms * 4;
    int zch = (int)std::max<long long>(1, (target + tiles - 1) / tiles);
    zch = std::min(zch, std::max(1, g.nz / (4 * W)));
    const int zlen = div_up(g.nz, zch);
    zch = div_up(g.nz, zlen);
    dim3 grid(tx, ty, zch);
    if constexpr (PM != 0) set_segments(pc, grid, used);
    k_pencil<ORDER, PM, SLAB><<<grid, C::NT, C::SMEM, st>>>(g, p, off, cnt, q, j, j + g.ncells,
                                                           j + 2 * (size_t)g.ncells, zlen, pc);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

template <int ORDER>
void pencil_push_order(const GridD& g, PushCtx& pc, const uint32_t* off, const uint32_t* cnt, double q, double* j,
                       int num_sms, cudaStream_t st) {
    const bool p2 = g.pow2x && g.pow2y && g.pow2z && g.gpow2Lx && g.pow2Ly && g.pow2Lz;
    const CAos p(pc.A);
    if (g.slab) {
        if (p2)
            launch_pencil<ORDER, 2, true>(g, p, off, cnt, q, j, num_sms, st, pc, &pc);
        else
            launch_pencil<ORDER, 1, true>(g, p, off, cnt, q, j, num_sms, st, pc, &pc);
    } else if (p2) {
        launch_pencil<ORDER, 2, false>(g, p, off, cnt, q, j, num_sms, st, pc, &pc);
    } else {
        launch_pencil<ORDER, 1, false>(g, p, off, cnt, q, j, num_sms, st, pc, &pc);
    }
}

}  // namespace

void launch_pencil_current(int order, const GridD& g, const CAos& p, const uint32_t* off, const uint32_t* cnt,
                           double q, double* j, int num_sms, cudaStream_t st) {
    switch (order) {
        case 1: launch_pencil<1, 0, false>(g, p, off, cnt, q, j, num_sms, st, PushCtx{}, nullptr); break;
        case 2: launch_pencil<2, 0, false>(g, p, off, cnt, q, j, num_sms, st, PushCtx{}, nullptr); break;
        case 3: launch_pencil<3, 0, false>(g, p, off, cnt, q, j, num_sms, st, PushCtx{}, nullptr); break;
        default: throw Status{PICGPU_EINVAL, "deposit: shape order must be 1, 2 or 3"};
    }
}

void launch_pencil_current_push(int order, const GridD& g, PushCtx& pc, const uint32_t* off, const uint32_t* cnt,
                                double q, double* j, int num_sms, cudaStream_t st) {
    switch (order) {
        case 1: pencil_push_order<1>(g, pc, off, cnt, q, j, num_sms, st); break;
        case 2: pencil_push_order<2>(g, pc, off, cnt, q, j, num_sms, st); break;
        case 3: pencil_push_order<3>(g, pc, off, cnt, q, j, num_sms, st); break;
        default: throw Status{PICGPU_EINVAL, "deposit: shape order must be 1, 2 or 3"};
    }
}

}  // namespace picgpu
