// jcommon.cuh -- per-particle device helpers shared by the J kernels
// (deposit_current.cu: lane/warp DFMA kernels, movers; deposit_pencil.cu: the
// default DMMA pencil kernel): record loads, the J shape weights, the fused
// bit-exact push + move detection, and the sm_100a primitives (FP64 DMMA,
// mbarrier) the pencil kernel is built on.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.hpp"

// The fused kernels' record loads carry an L2 256-byte prefetch hint (the same hint on the J-only kernels'
// read-only loads measured no effect: profiles/r02/lane_memory_ab.txt).
#ifndef PICGPU_LD_L2HINT
#define PICGPU_LD_L2HINT 1
#endif

namespace picgpu {
namespace jdev {

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
#if PICGPU_LD_L2HINT
    if constexpr (RW) {
        // the first load of the record asks L2 for the whole 256-byte block around it on
        // a miss: the next records of the bin (the following chunks) come along
        asm volatile("ld.global.L2::256B.v2.f64 {%0, %1}, [%2];" : "=d"(a.x), "=d"(a.y) : "l"(r));
        b = r[1];
        c = r[2];
        d.w = p.p[s].w;
    } else
#endif
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
#if PICGPU_WB_SECTOR
    // the record's whole first sector (x y z vx; vx unchanged): no partial-sector write
    reinterpret_cast<double2*>(pc.A.p + s)[0] = make_double2(d.x, d.y);
    reinterpret_cast<double2*>(pc.A.p + s)[1] = make_double2(d.z, d.vx);
#else
    reinterpret_cast<double2*>(pc.A.p + s)[0] = make_double2(d.x, d.y);
    pc.A.p[s].z = d.z;
#endif
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

// A slab leaver of a fused kernel that found its CTA's mover segment full:
// exported right here -- its exchange record (x y z vx vy vz w id-bits, the
// pushed position already written back) and the hole in its old bin, as
// k_movers does for the listed ones -- instead of going through the bounded
// overflow segment, so no leaver is ever dropped.
__device__ __forceinline__ void export_leaver_now(const PushCtx& pc, uint32_t s, uint32_t b, uint32_t code) {
    const Part r = pc.A.p[s];
    const int dir = code == kLeaveLeft ? 0 : 1;
    const unsigned li = atomicAdd(&pc.ctr->nleave[dir], 1u);
    if (li < pc.lcap) {
        double* rr = pc.L + ((size_t)dir * pc.lcap + li) * 8;
        rr[0] = r.x;
        rr[1] = r.y;
        rr[2] = r.z;
        rr[3] = r.vx;
        rr[4] = r.vy;
        rr[5] = r.vz;
        rr[6] = r.w;
        rr[7] = __longlong_as_double((long long)r.id);
        push_hole(pc.A, s, b, pc.off, pc.holes, pc.hl);
        atomicAdd(&pc.ctr->moved, 1ull);
    } else {
        raise_error(&pc.ctr->err, PICGPU_ELENGTH);
    }
}

// One mover segment per CTA of a fused kernel: its size and count.
inline void set_segments(PushCtx& pc, const dim3& grid, PushCtx* used) {
    const uint64_t nseg = (uint64_t)grid.x * grid.y * grid.z;
    if (nseg > kMaxFusedCtas) throw Status{PICGPU_ELENGTH, "fused step: too many CTAs for the mover segments"};
    pc.nseg = (uint32_t)nseg;
    pc.segcap = (uint32_t)(pc.mcap / 2 / nseg);
    pc.ovcap = pc.mcap - pc.nseg * pc.segcap;
    if (used) *used = pc;
}

// D += A * B on the FP64 tensor cores, one m8n8k4 tile (mma.sync, SASS DMMA.884).
// Fragments: A[row = lane>>2][k = lane&3], B[k = lane&3][col = lane>>2],
// D[row = lane>>2][col = 2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// cp.async (LDGSTS): 16 bytes global -> shared, cached in L2 only.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// mbarrier (shared::cta) primitives.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Waits for the phase of `parity` to complete; a waiter that finds it open
// backs off with nanosleep so it does not take issue slots from working warps.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    if (mbar_try_wait(bar, parity)) return;
    unsigned ns = 32;
    while (!mbar_try_wait(bar, parity)) {
        __nanosleep(ns);
        ns = ns < 256 ? ns * 2 : 256;
    }
}

}  // namespace jdev
}  // namespace picgpu
