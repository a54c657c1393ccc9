// common.cuh -- device primitives shared by the sm_100a kernels.
//
// Everything on the parity-critical path (cell location, shape weights, push,
// rho accumulation) uses explicit round-to-nearest intrinsics (__dmul_rn,
// __dadd_rn, __dsub_rn, __ddiv_rn) so nvcc can never contract them into FMAs:
// the reference build has no FMA.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "picgpu.h"

// Write-back of a pushed position: 1 = the record's whole first sector (x y z vx,
// two 16-byte stores), 0 = x y z only (24 of the sector's 32 bytes).
#ifndef PICGPU_WB_SECTOR
#define PICGPU_WB_SECTOR 1
#endif

namespace picgpu {

// Device view of the periodic box (pic::GridSpec, grid.hpp:26-72) plus values
// precomputed on the host exactly as the reference computes them.
struct GridD {
    int nx, ny, nz;
    double dx, dy, dz;
    double ox, oy, oz;
    double Lx, Ly, Lz;        // GridSpec::length(axis) = cells * spacing (grid.hpp:46)
    double inv_dx, inv_dy, inv_dz;
    int pow2x, pow2y, pow2z;  // spacing is a power of two: (x-o)*inv == (x-o)/h exactly
    double inv_Lx, inv_Ly, inv_Lz;
    int pow2Lx, pow2Ly, pow2Lz;  // same for the box lengths (wrap_position)
    uint32_t ncells;
    // x-slab of a box decomposed over ranks; the identity for a
    // whole box.  x is always located on the GLOBAL axis (origin gox, gnx
    // cells, periodic length gLx) and shifted by sx_shift into the slab's
    // ghost-extended local grid, so every per-particle quantity (cell,
    // fraction, weights, wrapped position) is bit-identical to the
    // undecomposed run.  The slab owns local x-cells [sx_lo, sx_hi).
    int slab;
    int gnx, sx_shift, sx_lo, sx_hi;
    double gox, gLx, ginv_Lx;
    int gpow2Lx;
};

// A slot whose x holds the all-ones sentinel (a NaN no valid particle can
// carry) is empty: bin slack, or a hole left by a departed particle.
__device__ __forceinline__ bool is_gap(double x) { return __double_as_longlong(x) == -1LL; }
constexpr long long kGapBits = -1LL;

// Store-cell codes of particles that left a slab (push / import routing).
constexpr uint32_t kLeaveLeft = 0xFFFFFFFEu;
constexpr uint32_t kLeaveRight = 0xFFFFFFFDu;
constexpr uint32_t kNoCell = 0xFFFFFFFFu;  // a mover-list entry without a particle (exported leaver)

GridD make_grid(const picgpu_grid& g);

// Particle store, structure of arrays (pic::ParticleSoA, particles.hpp:14-19).
struct Soa {
    double *x, *y, *z, *vx, *vy, *vz, *w;
    uint64_t* id;
};

struct CSoa {
    const double *x, *y, *z, *vx, *vy, *vz, *w;
    const uint64_t* id;
    CSoa() = default;
    CSoa(const Soa& s) : x(s.x), y(s.y), z(s.z), vx(s.vx), vy(s.vy), vz(s.vz), w(s.w), id(s.id) {}
};

// The binned particle store is an ARRAY OF 64-BYTE RECORDS, one per slot
// (x y z vx vy vz w id: two 32-byte sectors, half a 128-byte line).  Every
// particle move of the sorter (an arrival into its new bin, a hole filled from
// a bin's tail, a relayout) then reads and writes whole sectors -- with eight
// separate arrays a scattered move touched eight sectors and made HBM
// read-modify-write seven partial ones -- and the deposits still stream
// consecutive slots of a bin.  Packed host-facing staging (uploads, downloads,
// mover records) stays structure-of-arrays (Soa).
struct __align__(64) Part {
    double x, y, z, vx, vy, vz, w;
    uint64_t id;
};
static_assert(sizeof(Part) == 64, "particle record must be 64 bytes");

struct Aos {
    Part* p;
};

struct CAos {
    const Part* p;
    CAos() = default;
    CAos(const Aos& a) : p(a.p) {}
};

// Whole-record moves (four 16-byte accesses each way).
__device__ __forceinline__ void copy_record(const Part* __restrict__ src, Part* __restrict__ dst) {
    const double2* s = reinterpret_cast<const double2*>(src);
    double2* d = reinterpret_cast<double2*>(dst);
    const double2 a = s[0], b = s[1], c = s[2], e = s[3];
    d[0] = a;
    d[1] = b;
    d[2] = c;
    d[3] = e;
}

__device__ __forceinline__ void store_record(Part* dst, double x, double y, double z, double vx, double vy,
                                             double vz, double w, uint64_t id) {
    double2* d = reinterpret_cast<double2*>(dst);
    d[0] = make_double2(x, y);
    d[1] = make_double2(z, vx);
    d[2] = make_double2(vy, vz);
    d[3] = make_double2(w, __longlong_as_double((long long)id));
}

// An empty slot: all-ones record (its x is the gap sentinel, see is_gap).
__device__ __forceinline__ void store_gap_record(Part* dst) {
    const double g = __longlong_as_double(-1LL);
    double2* d = reinterpret_cast<double2*>(dst);
    const double2 v = make_double2(g, g);
    d[0] = v;
    d[1] = v;
    d[2] = v;
    d[3] = v;
}

// Device error word: first error code wins (host reads it back once per call).
__device__ __forceinline__ void raise_error(int* err, int code) {
    if (err) atomicCAS(err, 0, code);
}

// grid.hpp:64-67
__host__ __device__ __forceinline__ int wrap_index(int i, int n) {
    int r = i % n;
    return r < 0 ? r + n : r;
}

// detail::locate_axis, grid.hpp:81-100.  Bit-identical to the reference:
// u = (x - origin) / spacing (a multiply by the exact reciprocal when the
// spacing is a power of two, which yields the same correctly rounded value).
// P2: the caller knows every spacing is a power of two (no division code at all).
template <bool P2 = false>
__device__ __forceinline__ int locate_axis(double x, double origin, double spacing, double inv, int pow2, int n,
                                           double& frac) {
    const double t = __dsub_rn(x, origin);
    const double u = (P2 || pow2) ? __dmul_rn(t, inv) : __ddiv_rn(t, spacing);
    double fu = floor(u);
    double fr = __dsub_rn(u, fu);
    if (fr >= 1.0) {
        fr = 0.0;
        fu = __dadd_rn(fu, 1.0);
    }
    frac = fr;
    if (fu >= 0.0 && fu < (double)n) return (int)fu;
    if (fabs(fu) < 2147483648.0) {  // exact integer remainder: fmod of an integral double
        const int r = (int)fu % n;
        return r < 0 ? r + n : r;
    }
    double c = fmod(fu, (double)n);
    if (c < 0.0) c = __dadd_rn(c, (double)n);
    int ci = (int)c;
    if (ci == n) ci = 0;
    return ci;
}

__device__ __forceinline__ bool finite3(double x, double y, double z) {
    return isfinite(x) && isfinite(y) && isfinite(z);
}

// Local x-cell of a position (global locate, then the slab shift).
template <bool P2 = false>
__device__ __forceinline__ int locate_x(const GridD& g, double x, double& frac) {
    return locate_axis<P2>(x, g.gox, g.dx, g.inv_dx, g.pow2x, g.gnx, frac) - g.sx_shift;
}

// cell_of, grid.hpp:106-113 (caller checks finiteness).
template <bool P2 = false>
__device__ __forceinline__ uint32_t cell_linear(const GridD& g, double x, double y, double z, int& i, int& j,
                                                int& k, double& fx, double& fy, double& fz) {
    i = locate_x<P2>(g, x, fx);
    j = locate_axis<P2>(y, g.oy, g.dy, g.inv_dy, g.pow2y, g.ny, fy);
    k = locate_axis<P2>(z, g.oz, g.dz, g.inv_dz, g.pow2z, g.nz, fz);
    return (uint32_t)i + (uint32_t)g.nx * ((uint32_t)j + (uint32_t)g.ny * (uint32_t)k);
}

__device__ __forceinline__ uint32_t cell_linear(const GridD& g, double x, double y, double z) {
    int i, j, k;
    double fx, fy, fz;
    return cell_linear(g, x, y, z, i, j, k, fx, fy, fz);
}

// Bin of a particle in a session store: its cell, or kLeaveLeft/kLeaveRight
// when a slab does not own it (the nearer neighbour on the periodic x-axis).
template <bool P2 = false>
__device__ __forceinline__ uint32_t store_cell(const GridD& g, double x, double y, double z) {
    int i, j, k;
    double fx, fy, fz;
    const uint32_t c = cell_linear<P2>(g, x, y, z, i, j, k, fx, fy, fz);
    if (!g.slab || (i >= g.sx_lo && i < g.sx_hi)) return c;
    const int ig = i + g.sx_shift, x0 = g.sx_lo + g.sx_shift, x1 = g.sx_hi + g.sx_shift;
    const int dl = ((x0 - ig) % g.gnx + g.gnx) % g.gnx;
    const int dr = ((ig - x1 + 1) % g.gnx + g.gnx) % g.gnx;
    return dl <= dr ? kLeaveLeft : kLeaveRight;
}

// Device counters of one step (read back once per step).
struct StepCounters {
    unsigned long long moved;
    unsigned int nmovers;     // movers detected (may exceed mover capacity)
    unsigned int noverflow;   // arrivals that found no slack in their own bin
    int err;                  // picgpu_status of the first device-side error
    unsigned int nborrowed;   // ... placed by borrowing a following bin's slack
    unsigned int nleft;       // ... with no donor (-> rebuild)
    unsigned int nimport;     // arrivals from neighbour slabs appended to the movers
    unsigned int nleave[2];   // particles that left the slab to the left / right
    // fused step: movers beyond their CTA's segment go to the shared overflow
    // segment (ovf_movers, global atomic); beyond that they are dropped (-> full re-sort)
    unsigned int ovf_movers;
    unsigned int mover_drop;
    // device-resident slab exchange (picgpu_session_slab_step)
    unsigned int import_left;  // arrivals from the left (the right ones follow them)
    unsigned int ovf_import;   // bit 0/1: the left/right neighbour sent more than the bucket
};

// floor((x - o) / h) exactly as locate_axis computes it (before its range
// handling).  For u >= 0 the fraction u - floor(u) is exact and < 1, so equal
// non-negative floors on every axis mean the same cell.
__device__ __forceinline__ double axis_floor(double x, double o, double h, double inv, int pow2) {
    const double t = __dsub_rn(x, o);
    return floor(pow2 ? __dmul_rn(t, inv) : __ddiv_rn(t, h));
}

// detail::wrap_position, workload.hpp:128-132 (a power-of-two length divides
// exactly as a multiply by its reciprocal).
__device__ __forceinline__ double wrap_position(double x, double origin, double length, double inv, int pow2) {
    const double t = __dsub_rn(x, origin);
    double r = __dsub_rn(x, __dmul_rn(length, floor(pow2 ? __dmul_rn(t, inv) : __ddiv_rn(t, length))));
    if (__dsub_rn(r, origin) >= length) r = origin;
    return r;
}

// One particle of pic::advance (workload.hpp:144-153); returns false on a cap
// violation (the reference throws std::domain_error).
// P2: every spacing and box length is a power of two (checked on the host),
// so the divide-or-multiply choice folds away at compile time.
template <bool P2 = false>
__device__ __forceinline__ bool push_one(const GridD& g, double dt, double cap2, double& x, double& y, double& z,
                                         double vx, double vy, double vz) {
    const double v2 = __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
    if (v2 > cap2) return false;
    x = wrap_position(__dadd_rn(x, __dmul_rn(vx, dt)), g.gox, g.gLx, g.ginv_Lx, P2 || g.gpow2Lx);
    y = wrap_position(__dadd_rn(y, __dmul_rn(vy, dt)), g.oy, g.Ly, g.inv_Ly, P2 || g.pow2Ly);
    z = wrap_position(__dadd_rn(z, __dmul_rn(vz, dt)), g.oz, g.Lz, g.inv_Lz, P2 || g.pow2Lz);
    return true;
}

// A departure: the slot becomes a hole of its bin (sentinel x) and joins the
// bin's hole list.
__device__ __forceinline__ void push_hole(const Aos& A, uint64_t s, uint32_t b, const uint32_t* __restrict__ off,
                                          uint32_t* __restrict__ holes, uint32_t* __restrict__ hl) {
    store_gap_record(A.p + s);  // whole record: two full sectors, no partial-sector write
    hl[off[b] + atomicAdd(&holes[b], 1u)] = (uint32_t)s;
}

// Shape weights in a fixed window of W taps starting at node cell + OFF.
//   order 1: CIC, cic_shape_1d (shape.hpp:26-29), W = 2, OFF = 0.
//   order 3: QSP, qsp_shape_1d (shape.hpp:33-43), W = 4, OFF = -1.
//   order 2: TSC (this project's restatement, oracle/picoracle.c po_shape_1d):
//            3 taps from base cell-1+up, padded into a W = 4 window at OFF = -1;
//            `up` (d >= 0.5) says which end of the window holds the zero.
// Expression order matches the reference exactly (bit-identical weights).
template <int ORDER>
struct Shape;

template <>
struct Shape<1> {
    static constexpr int W = 2, OFF = 0, TAPS = 2;
    __device__ __forceinline__ static void weights(double d, double (&s)[W], int& up) {
        s[0] = __dsub_rn(1.0, d);
        s[1] = d;
        up = 0;
    }
};

template <>
struct Shape<3> {
    static constexpr int W = 4, OFF = -1, TAPS = 4;
    __device__ __forceinline__ static void weights(double d, double (&s)[W], int& up) {
        const double t = d;
        const double t2 = __dmul_rn(t, t);
        const double t3 = __dmul_rn(t2, t);
        const double u = __dsub_rn(1.0, t);
        const double k6 = 1.0 / 6.0;
        s[0] = __dmul_rn(__dmul_rn(__dmul_rn(u, u), u), k6);
        s[1] = __dmul_rn(__dadd_rn(__dsub_rn(__dmul_rn(3.0, t3), __dmul_rn(6.0, t2)), 4.0), k6);
        s[2] = __dmul_rn(
            __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(-3.0, t3), __dmul_rn(3.0, t2)), __dmul_rn(3.0, t)), 1.0), k6);
        s[3] = __dmul_rn(t3, k6);
        up = 0;
    }
};

template <>
struct Shape<2> {
    static constexpr int W = 4, OFF = -1, TAPS = 3;
    // Unpadded 3 taps (base = cell - 1 + up).
    __device__ __forceinline__ static void taps(double d, double (&w)[3], int& up) {
        up = d >= 0.5;
        const double dl = up ? __dsub_rn(d, 1.0) : d;
        const double a = __dsub_rn(0.5, dl);
        const double b = __dadd_rn(0.5, dl);
        w[0] = __dmul_rn(0.5, __dmul_rn(a, a));
        w[1] = __dsub_rn(0.75, __dmul_rn(dl, dl));
        w[2] = __dmul_rn(0.5, __dmul_rn(b, b));
    }
    __device__ __forceinline__ static void weights(double d, double (&s)[W], int& up) {
        double w[3];
        taps(d, w, up);
        s[0] = up ? 0.0 : w[0];
        s[1] = up ? w[0] : w[1];
        s[2] = up ? w[1] : w[2];
        s[3] = up ? w[2] : 0.0;
    }
};

// Launch bookkeeping: every kernel launch of this library bumps the counter
// reported by picgpu_kernel_launches() (evidence that the native path ran).
void note_launch(uint64_t n = 1);

#define PICGPU_CUDA_TRY(expr)                                              \
    do {                                                                   \
        cudaError_t e__ = (expr);                                          \
        if (e__ != cudaSuccess) throw ::picgpu::CudaError(e__, #expr);     \
    } while (0)

struct CudaError {
    cudaError_t code;
    const char* what;
    CudaError(cudaError_t c, const char* w) : code(c), what(w) {}
};

struct Status {  // thrown inside the library, converted to a return code at the C boundary
    int code;
    const char* msg;
};

inline int div_up(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace picgpu
