// sorter.cu -- the GPU cell sorter (bins with slack, incremental migration,
// full stable re-sort), the bit-exact push and the device plasma generator.
//
// Reference anchors (proj/include/pic/):
//   gpma_build          gpma.hpp:379-402  -> BinStore::full_sort_from_B (stable radix sort by cell,
//                                            radix_sort.cu)
//   Gpma::layout        gpma.hpp:269-302  -> k_counts_caps + scan (same capacity rule)
//   detect_moves        gpma.hpp:162-177  -> k_push + k_departures (unfused step: departures leave
//                                            holes), or the fused J pass + k_movers (deposit_current.cu)
//   apply_moves/insert  gpma.hpp:110-125, :248-262 -> k_insert (a hole of the bin, else its slack)
//   borrow_insert       gpma.hpp:337-370  -> k_borrow (next 4 bins), else the rebuild below
//   rebuild             gpma.hpp:130-143  -> BinStore::finish_incremental (relayout with fresh slack)
//   global_sort         sort_policy.hpp:83-85 -> BinStore::relayout
//   advance             workload.hpp:128-155 -> push_one (round-to-nearest intrinsics, bit-identical)
// The store is an array of 64-byte particle records (common.cuh, Part).
#include <type_traits>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <utility>

#include "kernels.hpp"
#include "store.hpp"

namespace picgpu {

// ---------------------------------------------------------------------------
// buffers

DevBuf::~DevBuf() { release(); }

void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}

void DevBuf::ensure(size_t b) {
    if (b <= bytes) return;
    // regrowth keeps 12.5% headroom: a store whose capacity creeps up after
    // rebuilds must not pay cudaFree/cudaMalloc (device-synchronising) each time
    const size_t grown = bytes ? b + b / 8 : b;
    release();
    const size_t nb = std::max<size_t>(grown, 256);
    if (cudaMalloc(&p, nb) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        throw Status{PICGPU_ENOMEM, "device allocation failed"};
    }
    bytes = nb;
}

void SoaBuf::ensure(size_t n) {
    for (auto& b : a) b.ensure(std::max<size_t>(n, 1) * 8);
    cap = std::max(cap, n);
}

Soa SoaBuf::soa() const {
    return Soa{a[0].as<double>(), a[1].as<double>(), a[2].as<double>(), a[3].as<double>(),
               a[4].as<double>(), a[5].as<double>(), a[6].as<double>(), a[7].as<uint64_t>()};
}

// Record stores are swapped with their re-layout spare (A <-> A2), so BOTH
// keep 12.5% headroom from their first allocation: a rebuild whose layout is a
// few slots larger must not pay a cudaFree + cudaMalloc of the whole store
// (C3: 45 GB, ~240 ms on the host).
void AosBuf::ensure(size_t n) {
    n = std::max<size_t>(n, 1);
    if (n * sizeof(Part) > a.bytes) a.ensure((n + n / 8) * sizeof(Part));
    cap = std::max(cap, n);
}

static void swap_aos(AosBuf& x, AosBuf& y) {
    std::swap(x.a.p, y.a.p);
    std::swap(x.a.bytes, y.a.bytes);
    std::swap(x.cap, y.cap);
}

static void swap_soa(SoaBuf& x, SoaBuf& y) {
    for (int i = 0; i < 8; ++i) {
        std::swap(x.a[i].p, y.a[i].p);
        std::swap(x.a[i].bytes, y.a[i].bytes);
    }
    std::swap(x.cap, y.cap);
}

static void swap_buf(DevBuf& x, DevBuf& y) {
    std::swap(x.p, y.p);
    std::swap(x.bytes, y.bytes);
}

// ---------------------------------------------------------------------------
// device helpers

// record -> record
__device__ __forceinline__ void copy_particle(const Aos src, uint64_t s, const Aos dst, uint64_t d) {
    copy_record(src.p + s, dst.p + d);
}

// packed arrays -> record
__device__ __forceinline__ void copy_particle(const Soa src, uint64_t s, const Aos dst, uint64_t d) {
    store_record(dst.p + d, src.x[s], src.y[s], src.z[s], src.vx[s], src.vy[s], src.vz[s], src.w[s], src.id[s]);
}

// record -> packed arrays
__device__ __forceinline__ void copy_particle(const Aos src, uint64_t s, const Soa dst, uint64_t d) {
    const double2* r = reinterpret_cast<const double2*>(src.p + s);
    const double2 a = r[0], b = r[1], c = r[2], e = r[3];
    dst.x[d] = a.x;
    dst.y[d] = a.y;
    dst.z[d] = b.x;
    dst.vx[d] = b.y;
    dst.vy[d] = c.x;
    dst.vz[d] = c.y;
    dst.w[d] = e.x;
    dst.id[d] = (uint64_t)__double_as_longlong(e.y);
}

__device__ __forceinline__ void copy_particle(const Soa src, uint64_t s, const Soa dst, uint64_t d) {
    dst.x[d] = src.x[s];
    dst.y[d] = src.y[s];
    dst.z[d] = src.z[s];
    dst.vx[d] = src.vx[s];
    dst.vy[d] = src.vy[s];
    dst.vz[d] = src.vz[s];
    dst.w[d] = src.w[s];
    dst.id[d] = src.id[s];
}

// Largest b in [0, nb) with so[b] <= s (bins of one CTA, offsets in smem).
__device__ __forceinline__ int find_bin(const uint32_t* so, int nb, uint32_t s) {
    int lo = 0, hi = nb - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (so[mid] <= s)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

// ---------------------------------------------------------------------------
// kernels

__global__ void k_cells(const GridD g, const double* __restrict__ x, const double* __restrict__ y,
                        const double* __restrict__ z, uint64_t n, uint32_t* __restrict__ cell, int* err) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const double px = x[p], py = y[p], pz = z[p];
    if (!finite3(px, py, pz)) {
        raise_error(err, PICGPU_EINVAL);
        cell[p] = 0;
        return;
    }
    const uint32_t c = store_cell(g, px, py, pz);
    if (c >= kLeaveRight) {  // not owned by this slab
        raise_error(err, PICGPU_EINVAL);
        cell[p] = 0;
        return;
    }
    cell[p] = c;
}

// Run boundaries of the sorted keys: start[c] = first rank, endp[c] = last rank + 1.
__global__ void k_boundaries(const uint32_t* __restrict__ key, uint64_t n, uint32_t* start, uint32_t* endp) {
    const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t k = key[r];
    if (r == 0 || key[r - 1] != k) start[k] = (uint32_t)r;
    if (r == n - 1 || key[r + 1] != k) endp[k] = (uint32_t)(r + 1);
}

// Capacity rule of Gpma::layout (gpma.hpp:275-278): ceil(count*(1+gap)) + min_gap.
__device__ __forceinline__ uint32_t bin_capacity(uint32_t count, double onepg, uint32_t min_gap) {
    return (uint32_t)ceil(__dmul_rn((double)count, onepg)) + min_gap;
}

__global__ void k_counts_caps(const uint32_t* start, const uint32_t* endp, uint32_t ncells, uint32_t* cnt,
                              uint32_t* caps, double onepg, uint32_t min_gap) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c > ncells) return;
    if (c == ncells) {
        caps[c] = 0;
        return;
    }
    const uint32_t k = endp[c] - start[c];
    cnt[c] = k;
    caps[c] = bin_capacity(k, onepg, min_gap);
}

__global__ void k_caps_from_cnt(const uint32_t* cnt, uint32_t ncells, uint32_t* caps, double onepg,
                                uint32_t min_gap) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c > ncells) return;
    caps[c] = c == ncells ? 0 : bin_capacity(cnt[c], onepg, min_gap);
}

// min(cnt, bin capacity): what a bin physically holds (after an overflow cnt
// counts the overflowed arrivals too).
__global__ void k_held(const uint32_t* cnt, const uint32_t* off, uint32_t ncells, uint32_t* held) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c > ncells) return;
    held[c] = c == ncells ? 0 : min(cnt[c], off[c + 1] - off[c]);
}

__global__ void k_u64_to_u32(const unsigned long long* in, uint32_t* out, uint64_t n) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (uint32_t)in[i];
}

// Sort keys of a binned store's slots, in storage order: the cell of each
// particle, ncells for holes and slack (they sort last).
__global__ void k_slot_keys(const GridD g, const Aos A, uint64_t slots, uint32_t* __restrict__ key, int* err) {
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= slots) return;
    const double2 r0 = reinterpret_cast<const double2*>(A.p + s)[0];
    if (is_gap(r0.x)) {
        key[s] = g.ncells;
        return;
    }
    const double z = A.p[s].z;
    if (!finite3(r0.x, r0.y, z)) {
        raise_error(err, PICGPU_EINVAL);
        key[s] = 0;
        return;
    }
    key[s] = store_cell(g, r0.x, r0.y, z);
}

template <class Src>
__global__ void k_gather_sorted(const Src src, const uint32_t* __restrict__ perm, const uint32_t* __restrict__ key,
                                const uint32_t* __restrict__ start, const uint32_t* __restrict__ off, const Aos dst,
                                uint64_t n) {
    const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t c = key[r];
    copy_particle(src, perm[r], dst, (uint64_t)off[c] + (r - start[c]));
}

#ifndef PICGPU_RELAYOUT_UNR2
#define PICGPU_RELAYOUT_UNR2 1
#endif
#ifndef PICGPU_BPB
#define PICGPU_BPB 64
#endif
constexpr int BPB = PICGPU_BPB;  // bins per CTA for the slot-range kernels

// Copy every bin's held particles (slot order kept) from src to dst offsets
// (Dst = Aos: a new layout of the store; Soa: packed staging).
template <class Dst>
__global__ void __launch_bounds__(256) k_relayout(const Aos src, const uint32_t* __restrict__ soff,
                                                  const uint32_t* __restrict__ cnt, const Dst dst,
                                                  const uint32_t* __restrict__ doff, uint32_t ncells) {
    __shared__ uint32_t so[BPB + 1], sc[BPB], dof[BPB];
    const uint32_t c0 = blockIdx.x * BPB;
    const int nb = (int)umin((uint32_t)BPB, ncells - c0);
    for (int b = threadIdx.x; b <= nb; b += blockDim.x) {
        so[b] = soff[c0 + b];
        if (b < nb) {
            sc[b] = min(cnt[c0 + b], soff[c0 + b + 1] - soff[c0 + b]);
            dof[b] = doff[c0 + b];
        }
    }
    __syncthreads();
    uint32_t s = so[0] + threadIdx.x;
    if constexpr (PICGPU_RELAYOUT_UNR2 && std::is_same<Dst, Aos>::value) {
        // two records in flight per thread (the loads of both before either store)
        for (; s + blockDim.x < so[nb]; s += 2 * blockDim.x) {
            const uint32_t t = s + blockDim.x;
            const int b0 = find_bin(so, nb, s), b1 = find_bin(so, nb, t);
            const uint32_t r0 = s - so[b0], r1 = t - so[b1];
            const bool k0 = r0 < sc[b0], k1 = r1 < sc[b1];
            const double2* p0 = reinterpret_cast<const double2*>(src.p + s);
            const double2* p1 = reinterpret_cast<const double2*>(src.p + t);
            double2 a0, a1, a2, a3, c0, c1, c2, c3;
            if (k0) { a0 = p0[0]; a1 = p0[1]; a2 = p0[2]; a3 = p0[3]; }
            if (k1) { c0 = p1[0]; c1 = p1[1]; c2 = p1[2]; c3 = p1[3]; }
            if (k0) {
                double2* d = reinterpret_cast<double2*>(dst.p + (uint64_t)dof[b0] + r0);
                d[0] = a0; d[1] = a1; d[2] = a2; d[3] = a3;
            }
            if (k1) {
                double2* d = reinterpret_cast<double2*>(dst.p + (uint64_t)dof[b1] + r1);
                d[0] = c0; d[1] = c1; d[2] = c2; d[3] = c3;
            }
        }
    }
    for (; s < so[nb]; s += blockDim.x) {
        const int b = find_bin(so, nb, s);
        const uint32_t r = s - so[b];
        if (r < sc[b]) copy_particle(src, s, dst, (uint64_t)dof[b] + r);
    }
}

// Aos -> Aos re-layout with the slack fill in ONE pass, a warp per bin: the
// bin's held records (slot order kept) are copied as 16-byte pieces, 32
// consecutive pieces per warp instruction (source and destination are both
// contiguous: no per-slot bin search, every access a full line), then the
// warp writes empty records into the bin's new slack [fill[c], new capacity)
// (slots [held, fill[c]) are left to k_place_left: the unplaced arrivals of a
// rebuild).  A warp takes 32 consecutive bins: lane i loads bin i's offsets
// and counts (coalesced), the per-bin values are then broadcast with shuffles.
// Replaces k_fill_slack + k_relayout<Aos> (one thread per slot, a binary search
// per slot, 64-byte records per thread: 2.3 TB/s of the copy's 6.5).
__global__ void __launch_bounds__(256) k_relayout_fill(const Aos src, const uint32_t* __restrict__ soff,
                                                       const uint32_t* __restrict__ cnt,
                                                       const uint32_t* __restrict__ fill, const Aos dst,
                                                       const uint32_t* __restrict__ doff, uint32_t ncells) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const uint64_t c0 = (uint64_t)warp * 32;
    if (c0 >= ncells) return;
    uint32_t so = 0, held = 0, d0 = 0, nfill = 0, ncap = 0;
    if (c0 + lane < ncells) {
        const uint32_t c = (uint32_t)c0 + lane;
        so = soff[c];
        held = min(cnt[c], soff[c + 1] - so);
        d0 = doff[c];
        ncap = doff[c + 1] - d0;
        nfill = min(fill[c], ncap);
    }
    const int nb = (int)min((uint64_t)32, ncells - c0);
    const double2 ones = make_double2(__longlong_as_double(-1LL), __longlong_as_double(-1LL));
    for (int b = 0; b < nb; ++b) {
        const uint32_t bso = __shfl_sync(0xffffffffu, so, b), bheld = __shfl_sync(0xffffffffu, held, b);
        const uint32_t bd0 = __shfl_sync(0xffffffffu, d0, b), bfill = __shfl_sync(0xffffffffu, nfill, b);
        const uint32_t bcap = __shfl_sync(0xffffffffu, ncap, b);
        const double2* __restrict__ s16 = reinterpret_cast<const double2*>(src.p + bso);
        double2* __restrict__ d16 = reinterpret_cast<double2*>(dst.p + bd0);
        const uint32_t np = 4u * bheld;
        for (uint32_t q = lane; q < np; q += 128) {  // up to four pieces in flight per lane
            double2 v0, v1, v2, v3;
            const bool k1 = q + 32 < np, k2 = q + 64 < np, k3 = q + 96 < np;
            v0 = s16[q];
            if (k1) v1 = s16[q + 32];
            if (k2) v2 = s16[q + 64];
            if (k3) v3 = s16[q + 96];
            d16[q] = v0;
            if (k1) d16[q + 32] = v1;
            if (k2) d16[q + 64] = v2;
            if (k3) d16[q + 96] = v3;
        }
        for (uint32_t q = 4u * bfill + lane; q < 4u * bcap; q += 32) d16[q] = ones;
    }
}

// Empty records into the slack of every bin of a fresh layout: slots
// [off[c] + fill[c], off[c+1]) (the particles are copied into the other slots
// by the layout's copy kernel; the two write disjoint slots).
__global__ void __launch_bounds__(256) k_fill_slack(const Aos A, const uint32_t* __restrict__ off,
                                                    const uint32_t* __restrict__ fill, uint32_t ncells) {
    __shared__ uint32_t so[BPB + 1], sf[BPB];
    const uint32_t c0 = blockIdx.x * BPB;
    const int nb = (int)umin((uint32_t)BPB, ncells - c0);
    for (int b = threadIdx.x; b <= nb; b += blockDim.x) {
        so[b] = off[c0 + b];
        if (b < nb) sf[b] = fill[c0 + b];
    }
    __syncthreads();
    for (uint32_t s = so[0] + threadIdx.x; s < so[nb]; s += blockDim.x) {
        const int b = find_bin(so, nb, s);
        if (s - so[b] >= sf[b]) store_gap_record(A.p + s);
    }
}

// Every slack slot holds a sentinel x (all-ones bit pattern, a NaN no valid
// particle can carry: non-finite positions are rejected), so the push can
// stream over raw slots without knowing the bin layout.

// Push (optional) + move detection (pic::advance + Gpma::detect_moves,
// workload.hpp:139-155, gpma.hpp:162-177).  Each CTA streams one contiguous
// chunk of UNR*256 slots.  Measured at C2 (tools/push_sweep.sh): one slot per
// thread at 6 CTAs/SM (0.83 ms, 4.0 TB/s, SoA store; with the record store a slot
// is loaded as three 16-byte pieces) beats loading only the valid slots after x, whose
// second round trip costs more than the slack bytes it saves.  The cell test is exact and
// cheap: a particle moves at most one cell, so when every axis' floor is
// unchanged (and non-negative) its cell is unchanged; only otherwise are the
// full cell ids of both positions computed (pic::cell_of).
// A particle whose cell changed is flagged and appended to the mover list:
// slots are numbered with a shared-memory atomic and the CTA reserves its
// range with ONE global atomic (no per-warp atomic round trips on the hot
// path); departures are counted per bin with fire-and-forget reductions.
// Movers that do not fit the mover buffer stay in their (now stale) bin with
// flag 2; the host then re-sorts fully.
// UNR 2 (both records in flight before any push) measured slower at C3:
// push + sort 46.4 (512 threads, 64 registers, spills) / 44.2 (256 threads,
// 80 registers) / 47.7 (w, id early) vs 43.5 ms at UNR 1 (profiles/r02/kpush_unr_ab.txt).
#ifndef PICGPU_PUSH_UNR
#define PICGPU_PUSH_UNR 1
#endif
#ifndef PICGPU_PUSH_EARLY_WID  // w, id with the rest of the record (UNR 1: C3 48.1 -> 46.0 ms)
#define PICGPU_PUSH_EARLY_WID (PICGPU_PUSH_UNR == 1)
#endif
// Threads per CTA: the CTA's ONE global reservation on ctr->nmovers is a
// same-address atomic, serialised in L2 -- C3 has 2.7M CTAs of 256 slots,
// so the reservations (and the moved-count reductions on the same line, now
// spread over kMovedParts counters) bound the kernel; wider CTAs need fewer.
#ifndef PICGPU_PUSH_NT
#define PICGPU_PUSH_NT 512
#endif
#ifndef PICGPU_PUSH_MINB
// record store: 5 CTAs/SM (48 registers) beat 6 (40, spills): C3 push+sort 54 -> 48 ms; with
// w/id loaded up front (64 registers) 4 CTAs/SM: 48.1 -> 46.0 ms (5 CTAs spill: 50.2 ms)
#define PICGPU_PUSH_MINB (4 * 256 / PICGPU_PUSH_NT)
#endif

// RECORD = false: push and count the moved particles only (the store is
// re-sorted from scratch afterwards; no flags, movers or departures).
// One slot of k_push: its record (w, id loaded with the rest: the mover copy
// needs no second round trip), then push + move test.
struct PushSlot {
    double x, y, z, vx, vy, vz;
    double2 wid;
    uint32_t nc, before;
    int lidx;
    bool moved;
};

template <bool RECORD>
__device__ __forceinline__ void push_load(const Aos& A, uint64_t s, uint64_t slots, PushSlot& q) {
    q.x = __longlong_as_double(-1LL);
    q.y = q.z = q.vx = q.vy = q.vz = 0.0;
    q.wid = make_double2(0.0, 0.0);
    q.nc = q.before = 0;
    q.lidx = -1;
    q.moved = false;
    if (s < slots) {  // x y | z vx | vy vz (| w id) of the record
        const double2* r = reinterpret_cast<const double2*>(A.p + s);
        const double2 a = r[0], b = r[1], c = r[2];
        if (PICGPU_PUSH_EARLY_WID && RECORD) q.wid = r[3];  // same two sectors
        q.x = a.x;
        q.y = a.y;
        q.z = b.x;
        q.vx = b.y;
        q.vy = c.x;
        q.vz = c.y;
    }
}

template <bool PUSH, bool P2, bool RECORD>
__device__ __forceinline__ void push_slot(const GridD& g, const Aos& A, uint64_t s, double dt, double cap2,
                                          PushSlot& q, const uint32_t* __restrict__ off,
                                          uint32_t* __restrict__ holes, uint32_t* __restrict__ hl,
                                          StepCounters* ctr, double* __restrict__ L, uint32_t lcap, unsigned* s_cnt) {
    if (is_gap(q.x)) return;
    if (!finite3(q.x, q.y, q.z)) {
        raise_error(&ctr->err, PICGPU_EINVAL);
        return;
    }
    if (PUSH) {
        const double ox = q.x, oy = q.y, oz = q.z;
        bool ok = push_one<P2>(g, dt, cap2, q.x, q.y, q.z, q.vx, q.vy, q.vz);
        if (!ok) {
            raise_error(&ctr->err, PICGPU_EDOMAIN);
        } else {
#if PICGPU_WB_SECTOR
            reinterpret_cast<double2*>(A.p + s)[0] = make_double2(q.x, q.y);
            reinterpret_cast<double2*>(A.p + s)[1] = make_double2(q.z, q.vx);
#else
            reinterpret_cast<double2*>(A.p + s)[0] = make_double2(q.x, q.y);
            A.p[s].z = q.z;
#endif
            if (!finite3(q.x, q.y, q.z)) {
                raise_error(&ctr->err, PICGPU_EINVAL);
                ok = false;
            }
        }
        if (ok) {
            const int p2x = P2 || g.pow2x, p2y = P2 || g.pow2y, p2z = P2 || g.pow2z;
            const double fx0 = axis_floor(ox, g.gox, g.dx, g.inv_dx, p2x);
            const double fy0 = axis_floor(oy, g.oy, g.dy, g.inv_dy, p2y);
            const double fz0 = axis_floor(oz, g.oz, g.dz, g.inv_dz, p2z);
            const bool same = fx0 >= 0.0 && fy0 >= 0.0 && fz0 >= 0.0 &&
                              fx0 == axis_floor(q.x, g.gox, g.dx, g.inv_dx, p2x) &&
                              fy0 == axis_floor(q.y, g.oy, g.dy, g.inv_dy, p2y) &&
                              fz0 == axis_floor(q.z, g.oz, g.dz, g.inv_dz, p2z);
            if (!same) {
                q.before = store_cell<P2>(g, ox, oy, oz);
                q.nc = store_cell<P2>(g, q.x, q.y, q.z);
                q.moved = q.nc != q.before;
            }
        }
    }
    if (RECORD && q.moved) {
        if (q.nc >= kLeaveRight) {  // left the slab: exchange record for the neighbour rank
            const int dir = q.nc == kLeaveLeft ? 0 : 1;
            const unsigned li = atomicAdd(&ctr->nleave[dir], 1u);
            if (li < lcap) {
                double* r = L + ((size_t)dir * lcap + li) * 8;
                r[0] = q.x; r[1] = q.y; r[2] = q.z;
                r[3] = q.vx; r[4] = q.vy; r[5] = q.vz;
                if (!PICGPU_PUSH_EARLY_WID) q.wid = reinterpret_cast<const double2*>(A.p + s)[3];
                r[6] = q.wid.x;
                r[7] = q.wid.y;
                push_hole(A, s, q.before, off, holes, hl);
            } else {
                raise_error(&ctr->err, PICGPU_ELENGTH);
            }
        } else {
            q.lidx = (int)atomicAdd(s_cnt, 1u);
        }
    }
}

template <bool RECORD>
__device__ __forceinline__ void push_store_mover(const Aos& A, uint64_t s, const PushSlot& q, unsigned base,
                                                 const Soa& M, uint32_t* __restrict__ mcell, uint32_t mcap,
                                                 uint32_t* __restrict__ mslot, uint32_t* __restrict__ mbin) {
    if (q.lidx < 0) return;
    const unsigned idx = base + (unsigned)q.lidx;
    if (idx >= mcap) return;  // not recorded (mover buffer full): stays in its stale bin; the host re-sorts
    double2 wid = q.wid;
    if (!PICGPU_PUSH_EARLY_WID) wid = reinterpret_cast<const double2*>(A.p + s)[3];
    M.x[idx] = q.x;
    M.y[idx] = q.y;
    M.z[idx] = q.z;
    M.vx[idx] = q.vx;
    M.vy[idx] = q.vy;
    M.vz[idx] = q.vz;
    M.w[idx] = wid.x;
    M.id[idx] = (uint64_t)__double_as_longlong(wid.y);
    mcell[idx] = q.nc;
    // the slot becomes a hole now; it joins its bin's hole list in
    // k_departures (no atomic round trip in this streaming kernel)
    store_gap_record(A.p + s);
    mslot[idx] = (uint32_t)s;
    mbin[idx] = q.before;
}

// UNR slots per thread (slot t and t + NT, ... of the CTA's range): every
// record is loaded before any is pushed and one reservation covers UNR x NT
// slots (measured: UNR 1 is fastest, see PICGPU_PUSH_UNR).
template <bool PUSH, int UNR, bool P2, bool RECORD = true>
__global__ void __launch_bounds__(PICGPU_PUSH_NT, PICGPU_PUSH_MINB) k_push(const GridD g, const Aos A, uint64_t slots,
                                              double dt, double cap2, const Soa M, uint32_t* __restrict__ mcell,
                                              uint32_t mcap, const uint32_t* __restrict__ off,
                                              uint32_t* __restrict__ holes, uint32_t* __restrict__ hl,
                                              StepCounters* ctr, double* __restrict__ L, uint32_t lcap,
                                              uint32_t* __restrict__ mslot, uint32_t* __restrict__ mbin,
                                              unsigned long long* __restrict__ mvpart) {
    __shared__ unsigned s_cnt, s_base, s_mv;
    if (threadIdx.x == 0) s_cnt = s_mv = 0;
    __syncthreads();
    const uint64_t s0 = (uint64_t)blockIdx.x * blockDim.x * UNR + threadIdx.x;
    PushSlot q[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) push_load<RECORD>(A, s0 + (uint64_t)u * blockDim.x, slots, q[u]);
    unsigned nmv = 0;
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
        push_slot<PUSH, P2, RECORD>(g, A, s0 + (uint64_t)u * blockDim.x, dt, cap2, q[u], off, holes, hl, ctr, L,
                                    lcap, &s_cnt);
        nmv += q[u].moved ? 1u : 0u;
    }
    // moved count: one shared-memory add per warp, one RED per block on one of
    // kMovedParts counters (k_fold_moved sums them into ctr->moved)
    const unsigned wm = __reduce_add_sync(0xffffffffu, nmv);
    if ((threadIdx.x & 31) == 0 && wm) atomicAdd(&s_mv, wm);
    __syncthreads();
    unsigned long long* part = mvpart + (size_t)(blockIdx.x % kMovedParts) * 16;
    if (!RECORD) {
        if (threadIdx.x == 0 && s_mv) atomicAdd(part, (unsigned long long)s_mv);
        return;
    }
    if (threadIdx.x == 0) {
        s_base = s_cnt ? atomicAdd(&ctr->nmovers, s_cnt) : 0u;
        if (s_mv) atomicAdd(part, (unsigned long long)s_mv);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < UNR; ++u)
        push_store_mover<RECORD>(A, s0 + (uint64_t)u * blockDim.x, q[u], s_base, M, mcell, mcap, mslot, mbin);
}

// Gaps, as in the reference's GPMA: a departing particle leaves a hole in its
// bin (delete_in_bin only marks the slot empty, gpma.hpp:328-335) and the next
// arrivals into that bin fill holes before they take tail slack (insert uses a
// spare slot of the bin, gpma.hpp:248-267).  A bin's extent [off, off+cnt)
// then holds particles and holes (sentinel x); holes[c] counts the holes.  The
// deposits skip holes; the per-step compaction pass of a packed store is gone.
//
// k_fill_holes makes every bin packed again before an operation that needs it
// (rebuild, global sort, downloads, window shift): a warp watches 32 bins'
// hole counts with one ballot and fills four holey bins at a time, one per
// 8-lane group.  With nd holes in an extent of len slots, each hole among the
// first len-nd slots takes one particle from the tail [len-nd, len) (the k-th
// front hole the k-th tail particle), and the tail becomes slack.  Bins with
// more than kHoleCap front holes fall back to a stable slide.
constexpr int kHoleCap = 32;

// ctr->moved += the spread partial counts of k_push; the partials are reset.
__global__ void k_fold_moved(unsigned long long* __restrict__ mvpart, StepCounters* ctr) {
    unsigned long long v = 0;
    for (int i = threadIdx.x; i < kMovedParts; i += blockDim.x) {
        v += mvpart[(size_t)i * 16];
        mvpart[(size_t)i * 16] = 0;
    }
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __shared__ unsigned long long w[32];
    if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int k = 0; k < (int)(blockDim.x + 31) / 32; ++k) t += w[k];
        if (t) ctr->moved += t;
    }
}

#ifndef PICGPU_COMPACT_MINB
#define PICGPU_COMPACT_MINB 8  // latency-bound: full occupancy beats spill-free registers (191 vs 209+ us at C2)
#endif
__global__ void __launch_bounds__(256, PICGPU_COMPACT_MINB) k_fill_holes(const Aos A, const uint32_t* __restrict__ off,
                                                                    uint32_t* cnt, uint32_t* dep, uint32_t ncells) {
    __shared__ uint32_t holes[256 / 8][kHoleCap];
    const int lane = threadIdx.x & 31;
    const int grp = lane >> 3, gl = lane & 7;  // four groups of 8 lanes, one dirty bin each
    const int gid = threadIdx.x >> 3;          // group index in the CTA
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t cl = wid * 32 + lane;
    const uint32_t mydep = cl < ncells ? dep[cl] : 0u;
    unsigned todo = __ballot_sync(0xffffffffu, mydep != 0);
    while (todo) {  // warp-uniform: the next (up to) four dirty bins, one per group
        int bin = -1;
#pragma unroll
        for (int gq = 0; gq < 4; ++gq) {
            const int b = todo ? __ffs(todo) - 1 : -1;
            if (todo) todo &= todo - 1;
            if (gq == grp) bin = b;
        }
        const bool active = bin >= 0;
        const uint32_t c = wid * 32 + (uint32_t)(active ? bin : 0);
        const uint32_t nd = __shfl_sync(0xffffffffu, mydep, active ? bin : 0);
        uint32_t lo = 0, len = 0;
        if (active) {
            lo = off[c];
            len = cnt[c];
        }
        const uint32_t front = len - min(nd, len);
        // front holes -> shared list (ranked by position)
        uint32_t nh = 0;
        bool spill = false;
        const uint32_t maxfront = __reduce_max_sync(0xffffffffu, front);
        for (uint32_t o = 0; o < maxfront; o += 8) {
            const uint32_t r = lo + o + gl;
            const bool hole = o + gl < front && is_gap(A.p[r].x);
            const unsigned hm = (__ballot_sync(0xffffffffu, hole) >> (grp * 8)) & 0xffu;
            const uint32_t k = nh + __popc(hm & ((1u << gl) - 1u));
            if (hole && k < kHoleCap) holes[gid][k] = r;
            nh += __popc(hm);
        }
        spill = nh > kHoleCap;
        __syncwarp();
        // tail survivors fill the holes, in order
        const uint32_t maxlen = __reduce_max_sync(0xffffffffu, len);
        uint32_t nk = 0;
        for (uint32_t o = front; __any_sync(0xffffffffu, o < maxlen); o += 8) {
            const uint32_t r = lo + o + gl;
            const bool kept = !spill && o + gl < len && !is_gap(A.p[r].x);
            const unsigned km = (__ballot_sync(0xffffffffu, kept) >> (grp * 8)) & 0xffu;
            if (kept) copy_particle(A, r, A, holes[gid][nk + __popc(km & ((1u << gl) - 1u))]);
            nk += __popc(km);
        }
        __syncwarp();
        if (active && !spill) {
            for (uint32_t r = lo + front + gl; r < lo + len; r += 8) store_gap_record(A.p + r);
            if (gl == 0) cnt[c] = front;
        }
        // a bin with more front holes than the list holds: stable slide
        if (__any_sync(0xffffffffu, spill)) {
            uint32_t wpos = lo;
            const uint32_t sl_len = spill ? len : 0u;
            const uint32_t maxs = __reduce_max_sync(0xffffffffu, sl_len);
            for (uint32_t o = 0; o < maxs; o += 8) {
                const uint32_t r = lo + o + gl;
                const bool keep = o + gl < sl_len && !is_gap(A.p[r].x);
                const unsigned km = (__ballot_sync(0xffffffffu, keep) >> (grp * 8)) & 0xffu;
                const uint32_t dst = wpos + __popc(km & ((1u << gl) - 1u));
                double2 q0{}, q1{}, q2{}, q3{};
                const bool mv = keep && dst != r;
                if (mv) {
                    const double2* src = reinterpret_cast<const double2*>(A.p + r);
                    q0 = src[0]; q1 = src[1]; q2 = src[2]; q3 = src[3];
                }
                __syncwarp();
                if (mv) {
                    double2* d2 = reinterpret_cast<double2*>(A.p + dst);
                    d2[0] = q0; d2[1] = q1; d2[2] = q2; d2[3] = q3;
                }
                __syncwarp();
                wpos += __popc(km);
            }
            if (spill) {
                for (uint32_t r = wpos + gl; r < lo + len; r += 8) store_gap_record(A.p + r);
                if (gl == 0) cnt[c] = wpos - lo;
            }
        }
    }
    if (mydep) dep[cl] = 0;
}

// Departures of k_push's movers join their old bins' hole lists (delete_in_bin,
// gpma.hpp:328-335); the slots already hold gap records.
__global__ void k_departures(const StepCounters* ctr, uint32_t mcap, const uint32_t* __restrict__ mslot,
                             const uint32_t* __restrict__ mbin, const uint32_t* __restrict__ off,
                             uint32_t* __restrict__ holes, uint32_t* __restrict__ hl) {
    const uint32_t nm = min(ctr->nmovers, mcap);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nm; i += gridDim.x * blockDim.x) {
        const uint32_t b = mbin[i];
        hl[off[b] + atomicAdd(&holes[b], 1u)] = mslot[i];
    }
}

// Migration: an arrival first takes a hole of its bin, else the next slot of
// its slack (atomic tail cursor); arrivals beyond the slack go to the overflow
// list.  Holes are popped from the bin's list with one atomicSub on holes[d]:
// the first holes[d] decrements return holes[d], ..., 1 (list entries, each
// once -- no departures run concurrently); a decrement that returns <= 0 found
// the list empty and gives its unit back, so holes[d] ends at max(h0 - a, 0).
__global__ void k_insert(const Soa M, const uint32_t* __restrict__ mcell, uint32_t mcap,
                         StepCounters* ctr, const Aos A, const uint32_t* __restrict__ off, uint32_t* cnt,
                         uint32_t* __restrict__ ovf, uint32_t* __restrict__ holes, const uint32_t* __restrict__ hl) {
    const uint32_t nm = min(ctr->nmovers, mcap) + ctr->nimport;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nm; i += gridDim.x * blockDim.x) {
        const uint32_t d = mcell[i];
        if (d == kNoCell) continue;  // a leaver exported by the fused slab step
        const uint32_t lo = off[d];
        const int h = (int)atomicSub(&holes[d], 1u);
        if (h > 0) {
            copy_particle(M, i, A, hl[lo + (uint32_t)h - 1u]);
            continue;
        }
        atomicAdd(&holes[d], 1u);  // RED
        const uint32_t pos = atomicAdd(&cnt[d], 1u);
        if (pos < off[d + 1] - lo) {
            copy_particle(M, i, A, (uint64_t)lo + pos);
        } else {
            ovf[atomicAdd(&ctr->noverflow, 1u)] = i;
        }
    }
}

// borrow_insert (gpma.hpp:337-370) for the arrivals that found their bin
// full: the nearest of the next `scan` bins with a free slot -- tail slack or
// a hole, as the reference's slot scan takes the first empty slot of either
// kind -- lends one slot; every boundary in (d, donor] moves up by one and
// each (full, hole-free) bin in between hands its first particle to its own
// tail (the slot just vacated above it), so bins stay contiguous and
// cell-exact.  A hole-free donor does the same into its tail slack; a donor
// with holes gives one up instead: its first slot's particle moves into one of
// them (or the first slot is itself the hole) and its hole list follows its
// base.  One
// thread per overflowed arrival; a thread works only while it holds try-locks
// on its whole window [d, d+scan] (taken in ascending order, released on any
// failure, so no thread ever waits while holding a lock).  Arrivals with no
// donor go to `left` for the re-sort.
__global__ void k_borrow(StepCounters* ctr, const Soa M, const uint32_t* __restrict__ mcell,
                         const uint32_t* __restrict__ ovf, uint32_t* __restrict__ left, const Aos A, uint32_t* off,
                         uint32_t* cnt, uint32_t* holes, uint32_t* hl, unsigned int* lock, uint32_t ncells, int scan) {
    const uint32_t n = *(volatile unsigned int*)&ctr->noverflow;
    for (uint32_t o = blockIdx.x * blockDim.x + threadIdx.x; o < n; o += gridDim.x * blockDim.x) {
        const uint32_t i = ovf[o];
        const uint32_t d = mcell[i];
        const uint64_t lim = (uint64_t)d + (uint64_t)scan;
        const uint32_t last = (uint32_t)(lim < (uint64_t)ncells - 1 ? lim : (uint64_t)ncells - 1);
        if (last <= d) {  // last bin: nothing follows it
            left[atomicAdd(&ctr->nleft, 1u)] = i;
            continue;
        }
        for (int attempt = 0;; ++attempt) {
            uint32_t got = d;
            while (got <= last && atomicCAS(&lock[got], 0u, 1u) == 0u) ++got;
            if (got <= last) {
                for (uint32_t b = d; b < got; ++b) atomicExch(&lock[b], 0u);
                __nanosleep(64u << (attempt < 6 ? attempt : 6));
                continue;
            }
            __threadfence();
            volatile uint32_t* voff = off;
            volatile uint32_t* vcnt = cnt;
            volatile uint32_t* vholes = holes;
            volatile uint32_t* vhl = hl;
            int64_t donor = -1;
            for (uint32_t b = d + 1; b <= last; ++b)
                if (vcnt[b] < voff[b + 1] - voff[b] || vholes[b] > 0) {
                    donor = b;
                    break;
                }
            if (donor < 0) {
                left[atomicAdd(&ctr->nleft, 1u)] = i;
            } else {
                const uint32_t slot = voff[d + 1];  // becomes bin d's new last slot
                uint32_t above = voff[(uint32_t)donor + 1];
                for (uint32_t j = (uint32_t)donor; j > d; --j) {
                    const uint32_t oj = voff[j];
                    const uint32_t len = vcnt[j];
                    const uint32_t hj = j == (uint32_t)donor ? vholes[j] : 0u;  // bins in between have none
                    uint64_t dst = (uint64_t)oj + min(len, above - oj);  // tail slack, or `above` (vacated by bin j+1)
                    if (hj) {  // a donor with holes gives one up (they are the spare slots arrivals missed)
                        uint32_t k = hj - 1;
                        if (is_gap(__ldcg(&A.p[oj].x))) {
                            while (k > 0 && vhl[oj + k] != oj) --k;  // the first slot is a listed hole
                            vhl[oj + k] = vhl[oj + hj - 1];
                            dst = oj;                       // nothing to move
                        } else {
                            dst = vhl[oj + k];
                        }
                        for (uint32_t q = hj - 1; q-- > 0;) vhl[oj + 1 + q] = vhl[oj + q];
                        vholes[j] = hj - 1;
                        vcnt[j] = len - 1;
                    }
                    if (len > 0 && dst != oj) {
                        const double2* src = reinterpret_cast<const double2*>(A.p + oj);
                        double2* d2 = reinterpret_cast<double2*>(A.p + dst);
                        const double2 q0 = __ldcg(src), q1 = __ldcg(src + 1), q2 = __ldcg(src + 2), q3 = __ldcg(src + 3);
                        d2[0] = q0; d2[1] = q1; d2[2] = q2; d2[3] = q3;
                    }
                    voff[j] = oj + 1;
                    above = oj;
                }
                copy_particle(M, i, A, slot);
                atomicAdd(&ctr->nborrowed, 1u);
            }
            __threadfence();
            for (uint32_t b = d; b <= last; ++b) atomicExch(&lock[b], 0u);
            break;
        }
    }
}

// Gpma::rebuild tail (gpma.hpp:137): arrivals that found no slack even after
// borrowing go after their bin's held particles in the fresh layout.
__global__ void k_place_left(const Soa M, const uint32_t* __restrict__ mcell, const uint32_t* __restrict__ left,
                             uint32_t nleft, const Aos dst, const uint32_t* __restrict__ doff, uint32_t* held) {
    const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= nleft) return;
    const uint32_t i = left[o];
    const uint32_t d = mcell[i];
    copy_particle(M, i, dst, (uint64_t)doff[d] + atomicAdd(&held[d], 1u));
}

// Overflowed movers appended after a packed store (mover-buffer fallback).
__global__ void k_append_overflow(const Soa M, const uint32_t* __restrict__ ovf, uint32_t novf, const Soa dst,
                                  uint64_t base) {
    const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o < novf) copy_particle(M, ovf[o], dst, base + o);
}

// Arrivals from the neighbour slabs (8-double records: x y z vx vy vz w id)
// appended to the mover list after this rank's own movers; k_insert and
// k_borrow then place them like any mover.
__global__ void k_import(const GridD g, const double* __restrict__ rec, uint32_t n, uint32_t base, const Soa M,
                         uint32_t* __restrict__ mcell, StepCounters* ctr) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {
        ctr->nimport = n;
        ctr->nmovers = base;  // own movers beyond the old capacity stay in their bins (flag 2)
    }
    if (i >= n) return;
    const double* r = rec + (size_t)i * 8;
    const double x = r[0], y = r[1], z = r[2];
    uint32_t c = 0;
    if (!finite3(x, y, z)) {
        raise_error(&ctr->err, PICGPU_EINVAL);
    } else {
        c = store_cell(g, x, y, z);
        if (c >= kLeaveRight) {  // routed to the wrong slab
            raise_error(&ctr->err, PICGPU_EINVAL);
            c = 0;
        }
    }
    const uint32_t d = base + i;
    M.x[d] = x; M.y[d] = y; M.z[d] = z;
    M.vx[d] = r[3]; M.vy[d] = r[4]; M.vz[d] = r[5];
    M.w[d] = r[6];
    M.id[d] = (uint64_t)__double_as_longlong(r[7]);
    mcell[d] = c;
}

// Arrivals of a device-resident exchange (picgpu_session_slab_step): the
// counts came with the records (cnt[0] from the left, cnt[1] from the right),
// so the host never reads them.  k_import_plan fixes the list: own movers
// [0, base), base = min(nmovers, mcap), then min(cnt, B) records per side;
// a side that sent more than its bucket B raises ovf_import (the host
// finishes those in a second, exactly sized round).
__global__ void k_import_plan(const uint32_t* __restrict__ cnt, uint32_t B, uint32_t mcap, StepCounters* ctr) {
    const uint32_t base = min(ctr->nmovers, mcap);
    const uint32_t nl = min(cnt[0], B), nr = min(cnt[1], B);
    if (ctr->nmovers > mcap) ctr->mover_drop += ctr->nmovers - mcap;  // unrecorded own movers -> full re-sort
    ctr->nmovers = base;
    if (base + nl + nr > mcap) {  // the host sized the mover buffers for 2B arrivals: never
        raise_error(&ctr->err, PICGPU_ELENGTH);
        ctr->nimport = 0;
        return;
    }
    ctr->nimport = nl + nr;
    ctr->import_left = nl;
    ctr->ovf_import = (cnt[0] > B ? 1u : 0u) | (cnt[1] > B ? 2u : 0u);
}

__global__ void k_import_dev(const GridD g, const double* __restrict__ from_left, const double* __restrict__ from_right,
                             uint32_t B, const Soa M, uint32_t* __restrict__ mcell, StepCounters* ctr) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t nl = ctr->import_left, n = ctr->nimport;
    if (t >= 2 * B) return;
    const bool right = t >= B;
    const uint32_t j = right ? t - B : t;
    const uint32_t i = right ? nl + j : j;  // rank in the arrival list
    if (right ? (i >= n) : (j >= nl)) return;
    const double* r = (right ? from_right : from_left) + (size_t)j * 8;
    const double x = r[0], y = r[1], z = r[2];
    uint32_t c = 0;
    if (!finite3(x, y, z)) {
        raise_error(&ctr->err, PICGPU_EINVAL);
    } else {
        c = store_cell(g, x, y, z);
        if (c >= kLeaveRight) {  // routed to the wrong slab
            raise_error(&ctr->err, PICGPU_EINVAL);
            c = 0;
        }
    }
    const uint32_t d = ctr->nmovers + i;
    M.x[d] = x; M.y[d] = y; M.z[d] = z;
    M.vx[d] = r[3]; M.vy[d] = r[4]; M.vz[d] = r[5];
    M.w[d] = r[6];
    M.id[d] = (uint64_t)__double_as_longlong(r[7]);
    mcell[d] = c;
}

// Guard planes of a slab's field (comps arrays of nx*ny*nz, x fastest):
// planes [p0, p0+np) packed as [comp][plane][z][y].
__global__ void k_pack_planes(const double* __restrict__ F, int comps, int nx, int ny, int nz, int p0, int np,
                              double* __restrict__ out) {
    const uint64_t total = (uint64_t)comps * np * ny * nz;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const int p = (int)(t % np);
        uint64_t r = t / np;
        const int j = (int)(r % ny);
        r /= ny;
        const int k = (int)(r % nz);
        const int c = (int)(r / nz);
        const size_t src = (size_t)c * nx * ny * nz + ((size_t)k * ny + j) * nx + p0 + p;
        out[(((size_t)c * np + p) * nz + k) * ny + j] = F[src];
    }
}

__global__ void k_add_planes(double* __restrict__ F, int comps, int nx, int ny, int nz, int p0, int np,
                             const double* __restrict__ in) {
    const uint64_t total = (uint64_t)comps * np * ny * nz;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const int p = (int)(t % np);
        uint64_t r = t / np;
        const int j = (int)(r % ny);
        r /= ny;
        const int k = (int)(r % nz);
        const int c = (int)(r / nz);
        const size_t dst = (size_t)c * nx * ny * nz + ((size_t)k * ny + j) * nx + p0 + p;
        F[dst] += in[(((size_t)c * np + p) * nz + k) * ny + j];
    }
}

__global__ void k_advance(const GridD g, double dt, double cap2, double* __restrict__ x, double* __restrict__ y,
                          double* __restrict__ z, const double* __restrict__ vx, const double* __restrict__ vy,
                          const double* __restrict__ vz, uint64_t n, unsigned long long* moved, int* err) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool m = false;
    if (p < n) {
        double px = x[p], py = y[p], pz = z[p];
        if (!finite3(px, py, pz)) {
            raise_error(err, PICGPU_EINVAL);
        } else {
            const uint32_t before = cell_linear(g, px, py, pz);
            if (!push_one<false>(g, dt, cap2, px, py, pz, vx[p], vy[p], vz[p])) {
                raise_error(err, PICGPU_EDOMAIN);
            } else {
                x[p] = px;
                y[p] = py;
                z[p] = pz;
                if (!finite3(px, py, pz))
                    raise_error(err, PICGPU_EINVAL);
                else
                    m = cell_linear(g, px, py, pz) != before;
            }
        }
    }
    const unsigned b = __ballot_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(moved, (unsigned long long)__popc(b));
}

// rng.hpp:12-27 (bit-identical), rng.hpp:30-34 (device libm: last-ulp
// differences from glibc are possible; benchmark inputs only).
__device__ __forceinline__ uint64_t hash_mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double uniform01(uint64_t seed, uint64_t stream, uint64_t counter) {
    const uint64_t bits = hash_mix(hash_mix(hash_mix(seed) ^ stream) ^ counter);
    return __dmul_rn(__dadd_rn((double)(bits >> 11), 0.5), 0x1.0p-53);
}
__device__ __forceinline__ double gaussian(uint64_t seed, uint64_t stream, uint64_t counter) {
    const double u1 = uniform01(seed, stream, 2 * counter);
    const double u2 = uniform01(seed, stream, 2 * counter + 1);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

// The generator of the whole box restricted to the owned x-cells: particle
// ids (and hence every hashed draw) are the global ones.
__global__ void k_generate(const GridD g, int ppc, double u_th, uint64_t seed, const Soa out, uint64_t n) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const uint64_t lin = p / (uint64_t)ppc;
    const uint64_t own = (uint64_t)(g.sx_hi - g.sx_lo);
    const int i = (int)(lin % own) + g.sx_lo + g.sx_shift;  // global x-cell
    const int j = (int)((lin / own) % (uint64_t)g.ny);
    const int k = (int)(lin / (own * (uint64_t)g.ny));
    const uint64_t pid = (((uint64_t)k * g.ny + j) * g.gnx + i) * (uint64_t)ppc + p % (uint64_t)ppc;
    out.x[p] = __dadd_rn(g.gox, __dmul_rn(__dadd_rn((double)i, uniform01(seed, pid, 6)), g.dx));
    out.y[p] = __dadd_rn(g.oy, __dmul_rn(__dadd_rn((double)j, uniform01(seed, pid, 7)), g.dy));
    out.z[p] = __dadd_rn(g.oz, __dmul_rn(__dadd_rn((double)k, uniform01(seed, pid, 8)), g.dz));
    const double ux = u_th * gaussian(seed, pid, 0);
    const double uy = u_th * gaussian(seed, pid, 1);
    const double uz = u_th * gaussian(seed, pid, 2);
    const double gam = sqrt(1.0 + ux * ux + uy * uy + uz * uz);
    out.vx[p] = ux / gam;
    out.vy[p] = uy / gam;
    out.vz[p] = uz / gam;
    out.w[p] = 1.0 / (double)ppc;
    out.id[p] = pid;
}

// SURVEY 8(d) C4 population (see picgpu_session_generate_lwfa): pfx[i] =
// background particles of x-cells < i in one (y, z) row.
__global__ void k_generate_lwfa(const GridD g, const uint32_t* __restrict__ pfx, uint64_t nbg, uint64_t n, int ppc,
                                double u_th, double ux_min, double ux_max, double bx0, double bx1, uint64_t seed,
                                const Soa out) {
    const uint64_t pid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pid >= n) return;
    double ux, uy, uz;
    if (pid < nbg) {
        const uint32_t R = pfx[g.nx];
        const uint64_t row = pid / R;
        const uint32_t r = (uint32_t)(pid % R);
        int lo = 0, hi = g.nx - 1;  // largest i with pfx[i] <= r
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (pfx[mid] <= r)
                lo = mid;
            else
                hi = mid - 1;
        }
        const int i = lo;
        const int j = (int)(row % (uint64_t)g.ny);
        const int k = (int)(row / (uint64_t)g.ny);
        out.x[pid] = __dadd_rn(g.ox, __dmul_rn(__dadd_rn((double)i, uniform01(seed, pid, 6)), g.dx));
        out.y[pid] = __dadd_rn(g.oy, __dmul_rn(__dadd_rn((double)j, uniform01(seed, pid, 7)), g.dy));
        out.z[pid] = __dadd_rn(g.oz, __dmul_rn(__dadd_rn((double)k, uniform01(seed, pid, 8)), g.dz));
        ux = u_th * gaussian(seed, pid, 0);
        uy = u_th * gaussian(seed, pid, 1);
        uz = u_th * gaussian(seed, pid, 2);
    } else {
        const double fx = __dadd_rn(bx0, __dmul_rn(__dsub_rn(bx1, bx0), uniform01(seed, pid, 6)));
        out.x[pid] = __dadd_rn(g.ox, __dmul_rn(fx, g.dx));
        out.y[pid] = __dadd_rn(g.oy, __dmul_rn(g.Ly, uniform01(seed, pid, 7)));
        out.z[pid] = __dadd_rn(g.oz, __dmul_rn(g.Lz, uniform01(seed, pid, 8)));
        ux = __dadd_rn(ux_min, __dmul_rn(__dsub_rn(ux_max, ux_min), uniform01(seed, pid, 9)));
        uy = uz = 0.0;
    }
    const double gam = sqrt(1.0 + ux * ux + uy * uy + uz * uz);
    out.vx[pid] = ux / gam;
    out.vy[pid] = uy / gam;
    out.vz[pid] = uz / gam;
    out.w[pid] = 1.0 / (double)ppc;
    out.id[pid] = pid;
}

// Moving window, counts of the shifted layout: new bin (i,j,k) = old bin
// (i+1,j,k) for i < nx-1; the last column receives the injected particles.
__global__ void k_shift_counts(const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ off, uint32_t ncells,
                               uint32_t nx, uint32_t ppc, uint32_t* __restrict__ cnt_new) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c > ncells) return;
    if (c == ncells) {
        cnt_new[c] = 0;
        return;
    }
    cnt_new[c] = c % nx == nx - 1 ? ppc : min(cnt[c + 1], off[c + 2] - off[c + 1]);
}

// Moving window relayout: new bin c <- old bin c+1 (the slots of an old
// column-0 bin, which lands on a new last-column bin, are the dropped ones);
// the new last-column bins are filled by the injector in place.
__global__ void __launch_bounds__(256) k_relayout_shift(const Aos src, const uint32_t* __restrict__ soff,
                                                        const uint32_t* __restrict__ cnt_new, const Aos dst,
                                                        const uint32_t* __restrict__ doff, uint32_t ncells,
                                                        const GridD gnew, int ppc, double u_th, uint64_t seed,
                                                        uint64_t pid0) {
    __shared__ uint32_t so[BPB + 1], sc[BPB], dof[BPB];
    const uint32_t nx = (uint32_t)gnew.nx;
    const uint32_t c0 = blockIdx.x * BPB;
    const int nb = (int)umin((uint32_t)BPB, ncells - c0);
    for (int b = threadIdx.x; b <= nb; b += blockDim.x) {
        so[b] = soff[umin(c0 + b + 1, ncells)];
        if (b < nb) {
            sc[b] = (c0 + b) % nx == nx - 1 ? 0u : cnt_new[c0 + b];
            dof[b] = doff[c0 + b];
        }
    }
    __syncthreads();
    for (uint32_t s = so[0] + threadIdx.x; s < so[nb]; s += blockDim.x) {
        const int b = find_bin(so, nb, s);
        const uint32_t r = s - so[b];
        if (r < sc[b]) copy_particle(src, s, dst, (uint64_t)dof[b] + r);
    }
    // injection into this block's last-column bins
    for (int t = threadIdx.x; t < nb * ppc; t += blockDim.x) {
        const int b = t / ppc, r = t % ppc;
        const uint32_t c = c0 + b;
        if (c % nx != nx - 1) continue;
        const uint32_t row = c / nx;  // j + ny*k
        const int j = (int)(row % (uint32_t)gnew.ny), k = (int)(row / (uint32_t)gnew.ny);
        const uint64_t pid = pid0 + (uint64_t)row * ppc + r;
        const uint64_t d = (uint64_t)dof[b] + r;
        const double px = __dadd_rn(gnew.ox, __dmul_rn(__dadd_rn((double)(nx - 1), uniform01(seed, pid, 6)), gnew.dx));
        const double py = __dadd_rn(gnew.oy, __dmul_rn(__dadd_rn((double)j, uniform01(seed, pid, 7)), gnew.dy));
        const double pz = __dadd_rn(gnew.oz, __dmul_rn(__dadd_rn((double)k, uniform01(seed, pid, 8)), gnew.dz));
        const double ux = u_th * gaussian(seed, pid, 0);
        const double uy = u_th * gaussian(seed, pid, 1);
        const double uz = u_th * gaussian(seed, pid, 2);
        const double gam = sqrt(1.0 + ux * ux + uy * uy + uz * uz);
        store_record(dst.p + d, px, py, pz, ux / gam, uy / gam, uz / gam, 1.0 / (double)ppc, pid);
    }
}

// make_workload (workload.hpp:75-125): particle pid = cell-major (x fastest),
// then a px*py*pz sub-lattice in the cell (x fastest); Maxwellian velocities,
// optional shear drift, truncation at the displacement cap; W = 1.
__global__ void k_make_workload(const GridD g, int ppc, int px, int py, int pz, double vth, int drift, double ax,
                                double ay, double az, double cap, uint64_t seed, const Soa out, uint64_t n) {
    const uint64_t pid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pid >= n) return;
    const uint64_t cell = pid / (uint64_t)ppc;
    const int r = (int)(pid % (uint64_t)ppc);
    const int a = r % px, b = (r / px) % py, c = r / (px * py);
    const int i = (int)(cell % (uint64_t)g.nx);
    const int j = (int)((cell / (uint64_t)g.nx) % (uint64_t)g.ny);
    const int k = (int)(cell / ((uint64_t)g.nx * (uint64_t)g.ny));
    const double X = __dadd_rn(g.ox, __dmul_rn(__dadd_rn((double)i, __ddiv_rn(__dadd_rn((double)a, 0.5), (double)px)), g.dx));
    const double Y = __dadd_rn(g.oy, __dmul_rn(__dadd_rn((double)j, __ddiv_rn(__dadd_rn((double)b, 0.5), (double)py)), g.dy));
    const double Z = __dadd_rn(g.oz, __dmul_rn(__dadd_rn((double)k, __ddiv_rn(__dadd_rn((double)c, 0.5), (double)pz)), g.dz));
    out.x[pid] = X;
    out.y[pid] = Y;
    out.z[pid] = Z;
    double VX = __dmul_rn(vth, gaussian(seed, pid, 0));
    double VY = __dmul_rn(vth, gaussian(seed, pid, 1));
    double VZ = __dmul_rn(vth, gaussian(seed, pid, 2));
    if (drift) {
        const double tau = 2.0 * 3.141592653589793;
        VX = __dadd_rn(VX, __dmul_rn(ax, cos(__ddiv_rn(__dmul_rn(tau, __dsub_rn(Y, g.oy)), g.Ly))));
        VY = __dadd_rn(VY, __dmul_rn(ay, cos(__ddiv_rn(__dmul_rn(tau, __dsub_rn(Z, g.oz)), g.Lz))));
        VZ = __dadd_rn(VZ, __dmul_rn(az, cos(__ddiv_rn(__dmul_rn(tau, __dsub_rn(X, g.ox)), g.Lx))));
    }
    const double speed = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(VX, VX), __dmul_rn(VY, VY)), __dmul_rn(VZ, VZ)));
    if (speed > cap) {
        const double sc = __dmul_rn(__ddiv_rn(cap, speed), 1.0 - 0x1.0p-40);
        VX = __dmul_rn(VX, sc);
        VY = __dmul_rn(VY, sc);
        VZ = __dmul_rn(VZ, sc);
    }
    out.vx[pid] = VX;
    out.vy[pid] = VY;
    out.vz[pid] = VZ;
    out.w[pid] = 1.0;
    out.id[pid] = pid;
}

// ---------------------------------------------------------------------------
// host launchers

void launch_cells(const GridD& g, const double* x, const double* y, const double* z, uint64_t n, uint32_t* cell,
                  int* err, cudaStream_t st) {
    if (!n) return;
    k_cells<<<div_up((long long)n, 256), 256, 0, st>>>(g, x, y, z, n, cell, err);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

void launch_advance(const GridD& g, double dt, double cap2, double* x, double* y, double* z, const double* vx,
                    const double* vy, const double* vz, uint64_t n, unsigned long long* moved, int* err,
                    cudaStream_t st) {
    if (!n) return;
    k_advance<<<div_up((long long)n, 256), 256, 0, st>>>(g, dt, cap2, x, y, z, vx, vy, vz, n, moved, err);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

void launch_generate_plasma(const GridD& g, int ppc, double u_th, uint64_t seed, Soa out, cudaStream_t st) {
    const uint64_t n = (uint64_t)(g.sx_hi - g.sx_lo) * g.ny * g.nz * (uint64_t)ppc;
    if (!n) return;
    k_generate<<<div_up((long long)n, 256), 256, 0, st>>>(g, ppc, u_th, seed, out, n);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

void launch_pack_planes(const double* F, int comps, int nx, int ny, int nz, int p0, int np, double* out,
                        cudaStream_t st) {
    const long long total = (long long)comps * np * ny * nz;
    if (!total) return;
    k_pack_planes<<<(int)std::min<long long>(div_up(total, 256), 148 * 8), 256, 0, st>>>(F, comps, nx, ny, nz, p0, np,
                                                                                        out);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

void launch_add_planes(double* F, int comps, int nx, int ny, int nz, int p0, int np, const double* in,
                       cudaStream_t st) {
    const long long total = (long long)comps * np * ny * nz;
    if (!total) return;
    k_add_planes<<<(int)std::min<long long>(div_up(total, 256), 148 * 8), 256, 0, st>>>(F, comps, nx, ny, nz, p0, np,
                                                                                       in);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

void launch_generate_lwfa(const GridD& g, const uint32_t* pfx_dev, uint64_t nbg, uint64_t n, int ppc, double u_th,
                          double ux_min, double ux_max, double bx0, double bx1, uint64_t seed, Soa out,
                          cudaStream_t st) {
    if (!n) return;
    k_generate_lwfa<<<div_up((long long)n, 256), 256, 0, st>>>(g, pfx_dev, nbg, n, ppc, u_th, ux_min, ux_max, bx0, bx1,
                                                              seed, out);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

void launch_make_workload(const GridD& g, int ppc, double vth, int drift, const double amp[3], double cap,
                          uint64_t seed, Soa out, cudaStream_t st) {
    // detail::sublattice_dims (workload.hpp:50-65): px >= py >= pz, px*py*pz == ppc
    int cb = 1;
    while ((cb + 1) * (cb + 1) * (cb + 1) <= ppc) ++cb;
    int pz = 1;
    for (int d = cb; d >= 1; --d)
        if (ppc % d == 0) {
            pz = d;
            break;
        }
    const int rem = ppc / pz;
    int sq = 1;
    while ((sq + 1) * (sq + 1) <= rem) ++sq;
    int py = 1;
    for (int d = sq; d >= 1; --d)
        if (rem % d == 0) {
            py = d;
            break;
        }
    const int px = rem / py;
    const uint64_t n = (uint64_t)g.ncells * (uint64_t)ppc;
    if (!n) return;
    k_make_workload<<<div_up((long long)n, 256), 256, 0, st>>>(g, ppc, px, py, pz, vth, drift, amp[0], amp[1], amp[2],
                                                              cap, seed, out, n);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// BinStore

BinStore::~BinStore() {
    if (hcounters) cudaFreeHost(hcounters);
}

void BinStore::init(const picgpu_grid& grid, double gap_ratio, uint32_t mg, cudaStream_t stream) {
    hg = grid;
    g = make_grid(grid);
    onepg = 1.0 + gap_ratio;
    min_gap = mg;
    st = stream;
    int dev = 0;
    PICGPU_CUDA_TRY(cudaGetDevice(&dev));
    PICGPU_CUDA_TRY(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t nc = g.ncells;
    off.ensure((nc + 1) * 4);
    off2.ensure((nc + 1) * 4);
    cnt.ensure(nc * 4);
    // start doubles as the (nc+1)-entry held-count scratch of a rebuild:
    // sized now, so no rebuild pays a (device-synchronising) regrowth
    start.ensure((nc + 1) * 4);
    endp.ensure(nc * 4);
    cnt2.ensure((nc + 1) * 4);
    caps.ensure((nc + 1) * 8);
    counters.ensure(sizeof(StepCounters));
    if (!hcounters) PICGPU_CUDA_TRY(cudaMallocHost((void**)&hcounters, sizeof(StepCounters)));
    PICGPU_CUDA_TRY(cudaMemsetAsync(off.p, 0, (nc + 1) * 4, st));
    PICGPU_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, nc * 4, st));
    locks.ensure(nc * 4 + 4);
    PICGPU_CUDA_TRY(cudaMemsetAsync(locks.p, 0, nc * 4 + 4, st));
    holes.ensure(nc * 4 + 4);
    PICGPU_CUDA_TRY(cudaMemsetAsync(holes.p, 0, nc * 4 + 4, st));
    capacity = 0;
    n = 0;
}

// caps (u32, ncells+1 entries, last 0) -> off2 (u32 offsets) ; capacity_next.
void BinStore::layout_from_counts(uint64_t) {
    const size_t nc = g.ncells;
    DevBuf& off64 = keys2;  // scratch: (nc+1) u64
    off64.ensure((nc + 1) * 8);
    exclusive_sum_u32_to_u64(caps.as<uint32_t>(), off64.as<unsigned long long>(), nc + 1, sort_tmp, st);
    unsigned long long total = 0;
    PICGPU_CUDA_TRY(cudaMemcpyAsync(&total, off64.as<unsigned long long>() + nc, 8, cudaMemcpyDeviceToHost, st));
    PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
    if (total >= 0xffffffffull) throw Status{PICGPU_ELENGTH, "gpma: capacity overflow"};
    k_u64_to_u32<<<div_up((long long)nc + 1, 256), 256, 0, st>>>(off64.as<unsigned long long>(),
                                                                 off2.as<uint32_t>(), nc + 1);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
    capacity_next = total;
}

void BinStore::full_sort_from_B(uint64_t np, uint32_t* perm_out_dev, cudaEvent_t fields_ready) {
    const size_t nc = g.ncells;
    if (np >= 0xffffffffull) throw Status{PICGPU_ELENGTH, "gpma: particle count exceeds 32-bit slots"};
    keys.ensure(np * 4 + 4);
    vals.ensure(np * 4 + 4);
    vals2.ensure(np * 4 + 4);
    skeys.ensure(np * 4 + 4);
    const Soa b = B.soa();
    const uint32_t *sk = skeys.as<uint32_t>(), *sv = vals2.as<uint32_t>();  // sorted keys / permutation
    StepCounters* ctr = counters.as<StepCounters>();
    PICGPU_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(StepCounters), st));
    PICGPU_CUDA_TRY(cudaMemsetAsync(start.p, 0, nc * 4, st));
    PICGPU_CUDA_TRY(cudaMemsetAsync(endp.p, 0, nc * 4, st));
    if (np) {
        launch_cells(g, b.x, b.y, b.z, np, keys.as<uint32_t>(), &ctr->err, st);
        int bits = 1;
        while (bits < 32 && (1ull << bits) < nc) ++bits;
        keys2.ensure(np * 4 + 4);
        radix_sort_pairs(keys.as<uint32_t>(), skeys.as<uint32_t>(), keys2.as<uint32_t>(), nullptr, vals2.as<uint32_t>(),
                         vals.as<uint32_t>(), np, bits, sort_tmp, st);
        k_boundaries<<<div_up((long long)np, 256), 256, 0, st>>>(sk, np, start.as<uint32_t>(), endp.as<uint32_t>());
        note_launch();
    }
    k_counts_caps<<<div_up((long long)nc + 1, 256), 256, 0, st>>>(start.as<uint32_t>(), endp.as<uint32_t>(),
                                                                  (uint32_t)nc, cnt.as<uint32_t>(),
                                                                  caps.as<uint32_t>(), onepg, min_gap);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
    PICGPU_CUDA_TRY(cudaMemcpyAsync(hcounters, ctr, sizeof(StepCounters), cudaMemcpyDeviceToHost, st));
    layout_from_counts(np);  // synchronises
    if (hcounters->err)
        throw Status{hcounters->err, g.slab ? "slab: particle outside the slab's owned cells (or non-finite)"
                                            : "cell_of: non-finite particle position"};
    A.ensure(capacity_next);
    swap_buf(off, off2);
    if (nc) {
        k_fill_slack<<<div_up((long long)nc, BPB), 256, 0, st>>>(A.aos(), off.as<uint32_t>(), cnt.as<uint32_t>(),
                                                                 (uint32_t)nc);
        note_launch();
    }
    if (np) {
        if (fields_ready) PICGPU_CUDA_TRY(cudaStreamWaitEvent(st, fields_ready, 0));
        k_gather_sorted<Soa><<<div_up((long long)np, 256), 256, 0, st>>>(b, sv, sk, start.as<uint32_t>(),
                                                                    off.as<uint32_t>(), A.aos(), np);
        note_launch();
        PICGPU_CUDA_TRY(cudaGetLastError());
        if (perm_out_dev) PICGPU_CUDA_TRY(cudaMemcpyAsync(perm_out_dev, sv, np * 4, cudaMemcpyDeviceToDevice, st));
    }
    capacity = capacity_next;
    n = np;
    PICGPU_CUDA_TRY(cudaMemsetAsync(holes.p, 0, nc * 4 + 4, st));  // fresh bins are packed
    // the spare store (relayout / rebuild target) gets the same capacity + headroom
    // now, outside any timed step, instead of at the first rebuild
    A2.ensure(capacity + capacity / 8);
    hl.ensure((capacity + capacity / 8) * 4 + 4);
}

unsigned long long* BinStore::moved_parts() {
    if (!mvpart.p) {
        mvpart.ensure((size_t)kMovedParts * 128);
        PICGPU_CUDA_TRY(cudaMemsetAsync(mvpart.p, 0, (size_t)kMovedParts * 128, st));
    }
    return mvpart.as<unsigned long long>();
}

void BinStore::fill_holes() {
    const size_t nc = g.ncells;
    if (!nc) return;
    k_fill_holes<<<div_up((long long)nc, 256), 256, 0, st>>>(A.aos(), off.as<uint32_t>(), cnt.as<uint32_t>(),
                                                             holes.as<uint32_t>(), (uint32_t)nc);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

void BinStore::relayout() {
    const size_t nc = g.ncells;
    fill_holes();
    k_caps_from_cnt<<<div_up((long long)nc + 1, 256), 256, 0, st>>>(cnt.as<uint32_t>(), (uint32_t)nc,
                                                                    caps.as<uint32_t>(), onepg, min_gap);
    note_launch();
    layout_from_counts(n);
    A2.ensure(capacity_next);
    if (nc) {
        k_relayout_fill<<<div_up((long long)nc, 256), 256, 0, st>>>(A.aos(), off.as<uint32_t>(), cnt.as<uint32_t>(),
                                                                    cnt.as<uint32_t>(), A2.aos(),
                                                                    off2.as<uint32_t>(), (uint32_t)nc);
        note_launch();
        PICGPU_CUDA_TRY(cudaGetLastError());
    }
    swap_aos(A, A2);
    swap_buf(off, off2);
    capacity = capacity_next;
}

void BinStore::compact_to_B() {
    const size_t nc = g.ncells;
    fill_holes();
    DevBuf& held = start;  // u32 scratch (nc) -- holds min(cnt, cap); needs nc+1
    held.ensure((nc + 1) * 4);
    k_held<<<div_up((long long)nc + 1, 256), 256, 0, st>>>(cnt.as<uint32_t>(), off.as<uint32_t>(), (uint32_t)nc,
                                                           held.as<uint32_t>());
    note_launch();
    DevBuf& off64 = keys2;
    off64.ensure((nc + 1) * 8);
    exclusive_sum_u32_to_u64(held.as<uint32_t>(), off64.as<unsigned long long>(), nc + 1, sort_tmp, st);
    k_u64_to_u32<<<div_up((long long)nc + 1, 256), 256, 0, st>>>(off64.as<unsigned long long>(),
                                                                 off2.as<uint32_t>(), nc + 1);
    note_launch();
    B.ensure(n + mcap + 1);
    if (nc) {
        k_relayout<<<div_up((long long)nc, BPB), 256, 0, st>>>(A.aos(), off.as<uint32_t>(), cnt.as<uint32_t>(),
                                                               B.soa(), off2.as<uint32_t>(), (uint32_t)nc);
        note_launch();
        PICGPU_CUDA_TRY(cudaGetLastError());
    }
}

void BinStore::ensure_movers(size_t m) {
    if (m <= mcap) return;
    M.ensure(m);
    mcell.ensure(m * 4);
    mslot.ensure(m * 4);
    mbin.ensure(m * 4);
    mcellseg.ensure(m * 4);
    ovf.ensure(m * 4);
    ovf_left.ensure(m * 4);
    mcap = m;
}

void BinStore::ensure_movers_keep(size_t m, size_t keep) {
    if (m <= mcap) return;
    SoaBuf M2;
    DevBuf mcell2;
    M2.ensure(m);
    mcell2.ensure(m * 4);
    if (keep) {
        for (int a = 0; a < 8; ++a)
            PICGPU_CUDA_TRY(cudaMemcpyAsync(M2.a[a].p, M.a[a].p, keep * 8, cudaMemcpyDeviceToDevice, st));
        PICGPU_CUDA_TRY(cudaMemcpyAsync(mcell2.p, mcell.p, keep * 4, cudaMemcpyDeviceToDevice, st));
    }
    PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
    swap_soa(M, M2);
    swap_buf(mcell, mcell2);
    mslot.ensure(m * 4);
    mbin.ensure(m * 4);
    mcellseg.ensure(m * 4);
    ovf.ensure(m * 4);
    ovf_left.ensure(m * 4);
    mcap = m;
}

void BinStore::enqueue_detect(bool push, double dt, double cap2) {
    const size_t nc = g.ncells;
    ensure_movers(std::max<size_t>(size_t(1) << 16, n / 4));
    if (g.slab) {
        const size_t want = std::max<size_t>(size_t(1) << 16, n / 4);
        if (want > lcap) {
            lrec.ensure(want * 2 * 8 * sizeof(double));
            lcap = want;
        }
    }
    StepCounters* ctr = counters.as<StepCounters>();
    PICGPU_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(StepCounters), st));
    if (!nc || !n) return;
    constexpr int UNR = PICGPU_PUSH_UNR;
    const int blocks = (int)((capacity + PICGPU_PUSH_NT * UNR - 1) / (PICGPU_PUSH_NT * UNR));
    const bool p2 = g.pow2x && g.pow2y && g.pow2z && g.gpow2Lx && g.pow2Ly && g.pow2Lz;
    hl.ensure(capacity * 4 + 4);
    auto* kern = push ? (p2 ? k_push<true, UNR, true> : k_push<true, UNR, false>)
                      : (p2 ? k_push<false, UNR, true> : k_push<false, UNR, false>);
    kern<<<blocks, PICGPU_PUSH_NT, 0, st>>>(g, A.aos(), capacity, dt, cap2, M.soa(), mcell.as<uint32_t>(),
                                            (uint32_t)mcap, off.as<uint32_t>(), holes.as<uint32_t>(),
                                            hl.as<uint32_t>(), ctr, lrec.as<double>(), (uint32_t)lcap,
                                            mslot.as<uint32_t>(), mbin.as<uint32_t>(), moved_parts());
    k_fold_moved<<<1, 256, 0, st>>>(moved_parts(), ctr);
    note_launch(2);
    PICGPU_CUDA_TRY(cudaGetLastError());
    if (push) {
        // the departures' hole-list entries (before any arrival looks for holes)
        k_departures<<<num_sms * 8, 256, 0, st>>>(counters.as<StepCounters>(), (uint32_t)mcap, mslot.as<uint32_t>(),
                                                  mbin.as<uint32_t>(), off.as<uint32_t>(), holes.as<uint32_t>(),
                                                  hl.as<uint32_t>());
        note_launch();
        PICGPU_CUDA_TRY(cudaGetLastError());
    }
    // no compaction: departures left holes (GPMA gaps), filled by the arrivals
}

void BinStore::enqueue_import(const double* rec_dev, uint32_t nimp, uint32_t base) {
    k_import<<<div_up((long long)std::max<uint32_t>(nimp, 1u), 256), 256, 0, st>>>(
        g, rec_dev, nimp, base, M.soa(), mcell.as<uint32_t>(), counters.as<StepCounters>());
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

void BinStore::enqueue_import_dev(const double* from_left, const double* from_right, const uint32_t* cnt_dev,
                                  uint32_t B) {
    k_import_plan<<<1, 1, 0, st>>>(cnt_dev, B, (uint32_t)mcap, counters.as<StepCounters>());
    k_import_dev<<<div_up(2ll * B, 256), 256, 0, st>>>(g, from_left, from_right, B, M.soa(), mcell.as<uint32_t>(),
                                                      counters.as<StepCounters>());
    note_launch(2);
    PICGPU_CUDA_TRY(cudaGetLastError());
}

void BinStore::enqueue_migrate() {
    const size_t nc = g.ncells;
    StepCounters* ctr = counters.as<StepCounters>();
    if (nc) {
        static const int mult = [] {
            const char* e = std::getenv("PICGPU_INSERT_BLOCKS");
            return e ? std::max(1, std::atoi(e)) : 4;
        }();
        k_insert<<<num_sms * mult, 256, 0, st>>>(M.soa(), mcell.as<uint32_t>(), (uint32_t)mcap, ctr, A.aos(),
                                              off.as<uint32_t>(), cnt.as<uint32_t>(), ovf.as<uint32_t>(),
                                              holes.as<uint32_t>(), hl.as<uint32_t>());
        note_launch();
        PICGPU_CUDA_TRY(cudaGetLastError());
        // borrow_insert for the full-bin arrivals; no work when there are none
        k_borrow<<<num_sms, 128, 0, st>>>(ctr, M.soa(), mcell.as<uint32_t>(), ovf.as<uint32_t>(),
                                          ovf_left.as<uint32_t>(), A.aos(), off.as<uint32_t>(), cnt.as<uint32_t>(),
                                          holes.as<uint32_t>(), hl.as<uint32_t>(), locks.as<unsigned int>(),
                                          (uint32_t)nc, kBorrowScanBins);
        note_launch();
        PICGPU_CUDA_TRY(cudaGetLastError());
    }
    PICGPU_CUDA_TRY(cudaMemcpyAsync(hcounters, ctr, sizeof(StepCounters), cudaMemcpyDeviceToHost, st));
}

void BinStore::enqueue_incremental(bool push, double dt, double cap2) {
    enqueue_detect(push, dt, cap2);
    if (!g.ncells || !n) {
        PICGPU_CUDA_TRY(cudaMemcpyAsync(hcounters, counters.p, sizeof(StepCounters), cudaMemcpyDeviceToHost, st));
        return;
    }
    enqueue_migrate();
}

void BinStore::enqueue_fused(int order, double q, double* J, double dt, double cap2, cudaEvent_t after_kernel,
                             bool migrate, int kernel) {
    ensure_movers(std::max<size_t>(size_t(1) << 16, n / 4));
    if (g.slab) {
        const size_t want = std::max<size_t>(size_t(1) << 16, n / 4);
        if (want > lcap) {
            lrec.ensure(want * 2 * 8 * sizeof(double));
            lcap = want;
        }
    }
    StepCounters* ctr = counters.as<StepCounters>();
    PICGPU_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(StepCounters), st));
    if (!g.ncells || !n) {
        PICGPU_CUDA_TRY(cudaMemcpyAsync(hcounters, ctr, sizeof(StepCounters), cudaMemcpyDeviceToHost, st));
        return;
    }
    hl.ensure(capacity * 4 + 4);
    segcnt.ensure(((size_t)kMaxFusedCtas + 1) * 4);
    PushCtx pc{A.aos(), dt, cap2, mslot.as<uint32_t>(), mbin.as<uint32_t>(), mcellseg.as<uint32_t>(),
               mcell.as<uint32_t>(), (uint32_t)mcap, 0u, 0u, 0u, segcnt.as<uint32_t>(), ctr,
               lrec.as<double>(), (uint32_t)lcap, off.as<uint32_t>(), holes.as<uint32_t>(), hl.as<uint32_t>()};
    launch_deposit_current_push(order, g, pc, d_off(), d_cnt(), q, J, num_sms, st, kernel);  // sets nseg, segcap
    if (after_kernel) PICGPU_CUDA_TRY(cudaEventRecord(after_kernel, st));
    launch_movers(order, g, pc, M.soa(), d_off(), holes.as<uint32_t>(), hl.as<uint32_t>(), q, J, num_sms, st);
    if (migrate)
        enqueue_migrate();
    else
        PICGPU_CUDA_TRY(cudaMemcpyAsync(hcounters, ctr, sizeof(StepCounters), cudaMemcpyDeviceToHost, st));
}

void BinStore::push_and_resort(bool push, double dt, double cap2, StepCounters& out) {
    const size_t nc = g.ncells;
    StepCounters* ctr = counters.as<StepCounters>();
    PICGPU_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(StepCounters), st));
    if (nc && n && push) {
        constexpr int UNR = PICGPU_PUSH_UNR;
        const int blocks = (int)((capacity + PICGPU_PUSH_NT * UNR - 1) / (PICGPU_PUSH_NT * UNR));
        const bool p2 = g.pow2x && g.pow2y && g.pow2z && g.gpow2Lx && g.pow2Ly && g.pow2Lz;
        auto* kern = p2 ? k_push<true, UNR, true, false> : k_push<true, UNR, false, false>;
        kern<<<blocks, PICGPU_PUSH_NT, 0, st>>>(g, A.aos(), capacity, dt, cap2, M.soa(), mcell.as<uint32_t>(),
                                                (uint32_t)mcap, off.as<uint32_t>(), holes.as<uint32_t>(),
                                                hl.as<uint32_t>(), ctr, lrec.as<double>(), (uint32_t)lcap,
                                                mslot.as<uint32_t>(), mbin.as<uint32_t>(), moved_parts());
        k_fold_moved<<<1, 256, 0, st>>>(moved_parts(), ctr);
        note_launch();
        note_launch();
        PICGPU_CUDA_TRY(cudaGetLastError());
    }
    PICGPU_CUDA_TRY(cudaMemcpyAsync(hcounters, ctr, sizeof(StepCounters), cudaMemcpyDeviceToHost, st));
    PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
    out = *hcounters;
    if (out.err) return;
    // global_sort (sort_policy.hpp:83): stable counting sort of the whole
    // store in storage order, fresh slack
    resort_records();
}

// global_sort straight from the records: after fill_holes (the packing every
// download applies, so the order sorted is the storage order a download
// reports) the store's slots in storage order are the packed store's order
// (slack keys ncells and sorts last), so a stable radix sort of (cell of
// slot, slot) followed by a record gather into the fresh layout IS
// gpma_build's counting sort of the packed store -- with no compaction pass
// and no detour through the SoA staging (C3: the compaction alone was 40 ms).
void BinStore::resort_records() {
    const size_t nc = g.ncells;
    const uint64_t slots = capacity;
    if (!nc) return;
    fill_holes();
    keys.ensure(slots * 4 + 4);
    vals.ensure(slots * 4 + 4);
    vals2.ensure(slots * 4 + 4);
    skeys.ensure(slots * 4 + 4);
    const uint32_t *sk = skeys.as<uint32_t>(), *sv = vals2.as<uint32_t>();  // sorted keys / slot permutation
    StepCounters* ctr = counters.as<StepCounters>();
    PICGPU_CUDA_TRY(cudaMemsetAsync(start.p, 0, nc * 4, st));
    PICGPU_CUDA_TRY(cudaMemsetAsync(endp.p, 0, nc * 4, st));
    if (slots) {
        k_slot_keys<<<div_up((long long)slots, 256), 256, 0, st>>>(g, A.aos(), slots, keys.as<uint32_t>(), &ctr->err);
        note_launch();
        int bits = 1;
        while (bits < 32 && (1ull << bits) < nc + 1) ++bits;
        keys2.ensure(slots * 4 + 4);
        radix_sort_pairs(keys.as<uint32_t>(), skeys.as<uint32_t>(), keys2.as<uint32_t>(), nullptr, vals2.as<uint32_t>(),
                         vals.as<uint32_t>(), slots, bits, sort_tmp, st);
        if (n) {  // the first n sorted keys are the particles' cells
            k_boundaries<<<div_up((long long)n, 256), 256, 0, st>>>(sk, n, start.as<uint32_t>(), endp.as<uint32_t>());
            note_launch();
        }
    }
    k_counts_caps<<<div_up((long long)nc + 1, 256), 256, 0, st>>>(start.as<uint32_t>(), endp.as<uint32_t>(),
                                                                  (uint32_t)nc, cnt.as<uint32_t>(),
                                                                  caps.as<uint32_t>(), onepg, min_gap);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
    PICGPU_CUDA_TRY(cudaMemcpyAsync(hcounters, ctr, sizeof(StepCounters), cudaMemcpyDeviceToHost, st));
    layout_from_counts(n);  // synchronises
    if (hcounters->err) throw Status{hcounters->err, "cell_of: non-finite particle position"};
    A2.ensure(capacity_next);
    k_fill_slack<<<div_up((long long)nc, BPB), 256, 0, st>>>(A2.aos(), off2.as<uint32_t>(), cnt.as<uint32_t>(),
                                                             (uint32_t)nc);
    note_launch();
    if (n) {
        k_gather_sorted<Aos><<<div_up((long long)n, 256), 256, 0, st>>>(A.aos(), sv, sk, start.as<uint32_t>(),
                                                                         off2.as<uint32_t>(), A2.aos(), n);
        note_launch();
    }
    PICGPU_CUDA_TRY(cudaGetLastError());
    swap_aos(A, A2);
    swap_buf(off, off2);
    capacity = capacity_next;
    PICGPU_CUDA_TRY(cudaMemsetAsync(holes.p, 0, nc * 4 + 4, st));  // fresh bins are packed
    hl.ensure(capacity * 4 + 4);
}

void BinStore::shift_window(const picgpu_grid& shifted, int ppc, double u_th, uint64_t seed, uint64_t pid0,
                            uint64_t& dropped, uint64_t& injected) {
    const size_t nc = g.ncells;
    injected = (uint64_t)g.ny * g.nz * (uint64_t)ppc;
    if (!nc) return;
    fill_holes();
    // counts and fresh-slack layout of the shifted grid (bins keep their order)
    cnt2.ensure((nc + 1) * 4);
    k_shift_counts<<<div_up((long long)nc + 1, 256), 256, 0, st>>>(cnt.as<uint32_t>(), off.as<uint32_t>(),
                                                                   (uint32_t)nc, (uint32_t)g.nx, (uint32_t)ppc,
                                                                   cnt2.as<uint32_t>());
    note_launch();
    DevBuf& tot64 = vals;  // particles of the new layout: sum of the new counts
    tot64.ensure((nc + 1) * 8);
    exclusive_sum_u32_to_u64(cnt2.as<uint32_t>(), tot64.as<unsigned long long>(), nc + 1, sort_tmp, st);
    unsigned long long nnew = 0;
    PICGPU_CUDA_TRY(cudaMemcpyAsync(&nnew, tot64.as<unsigned long long>() + nc, 8, cudaMemcpyDeviceToHost, st));
    k_caps_from_cnt<<<div_up((long long)nc + 1, 256), 256, 0, st>>>(cnt2.as<uint32_t>(), (uint32_t)nc,
                                                                    caps.as<uint32_t>(), onepg, min_gap);
    note_launch();
    layout_from_counts(0);  // synchronises
    A2.ensure(capacity_next + capacity_next / 8);
    hg = shifted;
    g = make_grid(shifted);
    k_fill_slack<<<div_up((long long)nc, BPB), 256, 0, st>>>(A2.aos(), off2.as<uint32_t>(), cnt2.as<uint32_t>(),
                                                             (uint32_t)nc);
    note_launch();
    k_relayout_shift<<<div_up((long long)nc, BPB), 256, 0, st>>>(A.aos(), off.as<uint32_t>(), cnt2.as<uint32_t>(),
                                                                 A2.aos(), off2.as<uint32_t>(), (uint32_t)nc, g, ppc,
                                                                 u_th, seed, pid0);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
    swap_aos(A, A2);
    swap_buf(off, off2);
    swap_buf(cnt, cnt2);
    capacity = capacity_next;
    dropped = n + injected - nnew;
    n = nnew;
}

bool BinStore::finish_incremental(StepCounters& out) {
    const size_t nc = g.ncells;
    PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
    out = *hcounters;
    if (out.err) return false;
    const bool mover_overflow = out.nmovers > mcap || out.mover_drop > 0 || movers_dropped;
    // (fused step: CTA segments hold half of mcap, the overflow segment the rest;
    // after a drop the buffers grow to twice the movers seen)
    const uint32_t nmovers_seen =
        movers_dropped ? (uint32_t)std::max<size_t>(mcap, out.nmovers)
                       : (uint32_t)std::min<uint64_t>(0xffffffffull / 4,
                                                      (uint64_t)(out.nmovers + out.mover_drop) *
                                                          (out.mover_drop ? 2 : 1));
    movers_dropped = false;
    // unplaced arrivals (no donor found); borrowed ones already sit in their bins
    const uint32_t left = out.nleft;
    const uint32_t* left_list = ovf_left.as<uint32_t>();
    borrowed += out.nborrowed;
    if (!mover_overflow && !left) return false;
    fill_holes();  // the layouts below need packed bins
    if (!mover_overflow) {
        // Gpma::rebuild (gpma.hpp:119-122, :130-143): fresh slack from the true
        // counts (cnt includes the unplaced arrivals), held particles keep their
        // slot order, the unplaced arrivals follow them.
        DevBuf& held = start;
        held.ensure((nc + 1) * 4);
        k_held<<<div_up((long long)nc + 1, 256), 256, 0, st>>>(cnt.as<uint32_t>(), off.as<uint32_t>(), (uint32_t)nc,
                                                               held.as<uint32_t>());
        note_launch();
        k_caps_from_cnt<<<div_up((long long)nc + 1, 256), 256, 0, st>>>(cnt.as<uint32_t>(), (uint32_t)nc,
                                                                        caps.as<uint32_t>(), onepg, min_gap);
        note_launch();
        layout_from_counts(n);
        A2.ensure(capacity_next);
        k_relayout_fill<<<div_up((long long)nc, 256), 256, 0, st>>>(A.aos(), off.as<uint32_t>(), cnt.as<uint32_t>(),
                                                                    cnt.as<uint32_t>(), A2.aos(),
                                                                    off2.as<uint32_t>(), (uint32_t)nc);
        note_launch();
        k_place_left<<<div_up(left, 256), 256, 0, st>>>(M.soa(), mcell.as<uint32_t>(), ovf_left.as<uint32_t>(), left,
                                                        A2.aos(), off2.as<uint32_t>(), held.as<uint32_t>());
        note_launch();
        PICGPU_CUDA_TRY(cudaGetLastError());
        swap_aos(A, A2);
        swap_buf(off, off2);
        capacity = capacity_next;
        ++rebuilds;
        return true;
    }
    // Mover-buffer overflow: stale movers still sit in their old bins.
    // Compact every held particle plus the unplaced arrivals and re-sort fully.
    compact_to_B();
    unsigned int h32 = 0;
    PICGPU_CUDA_TRY(cudaMemcpyAsync(&h32, off2.as<uint32_t>() + nc, 4, cudaMemcpyDeviceToHost, st));
    PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
    if (left) {
        k_append_overflow<<<div_up(left, 256), 256, 0, st>>>(M.soa(), left_list, left, B.soa(), h32);
        note_launch();
        PICGPU_CUDA_TRY(cudaGetLastError());
    }
    full_sort_from_B((uint64_t)h32 + left);
    ++rebuilds;
    ensure_movers(nmovers_seen + nmovers_seen / 2);
    return true;
}

}  // namespace picgpu
