// kernels.hpp -- host-side launchers shared between the translation units.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace picgpu {

// deposit_current.cu ---------------------------------------------------------
// J (3*ncells doubles: jx|jy|jz, pre-zeroed) += deposit of the binned store.
// J kernel families: the register-lane DFMA kernel ("lane", v3, the
// default), the warp-per-pencil DFMA kernel ("vector", orders 2/3; order 1
// falls back to the lane kernel) and the FP64 tensor-core DMMA pencil kernel
// ("matrix", deposit_pencil.cu, every order).
enum JKernel { kJDefault = -1, kJLane = 0, kJVector = 1, kJMatrix = 2 };
void launch_deposit_current(int order, const GridD& g, const CAos& p, const uint32_t* off, const uint32_t* cnt,
                            double q, double* j, int num_sms, cudaStream_t st, int kernel = kJDefault);

// Fused step kernel (the default session step): pic::advance + detect_moves +
// deposit_scalar in ONE pass over the bins.  Every particle is pushed in
// registers (bit-exact), written back, and -- if its cell did not change --
// deposited on the lane kernel's register window; a particle whose cell changed
// is listed (slot, old bin, new cell) for launch_movers, which copies it into
// the mover records, leaves a hole in its old bin and deposits its J with
// L2 reductions.  Slab stores: a particle that left the slab is listed with a
// kLeaveLeft/kLeaveRight code instead of a cell and exported by launch_movers.
struct PushCtx {
    Aos A;                   // the binned store (positions are updated in place)
    double dt, cap2;
    uint32_t* mslot;         // per mover, by CTA segment (nseg x segcap, then the overflow segment):
    uint32_t* mbin;          //   its slot, its old bin, its new cell
    uint32_t* mcellseg;
    uint32_t* mcell;         // compact target cells written by k_movers (k_insert's input)
    uint32_t mcap;           // compact mover capacity
    uint32_t segcap;         // entries per CTA segment (half of mcap over the CTAs of the fused kernel)
    uint32_t nseg;           // CTA segments (set by launch_deposit_current_push); segment nseg is
    uint32_t ovcap;          //   the shared overflow segment of ovcap entries at nseg * segcap
    uint32_t* seg_cnt;       // movers reserved per CTA segment (written at each CTA's end)
    StepCounters* ctr;       // -> nmovers / moved / mover_drop, err
    // slab stores: launch_movers writes particles that left the slab as exchange
    // records (x y z vx vy vz w id, by side) and leaves a hole; no deposit here
    double* L;               // [2][lcap][8]
    uint32_t lcap;
    const uint32_t* off;     // bin offsets, hole counts and lists (push_hole)
    uint32_t* holes;
    uint32_t* hl;
};
// Upper bound on the fused kernel's CTAs (size of seg_cnt).
constexpr uint32_t kMaxFusedCtas = 1u << 20;
// The fused form exists for the default lane kernel (v3) family only.
bool fused_step_available(int order, int kernel);
void launch_deposit_current_push(int order, const GridD& g, PushCtx& pc, const uint32_t* off,
                                 const uint32_t* cnt, double q, double* j, int num_sms, cudaStream_t st,
                                 int kernel = kJDefault);
// deposit_pencil.cu: the DMMA pencil kernel (J only / fused push + detect + J).
void launch_pencil_current(int order, const GridD& g, const CAos& p, const uint32_t* off, const uint32_t* cnt,
                           double q, double* j, int num_sms, cudaStream_t st);
void launch_pencil_current_push(int order, const GridD& g, PushCtx& pc, const uint32_t* off, const uint32_t* cnt,
                                double q, double* j, int num_sms, cudaStream_t st);
// Slab arrivals (mover records M[base .. base+n), appended by the import)
// deposited over their full window (RED.ADD.F64): the sender's fused pass
// left them out.
constexpr uint32_t kBaseFromCounters = 0xFFFFFFFFu;  // launch_deposit_records: arrivals start at ctr->nmovers
void launch_deposit_records(int order, const GridD& g, const Soa& M, const StepCounters* ctr, uint32_t base,
                            double q, double* j, int num_sms, cudaStream_t st);
// Movers of the fused kernel: slot -> mover record M[i] (+ hole in the old bin)
// and their J contribution (RED.ADD.F64); slab leavers -> exchange records.
void launch_movers(int order, const GridD& g, const PushCtx& pc, const Soa& M, const uint32_t* off,
                   uint32_t* holes, uint32_t* hl, double q, double* j, int num_sms, cudaStream_t st);

// deposit_density.cu ---------------------------------------------------------
// rho[node] = ordered sum (storage order) of quantity[s] * S (quantity NULL: qscale*w[s]), over binned,
// cell-sorted storage (bins ascending by cell, slot order within a bin).
// `scratch` holds (3*W + 1) doubles per slot (+1 byte per slot for TSC).
size_t density_scratch_bytes(int order, uint64_t slots);
void launch_deposit_density(int order, const GridD& g, const CAos& p, const double* quantity, double qscale,
                            const uint32_t* off,
                            const uint32_t* cnt, uint64_t slots, void* scratch, double* rho, cudaStream_t st);
// Unsorted storage: contributions to a node are merged by storage index across
// its source cells (k-way merge).  `rank[s]` is the storage index of slot s.
void launch_deposit_density_merge(int order, const GridD& g, const CAos& p, const double* quantity, double qscale,
                                  const uint32_t* rank, const uint32_t* off, const uint32_t* cnt, uint64_t slots,
                                  void* scratch, double* rho, cudaStream_t st);
// esirkepov.cu: charge-conserving J on the Yee faces (an extension; J zeroed by the caller).
void launch_deposit_esirkepov(int order, const GridD& g, const double* x0, const double* y0, const double* z0,
                              const double* x1, const double* y1, const double* z1, const double* w, double q,
                              double dt, uint64_t n, double* jx, double* jy, double* jz, int* err, cudaStream_t st);

// sorter.cu ------------------------------------------------------------------
// cell[p] = linear cell id (bit-identical cell_of); raises EINVAL on non-finite.
void launch_cells(const GridD& g, const double* x, const double* y, const double* z, uint64_t n, uint32_t* cell,
                  int* err, cudaStream_t st);
// Ballistic push, bit-identical to pic::advance; counts movers.
void launch_advance(const GridD& g, double dt, double cap2, double* x, double* y, double* z, const double* vx,
                    const double* vy, const double* vz, uint64_t n, unsigned long long* moved, int* err,
                    cudaStream_t st);
// Device-side SURVEY 8(d) plasma generator (cell-major, counter RNG).
void launch_generate_plasma(const GridD& g, int ppc, double u_th, uint64_t seed, Soa out, cudaStream_t st);
void launch_generate_lwfa(const GridD& g, const uint32_t* pfx_dev, uint64_t nbg, uint64_t n, int ppc, double u_th,
                          double ux_min, double ux_max, double bx0, double bx1, uint64_t seed, Soa out,
                          cudaStream_t st);
void launch_make_workload(const GridD& g, int ppc, double vth, int drift, const double amp[3], double cap,
                          uint64_t seed, Soa out, cudaStream_t st);
// Slab guard planes: pack planes [p0, p0+np) of a comps x (nx,ny,nz) field
// into [comp][plane][z][y], or add such a buffer back into them.
void launch_pack_planes(const double* F, int comps, int nx, int ny, int nz, int p0, int np, double* out,
                        cudaStream_t st);
void launch_add_planes(double* F, int comps, int nx, int ny, int nz, int p0, int np, const double* in,
                       cudaStream_t st);

}  // namespace picgpu
