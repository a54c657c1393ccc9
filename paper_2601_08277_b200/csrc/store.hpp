// store.hpp -- device-resident particle store in cell bins with slack (the GPU
// analogue of pic::Gpma, proj/include/pic/gpma.hpp:52-371).
//
// Unlike the reference GPMA, whose slots hold REFERENCES into an unsorted
// store, the bins here hold the particle data itself (one 64-byte record per
// slot: 7 FP64 + id): the deposition kernels then read particles cell-locally
// and coalesced straight from HBM.  Bin c owns slots [off[c], off[c+1]); its
// extent [off[c], off[c]+cnt[c]) holds its particles and holes, the slack
// follows; every slack slot and hole is an all-ones record (gap sentinel x) so
// the push and the deposits can stream over raw slots.  Capacities follow the
// reference's layout rule exactly, ceil(count*(1+gap_ratio)) + min_gap
// (gpma.hpp:274-281), so capacity and empty_slot_ratio match the reference.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace picgpu {

// Grow-only device allocation.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf();
    void ensure(size_t b);
    void release();
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

struct SoaBuf {
    DevBuf a[8];  // x y z vx vy vz w (double), id (uint64)
    size_t cap = 0;
    void ensure(size_t n);
    Soa soa() const;
};

// The binned store: one 64-byte record per slot (common.cuh, Part).
struct AosBuf {
    DevBuf a;
    size_t cap = 0;
    void ensure(size_t n);
    Aos aos() const { return Aos{a.as<Part>()}; }
};

constexpr int kBorrowScanBins = 4;
constexpr int kMovedParts = 256;  // k_push's moved-count partials (one 128-byte line each)  // GpmaConfig::borrow_scan_bins (gpma.hpp:25)

struct BinStore {
    GridD g{};
    picgpu_grid hg{};
    double onepg = 1.25;  // 1 + gap_ratio
    uint32_t min_gap = 2;
    int num_sms = 148;
    cudaStream_t st = nullptr;

    AosBuf A, A2;             // A: the binned store (records); A2: re-layout target
    SoaBuf B;                 // packed staging: uploads, generators, downloads, full re-sorts
    DevBuf off, cnt, off2;    // off: ncells+1 (u32), cnt: ncells (u32)
    DevBuf cnt2;              // counts of a layout being built (moving window)
    DevBuf keys, keys2, skeys, vals, vals2, start, endp, caps, sort_tmp;
    SoaBuf M;                 // mover records
    DevBuf mcell, ovf, ovf_left;  // mover target cell, overflow list, unplaced overflow
    DevBuf mslot, mbin;       // each mover's slot and old bin (fused step: by CTA segment)
    DevBuf mcellseg;          // fused step: movers' target cells by CTA segment
    DevBuf segcnt;            // fused step: movers per CTA segment
    DevBuf locks;             // per-bin try-locks of the borrow kernel (always released)
    DevBuf holes;             // per-bin holes in the extent [off, off+cnt) (GPMA gaps)
    DevBuf hl;                // per-bin hole lists, slot-indexed like the bins: bin c's holes
                              // are the slots hl[off[c] .. off[c]+holes[c]) (u32)
    DevBuf counters;          // StepCounters
    DevBuf mvpart;            // k_push's spread moved counts (kMovedParts x 128 bytes, kept zero between steps)
    StepCounters* hcounters = nullptr;  // pinned mirror

    uint64_t n = 0;           // particles
    uint64_t capacity = 0;    // slots in use (off[ncells])
    size_t mcap = 0;          // mover record capacity
    DevBuf lrec;              // slab leavers: [2][lcap][8] doubles (x y z vx vy vz w id)
    size_t lcap = 0;
    bool movers_dropped = false;  // a slab step dropped unrecorded movers (-> full re-sort)
    uint64_t rebuilds = 0;
    uint64_t borrowed = 0;    // arrivals placed by borrowing a neighbour's slack

    void init(const picgpu_grid& grid, double gap_ratio, uint32_t min_gap, cudaStream_t stream);
    ~BinStore();

    // B holds n packed particles: stable sort by cell into A with fresh slack
    // (gpma_build, gpma.hpp:379-402).  perm/starts/counts optionally exported.
    // `fields_ready` (optional): B's non-position fields may still be in flight
    // until this event -- the cell keys, the sort and the layout only need
    // x y z, so they overlap the rest of an upload; the gather waits for it.
    void full_sort_from_B(uint64_t n_particles, uint32_t* perm_out_dev = nullptr, cudaEvent_t fields_ready = nullptr);
    // Re-layout A's bins with fresh slack from the current counts (global_sort
    // on an already-binned store == identity permutation inside bins).
    void relayout();
    // Full stable re-sort of the binned store by the particles' current cells
    // (global_sort after a push: gpma_build on the packed store), records
    // gathered straight into a fresh layout.
    void resort_records();
    // A's valid particles compacted into B in storage order (bins ascending);
    // returns the packed offsets in `off2` (exclusive scan of cnt).
    void compact_to_B();
    // One incremental step, enqueued without host synchronisation: push
    // (optional) + detect (departures leave holes), migration into holes and
    // slack, borrow from the following bins for full bins; counters copied to
    // the host.
    void enqueue_incremental(bool push, double dt, double cap2);
    // The fused step (non-slab): push + detect + J of the particles that stay
    // in their cell in one pass over the bins, then the movers (records,
    // holes, their J) and the migration as in enqueue_incremental.  J (3 x
    // ncells, zeroed) receives the whole deposit unless the mover buffer
    // overflows (finish_incremental then re-sorts; the caller re-deposits).
    // `after_kernel` (optional) is recorded between the fused kernel and the movers.
    // migrate = false (slab step_begin): stop after the movers (the arrivals
    // are imported, deposited and migrated in step_end).
    void enqueue_fused(int order, double q, double* J, double dt, double cap2, cudaEvent_t after_kernel = nullptr,
                       bool migrate = true, int kernel = -1);
    // The same step in two halves around a slab exchange: detect (push +
    // move detection; leavers go to the exchange buffer
    // `lrec`), then migrate (optional arrivals appended to the movers,
    // insert, borrow).
    void enqueue_detect(bool push, double dt, double cap2);
    void enqueue_import(const double* rec_dev, uint32_t n, uint32_t base);
    // arrivals from a device-resident exchange: counts on the device (cnt_dev[0]
    // from the left, [1] from the right), at most B records per side
    void enqueue_import_dev(const double* from_left, const double* from_right, const uint32_t* cnt_dev, uint32_t B);
    void enqueue_migrate();
    // Synchronises, reads the counters and, if an arrival found no slack even
    // after borrowing (or the mover buffer overflowed), rebuilds by a full
    // re-sort.  Returns true when it rebuilt (fields deposited since the
    // enqueue must then be recomputed).
    bool finish_incremental(StepCounters& out);
    // Push (optional) with only the moved count, then a full stable counting
    // sort of the store (PICGPU_STEP_RESORT).  Synchronous.
    void push_and_resort(bool push, double dt, double cap2, StepCounters& out);
    // C4 moving window: drop x-column 0, shift the grid origin by one cell
    // (`shifted`), inject a fresh last column, re-sort.  Synchronous.
    void shift_window(const picgpu_grid& shifted, int ppc, double u_th, uint64_t seed, uint64_t pid0,
                      uint64_t& dropped, uint64_t& injected);

    uint32_t* d_off() const { return off.as<uint32_t>(); }
    unsigned long long* moved_parts();
    uint32_t* d_cnt() const { return cnt.as<uint32_t>(); }

    void ensure_movers(size_t m);
    void ensure_movers_keep(size_t m, size_t keep);  // grow, preserving the first `keep` records
    // packs every bin (holes filled from the bin's tail); cnt = particle counts
    void fill_holes();

   private:
    void layout_from_counts(uint64_t total_particles);  // caps + scan -> off2; returns via capacity_next
    uint64_t capacity_next = 0;
};

// radix_sort.cu: out[i] = sum(in[0..i)) (n entries)
void exclusive_sum_u32_to_u64(const uint32_t* in, unsigned long long* out, size_t n, DevBuf& tmp, cudaStream_t st);
// Stable LSD radix sort of n (key, value) pairs on the low `bits` key bits:
// the sorted pairs land in keys_out / vals_out; keys_in / vals_in are never
// written (vals_in == nullptr: the values are the indices 0..n-1, so vals_out
// receives the stable permutation); keys_tmp / vals_tmp are ping-pong scratch.
void radix_sort_pairs(const uint32_t* keys_in, uint32_t* keys_out, uint32_t* keys_tmp, const uint32_t* vals_in,
                      uint32_t* vals_out, uint32_t* vals_tmp, uint64_t n, int bits, DevBuf& tmp, cudaStream_t st);

}  // namespace picgpu
