// picgpu.hpp -- C++20 mirror of the reference's `pic::` hot-path interface,
// implemented on the C ABI of picgpu.h (link with -lpicgpu).
//
// Same names, argument meaning, value semantics and exception types as the
// reference headers (paths under proj/include/pic/), so a call site switches
// from `pic::` to `picgpu::` without other changes:
//   GridSpec, CellIndex, cell_of                 grid.hpp:16-113
//   ParticleSoA                                  particles.hpp:14-47
//   ShapeOrder (+ tsc, this project's order 2)   shape.hpp:14
//   CurrentGrid                                  grid.hpp:127-150
//   deposit_scalar, deposit_density              deposit.hpp:62-83
//   deposit_tiled (+TiledOptions, StageTimes,
//   KernelCounters), deposit_rhocell_vector      deposit.hpp:87-130, :179-334
//   advance                                      workload.hpp:139-155
//   GpmaConfig, gpma_build (perm + bins)         gpma.hpp:22-26, :379-402
//   SortPolicy, RankSortStats, SortReason,
//   should_global_sort, reset_counters           sort_policy.hpp:12-79
//   Session: device-resident store + step loop   simulation.hpp:92-176
// Status codes map back onto the reference's exceptions: EINVAL ->
// std::invalid_argument, ERANGE -> std::out_of_range, ELENGTH ->
// std::length_error, ELOGIC -> std::logic_error, EDOMAIN -> std::domain_error,
// ECUDA / ENCCL -> std::runtime_error, ENOMEM -> std::bad_alloc.
#pragma once

#include <algorithm>
#include <array>
#include <cstring>
#include <cstdlib>
#include <cstdio>
#include <chrono>
#include <string_view>
#include <cstdint>
#include <new>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "picgpu.h"

namespace picgpu {

inline void check(int rc) {
    if (rc == PICGPU_OK) return;
    const std::string msg = picgpu_last_error();
    switch (rc) {
        case PICGPU_EINVAL: throw std::invalid_argument(msg);
        case PICGPU_ERANGE: throw std::out_of_range(msg);
        case PICGPU_ELENGTH: throw std::length_error(msg);
        case PICGPU_ELOGIC: throw std::logic_error(msg);
        case PICGPU_EDOMAIN: throw std::domain_error(msg);
        case PICGPU_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(msg);
    }
}

using Vec3 = std::array<double, 3>;

struct CellIndex {
    int i = 0, j = 0, k = 0;
    std::uint32_t linear = 0;
};

struct GridSpec {
    int nx = 1, ny = 1, nz = 1;
    double dx = 1.0, dy = 1.0, dz = 1.0;
    Vec3 origin{0.0, 0.0, 0.0};

    void validate() const {
        if (nx < 1 || ny < 1 || nz < 1) throw std::invalid_argument("grid: cell counts must be >= 1");
        if (!(dx > 0.0) || !(dy > 0.0) || !(dz > 0.0)) throw std::invalid_argument("grid: cell sizes must be positive");
    }
    std::uint32_t n_cells() const {
        return static_cast<std::uint32_t>(nx) * static_cast<std::uint32_t>(ny) * static_cast<std::uint32_t>(nz);
    }
    std::uint32_t n_nodes() const { return n_cells(); }
    std::uint32_t linear_id(int i, int j, int k) const {
        return static_cast<std::uint32_t>(i) +
               static_cast<std::uint32_t>(nx) * (static_cast<std::uint32_t>(j) + static_cast<std::uint32_t>(ny) *
                                                                                      static_cast<std::uint32_t>(k));
    }
    picgpu_grid c() const { return picgpu_grid{nx, ny, nz, 0, dx, dy, dz, origin[0], origin[1], origin[2]}; }
};

enum class ShapeOrder { cic = 1, tsc = 2, qsp = 3 };

struct ParticleSoA {
    std::vector<double> x, y, z;
    std::vector<double> vx, vy, vz;
    std::vector<double> w;
    std::vector<std::uint64_t> id;
    double q = 1.0;

    std::size_t size() const { return x.size(); }
    void resize(std::size_t n) {
        x.resize(n); y.resize(n); z.resize(n);
        vx.resize(n); vy.resize(n); vz.resize(n);
        w.resize(n); id.resize(n);
    }
    Vec3 position(std::size_t i) const { return {x[i], y[i], z[i]}; }
    void apply_permutation(std::span<const std::uint32_t> perm) {
        if (perm.size() != size()) throw std::invalid_argument("apply_permutation: size mismatch");
        auto permute = [&](auto& a) {
            auto out = a;
            for (std::size_t i = 0; i < perm.size(); ++i) out[i] = a[perm[i]];
            a.swap(out);
        };
        permute(x); permute(y); permute(z);
        permute(vx); permute(vy); permute(vz);
        permute(w); permute(id);
    }
};

struct CurrentGrid {
    GridSpec spec;
    std::vector<double> jx, jy, jz;
    CurrentGrid() = default;
    explicit CurrentGrid(const GridSpec& g) : spec(g), jx(g.n_nodes(), 0.0), jy(g.n_nodes(), 0.0), jz(g.n_nodes(), 0.0) {}
    std::vector<double>& component(int c) { return c == 0 ? jx : c == 1 ? jy : jz; }
    const std::vector<double>& component(int c) const { return c == 0 ? jx : c == 1 ? jy : jz; }
    std::array<double, 3> component_sums() const {
        std::array<double, 3> s{0.0, 0.0, 0.0};
        for (int c = 0; c < 3; ++c)
            for (double v : component(c)) s[c] += v;
        return s;
    }
};

inline CellIndex cell_of(const Vec3& p, const GridSpec& g) {
    const picgpu_grid cg = g.c();
    std::uint32_t lin = 0;
    check(picgpu_cell_of(&cg, &p[0], &p[1], &p[2], 1, &lin));
    CellIndex c;
    c.linear = lin;
    c.i = static_cast<int>(lin % static_cast<std::uint32_t>(g.nx));
    c.j = static_cast<int>((lin / static_cast<std::uint32_t>(g.nx)) % static_cast<std::uint32_t>(g.ny));
    c.k = static_cast<int>(lin / (static_cast<std::uint32_t>(g.nx) * static_cast<std::uint32_t>(g.ny)));
    return c;
}

struct Gpma;

// deposit.hpp:62-73.  The reference's optional Gpma* only changes the
// summation order (bins ascending instead of storage order); J is
// order-independent to 1e-12, so it is accepted and not needed.
inline CurrentGrid deposit_scalar(const ParticleSoA& soa, const GridSpec& g, ShapeOrder order,
                                  const Gpma* /*gpma*/ = nullptr) {
    CurrentGrid grid(g);
    const picgpu_grid cg = g.c();
    check(picgpu_deposit_current(&cg, static_cast<int>(order), soa.x.data(), soa.y.data(), soa.z.data(),
                                 soa.vx.data(), soa.vy.data(), soa.vz.data(), soa.w.data(), soa.q, soa.size(),
                                 grid.jx.data(), grid.jy.data(), grid.jz.data()));
    return grid;
}

// deposit.hpp:76-83: bit-identical to the reference (storage-order sum).
inline std::vector<double> deposit_density(const ParticleSoA& soa, const GridSpec& g, ShapeOrder order,
                                           std::span<const double> quantity) {
    if (quantity.size() != soa.size()) throw std::invalid_argument("deposit_density: quantity length mismatch");
    std::vector<double> rho(g.n_nodes(), 0.0);
    const picgpu_grid cg = g.c();
    check(picgpu_deposit_density(&cg, static_cast<int>(order), soa.x.data(), soa.y.data(), soa.z.data(),
                                 quantity.data(), soa.size(), rho.data()));
    return rho;
}

// workload.hpp:139-155: bit-identical push; returns the moved fraction.
inline double advance(ParticleSoA& soa, double dt, const GridSpec& g) {
    const std::size_t n = soa.size();
    if (n == 0) return 0.0;
    const picgpu_grid cg = g.c();
    std::uint64_t moved = 0;
    check(picgpu_advance(&cg, dt, soa.x.data(), soa.y.data(), soa.z.data(), soa.vx.data(), soa.vy.data(),
                         soa.vz.data(), n, &moved));
    return static_cast<double>(moved) / static_cast<double>(n);
}

struct GpmaConfig {
    double gap_ratio = 0.25;
    std::uint32_t min_gap = 2;
    int borrow_scan_bins = 4;
};

// Result of gpma_build's stable counting sort (gpma.hpp:379-394), standing
// in for the reference's pic::Gpma at its read-only call sites: `Gpma gpma =
// gpma_build(soa, g)`, `deposit_scalar(soa, g, order, &gpma)` (test_pipeline.cpp:
// 139-142), for_each_in_cell / cell_entries (gpma.hpp:146-158).  The
// incremental index lives on the device (picgpu::Session).
struct Gpma {
    std::vector<std::uint32_t> perm;    // new storage index -> old
    std::vector<std::uint32_t> starts;  // packed bin starts (exclusive scan of counts)
    std::vector<std::uint32_t> counts;
    GpmaConfig cfg;

    std::size_t num_cells() const { return counts.size(); }
    std::size_t size() const { return perm.size(); }
    const GpmaConfig& config() const { return cfg; }
    // the storage indices of the particles of `cell`, in slot order
    template <class Fn>
    void for_each_in_cell(std::uint32_t cell, Fn&& fn) const {
        if (cell >= counts.size()) throw std::out_of_range("Gpma::for_each_in_cell: cell out of range");
        for (std::uint32_t r = starts[cell], e = starts[cell] + counts[cell]; r < e; ++r) fn(r);
    }
    std::vector<std::uint32_t> cell_entries(std::uint32_t cell) const {
        std::vector<std::uint32_t> out;
        for_each_in_cell(cell, [&](std::uint32_t r) { out.push_back(r); });
        return out;
    }
};
using Bins = Gpma;

// gpma_build (gpma.hpp:379-402): physically reorders the store by cell with a
// stable counting sort (bit-identical permutation) and returns the bins.
inline Gpma gpma_build(ParticleSoA& soa, const GridSpec& g, GpmaConfig cfg = {}) {
    Gpma b;
    b.cfg = cfg;
    b.perm.resize(soa.size());
    b.starts.resize(g.n_cells());
    b.counts.resize(g.n_cells());
    const picgpu_grid cg = g.c();
    check(picgpu_counting_sort(&cg, soa.x.data(), soa.y.data(), soa.z.data(), soa.size(), b.perm.data(),
                               b.starts.data(), b.counts.data()));
    soa.apply_permutation(b.perm);
    return b;
}

// deposit.hpp:121-130, :179-184.
struct KernelCounters {
    std::uint64_t mopa_calls = 0;
    std::uint64_t extract_passes = 0;
};
struct StageTimes {
    double preproc = 0.0;
    double compute = 0.0;
    double reduce = 0.0;
};
struct TiledOptions {
    const Bins* gpma = nullptr;  // when set, particles stream bin by bin
    bool residency = true;
    bool dual_tile = false;
    KernelCounters* counters = nullptr;
};

// deposit_tiled (deposit.hpp:284-334): the same J as deposit_scalar, computed
// by the FP64 tensor-core (DMMA) kernel; counters get the reference tile
// engine's counts for this input and options.
inline CurrentGrid deposit_tiled(const ParticleSoA& soa, const GridSpec& g, ShapeOrder order,
                                 const TiledOptions& opt = {}, StageTimes* times = nullptr) {
    CurrentGrid grid(g);
    const picgpu_grid cg = g.c();
    const std::uint32_t flags = (opt.gpma ? PICGPU_TILED_BINS : 0u) | (opt.residency ? PICGPU_TILED_RESIDENCY : 0u) |
                                (opt.dual_tile ? PICGPU_TILED_DUAL : 0u);
    picgpu_stage_times st{};
    picgpu_kernel_counters kc{};
    check(picgpu_deposit_tiled(&cg, static_cast<int>(order), soa.x.data(), soa.y.data(), soa.z.data(),
                               soa.vx.data(), soa.vy.data(), soa.vz.data(), soa.w.data(), soa.q, soa.size(), flags,
                               grid.jx.data(), grid.jy.data(), grid.jz.data(), times ? &st : nullptr,
                               opt.counters ? &kc : nullptr));
    if (times) *times = {st.preproc, st.compute, st.reduce};
    if (opt.counters) {
        opt.counters->mopa_calls += kc.mopa_calls;  // the reference increments
        opt.counters->extract_passes += kc.extract_passes;
    }
    return grid;
}

// deposit_rhocell_vector (deposit.hpp:87-119): the same J, warp-DFMA kernel.
inline CurrentGrid deposit_rhocell_vector(const ParticleSoA& soa, const GridSpec& g, ShapeOrder order,
                                          const Bins* gpma = nullptr, double* reduce_seconds = nullptr) {
    CurrentGrid grid(g);
    const picgpu_grid cg = g.c();
    check(picgpu_deposit_rhocell_vector(&cg, static_cast<int>(order), soa.x.data(), soa.y.data(), soa.z.data(),
                                        soa.vx.data(), soa.vy.data(), soa.vz.data(), soa.w.data(), soa.q, soa.size(),
                                        gpma != nullptr, grid.jx.data(), grid.jy.data(), grid.jz.data(),
                                        reduce_seconds));
    return grid;
}

struct SortPolicy {
    std::uint32_t sort_interval = 50;
    std::uint32_t min_sort_interval = 10;
    std::uint32_t trigger_rebuild_count = 100;
    double trigger_empty_ratio = 0.15;
    double trigger_full_ratio = 0.85;
    bool perf_enable = true;
    double perf_degrad = 0.80;
};

struct RankSortStats {
    std::uint32_t steps_since_sort = 0;
    std::uint64_t cumulative_local_rebuilds = 0;
    double empty_slot_ratio = 0.0;
    double perf_metric = 0.0;
    double baseline_perf = 0.0;
    std::uint64_t total_inserts = 0;
    std::uint64_t total_shifts = 0;
};

enum class SortReason { none, interval, rebuilds, slot_ratio, perf_degradation };

inline SortReason should_global_sort(const RankSortStats& s, const SortPolicy& p) {
    const picgpu_rank_sort_stats cs{s.steps_since_sort, 0, s.cumulative_local_rebuilds, s.empty_slot_ratio,
                                    s.perf_metric, s.baseline_perf, s.total_inserts, s.total_shifts};
    const picgpu_sort_policy cp{p.sort_interval, p.min_sort_interval, p.trigger_rebuild_count,
                                static_cast<std::uint32_t>(p.perf_enable), p.trigger_empty_ratio,
                                p.trigger_full_ratio, p.perf_degrad};
    return static_cast<SortReason>(picgpu_should_global_sort(&cs, &cp));
}

inline void reset_counters(RankSortStats& s) {  // sort_policy.hpp:75-79
    s.steps_since_sort = 0;
    s.cumulative_local_rebuilds = 0;
    s.baseline_perf = 0.0;
}

// Device-resident store in cell bins with slack + deposition fields: the
// reference's step loop with the GPMA kept on the GPU.
class Session {
   public:
    Session(const GridSpec& g, ShapeOrder order, GpmaConfig gc = {}, int device = 0, bool timing = false)
        : grid_(g) {
        const picgpu_grid cg = g.c();
        const picgpu_session_config cfg{static_cast<int32_t>(order), device, gc.gap_ratio, gc.min_gap,
                                        timing ? PICGPU_SESSION_TIMING : 0u};
        check(picgpu_session_create(&cg, &cfg, &h_));
    }
    ~Session() { picgpu_session_destroy(h_); }
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;

    void upload(const ParticleSoA& s) {
        check(picgpu_session_upload(h_, s.size(), s.x.data(), s.y.data(), s.z.data(), s.vx.data(), s.vy.data(),
                                    s.vz.data(), s.w.data(), s.id.empty() ? nullptr : s.id.data(), s.q));
    }
    picgpu_step_stats step(double dt, std::uint32_t flags = PICGPU_STEP_DEFAULT) {
        picgpu_step_stats st{};
        check(picgpu_session_step(h_, dt, flags, &st));
        return st;
    }
    void global_sort() { check(picgpu_session_global_sort(h_)); }
    CurrentGrid current() const {
        CurrentGrid g(grid_);
        check(picgpu_session_download_current(h_, g.jx.data(), g.jy.data(), g.jz.data()));
        return g;
    }
    std::vector<double> density() const {
        std::vector<double> r(grid_.n_nodes());
        check(picgpu_session_download_density(h_, r.data()));
        return r;
    }
    ParticleSoA particles() const {
        ParticleSoA s;
        s.resize(picgpu_session_num_particles(h_));
        check(picgpu_session_download_particles(h_, s.x.data(), s.y.data(), s.z.data(), s.vx.data(), s.vy.data(),
                                                s.vz.data(), s.w.data(), s.id.data()));
        return s;
    }
    std::size_t capacity() const { return picgpu_session_capacity(h_); }
    std::size_t size() const { return picgpu_session_num_particles(h_); }
    void set_kernel(int family) { check(picgpu_session_set_kernel(h_, family)); }
    void set_fusion(double max_moved_fraction) { check(picgpu_session_set_fusion(h_, max_moved_fraction)); }
    void make_workload(const picgpu_workload& w) { check(picgpu_session_make_workload(h_, &w)); }
    std::array<double, PICGPU_NPHASES> phase_ms() const {
        std::array<double, PICGPU_NPHASES> ms{};
        check(picgpu_session_phase_times(h_, ms.data(), nullptr, PICGPU_NPHASES));
        return ms;
    }
    picgpu_session* handle() const { return h_; }

   private:
    GridSpec grid_;
    picgpu_session* h_ = nullptr;
};

// ---- multi-GPU: x-slab sessions over NCCL (no reference counterpart) -------
// One process per GPU.  Rank 0 makes the id, the host's launcher broadcasts it
// (MPI_Bcast, a file, torch.distributed ...), every rank joins:
//   auto id = picgpu::Comm::unique_id();            // rank 0
//   /* broadcast id */
//   picgpu::Comm comm(id, nranks, rank, device);
//   auto [x0, x1] = picgpu::slab_range(g.nx, nranks, rank);
//   picgpu::SlabSession S(g, x0, x1, picgpu::ShapeOrder::qsp, comm);
//   S.upload(owned_particles); for (...) S.step(dt);  // one host sync per step
class Comm {
   public:
    using Id = std::array<unsigned char, 128>;
    static Id unique_id() {
        Id id{};
        check(picgpu_comm_unique_id(id.data()));
        return id;
    }
    Comm(const Id& id, int nranks, int rank, int device) { check(picgpu_comm_init(id.data(), nranks, rank, device, &c_)); }
    ~Comm() { picgpu_comm_destroy(c_); }
    Comm(const Comm&) = delete;
    Comm& operator=(const Comm&) = delete;
    picgpu_comm* handle() const { return c_; }

   private:
    picgpu_comm* c_ = nullptr;
};

inline std::pair<int, int> slab_range(int nx, int nranks, int rank) {  // balanced contiguous split
    const int base = nx / nranks, rem = nx % nranks;
    const int x0 = rank * base + std::min(rank, rem);
    return {x0, x0 + base + (rank < rem ? 1 : 0)};
}

class SlabSession {
   public:
    SlabSession(const GridSpec& global, int x0, int x1, ShapeOrder order, Comm& comm, GpmaConfig gc = {},
                int device = 0, int ghost = 2, std::uint32_t bucket_records = 0)
        : global_(global) {
        const picgpu_grid G = global.c();
        picgpu_grid L{};
        check(picgpu_slab_grid(&G, x0, x1, ghost, &L));
        local_ = GridSpec{L.nx, L.ny, L.nz, L.dx, L.dy, L.dz, {L.ox, L.oy, L.oz}};
        const picgpu_session_config cfg{static_cast<int32_t>(order), device, gc.gap_ratio, gc.min_gap, 0u};
        check(picgpu_session_create(&L, &cfg, &h_));
        check(picgpu_session_set_slab(h_, &G, x0, x1, ghost));
        check(picgpu_session_set_comm(h_, comm.handle(), bucket_records));
    }
    ~SlabSession() { picgpu_session_destroy(h_); }
    SlabSession(const SlabSession&) = delete;
    SlabSession& operator=(const SlabSession&) = delete;
    void upload(const ParticleSoA& s) {  // particles of the owned cells, global coordinates
        check(picgpu_session_upload(h_, s.size(), s.x.data(), s.y.data(), s.z.data(), s.vx.data(), s.vy.data(),
                                    s.vz.data(), s.w.data(), s.id.empty() ? nullptr : s.id.data(), s.q));
    }
    picgpu_step_stats step(double dt, std::uint32_t flags = PICGPU_STEP_DEFAULT) {  // collective
        picgpu_step_stats st{};
        check(picgpu_session_slab_step(h_, dt, flags, &st));
        return st;
    }
    CurrentGrid current() const {  // the slab grid's J (owned planes complete after the step)
        CurrentGrid g(local_);
        check(picgpu_session_download_current(h_, g.jx.data(), g.jy.data(), g.jz.data()));
        return g;
    }
    picgpu_session* handle() const { return h_; }

   private:
    GridSpec global_, local_;
    picgpu_session* h_ = nullptr;
};

// ---- charge-conserving current (an extension; no reference counterpart) ----
// Esirkepov J on the Yee faces for particles moved from `before` to `after`
// (same order of particles); see picgpu_deposit_current_esirkepov.
inline CurrentGrid deposit_current_esirkepov(const ParticleSoA& before, const ParticleSoA& after, const GridSpec& g,
                                             ShapeOrder order, double dt) {
    if (before.size() != after.size()) throw std::invalid_argument("deposit_current_esirkepov: size mismatch");
    CurrentGrid J(g);
    const picgpu_grid cg = g.c();
    check(picgpu_deposit_current_esirkepov(&cg, static_cast<int>(order), before.x.data(), before.y.data(),
                                           before.z.data(), after.x.data(), after.y.data(), after.z.data(),
                                           before.w.data(), before.q, dt, before.size(), J.jx.data(), J.jy.data(),
                                           J.jz.data()));
    return J;
}

// ---- the reference's harness loop (simulation.hpp:19-176) -------------------

enum class AblationMode {
    baseline,
    matrix_only,
    hybrid_nosort,
    hybrid_globalsort,
    fullopt,
    rhocell_vector,
    baseline_incrsort,
    rhocell_incrsort,
};
inline constexpr std::array<AblationMode, 8> kAllModes{
    AblationMode::baseline,          AblationMode::matrix_only,      AblationMode::hybrid_nosort,
    AblationMode::hybrid_globalsort, AblationMode::fullopt,          AblationMode::rhocell_vector,
    AblationMode::baseline_incrsort, AblationMode::rhocell_incrsort};

inline const char* to_string(AblationMode m) {
    switch (m) {
        case AblationMode::baseline: return "baseline";
        case AblationMode::matrix_only: return "matrix-only";
        case AblationMode::hybrid_nosort: return "hybrid-nosort";
        case AblationMode::hybrid_globalsort: return "hybrid-globalsort";
        case AblationMode::fullopt: return "fullopt";
        case AblationMode::rhocell_vector: return "rhocell-vector";
        case AblationMode::baseline_incrsort: return "baseline-incrsort";
        case AblationMode::rhocell_incrsort: return "rhocell-incrsort";
    }
    return "?";
}
inline AblationMode mode_from_string(std::string_view s) {
    for (AblationMode m : kAllModes)
        if (s == to_string(m)) return m;
    throw std::invalid_argument("unknown mode: " + std::string(s));
}
inline bool mode_uses_gpma(AblationMode m) {
    return m == AblationMode::hybrid_globalsort || m == AblationMode::fullopt ||
           m == AblationMode::baseline_incrsort || m == AblationMode::rhocell_incrsort;
}
inline bool mode_incremental_sort(AblationMode m) {
    return m == AblationMode::fullopt || m == AblationMode::baseline_incrsort || m == AblationMode::rhocell_incrsort;
}
// GPU kernel family of a mode: the scalar modes run the register-lane DFMA
// kernel, the rhocell-vector modes the warp-DFMA kernel, the tile-engine modes
// the FP64 tensor-core (DMMA) kernel.
inline int mode_kernel_family(AblationMode m) {
    switch (m) {
        case AblationMode::baseline:
        case AblationMode::baseline_incrsort: return 0;
        case AblationMode::rhocell_vector:
        case AblationMode::rhocell_incrsort: return 1;
        default: return 2;
    }
}

enum class WorkloadKind { uniform_plasma, drift_gradient };
struct WorkloadConfig {  // workload.hpp:16-44
    GridSpec grid;
    int ppc = 8;
    WorkloadKind kind = WorkloadKind::uniform_plasma;
    double thermal_speed = 0.01;
    Vec3 drift_velocity{0.0, 0.0, 0.0};
    std::uint64_t seed = 1;
    int steps = 10;
    double dt = 1.0;
    double charge = 1.0;
    ShapeOrder order = ShapeOrder::cic;
    double speed_cap() const { return std::min(grid.dx, std::min(grid.dy, grid.dz)) / dt; }
    picgpu_workload c() const {
        return picgpu_workload{grid.c(), ppc, static_cast<int32_t>(kind), thermal_speed,
                               {drift_velocity[0], drift_velocity[1], drift_velocity[2]}, seed, steps,
                               static_cast<int32_t>(order), dt, charge};
    }
};

struct StepMetrics {  // simulation.hpp:67-78
    std::uint32_t step = 0;
    double wall_s = 0.0;
    double preproc_s = 0.0;
    double compute_s = 0.0;
    double sort_s = 0.0;
    double reduce_s = 0.0;
    double particles_per_second = 0.0;
    double fraction_moved = 0.0;
    std::uint32_t rebuilds = 0;
    SortReason global_sort = SortReason::none;
};

struct RunResult {  // simulation.hpp:80-86
    std::vector<StepMetrics> steps;
    std::array<double, 3> checksum{0.0, 0.0, 0.0};
    CurrentGrid final_grid;
    ParticleSoA particles;
    RankSortStats stats;
};

// run_simulation (simulation.hpp:92-176) on one GPU: per step, advance fused
// with the mode's sort (incremental for the *-incrsort / fullopt modes, a full
// stable counting sort of the store otherwise -- the GPU kernels always read
// bins), deposition with the mode's kernel family, metrics from device event
// times (sort_s includes the fused push; preproc_s and reduce_s are 0, the
// staging and the node reduction live inside the kernels), then fullopt's
// adaptive global-resort decision.  `initial` replaces make_workload (e.g. the
// reference's own population, for bit-exact lockstep runs).
inline RunResult run_simulation(const WorkloadConfig& cfg, AblationMode mode, const SortPolicy& policy = {},
                                const GpmaConfig& gcfg = {}, int device = 0, const ParticleSoA* initial = nullptr) {
    // SortPolicy::validate (sort_policy.hpp:20-28)
    if (policy.min_sort_interval > policy.sort_interval)
        throw std::invalid_argument("policy: min_sort_interval exceeds sort_interval");
    if (!(policy.trigger_empty_ratio > 0.0 && policy.trigger_empty_ratio < 1.0) ||
        !(policy.trigger_full_ratio > 0.0 && policy.trigger_full_ratio < 1.0))
        throw std::invalid_argument("policy: slot-ratio triggers must lie in (0,1)");
    if (!(policy.perf_degrad > 0.0 && policy.perf_degrad <= 1.0))
        throw std::invalid_argument("policy: perf_degrad must lie in (0,1]");
    RunResult out;
    const GridSpec& g = cfg.grid;
    Session sess(g, cfg.order, gcfg, device, /*timing=*/true);
    sess.set_kernel(mode_kernel_family(mode));
    if (initial)
        sess.upload(*initial);
    else
        sess.make_workload(cfg.c());
    const std::size_t n = sess.size();
    const std::uint32_t flags = PICGPU_STEP_PUSH | PICGPU_STEP_CURRENT |
                                (mode_incremental_sort(mode) ? PICGPU_STEP_SORT : PICGPU_STEP_RESORT);
    std::array<double, PICGPU_NPHASES> prev = sess.phase_ms();
    for (int step = 0; step < cfg.steps; ++step) {
        StepMetrics m;
        m.step = static_cast<std::uint32_t>(step);
        const auto t0 = std::chrono::steady_clock::now();
        const picgpu_step_stats st = sess.step(cfg.dt, flags);
        const std::array<double, PICGPU_NPHASES> ph = sess.phase_ms();
        m.sort_s = (ph[0] - prev[0] + ph[2] - prev[2]) * 1e-3;
        m.compute_s = (ph[3] - prev[3] + ph[5] - prev[5]) * 1e-3;
        prev = ph;
        m.fraction_moved = n ? static_cast<double>(st.moved) / static_cast<double>(n) : 0.0;
        m.rebuilds = st.rebuilt;
        out.stats.total_inserts += st.inserts;
        m.particles_per_second =
            static_cast<double>(n) / std::max(m.preproc_s + m.compute_s + m.sort_s + m.reduce_s, 1e-12);
        out.stats.perf_metric = m.particles_per_second;
        out.stats.steps_since_sort += 1;
        out.stats.cumulative_local_rebuilds += m.rebuilds;
        if (mode_uses_gpma(mode)) out.stats.empty_slot_ratio = st.empty_slot_ratio;
        if (mode == AblationMode::fullopt) {
            if (out.stats.baseline_perf == 0.0) out.stats.baseline_perf = m.particles_per_second;
            const SortReason reason = should_global_sort(out.stats, policy);
            if (reason != SortReason::none) {
                sess.step(cfg.dt, PICGPU_STEP_GLOBAL_SORT);  // global_sort, timed
                const std::array<double, PICGPU_NPHASES> ph2 = sess.phase_ms();
                m.sort_s += (ph2[2] - prev[2]) * 1e-3;
                prev = ph2;
                reset_counters(out.stats);
                m.global_sort = reason;
            }
        }
        m.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        out.steps.push_back(m);
    }
    out.final_grid = sess.current();
    out.checksum = out.final_grid.component_sums();
    out.particles = sess.particles();
    return out;
}

// ---- reports (report.hpp:23-103): the reference's CSV / JSON schema ----------

inline const char* to_string(SortReason r) {  // sort_policy.hpp:48-56
    switch (r) {
        case SortReason::interval: return "interval";
        case SortReason::rebuilds: return "rebuilds";
        case SortReason::slot_ratio: return "slot_ratio";
        case SortReason::perf_degradation: return "perf_degradation";
        default: return "none";
    }
}

// The writer is table-driven: one Column per schema field says how a step
// row renders it and how the summary row aggregates it (a total, a mean, or a
// count).  CSV emits the columns in schema order, JSON in key order -- the
// reference's report.hpp:49-103 layout, produced from this one table.
namespace report_detail {

enum class Agg { total, mean, count_nonzero, label };

struct Cell {  // one rendered value: number or string
    bool is_text = false, is_int = false;
    double num = 0.0;
    std::uint64_t integer = 0;
    std::string text;
};

struct Column {
    const char* csv_name;      // step-row key (CSV header and JSON "steps" key)
    const char* summary_key;   // JSON "summary" key
    Agg agg;
    Cell (*get)(const StepMetrics&);
};

inline Cell num(double v) { Cell c; c.num = v; return c; }
inline Cell integer(std::uint64_t v) { Cell c; c.is_int = true; c.integer = v; return c; }
inline Cell text(std::string v) { Cell c; c.is_text = true; c.text = std::move(v); return c; }

inline const std::vector<Column>& columns() {
    static const std::vector<Column> cols = {
        {"step", nullptr, Agg::label, [](const StepMetrics& m) { return integer(m.step); }},
        {"wall_s", "wall_s", Agg::total, [](const StepMetrics& m) { return num(m.wall_s); }},
        {"preproc_s", "preproc_s", Agg::total, [](const StepMetrics& m) { return num(m.preproc_s); }},
        {"compute_s", "compute_s", Agg::total, [](const StepMetrics& m) { return num(m.compute_s); }},
        {"sort_s", "sort_s", Agg::total, [](const StepMetrics& m) { return num(m.sort_s); }},
        {"reduce_s", "reduce_s", Agg::total, [](const StepMetrics& m) { return num(m.reduce_s); }},
        {"pps", "mean_pps", Agg::mean, [](const StepMetrics& m) { return num(m.particles_per_second); }},
        {"fraction_moved", "mean_fraction_moved", Agg::mean,
         [](const StepMetrics& m) { return num(m.fraction_moved); }},
        {"rebuilds", "rebuilds", Agg::total, [](const StepMetrics& m) { return integer(m.rebuilds); }},
        {"global_sort_reason", "global_sorts", Agg::count_nonzero,
         [](const StepMetrics& m) { return text(to_string(m.global_sort)); }},
    };
    return cols;
}

// The summary value of column c over the steps.
inline Cell aggregate(const Column& c, std::span<const StepMetrics> steps) {
    if (c.agg == Agg::count_nonzero) {
        std::uint64_t n = 0;
        for (const StepMetrics& m : steps) n += m.global_sort != SortReason::none;
        return integer(n);
    }
    double acc = 0.0;
    std::uint64_t iacc = 0;
    bool ints = false;
    for (const StepMetrics& m : steps) {
        const Cell v = c.get(m);
        ints = v.is_int;
        if (v.is_int) iacc += v.integer; else acc += v.num;
    }
    if (ints) return integer(iacc);
    if (c.agg == Agg::mean && !steps.empty()) acc /= static_cast<double>(steps.size());
    return num(acc);
}

// %.17g for CSV; the shortest round-trip form (nlohmann::json's) for JSON.
inline std::string csv_num(double v) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return buf;
}
inline std::string json_num(double v) {
    char buf[40];
    int prec = 1;
    do {
        std::snprintf(buf, sizeof(buf), "%.*g", prec, v);
    } while (std::strtod(buf, nullptr) != v && ++prec <= 17);
    std::string s = buf;
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}
inline std::string render(const Cell& c, bool json) {
    if (c.is_text) return json ? "\"" + c.text + "\"" : c.text;
    if (c.is_int) return std::to_string(c.integer);
    return json ? json_num(c.num) : csv_num(c.num);
}

// JSON object from (key, value) pairs, keys in sorted order, no whitespace.
inline std::string json_object(std::vector<std::pair<std::string, std::string>> kv) {
    std::sort(kv.begin(), kv.end());
    std::string out = "{";
    for (std::size_t i = 0; i < kv.size(); ++i) out += (i ? ",\"" : "\"") + kv[i].first + "\":" + kv[i].second;
    return out + "}";
}

}  // namespace report_detail

inline const std::string& csv_header() {
    static const std::string h = [] {
        std::string s;
        for (const auto& c : report_detail::columns()) s += (s.empty() ? "" : ",") + std::string(c.csv_name);
        return s;
    }();
    return h;
}

// One row per step, then a summary row (label "summary"; totals, means and
// the count of fired global sorts), as report_csv (report.hpp:51-71).
inline std::string report_csv(std::span<const StepMetrics> steps) {
    using namespace report_detail;
    std::string out = csv_header() + "\n";
    if (steps.empty()) return out;
    for (const StepMetrics& m : steps) {
        std::string row;
        for (const auto& c : columns()) row += (row.empty() ? "" : ",") + render(c.get(m), false);
        out += row + "\n";
    }
    std::string row = "summary";
    for (const auto& c : columns())
        if (c.agg != Agg::label) row += "," + render(aggregate(c, steps), false);
    return out + row + "\n";
}

// report_json's records (report.hpp:74-103) serialised like
// nlohmann::json::dump(): keys sorted, no whitespace.
inline std::string report_json(std::span<const StepMetrics> steps) {
    using namespace report_detail;
    std::vector<std::pair<std::string, std::string>> top;
    std::string arr = "[";
    for (std::size_t i = 0; i < steps.size(); ++i) {
        std::vector<std::pair<std::string, std::string>> kv;
        for (const auto& c : columns()) kv.emplace_back(c.csv_name, render(c.get(steps[i]), true));
        arr += (i ? "," : "") + json_object(std::move(kv));
    }
    top.emplace_back("steps", arr + "]");
    if (!steps.empty()) {
        std::vector<std::pair<std::string, std::string>> kv;
        for (const auto& c : columns())
            if (c.summary_key) kv.emplace_back(c.summary_key, render(aggregate(c, steps), true));
        top.emplace_back("summary", json_object(std::move(kv)));
    }
    return json_object(std::move(top));
}

}  // namespace picgpu
