/*
 * picgpu.h -- C ABI of the B200-native (sm_100a) MatrixPIC deposition + cell-sort path.
 *
 * Every entry point takes plain pointers and sizes; no torch or C++ types cross
 * this boundary.  The C++ shim include/picgpu.hpp restores the reference's
 * value-semantics API (namespace picgpu mirrors namespace pic) on top of it,
 * and INTEGRATION.md shows the binding a maintainer adds to the reference.
 *
 * Reference interface each export replaces (paths under the reference tree
 * proj/include/pic/):
 *   picgpu_deposit_current   <- pic::deposit_scalar          deposit.hpp:62-73
 *   picgpu_deposit_density   <- pic::deposit_density         deposit.hpp:76-83
 *   picgpu_counting_sort     <- pic::gpma_build's counting sort (perm/starts/counts) gpma.hpp:379-394
 *   picgpu_advance           <- pic::advance                 workload.hpp:139-155
 *   picgpu_cell_of           <- pic::cell_of                 grid.hpp:106-113
 *   picgpu_session_*         <- the run_simulation step loop simulation.hpp:92-176 with a
 *                               device-resident pic::Gpma (gpma.hpp:52-371): gpma_build,
 *                               detect_moves + apply_pending_moves, rebuild, global_sort
 *                               (sort_policy.hpp:83), deposit_scalar / deposit_density.
 *   picgpu_should_global_sort <- pic::should_global_sort     sort_policy.hpp:62-73
 *   picgpu_deposit_tiled     <- pic::deposit_tiled (+ KernelCounters, StageTimes) deposit.hpp:121-334
 *   picgpu_deposit_rhocell_vector <- pic::deposit_rhocell_vector deposit.hpp:87-119
 *   picgpu_session_make_workload <- pic::make_workload        workload.hpp:16-125
 *   picgpu_slab_grid, picgpu_session_set_slab / step_begin / step_end / guard planes
 *                            <- new: x-slab decomposition over ranks (the
 *                               reference has no domain decomposition)
 *
 * Errors: every call returns a status.  The codes map one-to-one onto the
 * exception types the reference throws; picgpu_last_error()
 * returns a thread-local message for the last failing call on this thread.
 */
#ifndef PICGPU_H
#define PICGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PICGPU_ABI_VERSION 1

#if defined(__GNUC__)
#define PICGPU_API __attribute__((visibility("default")))
#else
#define PICGPU_API
#endif

enum picgpu_status {
    PICGPU_OK = 0,
    PICGPU_EINVAL = 1,  /* std::invalid_argument (non-finite position, bad order, grid < stencil) */
    PICGPU_ERANGE = 2,  /* std::out_of_range */
    PICGPU_ELENGTH = 3, /* std::length_error (slot capacity >= 2^32, gpma.hpp:279) */
    PICGPU_ELOGIC = 4,  /* std::logic_error */
    PICGPU_EDOMAIN = 5, /* std::domain_error (advance: displacement above the cap, workload.hpp:147) */
    PICGPU_ECUDA = 6,   /* CUDA runtime failure (std::runtime_error in the shim) */
    PICGPU_ENCCL = 7,   /* NCCL failure */
    PICGPU_ENOMEM = 8   /* device allocation failure (std::bad_alloc in the shim) */
};

/* Periodic box (pic::GridSpec, grid.hpp:26-72).  Node arrays use the cell
 * layout id = i + nx*(j + ny*k) (grid.hpp:50-54). */
typedef struct picgpu_grid {
    int32_t nx, ny, nz, pad_;
    double dx, dy, dz;
    double ox, oy, oz;
} picgpu_grid;

/* ---- library ----------------------------------------------------------- */
PICGPU_API int picgpu_abi_version(void);
PICGPU_API const char* picgpu_last_error(void);
/* Number of this library's kernels launched since load (all entry points). */
PICGPU_API uint64_t picgpu_kernel_launches(void);
/* Reference flop tally per deposit (deposit.hpp:336-345): 76 / 238 / 534. */
PICGPU_API int picgpu_flop_count(int order);

/* ---- stateless, host buffers (synchronous, like the reference) --------- */
/* J = sum_p q*W_p*v_p*S(x_i - x_p) at shape order 1, 2 or 3; jx/jy/jz hold
 * ncells doubles each and are overwritten.  Order 2 is this project's TSC. */
PICGPU_API int picgpu_deposit_current(const picgpu_grid* g, int order, const double* x, const double* y, const double* z,
                           const double* vx, const double* vy, const double* vz, const double* w, double q,
                           uint64_t n, double* jx, double* jy, double* jz);
/* rho = one-component scatter of quantity[p] in STORAGE ORDER, bit-identical
 * to pic::deposit_density on the same arrays. */
PICGPU_API int picgpu_deposit_density(const picgpu_grid* g, int order, const double* x, const double* y, const double* z,
                           const double* quantity, uint64_t n, double* rho);
/* Stable counting sort by linear cell id: perm bit-identical to gpma_build's. */
PICGPU_API int picgpu_counting_sort(const picgpu_grid* g, const double* x, const double* y, const double* z, uint64_t n,
                         uint32_t* perm, uint32_t* bin_start, uint32_t* bin_count);
/* Ballistic push x = wrap(x + v*dt), bit-identical to pic::advance. */
PICGPU_API int picgpu_advance(const picgpu_grid* g, double dt, double* x, double* y, double* z, const double* vx,
                   const double* vy, const double* vz, uint64_t n, uint64_t* moved);
PICGPU_API int picgpu_cell_of(const picgpu_grid* g, const double* x, const double* y, const double* z, uint64_t n,
                   uint32_t* cell);

/* pic::StageTimes / pic::KernelCounters (deposit.hpp:121-130). */
typedef struct picgpu_stage_times {
    double preproc; /* s: device time of the bin build (the staging pass of deposit_tiled) */
    double compute; /* s: device time of the J kernel */
    double reduce;  /* s: 0 -- nodes are reduced inside the J kernel, no rhocell pass */
} picgpu_stage_times;
typedef struct picgpu_kernel_counters {
    uint64_t mopa_calls;     /* tile outer products the reference's engine issues for this input */
    uint64_t extract_passes; /* tile extractions, same rule (deposit.hpp:191-274) */
} picgpu_kernel_counters;
/* pic::TiledOptions (deposit.hpp:179-184) as bit flags. */
#define PICGPU_TILED_BINS 1u      /* opt.gpma != nullptr: particles stream bin by bin */
#define PICGPU_TILED_RESIDENCY 2u /* opt.residency (CIC tiles resident across a cell's pairs) */
#define PICGPU_TILED_DUAL 4u      /* opt.dual_tile */
/* deposit_tiled (deposit.hpp:284-334): the reference's three-stage MOPA
 * pipeline.  Same J as deposit_scalar (<= 1e-12); computed by the FP64
 * tensor-core (DMMA) kernel at orders 2/3.  counters (may be NULL) get the
 * exact counts the reference's tile engine produces on this input and options.
 * Grids smaller than the stencil are rejected like NodeMap (rhocell.hpp:49);
 * the reference's 1 GiB rhocell budget (rhocell.hpp:68-73) does not apply. */
PICGPU_API int picgpu_deposit_tiled(const picgpu_grid* g, int order, const double* x, const double* y, const double* z,
                                    const double* vx, const double* vy, const double* vz, const double* w, double q,
                                    uint64_t n, uint32_t options, double* jx, double* jy, double* jz,
                                    picgpu_stage_times* times, picgpu_kernel_counters* counters);
/* deposit_rhocell_vector (deposit.hpp:87-119): the per-cell vector-unit
 * variant; same J, computed by the warp-per-pencil DFMA kernel at orders 2/3.
 * reduce_seconds (may be NULL) gets 0 (no separate reduce pass). */
PICGPU_API int picgpu_deposit_rhocell_vector(const picgpu_grid* g, int order, const double* x, const double* y,
                                             const double* z, const double* vx, const double* vy, const double* vz,
                                             const double* w, double q, uint64_t n, int use_bins, double* jx,
                                             double* jy, double* jz, double* reduce_seconds);

/* ---- stateless, device buffers (asynchronous on `stream`) -------------- */
/* Inputs and outputs are device pointers; scratch is allocated internally.
 * These are the hot-path entry points when particles already live in HBM. */
PICGPU_API int picgpu_deposit_current_dev(const picgpu_grid* g, int order, const double* x, const double* y, const double* z,
                               const double* vx, const double* vy, const double* vz, const double* w, double q,
                               uint64_t n, double* jx, double* jy, double* jz, void* stream);

/* ---- charge-conserving current (an EXTENSION: no reference counterpart) -- */
/* Esirkepov's scheme on the staggered Yee grid at shape order 1/2/3: particles
 * move from (x0,y0,z0) to (x1,y1,z1) in dt (x1 as pushed, i.e. possibly
 * wrapped into the box; the cell step per axis must be -1, 0 or +1, else
 * PICGPU_EDOMAIN).  jx[i + nx*(j + ny*k)] is J_x on the face (i+1/2, j, k),
 * likewise jy (i, j+1/2, k) and jz (i, j, k+1/2); they satisfy the discrete
 * continuity equation with rho = q*w*S (picgpu_deposit_density) to round-off.
 * The reference deposits J collocated (pic::deposit_scalar, deposit.hpp:60-73)
 * and lists charge-conserving schemes as future work: parity is
 * against this project's restatement (oracle/picoracle.c) and continuity. */
PICGPU_API int picgpu_deposit_current_esirkepov(const picgpu_grid* g, int order, const double* x0, const double* y0,
                                                const double* z0, const double* x1, const double* y1,
                                                const double* z1, const double* w, double q, double dt, uint64_t n,
                                                double* jx, double* jy, double* jz);
PICGPU_API int picgpu_deposit_current_esirkepov_dev(const picgpu_grid* g, int order, const double* x0,
                                                    const double* y0, const double* z0, const double* x1,
                                                    const double* y1, const double* z1, const double* w, double q,
                                                    double dt, uint64_t n, double* jx, double* jy, double* jz,
                                                    void* stream);

/* ---- resort policy (host logic, sort_policy.hpp:12-79) ------------------ */
typedef struct picgpu_sort_policy {
    uint32_t sort_interval;         /* 50 */
    uint32_t min_sort_interval;     /* 10 */
    uint32_t trigger_rebuild_count; /* 100 */
    uint32_t perf_enable;           /* 1 */
    double trigger_empty_ratio;     /* 0.15 */
    double trigger_full_ratio;      /* 0.85 */
    double perf_degrad;             /* 0.80 */
} picgpu_sort_policy;

typedef struct picgpu_rank_sort_stats {
    uint32_t steps_since_sort;
    uint32_t pad_;
    uint64_t cumulative_local_rebuilds;
    double empty_slot_ratio;
    double perf_metric;
    double baseline_perf;
    uint64_t total_inserts;
    uint64_t total_shifts;
} picgpu_rank_sort_stats;

enum picgpu_sort_reason {
    PICGPU_SORT_NONE = 0,
    PICGPU_SORT_INTERVAL = 1,
    PICGPU_SORT_REBUILDS = 2,
    PICGPU_SORT_SLOT_RATIO = 3,
    PICGPU_SORT_PERF = 4
};

PICGPU_API void picgpu_sort_policy_defaults(picgpu_sort_policy* p);
PICGPU_API int picgpu_should_global_sort(const picgpu_rank_sort_stats* s, const picgpu_sort_policy* p);

/* ---- device-resident session: bins-with-slack sorter + deposition ------ */
typedef struct picgpu_session picgpu_session;

typedef struct picgpu_session_config {
    int32_t order;        /* 1, 2, 3 */
    int32_t device;       /* CUDA device ordinal */
    double gap_ratio;     /* GpmaConfig::gap_ratio (0.25) */
    uint32_t min_gap;     /* GpmaConfig::min_gap (2) */
    uint32_t flags;       /* PICGPU_SESSION_* */
} picgpu_session_config;

#define PICGPU_SESSION_TIMING 1u        /* record CUDA events around each phase */

/* per-step flags */
#define PICGPU_STEP_PUSH 1u       /* advance (bit-exact pic::advance) */
#define PICGPU_STEP_SORT 2u       /* incremental sort (detect + migrate) */
#define PICGPU_STEP_CURRENT 4u    /* deposit J */
#define PICGPU_STEP_DENSITY 8u    /* deposit rho = q*W (bit-exact ordered gather) */
#define PICGPU_STEP_GLOBAL_SORT 16u /* force a full re-sort (global_sort) after the deposit */
#define PICGPU_STEP_NO_SYNC 32u   /* do not read back step stats (counts stay on device) */
#define PICGPU_STEP_RESORT 64u    /* instead of SORT: after the push, a full stable counting sort of the
                                     whole store (hybrid-globalsort and the modes without an index) */
#define PICGPU_STEP_UNFUSED 128u  /* PUSH|SORT|CURRENT on the default kernel run as ONE fused pass
                                     (push + move detection + J of the particles that stay in their
                                     cell; movers deposited separately) unless this flag is set:
                                     then a push kernel, the sort and the J kernel run one after another */
#define PICGPU_STEP_DEFAULT (PICGPU_STEP_PUSH | PICGPU_STEP_SORT | PICGPU_STEP_CURRENT)

typedef struct picgpu_step_stats {
    uint64_t moved;        /* particles whose cell changed (advance's moved count) */
    uint64_t inserts;      /* migrated particles placed into bins */
    uint64_t overflowed;   /* arrivals that found no slack -> rebuild */
    uint32_t rebuilt;      /* 1 if this step rebuilt the bins */
    uint32_t global_sorted;
    double empty_slot_ratio;
    uint64_t capacity;
    uint64_t num_particles;
    uint32_t fused;        /* 1 if push + detect + J ran as one fused pass (PICGPU_STEP_UNFUSED) */
    uint32_t reserved_;
} picgpu_step_stats;

PICGPU_API int picgpu_session_create(const picgpu_grid* g, const picgpu_session_config* cfg, picgpu_session** out);
PICGPU_API int picgpu_session_destroy(picgpu_session* s);
/* Upload a particle store (host pointers) and build the bins: stable counting
 * sort by cell + layout with slack = ceil(count*(1+gap_ratio)) + min_gap per
 * bin (gpma_build, gpma.hpp:379-402, layout :269-302).  id may be NULL (ids =
 * storage index).  Replaces any previous content. */
PICGPU_API int picgpu_session_upload(picgpu_session* s, uint64_t n, const double* x, const double* y, const double* z,
                          const double* vx, const double* vy, const double* vz, const double* w,
                          const uint64_t* id, double q);
/* Generate the SURVEY 8(d) seeded plasma directly in HBM (device-side
 * generator on the reference counter RNG; inputs for benchmarks). */
PICGPU_API int picgpu_session_generate_plasma(picgpu_session* s, int ppc, double u_th, uint64_t seed);
/* SURVEY 8(d) C4 (laser-wakefield-like) population on the session grid:
 * background electrons in x-cells i >= ramp_start, round(ppc * ramp_i) per
 * cell with ramp_i = clamp((i + 0.5 - ramp_start) / ramp_len, 0, 1), uniform
 * in the cell (counters 6, 7, 8), Maxwellian u_th (counters 0..5), pid
 * cell-major; plus a beam of llround(beam_fraction * background) particles
 * with ux ~ U(ux_min, ux_max) (counter 9), uy = uz = 0, uniform in x-cells
 * [beam_x0, beam_x1) and over the whole y-z plane, pids after the background.
 * v = u / gamma, W = 1/ppc, q = -1. */
typedef struct picgpu_lwfa {
    int32_t ppc, ramp_start, ramp_len, pad_;
    double u_th, beam_fraction, ux_min, ux_max, beam_x0, beam_x1;
    uint64_t seed;
} picgpu_lwfa;
PICGPU_API int picgpu_session_generate_lwfa(picgpu_session* s, const picgpu_lwfa* cfg);
/* C4 moving window: the grid origin moves +dx in x, particles
 * behind it (the old x-column 0) are dropped, and a fresh column of ppc
 * particles per cell is injected at the front (x-column nx-1): uniform in the
 * cell (counters 6, 7, 8), Maxwellian u_th (counters 0..5), ids / RNG streams
 * pid0, pid0+1, ... (cell-major).  The bins are rebuilt (stable counting sort).
 * Not available on slab sessions. */
PICGPU_API int picgpu_session_shift_window(picgpu_session* s, int ppc, double u_th, uint64_t seed, uint64_t pid0,
                                           uint64_t* n_dropped, uint64_t* n_injected);
/* The session's current grid (its origin moves with shift_window). */
PICGPU_API int picgpu_session_grid(picgpu_session* s, picgpu_grid* out);
/* One step: [push] -> [incremental sort] -> [deposit J] -> [deposit rho] -> [global sort]. */
PICGPU_API int picgpu_session_step(picgpu_session* s, double dt, uint32_t flags, picgpu_step_stats* out);
PICGPU_API int picgpu_session_global_sort(picgpu_session* s);
/* J kernel family used by this session's steps (orders 2/3): 0 register-lane
 * DFMA (default), 1 warp-per-pencil DFMA ("vector", rhocell-vector modes),
 * 2 FP64 tensor-core DMMA ("matrix", tile-engine modes). */
PICGPU_API int picgpu_session_set_kernel(picgpu_session* s, int family);
/* Fusion policy of PUSH|SORT|CURRENT steps: the fused pass runs while the
 * previous pushed step moved less than this fraction of the particles (default
 * 0.06, or PICGPU_FUSE_MAX_MOVED); 0 never fuses, >1 always does.  EINVAL if
 * negative or NaN.  No reference counterpart (a performance knob). */
/* Adaptive slack (off by default): an overflow rebuild within 4 pushed steps
 * of the previous one doubles the gap ratio of every later layout (up to 1.0).
 * For persistent inflow (C4's beam); capacities then differ from the
 * reference's Gpma after such rebuilds (bin SETS do not). */
PICGPU_API int picgpu_session_set_adaptive_slack(picgpu_session* s, int enable);
PICGPU_API int picgpu_session_set_fusion(picgpu_session* s, double max_moved_fraction);

/* pic::WorkloadConfig (workload.hpp:16-44) and make_workload (:75-125): ppc
 * particles per cell on a regular sub-lattice, Maxwellian velocities
 * truncated at the displacement cap, optional shear drift, W = 1.  Generated
 * on the device (velocities may differ from glibc's in the last ulp of log /
 * cos); the reference's 2^28-particle limit does not apply. */
#define PICGPU_WORKLOAD_UNIFORM 0
#define PICGPU_WORKLOAD_DRIFT_GRADIENT 1
typedef struct picgpu_workload {
    picgpu_grid grid;
    int32_t ppc;
    int32_t kind;            /* PICGPU_WORKLOAD_* */
    double thermal_speed;
    double drift[3];         /* drift_gradient amplitude; all zero selects 0.5 * speed cap along x */
    uint64_t seed;
    int32_t steps;
    int32_t order;           /* ShapeOrder */
    double dt;
    double charge;
} picgpu_workload;
/* Replaces the session's particles by make_workload(cfg) (grid must match). */
PICGPU_API int picgpu_session_make_workload(picgpu_session* s, const picgpu_workload* cfg);
PICGPU_API int picgpu_session_synchronize(picgpu_session* s);
PICGPU_API uint64_t picgpu_session_num_particles(picgpu_session* s);
PICGPU_API uint64_t picgpu_session_capacity(picgpu_session* s);
PICGPU_API void* picgpu_session_stream(picgpu_session* s);
/* Downloads (synchronous).  Particles come out in storage order: bins
 * ascending by cell, slot order within a bin (valid slots only, compacted). */
PICGPU_API int picgpu_session_download_particles(picgpu_session* s, double* x, double* y, double* z, double* vx, double* vy,
                                      double* vz, double* w, uint64_t* id);
PICGPU_API int picgpu_session_download_bins(picgpu_session* s, uint32_t* bin_offset, uint32_t* bin_count);
PICGPU_API int picgpu_session_download_current(picgpu_session* s, double* jx, double* jy, double* jz);
PICGPU_API int picgpu_session_download_density(picgpu_session* s, double* rho);
/* Device pointers of J (3*ncells doubles, jx|jy|jz) and rho (ncells). */
PICGPU_API int picgpu_session_device_fields(picgpu_session* s, double** j, double** rho);
/* Accumulated per-phase device times (ms) and launch counts since the last
 * reset, recorded only with PICGPU_SESSION_TIMING.  Phases:
 * 0 push + detect + migrate + borrow, 1 reserved, 2 rebuild/global sort, 3 deposit J,
 * 4 deposit rho, 5 zero fields.  In a fused step (PICGPU_STEP_UNFUSED not set)
 * phase 3 is the fused push + detect + J kernel and phase 0 the movers'
 * records/holes/J plus the migration. */
#define PICGPU_NPHASES 6
PICGPU_API int picgpu_session_phase_times(picgpu_session* s, double* ms, uint64_t* launches, int nphases);
PICGPU_API int picgpu_session_reset_phase_times(picgpu_session* s);

/* ---- x-slab decomposition over ranks -----------------------
 * The reference runs one single-threaded process over the whole periodic box
 * (simulation.hpp:92-176) and has no domain decomposition (SPEC.md:507 only
 * allows distinct Gpma tiles to run concurrently).  Here each rank (one
 * process per GPU) owns the global
 * x-cells [x0, x1) of `global` and runs one session on its slab grid: the
 * owned cells plus `ghost` (>= 2, the QSP stencil reach) guard cells on each
 * side.  Positions stay in global coordinates and wrap on the global box, so
 * every per-particle value is bit-identical to the undecomposed run.  A step
 * is split around two neighbour exchanges (done by the caller, e.g. NCCL
 * send/recv between ranks r-1, r, r+1 on the periodic ring):
 *   step_begin        push + move detection; particles that left the slab are
 *                     packed as 8-double records (x y z vx vy vz w id-bits)
 *   copy_leavers      -> caller's device buffers, sent to the left / right rank
 *   step_end          arrivals (records from both neighbours) inserted like
 *                     movers, then J / rho deposited on the slab grid
 *   guard_planes      planes [0,ghost) -> left rank, [ghost+own, own+2*ghost) -> right
 *   add_guard_planes  the left rank's high planes add into [ghost, 2*ghost),
 *                     the right rank's low planes into [own, own+ghost)
 * Device pointers passed in must be complete (synchronised) when the call is
 * made; outputs are complete when it returns. */
/* The slab grid of [x0, x1) with `ghost` guard cells per side. */
PICGPU_API int picgpu_slab_grid(const picgpu_grid* global, int x0, int x1, int ghost, picgpu_grid* local);
/* Turns an empty session created on picgpu_slab_grid(global, x0, x1, ghost)
 * into a slab session.  Upload / generate_plasma then take only owned particles
 * (generate_plasma produces the global generator's particles of the owned cells,
 * global ids). */
PICGPU_API int picgpu_session_set_slab(picgpu_session* s, const picgpu_grid* global, int x0, int x1, int ghost);
/* flags as for picgpu_session_step (SORT required; GLOBAL_SORT / NO_SYNC ignored). */
PICGPU_API int picgpu_session_step_begin(picgpu_session* s, double dt, uint32_t flags, uint64_t* n_to_left,
                                         uint64_t* n_to_right);
PICGPU_API int picgpu_session_copy_leavers(picgpu_session* s, double* to_left, double* to_right);
PICGPU_API int picgpu_session_step_end(picgpu_session* s, const double* arrivals, uint64_t n_arrivals,
                                       picgpu_step_stats* out);
/* field 0: J (3 components), 1: rho.  Each buffer holds comps*ghost*nz*ny
 * doubles laid out [comp][plane][z][y]. */
PICGPU_API int picgpu_session_guard_planes(picgpu_session* s, int field, double* lo, double* hi);
PICGPU_API int picgpu_session_add_guard_planes(picgpu_session* s, int field, const double* from_left,
                                               const double* from_right);

/* ---- microbenchmarks (roofline denominators measured in-run) ------------ */
/* Runs a dependent-free DFMA loop on all SMs; returns measured FP64 TFLOP/s. */
PICGPU_API int picgpu_fp64_peak(int device, double* tflops);

/* ---- multi-GPU: NCCL behind the C ABI (x-slab sessions) ----- */
/* New (the reference has no decomposition; its step loop is
 * simulation.hpp:105-181).  One process per GPU; rank r of the communicator
 * owns slab r of the x-decomposition and exchanges with ranks r-1 and r+1 on
 * the periodic ring.  The library binds the libnccl.so.2 already loaded in
 * the process (else loads it), so a communicator from the host application's
 * own NCCL can be wrapped. */
typedef struct picgpu_comm picgpu_comm;
PICGPU_API int picgpu_comm_unique_id(unsigned char id[128]);  /* ncclGetUniqueId: on one rank, then broadcast */
PICGPU_API int picgpu_comm_init(const unsigned char id[128], int nranks, int rank, int device, picgpu_comm** out);
PICGPU_API int picgpu_comm_wrap(void* nccl_comm, int device, picgpu_comm** out); /* an existing ncclComm_t */
PICGPU_API int picgpu_comm_rank(const picgpu_comm* c, int* rank, int* nranks);
PICGPU_API int picgpu_comm_destroy(picgpu_comm* c);
/* Attach a communicator to a slab session (picgpu_session_set_slab first).
 * bucket_records: leaver records per side sent in the step's first exchange
 * round (0: 32768); more leavers than that go in a second, exactly sized round. */
PICGPU_API int picgpu_session_set_comm(picgpu_session* s, picgpu_comm* c, uint32_t bucket_records);
/* One whole slab step with ONE host synchronisation: push + detect (fused
 * with J at low migration) -> leaver counts and records to the ring
 * neighbours (one NCCL group, counts stay on the device) -> arrivals imported,
 * deposited and inserted -> step counters read -> guard planes of J (and rho)
 * summed with the neighbours (NCCL, enqueued; no trailing synchronisation).
 * Collective: every rank of the communicator calls it with the same flags. */
PICGPU_API int picgpu_session_slab_step(picgpu_session* s, double dt, uint32_t flags, picgpu_step_stats* out);

#ifdef __cplusplus
}
#endif
#endif /* PICGPU_H */
