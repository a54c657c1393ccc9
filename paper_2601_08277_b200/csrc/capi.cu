// capi.cu -- the C ABI (include/picgpu.h): stateless drop-ins for the
// reference's deposition / sort / push functions and the device-resident
// session that runs the reference's step loop (simulation.hpp:92-176) on HBM.
#include <atomic>
#include <cmath>
#include <cstring>
#include <functional>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "comm.hpp"
#include "kernels.hpp"
#include "store.hpp"

namespace picgpu {

static std::atomic<uint64_t> g_launches{0};
void note_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static thread_local std::string g_error;

static int set_error(int code, const std::string& msg) {
    g_error = msg;
    return code;
}

template <class F>
static int guard(F&& f) {
    try {
        f();
        return PICGPU_OK;
    } catch (const Status& s) {
        return set_error(s.code, s.msg ? s.msg : "error");
    } catch (const CudaError& e) {
        return set_error(PICGPU_ECUDA, std::string(e.what) + ": " + cudaGetErrorString(e.code));
    } catch (const std::bad_alloc&) {
        return set_error(PICGPU_ENOMEM, "host allocation failed");
    } catch (...) {
        return set_error(PICGPU_ELOGIC, "unexpected exception");
    }
}

static bool is_pow2(double h) {
    int e = 0;
    return std::frexp(h, &e) == 0.5;
}

// GridSpec::validate (grid.hpp:32-36) + the derived constants.
GridD make_grid(const picgpu_grid& h) {
    if (h.nx < 1 || h.ny < 1 || h.nz < 1) throw Status{PICGPU_EINVAL, "grid: cell counts must be >= 1"};
    if (!(h.dx > 0.0) || !(h.dy > 0.0) || !(h.dz > 0.0))
        throw Status{PICGPU_EINVAL, "grid: cell sizes must be positive"};
    const uint64_t nc = (uint64_t)h.nx * (uint64_t)h.ny * (uint64_t)h.nz;
    if (nc >= 0xffffffffull) throw Status{PICGPU_ELENGTH, "grid: more than 2^32-1 cells"};
    GridD g{};
    g.nx = h.nx; g.ny = h.ny; g.nz = h.nz;
    g.dx = h.dx; g.dy = h.dy; g.dz = h.dz;
    g.ox = h.ox; g.oy = h.oy; g.oz = h.oz;
    g.Lx = h.nx * h.dx;  // GridSpec::length: cells(axis) * spacing(axis)
    g.Ly = h.ny * h.dy;
    g.Lz = h.nz * h.dz;
    g.pow2x = is_pow2(h.dx); g.pow2y = is_pow2(h.dy); g.pow2z = is_pow2(h.dz);
    g.inv_dx = 1.0 / h.dx; g.inv_dy = 1.0 / h.dy; g.inv_dz = 1.0 / h.dz;
    g.pow2Lx = is_pow2(g.Lx); g.pow2Ly = is_pow2(g.Ly); g.pow2Lz = is_pow2(g.Lz);
    g.inv_Lx = 1.0 / g.Lx; g.inv_Ly = 1.0 / g.Ly; g.inv_Lz = 1.0 / g.Lz;
    g.ncells = (uint32_t)nc;
    g.slab = 0;
    g.gnx = g.nx;
    g.sx_shift = 0;
    g.sx_lo = 0;
    g.sx_hi = g.nx;
    g.gox = g.ox;
    g.gLx = g.Lx;
    g.ginv_Lx = g.inv_Lx;
    g.gpow2Lx = g.pow2Lx;
    return g;
}

static void check_order(int order) {
    if (order < 1 || order > 3) throw Status{PICGPU_EINVAL, "shape order must be 1, 2 or 3"};
}

static int window(int order) { return order == 1 ? 2 : 4; }

static void check_density_grid(const picgpu_grid& g, int order) {
    const int W = window(order);
    if (g.nx < W || g.ny < W || g.nz < W)
        throw Status{PICGPU_EINVAL, "deposit_density: grid smaller than the shape window"};
}

// advance's displacement cap (workload.hpp:141): (min_spacing/dt)^2.
static double cap2_of(const picgpu_grid& g, double dt) {
    if (!(dt > 0.0)) throw Status{PICGPU_EINVAL, "advance: dt must be positive"};
    const double ms = std::min(g.dx, std::min(g.dy, g.dz));
    return (ms / dt) * (ms / dt);
}

__global__ void k_fill_ids(uint64_t* id, uint64_t n) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) id[p] = p;
}

__global__ void k_not_identity(const uint32_t* perm, uint64_t n, int* flag) {
    const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n && perm[r] != (uint32_t)r) *flag = 1;
}

static void h2d(void* d, const void* h, size_t bytes, cudaStream_t st) {
    if (bytes) PICGPU_CUDA_TRY(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
}
static void d2h(void* h, const void* d, size_t bytes, cudaStream_t st) {
    if (bytes && h) PICGPU_CUDA_TRY(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st));
}

static int current_sms() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// Workspace of the stateless entry points (packed bins, gap 0 / min_gap 0).
struct Stateless {
    std::mutex mu;
    cudaStream_t st = nullptr;
    cudaStream_t st2 = nullptr;     // second upload stream (velocities, weights)
    cudaEvent_t fields = nullptr;   // ... recorded after them
    BinStore store;
    DevBuf J, aux, flag;
    picgpu_grid grid{};
    bool ready = false;

    void prepare(const picgpu_grid& g) {
        if (!st) PICGPU_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        if (!st2) PICGPU_CUDA_TRY(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
        if (!fields) PICGPU_CUDA_TRY(cudaEventCreateWithFlags(&fields, cudaEventDisableTiming));
        if (!ready || std::memcmp(&g, &grid, sizeof g) != 0) {
            store.init(g, 0.0, 0, st);
            grid = g;
            ready = true;
        }
        flag.ensure(16);
    }
};

// Tile-engine counts of deposit_tiled (deposit.hpp:191-274) from the grouping
// the reference would see: out[0] += groups, out[1] += sum of ceil(len/2).
// Bins: one group per non-empty cell.  Runs: maximal runs of equal cell id in
// storage order (the residency-on path without an index, deposit.hpp:303-313).
__global__ void k_bin_groups(const uint32_t* __restrict__ cnt, uint32_t ncells, unsigned long long* out) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long grp = 0, pairs = 0;
    if (c < ncells && cnt[c]) {
        grp = 1;
        pairs = (cnt[c] + 1u) / 2u;
    }
    grp = __reduce_add_sync(0xffffffffu, (unsigned)grp);
    pairs = __reduce_add_sync(0xffffffffu, (unsigned)pairs);
    if ((threadIdx.x & 31) == 0 && grp) {
        atomicAdd(out, grp);
        atomicAdd(out + 1, pairs);
    }
}

__global__ void k_run_groups(const uint32_t* __restrict__ key, uint64_t n, unsigned long long* out) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long grp = 0, pairs = 0;
    if (p < n && (p == 0 || key[p] != key[p - 1])) {
        uint64_t e = p + 1;
        while (e < n && key[e] == key[p]) ++e;
        grp = 1;
        pairs = (e - p + 1) / 2;
    }
    if (grp) {
        atomicAdd(out, grp);
        atomicAdd(out + 1, pairs);
    }
}

static Stateless& stateless() {
    static Stateless* s = new Stateless;  // never destroyed (driver may be gone at exit)
    return *s;
}

}  // namespace picgpu

using namespace picgpu;

// ===========================================================================
// session

struct picgpu_session {
    int device = 0;
    int order = 3;
    uint32_t flags = 0;
    double q = 1.0;
    cudaStream_t st = nullptr;
    BinStore store;
    DevBuf J, rho, dscratch;
    bool timing = false;
    cudaEvent_t ev[8] = {};
    double phase_ms[PICGPU_NPHASES] = {};
    uint64_t phase_launches[PICGPU_NPHASES] = {};
    int kernel = -1;  // JKernel family; -1: library default
    double last_moved = 0.0;  // moved fraction of the previous pushed step (fusion policy)
    double fuse_max = [] {    // fuse while last_moved < fuse_max (picgpu_session_set_fusion)
        const char* e = std::getenv("PICGPU_FUSE_MAX_MOVED");
        return e ? std::atof(e) : 0.06;
    }();
    // x-slab decomposition (picgpu_session_set_slab)
    bool slab = false;
    int ghost = 0;
    int own = 0;
    bool pending = false;      // between step_begin and step_end
    bool pending_fused = false;  // ... of a fused step (J deposited in step_begin)
    uint32_t pending_flags = 0;
    uint64_t nleave[2] = {0, 0};
    StepCounters cbegin{};
    uint64_t begin_launches = 0;
    // adaptive slack (picgpu_session_set_adaptive_slack): rebuild storms widen the gap ratio
    bool adaptive_slack = false;
    uint32_t since_rebuild = 1000;  // pushed steps since the last rebuild
    // device-resident exchange over NCCL (picgpu_session_set_comm / slab_step)
    picgpu_comm* comm = nullptr;
    uint32_t bucket = 0;            // records per side per step in the first exchange round
    DevBuf xin, xcnt, xin2;         // arrivals (2 buckets), their counts, second-round remainders
    DevBuf psend, precv;            // guard planes: [lo | hi] and [from left | from right]
    uint32_t* hxcnt = nullptr;      // pinned mirror of xcnt
};

static void set_device(const picgpu_session* s) { PICGPU_CUDA_TRY(cudaSetDevice(s->device)); }

extern "C" {

int picgpu_abi_version(void) { return PICGPU_ABI_VERSION; }
const char* picgpu_last_error(void) { return g_error.c_str(); }
uint64_t picgpu_kernel_launches(void) { return g_launches.load(); }

int picgpu_flop_count(int order) {
    if (order == 1) return 9 + 3 + 4 + 60;   // deposit.hpp:343-344
    if (order == 3) return 9 + 57 + 4 + 464;
    if (order == 2) return 9 + 27 + 4 + 9 + 7 * 27;  // this project's TSC tally (f_shape = 9)
    return -1;
}

void picgpu_sort_policy_defaults(picgpu_sort_policy* p) {
    p->sort_interval = 50;  // sort_policy.hpp:17-23
    p->min_sort_interval = 10;
    p->trigger_rebuild_count = 100;
    p->perf_enable = 1;
    p->trigger_empty_ratio = 0.15;
    p->trigger_full_ratio = 0.85;
    p->perf_degrad = 0.80;
}

// sort_policy.hpp:62-73, same priority order.
int picgpu_should_global_sort(const picgpu_rank_sort_stats* s, const picgpu_sort_policy* p) {
    if (s->steps_since_sort < p->min_sort_interval) return PICGPU_SORT_NONE;
    if (s->steps_since_sort >= p->sort_interval) return PICGPU_SORT_INTERVAL;
    if (s->cumulative_local_rebuilds > p->trigger_rebuild_count) return PICGPU_SORT_REBUILDS;
    if (s->empty_slot_ratio < p->trigger_empty_ratio || s->empty_slot_ratio > p->trigger_full_ratio)
        return PICGPU_SORT_SLOT_RATIO;
    if (p->perf_enable && s->baseline_perf > 0.0 && s->perf_metric < p->perf_degrad * s->baseline_perf)
        return PICGPU_SORT_PERF;
    return PICGPU_SORT_NONE;
}

// ---- stateless -------------------------------------------------------------

}  // extern "C"

// deposit_scalar / deposit_tiled / deposit_rhocell_vector on host buffers:
// H2D, bin build (stable counting sort), J with the requested kernel family,
// D2H.  Device times of the build and of J in *sort_ms / *j_ms.
static void stateless_current(const picgpu_grid* g, int order, const double* x, const double* y, const double* z,
                              const double* vx, const double* vy, const double* vz, const double* w, double q,
                              uint64_t n, int kernel, double* jx, double* jy, double* jz, float* sort_ms,
                              float* j_ms, const uint32_t* tiled_options, picgpu_kernel_counters* counters) {
    check_order(order);
    const GridD gd = make_grid(*g);
    Stateless& S = stateless();
    std::lock_guard<std::mutex> lk(S.mu);
    S.prepare(*g);
    BinStore& bs = S.store;
    const cudaStream_t st = S.st;
    const bool timed = sort_ms || j_ms;
    cudaEvent_t ev[3] = {};
    if (timed)
        for (auto& e : ev) PICGPU_CUDA_TRY(cudaEventCreate(&e));
    bs.B.ensure(n);
    const Soa b = bs.B.soa();
    // positions first on the sort's stream, the other fields on a second
    // stream: cells, radix sort and layout run while velocities and weights
    // are still crossing PCIe (the gather waits for them)
    h2d(b.x, x, n * 8, st); h2d(b.y, y, n * 8, st); h2d(b.z, z, n * 8, st);
    PICGPU_CUDA_TRY(cudaEventRecord(S.fields, st));  // B is free (previous users on st are done)
    PICGPU_CUDA_TRY(cudaStreamWaitEvent(S.st2, S.fields, 0));
    h2d(b.vx, vx, n * 8, S.st2); h2d(b.vy, vy, n * 8, S.st2); h2d(b.vz, vz, n * 8, S.st2);
    h2d(b.w, w, n * 8, S.st2);
    PICGPU_CUDA_TRY(cudaEventRecord(S.fields, S.st2));
    if (timed) PICGPU_CUDA_TRY(cudaEventRecord(ev[0], st));
    bs.full_sort_from_B(n, nullptr, S.fields);
    if (timed) PICGPU_CUDA_TRY(cudaEventRecord(ev[1], st));
    S.J.ensure((size_t)gd.ncells * 24);
    double* J = S.J.as<double>();
    PICGPU_CUDA_TRY(cudaMemsetAsync(J, 0, (size_t)gd.ncells * 24, st));
    if (n) launch_deposit_current(order, gd, bs.A.aos(), bs.d_off(), bs.d_cnt(), q, J, bs.num_sms, st, kernel);
    if (timed) PICGPU_CUDA_TRY(cudaEventRecord(ev[2], st));
    if (counters) {
        const uint32_t opt = *tiled_options;
        unsigned long long* d = S.flag.as<unsigned long long>();
        PICGPU_CUDA_TRY(cudaMemsetAsync(d, 0, 16, st));
        if (opt & PICGPU_TILED_BINS) {
            k_bin_groups<<<div_up((long long)gd.ncells, 256), 256, 0, st>>>(bs.d_cnt(), gd.ncells, d);
            note_launch();
        } else if (n) {  // storage-order cell ids of the input (k_cells output of the sort)
            k_run_groups<<<div_up((long long)n, 256), 256, 0, st>>>(bs.keys.as<uint32_t>(), n, d);
            note_launch();
        }
        PICGPU_CUDA_TRY(cudaGetLastError());
        unsigned long long h[2] = {0, 0};
        PICGPU_CUDA_TRY(cudaMemcpyAsync(h, d, 16, cudaMemcpyDeviceToHost, st));
        PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
        const bool runs = (opt & (PICGPU_TILED_BINS | PICGPU_TILED_RESIDENCY)) != 0;
        const uint64_t pairs = runs ? h[1] : (n + 1) / 2;
        counters->mopa_calls = 3 * pairs;
        if (order == 1 && runs && (opt & PICGPU_TILED_RESIDENCY))  // cic_group_resident
            counters->extract_passes = 3 * h[0] * ((opt & PICGPU_TILED_DUAL) ? 2 : 1);
        else  // cic_pair_flush / qsp_pair: one extraction per pair and component
            counters->extract_passes = 3 * pairs;
    }
    d2h(jx, J, (size_t)gd.ncells * 8, st);
    d2h(jy, J + gd.ncells, (size_t)gd.ncells * 8, st);
    d2h(jz, J + 2 * (size_t)gd.ncells, (size_t)gd.ncells * 8, st);
    PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
    if (timed) {
        float a = 0, c = 0;
        PICGPU_CUDA_TRY(cudaEventElapsedTime(&a, ev[0], ev[1]));
        PICGPU_CUDA_TRY(cudaEventElapsedTime(&c, ev[1], ev[2]));
        if (sort_ms) *sort_ms = a;
        if (j_ms) *j_ms = c;
        for (auto& e : ev) cudaEventDestroy(e);
    }
}

extern "C" {

int picgpu_deposit_current(const picgpu_grid* g, int order, const double* x, const double* y, const double* z,
                           const double* vx, const double* vy, const double* vz, const double* w, double q,
                           uint64_t n, double* jx, double* jy, double* jz) {
    return guard([&] {
        stateless_current(g, order, x, y, z, vx, vy, vz, w, q, n, kJDefault, jx, jy, jz, nullptr, nullptr, nullptr,
                          nullptr);
    });
}

int picgpu_deposit_tiled(const picgpu_grid* g, int order, const double* x, const double* y, const double* z,
                         const double* vx, const double* vy, const double* vz, const double* w, double q, uint64_t n,
                         uint32_t options, double* jx, double* jy, double* jz, picgpu_stage_times* times,
                         picgpu_kernel_counters* counters) {
    return guard([&] {
        check_order(order);
        check_density_grid(*g, order);  // NodeMap: grid smaller than the stencil support
        float sort_ms = 0, j_ms = 0;
        stateless_current(g, order, x, y, z, vx, vy, vz, w, q, n, kJMatrix, jx, jy, jz, times ? &sort_ms : nullptr,
                          times ? &j_ms : nullptr, &options, counters);
        if (times) {
            times->preproc = sort_ms * 1e-3;
            times->compute = j_ms * 1e-3;
            times->reduce = 0.0;
        }
    });
}

int picgpu_deposit_rhocell_vector(const picgpu_grid* g, int order, const double* x, const double* y, const double* z,
                                  const double* vx, const double* vy, const double* vz, const double* w, double q,
                                  uint64_t n, int use_bins, double* jx, double* jy, double* jz,
                                  double* reduce_seconds) {
    (void)use_bins;  // the same J either way; the GPU always deposits from bins
    return guard([&] {
        check_order(order);
        check_density_grid(*g, order);
        stateless_current(g, order, x, y, z, vx, vy, vz, w, q, n, kJVector, jx, jy, jz, nullptr, nullptr, nullptr,
                          nullptr);
        if (reduce_seconds) *reduce_seconds = 0.0;
    });
}

// Esirkepov deposit on device buffers, enqueued on the stateless stream after
// `stream`, with `stream` waiting for it; the device error word is read once.
static void esirkepov_enqueue(const picgpu_grid* g, int order, const double* const in[7], double q, double dt,
                              uint64_t n, double* const out[3], cudaStream_t user, bool host_io) {
    check_order(order);
    if (!(dt > 0.0)) throw Status{PICGPU_EINVAL, "deposit_esirkepov: dt must be positive"};
    const GridD gd = make_grid(*g);
    Stateless& S = stateless();
    std::lock_guard<std::mutex> lk(S.mu);
    S.prepare(*g);
    const cudaStream_t st = S.st;
    BinStore& bs = S.store;
    const double* src[7];
    if (host_io) {
        bs.B.ensure(n);
        const Soa b = bs.B.soa();
        double* dst[7] = {b.x, b.y, b.z, b.vx, b.vy, b.vz, b.w};
        for (int a = 0; a < 7; ++a) {
            h2d(dst[a], in[a], n * 8, st);
            src[a] = dst[a];
        }
    } else {
        cudaEvent_t ev;
        PICGPU_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        PICGPU_CUDA_TRY(cudaEventRecord(ev, user));
        PICGPU_CUDA_TRY(cudaStreamWaitEvent(st, ev, 0));
        PICGPU_CUDA_TRY(cudaEventDestroy(ev));
        for (int a = 0; a < 7; ++a) src[a] = in[a];
    }
    S.J.ensure((size_t)gd.ncells * 24);
    double* J = S.J.as<double>();
    PICGPU_CUDA_TRY(cudaMemsetAsync(J, 0, (size_t)gd.ncells * 24, st));
    int* err = S.flag.as<int>();
    PICGPU_CUDA_TRY(cudaMemsetAsync(err, 0, 4, st));
    launch_deposit_esirkepov(order, gd, src[0], src[1], src[2], src[3], src[4], src[5], src[6], q, dt, n, J,
                             J + gd.ncells, J + 2 * (size_t)gd.ncells, err, st);
    int h = 0;
    PICGPU_CUDA_TRY(cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, st));
    PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
    if (h == PICGPU_EDOMAIN) throw Status{PICGPU_EDOMAIN, "deposit_esirkepov: a particle moved more than one cell"};
    if (h) throw Status{h, "deposit_esirkepov: non-finite particle position"};
    for (int c = 0; c < 3; ++c) {
        if (host_io)
            d2h(out[c], J + c * (size_t)gd.ncells, (size_t)gd.ncells * 8, st);
        else
            PICGPU_CUDA_TRY(cudaMemcpyAsync(out[c], J + c * (size_t)gd.ncells, (size_t)gd.ncells * 8,
                                            cudaMemcpyDeviceToDevice, st));
    }
    PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
}

int picgpu_deposit_current_esirkepov(const picgpu_grid* g, int order, const double* x0, const double* y0,
                                     const double* z0, const double* x1, const double* y1, const double* z1,
                                     const double* w, double q, double dt, uint64_t n, double* jx, double* jy,
                                     double* jz) {
    return guard([&] {
        const double* in[7] = {x0, y0, z0, x1, y1, z1, w};
        double* out[3] = {jx, jy, jz};
        esirkepov_enqueue(g, order, in, q, dt, n, out, nullptr, true);
    });
}

int picgpu_deposit_current_esirkepov_dev(const picgpu_grid* g, int order, const double* x0, const double* y0,
                                         const double* z0, const double* x1, const double* y1, const double* z1,
                                         const double* w, double q, double dt, uint64_t n, double* jx, double* jy,
                                         double* jz, void* stream) {
    return guard([&] {
        const double* in[7] = {x0, y0, z0, x1, y1, z1, w};
        double* out[3] = {jx, jy, jz};
        esirkepov_enqueue(g, order, in, q, dt, n, out, (cudaStream_t)stream, false);
    });
}

int picgpu_deposit_current_dev(const picgpu_grid* g, int order, const double* x, const double* y, const double* z,
                               const double* vx, const double* vy, const double* vz, const double* w, double q,
                               uint64_t n, double* jx, double* jy, double* jz, void* stream) {
    return guard([&] {
        check_order(order);
        const GridD gd = make_grid(*g);
        Stateless& S = stateless();
        std::lock_guard<std::mutex> lk(S.mu);
        S.prepare(*g);
        BinStore& bs = S.store;
        const cudaStream_t st = S.st;
        cudaEvent_t ev;
        PICGPU_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        PICGPU_CUDA_TRY(cudaEventRecord(ev, (cudaStream_t)stream));
        PICGPU_CUDA_TRY(cudaStreamWaitEvent(st, ev, 0));
        bs.B.ensure(n);
        const Soa b = bs.B.soa();
        const double* src[7] = {x, y, z, vx, vy, vz, w};
        double* dst[7] = {b.x, b.y, b.z, b.vx, b.vy, b.vz, b.w};
        for (int a = 0; a < 7; ++a)
            if (n) PICGPU_CUDA_TRY(cudaMemcpyAsync(dst[a], src[a], n * 8, cudaMemcpyDeviceToDevice, st));
        bs.full_sort_from_B(n);
        S.J.ensure((size_t)gd.ncells * 24);
        double* J = S.J.as<double>();
        PICGPU_CUDA_TRY(cudaMemsetAsync(J, 0, (size_t)gd.ncells * 24, st));
        if (n) launch_deposit_current(order, gd, bs.A.aos(), bs.d_off(), bs.d_cnt(), q, J, bs.num_sms, st);
        PICGPU_CUDA_TRY(cudaMemcpyAsync(jx, J, (size_t)gd.ncells * 8, cudaMemcpyDeviceToDevice, st));
        PICGPU_CUDA_TRY(cudaMemcpyAsync(jy, J + gd.ncells, (size_t)gd.ncells * 8, cudaMemcpyDeviceToDevice, st));
        PICGPU_CUDA_TRY(
            cudaMemcpyAsync(jz, J + 2 * (size_t)gd.ncells, (size_t)gd.ncells * 8, cudaMemcpyDeviceToDevice, st));
        PICGPU_CUDA_TRY(cudaEventRecord(ev, st));
        PICGPU_CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, ev, 0));
        PICGPU_CUDA_TRY(cudaEventDestroy(ev));
    });
}

int picgpu_deposit_density(const picgpu_grid* g, int order, const double* x, const double* y, const double* z,
                           const double* quantity, uint64_t n, double* rho) {
    return guard([&] {
        check_order(order);
        const GridD gd = make_grid(*g);
        check_density_grid(*g, order);
        Stateless& S = stateless();
        std::lock_guard<std::mutex> lk(S.mu);
        S.prepare(*g);
        BinStore& bs = S.store;
        const cudaStream_t st = S.st;
        bs.B.ensure(n);
        const Soa b = bs.B.soa();
        h2d(b.x, x, n * 8, st); h2d(b.y, y, n * 8, st); h2d(b.z, z, n * 8, st);
        h2d(b.w, quantity, n * 8, st);  // quantity rides in the w slot through the sort
        bs.full_sort_from_B(n);
        S.J.ensure((size_t)gd.ncells * 8);
        double* R = S.J.as<double>();
        if (n == 0) {
            PICGPU_CUDA_TRY(cudaMemsetAsync(R, 0, (size_t)gd.ncells * 8, st));
        } else {
            int* flag = S.flag.as<int>();
            PICGPU_CUDA_TRY(cudaMemsetAsync(flag, 0, 4, st));
            k_not_identity<<<div_up((long long)n, 256), 256, 0, st>>>(bs.vals2.as<uint32_t>(), n, flag);
            note_launch();
            int h = 0;
            PICGPU_CUDA_TRY(cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, st));
            PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
            S.aux.ensure(density_scratch_bytes(order, n));
            // the quantity rode in the records' w field: quantity = 1.0 * w (exact)
            const Aos a = bs.A.aos();
            if (!h)  // storage already cell-sorted: source-cell order == storage order
                launch_deposit_density(order, gd, a, nullptr, 1.0, bs.d_off(), bs.d_cnt(), n, S.aux.p, R, st);
            else
                launch_deposit_density_merge(order, gd, a, nullptr, 1.0, bs.vals2.as<uint32_t>(), bs.d_off(),
                                             bs.d_cnt(), n, S.aux.p, R, st);
        }
        d2h(rho, R, (size_t)gd.ncells * 8, st);
        PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
    });
}

int picgpu_counting_sort(const picgpu_grid* g, const double* x, const double* y, const double* z, uint64_t n,
                         uint32_t* perm, uint32_t* bin_start, uint32_t* bin_count) {
    return guard([&] {
        const GridD gd = make_grid(*g);
        Stateless& S = stateless();
        std::lock_guard<std::mutex> lk(S.mu);
        S.prepare(*g);
        BinStore& bs = S.store;
        const cudaStream_t st = S.st;
        bs.B.ensure(n);
        const Soa b = bs.B.soa();
        h2d(b.x, x, n * 8, st); h2d(b.y, y, n * 8, st); h2d(b.z, z, n * 8, st);
        bs.full_sort_from_B(n);
        d2h(perm, bs.vals2.p, n * 4, st);
        d2h(bin_start, bs.off.p, (size_t)gd.ncells * 4, st);  // packed layout: off == exclusive scan of counts
        d2h(bin_count, bs.cnt.p, (size_t)gd.ncells * 4, st);
        PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
    });
}

int picgpu_advance(const picgpu_grid* g, double dt, double* x, double* y, double* z, const double* vx,
                   const double* vy, const double* vz, uint64_t n, uint64_t* moved) {
    return guard([&] {
        const GridD gd = make_grid(*g);
        const double cap2 = cap2_of(*g, dt);
        Stateless& S = stateless();
        std::lock_guard<std::mutex> lk(S.mu);
        S.prepare(*g);
        BinStore& bs = S.store;
        const cudaStream_t st = S.st;
        bs.B.ensure(n);
        const Soa b = bs.B.soa();
        h2d(b.x, x, n * 8, st); h2d(b.y, y, n * 8, st); h2d(b.z, z, n * 8, st);
        h2d(b.vx, vx, n * 8, st); h2d(b.vy, vy, n * 8, st); h2d(b.vz, vz, n * 8, st);
        S.flag.ensure(16);
        unsigned long long* dm = S.flag.as<unsigned long long>();
        int* err = reinterpret_cast<int*>(dm + 1);
        PICGPU_CUDA_TRY(cudaMemsetAsync(dm, 0, 16, st));
        launch_advance(gd, dt, cap2, b.x, b.y, b.z, b.vx, b.vy, b.vz, n, dm, err, st);
        unsigned long long hm[2] = {0, 0};
        PICGPU_CUDA_TRY(cudaMemcpyAsync(hm, dm, 16, cudaMemcpyDeviceToHost, st));
        PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
        const int e = (int)(hm[1] & 0xffffffffu);
        if (e == PICGPU_EDOMAIN) throw Status{e, "advance: particle displacement exceeds the single-cell cap"};
        if (e) throw Status{e, "cell_of: non-finite particle position"};
        d2h(x, b.x, n * 8, st); d2h(y, b.y, n * 8, st); d2h(z, b.z, n * 8, st);
        PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
        if (moved) *moved = hm[0];
    });
}

int picgpu_cell_of(const picgpu_grid* g, const double* x, const double* y, const double* z, uint64_t n,
                   uint32_t* cell) {
    return guard([&] {
        const GridD gd = make_grid(*g);
        Stateless& S = stateless();
        std::lock_guard<std::mutex> lk(S.mu);
        S.prepare(*g);
        BinStore& bs = S.store;
        const cudaStream_t st = S.st;
        bs.B.ensure(n);
        bs.keys.ensure(n * 4 + 4);
        const Soa b = bs.B.soa();
        h2d(b.x, x, n * 8, st); h2d(b.y, y, n * 8, st); h2d(b.z, z, n * 8, st);
        int* err = S.flag.as<int>();
        PICGPU_CUDA_TRY(cudaMemsetAsync(err, 0, 4, st));
        launch_cells(gd, b.x, b.y, b.z, n, bs.keys.as<uint32_t>(), err, st);
        int h = 0;
        PICGPU_CUDA_TRY(cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, st));
        d2h(cell, bs.keys.p, n * 4, st);
        PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
        if (h) throw Status{h, "cell_of: non-finite particle position"};
    });
}

// ---- session ---------------------------------------------------------------

// Keep J resident in L2 while the step streams the particle store through it
// (a persisting access-policy window on the session stream): the fused step's
// movers and the halo nodes reduce into J with RED.ADD.F64, which otherwise
// miss L2 after the particle stream and pay a DRAM read-modify-write each.
// Best effort (PICGPU_L2_PERSIST=0 disables it); C2's J is 50 MB of the 126 MB L2.
static void keep_fields_in_l2(picgpu_session* s) {
    const char* e = std::getenv("PICGPU_L2_PERSIST");
    if (e && e[0] == '0') return;
    int max_persist = 0, max_window = 0;
    if (cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, s->device) != cudaSuccess ||
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, s->device) != cudaSuccess ||
        max_persist <= 0 || max_window <= 0) {
        cudaGetLastError();
        return;
    }
    const size_t bytes = (size_t)s->store.g.ncells * 24;
    const size_t persist = std::min(bytes, (size_t)max_persist);
    const size_t window = std::min(bytes, (size_t)max_window);
    cudaStreamAttrValue a{};
    a.accessPolicyWindow.base_ptr = s->J.p;
    a.accessPolicyWindow.num_bytes = window;
    a.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)persist / (double)window);
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist) != cudaSuccess ||
        cudaStreamSetAttribute(s->st, cudaStreamAttributeAccessPolicyWindow, &a) != cudaSuccess)
        cudaGetLastError();
}

int picgpu_session_create(const picgpu_grid* g, const picgpu_session_config* cfg, picgpu_session** out) {
    *out = nullptr;
    picgpu_session* s = nullptr;
    const int rc = guard([&] {
        check_order(cfg->order);
        make_grid(*g);
        if (!(cfg->gap_ratio >= 0.0)) throw Status{PICGPU_EINVAL, "gpma: gap_ratio must be >= 0"};
        s = new picgpu_session;
        s->device = cfg->device;
        s->order = cfg->order;
        s->flags = cfg->flags;
        set_device(s);
        PICGPU_CUDA_TRY(cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking));
        s->store.init(*g, cfg->gap_ratio, cfg->min_gap, s->st);
        s->J.ensure((size_t)s->store.g.ncells * 24);
        PICGPU_CUDA_TRY(cudaMemsetAsync(s->J.p, 0, (size_t)s->store.g.ncells * 24, s->st));
        keep_fields_in_l2(s);
        s->timing = (cfg->flags & PICGPU_SESSION_TIMING) != 0;
        for (auto& e : s->ev) PICGPU_CUDA_TRY(cudaEventCreate(&e));
        PICGPU_CUDA_TRY(cudaStreamSynchronize(s->st));
    });
    if (rc) {
        delete s;
        return rc;
    }
    *out = s;
    return PICGPU_OK;
}

int picgpu_session_destroy(picgpu_session* s) {
    if (!s) return PICGPU_OK;
    return guard([&] {
        set_device(s);
        cudaStreamSynchronize(s->st);
        for (auto& e : s->ev)
            if (e) cudaEventDestroy(e);
        if (s->hxcnt) cudaFreeHost(s->hxcnt);
        cudaStream_t st = s->st;
        delete s;
        if (st) cudaStreamDestroy(st);
    });
}

int picgpu_session_upload(picgpu_session* s, uint64_t n, const double* x, const double* y, const double* z,
                          const double* vx, const double* vy, const double* vz, const double* w, const uint64_t* id,
                          double q) {
    return guard([&] {
        set_device(s);
        BinStore& bs = s->store;
        const cudaStream_t st = s->st;
        bs.B.ensure(n);
        const Soa b = bs.B.soa();
        h2d(b.x, x, n * 8, st); h2d(b.y, y, n * 8, st); h2d(b.z, z, n * 8, st);
        h2d(b.vx, vx, n * 8, st); h2d(b.vy, vy, n * 8, st); h2d(b.vz, vz, n * 8, st);
        h2d(b.w, w, n * 8, st);
        if (id)
            h2d(b.id, id, n * 8, st);
        else if (n) {
            k_fill_ids<<<div_up((long long)n, 256), 256, 0, st>>>(b.id, n);
            note_launch();
        }
        bs.full_sort_from_B(n);
        s->q = q;
        PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
    });
}

int picgpu_session_generate_plasma(picgpu_session* s, int ppc, double u_th, uint64_t seed) {
    return guard([&] {
        set_device(s);
        if (ppc < 1) throw Status{PICGPU_EINVAL, "workload: ppc must be >= 1"};
        BinStore& bs = s->store;
        const uint64_t n = (uint64_t)(bs.g.sx_hi - bs.g.sx_lo) * bs.g.ny * bs.g.nz * (uint64_t)ppc;
        bs.B.ensure(n);
        launch_generate_plasma(bs.g, ppc, u_th, seed, bs.B.soa(), s->st);
        bs.full_sort_from_B(n);
        s->q = -1.0;  // electrons
        PICGPU_CUDA_TRY(cudaStreamSynchronize(s->st));
    });
}

int picgpu_session_generate_lwfa(picgpu_session* s, const picgpu_lwfa* c) {
    return guard([&] {
        set_device(s);
        BinStore& bs = s->store;
        if (s->slab) throw Status{PICGPU_ELOGIC, "generate_lwfa: not available on a slab session"};
        const GridD& g = bs.g;
        if (c->ppc < 1 || c->ramp_len < 1 || c->ramp_start < 0)
            throw Status{PICGPU_EINVAL, "generate_lwfa: ppc, ramp_len must be >= 1, ramp_start >= 0"};
        if (!(c->beam_fraction >= 0.0) || !(c->ux_max >= c->ux_min) || !(c->beam_x1 >= c->beam_x0) ||
            c->beam_x0 < 0.0 || c->beam_x1 > g.nx)
            throw Status{PICGPU_EINVAL, "generate_lwfa: bad beam parameters"};
        std::vector<uint32_t> pfx(g.nx + 1, 0u);
        for (int i = 0; i < g.nx; ++i) {
            const double ramp = std::min(1.0, std::max(0.0, (i + 0.5 - c->ramp_start) / c->ramp_len));
            const uint32_t ci = i >= c->ramp_start ? (uint32_t)std::llround(c->ppc * ramp) : 0u;
            pfx[i + 1] = pfx[i] + ci;
        }
        const uint64_t nbg = (uint64_t)pfx[g.nx] * g.ny * g.nz;
        const uint64_t nbeam = (uint64_t)std::llround(c->beam_fraction * (double)nbg);
        const uint64_t n = nbg + nbeam;
        if (n >= 0xffffffffull) throw Status{PICGPU_ELENGTH, "generate_lwfa: more than 2^32-1 particles"};
        DevBuf dp;
        dp.ensure(pfx.size() * 4);
        PICGPU_CUDA_TRY(cudaMemcpyAsync(dp.p, pfx.data(), pfx.size() * 4, cudaMemcpyHostToDevice, s->st));
        bs.B.ensure(n);
        launch_generate_lwfa(g, dp.as<uint32_t>(), nbg, n, c->ppc, c->u_th, c->ux_min, c->ux_max, c->beam_x0,
                             c->beam_x1, c->seed, bs.B.soa(), s->st);
        bs.full_sort_from_B(n);
        s->q = -1.0;
        PICGPU_CUDA_TRY(cudaStreamSynchronize(s->st));
    });
}

int picgpu_session_shift_window(picgpu_session* s, int ppc, double u_th, uint64_t seed, uint64_t pid0,
                                uint64_t* n_dropped, uint64_t* n_injected) {
    return guard([&] {
        set_device(s);
        if (s->slab) throw Status{PICGPU_ELOGIC, "shift_window: not available on a slab session"};
        if (ppc < 0) throw Status{PICGPU_EINVAL, "shift_window: ppc must be >= 0"};
        BinStore& bs = s->store;
        picgpu_grid shifted = bs.hg;
        shifted.ox = bs.hg.ox + bs.hg.dx;
        uint64_t d = 0, in = 0;
        bs.shift_window(shifted, ppc, u_th, seed, pid0, d, in);
        PICGPU_CUDA_TRY(cudaStreamSynchronize(s->st));
        if (n_dropped) *n_dropped = d;
        if (n_injected) *n_injected = in;
    });
}

int picgpu_session_grid(picgpu_session* s, picgpu_grid* out) {
    *out = s->store.hg;
    return PICGPU_OK;
}

static void accumulate_phase(picgpu_session* s, int phase, int e0, int e1, uint64_t launches) {
    float ms = 0.f;
    PICGPU_CUDA_TRY(cudaEventElapsedTime(&ms, s->ev[e0], s->ev[e1]));
    s->phase_ms[phase] += ms;
    s->phase_launches[phase] += launches;
}

// Deposits requested by `flags`, enqueued on the session stream; events
// ev[2..6] bracket them when timing is on.
static void enqueue_deposits(picgpu_session* s, uint32_t flags, uint64_t* lj, uint64_t* lr) {
    BinStore& bs = s->store;
    const cudaStream_t st = s->st;
    const GridD& g = bs.g;
    const bool T = s->timing;
    if (flags & PICGPU_STEP_CURRENT) {
        const uint64_t l0 = g_launches.load();
        if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[2], st));
        PICGPU_CUDA_TRY(cudaMemsetAsync(s->J.p, 0, (size_t)g.ncells * 24, st));
        if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[3], st));
        if (bs.n)
            launch_deposit_current(s->order, g, bs.A.aos(), bs.d_off(), bs.d_cnt(), s->q, s->J.as<double>(),
                                   bs.num_sms, st, s->kernel);
        if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[4], st));
        *lj = g_launches.load() - l0;
    }
    if (flags & PICGPU_STEP_DENSITY) {
        check_density_grid(bs.hg, s->order);
        const uint64_t l0 = g_launches.load();
        if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[5], st));
        // rho is bit-exact on the storage order: pack the bins first, so the
        // order it sums in is the order downloads report
        bs.fill_holes();
        s->rho.ensure((size_t)g.ncells * 8);
        s->dscratch.ensure(density_scratch_bytes(s->order, bs.capacity));
        launch_deposit_density(s->order, g, bs.A.aos(), nullptr, s->q, bs.d_off(), bs.d_cnt(), bs.capacity,
                               s->dscratch.p, s->rho.as<double>(), st);
        if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[6], st));
        *lr = g_launches.load() - l0;
    }
}

// One step of the reference loop (simulation.hpp:92-176), device-resident:
// [push + incremental sort] -> [J] -> [rho] -> [global sort].  The sorter's
// counters are read once after the sort kernels (one host wait per step):
// when an arrival found no slack even after borrowing, the bins are rebuilt
// before anything is deposited on them.
static void adapt_slack(picgpu_session* s, bool rebuilt, bool pushed);

int picgpu_session_step(picgpu_session* s, double dt, uint32_t flags, picgpu_step_stats* out) {
    return guard([&] {
        set_device(s);
        BinStore& bs = s->store;
        const cudaStream_t st = s->st;
        if (s->slab) throw Status{PICGPU_ELOGIC, "session_step: slab sessions step with step_begin / step_end"};
        if ((flags & PICGPU_STEP_SORT) && (flags & PICGPU_STEP_RESORT))
            throw Status{PICGPU_EINVAL, "session_step: SORT and RESORT are exclusive"};
        if ((flags & PICGPU_STEP_PUSH) && !(flags & (PICGPU_STEP_SORT | PICGPU_STEP_RESORT)))
            throw Status{PICGPU_EINVAL, "session_step: PUSH requires SORT or RESORT (the push is fused with them)"};
        if ((flags & PICGPU_STEP_DENSITY)) check_density_grid(bs.hg, s->order);
        picgpu_step_stats stats{};
        const uint64_t rebuilds0 = bs.rebuilds;
        const bool T = s->timing;
        uint64_t lj = 0, lr = 0;
        if (flags & PICGPU_STEP_RESORT) {
            const double cap2 = (flags & PICGPU_STEP_PUSH) ? cap2_of(bs.hg, dt) : 0.0;
            const uint64_t l0 = g_launches.load();
            if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[0], st));
            StepCounters c{};
            bs.push_and_resort((flags & PICGPU_STEP_PUSH) != 0, dt, cap2, c);
            if (c.err == PICGPU_EDOMAIN)
                throw Status{c.err, "advance: particle displacement exceeds the single-cell cap"};
            if (c.err) throw Status{c.err, "cell_of: non-finite particle position"};
            stats.moved = c.moved;
            stats.global_sorted = 1;
            if (T) {
                PICGPU_CUDA_TRY(cudaEventRecord(s->ev[1], st));
                PICGPU_CUDA_TRY(cudaEventSynchronize(s->ev[1]));
                accumulate_phase(s, 2, 0, 1, g_launches.load() - l0);
            }
        }
        // the fused step: push + detect + J in one pass over the bins (movers
        // deposited by their own kernel), then the migration
        const uint32_t fuse_mask = PICGPU_STEP_PUSH | PICGPU_STEP_SORT | PICGPU_STEP_CURRENT;
        // Policy: the fused pass deposits movers' out-of-window taps with L2
        // reductions, so it pays off at low migration and loses at high
        // migration (record store, step times: C2 1.2% per step, fused 1.95 vs
        // 2.3 ms; C4 5.6%, 15.6 vs 16.1 ms; C3 11%, 177 vs 143 ms): fuse while
        // the previous step moved less than PICGPU_FUSE_MAX_MOVED (default 6%).
        const bool fused = (flags & fuse_mask) == fuse_mask && !(flags & PICGPU_STEP_UNFUSED) &&
                           s->last_moved < s->fuse_max && fused_step_available(s->order, s->kernel);
        if (fused) {
            const double cap2 = cap2_of(bs.hg, dt);
            const uint64_t l0 = g_launches.load();
            if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[2], st));
            PICGPU_CUDA_TRY(cudaMemsetAsync(s->J.p, 0, (size_t)bs.g.ncells * 24, st));
            if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[3], st));
            bs.enqueue_fused(s->order, s->q, s->J.as<double>(), dt, cap2, T ? s->ev[4] : nullptr, true, s->kernel);
            if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[1], st));
            lj = g_launches.load() - l0;
            StepCounters c{};
            const size_t mcap0 = bs.mcap;
            const bool rebuilt = bs.finish_incremental(c);  // host waits here
            if (c.err == PICGPU_EDOMAIN)
                throw Status{c.err, "advance: particle displacement exceeds the single-cell cap"};
            if (c.err) throw Status{c.err, "cell_of: non-finite particle position"};
            stats.moved = c.moved;
            stats.fused = 1;
            stats.inserts = std::min<uint64_t>(c.nmovers, mcap0);
            stats.overflowed = c.noverflow;
            if (T) {
                // zero -> ev3 -> fused push + detect + J kernel -> ev4 -> movers + migration -> ev1
                accumulate_phase(s, 5, 2, 3, 0);
                accumulate_phase(s, 3, 3, 4, 1);
                accumulate_phase(s, 0, 4, 1, lj - 1);
                if (rebuilt) {
                    PICGPU_CUDA_TRY(cudaEventRecord(s->ev[7], st));
                    PICGPU_CUDA_TRY(cudaEventSynchronize(s->ev[7]));
                    accumulate_phase(s, 2, 1, 7, g_launches.load() - l0 - lj);
                }
            }
            if (rebuilt && (c.nmovers > mcap0 || c.mover_drop > 0)) {
                // movers beyond the buffer were pushed but neither recorded nor
                // deposited: the store was re-sorted fully, deposit J again
                flags &= ~PICGPU_STEP_SORT;  // (handled) -- J below is redone from scratch
            } else {
                flags &= ~(PICGPU_STEP_SORT | PICGPU_STEP_CURRENT);
            }
        }
        if (flags & PICGPU_STEP_SORT) {
            const double cap2 = (flags & PICGPU_STEP_PUSH) ? cap2_of(bs.hg, dt) : 0.0;
            const uint64_t l0 = g_launches.load();
            if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[0], st));
            bs.enqueue_incremental((flags & PICGPU_STEP_PUSH) != 0, dt, cap2);
            if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[1], st));
            const uint64_t ls = g_launches.load() - l0;
            StepCounters c{};
            const bool rebuilt = bs.finish_incremental(c);  // host waits here
            if (c.err == PICGPU_EDOMAIN)
                throw Status{c.err, "advance: particle displacement exceeds the single-cell cap"};
            if (c.err) throw Status{c.err, "cell_of: non-finite particle position"};
            stats.moved = c.moved;
            stats.inserts = std::min<uint64_t>(c.nmovers, bs.mcap);
            stats.overflowed = c.noverflow;
            if (T) {
                accumulate_phase(s, 0, 0, 1, ls);
                if (rebuilt) {
                    PICGPU_CUDA_TRY(cudaEventRecord(s->ev[7], st));
                    PICGPU_CUDA_TRY(cudaEventSynchronize(s->ev[7]));
                    accumulate_phase(s, 2, 1, 7, g_launches.load() - l0 - ls);
                }
            }
        }
        enqueue_deposits(s, flags, &lj, &lr);
        if (flags & PICGPU_STEP_GLOBAL_SORT) {
            const uint64_t l0 = g_launches.load();
            if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[0], st));
            bs.relayout();
            stats.global_sorted = 1;
            if (T) {
                PICGPU_CUDA_TRY(cudaEventRecord(s->ev[1], st));
                PICGPU_CUDA_TRY(cudaEventSynchronize(s->ev[1]));
                accumulate_phase(s, 2, 0, 1, g_launches.load() - l0);
            }
        }
        if (!(flags & PICGPU_STEP_NO_SYNC) || T) PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
        if (T) {
            if (flags & PICGPU_STEP_CURRENT) {
                accumulate_phase(s, 5, 2, 3, 0);
                accumulate_phase(s, 3, 3, 4, lj);
            }
            if (flags & PICGPU_STEP_DENSITY) accumulate_phase(s, 4, 5, 6, lr);
        }
        if (flags & PICGPU_STEP_PUSH)
            s->last_moved = bs.n ? (double)stats.moved / (double)bs.n : 0.0;
        stats.rebuilt = bs.rebuilds != rebuilds0;
        adapt_slack(s, stats.rebuilt != 0, (flags & PICGPU_STEP_PUSH) != 0);
        stats.capacity = bs.capacity;
        stats.num_particles = bs.n;
        stats.empty_slot_ratio = bs.capacity ? (double)(bs.capacity - bs.n) / (double)bs.capacity : 1.0;
        if (out) *out = stats;
    });
}

// Rebuild storm (an overflow rebuild within 4 pushed steps of the previous
// one): the gap ratio of every later layout (rebuild, window shift, global
// sort) doubles, up to 1.0 (Gpma::layout's rule with a larger gap_ratio,
// gpma.hpp:274-281).  Off by default: capacities then follow the reference.
static void adapt_slack(picgpu_session* s, bool rebuilt, bool pushed) {
    if (!s->adaptive_slack || !pushed) return;
    if (rebuilt) {
        BinStore& bs = s->store;
        if (s->since_rebuild <= 4) bs.onepg = 1.0 + std::min(1.0, 2.0 * (bs.onepg - 1.0) + 0.05);
        s->since_rebuild = 0;
    } else if (s->since_rebuild < 1000) {
        ++s->since_rebuild;
    }
}

int picgpu_session_set_adaptive_slack(picgpu_session* s, int enable) {
    return guard([&] { s->adaptive_slack = enable != 0; });
}

int picgpu_session_set_fusion(picgpu_session* s, double max_moved_fraction) {
    return guard([&] {
        if (!(max_moved_fraction >= 0.0)) throw Status{PICGPU_EINVAL, "set_fusion: threshold must be >= 0"};
        s->fuse_max = max_moved_fraction;
    });
}

int picgpu_session_set_kernel(picgpu_session* s, int family) {
    return guard([&] {
        if (family < -1 || family > 2) throw Status{PICGPU_EINVAL, "set_kernel: family must be 0, 1 or 2"};
        s->kernel = family;
    });
}

int picgpu_session_make_workload(picgpu_session* s, const picgpu_workload* cfg) {
    return guard([&] {
        set_device(s);
        BinStore& bs = s->store;
        if (s->slab) throw Status{PICGPU_ELOGIC, "make_workload: not available on a slab session"};
        const picgpu_grid& h = bs.hg;
        const picgpu_grid& c = cfg->grid;
        if (h.nx != c.nx || h.ny != c.ny || h.nz != c.nz || h.dx != c.dx || h.dy != c.dy || h.dz != c.dz ||
            h.ox != c.ox || h.oy != c.oy || h.oz != c.oz)
            throw Status{PICGPU_EINVAL, "make_workload: grid differs from the session's"};
        // WorkloadConfig::validate (workload.hpp:29-40)
        if (cfg->ppc < 1) throw Status{PICGPU_EINVAL, "workload: ppc must be >= 1"};
        if (!(cfg->dt > 0.0)) throw Status{PICGPU_EINVAL, "workload: dt must be positive"};
        if (cfg->steps < 0) throw Status{PICGPU_EINVAL, "workload: steps must be >= 0"};
        if (cfg->thermal_speed < 0.0) throw Status{PICGPU_EINVAL, "workload: thermal_speed must be >= 0"};
        check_order(cfg->order);
        const int W = cfg->order == 1 ? 2 : cfg->order == 2 ? 3 : 4;
        if (c.nx < W || c.ny < W || c.nz < W)
            throw Status{PICGPU_EINVAL, "workload: grid smaller than the shape stencil"};
        const double cap = std::min(c.dx, std::min(c.dy, c.dz)) / cfg->dt;  // speed_cap
        double amp[3] = {cfg->drift[0], cfg->drift[1], cfg->drift[2]};
        const int drift = cfg->kind == PICGPU_WORKLOAD_DRIFT_GRADIENT;
        if (drift && amp[0] == 0.0 && amp[1] == 0.0 && amp[2] == 0.0) amp[0] = 0.5 * cap;
        const uint64_t n = (uint64_t)bs.g.ncells * (uint64_t)cfg->ppc;
        bs.B.ensure(n);
        launch_make_workload(bs.g, cfg->ppc, cfg->thermal_speed, drift, amp, cap, cfg->seed, bs.B.soa(), s->st);
        bs.full_sort_from_B(n);
        s->q = cfg->charge;
        PICGPU_CUDA_TRY(cudaStreamSynchronize(s->st));
    });
}

int picgpu_session_global_sort(picgpu_session* s) {
    return guard([&] {
        set_device(s);
        s->store.relayout();
        PICGPU_CUDA_TRY(cudaStreamSynchronize(s->st));
    });
}

int picgpu_session_synchronize(picgpu_session* s) {
    return guard([&] {
        set_device(s);
        PICGPU_CUDA_TRY(cudaStreamSynchronize(s->st));
    });
}

uint64_t picgpu_session_num_particles(picgpu_session* s) { return s->store.n; }
uint64_t picgpu_session_capacity(picgpu_session* s) { return s->store.capacity; }
void* picgpu_session_stream(picgpu_session* s) { return (void*)s->st; }

int picgpu_session_download_particles(picgpu_session* s, double* x, double* y, double* z, double* vx, double* vy,
                                      double* vz, double* w, uint64_t* id) {
    return guard([&] {
        set_device(s);
        BinStore& bs = s->store;
        const cudaStream_t st = s->st;
        bs.compact_to_B();
        const Soa b = bs.B.soa();
        const size_t n = bs.n;
        d2h(x, b.x, n * 8, st); d2h(y, b.y, n * 8, st); d2h(z, b.z, n * 8, st);
        d2h(vx, b.vx, n * 8, st); d2h(vy, b.vy, n * 8, st); d2h(vz, b.vz, n * 8, st);
        d2h(w, b.w, n * 8, st); d2h(id, b.id, n * 8, st);
        PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
    });
}

int picgpu_session_download_bins(picgpu_session* s, uint32_t* bin_offset, uint32_t* bin_count) {
    return guard([&] {
        set_device(s);
        const size_t nc = s->store.g.ncells;
        std::vector<uint32_t> h(nc);
        d2h(bin_offset, s->store.off.p, (nc + 1) * 4, s->st);
        d2h(bin_count, s->store.cnt.p, nc * 4, s->st);
        if (nc) d2h(h.data(), s->store.holes.p, nc * 4, s->st);
        PICGPU_CUDA_TRY(cudaStreamSynchronize(s->st));
        for (size_t c = 0; c < nc; ++c) bin_count[c] -= h[c];  // particles, not extent (holes are gaps)
    });
}

int picgpu_session_download_current(picgpu_session* s, double* jx, double* jy, double* jz) {
    return guard([&] {
        set_device(s);
        const size_t nc = s->store.g.ncells;
        const double* J = s->J.as<double>();
        d2h(jx, J, nc * 8, s->st);
        d2h(jy, J + nc, nc * 8, s->st);
        d2h(jz, J + 2 * nc, nc * 8, s->st);
        PICGPU_CUDA_TRY(cudaStreamSynchronize(s->st));
    });
}

int picgpu_session_download_density(picgpu_session* s, double* rho) {
    return guard([&] {
        set_device(s);
        if (!s->rho.p) throw Status{PICGPU_ELOGIC, "session: no density deposited yet"};
        d2h(rho, s->rho.p, (size_t)s->store.g.ncells * 8, s->st);
        PICGPU_CUDA_TRY(cudaStreamSynchronize(s->st));
    });
}

int picgpu_session_device_fields(picgpu_session* s, double** j, double** rho) {
    if (j) *j = s->J.as<double>();
    if (rho) *rho = s->rho.as<double>();
    return PICGPU_OK;
}

int picgpu_session_phase_times(picgpu_session* s, double* ms, uint64_t* launches, int nphases) {
    for (int i = 0; i < nphases && i < PICGPU_NPHASES; ++i) {
        if (ms) ms[i] = s->phase_ms[i];
        if (launches) launches[i] = s->phase_launches[i];
    }
    return PICGPU_OK;
}

int picgpu_session_reset_phase_times(picgpu_session* s) {
    for (int i = 0; i < PICGPU_NPHASES; ++i) {
        s->phase_ms[i] = 0.0;
        s->phase_launches[i] = 0;
    }
    return PICGPU_OK;
}

// ---- x-slab decomposition ---------------------------------------------------

static void slab_grid(const picgpu_grid* G, int x0, int x1, int ghost, picgpu_grid* L) {
    make_grid(*G);
    if (!(0 <= x0 && x0 < x1 && x1 <= G->nx)) throw Status{PICGPU_EINVAL, "slab: need 0 <= x0 < x1 <= nx"};
    if (ghost < 2) throw Status{PICGPU_EINVAL, "slab: ghost must be >= 2 (QSP stencil reach)"};
    if (x1 - x0 < ghost) throw Status{PICGPU_EINVAL, "slab: a slab must own at least `ghost` x-cells"};
    *L = *G;
    L->nx = x1 - x0 + 2 * ghost;
    L->ox = G->ox + (double)(x0 - ghost) * G->dx;
}

int picgpu_slab_grid(const picgpu_grid* G, int x0, int x1, int ghost, picgpu_grid* L) {
    return guard([&] { slab_grid(G, x0, x1, ghost, L); });
}

int picgpu_session_set_slab(picgpu_session* s, const picgpu_grid* G, int x0, int x1, int ghost) {
    return guard([&] {
        BinStore& bs = s->store;
        if (bs.n || bs.capacity) throw Status{PICGPU_ELOGIC, "set_slab: the session must be empty"};
        picgpu_grid L{};
        slab_grid(G, x0, x1, ghost, &L);
        const picgpu_grid& h = bs.hg;
        if (h.nx != L.nx || h.ny != L.ny || h.nz != L.nz || h.dx != L.dx || h.dy != L.dy || h.dz != L.dz ||
            h.ox != L.ox || h.oy != L.oy || h.oz != L.oz)
            throw Status{PICGPU_EINVAL, "set_slab: session grid is not picgpu_slab_grid(global, x0, x1, ghost)"};
        GridD& g = bs.g;
        g.slab = 1;
        g.gnx = G->nx;
        g.sx_shift = x0 - ghost;
        g.sx_lo = ghost;
        g.sx_hi = ghost + (x1 - x0);
        g.gox = G->ox;
        g.gLx = G->nx * G->dx;
        g.ginv_Lx = 1.0 / g.gLx;
        g.gpow2Lx = is_pow2(g.gLx);
        s->slab = true;
        s->ghost = ghost;
        s->own = x1 - x0;
    });
}

static void throw_step_error(int err) {
    if (err == PICGPU_EDOMAIN) throw Status{err, "advance: particle displacement exceeds the single-cell cap"};
    if (err == PICGPU_ELENGTH) throw Status{err, "slab: leaver exchange buffer overflow"};
    throw Status{err, "cell_of: non-finite particle position (or arrival outside the slab)"};
}

int picgpu_session_step_begin(picgpu_session* s, double dt, uint32_t flags, uint64_t* n_to_left,
                              uint64_t* n_to_right) {
    return guard([&] {
        set_device(s);
        BinStore& bs = s->store;
        if (s->pending) throw Status{PICGPU_ELOGIC, "step_begin: previous step not ended"};
        if (!(flags & PICGPU_STEP_SORT)) throw Status{PICGPU_EINVAL, "step_begin: SORT is required"};
        if (flags & PICGPU_STEP_DENSITY) check_density_grid(bs.hg, s->order);
        const double cap2 = (flags & PICGPU_STEP_PUSH) ? cap2_of(bs.hg, dt) : 0.0;
        const uint64_t l0 = g_launches.load();
        // the fused step as on a whole box: push + detect + J of the particles
        // that stay on the slab (leavers are exported undeposited; the receiver
        // deposits its arrivals in step_end)
        const uint32_t fuse_mask = PICGPU_STEP_PUSH | PICGPU_STEP_SORT | PICGPU_STEP_CURRENT;
        const bool fused = (flags & fuse_mask) == fuse_mask && !(flags & PICGPU_STEP_UNFUSED) &&
                           s->last_moved < s->fuse_max && fused_step_available(s->order, s->kernel);
        if (s->timing) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[0], s->st));
        if (fused) {
            PICGPU_CUDA_TRY(cudaMemsetAsync(s->J.p, 0, (size_t)bs.g.ncells * 24, s->st));
            bs.enqueue_fused(s->order, s->q, s->J.as<double>(), dt, cap2, s->timing ? s->ev[4] : nullptr,
                             /*migrate=*/false, s->kernel);
        } else {
            bs.enqueue_detect((flags & PICGPU_STEP_PUSH) != 0, dt, cap2);
        }
        if (s->timing) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[1], s->st));
        PICGPU_CUDA_TRY(
            cudaMemcpyAsync(bs.hcounters, bs.counters.p, sizeof(StepCounters), cudaMemcpyDeviceToHost, s->st));
        PICGPU_CUDA_TRY(cudaStreamSynchronize(s->st));
        const StepCounters c = *bs.hcounters;
        if (c.err) throw_step_error(c.err);
        if (s->timing) {
            if (fused) {  // zero + fused kernel -> deposit J; the movers -> sort
                accumulate_phase(s, 3, 0, 4, 1);
                accumulate_phase(s, 0, 4, 1, g_launches.load() - l0 - 1);
            } else {
                accumulate_phase(s, 0, 0, 1, g_launches.load() - l0);
            }
        }
        s->pending_fused = fused;
        s->cbegin = c;
        s->nleave[0] = c.nleave[0];
        s->nleave[1] = c.nleave[1];
        s->pending = true;
        s->pending_flags = flags;
        if (n_to_left) *n_to_left = c.nleave[0];
        if (n_to_right) *n_to_right = c.nleave[1];
    });
}

int picgpu_session_copy_leavers(picgpu_session* s, double* to_left, double* to_right) {
    return guard([&] {
        set_device(s);
        if (!s->pending) throw Status{PICGPU_ELOGIC, "copy_leavers: no step in progress"};
        BinStore& bs = s->store;
        const double* L = bs.lrec.as<double>();
        if (s->nleave[0])
            PICGPU_CUDA_TRY(cudaMemcpyAsync(to_left, L, s->nleave[0] * 64, cudaMemcpyDeviceToDevice, s->st));
        if (s->nleave[1])
            PICGPU_CUDA_TRY(
                cudaMemcpyAsync(to_right, L + bs.lcap * 8, s->nleave[1] * 64, cudaMemcpyDeviceToDevice, s->st));
        PICGPU_CUDA_TRY(cudaStreamSynchronize(s->st));
    });
}

int picgpu_session_step_end(picgpu_session* s, const double* arrivals, uint64_t n_arr, picgpu_step_stats* out) {
    return guard([&] {
        set_device(s);
        if (!s->pending) throw Status{PICGPU_ELOGIC, "step_end: no step in progress"};
        s->pending = false;
        BinStore& bs = s->store;
        const cudaStream_t st = s->st;
        const uint32_t flags = s->pending_flags;
        const bool T = s->timing;
        const uint64_t rebuilds0 = bs.rebuilds;
        const StepCounters& cb = s->cbegin;
        const uint64_t l0 = g_launches.load();
        if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[0], st));
        const size_t base = std::min<size_t>(cb.nmovers, bs.mcap);
        if (cb.nmovers > bs.mcap) bs.movers_dropped = true;
        const size_t mcap0 = bs.mcap;
        if (n_arr) {
            if (n_arr >= 0xffffffffull) throw Status{PICGPU_ELENGTH, "slab: too many arrivals"};
            bs.ensure_movers_keep(base + n_arr + (base + n_arr) / 4, base);
            bs.enqueue_import(arrivals, (uint32_t)n_arr, (uint32_t)base);
            if (s->pending_fused)  // the sender left them out of its fused deposit
                launch_deposit_records(s->order, bs.g, bs.M.soa(), bs.counters.as<StepCounters>(), (uint32_t)base,
                                       s->q, s->J.as<double>(), bs.num_sms, st);
        }
        bs.n = bs.n - s->nleave[0] - s->nleave[1] + n_arr;
        bs.enqueue_migrate();
        if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[1], st));
        const uint64_t lm = g_launches.load() - l0;
        StepCounters c{};
        const bool rebuilt = bs.finish_incremental(c);  // host waits here
        if (c.err) throw_step_error(c.err);
        picgpu_step_stats stats{};
        stats.moved = cb.moved;
        stats.inserts = base + n_arr;
        stats.overflowed = c.noverflow;
        uint32_t dflags = flags;
        if (s->pending_fused) {
            stats.fused = 1;
            // J is complete unless movers were dropped (full re-sort): redo it then
            if (!(rebuilt && (c.mover_drop > 0 || cb.nmovers > mcap0))) dflags &= ~PICGPU_STEP_CURRENT;
        }
        if (T) {
            accumulate_phase(s, 0, 0, 1, lm);
            if (rebuilt) {
                PICGPU_CUDA_TRY(cudaEventRecord(s->ev[7], st));
                PICGPU_CUDA_TRY(cudaEventSynchronize(s->ev[7]));
                accumulate_phase(s, 2, 1, 7, g_launches.load() - l0 - lm);
            }
        }
        uint64_t lj = 0, lr = 0;
        enqueue_deposits(s, dflags, &lj, &lr);
        PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
        if (T) {
            if (dflags & PICGPU_STEP_CURRENT) {
                accumulate_phase(s, 5, 2, 3, 0);
                accumulate_phase(s, 3, 3, 4, lj);
            }
            if (dflags & PICGPU_STEP_DENSITY) accumulate_phase(s, 4, 5, 6, lr);
        }
        if (flags & PICGPU_STEP_PUSH)
            s->last_moved = bs.n ? (double)stats.moved / (double)bs.n : 0.0;
        stats.rebuilt = bs.rebuilds != rebuilds0;
        adapt_slack(s, stats.rebuilt != 0, (flags & PICGPU_STEP_PUSH) != 0);
        stats.capacity = bs.capacity;
        stats.num_particles = bs.n;
        stats.empty_slot_ratio = bs.capacity ? (double)(bs.capacity - bs.n) / (double)bs.capacity : 1.0;
        if (out) *out = stats;
    });
}

static double* slab_field(picgpu_session* s, int field, int& comps) {
    if (!s->slab) throw Status{PICGPU_ELOGIC, "guard planes: not a slab session"};
    if (field == 0) {
        comps = 3;
        return s->J.as<double>();
    }
    if (field == 1) {
        if (!s->rho.p) throw Status{PICGPU_ELOGIC, "guard planes: no density deposited yet"};
        comps = 1;
        return s->rho.as<double>();
    }
    throw Status{PICGPU_EINVAL, "guard planes: field must be 0 (J) or 1 (rho)"};
}

int picgpu_session_guard_planes(picgpu_session* s, int field, double* lo, double* hi) {
    return guard([&] {
        set_device(s);
        int comps = 0;
        double* F = slab_field(s, field, comps);
        const GridD& g = s->store.g;
        launch_pack_planes(F, comps, g.nx, g.ny, g.nz, 0, s->ghost, lo, s->st);
        launch_pack_planes(F, comps, g.nx, g.ny, g.nz, s->ghost + s->own, s->ghost, hi, s->st);
        PICGPU_CUDA_TRY(cudaStreamSynchronize(s->st));
    });
}

int picgpu_session_add_guard_planes(picgpu_session* s, int field, const double* from_left,
                                    const double* from_right) {
    return guard([&] {
        set_device(s);
        int comps = 0;
        double* F = slab_field(s, field, comps);
        const GridD& g = s->store.g;
        launch_add_planes(F, comps, g.nx, g.ny, g.nz, s->ghost, s->ghost, from_left, s->st);
        launch_add_planes(F, comps, g.nx, g.ny, g.nz, s->own, s->ghost, from_right, s->st);
        PICGPU_CUDA_TRY(cudaStreamSynchronize(s->st));
    });
}

}  // extern "C"

// ---- FP64 peak microbenchmark (roofline denominator, measured in-run) -------

namespace picgpu {
__global__ void k_dfma_peak(double* out, int iters, double a, double b) {
    double r0 = threadIdx.x, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3, r4 = r0 + 4, r5 = r0 + 5, r6 = r0 + 6,
           r7 = r0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            r0 = fma(r0, a, b); r1 = fma(r1, a, b); r2 = fma(r2, a, b); r3 = fma(r3, a, b);
            r4 = fma(r4, a, b); r5 = fma(r5, a, b); r6 = fma(r6, a, b); r7 = fma(r7, a, b);
        }
    }
    const double s = r0 + r1 + r2 + r3 + r4 + r5 + r6 + r7;
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}
}  // namespace picgpu

extern "C" int picgpu_fp64_peak(int device, double* tflops) {
    return guard([&] {
        PICGPU_CUDA_TRY(cudaSetDevice(device));
        const int sms = current_sms();
        DevBuf out;
        out.ensure(64);
        cudaStream_t st;
        PICGPU_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        cudaEvent_t e0, e1;
        PICGPU_CUDA_TRY(cudaEventCreate(&e0));
        PICGPU_CUDA_TRY(cudaEventCreate(&e1));
        const int blocks = sms * 4, threads = 256, iters = 4096;
        k_dfma_peak<<<blocks, threads, 0, st>>>(out.as<double>(), 64, 0.999, 1e-3);  // warm-up
        note_launch();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            PICGPU_CUDA_TRY(cudaEventRecord(e0, st));
            k_dfma_peak<<<blocks, threads, 0, st>>>(out.as<double>(), iters, 0.999, 1e-3);
            note_launch();
            PICGPU_CUDA_TRY(cudaEventRecord(e1, st));
            PICGPU_CUDA_TRY(cudaEventSynchronize(e1));
            float ms = 0;
            PICGPU_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
            best = std::min(best, ms);
        }
        PICGPU_CUDA_TRY(cudaGetLastError());
        const double flops = 2.0 * 64.0 * iters * (double)blocks * threads;
        *tflops = flops / (best * 1e-3) / 1e12;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaStreamDestroy(st);
    });
}

// ===========================================================================
// multi-GPU: NCCL behind the C ABI (comm.hpp)

int picgpu_comm_unique_id(unsigned char id[128]) {
    return guard([&] {
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
        ncclUniqueId u;
        nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId failed");
        std::memcpy(id, &u, 128);
    });
}

int picgpu_comm_init(const unsigned char id[128], int nranks, int rank, int device, picgpu_comm** out) {
    *out = nullptr;
    return guard([&] {
        if (nranks < 1 || rank < 0 || rank >= nranks) throw Status{PICGPU_EINVAL, "comm_init: bad rank / size"};
        PICGPU_CUDA_TRY(cudaSetDevice(device));
        ncclUniqueId u;
        std::memcpy(&u, id, 128);
        auto* c = new picgpu_comm;
        const ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, u, rank);
        if (r != ncclSuccess) {
            delete c;
            nccl_check(r, "ncclCommInitRank failed");
        }
        c->rank = rank;
        c->nranks = nranks;
        c->device = device;
        c->owned = true;
        *out = c;
    });
}

int picgpu_comm_wrap(void* nccl_comm, int device, picgpu_comm** out) {
    *out = nullptr;
    return guard([&] {
        if (!nccl_comm) throw Status{PICGPU_EINVAL, "comm_wrap: null communicator"};
        auto* c = new picgpu_comm;
        c->comm = static_cast<ncclComm_t>(nccl_comm);
        const Nccl& N = nccl();
        int n = 0, r = 0;
        const ncclResult_t a = N.CommCount(c->comm, &n), b = N.CommUserRank(c->comm, &r);
        if (a != ncclSuccess || b != ncclSuccess) {
            delete c;
            throw Status{PICGPU_ENCCL, "comm_wrap: not a usable ncclComm_t of this process's NCCL"};
        }
        c->nranks = n;
        c->rank = r;
        c->device = device;
        *out = c;
    });
}

int picgpu_comm_destroy(picgpu_comm* c) {
    if (!c) return PICGPU_OK;
    return guard([&] {
        if (c->owned && c->comm) nccl().CommDestroy(c->comm);
        delete c;
    });
}

int picgpu_comm_rank(const picgpu_comm* c, int* rank, int* nranks) {
    return guard([&] {
        if (!c) throw Status{PICGPU_EINVAL, "comm_rank: null communicator"};
        if (rank) *rank = c->rank;
        if (nranks) *nranks = c->nranks;
    });
}

int picgpu_session_set_comm(picgpu_session* s, picgpu_comm* c, uint32_t bucket_records) {
    return guard([&] {
        if (!s->slab) throw Status{PICGPU_ELOGIC, "set_comm: not a slab session (picgpu_session_set_slab first)"};
        if (c && c->device != s->device) throw Status{PICGPU_EINVAL, "set_comm: communicator of another device"};
        s->comm = c;
        s->bucket = bucket_records ? bucket_records : 32768u;
        set_device(s);
        if (!s->hxcnt) PICGPU_CUDA_TRY(cudaMallocHost((void**)&s->hxcnt, 16));
    });
}

// Send my `to_right` / `to_left` and receive `from_left` / `from_right` (ring
// neighbours of the communicator) in one NCCL group on the session stream.
// Issue order per peer is [right-going, left-coming, left-going, right-coming],
// so the pairing holds when both neighbours are one rank (2 ranks) or this
// rank itself (1 rank).
static void ring_exchange(picgpu_session* s, const void* to_right, const void* to_left, void* from_left,
                          void* from_right, size_t count_r, size_t count_l, size_t count_fl, size_t count_fr,
                          ncclDataType_t type) {
    const Nccl& N = nccl();
    const picgpu_comm* c = s->comm;
    const int L = (c->rank - 1 + c->nranks) % c->nranks, R = (c->rank + 1) % c->nranks;
    nccl_check(N.GroupStart(), "ncclGroupStart failed");
    if (count_r) nccl_check(N.Send(to_right, count_r, type, R, c->comm, s->st), "ncclSend failed");
    if (count_fl) nccl_check(N.Recv(from_left, count_fl, type, L, c->comm, s->st), "ncclRecv failed");
    if (count_l) nccl_check(N.Send(to_left, count_l, type, L, c->comm, s->st), "ncclSend failed");
    if (count_fr) nccl_check(N.Recv(from_right, count_fr, type, R, c->comm, s->st), "ncclRecv failed");
    nccl_check(N.GroupEnd(), "ncclGroupEnd failed");
}

// Guard-plane sums of J (and rho) over NCCL: planes [0, ghost) go left and
// [ghost + own, 2 ghost + own) right, added into the neighbours' first / last
// owned planes (picgpu_session_guard_planes + add_guard_planes, device-resident).
static void exchange_planes(picgpu_session* s, int field) {
    int comps = 0;
    double* F = slab_field(s, field, comps);
    const GridD& g = s->store.g;
    const size_t np = (size_t)comps * s->ghost * g.ny * g.nz;
    s->psend.ensure(2 * np * 8);
    s->precv.ensure(2 * np * 8);
    double* lo = s->psend.as<double>();
    double* hi = lo + np;
    double* fl = s->precv.as<double>();
    double* fr = fl + np;
    launch_pack_planes(F, comps, g.nx, g.ny, g.nz, 0, s->ghost, lo, s->st);
    launch_pack_planes(F, comps, g.nx, g.ny, g.nz, s->ghost + s->own, s->ghost, hi, s->st);
    ring_exchange(s, hi, lo, fl, fr, np, np, np, np, ncclFloat64);
    launch_add_planes(F, comps, g.nx, g.ny, g.nz, s->ghost, s->ghost, fl, s->st);
    launch_add_planes(F, comps, g.nx, g.ny, g.nz, s->own, s->ghost, fr, s->st);
}

int picgpu_session_slab_step(picgpu_session* s, double dt, uint32_t flags, picgpu_step_stats* out) {
    return guard([&] {
        set_device(s);
        if (!s->slab || !s->comm) throw Status{PICGPU_ELOGIC, "slab_step: no communicator (picgpu_session_set_comm)"};
        if (s->pending) throw Status{PICGPU_ELOGIC, "slab_step: a step_begin is pending"};
        if (!(flags & PICGPU_STEP_SORT)) throw Status{PICGPU_EINVAL, "slab_step: SORT is required"};
        BinStore& bs = s->store;
        if (flags & PICGPU_STEP_DENSITY) check_density_grid(bs.hg, s->order);
        const cudaStream_t st = s->st;
        const bool T = s->timing;
        const uint32_t B = s->bucket;
        const double cap2 = (flags & PICGPU_STEP_PUSH) ? cap2_of(bs.hg, dt) : 0.0;
        const uint64_t l0 = g_launches.load();
        const uint64_t rebuilds0 = bs.rebuilds;
        // room for the own movers and two buckets of arrivals; leaver records for a bucket
        bs.ensure_movers(std::max<size_t>(size_t(1) << 16, bs.n / 4) + 2 * (size_t)B);
        if (bs.lcap < B) {
            bs.lrec.ensure((size_t)B * 2 * 8 * sizeof(double));
            bs.lcap = B;
        }
        const uint32_t fuse_mask = PICGPU_STEP_PUSH | PICGPU_STEP_SORT | PICGPU_STEP_CURRENT;
        const bool fused = (flags & fuse_mask) == fuse_mask && !(flags & PICGPU_STEP_UNFUSED) &&
                           s->last_moved < s->fuse_max && fused_step_available(s->order, s->kernel);
        if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[0], st));
        if (fused) {
            PICGPU_CUDA_TRY(cudaMemsetAsync(s->J.p, 0, (size_t)bs.g.ncells * 24, st));
            bs.enqueue_fused(s->order, s->q, s->J.as<double>(), dt, cap2, T ? s->ev[4] : nullptr, /*migrate=*/false,
                             s->kernel);
        } else {
            bs.enqueue_detect((flags & PICGPU_STEP_PUSH) != 0, dt, cap2);
        }
        if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[1], st));
        // leaver counts and the first B records per side, device to device
        StepCounters* ctr = bs.counters.as<StepCounters>();
        s->xcnt.ensure(16);
        s->xin.ensure((size_t)2 * B * 64);
        uint32_t* xcnt = s->xcnt.as<uint32_t>();
        double* xin = s->xin.as<double>();
        const double* lrec = bs.lrec.as<double>();
        ring_exchange(s, &ctr->nleave[1], &ctr->nleave[0], xcnt, xcnt + 1, 1, 1, 1, 1, ncclUint32);
        ring_exchange(s, lrec + bs.lcap * 8, lrec, xin, xin + (size_t)B * 8, (size_t)B * 8, (size_t)B * 8,
                      (size_t)B * 8, (size_t)B * 8, ncclFloat64);
        bs.enqueue_import_dev(xin, xin + (size_t)B * 8, xcnt, B);
        if (fused)  // the senders left their leavers out of the fused deposit
            launch_deposit_records(s->order, bs.g, bs.M.soa(), ctr, kBaseFromCounters, s->q, s->J.as<double>(),
                                   bs.num_sms, st);
        bs.enqueue_migrate();  // (copies the counters to the host)
        PICGPU_CUDA_TRY(cudaMemcpyAsync(s->hxcnt, xcnt, 8, cudaMemcpyDeviceToHost, st));
        if (T) PICGPU_CUDA_TRY(cudaEventRecord(s->ev[2], st));
        // ---- the step's one host synchronisation
        PICGPU_CUDA_TRY(cudaStreamSynchronize(st));
        StepCounters c1 = *bs.hcounters;
        if (c1.err) throw_step_error(c1.err);
        const uint32_t got_l = s->hxcnt[0], got_r = s->hxcnt[1];
        const uint64_t sent = (uint64_t)c1.nleave[0] + c1.nleave[1];
        bs.n = bs.n - sent + c1.nimport;
        if (T) {
            if (fused) {
                accumulate_phase(s, 3, 0, 4, 1);
                accumulate_phase(s, 0, 4, 2, g_launches.load() - l0 - 1);
            } else {
                accumulate_phase(s, 0, 0, 2, g_launches.load() - l0);
            }
        }
        const bool movers_lost = c1.nmovers > bs.mcap || c1.mover_drop > 0;
        StepCounters c{};
        bool rebuilt = bs.finish_incremental(c);
        if (c.err) throw_step_error(c.err);
        uint64_t imported = c1.nimport;
        // ---- rare: a side sent more than its bucket -> the remainder, exactly sized
        const uint32_t rs_r = c1.nleave[1] > B ? c1.nleave[1] - B : 0, rs_l = c1.nleave[0] > B ? c1.nleave[0] - B : 0;
        const uint32_t rr_l = got_l > B ? got_l - B : 0, rr_r = got_r > B ? got_r - B : 0;
        if (rs_r | rs_l | rr_l | rr_r) {
            const uint32_t nrem = rr_l + rr_r;
            s->xin2.ensure(((size_t)nrem + 1) * 64);
            double* x2 = s->xin2.as<double>();
            ring_exchange(s, lrec + (bs.lcap + B) * 8, lrec + (size_t)B * 8, x2, x2 + (size_t)rr_l * 8,
                          (size_t)rs_r * 8, (size_t)rs_l * 8, (size_t)rr_l * 8, (size_t)rr_r * 8, ncclFloat64);
            PICGPU_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(StepCounters), st));
            bs.ensure_movers_keep(std::max<size_t>(bs.mcap, nrem + nrem / 4), 0);
            bs.enqueue_import(x2, nrem, 0);
            if (fused)
                launch_deposit_records(s->order, bs.g, bs.M.soa(), ctr, 0, s->q, s->J.as<double>(), bs.num_sms, st);
            bs.enqueue_migrate();
            bs.n += nrem;
            imported += nrem;
            StepCounters c2{};
            rebuilt |= bs.finish_incremental(c2);
            if (c2.err) throw_step_error(c2.err);
        }
        picgpu_step_stats stats{};
        stats.moved = c1.moved;
        stats.inserts = std::min<uint64_t>(c1.nmovers, bs.mcap) + imported;
        stats.overflowed = c.noverflow;
        uint32_t dflags = flags;
        if (fused) {
            stats.fused = 1;
            if (!(rebuilt && movers_lost)) dflags &= ~PICGPU_STEP_CURRENT;  // J complete
        }
        uint64_t lj = 0, lr = 0;
        enqueue_deposits(s, dflags, &lj, &lr);
        if (flags & PICGPU_STEP_CURRENT) exchange_planes(s, 0);
        if (flags & PICGPU_STEP_DENSITY) exchange_planes(s, 1);
        if (flags & PICGPU_STEP_PUSH) s->last_moved = bs.n ? (double)stats.moved / (double)bs.n : 0.0;
        stats.rebuilt = bs.rebuilds != rebuilds0;
        adapt_slack(s, stats.rebuilt != 0, (flags & PICGPU_STEP_PUSH) != 0);
        stats.capacity = bs.capacity;
        stats.num_particles = bs.n;
        stats.empty_slot_ratio = bs.capacity ? (double)(bs.capacity - bs.n) / (double)bs.capacity : 1.0;
        if (out) *out = stats;
        // no trailing synchronisation: the deposits and the plane exchange stay
        // enqueued on the session stream (downloads and the next step follow them)
    });
}
