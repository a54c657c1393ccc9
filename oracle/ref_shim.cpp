// ref_shim.cpp -- extern "C" wrappers around the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile straight from the
// read-only reference tree (-I /root/reference/proj/include) into
// oracle/_ref/libpicref.so.  No reference source is copied into this repo:
// this file only includes the headers and marshals plain pointers in and out,
// so tests and bench.py's CPU baseline can run the reference's own functions:
//   pic::deposit_scalar      proj/include/pic/deposit.hpp:62
//   pic::deposit_density     proj/include/pic/deposit.hpp:76
//   pic::deposit_tiled       proj/include/pic/deposit.hpp:284
//   pic::gpma_build          proj/include/pic/gpma.hpp:379
//   pic::Gpma::detect_moves  proj/include/pic/gpma.hpp:162
//   pic::apply_pending_moves proj/include/pic/gpma.hpp:373
//   pic::advance             proj/include/pic/workload.hpp:139
//   pic::should_global_sort  proj/include/pic/sort_policy.hpp:62
#include <pic/deposit.hpp>
#include <pic/gpma.hpp>
#include <pic/rng.hpp>
#include <pic/simulation.hpp>
#include <pic/sort_policy.hpp>
#include <pic/workload.hpp>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

struct RefGrid {  // same layout as picgpu_grid (include/picgpu.h)
    int32_t nx, ny, nz, pad;
    double dx, dy, dz;
    double ox, oy, oz;
};

pic::GridSpec to_spec(const RefGrid* g) {
    pic::GridSpec s;
    s.nx = g->nx; s.ny = g->ny; s.nz = g->nz;
    s.dx = g->dx; s.dy = g->dy; s.dz = g->dz;
    s.origin = {g->ox, g->oy, g->oz};
    return s;
}

pic::ShapeOrder to_order(int o) {
    if (o == 1) return pic::ShapeOrder::cic;
    if (o == 3) return pic::ShapeOrder::qsp;
    throw std::invalid_argument("reference supports shape orders 1 and 3 only");
}

thread_local std::string g_err;

// Status codes mirror include/picgpu.h.
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) { g_err = e.what(); return 1; }
    catch (const std::out_of_range& e) { g_err = e.what(); return 2; }
    catch (const std::length_error& e) { g_err = e.what(); return 3; }
    catch (const std::domain_error& e) { g_err = e.what(); return 5; }
    catch (const std::logic_error& e) { g_err = e.what(); return 4; }
    catch (const std::exception& e) { g_err = e.what(); return 9; }
}

struct RefState {
    pic::GridSpec grid;
    pic::ParticleSoA soa;
    pic::Gpma gpma;
    bool has_gpma = false;
};

void copy_out(const std::vector<double>& v, double* out) {
    if (out) std::memcpy(out, v.data(), v.size() * sizeof(double));
}

struct RefWorkload {  // same layout as picgpu_workload
    RefGrid grid;
    int32_t ppc, kind;
    double thermal_speed;
    double drift[3];
    uint64_t seed;
    int32_t steps, order;
    double dt, charge;
};

struct RefPolicy {  // same layout as picgpu_sort_policy
    uint32_t sort_interval, min_sort_interval, trigger_rebuild_count, perf_enable;
    double trigger_empty_ratio, trigger_full_ratio, perf_degrad;
};

pic::WorkloadConfig to_cfg(const RefWorkload* w) {
    pic::WorkloadConfig c;
    c.grid = to_spec(&w->grid);
    c.ppc = w->ppc;
    c.kind = w->kind ? pic::WorkloadKind::drift_gradient : pic::WorkloadKind::uniform_plasma;
    c.thermal_speed = w->thermal_speed;
    c.drift_velocity = {w->drift[0], w->drift[1], w->drift[2]};
    c.seed = w->seed;
    c.steps = w->steps;
    c.dt = w->dt;
    c.charge = w->charge;
    c.order = to_order(w->order);
    return c;
}

void soa_out(const pic::ParticleSoA& s, double* x, double* y, double* z, double* vx, double* vy, double* vz,
             double* w, uint64_t* id) {
    copy_out(s.x, x); copy_out(s.y, y); copy_out(s.z, z);
    copy_out(s.vx, vx); copy_out(s.vy, vy); copy_out(s.vz, vz); copy_out(s.w, w);
    if (id) std::memcpy(id, s.id.data(), s.id.size() * sizeof(uint64_t));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_make_workload(const RefWorkload* w, double* x, double* y, double* z, double* vx, double* vy, double* vz,
                      double* wt, uint64_t* id) {
    return guarded([&] { soa_out(pic::make_workload(to_cfg(w)), x, y, z, vx, vy, vz, wt, id); });
}

// run_simulation (simulation.hpp:92-176): per-step fraction moved, rebuilds and
// global-sort reason, the checksum, the final grid and particles.
int ref_run_simulation(const RefWorkload* w, const char* mode, const RefPolicy* p, double gap_ratio,
                       uint32_t min_gap, double* fraction_moved, uint32_t* rebuilds, int* reasons, double* checksum,
                       double* jx, double* jy, double* jz, double* x, double* y, double* z, double* vx, double* vy,
                       double* vz, double* wt, uint64_t* id) {
    return guarded([&] {
        pic::SortPolicy pol;
        pol.sort_interval = p->sort_interval;
        pol.min_sort_interval = p->min_sort_interval;
        pol.trigger_rebuild_count = p->trigger_rebuild_count;
        pol.perf_enable = p->perf_enable != 0;
        pol.trigger_empty_ratio = p->trigger_empty_ratio;
        pol.trigger_full_ratio = p->trigger_full_ratio;
        pol.perf_degrad = p->perf_degrad;
        pic::GpmaConfig gc;
        gc.gap_ratio = gap_ratio;
        gc.min_gap = min_gap;
        const pic::RunResult r = pic::run_simulation(to_cfg(w), pic::mode_from_string(mode), pol, gc);
        for (std::size_t i = 0; i < r.steps.size(); ++i) {
            fraction_moved[i] = r.steps[i].fraction_moved;
            rebuilds[i] = r.steps[i].rebuilds;
            reasons[i] = static_cast<int>(r.steps[i].global_sort);
        }
        for (int c = 0; c < 3; ++c) checksum[c] = r.checksum[c];
        copy_out(r.final_grid.jx, jx); copy_out(r.final_grid.jy, jy); copy_out(r.final_grid.jz, jz);
        soa_out(r.particles, x, y, z, vx, vy, vz, wt, id);
    });
}

void* ref_create(const RefGrid* g, uint64_t n, const double* x, const double* y, const double* z,
                 const double* vx, const double* vy, const double* vz, const double* w,
                 const uint64_t* id, double q) {
    auto* s = new RefState;
    s->grid = to_spec(g);
    s->soa.resize(n);
    s->soa.q = q;
    for (uint64_t p = 0; p < n; ++p) {
        s->soa.x[p] = x[p]; s->soa.y[p] = y[p]; s->soa.z[p] = z[p];
        s->soa.vx[p] = vx[p]; s->soa.vy[p] = vy[p]; s->soa.vz[p] = vz[p];
        s->soa.w[p] = w[p];
        s->soa.id[p] = id ? id[p] : p;
    }
    return s;
}

void ref_destroy(void* h) { delete static_cast<RefState*>(h); }

uint64_t ref_size(void* h) { return static_cast<RefState*>(h)->soa.size(); }

void ref_get_particles(void* h, double* x, double* y, double* z, double* vx, double* vy, double* vz,
                       double* w, uint64_t* id) {
    auto& s = static_cast<RefState*>(h)->soa;
    copy_out(s.x, x); copy_out(s.y, y); copy_out(s.z, z);
    copy_out(s.vx, vx); copy_out(s.vy, vy); copy_out(s.vz, vz);
    copy_out(s.w, w);
    if (id) std::memcpy(id, s.id.data(), s.id.size() * sizeof(uint64_t));
}

// pic::deposit_scalar; use_gpma selects bin-order iteration.
int ref_deposit_scalar(void* h, int order, int use_gpma, double* jx, double* jy, double* jz) {
    auto* s = static_cast<RefState*>(h);
    return guarded([&] {
        const pic::CurrentGrid cg = pic::deposit_scalar(s->soa, s->grid, to_order(order),
                                                        use_gpma && s->has_gpma ? &s->gpma : nullptr);
        copy_out(cg.jx, jx); copy_out(cg.jy, jy); copy_out(cg.jz, jz);
    });
}

// pic::deposit_scalar run by `threads` workers on disjoint particle chunks
// (each worker calls the reference kernel on its own sub-SoA), then the
// per-worker grids are summed.  Used only as the multi-core CPU baseline.
int ref_deposit_scalar_mt(void* h, int order, int threads, double* jx, double* jy, double* jz) {
    auto* s = static_cast<RefState*>(h);
    return guarded([&] {
        const std::size_t n = s->soa.size();
        if (threads < 1) threads = 1;
        std::vector<pic::ParticleSoA> parts(threads);
        std::vector<pic::CurrentGrid> grids(threads);
        for (int t = 0; t < threads; ++t) {
            const std::size_t lo = n * t / threads, hi = n * (t + 1) / threads;
            auto& ps = parts[t];
            ps.q = s->soa.q;
            ps.x.assign(s->soa.x.begin() + lo, s->soa.x.begin() + hi);
            ps.y.assign(s->soa.y.begin() + lo, s->soa.y.begin() + hi);
            ps.z.assign(s->soa.z.begin() + lo, s->soa.z.begin() + hi);
            ps.vx.assign(s->soa.vx.begin() + lo, s->soa.vx.begin() + hi);
            ps.vy.assign(s->soa.vy.begin() + lo, s->soa.vy.begin() + hi);
            ps.vz.assign(s->soa.vz.begin() + lo, s->soa.vz.begin() + hi);
            ps.w.assign(s->soa.w.begin() + lo, s->soa.w.begin() + hi);
            ps.id.assign(s->soa.id.begin() + lo, s->soa.id.begin() + hi);
        }
        std::vector<std::thread> pool;
        std::vector<std::exception_ptr> errs(threads);
        for (int t = 0; t < threads; ++t)
            pool.emplace_back([&, t] {
                try {
                    grids[t] = pic::deposit_scalar(parts[t], s->grid, to_order(order));
                } catch (...) {
                    errs[t] = std::current_exception();
                }
            });
        for (auto& th : pool) th.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        const std::size_t nn = s->grid.n_nodes();
        double* outs[3] = {jx, jy, jz};
        std::vector<std::thread> red;
        for (int t = 0; t < threads; ++t)
            red.emplace_back([&, t] {
                const std::size_t lo = nn * t / threads, hi = nn * (t + 1) / threads;
                for (int c = 0; c < 3; ++c)
                    for (std::size_t i = lo; i < hi; ++i) {
                        double acc = 0.0;
                        for (int u = 0; u < threads; ++u) acc += grids[u].component(c)[i];
                        if (outs[c]) outs[c][i] = acc;
                    }
            });
        for (auto& th : red) th.join();
    });
}

int ref_deposit_density(void* h, int order, const double* quantity, double* rho) {
    auto* s = static_cast<RefState*>(h);
    return guarded([&] {
        std::span<const double> qs(quantity, s->soa.size());
        const std::vector<double> r = pic::deposit_density(s->soa, s->grid, to_order(order), qs);
        copy_out(r, rho);
    });
}

int ref_deposit_tiled(void* h, int order, int use_gpma, double* jx, double* jy, double* jz) {
    auto* s = static_cast<RefState*>(h);
    return guarded([&] {
        pic::TiledOptions opt;
        opt.gpma = use_gpma && s->has_gpma ? &s->gpma : nullptr;
        const pic::CurrentGrid cg = pic::deposit_tiled(s->soa, s->grid, to_order(order), opt);
        copy_out(cg.jx, jx); copy_out(cg.jy, jy); copy_out(cg.jz, jz);
    });
}

// deposit_tiled with every TiledOptions field, plus the engine's counters.
int ref_deposit_tiled_opt(void* h, int order, int use_gpma, int residency, int dual_tile, double* jx, double* jy,
                          double* jz, uint64_t* mopa_calls, uint64_t* extract_passes) {
    auto* s = static_cast<RefState*>(h);
    return guarded([&] {
        pic::KernelCounters kc;
        pic::TiledOptions opt;
        opt.gpma = use_gpma && s->has_gpma ? &s->gpma : nullptr;
        opt.residency = residency != 0;
        opt.dual_tile = dual_tile != 0;
        opt.counters = &kc;
        const pic::CurrentGrid cg = pic::deposit_tiled(s->soa, s->grid, to_order(order), opt);
        copy_out(cg.jx, jx); copy_out(cg.jy, jy); copy_out(cg.jz, jz);
        *mopa_calls = kc.mopa_calls;
        *extract_passes = kc.extract_passes;
    });
}

int ref_deposit_rhocell(void* h, int order, int use_gpma, double* jx, double* jy, double* jz) {
    auto* s = static_cast<RefState*>(h);
    return guarded([&] {
        const pic::CurrentGrid cg = pic::deposit_rhocell_vector(s->soa, s->grid, to_order(order),
                                                                use_gpma && s->has_gpma ? &s->gpma : nullptr);
        copy_out(cg.jx, jx); copy_out(cg.jy, jy); copy_out(cg.jz, jz);
    });
}

// pic::gpma_build: physically sorts the store (stable counting sort) and
// indexes it.  With ids equal to the pre-sort storage index, id[i] after the
// call is perm[i].
int ref_gpma_build(void* h, double gap_ratio, uint32_t min_gap) {
    auto* s = static_cast<RefState*>(h);
    return guarded([&] {
        pic::GpmaConfig cfg;
        cfg.gap_ratio = gap_ratio;
        cfg.min_gap = min_gap;
        s->gpma = pic::gpma_build(s->soa, s->grid, cfg);
        s->has_gpma = true;
    });
}

// pic::advance; *moved_fraction as returned by the reference.
int ref_advance(void* h, double dt, double* moved_fraction) {
    auto* s = static_cast<RefState*>(h);
    return guarded([&] {
        const double f = pic::advance(s->soa, dt, s->grid);
        if (moved_fraction) *moved_fraction = f;
    });
}

// detect_moves + apply_pending_moves (the baseline-incrsort composition,
// simulation.hpp:117-124).  out[0]=pending, out[1]=inserts, out[2]=shifted,
// out[3]=overflowed, out[4]=rebuilt.
int ref_incremental_sort(void* h, uint64_t* out) {
    auto* s = static_cast<RefState*>(h);
    return guarded([&] {
        if (!s->has_gpma) throw std::logic_error("ref_incremental_sort: no gpma");
        auto pending = s->gpma.detect_moves(s->soa, s->grid);
        const uint64_t np = pending.size();
        const pic::ApplyMovesResult r = pic::apply_pending_moves(s->gpma, pending);
        if (out) {
            out[0] = np; out[1] = r.inserts; out[2] = r.shifted;
            out[3] = r.overflowed; out[4] = r.rebuilt ? 1 : 0;
        }
    });
}

// One baseline-incrsort step of the reference (simulation.hpp:117-136), each
// stage timed with the reference's own pic::Timer: secs[0] = advance,
// secs[1] = detect_moves + apply_pending_moves, secs[2] = deposit_scalar over
// the Gpma's bins.  out[0] = movers, out[1] = rebuilt.  No copies.
int ref_step_timed(void* h, int order, double dt, double* secs, uint64_t* out) {
    auto* s = static_cast<RefState*>(h);
    return guarded([&] {
        if (!s->has_gpma) throw std::logic_error("ref_step_timed: no gpma");
        const pic::ShapeOrder so = to_order(order);
        pic::Timer t0;
        pic::advance(s->soa, dt, s->grid);
        secs[0] = t0.elapsed();
        pic::Timer t1;
        auto pending = s->gpma.detect_moves(s->soa, s->grid);
        const uint64_t np = pending.size();
        const pic::ApplyMovesResult r = pic::apply_pending_moves(s->gpma, pending);
        secs[1] = t1.elapsed();
        pic::Timer t2;
        const pic::CurrentGrid cg = pic::deposit_scalar(s->soa, s->grid, so, &s->gpma);
        secs[2] = t2.elapsed();
        if (cg.jx.empty()) throw std::logic_error("empty grid");
        if (out) { out[0] = np; out[1] = r.rebuilt ? 1 : 0; }
    });
}

// pic::deposit_density of q*w, timed (seconds), no copy-out.
int ref_density_timed(void* h, int order, double* secs) {
    auto* s = static_cast<RefState*>(h);
    return guarded([&] {
        std::vector<double> qw(s->soa.size());
        for (std::size_t p = 0; p < qw.size(); ++p) qw[p] = s->soa.q * s->soa.w[p];
        pic::Timer t;
        const std::vector<double> r = pic::deposit_density(s->soa, s->grid, to_order(order), qw);
        *secs = t.elapsed();
        if (r.empty()) throw std::logic_error("empty grid");
    });
}

// bin_of[p] = cell whose bin holds storage index p (UINT32_MAX if none).
int ref_bins(void* h, uint32_t* bin_of, uint32_t* bin_len) {
    auto* s = static_cast<RefState*>(h);
    return guarded([&] {
        if (!s->has_gpma) throw std::logic_error("ref_bins: no gpma");
        for (std::size_t p = 0; p < s->soa.size(); ++p) bin_of[p] = UINT32_MAX;
        for (std::uint32_t c = 0; c < s->gpma.n_cells(); ++c) {
            if (bin_len) bin_len[c] = s->gpma.bin_length(c);
            s->gpma.for_each_in_cell(c, [&](pic::ParticleRef p) { bin_of[p] = c; });
        }
    });
}

// Gpma scalar state: out[0]=capacity, out[1]=num_particles, out[2]=num_empty, out[3]=rebuild_count
void ref_gpma_stats(void* h, uint64_t* out, double* empty_ratio) {
    auto* s = static_cast<RefState*>(h);
    out[0] = s->gpma.capacity(); out[1] = s->gpma.num_particles();
    out[2] = s->gpma.num_empty_slots(); out[3] = s->gpma.rebuild_count();
    if (empty_ratio) *empty_ratio = s->gpma.empty_slot_ratio();
}

int ref_cell_of(const RefGrid* g, double x, double y, double z, int32_t* ijk, uint32_t* linear) {
    return guarded([&] {
        const auto c = pic::cell_of({x, y, z}, to_spec(g));
        ijk[0] = c.i; ijk[1] = c.j; ijk[2] = c.k;
        *linear = c.linear;
    });
}

int ref_intra_cell(const RefGrid* g, double x, double y, double z, double* d) {
    return guarded([&] {
        const auto v = pic::intra_cell_coords({x, y, z}, to_spec(g));
        d[0] = v[0]; d[1] = v[1]; d[2] = v[2];
    });
}

int ref_shape_1d(int order, double d, double* out) {
    return guarded([&] {
        if (order == 1) {
            const auto s = pic::cic_shape_1d(d);
            out[0] = s[0]; out[1] = s[1];
        } else {
            const auto s = pic::qsp_shape_1d(d);
            for (int i = 0; i < 4; ++i) out[i] = s[i];
        }
    });
}

int ref_flop_count(int order) { return pic::flop_count_scalar(to_order(order)); }

int ref_should_global_sort(uint32_t steps, uint64_t rebuilds, double ratio, double perf, double base,
                           uint32_t sort_interval, uint32_t min_sort_interval, uint32_t trigger_rebuild_count,
                           double trigger_empty_ratio, double trigger_full_ratio, int perf_enable,
                           double perf_degrad) {
    pic::RankSortStats s;
    s.steps_since_sort = steps;
    s.cumulative_local_rebuilds = rebuilds;
    s.empty_slot_ratio = ratio;
    s.perf_metric = perf;
    s.baseline_perf = base;
    pic::SortPolicy p;
    p.sort_interval = sort_interval;
    p.min_sort_interval = min_sort_interval;
    p.trigger_rebuild_count = trigger_rebuild_count;
    p.trigger_empty_ratio = trigger_empty_ratio;
    p.trigger_full_ratio = trigger_full_ratio;
    p.perf_enable = perf_enable != 0;
    p.perf_degrad = perf_degrad;
    return static_cast<int>(pic::should_global_sort(s, p));
}

double ref_uniform01(uint64_t seed, uint64_t stream, uint64_t counter) {
    return pic::uniform01(seed, stream, counter);
}
double ref_gaussian(uint64_t seed, uint64_t stream, uint64_t counter) {
    return pic::gaussian(seed, stream, counter);
}

// CPU baseline / --impl reference: `threads` workers, each running the
// reference's own baseline-incrsort step (simulation.hpp:117-136 composition:
// advance -> detect_moves + apply_pending_moves -> deposit_scalar in bin order)
// on its own independent periodic sub-box of nx^3 cells x ppc particles
// (SURVEY 8(d) generator on the reference RNG, seed + worker).  Setup
// (generation, gpma_build) is untimed; returns the max over workers of the
// timed seconds for `steps` steps, and the particles per worker.
int ref_bench_steps(int nx, int ppc, double u_th, uint64_t seed, int order, double dt, int steps, int threads,
                    double* max_seconds, uint64_t* particles_per_worker) {
    return guarded([&] {
        if (threads < 1) threads = 1;
        pic::GridSpec g;
        g.nx = g.ny = g.nz = nx;
        const pic::ShapeOrder so = to_order(order);
        std::vector<double> secs(threads, 0.0);
        std::vector<std::exception_ptr> errs(threads);
        const std::size_t n = static_cast<std::size_t>(nx) * nx * nx * ppc;
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t)
            pool.emplace_back([&, t] {
                try {
                    pic::ParticleSoA soa;
                    soa.resize(n);
                    soa.q = -1.0;
                    const uint64_t sd = seed + static_cast<uint64_t>(t);
                    std::size_t pid = 0;
                    for (int k = 0; k < nx; ++k)
                        for (int j = 0; j < nx; ++j)
                            for (int i = 0; i < nx; ++i)
                                for (int p = 0; p < ppc; ++p, ++pid) {
                                    soa.x[pid] = i + pic::uniform01(sd, pid, 6);
                                    soa.y[pid] = j + pic::uniform01(sd, pid, 7);
                                    soa.z[pid] = k + pic::uniform01(sd, pid, 8);
                                    const double ux = u_th * pic::gaussian(sd, pid, 0);
                                    const double uy = u_th * pic::gaussian(sd, pid, 1);
                                    const double uz = u_th * pic::gaussian(sd, pid, 2);
                                    const double gam = std::sqrt(1.0 + ux * ux + uy * uy + uz * uz);
                                    soa.vx[pid] = ux / gam; soa.vy[pid] = uy / gam; soa.vz[pid] = uz / gam;
                                    soa.w[pid] = 1.0 / ppc;
                                    soa.id[pid] = pid;
                                }
                    pic::Gpma gpma = pic::gpma_build(soa, g, {});
                    pic::Timer timer;
                    for (int s = 0; s < steps; ++s) {
                        pic::advance(soa, dt, g);
                        auto pending = gpma.detect_moves(soa, g);
                        pic::apply_pending_moves(gpma, pending);
                        const pic::CurrentGrid cg = pic::deposit_scalar(soa, g, so, &gpma);
                        if (cg.jx.empty()) throw std::logic_error("empty grid");
                    }
                    secs[t] = timer.elapsed();
                } catch (...) {
                    errs[t] = std::current_exception();
                }
            });
        for (auto& th : pool) th.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        double mx = 0.0;
        for (double s : secs) mx = std::max(mx, s);
        *max_seconds = mx;
        *particles_per_worker = n;
    });
}

}  // extern "C"

