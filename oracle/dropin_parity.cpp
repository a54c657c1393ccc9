// dropin_parity.cpp -- TEST INFRASTRUCTURE: the reference's own C++ calls and
// the picgpu drop-in (include/picgpu.hpp) on identical inputs, side by side.
//
// Built by oracle/Makefile (only where /root/reference exists; the binary in
// oracle/_ref/ travels to the GPU box) from the UNMODIFIED reference headers
// plus picgpu.hpp, linked against paper_2601_08277_b200/libpicgpu.so.  Each
// block below is the same call site written once against `pic::` and once
// against `picgpu::`; the program exits non-zero on any parity failure.
//   positions after advance, rho, full-sort permutation: bit-identical
//   J: <= 1e-12 peak-normalised (proj/tests/test_pipeline.cpp:27-40 metric)
#include <pic/deposit.hpp>
#include <pic/gpma.hpp>
#include <pic/rng.hpp>
#include <pic/simulation.hpp>
#include <pic/sort_policy.hpp>
#include <pic/workload.hpp>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>

#include "picgpu.hpp"

namespace {

int failures = 0;

void expect(bool ok, const char* what) {
    std::printf("%-58s %s\n", what, ok ? "ok" : "FAIL");
    if (!ok) ++failures;
}

template <class A, class B>
double peak_rel_err(const A& got, const B& want) {
    double err = 0.0;
    for (int c = 0; c < 3; ++c) {
        double peak = 0.0;
        for (double v : want.component(c)) peak = std::max(peak, std::abs(v));
        for (std::size_t i = 0; i < want.component(c).size(); ++i) {
            const double d = std::abs(got.component(c)[i] - want.component(c)[i]);
            if (d == 0.0) continue;
            if (peak == 0.0) return INFINITY;
            err = std::max(err, d / peak);
        }
    }
    return err;
}

// SURVEY 8(d) plasma on the reference counter RNG.
pic::ParticleSoA plasma(const pic::GridSpec& g, int ppc, double u_th, std::uint64_t seed) {
    pic::ParticleSoA s;
    s.resize(static_cast<std::size_t>(g.n_cells()) * ppc);
    s.q = -1.0;
    std::size_t pid = 0;
    for (int k = 0; k < g.nz; ++k)
        for (int j = 0; j < g.ny; ++j)
            for (int i = 0; i < g.nx; ++i)
                for (int p = 0; p < ppc; ++p, ++pid) {
                    s.x[pid] = g.origin[0] + (i + pic::uniform01(seed, pid, 6)) * g.dx;
                    s.y[pid] = g.origin[1] + (j + pic::uniform01(seed, pid, 7)) * g.dy;
                    s.z[pid] = g.origin[2] + (k + pic::uniform01(seed, pid, 8)) * g.dz;
                    const double ux = u_th * pic::gaussian(seed, pid, 0), uy = u_th * pic::gaussian(seed, pid, 1),
                                 uz = u_th * pic::gaussian(seed, pid, 2);
                    const double gam = std::sqrt(1.0 + ux * ux + uy * uy + uz * uz);
                    s.vx[pid] = ux / gam; s.vy[pid] = uy / gam; s.vz[pid] = uz / gam;
                    s.w[pid] = 1.0 / ppc;
                    s.id[pid] = pid;
                }
    return s;
}

// deposit_tiled (deposit.hpp:284) and deposit_rhocell_vector (:87): same J,
// and the GPU reports the reference tile engine's counters exactly.
template <class RefOpt, class GpuOpt>
void tiled_case(const pic::ParticleSoA& ref, const pic::GridSpec& g, const picgpu::ParticleSoA& gpu,
                const picgpu::GridSpec& gg, RefOpt ropt, GpuOpt gopt, const char* what) {
    for (auto [po, go] : {std::pair{pic::ShapeOrder::cic, picgpu::ShapeOrder::cic},
                          std::pair{pic::ShapeOrder::qsp, picgpu::ShapeOrder::qsp}}) {
        for (int mode = 0; mode < 3; ++mode) {  // residency on, off, on + dual tile
            pic::KernelCounters kr;
            picgpu::KernelCounters kg;
            ropt.residency = gopt.residency = mode != 1;
            ropt.dual_tile = gopt.dual_tile = mode == 2;
            ropt.counters = &kr;
            gopt.counters = &kg;
            picgpu::StageTimes st;
            const pic::CurrentGrid jr = pic::deposit_tiled(ref, g, po, ropt);
            const picgpu::CurrentGrid jt = picgpu::deposit_tiled(gpu, gg, go, gopt, &st);
            char msg[160];
            const double e = peak_rel_err(jt, jr);
            std::snprintf(msg, sizeof msg, "deposit_tiled %s order %d mode %d: J err %.2e, counters %llu/%llu vs %llu/%llu",
                          what, static_cast<int>(po), mode, e, (unsigned long long)kg.mopa_calls,
                          (unsigned long long)kg.extract_passes, (unsigned long long)kr.mopa_calls,
                          (unsigned long long)kr.extract_passes);
            expect(e <= 1e-12 && kg.mopa_calls == kr.mopa_calls && kg.extract_passes == kr.extract_passes &&
                       st.compute > 0.0, msg);
        }
        const pic::CurrentGrid jr = pic::deposit_rhocell_vector(ref, g, po, ropt.gpma);
        const picgpu::CurrentGrid jv = picgpu::deposit_rhocell_vector(gpu, gg, go, gopt.gpma);
        char msg[96];
        const double e = peak_rel_err(jv, jr);
        std::snprintf(msg, sizeof msg, "deposit_rhocell_vector %s order %d: J err %.2e", what, static_cast<int>(po), e);
        expect(e <= 1e-12, msg);
    }
}

picgpu::ParticleSoA to_gpu(const pic::ParticleSoA& s) {
    picgpu::ParticleSoA o;
    o.x = s.x; o.y = s.y; o.z = s.z; o.vx = s.vx; o.vy = s.vy; o.vz = s.vz; o.w = s.w; o.id = s.id; o.q = s.q;
    return o;
}

}  // namespace

int main() {
    pic::GridSpec g;
    g.nx = 12; g.ny = 10; g.nz = 9;
    g.dx = 1.0; g.dy = 0.5; g.dz = 1.0;
    g.origin = {-2.0, 1.0, 0.5};
    picgpu::GridSpec gg;
    gg.nx = g.nx; gg.ny = g.ny; gg.nz = g.nz;
    gg.dx = g.dx; gg.dy = g.dy; gg.dz = g.dz;
    gg.origin = g.origin;

    pic::ParticleSoA ref = plasma(g, 6, 0.15, 3);
    picgpu::ParticleSoA gpu = to_gpu(ref);
    const double dt = 0.5;

    // --- advance (workload.hpp:139) ---
    for (int s = 0; s < 3; ++s) {
        const double fr = pic::advance(ref, dt, g);
        const double fg = picgpu::advance(gpu, dt, gg);
        expect(fr == fg, "advance: moved fraction identical");
    }
    expect(ref.x == gpu.x && ref.y == gpu.y && ref.z == gpu.z, "advance: positions bit-identical");

    // --- deposit_scalar (deposit.hpp:62) at orders 1 and 3 ---
    for (auto [po, go] : {std::pair{pic::ShapeOrder::cic, picgpu::ShapeOrder::cic},
                          std::pair{pic::ShapeOrder::qsp, picgpu::ShapeOrder::qsp}}) {
        const pic::CurrentGrid jr = pic::deposit_scalar(ref, g, po);
        const picgpu::CurrentGrid jg = picgpu::deposit_scalar(gpu, gg, go);
        char msg[96];
        const double e = peak_rel_err(jg, jr);
        std::snprintf(msg, sizeof msg, "deposit_scalar order %d: J err %.2e <= 1e-12", static_cast<int>(po), e);
        expect(e <= 1e-12, msg);
    }

    // --- deposit_density (deposit.hpp:76): storage order, bit-identical ---
    std::vector<double> charge(ref.size());
    for (std::size_t p = 0; p < ref.size(); ++p) charge[p] = ref.q * ref.w[p];
    for (auto [po, go] : {std::pair{pic::ShapeOrder::cic, picgpu::ShapeOrder::cic},
                          std::pair{pic::ShapeOrder::qsp, picgpu::ShapeOrder::qsp}}) {
        const auto rr = pic::deposit_density(ref, g, po, charge);
        const auto rg = picgpu::deposit_density(gpu, gg, go, charge);
        expect(rr.size() == rg.size() && std::memcmp(rr.data(), rg.data(), rr.size() * 8) == 0,
               "deposit_density: rho bit-identical (unsorted store)");
    }

    // --- deposit_tiled / deposit_rhocell_vector on the unsorted store ---
    tiled_case(ref, g, gpu, gg, pic::TiledOptions{}, picgpu::TiledOptions{}, "unsorted");

    // --- gpma_build (gpma.hpp:379): same stable permutation of the store ---
    pic::Gpma gpma = pic::gpma_build(ref, g);
    const picgpu::Gpma bins = picgpu::gpma_build(gpu, gg);  // the reference call site, namespace switched
    {
        // deposit_scalar(soa, g, order, &gpma) as test_pipeline.cpp:139-142 calls it
        const pic::CurrentGrid jr = pic::deposit_scalar(ref, g, pic::ShapeOrder::qsp, &gpma);
        const picgpu::CurrentGrid jg = picgpu::deposit_scalar(gpu, gg, picgpu::ShapeOrder::qsp, &bins);
        expect(peak_rel_err(jg, jr) <= 1e-12, "deposit_scalar(..., &gpma): J within 1e-12");
        bool entries_ok = true;
        for (std::uint32_t c = 0; c < g.n_cells(); ++c) {
            std::vector<std::uint32_t> want;
            gpma.for_each_in_cell(c, [&](pic::ParticleRef r) { want.push_back(r); });
            entries_ok &= want == bins.cell_entries(c);
        }
        expect(entries_ok, "gpma_build: for_each_in_cell / cell_entries identical (fresh build)");
    }
    {
        pic::TiledOptions ro;
        ro.gpma = &gpma;
        picgpu::TiledOptions go;
        go.gpma = &bins;
        tiled_case(ref, g, gpu, gg, ro, go, "bins");
        tiled_case(ref, g, gpu, gg, pic::TiledOptions{}, picgpu::TiledOptions{}, "sorted");
    }
    expect(ref.id == gpu.id && ref.x == gpu.x, "gpma_build: store permuted identically");
    {
        const auto rr = pic::deposit_density(ref, g, pic::ShapeOrder::qsp, charge);  // charge is uniform per species
        const auto rg = picgpu::deposit_density(gpu, gg, picgpu::ShapeOrder::qsp, charge);
        expect(std::memcmp(rr.data(), rg.data(), rr.size() * 8) == 0, "deposit_density: rho bit-identical (sorted store)");
    }
    bool counts_ok = true;
    for (std::uint32_t c = 0; c < g.n_cells(); ++c) counts_ok &= gpma.bin_length(c) == bins.counts[c];
    expect(counts_ok, "gpma_build: per-cell counts identical");

    // --- incremental sort: bins as sets after push + detect/apply ---
    {
        picgpu::GpmaConfig gc;
        picgpu::Session sess(gg, picgpu::ShapeOrder::qsp, gc);
        sess.upload(gpu);
        expect(sess.capacity() == gpma.capacity(), "session capacity == Gpma capacity (layout rule)");
        for (int s = 0; s < 4; ++s) {
            pic::advance(ref, dt, g);
            auto pending = gpma.detect_moves(ref, g);
            pic::apply_pending_moves(gpma, pending);
            sess.step(dt, PICGPU_STEP_PUSH | PICGPU_STEP_SORT | PICGPU_STEP_CURRENT);
        }
        const picgpu::ParticleSoA got = sess.particles();
        std::map<std::uint64_t, std::uint32_t> want_bin, got_bin;
        for (std::uint32_t c = 0; c < g.n_cells(); ++c)
            gpma.for_each_in_cell(c, [&](pic::ParticleRef p) { want_bin[ref.id[p]] = c; });
        bool pos_ok = true;
        std::map<std::uint64_t, std::size_t> slot;
        for (std::size_t p = 0; p < ref.size(); ++p) slot[ref.id[p]] = p;
        for (std::size_t p = 0; p < got.size(); ++p) {
            got_bin[got.id[p]] = pic::cell_of(got.position(p), g).linear;
            const std::size_t r = slot[got.id[p]];
            pos_ok &= got.x[p] == ref.x[r] && got.y[p] == ref.y[r] && got.z[p] == ref.z[r];
        }
        expect(pos_ok, "session: positions bit-identical to pic::advance");
        expect(want_bin == got_bin, "session: bin sets == reference Gpma bins");
        const pic::CurrentGrid jr = pic::deposit_scalar(ref, g, pic::ShapeOrder::qsp, &gpma);
        expect(peak_rel_err(sess.current(), jr) <= 1e-12, "session: J (bin order) within 1e-12");
    }

    // --- should_global_sort (sort_policy.hpp:62) ---
    {
        bool ok = true;
        for (std::uint32_t steps : {5u, 10u, 20u, 50u, 200u})
            for (std::uint64_t rb : {0ull, 100ull, 101ull})
                for (double ratio : {0.1, 0.5, 0.9})
                    for (double perf : {79.9, 80.1}) {
                        pic::RankSortStats rs;
                        rs.steps_since_sort = steps; rs.cumulative_local_rebuilds = rb;
                        rs.empty_slot_ratio = ratio; rs.perf_metric = perf; rs.baseline_perf = 100.0;
                        picgpu::RankSortStats gs;
                        gs.steps_since_sort = steps; gs.cumulative_local_rebuilds = rb;
                        gs.empty_slot_ratio = ratio; gs.perf_metric = perf; gs.baseline_perf = 100.0;
                        ok &= static_cast<int>(pic::should_global_sort(rs, {})) ==
                              static_cast<int>(picgpu::should_global_sort(gs, {}));
                    }
        expect(ok, "should_global_sort: identical decisions");
    }

    // --- error behaviour: the same exception types ---
    {
        picgpu::ParticleSoA bad = gpu;
        bad.x[0] = NAN;
        bool got_invalid = false;
        try {
            picgpu::deposit_scalar(bad, gg, picgpu::ShapeOrder::cic);
        } catch (const std::invalid_argument&) {
            got_invalid = true;
        }
        expect(got_invalid, "non-finite position -> std::invalid_argument");
        picgpu::ParticleSoA fast = gpu;
        fast.vx[0] = 10.0;
        bool got_domain = false;
        try {
            picgpu::advance(fast, dt, gg);
        } catch (const std::domain_error&) {
            got_domain = true;
        }
        expect(got_domain, "displacement above the cap -> std::domain_error");
    }

    // --- run_simulation (simulation.hpp:92) in every mode, same population ---
    {
        pic::WorkloadConfig rc;
        rc.grid = g;
        rc.ppc = 4;
        rc.thermal_speed = 0.2;
        rc.seed = 5;
        rc.steps = 6;
        rc.dt = 0.5;
        rc.charge = -1.0;
        rc.order = pic::ShapeOrder::qsp;
        picgpu::WorkloadConfig gc;
        gc.grid = gg;
        gc.ppc = rc.ppc;
        gc.thermal_speed = rc.thermal_speed;
        gc.seed = rc.seed;
        gc.steps = rc.steps;
        gc.dt = rc.dt;
        gc.charge = rc.charge;
        gc.order = picgpu::ShapeOrder::qsp;
        pic::SortPolicy rp;
        rp.perf_enable = false;  // deterministic decisions
        rp.sort_interval = 3;
        rp.min_sort_interval = 2;
        picgpu::SortPolicy gp;
        gp.perf_enable = false;
        gp.sort_interval = 3;
        gp.min_sort_interval = 2;
        const picgpu::ParticleSoA init = to_gpu(pic::make_workload(rc));
        for (pic::AblationMode m : pic::kAllModes) {
            const pic::RunResult rr = pic::run_simulation(rc, m, rp);
            const picgpu::RunResult gr =
                picgpu::run_simulation(gc, picgpu::mode_from_string(pic::to_string(m)), gp, {}, 0, &init);
            bool same_moved = rr.steps.size() == gr.steps.size(), same_sorts = same_moved;
            for (std::size_t i = 0; same_moved && i < rr.steps.size(); ++i) {
                same_moved = rr.steps[i].fraction_moved == gr.steps[i].fraction_moved;
                same_sorts = same_sorts && static_cast<int>(rr.steps[i].global_sort) ==
                                               static_cast<int>(gr.steps[i].global_sort);
            }
            std::map<std::uint64_t, std::size_t> at;
            for (std::size_t p = 0; p < gr.particles.size(); ++p) at[gr.particles.id[p]] = p;
            bool same_state = at.size() == rr.particles.size();
            for (std::size_t p = 0; same_state && p < rr.particles.size(); ++p) {
                const auto it = at.find(rr.particles.id[p]);
                same_state = it != at.end() && gr.particles.x[it->second] == rr.particles.x[p] &&
                             gr.particles.y[it->second] == rr.particles.y[p] &&
                             gr.particles.z[it->second] == rr.particles.z[p];
            }
            const double e = peak_rel_err(gr.final_grid, rr.final_grid);
            char msg[160];
            std::snprintf(msg, sizeof msg, "run_simulation %s: moved %s, sorts %s, state %s, J err %.2e",
                          pic::to_string(m), same_moved ? "same" : "DIFF", same_sorts ? "same" : "DIFF",
                          same_state ? "same" : "DIFF", e);
            expect(same_moved && same_sorts && same_state && e <= 1e-12, msg);
        }
    }

    // multi-GPU C++ host path (no reference counterpart): a one-rank NCCL ring
    // slab session steps like the whole-box session
    {
        picgpu::GridSpec gg{16, 8, 8, 1.0, 1.0, 1.0, {0.0, 0.0, 0.0}};
        pic::WorkloadConfig wc;
        wc.grid.nx = 16; wc.grid.ny = 8; wc.grid.nz = 8;
        wc.ppc = 4;
        wc.thermal_speed = 0.3;
        wc.seed = 3;
        const picgpu::ParticleSoA init = to_gpu(pic::make_workload(wc));
        picgpu::Session whole(gg, picgpu::ShapeOrder::qsp);
        whole.upload(init);
        const auto id = picgpu::Comm::unique_id();
        picgpu::Comm comm(id, 1, 0, 0);
        picgpu::SlabSession slab(gg, 0, 16, picgpu::ShapeOrder::qsp, comm);
        slab.upload(init);
        bool same = true;
        for (int k = 0; k < 3; ++k) {
            const auto a = whole.step(0.5), b = slab.step(0.5);
            same = same && a.moved == b.moved && a.num_particles == b.num_particles;
        }
        const picgpu::CurrentGrid Jw = whole.current(), Js = slab.current();
        double peak = 0.0, d = 0.0;  // owned planes x in [2, 18) of the slab grid = the whole box
        for (int k = 0; k < 8; ++k)
            for (int j = 0; j < 8; ++j)
                for (int i = 0; i < 16; ++i) {
                    const std::size_t w = i + 16 * (j + 8 * k), sidx = (i + 2) + 20 * (j + 8 * k);
                    peak = std::max(peak, std::abs(Jw.jx[w]));
                    d = std::max(d, std::abs(Jw.jx[w] - Js.jx[sidx]));
                }
        char msg[160];
        std::snprintf(msg, sizeof msg, "picgpu::SlabSession over a one-rank NCCL ring: moved/count %s, jx err %.2e",
                      same ? "same" : "DIFF", peak > 0 ? d / peak : d);
        expect(same && d <= 1e-12 * peak, msg);
    }

    std::printf("%s (%d failures)\n", failures ? "DROP-IN PARITY FAILED" : "drop-in parity ok", failures);
    return failures ? 1 : 0;
}
