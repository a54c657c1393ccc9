"""The reference's harness loop on the GPU:
make_workload (workload.hpp:75-125), the full-resort step, and run_simulation
(simulation.hpp:92-176) in all eight ablation modes, in lockstep with the
reference's own run_simulation (oracle/_ref) started from the same population.

Bars: fraction moved per step and the final particle state bit-exact, the
final J within 1e-12 peak-normalised, fullopt's global-sort decisions identical
under a deterministic policy (perf trigger off)."""
import numpy as np
import pytest

from conftest import peak_rel_err

import oracle as O

pytestmark = pytest.mark.gpu


def _wl(pg, order=3, kind=0, steps=8, thermal=0.2, drift=(0.0, 0.0, 0.0)):
    g = pg.Grid.make(10, 8, 6, dx=1.0, dy=0.5, dz=1.0, origin=(-3.0, 1.0, 0.0))
    return pg.WorkloadConfig.make(g, ppc=4, kind=kind, thermal_speed=thermal, drift=drift, seed=3, steps=steps,
                                  dt=0.5, charge=-1.0, order=order)


@pytest.mark.parametrize("kind", [0, 1])
def test_make_workload_matches_reference(pg, ref, kind):
    wl = _wl(pg, kind=kind, thermal=0.9)  # hot: some velocities hit the cap truncation
    want = ref.make_workload(wl)
    S = pg.Session(wl.grid, 3)
    S.make_workload(wl)
    p = S.particles()
    o = np.argsort(p.id)
    got = {k: getattr(p, k)[o] for k in ("x", "y", "z", "vx", "vy", "vz", "w", "id")}
    for k in ("x", "y", "z", "w", "id"):
        assert np.array_equal(got[k], want[k]), k
    for k in ("vx", "vy", "vz"):  # device log/cos vs glibc: last-ulp differences allowed
        assert np.max(np.abs(got[k] - want[k])) <= 4e-16 * np.max(np.abs(want[k])), k
    speed = np.sqrt(got["vx"] ** 2 + got["vy"] ** 2 + got["vz"] ** 2)
    assert speed.max() <= wl.speed_cap()


def test_make_workload_validates(pg):
    wl = _wl(pg)
    S = pg.Session(wl.grid, 3)
    for field, bad in (("ppc", 0), ("dt", 0.0), ("thermal_speed", -1.0), ("steps", -1)):
        w2 = _wl(pg)
        setattr(w2, field, bad)
        with pytest.raises(pg.InvalidArgument):
            S.make_workload(w2)
    small = pg.WorkloadConfig.make(pg.Grid.make(3, 8, 8), order=3)
    with pytest.raises(pg.InvalidArgument):
        pg.Session(small.grid, 3).make_workload(small)


def test_resort_step_is_a_stable_counting_sort(pg, orc):
    wl = _wl(pg, thermal=0.4)
    S = pg.Session(wl.grid, 3)
    S.make_workload(wl)
    before = S.particles()
    st = S.step(0.5, pg.STEP_PUSH | pg.STEP_RESORT | pg.STEP_CURRENT)
    after = S.particles()
    g = O.Grid.make(wl.grid.nx, wl.grid.ny, wl.grid.nz, dx=wl.grid.dx, dy=wl.grid.dy, dz=wl.grid.dz,
                    origin=(wl.grid.ox, wl.grid.oy, wl.grid.oz))
    d = {k: getattr(before, k).copy() for k in ("x", "y", "z", "vx", "vy", "vz", "w")}
    moved = orc.advance(g, 0.5, d)
    perm, _, _ = orc.counting_sort(g, d)
    assert st["moved"] == moved and st["global_sorted"] == 1
    for k in ("x", "y", "z", "vx"):
        assert np.array_equal(getattr(after, k), d[k][perm]), k
    assert np.array_equal(after.id, before.id[perm])


def test_resort_after_incremental_steps_sorts_the_download_order(pg, orc):
    """Incremental steps leave holes in the bins; a following STEP_RESORT is the
    stable counting sort of the store in the order a download reports it."""
    wl = _wl(pg, thermal=0.4)
    S = pg.Session(wl.grid, 3)
    S.make_workload(wl)
    g = O.Grid.make(wl.grid.nx, wl.grid.ny, wl.grid.nz, dx=wl.grid.dx, dy=wl.grid.dy, dz=wl.grid.dz,
                    origin=(wl.grid.ox, wl.grid.oy, wl.grid.oz))
    for _ in range(3):
        S.step(0.5, pg.STEP_PUSH | pg.STEP_SORT | pg.STEP_CURRENT | pg.STEP_UNFUSED)
    before = S.particles()  # storage order after the incremental steps (holes packed)
    S.step(0.5, pg.STEP_PUSH | pg.STEP_RESORT | pg.STEP_CURRENT)
    after = S.particles()
    d = {k: getattr(before, k).copy() for k in ("x", "y", "z", "vx", "vy", "vz", "w")}
    orc.advance(g, 0.5, d)
    perm, _, _ = orc.counting_sort(g, d)
    for k in ("x", "y", "z", "vx"):
        assert np.array_equal(getattr(after, k), d[k][perm]), k
    assert np.array_equal(after.id, before.id[perm])


@pytest.mark.parametrize("order", [1, 3])
@pytest.mark.parametrize("mode", ["baseline", "matrix-only", "hybrid-nosort", "hybrid-globalsort", "fullopt",
                                  "rhocell-vector", "baseline-incrsort", "rhocell-incrsort"])
def test_run_simulation_lockstep_with_reference(pg, ref, order, mode):
    wl = _wl(pg, order=order)
    pol = pg.SortPolicy.defaults(perf_enable=0, sort_interval=3, min_sort_interval=2, trigger_rebuild_count=1000,
                                 trigger_empty_ratio=0.01, trigger_full_ratio=0.99)
    want = ref.run_simulation(wl, mode, pol)
    init = pg.ParticleSoA.from_dict(ref.make_workload(wl), q=wl.charge)
    got = pg.run_simulation(wl, mode, pol, initial=init)
    assert len(got.steps) == wl.steps
    assert [m.fraction_moved for m in got.steps] == list(want["fraction_moved"])
    if mode == "fullopt":
        assert [m.global_sort for m in got.steps] == [pg.SORT_REASONS[r] for r in want["reasons"]]
        assert any(m.global_sort == "interval" for m in got.steps)
    J = got.final_grid
    assert peak_rel_err((J.jx, J.jy, J.jz), want["J"]) <= 1e-12
    assert np.allclose(got.checksum, want["checksum"], rtol=1e-12, atol=1e-12 * np.abs(J.jx).max())
    p = got.particles
    o = np.argsort(p.id)
    wp = want["particles"]
    wo = np.argsort(wp["id"])
    for k in ("x", "y", "z", "vx", "vy", "vz", "w", "id"):
        assert np.array_equal(getattr(p, k)[o], wp[k][wo]), k
    for m in got.steps:
        assert m.compute_s > 0 and m.sort_s > 0 and m.particles_per_second > 0


def test_run_simulation_device_workload_and_errors(pg):
    wl = _wl(pg, order=3, kind=1, steps=4)
    r = pg.run_simulation(wl, "fullopt")
    assert len(r.steps) == 4 and r.particles.size() == 10 * 8 * 6 * 4
    with pytest.raises(pg.InvalidArgument):
        pg.run_simulation(wl, "no-such-mode")
    with pytest.raises(pg.InvalidArgument):
        pg.run_simulation(wl, "fullopt", pg.SortPolicy.defaults(min_sort_interval=60))
