"""SURVEY 8(d) C4 population (density ramp + relativistic beam) on the GPU:
the generator follows its recipe exactly (positions and counts bit-exact
against a restatement on the oracle's counter RNG), and sessions on this
strongly non-uniform plasma (empty cells, dense cells, particles moving half
a cell per step) stay in lockstep with the oracle."""
import math

import numpy as np
import pytest

from conftest import peak_rel_err

import oracle as O

pytestmark = pytest.mark.gpu


def _cfg(pg):
    G = pg.Grid.make(64, 8, 8, dx=1.0, dy=1.0, dz=1.0, origin=(0.0, -4.0, 2.0))
    c = pg.LwfaConfig.make(ppc=8, ramp_start=8, ramp_len=16, u_th=0.05, beam_fraction=0.1, ux=(5.0, 50.0),
                           beam_x=(24.0, 32.0), seed=3)
    return G, c


def _counts(c, nx):
    out = []
    for i in range(nx):
        ramp = min(1.0, max(0.0, (i + 0.5 - c.ramp_start) / c.ramp_len))
        out.append(int(math.floor(c.ppc * ramp + 0.5)) if i >= c.ramp_start else 0)  # llround, ramp >= 0
    return out


def test_lwfa_generator_follows_recipe(pg, orc):
    G, c = _cfg(pg)
    S = pg.Session(G, 3)
    S.generate_lwfa(c)
    p = S.particles()
    o = np.argsort(p.id)
    x, y, z, vx, vy, w = p.x[o], p.y[o], p.z[o], p.vx[o], p.vy[o], p.w[o]
    per_col = _counts(c, G.nx)
    nbg = sum(per_col) * G.ny * G.nz
    nbeam = int(round(c.beam_fraction * nbg))
    assert p.size() == nbg + nbeam and np.array_equal(p.id[o], np.arange(nbg + nbeam, dtype=np.uint64))
    # background: cell-major (x fastest) pids, per-cell counts from the ramp
    pfx = np.concatenate([[0], np.cumsum(per_col)])
    R = pfx[-1]
    for pid in list(range(0, nbg, 97)) + [nbg - 1]:
        row, r = divmod(pid, R)
        i = int(np.searchsorted(pfx, r, side="right") - 1)
        j, k = row % G.ny, row // G.ny
        assert x[pid] == G.ox + (i + orc.uniform01(c.seed, pid, 6)) * G.dx
        assert y[pid] == G.oy + (j + orc.uniform01(c.seed, pid, 7)) * G.dy
        assert z[pid] == G.oz + (k + orc.uniform01(c.seed, pid, 8)) * G.dz
    # beam: uniform in x-cells [24, 32), ux from counter 9, uy = uz = 0
    bx = (x[nbg:] - G.ox) / G.dx
    assert bx.min() >= c.beam_x0 and bx.max() < c.beam_x1
    for b in range(0, nbeam, 53):
        pid = nbg + b
        ux = c.ux_min + (c.ux_max - c.ux_min) * orc.uniform01(c.seed, pid, 9)
        assert vx[pid] == pytest.approx(ux / math.sqrt(1.0 + ux * ux), rel=1e-15) and vy[pid] == 0.0
    assert np.all(w == 1.0 / c.ppc)
    assert not np.any((x[:nbg] - G.ox) < c.ramp_start)  # vacuum below the ramp
    # bins: empty vacuum columns, ramp and plateau counts
    off, cnt = S.bins()
    cnt3 = cnt.reshape(G.nz, G.ny, G.nx)
    assert cnt3[:, :, : c.ramp_start].sum() == 0


@pytest.mark.parametrize("order", [1, 3])
def test_lwfa_steps_lockstep_with_oracle(pg, orc, order):
    G, c = _cfg(pg)
    S = pg.Session(G, order)
    S.generate_lwfa(c)
    p = S.particles()
    ref = {k: getattr(p, k).copy() for k in ("x", "y", "z", "vx", "vy", "vz", "w", "id")}
    g = O.Grid.make(G.nx, G.ny, G.nz, dx=G.dx, dy=G.dy, dz=G.dz, origin=(G.ox, G.oy, G.oz))
    flags = pg.STEP_DEFAULT | pg.STEP_DENSITY
    for step in range(6):
        st = S.step(0.5, flags)
        moved = orc.advance(g, 0.5, ref)
        assert st["moved"] == moved
        got = S.particles()
        o, w = np.argsort(got.id), np.argsort(ref["id"])
        for k in ("x", "y", "z"):
            assert np.array_equal(getattr(got, k)[o], ref[k][w]), (step, k)
        J = S.current()
        assert peak_rel_err((J.jx, J.jy, J.jz), orc.deposit_current(g, order, ref, -1.0)) <= 1e-12
        q = {k: getattr(got, k) for k in ("x", "y", "z")}
        rho = orc.deposit_density(g, order, q, -1.0 * got.w)
        assert np.array_equal(S.density(), rho)  # bit-exact, storage order
    assert st["moved"] > 0


def test_moving_window_shift(pg, orc):
    """Every 2 steps the window moves one cell: the particles of the back column
    are dropped, the rest keep their exact state, a fresh column (ids pid0..,
    recipe positions) enters at the front, and the steps that follow stay in
    lockstep with the oracle on the shifted grid."""
    G, c = _cfg(pg)
    S = pg.Session(G, 3)
    S.generate_lwfa(c)
    pid = S.num_particles
    for cycle in range(3):
        for _ in range(2):
            S.step(0.5)
        before = S.particles()
        ox_new = S.grid.ox + S.grid.dx
        dropped, injected = S.shift_window(8, 0.01, c.seed, pid)
        assert S.grid.ox == ox_new and injected == G.ny * G.nz * 8
        after = S.particles()
        keep = before.x >= ox_new
        assert dropped == int((~keep).sum())
        surv = np.argsort(before.id[keep])
        got = after.id < pid
        o = np.argsort(after.id[got])
        for k in ("x", "y", "z", "vx", "vy", "vz", "w", "id"):
            assert np.array_equal(getattr(after, k)[got][o], getattr(before, k)[keep][surv]), (cycle, k)
        new = np.nonzero(~got)[0]
        assert sorted(after.id[new]) == list(range(pid, pid + injected))
        for t in range(0, injected, 37):
            q = new[after.id[new] == pid + t][0]
            cell = t // 8
            j, k = cell % G.ny, cell // G.ny
            assert after.x[q] == S.grid.ox + (G.nx - 1 + orc.uniform01(c.seed, pid + t, 6)) * G.dx
            assert after.y[q] == S.grid.oy + (j + orc.uniform01(c.seed, pid + t, 7)) * G.dy
            assert after.z[q] == S.grid.oz + (k + orc.uniform01(c.seed, pid + t, 8)) * G.dz
        pid += injected
        # lockstep on the shifted grid, from the session's own state
        g = O.Grid.make(G.nx, G.ny, G.nz, dx=G.dx, dy=G.dy, dz=G.dz, origin=(S.grid.ox, S.grid.oy, S.grid.oz))
        ref = {k: getattr(after, k).copy() for k in ("x", "y", "z", "vx", "vy", "vz", "w", "id")}
        st = S.step(0.5)
        assert st["moved"] == orc.advance(g, 0.5, ref)
        J = S.current()
        assert peak_rel_err((J.jx, J.jy, J.jz), orc.deposit_current(g, 3, ref, -1.0)) <= 1e-12
        p2 = S.particles()
        o2, w2 = np.argsort(p2.id), np.argsort(ref["id"])
        assert np.array_equal(p2.x[o2], ref["x"][w2])


def test_adaptive_slack_keeps_lockstep_and_cuts_rebuilds(pg, orc):
    """picgpu_session_set_adaptive_slack: a rebuild storm (the beam flowing into
    bins sized at the last layout) widens the gap ratio of later layouts.  The
    particles, their bins and J stay in lockstep with the oracle; the session
    rebuilds no more often than one with the reference's fixed slack."""
    G, c = _cfg(pg)
    runs = {}
    for adaptive in (False, True):
        S = pg.Session(G, 3)
        if adaptive:
            S.set_adaptive_slack(True)
        S.generate_lwfa(c)
        p = S.particles()
        ref = {k: getattr(p, k).copy() for k in ("x", "y", "z", "vx", "vy", "vz", "w", "id")}
        rebuilds = 0
        for step in range(16):
            g = O.Grid.make(G.nx, G.ny, G.nz, dx=G.dx, dy=G.dy, dz=G.dz, origin=(S.grid.ox, S.grid.oy, S.grid.oz))
            st = S.step(0.5)
            assert st["moved"] == orc.advance(g, 0.5, ref)
            rebuilds += st["rebuilt"]
        got = S.particles()
        o, w = np.argsort(got.id), np.argsort(ref["id"])
        for k in ("x", "y", "z"):
            assert np.array_equal(getattr(got, k)[o], ref[k][w]), k
        off, cnt = S.bins()
        cells = np.repeat(np.arange(G.ncells, dtype=np.uint32), cnt.astype(np.int64))
        assert np.array_equal(cells, orc.cells(g, {"x": got.x, "y": got.y, "z": got.z}))
        J = S.current()
        assert peak_rel_err((J.jx, J.jy, J.jz), orc.deposit_current(g, 3, ref, -1.0)) <= 1e-12
        runs[adaptive] = rebuilds
    assert runs[True] <= runs[False]
