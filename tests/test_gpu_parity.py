"""GPU parity: the sm_100a path (through the C ABI) against the oracle and the
reference's golden fixtures.

Bars (north_star / SURVEY 8(c)):
  rho, sort permutation, push, cell ids, bin sets:  bit-exact
  J:  <= 1e-12 peak-normalised per component (reference metric,
      proj/tests/test_pipeline.cpp:27-40; the reference's own kernels agree to 1e-13)
"""
import numpy as np
import pytest

from conftest import golden_cases, load_golden, peak_rel_err, to_pg_grid

import oracle as O

pytestmark = pytest.mark.gpu

J_TOL = 1e-12


def scramble(s, seed):
    p = np.random.default_rng(seed).permutation(len(s["x"]))
    return {k: np.ascontiguousarray(v[p]) for k, v in s.items()}


GRIDS = [
    dict(nx=8),
    dict(nx=13, ny=6, nz=9, dx=0.5, dy=1.0, dz=0.25, origin=(-1.0, 2.0, 0.5)),
    dict(nx=5, ny=4, nz=7, dx=0.3, dy=1.7, dz=0.05, origin=(-1.0, 2.0, 0.25)),
    dict(nx=37, ny=11, nz=20),
    dict(nx=4, ny=4, nz=4),
]


# ------------------------------------------------------------- golden fixtures


@pytest.mark.parametrize("case", golden_cases())
def test_golden_current_density_perm(pg, case):
    d, g, s = load_golden(case)
    G = to_pg_grid(g)
    q = float(d["q"])
    for order in (1, 3):
        J = pg.deposit_scalar(s, G, order, q=q)
        assert peak_rel_err((J.jx, J.jy, J.jz), d[f"J_o{order}"]) <= J_TOL
        rho = pg.deposit_density(s, G, order, q * s["w"])
        assert np.array_equal(rho, d[f"rho_o{order}"]), f"rho order {order} not bit-exact"
    perm, starts, counts = pg.counting_sort(s, G)
    assert np.array_equal(perm, d["perm"])


@pytest.mark.parametrize("case", golden_cases())
def test_golden_session_lockstep(pg, case):
    """Session (device-resident bins): push + incremental sort each step must
    reproduce the reference's positions bit-for-bit and its bin sets."""
    d, g, s = load_golden(case)
    G = to_pg_grid(g)
    q = float(d["q"])
    with pg.Session(G, order=3) as S:
        S.upload(s, q=q)
        assert S.capacity == int(d["cap_gpma"])  # same layout rule as Gpma::layout
        k = 1
        while f"adv{k}_x" in d:
            st = S.step(float(d["dt"]), pg.STEP_PUSH | pg.STEP_SORT)
            assert st["moved"] / len(s["x"]) == float(d[f"adv{k}_frac"])
            p = S.particles()
            mine = np.argsort(p.id)
            want = np.argsort(d[f"adv{k}_id"])
            for a in ("x", "y", "z"):
                assert np.array_equal(getattr(p, a)[mine], d[f"adv{k}_{a}"][want])
            off, cnt = S.bins()
            bin_of = np.repeat(np.arange(G.ncells, dtype=np.uint32), cnt.astype(np.int64))
            assert np.array_equal(bin_of[mine], d[f"bins{k}"][want])
            k += 1
        S.step(0.5, pg.STEP_CURRENT | pg.STEP_DENSITY)
        J = S.current()
        assert peak_rel_err((J.jx, J.jy, J.jz), d["final_J_o3_bin_order"]) <= J_TOL


# ---------------------------------------------------------- oracle, many cases


@pytest.mark.parametrize("order", [1, 2, 3])
@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_current_vs_oracle(pg, orc, order, gi):
    g = O.Grid.make(**GRIDS[gi])
    s = scramble(orc.make_plasma(g, 7, 0.3 * min(g.dx, g.dy, g.dz), 100 + gi), gi)
    s["x"][:3] += np.array([1.0, -2.0, 5.0]) * g.nx * g.dx  # out-of-box positions wrap
    q = -0.75
    want = orc.deposit_current(g, order, s, q)
    J = pg.deposit_scalar(s, to_pg_grid(g), order, q=q)
    assert peak_rel_err((J.jx, J.jy, J.jz), want) <= J_TOL


@pytest.mark.parametrize("order", [1, 2, 3])
@pytest.mark.parametrize("sorted_input", [True, False])
@pytest.mark.parametrize("gi", [0, 1, 2, 3])
def test_density_bit_exact(pg, orc, order, sorted_input, gi):
    g = O.Grid.make(**GRIDS[gi])
    s = orc.make_plasma(g, 5, 0.2 * min(g.dx, g.dy, g.dz), 200 + gi)
    for _ in range(2):
        orc.advance(g, 0.5, s)
    if sorted_input:
        perm, _, _ = orc.counting_sort(g, s)
        s = {k: np.ascontiguousarray(v[perm]) for k, v in s.items()}
    else:
        s = scramble(s, gi)
    quantity = np.random.default_rng(gi).standard_normal(len(s["x"]))
    want = orc.deposit_density(g, order, s, quantity)
    got = pg.deposit_density(s, to_pg_grid(g), order, quantity)
    assert np.array_equal(got, want), f"{np.count_nonzero(got != want)} nodes differ"


@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_counting_sort_and_cells_exact(pg, orc, gi):
    g = O.Grid.make(**GRIDS[gi])
    s = scramble(orc.make_plasma(g, 6, 0.1, 300 + gi), gi)
    s["y"][:4] = [-1e-18, 1e30, -1e30, np.nextafter(g.oy + g.ny * g.dy, 0)]
    perm, starts, counts = orc.counting_sort(g, s)
    gp, gs, gc = pg.counting_sort(s, to_pg_grid(g))
    assert np.array_equal(gp, perm) and np.array_equal(gs, starts) and np.array_equal(gc, counts)
    assert np.array_equal(pg.cells(s, to_pg_grid(g)), orc.cells(g, s))


@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_advance_bit_exact(pg, orc, gi):
    g = O.Grid.make(**GRIDS[gi])
    ms = min(g.dx, g.dy, g.dz)
    s = orc.make_plasma(g, 4, 0.9 * ms, 400 + gi)  # hot: many crossings and wraps
    for k in ("vx", "vy", "vz"):  # keep |v|*dt under the single-cell cap (workload.hpp:142-147)
        s[k] = np.clip(s[k], -0.55 * ms / 0.5, 0.55 * ms / 0.5)
    sp = pg.ParticleSoA.from_dict({k: v.copy() for k, v in s.items()})
    G = to_pg_grid(g)
    for _ in range(5):
        m = orc.advance(g, 0.5, s)
        f = pg.advance(sp, 0.5, G)
        assert f == m / len(s["x"])
        for a in ("x", "y", "z"):
            assert np.array_equal(getattr(sp, a), s[a])


def test_single_particle_kats(pg):
    G = pg.Grid.make(4)
    one = dict(x=[1.0], y=[2.0], z=[3.0], vx=[0.5], vy=[-1.0], vz=[0.25], w=[3.0])  # test_pipeline.cpp:76-90
    J = pg.deposit_scalar(one, G, pg.CIC, q=2.0)
    node = G.linear_id(1, 2, 3)
    assert J.jx[node] == pytest.approx(3.0, rel=1e-15) and J.jy[node] == pytest.approx(-6.0, rel=1e-15)
    assert np.count_nonzero(J.jx) == 1
    one.update(x=[1.3], y=[2.3], z=[3.3])
    J = pg.deposit_scalar(one, G, pg.QSP, q=2.0)
    assert np.count_nonzero(J.jx) == 64
    assert sum(J.component_sums()) == pytest.approx(3.0 - 6.0 + 1.5, rel=1e-13)
    J2 = pg.deposit_scalar(one, G, pg.TSC, q=2.0)
    assert np.count_nonzero(J2.jx) == 27
    G6 = pg.Grid.make(6)  # test_acceptance.cpp:322-341
    one = dict(x=[2.3], y=[3.45], z=[1.7], vx=[0.4], vy=[-0.2], vz=[0.1], w=[1.5])
    J = pg.deposit_scalar(one, G6, pg.QSP, q=-2.0)
    for c in range(3):
        assert np.count_nonzero(J.component(c)) == 64


def test_empty_inputs(pg):
    G = pg.Grid.make(4)
    empty = {k: np.zeros(0) for k in ("x", "y", "z", "vx", "vy", "vz", "w")}
    for order in (1, 2, 3):
        J = pg.deposit_scalar(empty, G, order)
        assert not np.any(J.jx) and not np.any(J.jy) and not np.any(J.jz)
        assert not np.any(pg.deposit_density(empty, G, order, np.zeros(0)))
    perm, starts, counts = pg.counting_sort(empty, G)
    assert len(perm) == 0 and not np.any(counts)


def test_errors_map_to_reference_exceptions(pg):
    G = pg.Grid.make(4)
    bad = dict(x=[np.nan], y=[1.0], z=[1.0], vx=[0.0], vy=[0.0], vz=[0.0], w=[1.0])
    with pytest.raises(pg.InvalidArgument):
        pg.deposit_scalar(bad, G, 1)
    with pytest.raises(pg.InvalidArgument):
        pg.counting_sort(bad, G)
    ok = dict(x=[1.0], y=[1.0], z=[1.0], vx=[0.0], vy=[0.0], vz=[0.0], w=[1.0])
    with pytest.raises(pg.InvalidArgument):
        pg.deposit_scalar(ok, G, 4)
    fast = pg.ParticleSoA.from_dict(dict(ok, vx=[2.5]))
    with pytest.raises(pg.DomainError):
        pg.advance(fast, 0.5, G)
    with pytest.raises(pg.InvalidArgument):
        pg.deposit_scalar(ok, pg.Grid.make(0, 4, 4), 1)


def test_current_on_tiny_grids_aliasing(pg, orc):
    """Grids smaller than the stencil window: the periodic footprint aliases
    onto itself; every halo node is reduced, never overwritten."""
    for dims in [(1, 1, 1), (2, 3, 1), (3, 3, 3), (2, 2, 9)]:
        g = O.Grid.make(*dims)
        s = orc.make_plasma(g, 9, 0.1, 9)
        for order in (1, 2, 3):
            want = orc.deposit_current(g, order, s, 1.0)
            J = pg.deposit_scalar(s, to_pg_grid(g), order, q=1.0)
            assert peak_rel_err((J.jx, J.jy, J.jz), want) <= J_TOL, (dims, order)


# ------------------------------------------------------------------- sessions


@pytest.mark.parametrize("order", [1, 2, 3])
def test_session_lockstep_vs_oracle(pg, orc, order):
    g = O.Grid.make(12, 10, 9)
    s = orc.make_plasma(g, 6, 0.35, 31)
    q = -1.0
    G = to_pg_grid(g)
    with pg.Session(G, order=order) as S:
        S.upload(s, q=q)
        perm, _, _ = orc.counting_sort(g, s)
        cur = {k: np.ascontiguousarray(v[perm]) for k, v in s.items()}
        for step in range(6):
            moved = orc.advance(g, 0.5, cur)
            st = S.step(0.5, pg.STEP_PUSH | pg.STEP_SORT | pg.STEP_CURRENT | pg.STEP_DENSITY)
            assert st["moved"] == moved
            p = S.particles()
            mine, want = np.argsort(p.id), np.argsort(cur["id"])
            for a in ("x", "y", "z", "vx", "vy", "vz", "w"):
                assert np.array_equal(getattr(p, a)[mine], cur[a][want])
            # bins: every particle sits in the bin of its cell; storage is cell-sorted
            off, cnt = S.bins()
            bin_of = np.repeat(np.arange(G.ncells, dtype=np.uint32), cnt.astype(np.int64))
            assert np.array_equal(bin_of, orc.cells(g, {"x": p.x, "y": p.y, "z": p.z}))
            # J against the oracle; rho bit-exact against the oracle on the GPU's storage order
            pd = {"x": p.x, "y": p.y, "z": p.z, "vx": p.vx, "vy": p.vy, "vz": p.vz, "w": p.w}
            J = S.current()
            assert peak_rel_err((J.jx, J.jy, J.jz), orc.deposit_current(g, order, pd, q)) <= J_TOL
            assert np.array_equal(S.density(), orc.deposit_density(g, order, pd, q * p.w))


def test_session_no_slack_stays_exact(pg, orc):
    """No slack at all (gap 0, min_gap 0): arrivals overflow every step and are
    placed by borrowing or a rebuild; the store stays exact."""
    g = O.Grid.make(8)
    s = orc.make_plasma(g, 4, 0.6, 5)
    G = to_pg_grid(g)
    with pg.Session(G, order=3, gap_ratio=0.0, min_gap=0) as S:
        S.upload(s, q=1.0)
        assert S.capacity == len(s["x"])
        perm, _, _ = orc.counting_sort(g, s)
        cur = {k: np.ascontiguousarray(v[perm]) for k, v in s.items()}
        for _ in range(4):
            orc.advance(g, 0.5, cur)
            st = S.step(0.5, pg.STEP_DEFAULT)
            assert st["overflowed"] > 0
            p = S.particles()
            off, cnt = S.bins()
            assert int(cnt.sum()) == len(s["x"])
            assert np.all(np.diff(off.astype(np.int64)) >= cnt)
            bin_of = np.repeat(np.arange(G.ncells, dtype=np.uint32), cnt.astype(np.int64))
            assert np.array_equal(bin_of, orc.cells(g, {"x": p.x, "y": p.y, "z": p.z}))
            assert np.array_equal(np.sort(p.id), np.sort(cur["id"]))
            J = S.current()
            pd = {"x": p.x, "y": p.y, "z": p.z, "vx": p.vx, "vy": p.vy, "vz": p.vz, "w": p.w}
            assert peak_rel_err((J.jx, J.jy, J.jz), orc.deposit_current(g, 3, pd, 1.0)) <= J_TOL


def _line_store(xs, vxs):
    n = len(xs)
    return {"x": np.array(xs, float), "y": np.full(n, 0.5), "z": np.full(n, 0.5), "vx": np.array(vxs, float),
            "vy": np.zeros(n), "vz": np.zeros(n), "w": np.ones(n), "id": np.arange(n, dtype=np.uint64)}


def test_session_borrow_from_next_bins(pg, orc):
    """borrow_insert analogue (gpma.hpp:337-370): bin 1 is full, bins 2/3 lend
    their slack, boundaries shift, no rebuild."""
    G = pg.Grid.make(8, 1, 1)
    # cell 0: three particles that move to cell 1; cell 1: one stayer; cells 2, 3 empty
    s = _line_store([0.9, 0.8, 0.7, 1.5], [0.6, 0.6, 0.8, 0.0])
    with pg.Session(G, order=1, gap_ratio=0.0, min_gap=1) as S:
        S.upload(s, q=1.0)
        off0, cnt0 = S.bins()
        assert list(np.diff(off0.astype(np.int64))) == [4, 2, 1, 1, 1, 1, 1, 1]
        st = S.step(0.5, pg.STEP_DEFAULT)
        assert st["moved"] == 3 and st["overflowed"] == 2 and st["rebuilt"] == 0
        off, cnt = S.bins()
        assert list(cnt) == [0, 4, 0, 0, 0, 0, 0, 0]
        assert list(np.diff(off.astype(np.int64))) == [4, 4, 0, 0, 1, 1, 1, 1]
        p = S.particles()
        assert sorted(p.id.tolist()) == [0, 1, 2, 3]
        want = orc.deposit_current(O.Grid.make(8, 1, 1), 1, {k: getattr(p, k) for k in
                                                              ("x", "y", "z", "vx", "vy", "vz", "w")}, 1.0)
        J = S.current()
        assert peak_rel_err((J.jx, J.jy, J.jz), want) <= J_TOL


def test_session_no_donor_rebuilds(pg, orc):
    """Arrivals with no slack within the 4-bin scan window trigger the rebuild
    (apply_moves -> rebuild, gpma.hpp:119-122)."""
    G = pg.Grid.make(8, 1, 1)
    s = _line_store([0.5] * 10, [1.2] * 10)
    with pg.Session(G, order=1, gap_ratio=0.0, min_gap=0) as S:
        S.upload(s, q=1.0)
        st = S.step(0.5, pg.STEP_DEFAULT)
        assert st["moved"] == 10 and st["rebuilt"] == 1
        off, cnt = S.bins()
        assert list(cnt) == [0, 10, 0, 0, 0, 0, 0, 0]
        assert list(np.diff(off.astype(np.int64))) == [0, 10, 0, 0, 0, 0, 0, 0]
        p = S.particles()
        assert np.allclose(p.x, 1.1) and sorted(p.id.tolist()) == list(range(10))


def test_session_global_sort_and_stats(pg, orc):
    g = O.Grid.make(10)
    s = orc.make_plasma(g, 8, 0.3, 8)
    G = to_pg_grid(g)
    with pg.Session(G, order=1) as S:
        S.upload(s, q=-1.0)
        cap0 = S.capacity
        rebuilt = 0
        for _ in range(3):
            st = S.step(0.5)
            rebuilt += st["rebuilt"]
        assert st["num_particles"] == len(s["x"])
        if not rebuilt:
            assert st["capacity"] == cap0
        cap0 = st["capacity"]
        assert st["empty_slot_ratio"] == pytest.approx((cap0 - len(s["x"])) / cap0)
        J0 = S.current()
        st = S.step(0.5, pg.STEP_CURRENT | pg.STEP_GLOBAL_SORT)
        assert st["global_sorted"] == 1
        off, cnt = S.bins()
        caps = np.diff(off.astype(np.int64))
        assert np.array_equal(caps, np.ceil(cnt * 1.25).astype(np.int64) + 2)
        S.step(0.5, pg.STEP_CURRENT)
        J1 = S.current()
        assert peak_rel_err((J1.jx, J1.jy, J1.jz), (J0.jx, J0.jy, J0.jz)) <= J_TOL


def test_session_generator_matches_cpu_generator(pg, orc):
    g = O.Grid.make(6, 5, 4)
    with pg.Session(to_pg_grid(g), order=3) as S:
        S.generate_plasma(4, 0.05, seed=3)
        p = S.particles()
    s = orc.make_plasma(g, 4, 0.05, 3)
    mine, want = np.argsort(p.id), np.argsort(s["id"])
    for a in ("x", "y", "z", "w"):
        assert np.array_equal(getattr(p, a)[mine], s[a][want])  # integer-hash uniforms: exact
    for a in ("vx", "vy", "vz"):
        assert np.allclose(getattr(p, a)[mine], s[a][want], rtol=1e-14, atol=1e-17)  # libm last ulp


def test_launch_counter_moves(pg, orc):
    before = pg.kernel_launches()
    g = O.Grid.make(4)
    s = orc.make_plasma(g, 2, 0.1, 1)
    pg.deposit_scalar(s, to_pg_grid(g), 3)
    assert pg.kernel_launches() > before


def _hp_deposit(p, g, order, q):
    """80-bit longdouble deposition (exact shape forms, shape.hpp:26-43 and the
    TSC restatement in oracle/picoracle.c po_shape_1d) -- an accuracy yardstick
    independent of summation order."""
    L = np.longdouble
    W = 2 if order == 1 else 4
    off = 0 if order == 1 else -1

    def shape(d):
        if order == 1:
            return [1 - d, d]
        if order == 3:
            u = 1 - d
            return [u ** 3 / 6, (4 - 6 * d * d + 3 * d ** 3) / 6, (1 + 3 * d + 3 * d * d - 3 * d ** 3) / 6, d ** 3 / 6]
        up = d >= L(0.5)
        dl = np.where(up, d - 1, d)
        a, b, m = L(0.5) * (L(0.5) - dl) ** 2, L(0.75) - dl * dl, L(0.5) * (L(0.5) + dl) ** 2
        z = np.zeros_like(d)
        return [np.where(up, z, a), np.where(up, a, b), np.where(up, b, m), np.where(up, m, z)]

    dims = (g.nx, g.ny, g.nz)
    org = (g.ox, g.oy, g.oz)
    hs = (g.dx, g.dy, g.dz)
    J = np.zeros((3, g.nz, g.ny, g.nx), dtype=L)
    ci, S = [], []
    for a, k in enumerate("xyz"):
        u = (np.asarray(getattr(p, k), dtype=L) - L(org[a])) / L(hs[a])
        c = np.floor(u)
        S.append(shape(u - c))
        ci.append(c.astype(np.int64))
    wq = [L(q) * np.asarray(p.w, dtype=L) * np.asarray(getattr(p, v), dtype=L) for v in ("vx", "vy", "vz")]
    for kz in range(W):
        for jy in range(W):
            for ix in range(W):
                X = (ci[0] + off + ix) % dims[0]
                Y = (ci[1] + off + jy) % dims[1]
                Z = (ci[2] + off + kz) % dims[2]
                s = S[0][ix] * S[1][jy] * S[2][kz]
                for c in range(3):
                    np.add.at(J[c], (Z, Y, X), wq[c] * s)
    return J.reshape(3, -1)


@pytest.mark.gpu
@pytest.mark.parametrize("order", [1, 2, 3])
def test_session_current_vs_extended_precision(pg, order):
    """The session's J after several push/sort steps of a hot plasma is within
    a few ulps (peak-normalised) of an 80-bit deposit of the same particles:
    the FMA weight polynomials and the register accumulation cost < 1e-14."""
    g = pg.Grid.make(16, 8, 8, dx=0.5, dy=0.5, dz=0.5, origin=(-2.0, 0.0, 1.0))
    S = pg.Session(g, order)
    S.generate_plasma(4, 0.6, seed=7)
    for _ in range(4):
        S.step(0.5)
    p = S.particles()
    J = S.current()
    hp = _hp_deposit(p, g, order, -1.0)
    got = np.stack([J.jx, J.jy, J.jz]).astype(np.longdouble)
    err = float(np.abs(got - hp).max() / np.abs(hp).max())
    assert err < 1e-14, err


def test_session_mover_buffer_overflow_resorts_exactly(pg, orc):
    """Every particle changes cell in one step: the movers exceed the mover
    buffer (64 records per 256-slot push block), the unrecorded ones stay in
    their stale bins and the step falls back to a full stable re-sort.  The
    state must still equal the oracle's, and the next steps run normally."""
    g = O.Grid.make(128, 32, 32)
    s = orc.make_plasma(g, 4, 0.0, seed=5)  # 524288 particles at rest
    s["vx"][:] = 1.5                        # dt 0.5: every particle moves +0.75 cell in x
    s["vx"][::7] = -1.9
    q = -1.0
    S = pg.Session(to_pg_grid(g), 3)
    S.upload(s, q=q)
    ref = {k: v.copy() for k, v in s.items()}
    for step in range(3):
        st = S.step(0.5)
        moved = orc.advance(g, 0.5, ref)
        assert st["moved"] == moved
        if step == 0:
            assert st["rebuilt"] == 1 and moved > S.num_particles // 4
        got = S.particles()
        o = np.argsort(got.id)
        w = np.argsort(ref["id"]) if "id" in ref else np.arange(len(ref["x"]))
        for k in ("x", "y", "z"):
            assert np.array_equal(getattr(got, k)[o], ref[k][w]), (step, k)
        cells = orc.cells(g, {k: getattr(got, k) for k in ("x", "y", "z")})
        assert np.all(np.diff(cells.astype(np.int64)) >= 0)  # storage is cell-sorted
        J = S.current()
        assert peak_rel_err((J.jx, J.jy, J.jz), orc.deposit_current(g, 3, ref, q)) <= J_TOL


@pytest.mark.parametrize("order", [1, 2, 3])
@pytest.mark.parametrize("gi", [0, 1, 3])
def test_fused_step_matches_unfused_and_oracle(pg, orc, order, gi):
    """The default step fuses push + move detection + J into one pass over the
    bins (movers deposited by their own kernel).  Against the unfused step
    (push kernel, sort, J kernel) and the oracle: positions and moved counts
    bit-exact, the same bin sets, J within the bar, rho bit-exact."""
    kw = GRIDS[gi]
    g = O.Grid.make(kw["nx"], kw.get("ny"), kw.get("nz"), kw.get("dx", 1.0), kw.get("dy", 1.0),
                    kw.get("dz", 1.0), kw.get("origin", (0.0, 0.0, 0.0)))
    s = orc.make_plasma(g, 5, 0.08 if gi == 1 else 0.4, 17 + gi)
    q = -1.0
    G = to_pg_grid(g)
    perm, _, _ = orc.counting_sort(g, s)
    cur = {k: np.ascontiguousarray(v[perm]) for k, v in s.items()}
    with pg.Session(G, order=order) as A, pg.Session(G, order=order) as B:
        A.set_fusion(2.0)  # fuse every step, whatever the migration
        A.upload(s, q=q)
        B.upload(s, q=q)
        for step in range(5):
            moved = orc.advance(g, 0.5, cur)
            sa = A.step(0.5, pg.STEP_DEFAULT | pg.STEP_DENSITY)
            sb = B.step(0.5, pg.STEP_DEFAULT | pg.STEP_DENSITY | pg.STEP_UNFUSED)
            assert sa["moved"] == sb["moved"] == moved
            pa, pb = A.particles(), B.particles()
            oa, ob, oc = np.argsort(pa.id), np.argsort(pb.id), np.argsort(cur["id"])
            for k in ("x", "y", "z", "vx", "vy", "vz", "w"):
                assert np.array_equal(getattr(pa, k)[oa], cur[k][oc]), (step, k)
                assert np.array_equal(getattr(pb, k)[ob], cur[k][oc]), (step, k)
            (offa, cnta), (offb, cntb) = A.bins(), B.bins()
            assert np.array_equal(cnta, cntb)
            ca = np.repeat(np.arange(G.ncells), cnta.astype(np.int64))
            assert np.array_equal(ca, orc.cells(g, {"x": pa.x, "y": pa.y, "z": pa.z}))
            # same set per bin
            assert np.array_equal(pa.id[np.lexsort((pa.id, ca))], pb.id[np.lexsort((pb.id, ca))])
            pd = {"x": pa.x, "y": pa.y, "z": pa.z, "vx": pa.vx, "vy": pa.vy, "vz": pa.vz, "w": pa.w}
            want = orc.deposit_current(g, order, pd, q)
            Ja, Jb = A.current(), B.current()
            assert peak_rel_err((Ja.jx, Ja.jy, Ja.jz), want) <= J_TOL
            assert peak_rel_err((Jb.jx, Jb.jy, Jb.jz), want) <= J_TOL
            assert np.array_equal(A.density(), orc.deposit_density(g, order, pd, q * pa.w))


def test_fused_step_cap_violation(pg):
    """The fused pass raises the reference's exception for a displacement above
    the one-cell cap (advance, workload.hpp:147: std::domain_error)."""
    G = pg.Grid.make(8, 8, 8)
    s = _line_store([0.5, 2.5], [0.1, 0.1])
    with pg.Session(G, order=3) as S:
        s2 = dict(s)
        s2["vx"] = np.array([0.1, 3.0])
        S.upload(s2, q=1.0)
        with pytest.raises(pg.DomainError):
            S.step(0.5)


def test_fusion_policy_follows_migration(pg, orc):
    """The fused pass runs while the previous step's moved fraction stays under
    the session's threshold (default 6%), the separate kernels otherwise."""
    g = O.Grid.make(16)
    cold = orc.make_plasma(g, 4, 0.01, 3)  # ~1% of the particles change cell per step
    hot = orc.make_plasma(g, 4, 0.3, 3)    # ~30%
    with pg.Session(to_pg_grid(g), order=3) as S:
        with pytest.raises(pg.InvalidArgument):
            S.set_fusion(-1.0)
        S.upload(cold, q=-1.0)
        assert [S.step(0.5)["fused"] for _ in range(3)] == [1, 1, 1]
        S.upload(hot, q=-1.0)
        first = S.step(0.5)  # decided on the previous (cold) step
        assert first["fused"] == 1 and first["moved"] > 0.03 * S.num_particles
        assert [S.step(0.5)["fused"] for _ in range(2)] == [0, 0]
        S.set_fusion(0.0)
        S.upload(cold, q=-1.0)
        assert S.step(0.5)["fused"] == 0
        S.set_fusion(2.0)
        S.upload(hot, q=-1.0)
        assert [S.step(0.5)["fused"] for _ in range(2)] == [1, 1]
        assert S.step(0.5, pg.STEP_DEFAULT | pg.STEP_UNFUSED)["fused"] == 0


def test_fused_mover_segment_overflow(pg, orc):
    """Movers concentrated in a few CTAs (a fast beam in one x-tile column, as
    C4's beam): their per-CTA segments overflow into the shared overflow
    segment (no drop, no full re-sort).  Same particles, bins and J as the
    unfused step and the oracle."""
    g = O.Grid.make(64)
    s = orc.make_plasma(g, 4, 0.0, seed=9)           # 1,048,576 particles at rest
    beam = s["x"] < 8.0                              # one 8-cell column of tiles
    s["vx"][beam] = 1.5                              # dt 0.5: +0.75 cell, ~3/4 change cell
    q = -1.0
    G = to_pg_grid(g)
    ref = {k: v.copy() for k, v in s.items()}
    with pg.Session(G, order=3) as A, pg.Session(G, order=3) as B:
        A.set_fusion(2.0)
        A.upload(s, q=q)
        B.upload(s, q=q)
        for step in range(3):
            moved = orc.advance(g, 0.5, ref)
            sa = A.step(0.5)
            sb = B.step(0.5, pg.STEP_DEFAULT | pg.STEP_UNFUSED)
            assert sa["fused"] == 1 and sb["fused"] == 0
            assert sa["moved"] == sb["moved"] == moved > 50000
            assert sa["rebuilt"] == 0  # the overflow segment held every mover
            pa, pb = A.particles(), B.particles()
            oa, ob, oc = np.argsort(pa.id), np.argsort(pb.id), np.argsort(ref["id"])
            for k in ("x", "y", "z"):
                assert np.array_equal(getattr(pa, k)[oa], ref[k][oc]), (step, k)
                assert np.array_equal(getattr(pb, k)[ob], ref[k][oc]), (step, k)
            (_, cnta), (_, cntb) = A.bins(), B.bins()
            assert np.array_equal(cnta, cntb)
            want = orc.deposit_current(g, 3, ref, q)
            Ja = A.current()
            assert peak_rel_err((Ja.jx, Ja.jy, Ja.jz), want) <= J_TOL


@pytest.mark.parametrize("order", [1, 3])
def test_fused_long_run_with_holes_and_rebuilds(pg, orc, order):
    """Forty fused steps (holes, borrows and rebuilds accumulate) in lockstep
    with the oracle: positions bit-exact every step, every particle in the bin
    of its cell, J within the bar and rho bit-exact at checkpoints."""
    g = O.Grid.make(24, 20, 16)
    s = orc.make_plasma(g, 8, 0.12, seed=21)
    q = -1.0
    G = to_pg_grid(g)
    perm, _, _ = orc.counting_sort(g, s)
    cur = {k: np.ascontiguousarray(v[perm]) for k, v in s.items()}
    rebuilt = 0
    with pg.Session(G, order=order, gap_ratio=0.1, min_gap=1) as S:
        S.set_fusion(2.0)
        S.upload(s, q=q)
        for step in range(40):
            moved = orc.advance(g, 0.5, cur)
            st = S.step(0.5)
            assert st["fused"] == 1 and st["moved"] == moved
            rebuilt += st["rebuilt"]
            if step % 8 == 7:
                p = S.particles()
                a, b = np.argsort(p.id), np.argsort(cur["id"])
                for k in ("x", "y", "z", "vx", "vy", "vz", "w"):
                    assert np.array_equal(getattr(p, k)[a], cur[k][b]), (step, k)
                off, cnt = S.bins()
                cells = np.repeat(np.arange(G.ncells, dtype=np.uint32), cnt.astype(np.int64))
                assert np.array_equal(cells, orc.cells(g, {"x": p.x, "y": p.y, "z": p.z}))
                pd = {"x": p.x, "y": p.y, "z": p.z, "vx": p.vx, "vy": p.vy, "vz": p.vz, "w": p.w}
                J = S.current()
                assert peak_rel_err((J.jx, J.jy, J.jz), orc.deposit_current(g, order, pd, q)) <= J_TOL
                S.step(0.5, pg.STEP_DENSITY)  # rho of the current store (no push)
                p = S.particles()  # storage order after the hole packing rho does first
                pd = {"x": p.x, "y": p.y, "z": p.z, "vx": p.vx, "vy": p.vy, "vz": p.vz, "w": p.w}
                assert np.array_equal(S.density(), orc.deposit_density(g, order, pd, q * p.w))
    assert rebuilt > 0  # tight slack: the run exercised rebuilds too
