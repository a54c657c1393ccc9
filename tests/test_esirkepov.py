"""Charge-conserving (Esirkepov) current deposition on the Yee grid -- this
project's extension (north_star's first clause).  The reference has only the
direct collocated deposit (proj/include/pic/deposit.hpp:60-73; SPEC.md:8 lists
charge-conserving schemes as future work), so this path is UNPINNED by the
reference.  Its pins:
  * the discrete continuity equation, (rho(x1) - rho(x0)) / dt + div J = 0 to
    round-off, with rho the reference-pinned deposit_density (q*w*S on nodes);
  * uniform translation: the summed face current equals q*w*v (CPU, oracle);
  * GPU (-m gpu): the sm_100a kernel equals the C restatement at 1e-12.
"""
import numpy as np
import pytest

import oracle as O


def _divergence(g, jx, jy, jz):
    sh = (g.nz, g.ny, g.nx)
    X, Y, Z = (a.reshape(sh) for a in (jx, jy, jz))
    return ((X - np.roll(X, 1, axis=2)) / g.dx + (Y - np.roll(Y, 1, axis=1)) / g.dy
            + (Z - np.roll(Z, 1, axis=0)) / g.dz).ravel()


def _pair(orc, g, n, seed, cap=0.9):
    """Old positions uniform in the box, new = old + a displacement under one
    cell per axis, wrapped into the box (the push's wrap_position)."""
    rng = np.random.default_rng(seed)
    L = np.array([g.nx * g.dx, g.ny * g.dy, g.nz * g.dz])
    o = np.array([g.ox, g.oy, g.oz])
    h = np.array([g.dx, g.dy, g.dz])
    x0 = o + rng.random((n, 3)) * L
    x1 = x0 + (rng.random((n, 3)) * 2 - 1) * cap * h
    x1 = o + np.mod(x1 - o, L)
    old = {k: np.ascontiguousarray(x0[:, a]) for a, k in enumerate("xyz")}
    new = {k: np.ascontiguousarray(x1[:, a]) for a, k in enumerate("xyz")}
    w = rng.random(n) + 0.5
    return old, new, w


def continuity_residual(orc, g, order, old, new, w, q, dt, J):
    r0 = orc.deposit_density(g, order, old, q * w)
    r1 = orc.deposit_density(g, order, new, q * w)
    res = (r1 - r0) / dt + _divergence(g, *J)
    scale = np.abs(r1 - r0).max() / dt
    return float(np.abs(res).max() / scale)


@pytest.mark.parametrize("order", [1, 2, 3])
@pytest.mark.parametrize("gi", [0, 1, 2])
def test_oracle_esirkepov_conserves_charge(orc, order, gi):
    g = [O.Grid.make(8), O.Grid.make(13, 6, 9, 0.5, 1.0, 0.25, origin=(-1.0, 2.0, 0.5)),
         O.Grid.make(5, 4, 7, 0.3, 1.7, 0.05)][gi]
    old, new, w = _pair(orc, g, 3000, 7 + gi)
    q, dt = -1.0, 0.37
    J = orc.deposit_esirkepov(g, order, old, new, w, q, dt)
    assert continuity_residual(orc, g, order, old, new, w, q, dt, J) < 1e-12


@pytest.mark.parametrize("order", [1, 2, 3])
def test_oracle_esirkepov_uniform_translation(orc, order):
    """Every particle moves by the same v*dt: sum of jx over the faces = q*sum(w)*vx."""
    g = O.Grid.make(10, 9, 8)
    old, _, w = _pair(orc, g, 500, 3)
    v = np.array([0.31, -0.22, 0.17])
    dt = 0.9
    new = {k: old[k] + v[a] * dt for a, k in enumerate("xyz")}
    Lx = np.array([g.nx, g.ny, g.nz], float)
    for a, k in enumerate("xyz"):
        new[k] = np.mod(new[k], Lx[a])
    q = 0.7
    jx, jy, jz = orc.deposit_esirkepov(g, order, old, new, w, q, dt)
    for J, vc in ((jx, v[0]), (jy, v[1]), (jz, v[2])):
        assert J.sum() == pytest.approx(q * w.sum() * vc, rel=1e-12)


def test_oracle_esirkepov_rejects_jumps(orc):
    g = O.Grid.make(8)
    old = {"x": np.array([1.5]), "y": np.array([1.5]), "z": np.array([1.5])}
    new = {"x": np.array([3.6]), "y": np.array([1.5]), "z": np.array([1.5])}
    with pytest.raises(ArithmeticError):
        orc.deposit_esirkepov(g, 3, old, new, np.ones(1), 1.0, 0.5)


# --------------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("order", [1, 2, 3])
@pytest.mark.parametrize("gi", [0, 1, 2])
def test_gpu_esirkepov_matches_oracle_and_conserves_charge(pg, orc, order, gi):
    from conftest import peak_rel_err, to_pg_grid

    g = [O.Grid.make(8), O.Grid.make(13, 6, 9, 0.5, 1.0, 0.25, origin=(-1.0, 2.0, 0.5)),
         O.Grid.make(5, 4, 7, 0.3, 1.7, 0.05)][gi]
    old, new, w = _pair(orc, g, 20000, 11 + gi)
    q, dt = -1.0, 0.37
    J = pg.deposit_esirkepov(old, new, w, to_pg_grid(g), order, q, dt)
    got = (J.jx, J.jy, J.jz)
    assert peak_rel_err(got, orc.deposit_esirkepov(g, order, old, new, w, q, dt)) <= 1e-12
    assert continuity_residual(orc, g, order, old, new, w, q, dt, got) < 1e-12


@pytest.mark.gpu
def test_gpu_esirkepov_session_step_conserves_charge(pg, orc):
    """Positions before and after a bit-exact session push (64^3 x 4 ppc, QSP):
    the GPU Esirkepov current closes the continuity equation with the
    bit-exact GPU rho of both states."""
    from conftest import to_pg_grid

    g = O.Grid.make(64)
    G = to_pg_grid(g)
    with pg.Session(G, order=3) as S:
        S.generate_plasma(4, 0.3, seed=5)
        p0 = S.particles()
        S.step(0.5)
        p1 = S.particles()
    a, b = np.argsort(p0.id), np.argsort(p1.id)
    old = {k: getattr(p0, k)[a] for k in "xyz"}
    new = {k: getattr(p1, k)[b] for k in "xyz"}
    w = p0.w[a]
    q, dt = -1.0, 0.5
    J = pg.deposit_esirkepov(old, new, w, G, 3, q, dt)
    zero = np.zeros_like(w)
    full = lambda d: {**d, "vx": zero, "vy": zero, "vz": zero, "w": w}  # noqa: E731
    r0 = pg.deposit_density(full(old), G, 3, q * w)
    r1 = pg.deposit_density(full(new), G, 3, q * w)
    res = (r1 - r0) / dt + _divergence(g, J.jx, J.jy, J.jz)
    assert np.abs(res).max() / (np.abs(r1 - r0).max() / dt) < 1e-12


@pytest.mark.gpu
def test_gpu_esirkepov_errors(pg):
    G = pg.Grid.make(8)
    one = {"x": np.array([1.5]), "y": np.array([1.5]), "z": np.array([1.5])}
    far = {"x": np.array([3.6]), "y": np.array([1.5]), "z": np.array([1.5])}
    with pytest.raises(pg.DomainError):
        pg.deposit_esirkepov(one, far, np.ones(1), G, 3, 1.0, 0.5)
    nan = {"x": np.array([np.nan]), "y": np.array([1.5]), "z": np.array([1.5])}
    with pytest.raises(pg.InvalidArgument):
        pg.deposit_esirkepov(one, nan, np.ones(1), G, 3, 1.0, 0.5)
    with pytest.raises(pg.InvalidArgument):
        pg.deposit_esirkepov(one, one, np.ones(1), G, 3, 1.0, 0.0)
