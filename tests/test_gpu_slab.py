"""x-slab decomposition on the GPU: P slab sessions driven in
lockstep on one device (the exchanges are device copies; test_slab_cpu.py covers
the same protocol over gloo) against the undecomposed session and the oracle.

Parity bar: pushed positions, velocities and ids bit-exact; moved counts exact;
assembled J within 1e-12 peak-normalised, rho within 1e-13 (only the summation
order across a seam differs); migration lossless (id multiset unchanged,
proj/tests/test_domain.cpp:202-218)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _grid(pg, nx=16, ny=8, nz=8):
    return pg.Grid.make(nx, ny, nz, dx=0.5, dy=0.5, dz=0.5, origin=(-2.0, 0.0, 1.0))


def _sorted(soa):
    o = np.argsort(soa.id)
    return {k: getattr(soa, k)[o] for k in ("x", "y", "z", "vx", "vy", "vz", "w", "id")}


def _slabs(pg, G, P, order, **kw):
    from paper_2601_08277_b200.slab import SlabSession, slab_range

    return [SlabSession(G, *slab_range(G.nx, P, r), order=order, **kw) for r in range(P)]


def _union(sessions):
    parts = [s.particles() for s in sessions]
    cat = {k: np.concatenate([getattr(p, k) for p in parts]) for k in ("x", "y", "z", "vx", "vy", "vz", "w", "id")}
    o = np.argsort(cat["id"])
    return {k: v[o] for k, v in cat.items()}


def _assemble(sessions, what):
    from paper_2601_08277_b200.slab import assemble_x

    if what == "rho":
        return assemble_x([s.owned_density() for s in sessions])
    comps = [s.owned_current() for s in sessions]
    return [assemble_x([c[i] for c in comps]) for i in range(3)]


def test_slab_generate_is_global_generator(pg):
    G = _grid(pg)
    ref = pg.Session(G, 3)
    ref.generate_plasma(4, 0.2, seed=5)
    slabs = _slabs(pg, G, 3, 3)
    for s in slabs:
        s.generate_plasma(4, 0.2, seed=5)
    got, want = _union(slabs), _sorted(ref.particles())
    for k in want:
        assert np.array_equal(got[k], want[k]), k
    assert sum(s.num_particles for s in slabs) == ref.num_particles


@pytest.mark.parametrize("order,P", [(1, 2), (2, 3), (3, 1), (3, 2), (3, 3), (3, 4)])
def test_slab_steps_match_undecomposed(pg, orc, order, P):
    import oracle
    from paper_2601_08277_b200.slab import local_ring_step

    G = _grid(pg)
    flags = pg.STEP_DEFAULT | pg.STEP_DENSITY
    ref = pg.Session(G, order)
    ref.generate_plasma(4, 0.6, seed=7)  # fast: many particles cross slab faces each step
    slabs = _slabs(pg, G, P, order)
    for s in slabs:
        s.generate_plasma(4, 0.6, seed=7)
    sent = 0
    for step in range(6):
        want = ref.step(0.5, flags)
        stats = local_ring_step(slabs, 0.5, flags)
        sent += sum(st["sent"] for st in stats)
        assert sum(st["moved"] for st in stats) == want["moved"]
        assert sum(st["num_particles"] for st in stats) == want["num_particles"]
        J = _assemble(slabs, "J")
        Jr = ref.current()
        assert oracle.peak_rel_err(J, [Jr.jx, Jr.jy, Jr.jz]) < 1e-12, step
        assert oracle.peak_rel_err([_assemble(slabs, "rho")], [ref.density()]) < 1e-13
    if P > 1:
        assert sent > 0
    got, want = _union(slabs), _sorted(ref.particles())
    for k in want:
        assert np.array_equal(got[k], want[k]), k
    # and against the oracle's global J of the final state
    s = {k: want[k] for k in ("x", "y", "z", "vx", "vy", "vz", "w")}
    Go = oracle.Grid.make(G.nx, G.ny, G.nz, dx=G.dx, dy=G.dy, dz=G.dz, origin=(G.ox, G.oy, G.oz))
    Jo = orc.deposit_current(Go, order, s, -1.0)
    assert oracle.peak_rel_err(_assemble(slabs, "J"), Jo) < 1e-12


def test_slab_tight_slack_rebuilds(pg):
    """No slack at all: every arrival (own movers and neighbours') borrows or
    forces a rebuild; the decomposition must stay lossless and exact."""
    import oracle
    from paper_2601_08277_b200.slab import local_ring_step

    G = _grid(pg, 12, 6, 6)
    ref = pg.Session(G, 3, gap_ratio=0.0, min_gap=0)
    ref.generate_plasma(3, 0.6, seed=3)
    slabs = _slabs(pg, G, 3, 3, gap_ratio=0.0, min_gap=0)
    for s in slabs:
        s.generate_plasma(3, 0.6, seed=3)
    rebuilt = 0
    for _ in range(5):
        ref.step(0.5)
        stats = local_ring_step(slabs, 0.5)
        rebuilt += sum(st["rebuilt"] for st in stats)
    assert rebuilt > 0
    got, want = _union(slabs), _sorted(ref.particles())
    for k in want:
        assert np.array_equal(got[k], want[k]), k
    Jr = ref.current()
    assert oracle.peak_rel_err(_assemble(slabs, "J"), [Jr.jx, Jr.jy, Jr.jz]) < 1e-12


def test_slab_upload_owned_and_errors(pg, orc):
    import oracle
    from paper_2601_08277_b200.slab import SlabSession, local_ring_step, slab_grid

    G = _grid(pg)
    Go = oracle.Grid.make(G.nx, G.ny, G.nz, dx=G.dx, dy=G.dy, dz=G.dz, origin=(G.ox, G.oy, G.oz))
    d = orc.make_plasma(Go, 2, 0.3, seed=9)
    soa = pg.ParticleSoA.from_dict(d, q=-1.0)
    slabs = _slabs(pg, G, 2, 3)
    for s in slabs:
        s.upload_owned(soa)
    assert sum(s.num_particles for s in slabs) == soa.size()
    local_ring_step(slabs, 0.5)
    assert sum(s.num_particles for s in slabs) == soa.size()
    s0 = slabs[0]
    with pytest.raises(pg.LogicError):
        s0.step(0.5)  # slab sessions use begin/end
    with pytest.raises(pg.LogicError):
        s0.end(None)  # no step in progress
    with pytest.raises(pg.LogicError):  # set_slab needs an empty session
        pg._check(pg.lib().picgpu_session_set_slab(s0._h, C.byref(G), 0, 8, 2))
    fresh = SlabSession(G, 0, 8, order=3)
    with pytest.raises(pg.InvalidArgument):  # particles outside the slab
        fresh.upload(soa)
    bad = pg.Session(slab_grid(G, 0, 6), 3)  # grid of another slab
    with pytest.raises(pg.InvalidArgument):
        pg._check(pg.lib().picgpu_session_set_slab(bad._h, C.byref(G), 0, 8, 2))


@pytest.mark.parametrize("order,bucket,uth", [(3, 0, 0.6), (1, 0, 0.6), (3, 16, 0.6), (2, 0, 0.02)])
def test_nccl_slab_step_matches_undecomposed(pg, order, bucket, uth):
    """The whole slab step behind the C ABI (picgpu_session_slab_step): leaver
    counts and records over NCCL on the session stream (a one-rank ring: this
    rank is both neighbours), arrivals imported from device-side counts, guard
    planes summed over NCCL.  Against the undecomposed session: particles
    bit-exact, J <= 1e-12, rho <= 1e-13.  bucket 16: most leavers travel in the
    second, exactly sized round.  u_th 0.02: the fused step (low migration)."""
    import oracle
    from paper_2601_08277_b200.slab import NcclComm, SlabSession, attach_comm, nccl_slab_step

    G = _grid(pg)
    flags = pg.STEP_DEFAULT | pg.STEP_DENSITY
    ref = pg.Session(G, order)
    ref.generate_plasma(4, uth, seed=7)
    comm = NcclComm(device=0, world=1, rank=0)
    s = SlabSession(G, 0, G.nx, order=order)
    s.generate_plasma(4, uth, seed=7)
    attach_comm(s, comm, bucket)
    fused = 0
    for step in range(6):
        want = ref.step(0.5, flags)
        got = nccl_slab_step(s, 0.5, flags)
        fused += got["fused"]
        assert got["moved"] == want["moved"] and got["num_particles"] == want["num_particles"], step
        a, b = _union([s]), _sorted(ref.particles())
        for k in b:
            assert np.array_equal(a[k], b[k]), (step, k)
        J = _assemble([s], "J")
        Jr = ref.current()
        assert oracle.peak_rel_err(J, (Jr.jx, Jr.jy, Jr.jz)) <= 1e-12, step
        rho = _assemble([s], "rho")
        assert np.abs(rho - ref.density()).max() <= 1e-13 * np.abs(ref.density()).max(), step
    if uth < 0.1:
        assert fused == 6
    comm.close()


def test_nccl_slab_step_errors(pg):
    from paper_2601_08277_b200.slab import SlabSession, nccl_slab_step

    G = _grid(pg)
    s = SlabSession(G, 0, G.nx, order=3)
    s.generate_plasma(2, 0.1, seed=1)
    with pytest.raises(pg.LogicError):  # no communicator attached
        nccl_slab_step(s, 0.5)
    plain = pg.Session(G, 3)
    from paper_2601_08277_b200 import _check, lib

    with pytest.raises(pg.LogicError):  # not a slab session
        _check(lib().picgpu_session_set_comm(plain._h, None, 0))
