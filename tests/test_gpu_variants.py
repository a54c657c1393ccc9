"""The reference's deposition variants (R10-R17): deposit_tiled (MOPA tile
pipeline, deposit.hpp:284-334) and deposit_rhocell_vector (deposit.hpp:87-119)
compute the same J as deposit_scalar.  On the GPU they run the FP64
tensor-core (DMMA) kernel and the warp-DFMA kernel; the tile engine's
KernelCounters are reproduced exactly from the grouping the reference sees."""
import numpy as np
import pytest

from conftest import peak_rel_err, to_pg_grid
from test_gpu_parity import GRIDS, J_TOL, scramble

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("order", [1, 2, 3])
@pytest.mark.parametrize("gi", [0, 1, 2, 3, 4])
def test_variant_kernels_vs_oracle(pg, orc, order, gi):
    g = O.Grid.make(**GRIDS[gi])
    s = scramble(orc.make_plasma(g, 6, 0.3 * min(g.dx, g.dy, g.dz), 300 + gi), gi)
    want = orc.deposit_current(g, order, s, -1.0)
    G = to_pg_grid(g)
    times = pg.StageTimes()
    Jt = pg.deposit_tiled(s, G, order, pg.TiledOptions(), times, q=-1.0)
    assert peak_rel_err((Jt.jx, Jt.jy, Jt.jz), want) <= J_TOL
    assert times.compute > 0.0 and times.preproc > 0.0 and times.reduce == 0.0
    Jv = pg.deposit_rhocell_vector(s, G, order, q=-1.0)
    assert peak_rel_err((Jv.jx, Jv.jy, Jv.jz), want) <= J_TOL


@pytest.mark.parametrize("order", [1, 3])
@pytest.mark.parametrize("layout", ["unsorted", "sorted", "bins"])
def test_tiled_counters_and_J_match_reference(pg, orc, ref, order, layout):
    g = O.Grid.make(9, 7, 6, dx=0.5, dy=1.0, dz=0.5, origin=(-1.0, 0.0, 2.0))
    s = orc.make_plasma(g, 5, 0.2, seed=17)
    if layout == "unsorted":
        s = scramble(s, 4)
    rs = ref.state(g, s, -1.0)
    if layout != "unsorted":
        rs.gpma_build()
        s = {k: v for k, v in rs.particles().items() if k in s}
    G = to_pg_grid(g)
    for residency, dual in ((True, False), (False, False), (True, True)):
        (jr, (m, e)) = rs.deposit_tiled_opt(order, use_gpma=layout == "bins", residency=residency, dual_tile=dual)
        kc = pg.KernelCounters()
        opt = pg.TiledOptions(gpma=layout == "bins", residency=residency, dual_tile=dual, counters=kc)
        J = pg.deposit_tiled(s, G, order, opt, q=-1.0)
        assert (kc.mopa_calls, kc.extract_passes) == (m, e), (residency, dual)
        assert peak_rel_err((J.jx, J.jy, J.jz), jr) <= J_TOL
    # counters accumulate across calls, like the reference's ++
    pg.deposit_tiled(s, G, order, opt, q=-1.0)
    assert (kc.mopa_calls, kc.extract_passes) == (2 * m, 2 * e)
    jr = rs.deposit_rhocell(order, use_gpma=layout == "bins")
    J = pg.deposit_rhocell_vector(s, G, order, gpma=layout == "bins", q=-1.0)
    assert peak_rel_err((J.jx, J.jy, J.jz), jr) <= J_TOL


def test_variants_reject_grid_below_stencil(pg):
    G = pg.Grid.make(3, 8, 8)  # NodeMap: QSP needs 4 nodes per axis (rhocell.hpp:49)
    s = {k: np.full(2, 0.5) for k in ("x", "y", "z", "vx", "vy", "vz", "w")}
    with pytest.raises(pg.InvalidArgument):
        pg.deposit_tiled(s, G, 3)
    with pytest.raises(pg.InvalidArgument):
        pg.deposit_rhocell_vector(s, G, 3)
    pg.deposit_tiled(s, G, 1)  # CIC needs 2


def test_variants_empty_input(pg):
    G = pg.Grid.make(6)
    s = {k: np.zeros(0) for k in ("x", "y", "z", "vx", "vy", "vz", "w")}
    kc = pg.KernelCounters()
    J = pg.deposit_tiled(s, G, 3, pg.TiledOptions(counters=kc))
    assert not J.jx.any() and (kc.mopa_calls, kc.extract_passes) == (0, 0)
    assert not pg.deposit_rhocell_vector(s, G, 3).jz.any()
