"""The hand-written stable radix sort (csrc/radix_sort.cu) behind gpma_build /
global_sort / every stateless call, through the C ABI (picgpu_counting_sort):
the permutation must equal a stable counting sort by cell
(proj/include/pic/gpma.hpp:379-394) on every key distribution the sorter
meets -- random, already sorted, nearly sorted (a binned store after a push),
reversed, one hot cell, all in one cell -- at tile-ragged sizes and key
widths of 1 to 4 radix passes."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _store_for_cells(g, cells, rng):
    """Particles placed inside the given cells (cell-relative uniform offsets)."""
    i = cells % g.nx
    j = (cells // g.nx) % g.ny
    k = cells // (g.nx * g.ny)
    n = len(cells)
    s = {"x": g.ox + (i + rng.random(n) * 0.999) * g.dx, "y": g.oy + (j + rng.random(n) * 0.999) * g.dy,
         "z": g.oz + (k + rng.random(n) * 0.999) * g.dz}
    for v in ("vx", "vy", "vz"):
        s[v] = np.zeros(n)
    s["w"] = np.ones(n)
    return s


def _check(pg, orc, g, s):
    from conftest import to_pg_grid

    cells = orc.cells(g, s)
    want = np.argsort(cells, kind="stable").astype(np.uint32)
    perm, starts, counts = pg.counting_sort(s, to_pg_grid(g))
    assert np.array_equal(perm, want)
    cnt = np.bincount(cells, minlength=g.ncells).astype(np.uint32)
    assert np.array_equal(counts, cnt)
    st = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.uint32)
    assert np.array_equal(starts[cnt > 0], st[cnt > 0])


@pytest.mark.parametrize("dist", ["random", "sorted", "nearly_sorted", "reversed", "hot_cell", "one_cell"])
@pytest.mark.parametrize("n", [1, 4095, 4097, 300001])
def test_stable_sort_distributions(pg, orc, dist, n):
    g = O.Grid.make(40, 30, 20)  # 24000 cells: 15-bit keys, 2 passes
    rng = np.random.default_rng(n + len(dist))
    nc = g.ncells
    if dist == "random":
        cells = rng.integers(0, nc, n)
    elif dist == "sorted":
        cells = np.sort(rng.integers(0, nc, n))
    elif dist == "nearly_sorted":
        cells = np.sort(rng.integers(0, nc, n))
        m = rng.random(n) < 0.05
        cells[m] = np.clip(cells[m] + rng.integers(-1, 2, m.sum()), 0, nc - 1)
    elif dist == "reversed":
        cells = np.sort(rng.integers(0, nc, n))[::-1].copy()
    elif dist == "hot_cell":
        cells = rng.integers(0, nc, n)
        cells[rng.random(n) < 0.6] = 12345
    else:
        cells = np.full(n, 777)
    _check(pg, orc, g, _store_for_cells(g, cells.astype(np.int64), rng))


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 1, 1), (16, 16, 1), (64, 64, 64), (256, 128, 128), (512, 256, 256)])
def test_stable_sort_key_widths(pg, orc, dims):
    """1 cell (1-bit keys) up to 2^25 cells (512x256x256: 4 radix passes)."""
    g = O.Grid.make(*dims)
    rng = np.random.default_rng(sum(dims))
    n = min(2_000_000, max(10, g.ncells * 2))
    cells = rng.integers(0, g.ncells, n)
    _check(pg, orc, g, _store_for_cells(g, cells.astype(np.int64), rng))


def test_stable_sort_full_c2_size(pg, orc):
    """C2's 33.5M particles (128^3 cells, 8136 tiles of the look-back chain)."""
    g = O.Grid.make(128)
    s = orc.make_plasma(g, 16, 0.01, seed=3)
    p = np.random.default_rng(1).permutation(len(s["x"]))
    s = {k: np.ascontiguousarray(v[p]) for k, v in s.items()}
    _check(pg, orc, g, s)
