"""Host side of the x-slab decomposition on CPU, world size
2 and 3 over gloo: the partition, the slab grid, the ring exchange, and the
guard-plane protocol end to end with the oracle standing in for each rank's
local deposit (the assembled J must equal the oracle's global J).  The GPU
kernels of the same protocol are covered in test_gpu_slab.py."""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    return dist


def test_slab_range_partitions():
    from paper_2601_08277_b200.slab import slab_range

    for nx in (4, 7, 12, 128, 1000):
        for world in (1, 2, 3, 5, 8):
            if world * 2 > nx:
                continue
            parts = [slab_range(nx, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == nx
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            widths = [b - a for a, b in parts]
            assert max(widths) - min(widths) <= 1


def test_slab_grid_host_only(pg):
    """picgpu_slab_grid is host arithmetic (works without a GPU)."""
    from paper_2601_08277_b200.slab import slab_grid

    g = pg.Grid.make(16, 8, 4, dx=0.25, dy=0.5, dz=1.0, origin=(-1.0, 0.5, 2.0))
    L = slab_grid(g, 4, 9, 2)
    assert (L.nx, L.ny, L.nz) == (5 + 4, 8, 4)
    assert L.ox == -1.0 + (4 - 2) * 0.25 and (L.oy, L.oz) == (0.5, 2.0)
    for bad in ((0, 0, 2), (3, 2, 2), (0, 17, 2), (0, 1, 2), (0, 8, 1)):
        with pytest.raises(pg.InvalidArgument):
            slab_grid(g, *bad)


def _exchange_worker(rank, world, port):
    import torch

    dist = _init(rank, world, port)
    from paper_2601_08277_b200.slab import RingExchange

    ring = RingExchange()
    # rank r sends (r, dir, i) rows; counts vary per rank and direction, some zero
    nl, nr = (rank * 3) % 4, (rank * 5 + 1) % 3

    def rows(n, d):
        return torch.tensor([[rank, d, i] + [0.0] * 5 for i in range(n)], dtype=torch.float64).reshape(n, 8)

    fl, fr = ring.exchange(rows(nl, 0), rows(nr, 1), sized=True)
    left, right = (rank - 1) % world, (rank + 1) % world
    want_l = (left * 5 + 1) % 3  # left rank's to_right count
    want_r = (right * 3) % 4  # right rank's to_left count
    assert fl.shape == (want_l, 8) and fr.shape == (want_r, 8)
    assert all(int(r[0]) == left and int(r[1]) == 1 for r in fl)
    assert all(int(r[0]) == right and int(r[1]) == 0 for r in fr)
    assert [int(r[2]) for r in fl] == list(range(want_l))
    # fixed-size exchange (guard planes)
    lo, hi = torch.full((1, 6), float(rank)), torch.full((1, 6), 100.0 + rank)
    gl, gr = ring.exchange(lo, hi)
    assert torch.all(gl == 100.0 + left) and torch.all(gr == float(right))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ring_exchange_gloo(world):
    import torch.multiprocessing as mp

    mp.spawn(_exchange_worker, args=(world, _free_port()), nprocs=world, join=True)


def _guard_worker(rank, world, port, order):
    import torch

    dist = _init(rank, world, port)
    import oracle
    import paper_2601_08277_b200 as pg
    from paper_2601_08277_b200.slab import GHOST, RingExchange, slab_grid, slab_range

    orc = oracle.Oracle()
    nx, ny, nz = 12, 6, 5
    G = oracle.Grid.make(nx, ny, nz, dx=0.5, dy=0.25, dz=0.5, origin=(-1.0, 0.0, 0.5))
    s = orc.make_plasma(G, 3, 0.05, seed=11)
    x0, x1 = slab_range(nx, world, rank)
    pgG = pg.Grid.make(nx, ny, nz, dx=0.5, dy=0.25, dz=0.5, origin=(-1.0, 0.0, 0.5))
    L = slab_grid(pgG, x0, x1, GHOST)
    Lo = oracle.Grid.make(L.nx, L.ny, L.nz, dx=L.dx, dy=L.dy, dz=L.dz, origin=(L.ox, L.oy, L.oz))
    ix = orc.cells(G, s) % nx
    mine = {k: np.ascontiguousarray(v[(ix >= x0) & (ix < x1)]) for k, v in s.items()}
    J = np.stack(orc.deposit_current(Lo, order, mine, -1.0)).reshape(3, nz, ny, L.nx)
    own = x1 - x0

    def pack(p0):  # [comp][plane][z][y], the kernels' layout
        return torch.from_numpy(np.ascontiguousarray(np.transpose(J[..., p0:p0 + GHOST], (0, 3, 1, 2))).reshape(1, -1))

    ring = RingExchange()
    gl, gr = ring.exchange(pack(0), pack(GHOST + own))

    def add(buf, p0):
        J[..., p0:p0 + GHOST] += np.transpose(buf.numpy().reshape(3, GHOST, nz, ny), (0, 2, 3, 1))

    add(gl, GHOST)
    add(gr, own)
    part = torch.from_numpy(np.ascontiguousarray(J[..., GHOST:GHOST + own]))
    parts = [None] * world
    dist.all_gather_object(parts, part)
    if rank == 0:
        full = np.concatenate([p.numpy() for p in parts], axis=3).reshape(3, -1)
        want = np.stack(orc.deposit_current(G, order, s, -1.0))
        assert oracle.peak_rel_err(list(full), list(want)) < 1e-12, order
    dist.destroy_process_group()


@pytest.mark.parametrize("world,order", [(2, 1), (2, 3), (3, 2), (3, 3)])
def test_guard_plane_protocol_gloo(world, order):
    import torch.multiprocessing as mp

    mp.spawn(_guard_worker, args=(world, _free_port(), order), nprocs=world, join=True)
