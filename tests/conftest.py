import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    import oracle

    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.reference_available():
        pytest.skip("oracle/_ref/libpicref.so not built (needs /root/reference at build time)")
    return oracle.Reference()


@pytest.fixture(scope="session")
def pg():
    import paper_2601_08277_b200 as pg

    pg.lib()
    return pg


def golden_cases():
    return sorted(os.path.splitext(os.path.basename(p))[0] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_golden(name):
    import oracle

    d = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    nx, ny, nz = (int(v) for v in d["grid"])
    g = oracle.Grid.make(nx, ny, nz, *d["spacing"], origin=tuple(d["origin"]))
    s = {k: d[k] for k in ("x", "y", "z", "vx", "vy", "vz", "w", "id")}
    return d, g, s


def to_pg_grid(g):
    import paper_2601_08277_b200 as pg

    return pg.Grid(g.nx, g.ny, g.nz, 0, g.dx, g.dy, g.dz, g.ox, g.oy, g.oz)


def peak_rel_err(got, want):
    import oracle

    return oracle.peak_rel_err(got, want)
