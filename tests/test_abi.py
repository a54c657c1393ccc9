"""CPU tests of the C-ABI boundary: the library loads, exports exactly what
include/picgpu.h declares, host-only entry points behave, and compute calls
FAIL LOUDLY without a GPU (there is no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "picgpu.h")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"PICGPU_API\s+[\w\s\*]*?\b(picgpu_\w+)\s*\(", txt)))


def test_header_declares_entry_points():
    names = declared()
    assert "picgpu_deposit_current" in names and "picgpu_session_step" in names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol(pg):
    out = subprocess.run(["nm", "-D", "--defined-only", pg.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (picgpu_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    L = pg.lib()
    for n in declared():
        assert hasattr(L, n)


def test_library_is_sm100a(pg):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pg.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_only_entry_points(pg):
    L = pg.lib()
    assert L.picgpu_abi_version() == 1
    assert pg.flop_count(1) == 76 and pg.flop_count(3) == 534 and pg.flop_count(2) == 238
    pol = pg.SortPolicy.defaults()
    assert (pol.sort_interval, pol.min_sort_interval, pol.trigger_rebuild_count) == (50, 10, 100)
    st = pg.RankSortStats()
    st.steps_since_sort = 50
    assert pg.should_global_sort(st, pol) == "interval"
    st.steps_since_sort = 20
    st.empty_slot_ratio = 0.5
    st.perf_metric, st.baseline_perf = 79.9, 100.0
    assert pg.should_global_sort(st, pol) == "perf_degradation"


def test_policy_table_matches_oracle(pg, orc):
    rng = np.random.default_rng(3)
    pol = pg.SortPolicy.defaults()
    for _ in range(300):
        st = pg.RankSortStats()
        st.steps_since_sort = int(rng.integers(0, 120))
        st.cumulative_local_rebuilds = int(rng.integers(0, 200))
        st.empty_slot_ratio = float(rng.random())
        st.perf_metric = float(rng.random() * 100)
        st.baseline_perf = float(rng.random() * 100) * (rng.random() < 0.7)
        want = orc.should_global_sort(st.steps_since_sort, st.cumulative_local_rebuilds, st.empty_slot_ratio,
                                      st.perf_metric, st.baseline_perf)
        assert pg.lib().picgpu_should_global_sort(C.byref(st), C.byref(pol)) == want


def _gpu_present():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_gpu_present(), reason="checks the no-GPU failure mode")
def test_compute_fails_loudly_without_gpu(pg):
    g = pg.Grid.make(4)
    s = {k: np.zeros(3) + 0.5 for k in ("x", "y", "z", "vx", "vy", "vz", "w")}
    with pytest.raises(pg.PicError):
        pg.deposit_scalar(s, g, 1)


def test_cpp_shim_compiles():
    """include/picgpu.hpp (the pic:: mirror) is self-contained C++20."""
    r = subprocess.run(["g++", "-std=gnu++20", "-fsyntax-only", "-x", "c++", "-I", os.path.join(ROOT, "include"), "-"],
                       input='#include "picgpu.hpp"\nint main() { picgpu::GridSpec g; g.validate(); return 0; }\n',
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
