"""ctypes bindings for the parity checkers.  TEST INFRASTRUCTURE ONLY.

`Oracle` wraps oracle/liboracle.so (this repo's C restatement, picoracle.c).
`Reference` wraps oracle/_ref/libpicref.so (the unmodified reference headers
compiled by oracle/Makefile).  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpicref.so")

_d = C.c_double
_u32 = C.c_uint32
_u64 = C.c_uint64
_i32 = C.c_int32
_p = C.c_void_p


class Grid(C.Structure):
    """Same layout as picgpu_grid (include/picgpu.h) / pic::GridSpec fields."""

    _fields_ = [("nx", _i32), ("ny", _i32), ("nz", _i32), ("pad", _i32),
                ("dx", _d), ("dy", _d), ("dz", _d),
                ("ox", _d), ("oy", _d), ("oz", _d)]

    @classmethod
    def make(cls, nx, ny=None, nz=None, dx=1.0, dy=1.0, dz=1.0, origin=(0.0, 0.0, 0.0)):
        ny = nx if ny is None else ny
        nz = nx if nz is None else nz
        return cls(nx, ny, nz, 0, dx, dy, dz, *origin)

    @property
    def ncells(self):
        return self.nx * self.ny * self.nz


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_p)


def build():
    subprocess.check_call(["make", "-s", "-C", HERE])


class Oracle:
    """The C restatement of the reference hot path (picoracle.c)."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.po_uniform01.restype = _d
        L.po_uniform01.argtypes = [_u64, _u64, _u64]
        L.po_gaussian.restype = _d
        L.po_gaussian.argtypes = [_u64, _u64, _u64]
        L.po_cell_of.argtypes = [C.POINTER(Grid), _d, _d, _d, _p, _p]
        L.po_shape_1d.argtypes = [C.c_int, _d, _p, _p]
        L.po_deposit_current.argtypes = [C.POINTER(Grid), C.c_int] + [_p] * 7 + [_d, _u64, _p, _p, _p, _p]
        L.po_deposit_density.argtypes = [C.POINTER(Grid), C.c_int, _p, _p, _p, _p, _u64, _p]
        L.po_counting_sort.argtypes = [C.POINTER(Grid), _p, _p, _p, _u64, _p, _p, _p]
        L.po_advance.argtypes = [C.POINTER(Grid), _d, _p, _p, _p, _p, _p, _p, _u64, _p]
        L.po_cells.argtypes = [C.POINTER(Grid), _p, _p, _p, _u64, _p]
        L.po_deposit_esirkepov.argtypes = [C.POINTER(Grid), C.c_int] + [_p] * 7 + [_d, _d, _u64, _p, _p, _p]
        L.po_make_plasma.argtypes = [C.POINTER(Grid), C.c_int, _d, _u64] + [_p] * 8
        L.po_make_plasma.restype = None
        L.po_should_global_sort.argtypes = [_u32, _u64, _d, _d, _d, _u32, _u32, _u32, _d, _d, C.c_int, _d]
        self.L = L

    def uniform01(self, seed, stream, counter):
        return self.L.po_uniform01(seed, stream, counter)

    def gaussian(self, seed, stream, counter):
        return self.L.po_gaussian(seed, stream, counter)

    def cell_of(self, g, x, y, z):
        ijk = np.zeros(3, np.int32)
        lin = np.zeros(1, np.uint32)
        rc = self.L.po_cell_of(C.byref(g), x, y, z, _ptr(ijk), _ptr(lin))
        if rc:
            raise ValueError("cell_of: non-finite particle position")
        return tuple(int(v) for v in ijk), int(lin[0])

    def shape_1d(self, order, d):
        out = np.zeros(4)
        off = np.zeros(1, np.int32)
        if self.L.po_shape_1d(order, d, _ptr(out), _ptr(off)):
            raise ValueError("shape: coordinate outside [0,1)")
        return out, int(off[0])

    def deposit_current(self, g, order, s, q, visit=None):
        jx, jy, jz = (np.zeros(g.ncells) for _ in range(3))
        n = len(s["x"])
        rc = self.L.po_deposit_current(C.byref(g), order, *(_ptr(s[k]) for k in ("x", "y", "z", "vx", "vy", "vz", "w")),
                                       q, n, _ptr(visit), _ptr(jx), _ptr(jy), _ptr(jz))
        if rc:
            raise ValueError(f"deposit_current failed ({rc})")
        return jx, jy, jz

    def deposit_esirkepov(self, g, order, old, new, w, q, dt):
        """Charge-conserving J on the Yee faces (this project's extension; unpinned by the reference)."""
        jx, jy, jz = (np.zeros(g.ncells) for _ in range(3))
        n = len(w)
        rc = self.L.po_deposit_esirkepov(C.byref(g), order, *(_ptr(np.ascontiguousarray(a)) for a in
                                                              (old["x"], old["y"], old["z"], new["x"], new["y"],
                                                               new["z"], w)), q, dt, n, _ptr(jx), _ptr(jy), _ptr(jz))
        if rc:
            raise {5: ArithmeticError}.get(rc, ValueError)(f"deposit_esirkepov failed ({rc})")
        return jx, jy, jz

    def deposit_density(self, g, order, s, quantity):
        rho = np.zeros(g.ncells)
        rc = self.L.po_deposit_density(C.byref(g), order, _ptr(s["x"]), _ptr(s["y"]), _ptr(s["z"]),
                                       _ptr(quantity), len(quantity), _ptr(rho))
        if rc:
            raise ValueError(f"deposit_density failed ({rc})")
        return rho

    def counting_sort(self, g, s):
        n = len(s["x"])
        perm = np.zeros(max(n, 1), np.uint32)[:n]
        starts = np.zeros(g.ncells, np.uint32)
        counts = np.zeros(g.ncells, np.uint32)
        rc = self.L.po_counting_sort(C.byref(g), _ptr(s["x"]), _ptr(s["y"]), _ptr(s["z"]), n,
                                     _ptr(perm), _ptr(starts), _ptr(counts))
        if rc:
            raise ValueError("counting_sort: non-finite position")
        return perm, starts, counts

    def advance(self, g, dt, s):
        """In place, like pic::advance.  Returns the moved count."""
        moved = np.zeros(1, np.uint64)
        rc = self.L.po_advance(C.byref(g), dt, *(_ptr(s[k]) for k in ("x", "y", "z", "vx", "vy", "vz")),
                               len(s["x"]), _ptr(moved))
        if rc == 5:
            raise ArithmeticError("advance: particle displacement exceeds the single-cell cap")
        if rc:
            raise ValueError("advance: non-finite particle position")
        return int(moved[0])

    def cells(self, g, s):
        cell = np.zeros(len(s["x"]), np.uint32)
        if self.L.po_cells(C.byref(g), _ptr(s["x"]), _ptr(s["y"]), _ptr(s["z"]), len(s["x"]), _ptr(cell)):
            raise ValueError("cells: non-finite position")
        return cell

    def make_plasma(self, g, ppc, u_th, seed=1):
        n = g.ncells * ppc
        s = {k: np.zeros(n) for k in ("x", "y", "z", "vx", "vy", "vz", "w")}
        s["id"] = np.zeros(n, np.uint64)
        self.L.po_make_plasma(C.byref(g), ppc, u_th, seed,
                              *(_ptr(s[k]) for k in ("x", "y", "z", "vx", "vy", "vz", "w", "id")))
        return s

    def should_global_sort(self, steps, rebuilds, ratio, perf, base, sort_interval=50, min_sort_interval=10,
                           trigger_rebuild_count=100, trigger_empty_ratio=0.15, trigger_full_ratio=0.85,
                           perf_enable=True, perf_degrad=0.80):
        return self.L.po_should_global_sort(steps, rebuilds, ratio, perf, base, sort_interval, min_sort_interval,
                                            trigger_rebuild_count, trigger_empty_ratio, trigger_full_ratio,
                                            int(perf_enable), perf_degrad)

    def flop_count(self, order):
        return self.L.po_flop_count(order)


def reference_available():
    return os.path.exists(REF_SO)


class Reference:
    """The reference's own functions (compiled headers, oracle/_ref/libpicref.so)."""

    def __init__(self, path=REF_SO):
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_create.restype = _p
        L.ref_create.argtypes = [C.POINTER(Grid), _u64] + [_p] * 8 + [_d]
        L.ref_destroy.argtypes = [_p]
        L.ref_size.restype = _u64
        L.ref_size.argtypes = [_p]
        L.ref_get_particles.argtypes = [_p] * 9
        L.ref_get_particles.restype = None
        L.ref_deposit_scalar.argtypes = [_p, C.c_int, C.c_int, _p, _p, _p]
        L.ref_deposit_scalar_mt.argtypes = [_p, C.c_int, C.c_int, _p, _p, _p]
        L.ref_deposit_density.argtypes = [_p, C.c_int, _p, _p]
        L.ref_deposit_tiled.argtypes = [_p, C.c_int, C.c_int, _p, _p, _p]
        L.ref_make_workload.argtypes = [_p] * 9
        L.ref_run_simulation.argtypes = [_p, C.c_char_p, _p, C.c_double, C.c_uint32] + [_p] * 15
        L.ref_deposit_tiled_opt.argtypes = [_p, C.c_int, C.c_int, C.c_int, C.c_int, _p, _p, _p, _p, _p]
        L.ref_deposit_rhocell.argtypes = [_p, C.c_int, C.c_int, _p, _p, _p]
        L.ref_gpma_build.argtypes = [_p, _d, _u32]
        L.ref_advance.argtypes = [_p, _d, _p]
        L.ref_incremental_sort.argtypes = [_p, _p]
        L.ref_bins.argtypes = [_p, _p, _p]
        L.ref_gpma_stats.argtypes = [_p, _p, _p]
        L.ref_gpma_stats.restype = None
        L.ref_step_timed.argtypes = [_p, C.c_int, _d, _p, _p]
        L.ref_density_timed.argtypes = [_p, C.c_int, _p]
        L.ref_cell_of.argtypes = [C.POINTER(Grid), _d, _d, _d, _p, _p]
        L.ref_intra_cell.argtypes = [C.POINTER(Grid), _d, _d, _d, _p]
        L.ref_shape_1d.argtypes = [C.c_int, _d, _p]
        L.ref_should_global_sort.argtypes = [_u32, _u64, _d, _d, _d, _u32, _u32, _u32, _d, _d, C.c_int, _d]
        L.ref_uniform01.restype = _d
        L.ref_uniform01.argtypes = [_u64, _u64, _u64]
        L.ref_gaussian.restype = _d
        L.ref_gaussian.argtypes = [_u64, _u64, _u64]
        self.L = L

    def _check(self, rc):
        if rc:
            msg = self.L.ref_last_error().decode()
            raise {1: ValueError, 2: IndexError, 3: MemoryError, 4: RuntimeError,
                   5: ArithmeticError}.get(rc, RuntimeError)(msg)

    def make_workload(self, wl):
        """pic::make_workload; wl is a paper_2601_08277_b200.WorkloadConfig (same C layout)."""
        n = wl.grid.nx * wl.grid.ny * wl.grid.nz * wl.ppc
        out = {k: np.zeros(n) for k in ("x", "y", "z", "vx", "vy", "vz", "w")}
        out["id"] = np.zeros(n, np.uint64)
        self._check(self.L.ref_make_workload(C.byref(wl), *(_ptr(out[k]) for k in
                                                            ("x", "y", "z", "vx", "vy", "vz", "w", "id"))))
        return out

    def run_simulation(self, wl, mode, policy, gap_ratio=0.25, min_gap=2):
        """pic::run_simulation; policy is a paper_2601_08277_b200.SortPolicy (same C layout)."""
        n = wl.grid.nx * wl.grid.ny * wl.grid.nz * wl.ppc
        nc = wl.grid.nx * wl.grid.ny * wl.grid.nz
        fm = np.zeros(max(wl.steps, 1))
        rb = np.zeros(max(wl.steps, 1), np.uint32)
        rs = np.zeros(max(wl.steps, 1), np.int32)
        ck = np.zeros(3)
        J = [np.zeros(nc) for _ in range(3)]
        out = {k: np.zeros(n) for k in ("x", "y", "z", "vx", "vy", "vz", "w")}
        out["id"] = np.zeros(n, np.uint64)
        self._check(self.L.ref_run_simulation(C.byref(wl), mode.encode(), C.byref(policy), gap_ratio, min_gap,
                                              _ptr(fm), _ptr(rb), _ptr(rs), _ptr(ck), *(_ptr(j) for j in J),
                                              *(_ptr(out[k]) for k in ("x", "y", "z", "vx", "vy", "vz", "w", "id"))))
        return dict(fraction_moved=fm[:wl.steps], rebuilds=rb[:wl.steps], reasons=rs[:wl.steps], checksum=ck,
                    J=J, particles=out)

    def state(self, g, s, q):
        return RefState(self, g, s, q)

    def cell_of(self, g, x, y, z):
        ijk = np.zeros(3, np.int32)
        lin = np.zeros(1, np.uint32)
        self._check(self.L.ref_cell_of(C.byref(g), x, y, z, _ptr(ijk), _ptr(lin)))
        return tuple(int(v) for v in ijk), int(lin[0])

    def intra_cell(self, g, x, y, z):
        d = np.zeros(3)
        self._check(self.L.ref_intra_cell(C.byref(g), x, y, z, _ptr(d)))
        return d

    def shape_1d(self, order, d):
        out = np.zeros(4)
        self._check(self.L.ref_shape_1d(order, d, _ptr(out)))
        return out

    def should_global_sort(self, *a):
        return self.L.ref_should_global_sort(*a)


class RefState:
    """A pic::ParticleSoA (+ optional pic::Gpma) living inside the reference."""

    def __init__(self, ref, g, s, q):
        self.ref, self.g, self.q = ref, g, q
        n = len(s["x"])
        ids = s.get("id")
        self.h = ref.L.ref_create(C.byref(g), n, *(_ptr(np.ascontiguousarray(s[k]))
                                                    for k in ("x", "y", "z", "vx", "vy", "vz", "w")),
                                  _ptr(None if ids is None else np.ascontiguousarray(ids, np.uint64)), q)
        self.n = n

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.L.ref_destroy(self.h)
            self.h = None

    def particles(self):
        out = {k: np.zeros(self.n) for k in ("x", "y", "z", "vx", "vy", "vz", "w")}
        out["id"] = np.zeros(self.n, np.uint64)
        self.ref.L.ref_get_particles(self.h, *(_ptr(out[k]) for k in ("x", "y", "z", "vx", "vy", "vz", "w", "id")))
        return out

    def deposit_scalar(self, order, use_gpma=False):
        jx, jy, jz = (np.zeros(self.g.ncells) for _ in range(3))
        self.ref._check(self.ref.L.ref_deposit_scalar(self.h, order, int(use_gpma), _ptr(jx), _ptr(jy), _ptr(jz)))
        return jx, jy, jz

    def deposit_scalar_mt(self, order, threads):
        jx, jy, jz = (np.zeros(self.g.ncells) for _ in range(3))
        self.ref._check(self.ref.L.ref_deposit_scalar_mt(self.h, order, threads, _ptr(jx), _ptr(jy), _ptr(jz)))
        return jx, jy, jz

    def deposit_density(self, order, quantity):
        rho = np.zeros(self.g.ncells)
        self.ref._check(self.ref.L.ref_deposit_density(self.h, order, _ptr(np.ascontiguousarray(quantity)), _ptr(rho)))
        return rho

    def deposit_tiled(self, order, use_gpma=False):
        jx, jy, jz = (np.zeros(self.g.ncells) for _ in range(3))
        self.ref._check(self.ref.L.ref_deposit_tiled(self.h, order, int(use_gpma), _ptr(jx), _ptr(jy), _ptr(jz)))
        return jx, jy, jz

    def deposit_tiled_opt(self, order, use_gpma=False, residency=True, dual_tile=False):
        jx, jy, jz = (np.zeros(self.g.ncells) for _ in range(3))
        m, e = C.c_uint64(), C.c_uint64()
        self.ref._check(self.ref.L.ref_deposit_tiled_opt(self.h, order, int(use_gpma), int(residency), int(dual_tile),
                                                         _ptr(jx), _ptr(jy), _ptr(jz), C.byref(m), C.byref(e)))
        return (jx, jy, jz), (m.value, e.value)

    def deposit_rhocell(self, order, use_gpma=False):
        jx, jy, jz = (np.zeros(self.g.ncells) for _ in range(3))
        self.ref._check(self.ref.L.ref_deposit_rhocell(self.h, order, int(use_gpma), _ptr(jx), _ptr(jy), _ptr(jz)))
        return jx, jy, jz

    def gpma_build(self, gap_ratio=0.25, min_gap=2):
        self.ref._check(self.ref.L.ref_gpma_build(self.h, gap_ratio, min_gap))

    def advance(self, dt):
        f = np.zeros(1)
        self.ref._check(self.ref.L.ref_advance(self.h, dt, _ptr(f)))
        return float(f[0])

    def incremental_sort(self):
        out = np.zeros(5, np.uint64)
        self.ref._check(self.ref.L.ref_incremental_sort(self.h, _ptr(out)))
        return dict(zip(("pending", "inserts", "shifted", "overflowed", "rebuilt"), (int(v) for v in out)))

    def step_timed(self, order, dt):
        """One baseline-incrsort step (simulation.hpp:117-136) timed per stage by
        the reference's pic::Timer: (advance_s, sort_s, deposit_s, movers, rebuilt)."""
        secs = np.zeros(3)
        out = np.zeros(2, np.uint64)
        self.ref._check(self.ref.L.ref_step_timed(self.h, order, dt, _ptr(secs), _ptr(out)))
        return float(secs[0]), float(secs[1]), float(secs[2]), int(out[0]), int(out[1])

    def density_timed(self, order):
        secs = np.zeros(1)
        self.ref._check(self.ref.L.ref_density_timed(self.h, order, _ptr(secs)))
        return float(secs[0])

    def bins(self):
        bin_of = np.zeros(self.n, np.uint32)
        bin_len = np.zeros(self.g.ncells, np.uint32)
        self.ref._check(self.ref.L.ref_bins(self.h, _ptr(bin_of), _ptr(bin_len)))
        return bin_of, bin_len

    def gpma_stats(self):
        out = np.zeros(4, np.uint64)
        r = np.zeros(1)
        self.ref.L.ref_gpma_stats(self.h, _ptr(out), _ptr(r))
        return dict(capacity=int(out[0]), num_particles=int(out[1]), num_empty=int(out[2]),
                    rebuild_count=int(out[3]), empty_ratio=float(r[0]))


def peak_rel_err(got, want):
    """Max per-node |diff| / component peak (proj/tests/test_pipeline.cpp:27-40)."""
    err = 0.0
    for a, b in zip(got, want):
        a = np.asarray(a)
        b = np.asarray(b)
        peak = float(np.max(np.abs(b))) if b.size else 0.0
        d = np.abs(a - b)
        if not np.any(d):
            continue
        if peak == 0.0:
            return float("inf")
        err = max(err, float(np.max(d)) / peak)
    return err
