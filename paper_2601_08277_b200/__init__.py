"""picgpu -- B200-native (sm_100a) MatrixPIC deposition + cell sorter.

Python mirror of the reference's `pic::` interface for the hot path, over the
C ABI in include/picgpu.h (ctypes; no torch types cross the boundary).  Names
and argument meaning follow the reference headers under proj/include/pic/:

    deposit_scalar(soa, grid, order)            deposit.hpp:62-73
    deposit_density(soa, grid, order, quantity) deposit.hpp:76-83
    deposit_tiled(soa, grid, order, opt, times) deposit.hpp:284-334 (DMMA tensor-core kernel)
    deposit_rhocell_vector(soa, grid, order)    deposit.hpp:87-119 (warp-DFMA kernel)
    counting_sort(soa, grid)                    gpma.hpp:379-394 (perm, starts, counts)
    gpma_build(soa, grid, cfg)                  gpma.hpp:379-402 (permutes soa in place)
    advance(soa, dt, grid)                      workload.hpp:139-155
    cell_of(pos, grid)                          grid.hpp:106-113
    should_global_sort(stats, policy)           sort_policy.hpp:62-73
    Session                                     run_simulation's step loop on a device-resident Gpma
    slab.SlabSession                            the same loop on one x-slab per rank (multi-GPU)

Errors raise the Python analogue of the reference's exception type.  The
product path has no CPU fallback: importing works anywhere, but every compute
call goes through libpicgpu.so and fails loudly without a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PICGPU_LIB", os.path.join(_HERE, "libpicgpu.so"))

CIC, TSC, QSP = 1, 2, 3

OK, EINVAL, ERANGE, ELENGTH, ELOGIC, EDOMAIN, ECUDA, ENCCL, ENOMEM = range(9)

STEP_PUSH, STEP_SORT, STEP_CURRENT, STEP_DENSITY, STEP_GLOBAL_SORT, STEP_NO_SYNC, STEP_RESORT = 1, 2, 4, 8, 16, 32, 64
STEP_UNFUSED = 128  # run push, sort and J as separate kernels (default: one fused push + detect + J pass)
KERNEL_LANE, KERNEL_VECTOR, KERNEL_MATRIX = 0, 1, 2
STEP_DEFAULT = STEP_PUSH | STEP_SORT | STEP_CURRENT
SESSION_TIMING = 1
PHASES = ("push_sort", "reserved", "rebuild_or_global_sort", "deposit_current", "deposit_density", "zero_fields")


class PicError(RuntimeError):
    code = -1


class InvalidArgument(PicError, ValueError):  # std::invalid_argument
    code = EINVAL


class OutOfRange(PicError, IndexError):  # std::out_of_range
    code = ERANGE


class LengthError(PicError, ValueError):  # std::length_error
    code = ELENGTH


class LogicError(PicError):  # std::logic_error
    code = ELOGIC


class DomainError(PicError, ArithmeticError):  # std::domain_error
    code = EDOMAIN


class CudaError(PicError):
    code = ECUDA


class NcclError(PicError):
    code = ENCCL


class DeviceOutOfMemory(PicError, MemoryError):
    code = ENOMEM


_ERRORS = {c.code: c for c in (InvalidArgument, OutOfRange, LengthError, LogicError, DomainError, CudaError,
                                NcclError, DeviceOutOfMemory)}


class Grid(C.Structure):
    """picgpu_grid == pic::GridSpec (grid.hpp:26-72), periodic on every axis."""

    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("pad_", C.c_int32),
                ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double),
                ("ox", C.c_double), ("oy", C.c_double), ("oz", C.c_double)]

    @classmethod
    def make(cls, nx, ny=None, nz=None, dx=1.0, dy=1.0, dz=1.0, origin=(0.0, 0.0, 0.0)):
        ny = nx if ny is None else ny
        nz = nx if nz is None else nz
        return cls(nx, ny, nz, 0, dx, dy, dz, *origin)

    @property
    def ncells(self) -> int:
        return self.nx * self.ny * self.nz

    def linear_id(self, i, j, k):  # grid.hpp:50-54
        return i + self.nx * (j + self.ny * k)


GridSpec = Grid


class StepStats(C.Structure):
    _fields_ = [("moved", C.c_uint64), ("inserts", C.c_uint64), ("overflowed", C.c_uint64),
                ("rebuilt", C.c_uint32), ("global_sorted", C.c_uint32), ("empty_slot_ratio", C.c_double),
                ("capacity", C.c_uint64), ("num_particles", C.c_uint64), ("fused", C.c_uint32),
                ("reserved_", C.c_uint32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class SessionConfig(C.Structure):
    _fields_ = [("order", C.c_int32), ("device", C.c_int32), ("gap_ratio", C.c_double), ("min_gap", C.c_uint32),
                ("flags", C.c_uint32)]


class StageTimes(C.Structure):
    """pic::StageTimes (deposit.hpp:126-130), seconds."""

    _fields_ = [("preproc", C.c_double), ("compute", C.c_double), ("reduce", C.c_double)]


class KernelCounters(C.Structure):
    """pic::KernelCounters (deposit.hpp:121-124)."""

    _fields_ = [("mopa_calls", C.c_uint64), ("extract_passes", C.c_uint64)]


@dataclass
class TiledOptions:
    """pic::TiledOptions (deposit.hpp:179-184); gpma: stream bin by bin."""

    gpma: bool = False
    residency: bool = True
    dual_tile: bool = False
    counters: KernelCounters | None = None

    def flags(self) -> int:
        return (1 if self.gpma else 0) | (2 if self.residency else 0) | (4 if self.dual_tile else 0)


class WorkloadConfig(C.Structure):
    """picgpu_workload == pic::WorkloadConfig (workload.hpp:16-44)."""

    _fields_ = [("grid", Grid), ("ppc", C.c_int32), ("kind", C.c_int32), ("thermal_speed", C.c_double),
                ("drift", C.c_double * 3), ("seed", C.c_uint64), ("steps", C.c_int32), ("order", C.c_int32),
                ("dt", C.c_double), ("charge", C.c_double)]

    UNIFORM_PLASMA, DRIFT_GRADIENT = 0, 1

    @classmethod
    def make(cls, grid, ppc=8, kind=0, thermal_speed=0.01, drift=(0.0, 0.0, 0.0), seed=1, steps=10, dt=1.0,
             charge=1.0, order=1):
        return cls(grid, ppc, kind, thermal_speed, (C.c_double * 3)(*drift), seed, steps, order, dt, charge)

    def speed_cap(self):
        return min(self.grid.dx, self.grid.dy, self.grid.dz) / self.dt


class LwfaConfig(C.Structure):
    """picgpu_lwfa: the SURVEY 8(d) C4 population (density ramp + relativistic beam)."""

    _fields_ = [("ppc", C.c_int32), ("ramp_start", C.c_int32), ("ramp_len", C.c_int32), ("pad_", C.c_int32),
                ("u_th", C.c_double), ("beam_fraction", C.c_double), ("ux_min", C.c_double), ("ux_max", C.c_double),
                ("beam_x0", C.c_double), ("beam_x1", C.c_double), ("seed", C.c_uint64)]

    @classmethod
    def make(cls, ppc=8, ramp_start=64, ramp_len=64, u_th=0.01, beam_fraction=0.1, ux=(5.0, 50.0),
             beam_x=(128.0, 160.0), seed=1):
        return cls(ppc, ramp_start, ramp_len, 0, u_th, beam_fraction, ux[0], ux[1], beam_x[0], beam_x[1], seed)


class SortPolicy(C.Structure):
    """pic::SortPolicy (sort_policy.hpp:12-30); defaults are Table 4's."""

    _fields_ = [("sort_interval", C.c_uint32), ("min_sort_interval", C.c_uint32),
                ("trigger_rebuild_count", C.c_uint32), ("perf_enable", C.c_uint32),
                ("trigger_empty_ratio", C.c_double), ("trigger_full_ratio", C.c_double),
                ("perf_degrad", C.c_double)]

    @classmethod
    def defaults(cls, **kw):
        p = cls()
        lib().picgpu_sort_policy_defaults(C.byref(p))
        for k, v in kw.items():
            setattr(p, k, v)
        return p


class RankSortStats(C.Structure):
    """pic::RankSortStats (sort_policy.hpp:35-44)."""

    _fields_ = [("steps_since_sort", C.c_uint32), ("pad_", C.c_uint32), ("cumulative_local_rebuilds", C.c_uint64),
                ("empty_slot_ratio", C.c_double), ("perf_metric", C.c_double), ("baseline_perf", C.c_double),
                ("total_inserts", C.c_uint64), ("total_shifts", C.c_uint64)]


SORT_REASONS = ("none", "interval", "rebuilds", "slot_ratio", "perf_degradation")

_lib = None
_P = C.c_void_p
_D = C.c_double
_U64 = C.c_uint64


def lib():
    """Load libpicgpu.so (the sm_100a build); there is no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    G = C.POINTER(Grid)
    L.picgpu_last_error.restype = C.c_char_p
    L.picgpu_kernel_launches.restype = _U64
    L.picgpu_deposit_current.argtypes = [G, C.c_int] + [_P] * 7 + [_D, _U64, _P, _P, _P]
    L.picgpu_deposit_current_dev.argtypes = [G, C.c_int] + [_P] * 7 + [_D, _U64, _P, _P, _P, _P]
    L.picgpu_session_set_adaptive_slack.argtypes = [_P, C.c_int]
    L.picgpu_comm_unique_id.argtypes = [_P]
    L.picgpu_comm_init.argtypes = [_P, C.c_int, C.c_int, C.c_int, _P]
    L.picgpu_comm_wrap.argtypes = [_P, C.c_int, _P]
    L.picgpu_comm_rank.argtypes = [_P, _P, _P]
    L.picgpu_comm_destroy.argtypes = [_P]
    L.picgpu_session_set_comm.argtypes = [_P, _P, C.c_uint32]
    L.picgpu_session_slab_step.argtypes = [_P, _D, C.c_uint32, _P]
    L.picgpu_deposit_current_esirkepov.argtypes = [G, C.c_int] + [_P] * 7 + [_D, _D, _U64, _P, _P, _P]
    L.picgpu_deposit_current_esirkepov_dev.argtypes = [G, C.c_int] + [_P] * 7 + [_D, _D, _U64, _P, _P, _P, _P]
    L.picgpu_deposit_density.argtypes = [G, C.c_int, _P, _P, _P, _P, _U64, _P]
    L.picgpu_counting_sort.argtypes = [G, _P, _P, _P, _U64, _P, _P, _P]
    L.picgpu_advance.argtypes = [G, _D, _P, _P, _P, _P, _P, _P, _U64, _P]
    L.picgpu_cell_of.argtypes = [G, _P, _P, _P, _U64, _P]
    L.picgpu_sort_policy_defaults.argtypes = [C.POINTER(SortPolicy)]
    L.picgpu_sort_policy_defaults.restype = None
    L.picgpu_should_global_sort.argtypes = [C.POINTER(RankSortStats), C.POINTER(SortPolicy)]
    L.picgpu_session_create.argtypes = [G, C.POINTER(SessionConfig), C.POINTER(_P)]
    L.picgpu_session_destroy.argtypes = [_P]
    L.picgpu_session_upload.argtypes = [_P, _U64] + [_P] * 8 + [_D]
    L.picgpu_session_generate_plasma.argtypes = [_P, C.c_int, _D, _U64]
    L.picgpu_session_step.argtypes = [_P, _D, C.c_uint32, C.POINTER(StepStats)]
    L.picgpu_session_global_sort.argtypes = [_P]
    L.picgpu_session_synchronize.argtypes = [_P]
    L.picgpu_session_num_particles.argtypes = [_P]
    L.picgpu_session_num_particles.restype = _U64
    L.picgpu_session_capacity.argtypes = [_P]
    L.picgpu_session_capacity.restype = _U64
    L.picgpu_session_stream.argtypes = [_P]
    L.picgpu_session_stream.restype = _P
    L.picgpu_session_download_particles.argtypes = [_P] * 9
    L.picgpu_session_download_bins.argtypes = [_P, _P, _P]
    L.picgpu_session_download_current.argtypes = [_P, _P, _P, _P]
    L.picgpu_session_download_density.argtypes = [_P, _P]
    L.picgpu_session_device_fields.argtypes = [_P, C.POINTER(_P), C.POINTER(_P)]
    L.picgpu_session_phase_times.argtypes = [_P, _P, _P, C.c_int]
    L.picgpu_session_reset_phase_times.argtypes = [_P]
    L.picgpu_fp64_peak.argtypes = [C.c_int, C.POINTER(_D)]
    L.picgpu_deposit_tiled.argtypes = [G, C.c_int] + [_P] * 7 + [_D, _U64, C.c_uint32, _P, _P, _P,
                                                                C.POINTER(StageTimes), C.POINTER(KernelCounters)]
    L.picgpu_deposit_rhocell_vector.argtypes = [G, C.c_int] + [_P] * 7 + [_D, _U64, C.c_int, _P, _P, _P,
                                                                         C.POINTER(_D)]
    L.picgpu_session_set_kernel.argtypes = [_P, C.c_int]
    L.picgpu_session_set_fusion.argtypes = [_P, C.c_double]
    L.picgpu_session_generate_lwfa.argtypes = [_P, C.POINTER(LwfaConfig)]
    L.picgpu_session_shift_window.argtypes = [_P, C.c_int, _D, _U64, _U64, C.POINTER(_U64), C.POINTER(_U64)]
    L.picgpu_session_grid.argtypes = [_P, G]
    L.picgpu_session_make_workload.argtypes = [_P, C.POINTER(WorkloadConfig)]
    L.picgpu_slab_grid.argtypes = [G, C.c_int, C.c_int, C.c_int, G]
    L.picgpu_session_set_slab.argtypes = [_P, G, C.c_int, C.c_int, C.c_int]
    L.picgpu_session_step_begin.argtypes = [_P, _D, C.c_uint32, C.POINTER(_U64), C.POINTER(_U64)]
    L.picgpu_session_copy_leavers.argtypes = [_P, _P, _P]
    L.picgpu_session_step_end.argtypes = [_P, _P, _U64, C.POINTER(StepStats)]
    L.picgpu_session_guard_planes.argtypes = [_P, C.c_int, _P, _P]
    L.picgpu_session_add_guard_planes.argtypes = [_P, C.c_int, _P, _P]
    _lib = L
    return L


def _check(rc):
    if rc:
        msg = lib().picgpu_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, PicError)(msg)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def kernel_launches() -> int:
    return int(lib().picgpu_kernel_launches())


def flop_count(order: int) -> int:
    """deposit.hpp:336-345 tally (76 / 534), 238 for this project's TSC."""
    return lib().picgpu_flop_count(order)


@dataclass
class ParticleSoA:
    """pic::ParticleSoA (particles.hpp:14-19)."""

    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    vx: np.ndarray
    vy: np.ndarray
    vz: np.ndarray
    w: np.ndarray
    id: np.ndarray = None
    q: float = 1.0

    def __post_init__(self):
        for k in ("x", "y", "z", "vx", "vy", "vz", "w"):
            setattr(self, k, np.array(getattr(self, k), dtype=np.float64, copy=True))
        if self.id is None:
            self.id = np.arange(len(self.x), dtype=np.uint64)
        self.id = np.array(self.id, dtype=np.uint64, copy=True)

    @classmethod
    def from_dict(cls, d, q=None):
        return cls(d["x"], d["y"], d["z"], d["vx"], d["vy"], d["vz"], d["w"], d.get("id"),
                   d.get("q", 1.0) if q is None else q)

    def size(self):
        return len(self.x)

    def apply_permutation(self, perm):  # particles.hpp:34-47
        for k in ("x", "y", "z", "vx", "vy", "vz", "w", "id"):
            setattr(self, k, np.ascontiguousarray(getattr(self, k)[perm]))


@dataclass
class CurrentGrid:
    """pic::CurrentGrid (grid.hpp:127-150)."""

    spec: Grid
    jx: np.ndarray
    jy: np.ndarray
    jz: np.ndarray

    def component(self, c):
        return (self.jx, self.jy, self.jz)[c]

    def component_sums(self):
        return [float(np.sum(a)) for a in (self.jx, self.jy, self.jz)]


def _soa(soa, q=None):
    if isinstance(soa, ParticleSoA):
        return soa
    return ParticleSoA.from_dict(soa, q)


def deposit_esirkepov(old, new, w, grid: Grid, order: int, q: float, dt: float) -> CurrentGrid:
    """Charge-conserving J on the Yee faces (picgpu_deposit_current_esirkepov):
    an extension with no reference counterpart (see include/picgpu.h)."""
    n = len(w)
    a = [_f64(old[k]) for k in ("x", "y", "z")] + [_f64(new[k]) for k in ("x", "y", "z")] + [_f64(w)]
    nc = grid.ncells
    jx, jy, jz = np.empty(nc), np.empty(nc), np.empty(nc)
    _check(lib().picgpu_deposit_current_esirkepov(C.byref(grid), order, *(_ptr(v) for v in a), q, dt, n, _ptr(jx),
                                                  _ptr(jy), _ptr(jz)))
    return CurrentGrid(grid, jx, jy, jz)


def deposit_scalar(soa, grid: Grid, order: int, q: float | None = None) -> CurrentGrid:
    """Current deposition at order 1/2/3 (deposit_scalar, deposit.hpp:62-73)."""
    s = _soa(soa, q)
    qq = s.q if q is None else q
    nc = grid.ncells
    jx, jy, jz = np.empty(nc), np.empty(nc), np.empty(nc)
    _check(lib().picgpu_deposit_current(C.byref(grid), order, _ptr(s.x), _ptr(s.y), _ptr(s.z), _ptr(s.vx),
                                        _ptr(s.vy), _ptr(s.vz), _ptr(s.w), qq, s.size(), _ptr(jx), _ptr(jy),
                                        _ptr(jz)))
    return CurrentGrid(grid, jx, jy, jz)


def deposit_tiled(soa, grid: Grid, order: int, opt: TiledOptions | None = None, times: StageTimes | None = None,
                  q: float | None = None) -> CurrentGrid:
    """deposit_tiled (deposit.hpp:284-334): same J, on the FP64 tensor-core (DMMA)
    kernel; opt.counters gets the reference tile engine's counts for this input."""
    s = _soa(soa, q)
    opt = opt or TiledOptions()
    nc = grid.ncells
    jx, jy, jz = np.empty(nc), np.empty(nc), np.empty(nc)
    kc = KernelCounters()
    _check(lib().picgpu_deposit_tiled(C.byref(grid), order, _ptr(s.x), _ptr(s.y), _ptr(s.z), _ptr(s.vx), _ptr(s.vy),
                                      _ptr(s.vz), _ptr(s.w), s.q if q is None else q, s.size(), opt.flags(),
                                      _ptr(jx), _ptr(jy), _ptr(jz), C.byref(times) if times is not None else None,
                                      C.byref(kc) if opt.counters is not None else None))
    if opt.counters is not None:  # the reference increments its counters
        opt.counters.mopa_calls += kc.mopa_calls
        opt.counters.extract_passes += kc.extract_passes
    return CurrentGrid(grid, jx, jy, jz)


def deposit_rhocell_vector(soa, grid: Grid, order: int, gpma: bool = False, q: float | None = None) -> CurrentGrid:
    """deposit_rhocell_vector (deposit.hpp:87-119): same J, on the warp-DFMA kernel."""
    s = _soa(soa, q)
    nc = grid.ncells
    jx, jy, jz = np.empty(nc), np.empty(nc), np.empty(nc)
    red = C.c_double(-1.0)
    _check(lib().picgpu_deposit_rhocell_vector(C.byref(grid), order, _ptr(s.x), _ptr(s.y), _ptr(s.z), _ptr(s.vx),
                                               _ptr(s.vy), _ptr(s.vz), _ptr(s.w), s.q if q is None else q, s.size(),
                                               int(gpma), _ptr(jx), _ptr(jy), _ptr(jz), C.byref(red)))
    return CurrentGrid(grid, jx, jy, jz)


def deposit_density(soa, grid: Grid, order: int, quantity) -> np.ndarray:
    """One-component deposition in storage order, bit-identical (deposit.hpp:76-83)."""
    s = _soa(soa)
    qv = _f64(quantity)
    if len(qv) != s.size():
        raise InvalidArgument("deposit_density: quantity length mismatch")
    rho = np.empty(grid.ncells)
    _check(lib().picgpu_deposit_density(C.byref(grid), order, _ptr(s.x), _ptr(s.y), _ptr(s.z), _ptr(qv),
                                        s.size(), _ptr(rho)))
    return rho


def counting_sort(soa, grid: Grid):
    """Stable counting sort by cell: (perm, starts, counts), perm == gpma_build's."""
    s = _soa(soa)
    n = s.size()
    perm = np.empty(n, np.uint32)
    starts = np.empty(grid.ncells, np.uint32)
    counts = np.empty(grid.ncells, np.uint32)
    _check(lib().picgpu_counting_sort(C.byref(grid), _ptr(s.x), _ptr(s.y), _ptr(s.z), n, _ptr(perm),
                                      _ptr(starts), _ptr(counts)))
    return perm, starts, counts


def gpma_build(soa: ParticleSoA, grid: Grid):
    """gpma_build's physical stable sort of the store (gpma.hpp:379-395).
    Returns (starts, counts) of the packed bins; the store is permuted in place."""
    perm, starts, counts = counting_sort(soa, grid)
    soa.apply_permutation(perm)
    return starts, counts


def advance(soa: ParticleSoA, dt: float, grid: Grid) -> float:
    """Ballistic push with periodic wrap, in place; returns the moved fraction."""
    n = soa.size()
    moved = np.zeros(1, np.uint64)
    _check(lib().picgpu_advance(C.byref(grid), dt, _ptr(soa.x), _ptr(soa.y), _ptr(soa.z), _ptr(soa.vx),
                                _ptr(soa.vy), _ptr(soa.vz), n, _ptr(moved)))
    return float(moved[0]) / n if n else 0.0


def cells(soa, grid: Grid) -> np.ndarray:
    s = _soa(soa)
    out = np.empty(s.size(), np.uint32)
    _check(lib().picgpu_cell_of(C.byref(grid), _ptr(s.x), _ptr(s.y), _ptr(s.z), s.size(), _ptr(out)))
    return out


def cell_of(pos, grid: Grid) -> int:
    x, y, z = (np.array([v], np.float64) for v in pos)
    out = np.empty(1, np.uint32)
    _check(lib().picgpu_cell_of(C.byref(grid), _ptr(x), _ptr(y), _ptr(z), 1, _ptr(out)))
    return int(out[0])


def should_global_sort(stats: RankSortStats, policy: SortPolicy | None = None) -> str:
    policy = policy or SortPolicy.defaults()
    return SORT_REASONS[lib().picgpu_should_global_sort(C.byref(stats), C.byref(policy))]


def fp64_peak_tflops(device: int = 0) -> float:
    out = C.c_double(0.0)
    _check(lib().picgpu_fp64_peak(device, C.byref(out)))
    return out.value


class Session:
    """Device-resident particles in cell bins with slack + deposition fields.

    One step = [advance] -> [incremental sort] -> [deposit J] -> [deposit rho]
    -> [global sort], the reference's run_simulation order (simulation.hpp:92-176).
    """

    def __init__(self, grid: Grid, order: int = QSP, gap_ratio: float = 0.25, min_gap: int = 2, device: int = 0,
                 timing: bool = False):
        self.grid = grid
        self.order = order
        cfg = SessionConfig(order, device, gap_ratio, min_gap, SESSION_TIMING if timing else 0)
        h = _P()
        _check(lib().picgpu_session_create(C.byref(grid), C.byref(cfg), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().picgpu_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def upload(self, soa, q=None):
        s = _soa(soa, q)
        _check(lib().picgpu_session_upload(self._h, s.size(), _ptr(s.x), _ptr(s.y), _ptr(s.z), _ptr(s.vx),
                                           _ptr(s.vy), _ptr(s.vz), _ptr(s.w), _ptr(s.id),
                                           s.q if q is None else q))

    def generate_plasma(self, ppc: int, u_th: float, seed: int = 1):
        _check(lib().picgpu_session_generate_plasma(self._h, ppc, u_th, seed))

    def shift_window(self, ppc: int, u_th: float, seed: int, pid0: int):
        """C4 moving window: origin += dx, drop x-column 0, inject a fresh last
        column (ids pid0..).  Returns (dropped, injected); self.grid follows."""
        d, i = C.c_uint64(), C.c_uint64()
        _check(lib().picgpu_session_shift_window(self._h, ppc, u_th, seed, pid0, C.byref(d), C.byref(i)))
        g = Grid()
        lib().picgpu_session_grid(self._h, C.byref(g))
        self.grid = g
        return int(d.value), int(i.value)

    def generate_lwfa(self, cfg: "LwfaConfig"):
        """SURVEY 8(d) C4 population (density ramp + relativistic beam), generated in HBM."""
        _check(lib().picgpu_session_generate_lwfa(self._h, C.byref(cfg)))

    def step(self, dt: float = 0.5, flags: int = STEP_DEFAULT) -> dict:
        st = StepStats()
        _check(lib().picgpu_session_step(self._h, dt, flags, C.byref(st)))
        return st.as_dict()

    def global_sort(self):
        _check(lib().picgpu_session_global_sort(self._h))

    def synchronize(self):
        _check(lib().picgpu_session_synchronize(self._h))

    @property
    def num_particles(self) -> int:
        return int(lib().picgpu_session_num_particles(self._h))

    @property
    def capacity(self) -> int:
        return int(lib().picgpu_session_capacity(self._h))

    @property
    def stream(self) -> int:
        return int(lib().picgpu_session_stream(self._h) or 0)

    def particles(self) -> ParticleSoA:
        n = self.num_particles
        a = {k: np.empty(n) for k in ("x", "y", "z", "vx", "vy", "vz", "w")}
        ids = np.empty(n, np.uint64)
        _check(lib().picgpu_session_download_particles(self._h, *(_ptr(a[k]) for k in
                                                                  ("x", "y", "z", "vx", "vy", "vz", "w")),
                                                       _ptr(ids)))
        return ParticleSoA(id=ids, **a)

    def bins(self):
        off = np.empty(self.grid.ncells + 1, np.uint32)
        cnt = np.empty(self.grid.ncells, np.uint32)
        _check(lib().picgpu_session_download_bins(self._h, _ptr(off), _ptr(cnt)))
        return off, cnt

    def current(self) -> CurrentGrid:
        nc = self.grid.ncells
        jx, jy, jz = np.empty(nc), np.empty(nc), np.empty(nc)
        _check(lib().picgpu_session_download_current(self._h, _ptr(jx), _ptr(jy), _ptr(jz)))
        return CurrentGrid(self.grid, jx, jy, jz)

    def density(self) -> np.ndarray:
        rho = np.empty(self.grid.ncells)
        _check(lib().picgpu_session_download_density(self._h, _ptr(rho)))
        return rho

    def device_fields(self):
        j, r = _P(), _P()
        lib().picgpu_session_device_fields(self._h, C.byref(j), C.byref(r))
        return j.value, r.value

    def set_kernel(self, family: int):
        """J kernel family: KERNEL_LANE (default), KERNEL_VECTOR (warp DFMA), KERNEL_MATRIX (DMMA)."""
        _check(lib().picgpu_session_set_kernel(self._h, family))

    def set_adaptive_slack(self, enable: bool = True):
        """picgpu_session_set_adaptive_slack: rebuild storms widen later layouts' gap ratio."""
        _check(lib().picgpu_session_set_adaptive_slack(self._h, int(enable)))

    def set_fusion(self, max_moved_fraction: float):
        """Fuse push + detect + J while the previous step moved less than this
        fraction of the particles (default 0.06; 0 never, > 1 always)."""
        _check(lib().picgpu_session_set_fusion(self._h, max_moved_fraction))

    def make_workload(self, cfg: WorkloadConfig):
        """Replace the particles by make_workload(cfg) generated on the device."""
        _check(lib().picgpu_session_make_workload(self._h, C.byref(cfg)))

    def phase_times(self):
        ms = np.zeros(len(PHASES))
        launches = np.zeros(len(PHASES), np.uint64)
        lib().picgpu_session_phase_times(self._h, _ptr(ms), _ptr(launches), len(PHASES))
        return {p: (float(m), int(l)) for p, m, l in zip(PHASES, ms, launches)}

    def reset_phase_times(self):
        lib().picgpu_session_reset_phase_times(self._h)


# ---- the reference's harness loop (simulation.hpp:19-176) ----------------------

MODES = ("baseline", "matrix-only", "hybrid-nosort", "hybrid-globalsort", "fullopt", "rhocell-vector",
         "baseline-incrsort", "rhocell-incrsort")


def mode_uses_gpma(mode: str) -> bool:
    return mode in ("hybrid-globalsort", "fullopt", "baseline-incrsort", "rhocell-incrsort")


def mode_incremental_sort(mode: str) -> bool:
    return mode in ("fullopt", "baseline-incrsort", "rhocell-incrsort")


def mode_kernel_family(mode: str) -> int:
    """Scalar modes -> lane DFMA kernel, rhocell modes -> warp DFMA, tile-engine modes -> DMMA."""
    if mode in ("baseline", "baseline-incrsort"):
        return KERNEL_LANE
    if mode in ("rhocell-vector", "rhocell-incrsort"):
        return KERNEL_VECTOR
    return KERNEL_MATRIX


@dataclass
class StepMetrics:  # simulation.hpp:67-78
    step: int
    wall_s: float = 0.0
    preproc_s: float = 0.0
    compute_s: float = 0.0
    sort_s: float = 0.0
    reduce_s: float = 0.0
    particles_per_second: float = 0.0
    fraction_moved: float = 0.0
    rebuilds: int = 0
    global_sort: str = "none"


@dataclass
class RunResult:  # simulation.hpp:80-86
    steps: list
    checksum: list
    final_grid: CurrentGrid
    particles: ParticleSoA
    stats: RankSortStats


def validate_policy(p: SortPolicy):  # sort_policy.hpp:20-28
    if p.min_sort_interval > p.sort_interval:
        raise InvalidArgument("policy: min_sort_interval exceeds sort_interval")
    if not (0.0 < p.trigger_empty_ratio < 1.0 and 0.0 < p.trigger_full_ratio < 1.0):
        raise InvalidArgument("policy: slot-ratio triggers must lie in (0,1)")
    if not (0.0 < p.perf_degrad <= 1.0):
        raise InvalidArgument("policy: perf_degrad must lie in (0,1]")


def run_simulation(cfg: WorkloadConfig, mode: str, policy: SortPolicy | None = None, gap_ratio: float = 0.25,
                   min_gap: int = 2, device: int = 0, initial=None) -> RunResult:
    """run_simulation (simulation.hpp:92-176) on one GPU.

    Per step: advance fused with the mode's sort (incremental for *-incrsort and
    fullopt, a full stable counting sort of the store otherwise: the GPU kernels
    always read bins), J with the mode's kernel family, metrics from device
    event times (sort_s includes the fused push; preproc_s and reduce_s are 0),
    then fullopt's adaptive global-resort decision.  `initial` (a ParticleSoA
    or dict) replaces make_workload, e.g. the reference's own population.
    """
    import time

    if mode not in MODES:
        raise InvalidArgument(f"unknown mode: {mode}")
    policy = policy or SortPolicy.defaults()
    validate_policy(policy)
    sess = Session(cfg.grid, cfg.order, gap_ratio, min_gap, device, timing=True)
    try:
        sess.set_kernel(mode_kernel_family(mode))
        if initial is not None:
            sess.upload(initial, q=cfg.charge)
        else:
            sess.make_workload(cfg)
        n = sess.num_particles
        flags = STEP_PUSH | STEP_CURRENT | (STEP_SORT if mode_incremental_sort(mode) else STEP_RESORT)
        stats = RankSortStats()
        prev = sess.phase_times()
        steps = []
        for step in range(cfg.steps):
            t0 = time.perf_counter()
            st = sess.step(cfg.dt, flags)
            ph = sess.phase_times()
            m = StepMetrics(step)
            m.sort_s = (ph["push_sort"][0] - prev["push_sort"][0] + ph["rebuild_or_global_sort"][0]
                        - prev["rebuild_or_global_sort"][0]) * 1e-3
            m.compute_s = (ph["deposit_current"][0] - prev["deposit_current"][0] + ph["zero_fields"][0]
                           - prev["zero_fields"][0]) * 1e-3
            prev = ph
            m.fraction_moved = st["moved"] / n if n else 0.0
            m.rebuilds = int(st["rebuilt"])
            stats.total_inserts += st["inserts"]
            m.particles_per_second = n / max(m.preproc_s + m.compute_s + m.sort_s + m.reduce_s, 1e-12)
            stats.perf_metric = m.particles_per_second
            stats.steps_since_sort += 1
            stats.cumulative_local_rebuilds += m.rebuilds
            if mode_uses_gpma(mode):
                stats.empty_slot_ratio = st["empty_slot_ratio"]
            if mode == "fullopt":
                if stats.baseline_perf == 0.0:
                    stats.baseline_perf = m.particles_per_second
                reason = should_global_sort(stats, policy)
                if reason != "none":
                    sess.step(cfg.dt, STEP_GLOBAL_SORT)  # global_sort, timed
                    ph = sess.phase_times()
                    m.sort_s += (ph["rebuild_or_global_sort"][0] - prev["rebuild_or_global_sort"][0]) * 1e-3
                    prev = ph
                    stats.steps_since_sort = 0  # reset_counters, sort_policy.hpp:75-79
                    stats.cumulative_local_rebuilds = 0
                    stats.baseline_perf = 0.0
                    m.global_sort = reason
            m.wall_s = time.perf_counter() - t0
            steps.append(m)
        grid = sess.current()
        return RunResult(steps, grid.component_sums(), grid, sess.particles(), stats)
    finally:
        sess.close()
