"""x-slab decomposition of the periodic box over ranks.

The reference runs one single-threaded process over the whole box
(run_simulation, proj/include/pic/simulation.hpp:92-176; its concurrency model
only allows distinct Gpma tiles to be processed concurrently, and
it has no domain decomposition).  Here one process drives one GPU and
owns the global x-cells [x0, x1) (`slab_range`, a balanced contiguous split;
SURVEY.md 8(e)); the slab's session grid is the owned cells plus `ghost` guard
cells on each side.  One step:

    begin        push + move detection; particles that left the slab are
                 packed as 8-double records (x y z vx vy vz w id-bits)
    exchange     records to the left / right rank on the periodic ring
    end          arrivals inserted like movers (slack, borrow, rebuild),
                 then J (and rho) deposited on the slab grid
    exchange     guard planes: the low ghost planes go left, the high ones
                 right, and are added into the neighbour's owned edge planes

Positions stay in global coordinates and wrap on the global box, so every
per-particle value (cell, weights, pushed position) is bit-identical to the
undecomposed run; only the summation order of J across a seam differs
(J agrees to the 1e-12 peak-normalised tolerance, rho to 1e-13).

torch is plumbing here: device buffers for the exchanges and
torch.distributed (NCCL on GPUs, gloo on CPU) for the send/recv.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import STEP_CURRENT, STEP_DEFAULT, STEP_DENSITY, Grid, ParticleSoA, Session, StepStats, _check, cells, lib

GHOST = 2  # QSP reach: nodes cell-1 .. cell+2
RECORD = 8  # doubles per exchanged particle


def slab_range(nx: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split of nx x-cells over `world` ranks."""
    base, rem = divmod(nx, world)
    x0 = rank * base + min(rank, rem)
    return x0, x0 + base + (1 if rank < rem else 0)


def slab_grid(grid: Grid, x0: int, x1: int, ghost: int = GHOST) -> Grid:
    out = Grid()
    _check(lib().picgpu_slab_grid(C.byref(grid), x0, x1, ghost, C.byref(out)))
    return out


def _torch():
    import torch

    return torch


class SlabSession(Session):
    """A Session on the slab [x0, x1) of `global_grid` (picgpu_session_set_slab)."""

    def __init__(self, global_grid: Grid, x0: int, x1: int, order: int = 3, ghost: int = GHOST, gap_ratio=0.25,
                 min_gap=2, device: int = 0, timing: bool = False):
        self.global_grid = global_grid
        self.x0, self.x1, self.ghost = x0, x1, ghost
        self.own = x1 - x0
        self.device = device
        super().__init__(slab_grid(global_grid, x0, x1, ghost), order, gap_ratio, min_gap, device, timing)
        _check(lib().picgpu_session_set_slab(self._h, C.byref(global_grid), x0, x1, ghost))
        g = self.grid
        self.plane_doubles = ghost * g.ny * g.nz
        self._flags = 0

    # ---- population --------------------------------------------------------
    def owned_mask(self, soa) -> np.ndarray:
        """Particles whose global cell lies in [x0, x1) (global cell_of)."""
        i = cells(soa, self.global_grid) % np.uint32(self.global_grid.nx)
        return (i >= self.x0) & (i < self.x1)

    def upload_owned(self, soa, q=None):
        m = self.owned_mask(soa)
        sub = {k: getattr(soa, k)[m] for k in ("x", "y", "z", "vx", "vy", "vz", "w", "id")}
        self.upload(ParticleSoA(**sub, q=soa.q if q is None else q), q)

    # ---- the step protocol ------------------------------------------------
    def begin(self, dt: float, flags: int = STEP_DEFAULT) -> tuple[int, int]:
        nl, nr = C.c_uint64(0), C.c_uint64(0)
        _check(lib().picgpu_session_step_begin(self._h, dt, flags, C.byref(nl), C.byref(nr)))
        self._flags = flags
        return int(nl.value), int(nr.value)

    def leavers(self, counts: tuple[int, int]):
        """(to_left, to_right) record tensors [n, 8] float64 on this GPU."""
        torch = _torch()
        dev = torch.device("cuda", self.device)
        _sync(self.device)  # the buffers below must not be in flight on torch's stream
        tl = torch.empty((counts[0], RECORD), dtype=torch.float64, device=dev)
        tr = torch.empty((counts[1], RECORD), dtype=torch.float64, device=dev)
        _check(lib().picgpu_session_copy_leavers(self._h, tl.data_ptr() if counts[0] else None,
                                                 tr.data_ptr() if counts[1] else None))
        return tl, tr

    def end(self, arrivals) -> dict:
        """arrivals: [n, 8] float64 device tensor (or None); complete when passed."""
        st = StepStats()
        n = 0 if arrivals is None else int(arrivals.shape[0])
        ptr = arrivals.contiguous().data_ptr() if n else None
        _check(lib().picgpu_session_step_end(self._h, ptr, n, C.byref(st)))
        return st.as_dict()

    def guard_planes(self, field: int = 0):
        torch = _torch()
        comps = 3 if field == 0 else 1
        dev = torch.device("cuda", self.device)
        lo = torch.empty(comps * self.plane_doubles, dtype=torch.float64, device=dev)
        hi = torch.empty_like(lo)
        _sync(self.device)
        _check(lib().picgpu_session_guard_planes(self._h, field, lo.data_ptr(), hi.data_ptr()))
        return lo, hi

    def add_guard_planes(self, field: int, from_left, from_right):
        _check(lib().picgpu_session_add_guard_planes(self._h, field, from_left.contiguous().data_ptr(),
                                                     from_right.contiguous().data_ptr()))

    # ---- owned views ----------------------------------------------------------
    def _owned(self, a: np.ndarray) -> np.ndarray:
        g = self.grid
        return a.reshape(g.nz, g.ny, g.nx)[:, :, self.ghost:self.ghost + self.own]

    def owned_current(self):
        """(jx, jy, jz), each [nz, ny, own]: this slab's part of the global J."""
        J = self.current()
        return tuple(np.ascontiguousarray(self._owned(a)) for a in (J.jx, J.jy, J.jz))

    def owned_density(self) -> np.ndarray:
        return np.ascontiguousarray(self._owned(self.density()))


# ---- neighbour exchange on the periodic ring ------------------------------------

class RingExchange:
    """Send to the left / right rank, receive from them (torch.distributed).

    One batch per exchange, ordered [send right, recv left, send left, recv
    right] on every rank, so when both neighbours are the same rank (world 2)
    the pairwise FIFO order still matches each send with the right receive.
    Empty messages travel as one padding row.  world 1: the ring is this rank.
    """

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        up = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if up else 1
        self.rank = dist.get_rank(group) if up else 0
        self.left = (self.rank - 1) % self.world
        self.right = (self.rank + 1) % self.world

    def _peer(self, r):
        return self.dist.get_global_rank(self.group, r) if self.group is not None else r

    def _p2p(self, send_r, recv_l, send_l, recv_r):
        d = self.dist
        ops = [d.P2POp(d.isend, send_r, self._peer(self.right), self.group),
               d.P2POp(d.irecv, recv_l, self._peer(self.left), self.group),
               d.P2POp(d.isend, send_l, self._peer(self.left), self.group),
               d.P2POp(d.irecv, recv_r, self._peer(self.right), self.group)]
        for req in d.batch_isend_irecv(ops):
            req.wait()

    def exchange(self, to_left, to_right, sized: bool = False):
        """Returns (from_left, from_right): the left rank's `to_right` and the
        right rank's `to_left`.  sized=True: row counts may differ per rank."""
        torch = _torch()
        if self.world == 1:
            return to_right, to_left
        row = tuple(to_left.shape[1:])
        if sized:
            cnt_r = torch.tensor([to_right.shape[0]], dtype=torch.int64, device=to_right.device)
            cnt_l = torch.tensor([to_left.shape[0]], dtype=torch.int64, device=to_left.device)
            got_l, got_r = torch.empty_like(cnt_r), torch.empty_like(cnt_l)
            self._p2p(cnt_r, got_l, cnt_l, got_r)
            n_l, n_r = int(got_l.item()), int(got_r.item())
        else:
            n_l, n_r = to_right.shape[0], to_left.shape[0]

        def pad(t):
            return t if t.shape[0] else torch.zeros((1,) + row, dtype=t.dtype, device=t.device)

        from_l = torch.empty((max(n_l, 1),) + row, dtype=to_left.dtype, device=to_left.device)
        from_r = torch.empty((max(n_r, 1),) + row, dtype=to_left.dtype, device=to_left.device)
        self._p2p(pad(to_right).contiguous(), from_l, pad(to_left).contiguous(), from_r)
        return from_l[:n_l], from_r[:n_r]


def _sync(dev):
    torch = _torch()
    if torch.cuda.is_available():
        torch.cuda.current_stream(dev).synchronize()


def slab_step(sess: SlabSession, ring: RingExchange, dt: float, flags: int = STEP_DEFAULT) -> dict:
    """One step of `sess` with its ring neighbours (collective over the ring)."""
    torch = _torch()
    counts = sess.begin(dt, flags)
    tl, tr = sess.leavers(counts)
    fl, fr = ring.exchange(tl, tr, sized=True)
    # the concatenation is queued on torch's stream; the session reads the
    # arrivals from its own (non-blocking) stream, so synchronise after it
    arr = torch.cat([fl, fr]) if fl.shape[0] + fr.shape[0] else None
    _sync(sess.device)
    stats = sess.end(arr)
    for field, bit in ((0, STEP_CURRENT), (1, STEP_DENSITY)):
        if flags & bit:
            lo, hi = sess.guard_planes(field)
            gl, gr = ring.exchange(lo.view(1, -1), hi.view(1, -1))
            _sync(sess.device)
            sess.add_guard_planes(field, gl.reshape(-1), gr.reshape(-1))
    stats["sent"] = counts[0] + counts[1]
    return stats


class NcclComm:
    """A communicator of the library's own NCCL path (picgpu_comm_*): rank 0's
    unique id is broadcast over the host application's process group (any
    torch.distributed backend), then every rank joins.  Slab r of the
    decomposition belongs to rank r of this communicator."""

    def __init__(self, device: int = 0, group=None, world: int | None = None, rank: int | None = None):
        torch = _torch()
        import torch.distributed as dist

        up = dist.is_available() and dist.is_initialized()
        self.world = world if world is not None else (dist.get_world_size(group) if up else 1)
        self.rank = rank if rank is not None else (dist.get_rank(group) if up else 0)
        uid = np.zeros(128, np.uint8)
        if self.rank == 0:
            _check(lib().picgpu_comm_unique_id(uid.ctypes.data_as(C.c_void_p)))
        if self.world > 1:
            backend = dist.get_backend(group)
            t = torch.from_numpy(uid.copy())
            if backend == "nccl":
                t = t.to(torch.device("cuda", device))
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast(t, src=src, group=group)
            uid = t.cpu().numpy().astype(np.uint8)
        self._h = C.c_void_p()
        _check(lib().picgpu_comm_init(uid.ctypes.data_as(C.c_void_p), self.world, self.rank, device,
                                      C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().picgpu_comm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        self.close()


def attach_comm(sess: SlabSession, comm: NcclComm, bucket: int = 0):
    """picgpu_session_set_comm: the session's exchanges go through `comm`."""
    _check(lib().picgpu_session_set_comm(sess._h, comm._h, bucket))
    sess._comm = comm  # keep it alive


def nccl_slab_step(sess: SlabSession, dt: float, flags: int = STEP_DEFAULT) -> dict:
    """One slab step entirely behind the C ABI (picgpu_session_slab_step):
    exchanges over NCCL on the session stream, one host synchronisation."""
    st = StepStats()
    _check(lib().picgpu_session_slab_step(sess._h, dt, flags, C.byref(st)))
    return st.as_dict()


def local_ring_step(sessions: list[SlabSession], dt: float, flags: int = STEP_DEFAULT) -> list[dict]:
    """The same step for P slab sessions driven in lockstep by one process
    (single-GPU validation of the decomposition; the exchanges are device
    copies instead of NCCL messages)."""
    torch = _torch()
    P = len(sessions)
    counts = [s.begin(dt, flags) for s in sessions]
    recs = [s.leavers(c) for s, c in zip(sessions, counts)]
    stats = []
    for r, s in enumerate(sessions):
        arr = torch.cat([recs[(r - 1) % P][1], recs[(r + 1) % P][0]])
        _sync(s.device)  # the cat runs on torch's stream; the session reads on its own stream
        st = s.end(arr if arr.shape[0] else None)
        st["sent"] = counts[r][0] + counts[r][1]
        stats.append(st)
    for field, bit in ((0, STEP_CURRENT), (1, STEP_DENSITY)):
        if flags & bit:
            planes = [s.guard_planes(field) for s in sessions]
            for r, s in enumerate(sessions):
                s.add_guard_planes(field, planes[(r - 1) % P][1], planes[(r + 1) % P][0])
    return stats


def assemble_x(parts: list[np.ndarray]) -> np.ndarray:
    """Concatenate per-slab [nz, ny, own] blocks along x into the flat global field."""
    return np.concatenate(parts, axis=2).reshape(-1)
