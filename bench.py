#!/usr/bin/env python
"""Benchmark: particle current deposits/s on B200 (BASELINE.json metric).

Workload (N=1): BASELINE configs[1] ("C2"): 128^3 cells, 16 particles/cell,
order 3 (QSP), Maxwellian u_th = 0.01c, dt = 0.5, seeded synthetic plasma
(SURVEY 8(d) generator, generated in HBM).  One STEP = the reference's step
(simulation.hpp:92-176): bit-exact push -> incremental cell sort (bins with
slack, migration) -> current deposition J.  Inputs stay resident in HBM.  At
low migration the step runs fused: ONE pass over the bins pushes every
particle, detects the movers and deposits J (movers' out-of-window taps by a
small reduction kernel), then the movers are inserted into their new bins.

value  = particles * steps * n_gpus / (max over ranks of the device time of K steps)
e2e    = the same metric through the stateless C-ABI drop-in for
         pic::deposit_scalar (picgpu_deposit_current) on pinned HOST buffers:
         H2D of the 7 particle arrays + sort + deposit + D2H of J every step.
roofline: the dominant kernel (the fused push + detect + J kernel, or the J
         kernel in unfused steps), timed with CUDA events on the session's
         stream inside the timed region.  Order 3 is FP64-bound: achieved =
         particles * 534 flops (reference tally, deposit.hpp:336-345; the
         push's flops are not counted) / launch time, against the FP64 peak
         measured in-run by a DFMA microbenchmark (MEASURED_PEAKS.json has no
         FP64 figure); the HBM view (56 [+ 24 written back when fused] +
         24/ppc bytes per deposit vs MEASURED_PEAKS hbm_gbs) is reported beside it.
cpu_baseline: the reference's own step (oracle/_ref, its headers compiled:
         advance + detect_moves + apply_pending_moves + deposit_scalar over the
         Gpma bins, simulation.hpp:117-136) on the SAME box (C2: 128^3 x 16 ppc,
         the same seeded plasma), pinned to ONE host core (the reference is
         single-threaded), 2 timed steps.
orders:  the same box and step at shape orders 1, 2 and 3 (the metric names all
         three), each with its kernel roofline fraction.
selfcheck: grid totals of the last J against q*sum(w*v) (partition of unity):
         the bench refuses to print a number from a wrong deposit.

--impl reference runs only the CPU arm: the same one-core reference step on the
config's box, warm-up 1 step, up to K timed steps within ~150 s, plus the
deposit_density rate and a labelled all-threads sub-box figure.
Multi-GPU (torchrun, N>1): x-slab decomposition of one periodic
box of (128*N) x 128 x 128 cells; each rank owns a C2-sized slab (weak
scaling) and every step exchanges leaving particles and J guard planes with its
two ring neighbours over NCCL (paper_2601_08277_b200/slab.py).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n, ppc, order, u_th, dt, default steps, description)
    "c1": (64, 8, 1, 0.01, 0.5, 10, "C1: 64^3 cells, 8 ppc, order 1 (CIC), u_th 0.01, dt 0.5"),
    "c2": (128, 16, 3, 0.01, 0.5, 20, "C2: 128^3 cells, 16 ppc, order 3 (QSP), u_th 0.01, dt 0.5"),
    "c3o1": (256, 32, 1, 0.1, 0.5, 5, "C3: 256^3 cells, 32 ppc, order 1, u_th 0.1, dt 0.5"),
    "c3o2": (256, 32, 2, 0.1, 0.5, 5, "C3: 256^3 cells, 32 ppc, order 2 (TSC), u_th 0.1, dt 0.5"),
    "c3o3": (256, 32, 3, 0.1, 0.5, 5, "C3: 256^3 cells, 32 ppc, order 3, u_th 0.1, dt 0.5"),
    "c4": ((512, 128, 128), 8, 3, 0.01, 0.5, 100,
           "C4 (LWFA-like, static window): 512x128x128 cells, order 3, electrons from x-cell 64 with a linear "
           "density ramp over [64,128) to 8 ppc, u_th 0.01, plus a 10% beam with ux ~ U(5,50) in x-cells "
           "[128,160); dt 0.5; moving window: origin +1 cell every 2 steps, back column dropped, a fresh 8-ppc "
           "column injected at the front (inside the timed region)"),
    # strong scaling over x-slabs; needs N >= 4 B200s (2.1e9 particles)
    "c5": ((2048, 256, 256), 16, 3, 0.05, 0.5, 50,
           "C5: 2048x256x256 cells, 16 ppc, order 3, u_th 0.05, dt 0.5, x-slabs of 2048/N cells per GPU "
           "(strong scaling)"),
}


def make_grid(pg, n):
    return pg.Grid.make(*n) if isinstance(n, tuple) else pg.Grid.make(n)


def populate(pg, S, name, ppc, u_th, seed=1):
    if name == "c4":
        S.generate_lwfa(pg.LwfaConfig.make(ppc=ppc, ramp_start=64, ramp_len=64, u_th=u_th, beam_fraction=0.1,
                                           ux=(5.0, 50.0), beam_x=(128.0, 160.0), seed=seed))
    else:
        S.generate_plasma(ppc, u_th, seed=seed)
METRIC = "particle current deposits/sec"
UNIT = "deposits/s"
FLOPS = {1: 76, 2: 238, 3: 534}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()  # the sampler is live before the timed region starts
            while not self.rows and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


class OneCore:
    """Pin this process to one host core for the duration (the reference is
    single-threaded; taskset -c 0)."""

    def __enter__(self):
        self.old = os.sched_getaffinity(0)
        self.core = min(self.old)
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *a):
        os.sched_setaffinity(0, self.old)


def cpu_box(cfgname):
    """(grid dims, note) of the box the CPU reference runs for this config."""
    nx, ppc, order, u_th, dt, _, desc = CONFIGS[cfgname]
    if cfgname.startswith("c3"):  # 537M particles do not fit a bounded CPU sample: the same per-cell workload
        return (128, 128, 128), "128^3 x 32 ppc box (C3's per-cell workload at 1/8 of its cells)"
    if cfgname == "c4":  # the LWFA generator is device-only: a uniform 8 ppc plasma on the C4 grid
        return nx, "uniform 8 ppc plasma on the C4 grid (stand-in for the ramp + beam population)"
    if cfgname == "c5":
        return (128, 128, 128), "C2-sized 128^3 x 16 ppc box (C5's per-GPU slab workload)"
    return (nx, nx, nx), "the config's own box"


def cpu_reference_box(cfgname, max_steps, budget_s, warmup=1, with_rho=False):
    """The reference's baseline-incrsort step (simulation.hpp:117-136: advance ->
    detect_moves + apply_pending_moves -> deposit_scalar over the Gpma bins),
    compiled from its own headers (oracle/_ref), on the config's box, pinned to
    ONE host core.  Each stage is timed by the reference's pic::Timer; the
    throughput is particles / (advance + sort + deposit) per step
    (simulation.hpp:158-160 counts sort + deposit).  Timed steps stop at
    max_steps or when the next step would exceed budget_s (a bounded sample)."""
    import oracle

    if not oracle.reference_available():
        return None
    nx, ppc, order, u_th, dt, _, desc = CONFIGS[cfgname]
    dims, note = cpu_box(cfgname)
    ref_order = order if order in (1, 3) else 3  # the reference has no order 2: its QSP step stands in
    g = oracle.Grid.make(*dims)
    with OneCore() as one:
        t_setup = time.perf_counter()
        s = oracle.Oracle().make_plasma(g, ppc, u_th, seed=1)  # the bench's seeded recipe
        st = oracle.RefState(oracle.Reference(), g, s, -1.0)
        del s
        st.gpma_build()
        for _ in range(warmup):
            st.step_timed(ref_order, dt)
        t_setup = time.perf_counter() - t_setup
        stages = [0.0, 0.0, 0.0]
        steps = moved = rebuilt = 0
        while steps < max_steps:
            a, b, c, m, r = st.step_timed(ref_order, dt)
            stages = [stages[0] + a, stages[1] + b, stages[2] + c]
            steps += 1
            moved += m
            rebuilt += r
            if sum(stages) * (steps + 1) / steps > budget_s:
                break
        rho_s = st.density_timed(ref_order) if with_rho else None
        n = st.n
        core = one.core
    total = sum(stages)
    out = {"value": n * steps / total, "n": n, "steps": steps, "seconds": total,
           "s_per_step": {"advance": stages[0] / steps, "sort": stages[1] / steps, "deposit_scalar": stages[2] / steps},
           "deposit_only_per_s": n * steps / stages[2], "moved_fraction": moved / (n * steps), "rebuilds": rebuilt,
           "grid": list(dims), "ppc": ppc, "order": ref_order, "box_note": note, "core": core,
           "warmup_steps": warmup, "setup_s": t_setup, **cpu_info()}
    if rho_s is not None:
        out["deposit_density_per_s"] = n / rho_s
    return out


def cpu_reference_subboxes(order, ppc, u_th, dt, steps, threads, nx=32, seed=1):
    """Labelled extra: `threads` independent 32^3 sub-boxes, one reference step loop each."""
    import oracle

    L = oracle.Reference().L
    L.ref_bench_steps.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_double, C.c_int, C.c_int,
                                  C.c_void_p, C.c_void_p]
    sec, n = C.c_double(), C.c_uint64()
    rc = L.ref_bench_steps(nx, ppc, u_th, seed, order if order in (1, 3) else 3, dt, steps, threads, C.byref(sec),
                           C.byref(n))
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    return {"value": n.value * threads * steps / sec.value, "threads": threads, "sub_box_particles": n.value,
            "steps": steps, "note": f"{threads} threads x independent {nx}^3 x {ppc} ppc periodic sub-boxes "
                                    "(NOT the config's box; the reference itself is single-threaded)"}


def cpu_sample_text(r):
    g = "x".join(map(str, r["grid"]))
    return (f"{g} x {r['ppc']} ppc ({r['n']} particles, {r['box_note']}), 1 core (#{r['core']} of {r['nproc']}, "
            f"{r['model']}), {r['steps']} timed reference steps (advance + detect_moves + apply_pending_moves + "
            f"deposit_scalar order {r['order']}) after {r['warmup_steps']} warm-up, {r['seconds']:.1f} s")


def run_reference_arm(args, cfgname):
    nx, ppc, order, u_th, dt, _, desc = CONFIGS[cfgname]
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    K = args.steps
    # one warm-up step (the CPU has no JIT or device state to warm) and at most
    # ~150 s of timed steps, so the arm ends within a few minutes at C2
    r = cpu_reference_box(cfgname, K, budget_s=float(os.environ.get("PICGPU_REF_BUDGET_S", "150")),
                          warmup=min(args.warmup, 1), with_rho=True)
    if r is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libpicref.so not built"}))
        return 0
    value = r["value"]
    extra = None
    try:
        extra = cpu_reference_subboxes(order, ppc, u_th, dt, 3, os.cpu_count() or 1)
    except Exception as e:  # a labelled extra only
        extra = {"error": str(e)}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": K, "warmup": args.warmup,
        "ms_per_step": r["seconds"] / r["steps"] * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY 8(d) generator, reference counter RNG)",
        "config": {"workload": desc + "; step = push + incremental sort + J deposit",
                   "grid": list(nx) if isinstance(nx, tuple) else [nx] * 3, "ppc": ppc, "order": order,
                   "parallelism": "single" if args.gpus == 1 else f"x-slabs x{args.gpus} (GPU arm); CPU: rank 0 only"},
        "impl": "reference",
        "same_config": r["box_note"] == "the config's own box" and r["order"] == order,
        "timed_steps": r["steps"],
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference", "sample": cpu_sample_text(r)},
        "cpu_detail": r,
        "cpu_parallel_subboxes": extra,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def load_traffic(cfgname, order, fused):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel, from an ncu --set full capture of THIS config/order/path
    (profiles/ncu_traffic.json, tools/traffic.sh); null when not captured."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"{cfgname}_o{order}_{'fused' if fused else 'unfused'}")
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--order", type=int, default=None, choices=[1, 2, 3], help="override the config's shape order")
    ap.add_argument("--steady-steps", type=int, default=130,
                    help="C2: time the step again after this many further steps (steady-state cell counts)")
    ap.add_argument("--no-orders", dest="orders", action="store_false",
                    help="skip the per-order (1/2/3) runs on the same box")
    ap.add_argument("--slab", action="store_true", help="use the slab-decomposed path even at N=1 (loopback ring)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "torch"],
                    help="slab exchanges: nccl = picgpu_session_slab_step (NCCL behind the C ABI, one host sync per "
                         "step); torch = the Python protocol over torch.distributed (slab.py slab_step)")
    ap.add_argument("--sort", default="incremental", choices=["incremental", "resort"],
                    help="incremental: bins with slack + migration (default); resort: a full stable counting "
                         "sort of the store every step (global_sort each step; the crossover study of C3)")
    args = ap.parse_args()
    nx, ppc, order, u_th, dt, default_steps, desc = CONFIGS[args.config]
    if args.order is not None and args.order != order:
        order = args.order
        desc += f" [shape order overridden: {order}]"
        CONFIGS[args.config] = (nx, ppc, order, u_th, dt, default_steps, desc)
    if args.steps is None:
        args.steps = default_steps
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference_arm(args, args.config)

    import numpy as np
    import torch

    import paper_2601_08277_b200 as pg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    grid = make_grid(pg, nx)
    strong = args.config == "c5"
    G_dims = nx if isinstance(nx, tuple) else (nx * world, nx, nx)
    if strong and world < 4:
        raise SystemExit("c5 (2.1e9 particles) needs at least 4 GPUs: torchrun --nproc-per-node 4|8 bench.py --config c5")
    if isinstance(nx, tuple) and world > 1 and not strong:
        raise SystemExit("multi-GPU runs use the cubic configs (x-slabs of a (n*N) x n x n box) or c5")
    single = world == 1 and not args.slab
    fp64_peak = pg.fp64_peak_tflops(local)
    try:  # SMs x 64 DFMA/clk x 2 flops x max SM clock (MEASURED_PEAKS.json sm_max_mhz)
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f).get("sm_max_mhz", 1965.0))
    except Exception:
        mhz = 1965.0
    fp64_nominal = torch.cuda.get_device_properties(local).multi_processor_count * 64 * 2 * mhz * 1e6 / 1e12
    hbm_peak, hbm_src = peaks()

    comm_box = [None]  # one NCCL communicator for every session of the run

    def open_session(order):
        if single:
            S = pg.Session(grid, order=order, device=local, timing=True)
            if args.sort == "resort":
                step = lambda: S.step(dt, pg.STEP_PUSH | pg.STEP_RESORT | pg.STEP_CURRENT)  # noqa: E731
            else:
                step = lambda: S.step(dt)  # noqa: E731
        else:
            from paper_2601_08277_b200.slab import RingExchange, SlabSession, slab_step

            if strong:  # one global box split into x-slabs
                from paper_2601_08277_b200.slab import slab_range

                G = pg.Grid.make(*nx)
                S = SlabSession(G, *slab_range(nx[0], world, rank), order=order, device=local, timing=True)
            else:  # weak scaling: a C2-sized slab per rank
                G = pg.Grid.make(nx * world, nx, nx)
                S = SlabSession(G, rank * nx, (rank + 1) * nx, order=order, device=local, timing=True)
            if args.exchange == "nccl":  # the whole slab step behind the C ABI (NCCL on the session stream)
                from paper_2601_08277_b200.slab import NcclComm, attach_comm, nccl_slab_step

                if comm_box[0] is None:
                    comm_box[0] = NcclComm(device=local)
                attach_comm(S, comm_box[0])
                step = lambda: nccl_slab_step(S, dt)  # noqa: E731
            else:
                ring = RingExchange()
                step = lambda: slab_step(S, ring, dt)  # noqa: E731
        if args.config == "c4":
            # C4's beam keeps flowing into bins sized at the last layout: every
            # second step rebuilt (50 of 100); a rebuild storm widens the slack
            S.set_adaptive_slack(True)
        populate(pg, S, args.config, ppc, u_th)
        return S, step

    def measure(order):
        """W warm-up + K timed steps of the session at `order`: the bench numbers."""
        S, step = open_session(order)
        n = S.num_particles
        window = None
        if args.config == "c4":
            next_pid = [n]

            def window():
                _, inj = S.shift_window(ppc, u_th, 1, next_pid[0])
                next_pid[0] += inj
        n_total = n * world
        if dist is not None:  # particles of all ranks (conserved by the migration)
            tn = torch.tensor([float(n)], device="cuda", dtype=torch.float64)
            dist.all_reduce(tn)
            n_total = int(tn.item())
        stream = torch.cuda.ExternalStream(S.stream)
        for it in range(args.warmup):
            step()
            if window is not None and it % 2 == 1:
                window()  # loads the window kernels and grows its buffers before timing
        if single:
            S.global_sort()  # also exercises the relayout kernels before the timed region
        S.reset_phase_times()
        barrier()
        launches0 = pg.kernel_launches()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        moved = rebuilds = fused_steps = 0
        with Clocks(local) as clk:
            barrier()
            e0.record(stream)
            for it in range(args.steps):
                st = step()
                moved += st["moved"]
                fused_steps += st.get("fused", 0)
                if window is not None and it % 2 == 1:  # C4 moving window: one cell every 2 steps
                    window()
                rebuilds += st["rebuilt"]
            e1.record(stream)
            e1.synchronize()
            barrier()
        launches = pg.kernel_launches() - launches0
        ms = e0.elapsed_time(e1)
        t = torch.tensor([ms], device="cuda")
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
        phases = S.phase_times()
        j_ms, j_launches = phases["deposit_current"]
        j_avg_s = j_ms / max(j_launches, 1) * 1e-3
        # roofline of the dominant kernel: J deposition, fused with the push (positions
        # read with the particle and written back: +24 B) when the steps ran fused
        fused = fused_steps == args.steps
        bytes_per = 56 + (24 if fused else 0) + 24 * grid.ncells / n  # J written once per node, amortised
        hbm_achieved = n * bytes_per / j_avg_s / 1e9
        fp64_achieved = n * FLOPS[order] / j_avg_s / 1e12
        frac_hbm, frac_fp64 = hbm_achieved / hbm_peak, fp64_achieved / fp64_peak
        traffic = load_traffic(args.config, order, fused)
        if frac_fp64 >= frac_hbm:
            roof = {"bound": "fp64", "achieved": fp64_achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                    "frac": frac_fp64, "traffic": traffic,
                    "peak_source": "measured in-run (DFMA microbenchmark, picgpu_fp64_peak); MEASURED_PEAKS.json "
                                   "and B200_PROFILING.md carry no FP64 figure",
                    "peak_nominal": fp64_nominal, "frac_vs_nominal": fp64_achieved / fp64_nominal,
                    "flops_per_deposit": FLOPS[order]}
        else:
            roof = {"bound": "hbm", "achieved": hbm_achieved, "peak": hbm_peak, "unit": "GB/s", "frac": frac_hbm,
                    "traffic": traffic, "peak_source": hbm_src, "bytes_per_deposit": bytes_per}
        roof.update({"kernel": "deposit_current_kernel_v3 (fused push + detect + J)" if fused else
                     "deposit_current_kernel_v3 (J)", "launch_ms": j_avg_s * 1e3,
                     "traffic_per_deposit": traffic / n if traffic else None,
                     "hbm_view": {"achieved_gbs": hbm_achieved, "peak_gbs": hbm_peak, "frac": frac_hbm},
                     "fp64_view": {"achieved_tflops": fp64_achieved, "peak_tflops": fp64_peak, "frac": frac_fp64},
                     "deposits_per_s_kernel_only": n / j_avg_s})
        value = n_total * args.steps / (ms_max * 1e-3)
        # step-inclusive roofline fraction: the whole step against the kernel's bound
        step_rate_bound = min(hbm_peak * 1e9 / (56 + 24 * grid.ncells / n), fp64_peak * 1e12 / FLOPS[order])
        res = {"value": value, "ms_per_step": ms_max / args.steps, "n": n, "n_total": n_total, "roofline": roof,
               "step_roofline_frac": (value / world) / step_rate_bound, "launches": launches,
               "clocks": clk.summary(), "phases_ms_total": {k: v[0] for k, v in phases.items()},
               "moved_fraction": moved / (n * args.steps), "rebuilds": rebuilds, "fused_steps": fused_steps}
        return S, res

    def selfcheck(S, p, order):
        """Size-independent properties of the last step's output, checked in the
        bench itself (every node weight set sums to one, so the grid totals of J
        are q*sum(w*v)): a wrong kernel cannot post a number.  Slabs: the owned
        planes of every rank (guard planes already summed into them), totals
        reduced over the ranks."""
        q = -1.0
        if single:
            J = S.current()
            got = [float(np.sum(a)) for a in (J.jx, J.jy, J.jz)]
        else:
            got = [float(np.sum(a)) for a in S.owned_current()]
        want = [q * float(np.dot(p.w, v)) for v in (p.vx, p.vy, p.vz)]
        scale = [float(np.dot(p.w, np.abs(v))) for v in (p.vx, p.vy, p.vz)]
        if dist is not None:
            t = torch.tensor(got + want + scale, dtype=torch.float64, device="cuda")
            dist.all_reduce(t)
            v = t.tolist()
            got, want, scale = v[0:3], v[3:6], v[6:9]
        out = {c: abs(got[i] - want[i]) / max(scale[i], 1e-300) for i, c in enumerate(("jx", "jy", "jz"))}
        out["ok"] = all(e < 1e-9 for e in out.values())
        return out

    S, res = measure(order)
    e2e = e2e_session = check = None
    p = S.particles()
    n = p.size()
    if args.config != "c4":  # the window moved after the last deposit
        check = selfcheck(S, p, order)
        if not check["ok"]:
            print(json.dumps({"error": "bench self-check failed", "selfcheck": check}), file=sys.stderr)
            return 1
    steady = None
    if single and args.config == "c2" and args.steady_steps > 0:
        # the bench window starts from the generator's exactly-ppc cells; migration
        # spreads the counts towards Poisson (a warp's 8 pencils then contract as
        # many particles as the fullest): the same step after `steady_steps` more
        # steps (no global sort in between), reported beside the headline
        for _ in range(args.steady_steps):
            S.step(dt)
        stream = torch.cuda.ExternalStream(S.stream)
        ph0 = S.phase_times()["deposit_current"]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            S.step(dt)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        ph1 = S.phase_times()["deposit_current"]
        kms = (ph1[0] - ph0[0]) / max(ph1[1] - ph0[1], 1)
        steady = {"value": res["n"] * args.steps / (ms * 1e-3), "ms_per_step": ms / args.steps,
                  "kernel_ms": kms, "after_steps": args.warmup + args.steps + args.steady_steps,
                  "roofline_frac": res["n"] * FLOPS[order] / (kms * 1e-3) / 1e12 / fp64_peak}
    if single and args.e2e_steps > 0:
        # the device-resident session as a PIC code drives it: particles uploaded
        # once from host memory, then every step push + sort + J on the device
        # and J read back into pinned host memory (the field solver's input)
        S.upload(p, q=-1.0)
        jh = [torch.empty(grid.ncells, dtype=torch.float64, pin_memory=True) for _ in range(3)]
        L = pg.lib()

        def sess_step():
            S.step(dt)
            rc = L.picgpu_session_download_current(S._h, *(C.c_void_p(t.data_ptr()) for t in jh))
            if rc:
                raise RuntimeError(L.picgpu_last_error().decode())

        sess_step()
        torch.cuda.synchronize()
        ks = max(args.steps, 3)
        t0 = time.perf_counter()
        for _ in range(ks):
            sess_step()
        ts = time.perf_counter() - t0
        e2e_session = {"value": n * ks / ts, "unit": UNIT, "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 3 * 8 * grid.ncells, "steps": ks,
                       "api": "picgpu_session_step + picgpu_session_download_current (particles uploaded "
                              "once from host memory before timing; J read back to pinned host memory "
                              "every step)",
                       "timer": "host wall clock around synchronous C-ABI calls"}
    S.close()  # the stateless call below allocates its own workspace (C3: ~86 GB each)
    if args.e2e_steps > 0:  # every rank (the max over ranks needs them all)
        host = {}
        for k in ("x", "y", "z", "vx", "vy", "vz", "w"):
            tt = torch.empty(n, dtype=torch.float64, pin_memory=True)
            tt.numpy()[:] = getattr(p, k)
            host[k] = tt
        outs = [torch.empty(grid.ncells, dtype=torch.float64, pin_memory=True) for _ in range(3)]
        L = pg.lib()
        ptr = lambda tt: C.c_void_p(tt.data_ptr())  # noqa: E731

        def call():
            rc = L.picgpu_deposit_current(C.byref(grid), order, *(ptr(host[k]) for k in
                                                                  ("x", "y", "z", "vx", "vy", "vz", "w")),
                                          -1.0, n, ptr(outs[0]), ptr(outs[1]), ptr(outs[2]))
            if rc:
                raise RuntimeError(L.picgpu_last_error().decode())

        call()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            call()
        barrier()
        e2e_s = time.perf_counter() - t0
        tt = torch.tensor([e2e_s], device="cuda")
        ne = torch.tensor([float(n)], device="cuda", dtype=torch.float64)
        if dist is not None:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dist.all_reduce(ne)
        e2e = {"value": float(ne.item()) * args.e2e_steps / float(tt.item()), "unit": UNIT,
               "h2d_bytes_per_step": 7 * 8 * n, "d2h_bytes_per_step": 3 * 8 * grid.ncells,
               "steps": args.e2e_steps, "api": "picgpu_deposit_current (drop-in for pic::deposit_scalar)",
               "timer": "host wall clock around synchronous C-ABI calls (copies inside)"}
    del p

    # the metric names orders 1/2/3: the same box and step at the other two orders
    orders = {str(order): {"value": res["value"], "ms_per_step": res["ms_per_step"],
                           "roofline_frac": res["roofline"]["frac"], "bound": res["roofline"]["bound"],
                           "kernel_ms": res["roofline"]["launch_ms"], "step_roofline_frac": res["step_roofline_frac"],
                           "fused_steps": res["fused_steps"]}}
    if args.orders and not isinstance(nx, tuple) and not args.config.startswith("c3"):
        for o in (1, 2, 3):
            if o == order:
                continue
            So, r = measure(o)
            So.close()
            orders[str(o)] = {"value": r["value"], "ms_per_step": r["ms_per_step"],
                              "roofline_frac": r["roofline"]["frac"], "bound": r["roofline"]["bound"],
                              "kernel_ms": r["roofline"]["launch_ms"], "step_roofline_frac": r["step_roofline_frac"],
                              "fused_steps": r["fused_steps"], "traffic": r["roofline"]["traffic"],
                              "clocks": r["clocks"]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_reference_box(args.config, 2, budget_s=30.0, warmup=0)
        if r is not None:
            cpu = {"value": r["value"], "unit": UNIT, "cores": 1, "kind": "reference", "sample": cpu_sample_text(r),
                   "same_config": r["box_note"] == "the config's own box" and r["order"] == order,
                   "cpu_model": r["model"], "nproc": r["nproc"]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SURVEY 8(d) seeded plasma generated in HBM; no dataset)",
            "config": {"workload": desc + ("; step = push + full stable re-sort + J deposit" if args.sort == "resort"
                                           else "; step = push + incremental sort + J deposit"),
                       "grid": list(G_dims), "ppc": ppc,
                       "order": order, "particles_per_gpu": res["n"],
                       "l2": f"inputs larger than L2 ({res['n'] * 64 / 1e9:.1f} GB particle store)",
                       "parallelism": "single" if world == 1 else
                       f"x-slabs x{world} of a {'x'.join(map(str, G_dims))} box, NCCL ring exchange "
                       f"(migration + J guards; {'picgpu_session_slab_step' if args.exchange == 'nccl' else 'torch.distributed'})"},
            "roofline": res["roofline"], "step_roofline_frac": res["step_roofline_frac"], "orders": orders,
            "steady_state": steady,
            "cpu_baseline": cpu, "e2e": e2e, "e2e_session": e2e_session, "gpu_launches": res["launches"],
            "clocks": res["clocks"], "selfcheck": check,
            "phases_ms_total": res["phases_ms_total"],
            "moved_fraction": res["moved_fraction"], "rebuilds": res["rebuilds"], "fused_steps": res["fused_steps"],
        }
        print(json.dumps(line))
    if comm_box[0] is not None:
        comm_box[0].close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
