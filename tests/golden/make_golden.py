"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libpicref.so,
the unmodified reference headers compiled by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures are small and committed; the GPU box never needs the reference.

Each case stores the input store (SURVEY 8(d) generator on the reference's
counter RNG), and what the reference's own functions return on it:
  J_o{1,3}        pic::deposit_scalar            (deposit.hpp:62-73)
  rho_o{1,3}      pic::deposit_density, q*W       (deposit.hpp:76-83)
  perm            pic::gpma_build's stable counting sort (gpma.hpp:379-394)
  adv{k}_x/y/z    pic::advance after k steps      (workload.hpp:139-155)
  bins{k}         bin of every particle after detect_moves + apply_pending_moves
  cap_gpma        Gpma capacity after gpma_build  (layout rule gpma.hpp:274-281)
Order 2 (TSC) has no reference; it is not in these fixtures.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402

CASES = {
    # name: (grid kwargs, ppc, u_th, seed, q, dt, steps)
    "cube8": (dict(nx=8), 4, 0.1, 1, -1.0, 0.5, 4),
    "box12x9x7": (dict(nx=12, ny=9, nz=7, dx=0.5, dy=1.0, dz=0.25, origin=(-1.0, 2.0, 0.5)), 3, 0.05, 7, 1.5, 0.5, 4),
    "cube5_ppc6": (dict(nx=5), 6, 0.2, 77, -2.0, 0.5, 3),
}


def make_case(ref, orc, name, gkw, ppc, u_th, seed, q, dt, steps):
    g = O.Grid.make(**gkw)
    s = orc.make_plasma(g, ppc, u_th, seed)
    out = {"grid": np.array([g.nx, g.ny, g.nz], np.int32),
           "spacing": np.array([g.dx, g.dy, g.dz]), "origin": np.array([g.ox, g.oy, g.oz]),
           "q": np.array(q), "dt": np.array(dt), "ppc": np.array(ppc)}
    for k in ("x", "y", "z", "vx", "vy", "vz", "w", "id"):
        out[k] = s[k].copy()
    st = ref.state(g, s, q)
    quantity = q * s["w"]
    for order in (1, 3):
        jx, jy, jz = st.deposit_scalar(order)
        out[f"J_o{order}"] = np.stack([jx, jy, jz])
        out[f"rho_o{order}"] = st.deposit_density(order, quantity)
    # gpma_build on a fresh copy (ids == storage index -> id after build is perm)
    st2 = ref.state(g, s, q)
    st2.gpma_build()
    out["perm"] = st2.particles()["id"].astype(np.uint32)
    out["cap_gpma"] = np.array(st2.gpma_stats()["capacity"])
    # advance + incremental sort in lockstep (baseline-incrsort composition)
    for k in range(1, steps + 1):
        frac = st2.advance(dt)
        res = st2.incremental_sort()
        p = st2.particles()
        out[f"adv{k}_x"], out[f"adv{k}_y"], out[f"adv{k}_z"] = p["x"], p["y"], p["z"]
        out[f"adv{k}_id"] = p["id"]
        out[f"adv{k}_frac"] = np.array(frac)
        bin_of, _ = st2.bins()
        out[f"bins{k}"] = bin_of
        out[f"pending{k}"] = np.array(res["pending"])
    p = st2.particles()
    jx, jy, jz = st2.deposit_scalar(3, use_gpma=True)
    out["final_J_o3_bin_order"] = np.stack([jx, jy, jz])
    out["final_rho_o3"] = st2.deposit_density(3, q * p["w"])
    return out


def main():
    if not O.reference_available():
        raise SystemExit("oracle/_ref/libpicref.so missing: run `make -C oracle` where /root/reference exists")
    ref = O.Reference()
    orc = O.Oracle()
    for name, (gkw, ppc, u_th, seed, q, dt, steps) in CASES.items():
        data = make_case(ref, orc, name, gkw, ppc, u_th, seed, q, dt, steps)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
