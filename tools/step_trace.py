"""Per-step wall time and step counters for the C2 bench loop."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_08277_b200 as pg
n = int(os.environ.get("NCELL", "128")); ppc = int(os.environ.get("PPC", "16")); uth = float(os.environ.get("UTH", "0.01"))
S = pg.Session(pg.Grid.make(n), order=3, timing=True)
S.generate_plasma(ppc, uth, seed=1)
for i in range(int(os.environ.get("STEPS", "16"))):
    S.reset_phase_times()
    t = time.perf_counter()
    st = S.step(0.5)
    w = (time.perf_counter() - t) * 1e3
    print(i, round(w, 2), {k: st[k] for k in ("moved", "inserts", "overflowed", "rebuilt")},
          {k: round(v[0], 2) for k, v in S.phase_times().items()}, flush=True)
