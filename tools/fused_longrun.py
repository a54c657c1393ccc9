"""Fused step over a long run from the uniform start: per-10-step averages."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2601_08277_b200 as pg
G = pg.Grid.make(128)
S = pg.Session(G, order=3, timing=True)
S.generate_plasma(16, 0.01, seed=1)
for blk in range(30):
    S.reset_phase_times()
    rb = 0
    for _ in range(10):
        rb += S.step(0.5)["rebuilt"]
    ph = S.phase_times()
    if blk % 3 == 0 or blk == 29:
        off, cnt = S.bins()
        print(f"steps {blk*10+10:4d}: fused {ph['deposit_current'][0]/10:.3f} ms  rest {ph['push_sort'][0]/10:.3f}"
              f"  rebuild {ph['rebuild_or_global_sort'][0]/10:.3f}  rebuilds {rb}  cell count std {cnt.std():.2f}")
