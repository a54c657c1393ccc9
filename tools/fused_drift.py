"""Fused kernel time per step after a global sort (do holes accumulate?)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08277_b200 as pg
G = pg.Grid.make(128)
S = pg.Session(G, order=3, timing=True)
S.generate_plasma(16, 0.01, seed=1)
for _ in range(3):
    S.step(0.5)
S.global_sort()
out = []
for it in range(40):
    S.reset_phase_times()
    st = S.step(0.5)
    ph = S.phase_times()
    out.append((it, round(ph["deposit_current"][0], 3), round(ph["push_sort"][0], 3), st["rebuilt"]))
print(out)
# after a hole fill (the density deposit packs the bins first)
S.step(0.5, pg.STEP_DENSITY)
res = []
for it in range(5):
    S.reset_phase_times()
    st = S.step(0.5)
    ph = S.phase_times()
    res.append(round(ph["deposit_current"][0], 3))
print("after fill_holes:", res)
