"""Per-kernel view of the incremental sort at C3 (256^3 x 32 ppc, u_th 0.1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08277_b200 as pg
G = pg.Grid.make(256)
S = pg.Session(G, order=3, timing=True)
S.generate_plasma(32, 0.1, seed=1)
for _ in range(2):
    S.step(0.5)
S.reset_phase_times()
for i in range(3):
    st = S.step(0.5)
    print({k: st[k] for k in ("moved", "inserts", "overflowed", "rebuilt")})
print({k: round(v[0] / 3, 2) for k, v in S.phase_times().items()})
