import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08277_b200 as pg
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ppc = int(sys.argv[2]) if len(sys.argv) > 2 else 16
G = pg.Grid.make(n)
S = pg.Session(G, order=3)
S.generate_plasma(ppc, 0.01, seed=1)
off, cnt = S.bins()
print("init cap", S.capacity, "n", S.num_particles, "cnt min/max", cnt.min(), cnt.max(), "caps min/max", np.diff(off.astype(np.int64)).min(), np.diff(off.astype(np.int64)).max())
for k in range(8):
    st = S.step(0.5, pg.STEP_PUSH | pg.STEP_SORT)
    off, cnt = S.bins()
    caps = np.diff(off.astype(np.int64))
    print(k, st, "cnt max", cnt.max(), "min slack", (caps - cnt).min(), "sum", cnt.sum())
