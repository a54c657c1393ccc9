import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2601_08277_b200 as pg
from paper_2601_08277_b200.slab import SlabSession, slab_range, local_ring_step, assemble_x
import oracle
G = pg.Grid.make(16, 8, 8, dx=0.5, dy=0.5, dz=0.5, origin=(-2.0, 0.0, 1.0))
for P in (1, 2):
    ref = pg.Session(G, 3); ref.generate_plasma(4, float(sys.argv[1]) if len(sys.argv) > 1 else 0.6, seed=7)
    slabs = [SlabSession(G, *slab_range(G.nx, P, r), order=3) for r in range(P)]
    for s in slabs: s.generate_plasma(4, float(sys.argv[1]) if len(sys.argv) > 1 else 0.6, seed=7)
    flags = pg.STEP_DEFAULT
    want = ref.step(0.5, flags)
    stats = local_ring_step(slabs, 0.5, flags)
    comps = [s.owned_current() for s in slabs]
    J = [assemble_x([c[i] for c in comps]) for i in range(3)]
    Jr = ref.current()
    R = [Jr.jx, Jr.jy, Jr.jz]
    print("P", P, "fused", [st["fused"] for st in stats], "moved", sum(st["moved"] for st in stats), want["moved"],
          "err", oracle.peak_rel_err(J, R))
    for c in range(3):
        d = (J[c] - R[c]).reshape(8, 8, 16)
        bad = np.argwhere(np.abs(d) > 1e-9 * np.abs(R[c]).max())
        print("  comp", c, "bad nodes", len(bad), "x-planes", sorted(set(bad[:, 2].tolist()))[:20])
