"""Fused step vs migration rate at C2 size: python tools/fused_uth.py [u_th ...]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08277_b200 as pg
G = pg.Grid.make(128)
for uth in [float(a) for a in sys.argv[1:]] or [0.0, 0.002, 0.01, 0.03]:
    S = pg.Session(G, order=3, timing=True)
    S.set_fusion(2.0)
    S.generate_plasma(16, uth, seed=1)
    for _ in range(3):
        S.step(0.5)
    S.reset_phase_times()
    moved = 0
    for _ in range(10):
        moved += S.step(0.5)["moved"]
    ph = S.phase_times()
    print(f"u_th {uth}: moved {moved / 10 / S.num_particles:.4f}  fused kernel {ph['deposit_current'][0] / 10:.3f} ms"
          f"  movers+insert+borrow {ph['push_sort'][0] / 10:.3f} ms")
    S.close()
