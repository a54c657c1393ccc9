"""Time the J deposition kernel alone on a C2-like session (order, n, ppc from argv)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08277_b200 as pg
order = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 128
ppc = int(sys.argv[3]) if len(sys.argv) > 3 else 16
G = pg.Grid.make(n)
S = pg.Session(G, order=order, timing=True)
S.generate_plasma(ppc, 0.01 if order == 3 else 0.1, seed=1)
for _ in range(3):
    S.step(0.5)
S.reset_phase_times()
for _ in range(10):
    S.step(0.5, pg.STEP_CURRENT)
ms, launches = S.phase_times()["deposit_current"]
N = S.num_particles
t = ms / launches * 1e-3
print(json.dumps({"variant": os.environ.get("PICGPU_J_VARIANT", "lane"), "order": order, "n": n, "ppc": ppc,
                  "ms": t * 1e3, "dep_per_s": N / t, "frac_fp64_tally": N * pg.flop_count(order) / t / 34.15e12}))
