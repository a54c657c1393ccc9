"""Time J (and rho) deposition alone on a session: jbench.py order n ppc [u_th]."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08277_b200 as pg

order = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 128
ppc = int(sys.argv[3]) if len(sys.argv) > 3 else 16
uth = float(sys.argv[4]) if len(sys.argv) > 4 else 0.01
G = pg.Grid.make(n)
S = pg.Session(G, order=order, timing=True)
S.generate_plasma(ppc, uth, seed=1)
for _ in range(3):
    S.step(0.5)
S.step(0.5, pg.STEP_CURRENT | pg.STEP_DENSITY)  # loads the deposition modules before timing
S.reset_phase_times()
for _ in range(5):
    S.step(0.5, pg.STEP_CURRENT | pg.STEP_DENSITY)
ph = S.phase_times()
N = S.num_particles
out = {"variant": os.environ.get("PICGPU_J_VARIANT", "lane"), "order": order, "n": n, "ppc": ppc, "N": N}
for k in ("deposit_current", "deposit_density"):
    ms, launches = ph[k]
    t = ms / 5 * 1e-3
    out[k + "_ms"] = t * 1e3
    out[k + "_dep_per_s"] = N / t
out["J_frac_fp64_tally"] = N * pg.flop_count(order) / (out["deposit_current_ms"] * 1e-3) / 34.15e12
out["J_hbm_gbs"] = N * (56 + 24 / ppc) / (out["deposit_current_ms"] * 1e-3) / 1e9
print(json.dumps(out))
