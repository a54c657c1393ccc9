"""Per-step wall time vs device phases for the C2 bench loop."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_08277_b200 as pg
G = pg.Grid.make(128)
S = pg.Session(G, order=3, timing=bool(int(os.environ.get("TIMING", "1"))))
S.generate_plasma(16, 0.01, seed=1)
for _ in range(3):
    S.step(0.5)
stream = torch.cuda.ExternalStream(S.stream)
S.reset_phase_times()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
walls = []
e0.record(stream)
for _ in range(10):
    t = time.perf_counter()
    S.step(0.5)
    walls.append((time.perf_counter() - t) * 1e3)
e1.record(stream)
e1.synchronize()
print("device ms/step", e0.elapsed_time(e1) / 10, "wall ms/step", sum(walls) / 10, [round(w, 2) for w in walls])
print({k: round(v[0] / 10, 3) for k, v in S.phase_times().items()})
