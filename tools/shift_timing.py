import sys, time
sys.path.insert(0, ".")
import paper_2601_08277_b200 as pg
fuse = float(sys.argv[1]) if len(sys.argv) > 1 else 0.03
G = pg.Grid.make(512, 128, 128)
S = pg.Session(G, 3, timing=True)
S.set_fusion(fuse)
S.generate_lwfa(pg.LwfaConfig.make())
pid = S.num_particles
for it in range(8):
    t0 = time.perf_counter(); st = S.step(0.5); t1 = time.perf_counter()
    if it % 2 == 1:
        d, i = S.shift_window(8, 0.01, 1, pid); pid += i
        S.synchronize()
        t2 = time.perf_counter()
        print(f"step {1e3*(t1-t0):.2f} ms  shift {1e3*(t2-t1):.2f} ms  dropped {d} injected {i} rebuilt {st['rebuilt']} fused {st['fused']} moved {st['moved']}")
    else:
        print(f"step {1e3*(t1-t0):.2f} ms rebuilt {st['rebuilt']} fused {st['fused']} moved {st['moved']}")
print(S.phase_times())
