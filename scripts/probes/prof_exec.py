import cProfile, pstats, sys, time
sys.path.insert(0, '.')
from paper_1805_00988_b200 import State, build_qft, execute
s = State(16); q = build_qft(16)
for _ in range(5): execute(q, s, fuse=False)
s.flush()
t = time.perf_counter()
for _ in range(20): execute(q, s, fuse=False)
s.flush()
print("per gate us", (time.perf_counter() - t) / 20 / 136 * 1e6)
t = time.perf_counter()
for _ in range(20):
    for j in range(16): s.h(j)
s.flush()
print("State.h per call us", (time.perf_counter() - t) / 20 / 16 * 1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(20): execute(q, s, fuse=False)
s.flush(); pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(12)
