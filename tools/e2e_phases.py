"""Where the end-to-end solve() time goes (config 2): session creation,
passes, state and dual download."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_10084_b200 import instances  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession, SolverConfig, solve  # noqa: E402

inst = instances.config_instance(2)
solve(inst, SolverConfig(tile_size=40, fixed_passes=2))  # warm: module load, JIT-free
for _ in range(2):
    t0 = time.perf_counter()
    s = DeviceSession(inst, "tiled", 40)
    t1 = time.perf_counter()
    for _ in range(23):
        s.run(1)
    t2 = time.perf_counter()
    x, f = s.state()
    t3 = time.perf_counter()
    k, v, pd = s.duals()
    t4 = time.perf_counter()
    s.close()
    t5 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  23 passes {1e3*(t2-t1):.1f} ms  state {1e3*(t3-t2):.1f}  "
          f"duals {1e3*(t4-t3):.1f}  close {1e3*(t5-t4):.1f}")
t0 = time.perf_counter()
sol = solve(inst, SolverConfig(tile_size=40, fixed_passes=23))
print(f"solve(): {1e3*(time.perf_counter()-t0):.1f} ms")
s = DeviceSession(inst, "tiled", 40)
s.run(2)
import time as _t
t0 = _t.perf_counter()
st = s.run(23)
t1 = _t.perf_counter()
print(f"run(23) in one call: {1e3*(t1-t0):.1f} ms  device sum {sum(x.wall_time for x in st)*1e3:.1f} ms")
s.close()
if os.environ.get("PROFILE"):
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    solve(inst, SolverConfig(tile_size=40, fixed_passes=23))
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
