"""Where the FIRST solve() of a process goes at config 3 (bench.py's e2e leg): session
creation by phase (MP_TIME_CREATE in a knobs build), passes, state and dual download."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_10084_b200 import instances  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession  # noqa: E402

inst = instances.config_instance(3)
for rep in range(2):
    t0 = time.perf_counter()
    s = DeviceSession(inst, "tiled", 40)
    t1 = time.perf_counter()
    st = s.run(23)
    t2 = time.perf_counter()
    x, f = s.state()
    t3 = time.perf_counter()
    k, v, pd = s.duals()
    t4 = time.perf_counter()
    s.close()
    t5 = time.perf_counter()
    print(f"call {rep}: create {1e3*(t1-t0):.1f} ms  23 passes {1e3*(t2-t1):.1f} ms (device sum "
          f"{sum(q.wall_time for q in st)*1e3:.1f})  state {1e3*(t3-t2):.1f}  duals {1e3*(t4-t3):.1f}  "
          f"close {1e3*(t5-t4):.1f}")
