"""Wall-clock of solve() phases (session create, passes, download) for config 2."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_10084_b200 import instances  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession  # noqa: E402
inst = instances.config_instance(2)
for rep in range(3):
    t0 = time.perf_counter(); s = DeviceSession(inst, "tiled", 40); t1 = time.perf_counter()
    s.run(1); t2 = time.perf_counter(); s.run(22); t3 = time.perf_counter()
    s.state(); s.duals(); t4 = time.perf_counter(); s.close()
    print(f"create {t1-t0:.3f} first pass {t2-t1:.3f} 22 passes {t3-t2:.3f} download {t4-t3:.3f}")
