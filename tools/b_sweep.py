"""ns per critical level vs tile size b (config 2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_10084_b200 import instances, schedule  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession  # noqa: E402

inst = instances.config_instance(int(os.environ.get("CFG", "2")))
for b in [int(x) for x in os.environ.get("BS", "16 24 32 40 48 56 64").split()]:
    s = DeviceSession(inst, "tiled", b)
    s.run(4)
    st = s.run(2)
    t = min(x.wall_time for x in st)
    lv = schedule.critical_levels(inst.n, b)
    rows = 3 * (inst.n * (inst.n - 1) * (inst.n - 2) // 6)
    print(f"b={b:3d} pass {t*1e3:7.2f} ms  barrier levels {lv:6d}  "
          f"{t/lv*1e9:6.1f} ns/level  {rows/t:.3e} proj/s", flush=True)
    s.close()
