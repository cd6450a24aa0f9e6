"""Metric-phase vs pair-phase device time of a few passes (config 2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_10084_b200 import instances  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession  # noqa: E402

inst = instances.config_instance(int(os.environ.get("CFG", "2")))
s = DeviceSession(inst, "tiled", 40)
s.run(4)
for _ in range(3):
    st = s.run(1)[0]
    m, p, nl = s.timing()
    print(f"total {st.wall_time*1e3:.3f} ms  metric {m:.3f}  pair {p:.3f}  launches {nl}")
