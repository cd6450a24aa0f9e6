"""Per-pass device time of a fresh config-3 session (first passes: pool growth, overflow retries?)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_10084_b200 import instances  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession  # noqa: E402
inst = instances.config_instance(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
s = DeviceSession(inst, "tiled", 40)
st = s.run(int(sys.argv[2]) if len(sys.argv) > 2 else 23)
print(" ".join(f"{q.wall_time*1e3:.1f}" for q in st))
print("nnz", [q.nnz_metric for q in st][:6], "...", st[-1].nnz_metric)
s.close()
