"""Pass time of schedule_kind='serial' on the device (config instance, a few passes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_10084_b200 import instances  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
inst = instances.config_instance(cfg, n=n)
s = DeviceSession(inst, "serial", 40)
for st in s.run(4):
    rows = 3 * inst.n * (inst.n - 1) * (inst.n - 2) // 6
    print(f"serial n={inst.n} pass {st.pass_index}: {st.wall_time*1e3:.2f} ms  {rows/st.wall_time:.3e} proj/s  nnz={st.nnz_metric}")
