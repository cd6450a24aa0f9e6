"""Small fixed workload for ncu: W untimed passes then K passes of a config."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_10084_b200 import instances  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--b", type=int, default=40)
ap.add_argument("--passes", type=int, default=4)
a = ap.parse_args()
inst = instances.config_instance(a.config, n=a.n)
s = DeviceSession(inst, "tiled", a.b)
for st in s.run(a.passes):
    print(st.pass_index, st.wall_time, st.nnz_metric, st.max_violation)
s.close()
