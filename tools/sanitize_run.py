"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
a few passes of a config-shaped instance, checked bitwise against the CPU
oracle so a tool run also shows the results are unchanged under it.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py --n 150 --passes 3
  (launch shapes through the library's environment switches: MP_FORCE_C,
   MP_NO_TMA, MP_NO_DF, MP_DF_C, MP_WAVE_C ...)
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402  (the checker)
from paper_1901_10084_b200 import instances  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--n", type=int, default=150)
ap.add_argument("--b", type=int, default=40)
ap.add_argument("--passes", type=int, default=3)
a = ap.parse_args()
inst = instances.config_instance(a.config, n=a.n)
s = DeviceSession(inst, "tiled", a.b)
ref = oracle.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, b=a.b)
for k in range(a.passes):
    s.run(1)
    ref.run_pass()
x, f = s.state()
rx, rf = ref.state()
ok = np.array_equal(x, rx) and np.array_equal(f, rf)
keys, vals, _ = s.duals()
rk, rv = ref.duals()
ok = ok and np.array_equal(np.sort(keys), np.sort(rk))
print(f"n={inst.n} b={a.b} passes={a.passes} env={{{', '.join(k + '=' + v for k, v in os.environ.items() if k.startswith('MP_'))}}}"
      f" bitwise_vs_oracle={ok}")
s.close()
ref.close()
sys.exit(0 if ok else 1)
