"""Large-config checks: device vs oracle for a few passes at full size, and timing."""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402
from paper_1901_10084_b200 import instances  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--passes", type=int, default=3)
ap.add_argument("--oracle", action="store_true")
ap.add_argument("--threads", type=int, default=os.cpu_count())
a = ap.parse_args()
t0 = time.time()
inst = instances.config_instance(a.config)
print(f"config {a.config} n={inst.n} generated in {time.time()-t0:.1f}s", flush=True)
t0 = time.time()
s = DeviceSession(inst, "tiled", 40)
print(f"session created in {time.time()-t0:.1f}s", flush=True)
ref = oracle.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, b=40,
                          workers=a.threads) if a.oracle else None
for k in range(a.passes):
    st = s.run(1)[0]
    line = f"pass {k}: {st.wall_time*1e3:.1f} ms  nnz={st.nnz_metric}  viol={st.max_violation:.6g}  primal={st.primal_objective:.10g}"
    if ref is not None:
        t1 = time.time()
        rs = ref.run_pass()
        x, f = s.state()
        rx, rf = ref.state()
        rk, rv = ref.duals()
        same = np.array_equal(x, rx) and np.array_equal(f, rf)
        line += f" | oracle {time.time()-t1:.1f}s bitwise_x={same} viol_eq={st.max_violation == rs.max_violation} nnz_eq={st.nnz_metric == len(rk)}"
    print(line, flush=True)
