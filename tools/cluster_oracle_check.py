"""Device vs oracle per forced cluster size (MP_CLUSTER) at sizes where the
j-rings wrap; prints the first differing pass per case."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = r'''
import os, sys, numpy as np
sys.path.insert(0, %r)
from oracle import oracle
from paper_1901_10084_b200 import instances
from paper_1901_10084_b200.solver import DeviceSession
cfg, n, passes = %d, %d, %d
inst = instances.config_instance(cfg, n=n)
s = DeviceSession(inst, "tiled", 40)
o = oracle.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, b=40, workers=os.cpu_count())
bad = None
for p in range(passes):
    st = s.run(1)[0]; rs = o.run_pass()
    x, f = s.state(); rx, rf = o.state()
    nd = int(np.sum(x != rx))
    if nd and bad is None: bad = (p, nd, float(np.max(np.abs(x - rx))))
print("cfg", cfg, "n", n, "MP_CLUSTER", os.environ.get("MP_CLUSTER"), "env", os.environ.get("MP_EXTRA", ""),
      "nnz", st.nnz_metric, "->", "OK" if bad is None else "DIFF first pass %%d: %%d entries, max %%.3g" %% bad, flush=True)
'''
cases = [(4, 600, 3), (2, 1000, 3), (4, 1200, 3)]
envs = [{"MP_CLUSTER": "1"}, {"MP_CLUSTER": "2"}, {"MP_CLUSTER": "8"}, {"MP_CLUSTER": "1", "MP_NO_TMA": "1"},
        {"MP_CLUSTER": "1", "MP_SLOTS": "1"}]
if len(sys.argv) > 1:
    envs = envs[:int(sys.argv[1])]
for cfg, n, passes in cases:
    for e in envs:
        env = dict(os.environ, **e, MP_EXTRA=",".join(f"{k}={v}" for k, v in e.items()))
        subprocess.run([sys.executable, "-c", CASE % (ROOT, cfg, n, passes)], env=env, timeout=600)
