"""x/f hashes after P passes for one instance under several launch-shape
environment variants (each in its own process): equal hashes = same trajectory."""
import hashlib
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = r'''
import hashlib, os, sys, numpy as np
sys.path.insert(0, %r)
from paper_1901_10084_b200 import instances
from paper_1901_10084_b200.solver import DeviceSession
inst = instances.config_instance(%d, n=%d)
s = DeviceSession(inst, "tiled", 40)
st = s.run(%d)[-1]
x, f = s.state()
h = hashlib.sha1(x.tobytes() + f.tobytes()).hexdigest()[:12]
print(os.environ.get("MP_EXTRA", "default"), "nnz", st.nnz_metric, "hash", h, flush=True)
'''
cfg, n, passes = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
variants = [v for v in sys.argv[4:]] or ["", "MP_CLUSTER=1", "MP_CLUSTER=2", "MP_CLUSTER=4"]
for v in variants:
    e = dict(kv.split("=") for kv in v.split(",") if kv)
    env = dict(os.environ, **e, MP_EXTRA=v or "default")
    subprocess.run([sys.executable, "-c", CASE % (ROOT, cfg, n, passes)], env=env, timeout=900)
