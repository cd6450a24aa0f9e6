import time, sys, os
sys.path.insert(0, os.getcwd())
from paper_1901_10084_b200 import instances
from paper_1901_10084_b200.solver import DeviceSession
inst = instances.config_instance(1, n=300)
for b in (40, 64, 40):
    t = time.time()
    s = DeviceSession(inst, "tiled", b)
    print("b", b, "create", time.time() - t, flush=True)
    t = time.time(); s.run(1); print("  pass", time.time() - t, flush=True)
    s.close()
