"""Small tiled solve (n=13, b=4) for debugging under compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_10084_b200 import instances  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 13
b = int(sys.argv[2]) if len(sys.argv) > 2 else 4
inst = instances.random_instance(n, seed=5)
s = DeviceSession(inst, "tiled", b)
print(s.run(3)[-1])
