"""Per-phase cycle breakdown of the tile kernel for one pass (mp_trace)."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_10084_b200 import _native, instances  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession  # noqa: E402

NAMES = ["pred_wait", "ring_wait", "hot", "cold", "release", "levels", "cold_calls", "-",
         "prologue", "loop", "epilogue", "epi_blocks", "ctas", "c_lookup", "c_math", "c_append"]
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--b", type=int, default=40)
ap.add_argument("--passes", type=int, default=4)
a = ap.parse_args()
inst = instances.config_instance(a.config, n=a.n)
s = DeviceSession(inst, "tiled", a.b)
L = _native.load()
s.run(a.passes - 1)
out = (ctypes.c_uint64 * 16)()
L.mp_trace(s._h, 1, None, 0)
st = s.run(1)[0]
L.mp_trace(s._h, 1, out, 16)
v = list(out)
print(f"pass time {st.wall_time*1e3:.3f} ms")
wl = v[5] or 1
for i, nm in enumerate(NAMES):
    if nm == "-":
        continue
    extra = f"  ({v[i]/wl:.1f} cyc per warp-level)" if i < 5 else ""
    print(f"{nm:12s} {v[i]:>16d}{extra}")
print(f"cold fraction of warp-levels: {v[6]/wl:.4f}")
ctas = v[12] or 1
print(f"per CTA: prologue {v[8]/ctas:.0f}  loop {v[9]/ctas:.0f}  epilogue {v[10]/ctas:.0f} cycles")
