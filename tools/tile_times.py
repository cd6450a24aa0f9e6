"""Per-tile times of one pass (MP_TILETIME build): which tile bounds each
round, and how its sweep splits into waits, hot and cold work.

  python -c "from paper_1901_10084_b200 import _native; _native.build(variant='tt', defines=['MP_TILETIME'])"
  MP_LIB_VARIANT=tt python tools/tile_times.py --config 3 --passes 4 [--dump out.npz]
"""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_10084_b200 import _native, instances  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession  # noqa: E402

R, T, B, REC = 256, 128, 8, 16
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--passes", type=int, default=4)
ap.add_argument("--dump", default="")
ap.add_argument("--show", type=int, default=40)
a = ap.parse_args()
inst = instances.config_instance(a.config)
s = DeviceSession(inst, "tiled", 40)
L = _native.load()
s.run(a.passes - 1)
ns = R * T * B * REC
out = (ctypes.c_uint64 * ns)()
L.mp_trace(s._h, 1, None, 0)
st = s.run(1)[0]
L.mp_trace(s._h, 1, out, ns)
L.mp_trace(s._h, 0, None, 0)
s.close()
d = np.frombuffer(out, dtype=np.uint64).reshape(R, T, B, REC).astype(np.int64)
if a.dump:
    np.savez_compressed(a.dump, d=d)
have = d[:, :, :, 12] > 0
nr = int(have.any(axis=(1, 2)).sum())
print(f"config {a.config}: {nr} rounds traced; pass metric time {st.metric_ms if hasattr(st, 'metric_ms') else ''}")
tot_round = 0
fam = np.zeros(2)
for r in range(nr):
    m = have[r]
    t0 = d[r][..., 0][m].min()
    t3 = d[r][..., 3][m].max()
    span = (t3 - t0) / 1e3
    tot_round += span
    # the tile finishing last
    ends = np.where(m, d[r][..., 3], 0).max(axis=1)
    tl = int(np.argmax(ends))
    rec = d[r, tl]
    bands = np.where(have[r, tl])[0]
    ilo, z = int(rec[bands[0], 12]) - 1, int(rec[bands[0], 13])
    C = int(rec[bands[0], 14])
    pro = (rec[bands, 1] - rec[bands, 0]).max() / 1e3
    swp = (rec[bands, 2] - rec[bands, 1]).max() / 1e3
    epi = (rec[bands, 3] - rec[bands, 2]).max() / 1e3
    cyc = rec[bands, 4:11].sum(axis=0)
    tc = max(cyc[0] + cyc[1] + cyc[2] + cyc[3] + cyc[4], 1)
    fam[0 if ilo <= 0 or r < nr // 2 else 1] += span
    if r < a.show or r % 10 == 0:
        print(f"r{r:3d} tiles {int(m.any(axis=1).sum()):3d} span {span:8.1f}us | last tile ({ilo},{z}) C={C} "
              f"pro {pro:6.1f} sweep {swp:8.1f} epi {epi:6.1f} | pred {cyc[0]/tc:4.0%} ring {cyc[1]/tc:4.0%} "
              f"hot {cyc[2]/tc:4.0%} cold {cyc[3]/tc:4.0%} rel {cyc[4]/tc:4.0%} levels {cyc[5]} coldb {cyc[6]}")
print(f"sum of round spans {tot_round/1e3:.2f} ms; first half {fam[0]/1e3:.2f} ms second {fam[1]/1e3:.2f} ms")
