"""Per-batch timeline of the first tile of one round (MP_TIMELINE build).

  python -c "from paper_1901_10084_b200 import _native; _native.build(variant='tl', defines=['MP_TIMELINE'])"
  MP_LIB_VARIANT=tl MP_TL_ROUND=25 python tools/timeline.py --passes 4
"""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_10084_b200 import _native, instances  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession  # noqa: E402

TL_MAXB = 512
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--passes", type=int, default=4)
ap.add_argument("--dump", default="")
a = ap.parse_args()
inst = instances.config_instance(a.config)
s = DeviceSession(inst, "tiled", 40)
L = _native.load()
s.run(a.passes - 1)
ns = 8 * 16 * TL_MAXB * 8
out = (ctypes.c_uint64 * ns)()
L.mp_trace(s._h, 1, None, 0)
st = s.run(1)[0]
L.mp_trace(s._h, 1, out, ns)
v = np.frombuffer(out, dtype=np.uint64).reshape(8, 16, TL_MAXB, 8).astype(np.int64)
print(f"pass {st.wall_time*1e3:.3f} ms")
if a.dump:
    np.save(a.dump, v)
bands = [c for c in range(8) if v[c, 15, 0, 0] != 0]
if os.environ.get("TL_CRIT"):
    # per band: sweep length, max warp work, mean wait; the warp with max work
    for c in bands:
        hdr = v[c, 15, 0]
        works, waits, colds = [], [], []
        for w in range(15):
            r = v[c, w]
            nb = int(np.count_nonzero(r[:, 2]))
            if not nb:
                continue
            r = r[:nb]
            works.append(int((r[:, 2] - r[:, 1]).sum()))
            waits.append(int((r[:, 1] - r[:, 0]).sum()))
            colds.append(int((r[:, 3] == 1).sum()))
        print(f"band {c}: sweep {hdr[2]-hdr[0]:8d}  warps {len(works):2d}  max work {max(works):8d}  "
              f"mean work {int(np.mean(works)):8d}  mean wait {int(np.mean(waits)):8d}  cold max {max(colds)}")
    sys.exit(0)
if os.environ.get("TL_SUMMARY"):
    for c in bands:
        r = v[c, :15].reshape(-1, 8)
        r = r[r[:, 2] != 0]
        cold = (r[:, 3] & 1) == 1
        rc = r[cold]
        lk = rc[:, 4] & ((1 << 48) - 1)
        nl = rc[:, 4] >> 48
        ap = rc[:, 7] & 0xFFFFFFFF
        tot = rc[:, 7] >> 32
        ent = rc[:, 5] >> 32
        ld = rc[:, 5] & 0xFFFFFFFF
        st = rc[:, 6] & 0xFFFFFFFF
        slow = (rc[:, 6] >> 32) & 0xFFFF
        nsw = rc[:, 6] >> 48
        wt = rc[:, 3] >> 8
        print(f"band {c}: cold batches {cold.sum():4d}  cold batch {np.mean(rc[:,2]-rc[:,1]):6.0f}  in call "
              f"{tot.mean():6.0f} levels {nl.mean():.2f}  lookup {lk.mean():5.0f}  load+check {ld.mean():5.0f}  "
              f"step {st.mean():5.0f}  append {ap.mean():5.0f}  hot batch {np.mean(r[~cold,2]-r[~cold,1]):5.0f} | "
              f"entries {ent.mean():.2f} slow lookups {slow.mean():.2f} chunk switches {nsw.mean():.2f} "
              f"switch wait {wt.mean():.0f}")
    sys.exit(0)
for c in bands:
    hdr = v[c, 15, 0]
    hdr2 = v[c, 15, 1]
    t0 = hdr[0]
    print(f"band {c}: sweep {hdr[2]-hdr[0]} cyc, gtimer {(hdr[3]-hdr[1])} ns, prologue {hdr2[1]-hdr2[0]} cyc, "
          f"start gtimer offset {hdr[1]-v[bands[0],15,0,1]} ns")
    for w in range(15):
        r = v[c, w]
        nb = int(np.count_nonzero(r[:, 2]))
        if nb == 0:
            continue
        r = r[:nb]
        wait = (r[:, 1] - r[:, 0]).sum()
        work = (r[:, 2] - r[:, 1]).sum()
        cold = (r[:, 3] & 1) == 1
        gaps = r[1:, 0] - r[:-1, 2]
        if cold.any():
            rc = r[cold]
            extra = (f" | per cold batch: levels {rc[:,4].mean():.2f} lookup {rc[:,5].mean():.0f} "
                     f"math {rc[:,6].mean():.0f} rest {rc[:,7].mean():.0f}")
        else:
            extra = ""
        print(f"  w{w:2d} batches {nb:3d} first {r[0,0]-t0:7d} last {r[-1,2]-t0:8d} wait {wait:8d} "
              f"work {work:8d} (hot {(r[~cold,2]-r[~cold,1]).mean():6.0f}/batch, cold {cold.sum():3d} x "
              f"{(r[cold,2]-r[cold,1]).mean() if cold.any() else 0:6.0f}) gap {gaps.mean() if len(gaps) else 0:.0f}{extra}")
s.close()
