"""Stored metric duals per row i (and per (row, column-band)) after a few passes: where the
exact steps of a config concentrate (the hub rows of Chung-Lu instances)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_10084_b200 import core, instances  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 6
inst = instances.config_instance(cfg)
s = DeviceSession(inst, "tiled", 40)
s.run(passes)
keys, vals, _ = s.duals()
n = inst.n
i, j, k, kind = core.decode_keys(keys, n)
cnt = np.bincount(i, minlength=n)
tot = cnt.sum()
print(f"config {cfg}: {tot} duals after {passes} passes")
# work per row of the hub tile's rows 1..40 (the first family's row band 1)
for r in list(range(0, 12)) + [20, 40, 41, 80, 120, 400, 1000]:
    print(f"row {r:5d}: {cnt[r]:8d} ({cnt[r] / tot:.3%})  rows 1..r: {cnt[1:r + 1].sum() / tot:.3%}")
np.save("gpurun_out/row_duals_c%d.npy" % cfg, cnt)
band = cnt[1:41].astype(float)
print("rows 1..40 share of the band:", np.round(band / band.sum(), 3).tolist())
