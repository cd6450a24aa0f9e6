"""Where does a sharded group's x differ from a single session's?"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_10084_b200 import distributed, instances  # noqa: E402
from paper_1901_10084_b200.solver import DeviceSession  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--world", type=int, default=2)
ap.add_argument("--passes", type=int, default=2)
a = ap.parse_args()
inst = instances.config_instance(a.config, n=a.n)
n = inst.n
iu = np.triu_indices(n, 1)
single = DeviceSession(inst, "tiled", 40)
grp = distributed.LocalShardGroup(inst, a.world, 40)
for p in range(a.passes):
    s = single.run(1)[0]
    g = grp.run(1)[0]
    x, f = single.state()
    print(f"pass {p}: single nnz={s.nnz_metric} viol={s.max_violation} primal={s.primal_objective!r}; "
          f"group nnz={g.nnz_metric} viol={g.max_violation} primal={g.primal_objective!r}", flush=True)
    for r in range(a.world):
        gx, gf = grp.state(r)
        dx = np.nonzero(gx != x)[0]
        df = np.nonzero(gf != f)[0]
        print(f"  rank {r}: {len(dx)} x differ, {len(df)} f differ", flush=True)
        if len(dx):
            ii, jj = iu[0][dx], iu[1][dx]
            print("   i range", ii.min(), ii.max(), " j range", jj.min(), jj.max())
            for t in range(min(12, len(dx))):
                q = dx[t]
                print(f"   ({ii[t]},{jj[t]}) single={x[q]!r} rank={gx[q]!r}")
            print("   max |dx| =", np.max(np.abs(gx[dx] - x[dx])))
