import numpy as np, sys
sys.path.insert(0, '.')
from oracle import oracle
from paper_1901_10084_b200 import instances, core
from paper_1901_10084_b200.solver import DeviceSession
inst = instances.config_instance(1)
n = inst.n
s = DeviceSession(inst, "tiled", 40)
ref = oracle.OracleSolver(n, inst.d_flat, inst.w_flat, inst.epsilon, b=40, workers=4)
for k in range(3):
    st = s.run(1)[0]; rs = ref.run_pass()
    x, f = s.state(); rx, rf = ref.state()
    bad = np.nonzero(x != rx)[0]
    print("pass", k, "viol", st.max_violation, rs.max_violation, "ndiff", len(bad))
    if len(bad):
        iu = [core.pair_from_index(n, p) if hasattr(core, 'pair_from_index') else None for p in bad[:10]]
        # decode packed index
        res = []
        for p in bad[:20]:
            i = 0
            while p >= (n - 1 - i):
                p -= (n - 1 - i); i += 1
            res.append((i, i + 1 + p))
        print(res)
        break
