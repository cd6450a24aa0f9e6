"""Pin the CPU oracle at the BASELINE configs' full sizes and check the
full-length fixtures (tests/golden/make_fullsize_golden.py) are consistent
with each other and with the instance generators.  CPU only.

* config 2 (n = 1000): the oracle replays the first passes of the
  reference's own 100-pass run bit for bit;
* config 3 (n = 4000): the oracle's 200-pass fixture begins with exactly the
  reference's passes 1-3 (both written by the generator script), so the
  remaining 197 oracle passes extend a pinned trajectory;
* projection.dykstra_step: the oracle's restatement equals the reference's
  single-row steps (tests/golden/steps.npz) bit for bit.
"""

import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden
from paper_1901_10084_b200 import instances

FIELDS = ("xsha", "fsha", "pdsha", "dkeys_sha", "dvals_sha", "viol", "nnz", "steps")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def have(name):
    return os.path.exists(os.path.join(GOLDEN, name + ".npz"))


def test_config2_instance_matches_fixture():
    g = golden("full_config2_n1000_p100_ref")
    inst = instances.config_instance(2)
    assert sha(inst.d_flat) == str(g["dsha"]) and sha(inst.w_flat) == str(g["wsha"])
    assert int(g["passes"]) == 100 == len(g["xsha"])
    assert str(g["source"]) == "reference"


def test_config2_oracle_replays_reference(oracle_lib):
    g = golden("full_config2_n1000_p100_ref")
    inst = instances.config_instance(2)
    o = oracle_lib.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, b=40,
                                workers=os.cpu_count() or 1)
    for k in range(8):
        st = o.run_pass()
        x, f = o.state()
        keys, vals = o.duals()
        ordr = np.argsort(keys, kind="stable")
        assert sha(x) == g["xsha"][k] and sha(f) == g["fsha"][k], k
        assert sha(o.pair_duals()) == g["pdsha"][k], k
        assert sha(keys[ordr]) == g["dkeys_sha"][k] and sha(vals[ordr]) == g["dvals_sha"][k], k
        assert st.max_violation == g["viol"][k] and st.steps == g["steps"][k], k
        assert st.primal_objective == pytest.approx(g["primal"][k], rel=1e-13)
    o.close()


@pytest.mark.skipif(not have("full_config3_n4000_p200_oracle"), reason="fixture not generated yet")
def test_config3_oracle_fixture_starts_with_reference_passes():
    ref = golden("full_config3_n4000_p3_ref")
    orc = golden("full_config3_n4000_p200_oracle")
    assert str(ref["dsha"]) == str(orc["dsha"]) and str(ref["wsha"]) == str(orc["wsha"])
    assert str(ref["source"]) == "reference" and str(orc["source"]) == "oracle"
    assert len(orc["xsha"]) == 200
    for fld in FIELDS:
        assert list(ref[fld][:3]) == list(orc[fld][:3]), fld
    np.testing.assert_allclose(ref["primal"], orc["primal"][:3], rtol=1e-13)


def test_config3_instance_matches_fixture():
    g = golden("full_config3_n4000_p3_ref")
    inst = instances.config_instance(3)
    assert sha(inst.d_flat) == str(g["dsha"]) and sha(inst.w_flat) == str(g["wsha"])


def test_dykstra_step_restatement_matches_reference():
    from oracle import oracle
    g = golden("steps")
    for c in range(6):
        n, eps = int(g[f"c{c}_n"]), float(g[f"c{c}_eps"])
        D = g[f"c{c}_D"]
        d_flat = D[np.triu_indices(n, 1)]
        x, f = g[f"c{c}_x0"].copy(), g[f"c{c}_f0"].copy()
        rx, rf = g[f"c{c}_regx"], g[f"c{c}_regf"]
        for t, (kind, i, j, k) in enumerate(g[f"c{c}_keys"]):
            th, ch = oracle.dykstra_step_py(x, f, rx, rf, eps, n, int(kind), int(i), int(j),
                                            int(k), float(g[f"c{c}_y"][t]), d_flat)
            assert th == g[f"c{c}_theta"][t] and ch == bool(g[f"c{c}_changed"][t]), (c, t)
        assert np.array_equal(x, g[f"c{c}_x1"]) and np.array_equal(f, g[f"c{c}_f1"]), c
