"""Every BASELINE config at its full size against reference-order fixtures,
pass by pass, bit for bit (tests/golden/make_fullsize_golden.py).

* config 2 (n = 1000): all 100 passes against the UNMODIFIED reference;
* config 3 (n = 4000): all 200 passes against the C oracle, whose first 3
  passes equal the reference's own (tests/test_oracle_full.py), and passes
  1-3 directly against the reference fixture;
* configs 4 and 5 (n = 10000 / 18000): passes 1-3 against the C oracle.

Per pass: sha256 of x, f, the pair duals and the metric duals sorted by
reference key (ConstraintKey.encode), plus max violation, nnz and the
objectives (north_star: x within 1e-9 relative, objective within 1e-6 -- we
require x bitwise, the primal objective to 1e-12 and the dual objective,
a cancelling sum, to 1e-9).
"""

import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden
from paper_1901_10084_b200 import instances
from paper_1901_10084_b200.solver import DeviceSession

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def have(name):
    return os.path.exists(os.path.join(GOLDEN, name + ".npz"))


def replay(config, fixture, passes=None, every=1):
    g = golden(fixture)
    inst = instances.config_instance(config)
    assert sha(inst.d_flat) == str(g["dsha"]) and sha(inst.w_flat) == str(g["wsha"])
    passes = passes or int(g["passes"])
    sess = DeviceSession(inst, "tiled", int(g["b"]))
    for k in range(passes):
        st = sess.run(1)[0]
        assert st.max_violation == g["viol"][k], k
        assert st.nnz_metric == g["nnz"][k], k
        assert st.steps == g["steps"][k], k
        assert st.primal_objective == pytest.approx(g["primal"][k], rel=1e-12, abs=1e-12), k
        # The dual objective sums ~C(n,2) terms with heavy cancellation (b.y - ||.||^2/2):
        # the state is bitwise equal, only the summation order differs from numpy's
        # pairwise dot, which moves the last few of its ~12 significant digits.
        assert st.dual_objective == pytest.approx(g["dual"][k], rel=1e-9, abs=1e-9), k
        if (k + 1) % every and k + 1 != passes:
            continue
        x, f = sess.state()
        assert sha(x) == g["xsha"][k], f"x differs after pass {k + 1}"
        assert sha(f) == g["fsha"][k], f"f differs after pass {k + 1}"
        keys, vals, pd = sess.duals()
        o = np.argsort(keys, kind="stable")
        assert sha(keys[o]) == g["dkeys_sha"][k], f"dual keys differ after pass {k + 1}"
        assert sha(vals[o]) == g["dvals_sha"][k], f"dual values differ after pass {k + 1}"
        assert sha(pd) == g["pdsha"][k], f"pair duals differ after pass {k + 1}"
    if passes == int(g["passes"]):
        x, f = sess.state()
        idx = g["sample_idx"]
        assert np.array_equal(x[idx], g["sample_x_final"])
        assert np.array_equal(f[idx], g["sample_f_final"])
    sess.close()


def test_config2_all_100_passes_vs_reference():
    replay(2, "full_config2_n1000_p100_ref")


def test_config3_passes_1_3_vs_reference():
    replay(3, "full_config3_n4000_p3_ref")


@pytest.mark.skipif(not have("full_config3_n4000_p200_oracle"), reason="fixture not generated")
def test_config3_all_200_passes_vs_oracle():
    replay(3, "full_config3_n4000_p200_oracle")


@pytest.mark.skipif(not have("full_config4_n10000_p3_oracle"), reason="fixture not generated")
def test_config4_passes_1_3_vs_oracle():
    replay(4, "full_config4_n10000_p3_oracle")


@pytest.mark.skipif(not have("full_config5_n18000_p3_oracle"), reason="fixture not generated")
def test_config5_passes_1_3_vs_oracle():
    replay(5, "full_config5_n18000_p3_oracle")
