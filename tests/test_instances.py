"""Seeded synthetic instances for BASELINE.json's configs.  CPU only."""

import hashlib

import numpy as np

from conftest import golden
from paper_1901_10084_b200 import core, instances


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_generators_are_deterministic_and_match_goldens():
    g1 = golden("config1_n100_b40")
    a = instances.config_instance(1)
    b = instances.config_instance(1)
    assert np.array_equal(a.d_flat, b.d_flat)
    assert sha(a.d_flat) == str(g1["dsha"]) and sha(a.w_flat) == str(g1["wsha"])
    g2 = golden("config2_n1000_b40_p4")
    assert sha(instances.config_instance(2).d_flat) == str(g2["dsha"])


def test_config_shapes():
    for cfg, (n, eps) in {1: (100, 0.2), 2: (1000, 0.2)}.items():
        inst = instances.config_instance(cfg)
        assert inst.n == n and inst.epsilon == eps
        assert set(np.unique(inst.d_flat)) <= {0.0, 1.0}
        assert np.all(inst.w_flat > 0)
    # planted partition: dense inside clusters, sparse across
    inst = instances.config_instance(1)
    i, j = np.triu_indices(100, 1)
    same = (i // 25) == (j // 25)
    assert (1 - inst.d_flat[same]).mean() > 0.6 and (1 - inst.d_flat[~same]).mean() < 0.2
    # G(n, 0.01): mean degree ~ 10
    A = 1 - instances.config_instance(2).d_flat
    assert 8 < 2 * A.sum() / 1000 < 12


def test_chung_lu_weights_and_lambda():
    inst = instances.config_instance(3, n=400)
    A = 1 - inst.d_flat
    assert np.all(inst.w_flat[A == 0] == 0.5) and np.all(inst.w_flat[A == 1] == 1.0)
    assert inst.epsilon == 0.1
    deg = np.zeros(400)
    i, j = np.triu_indices(400, 1)
    np.add.at(deg, i, A)
    np.add.at(deg, j, A)
    assert deg[:10].mean() > deg[-100:].mean()  # power-law head


def test_random_instance_is_valid_problem():
    inst = instances.random_instance(9, seed=4)
    assert inst.npairs == core.pair_count(9)
    assert np.all((inst.w_flat >= 0.5) & (inst.w_flat <= 1.5))
