import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


@pytest.fixture(scope="session")
def small_golden():
    return golden("small_cases")


@pytest.fixture(scope="session")
def config1_golden():
    return golden("config1_n100_b40")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import oracle
    oracle.build()
    return oracle


@pytest.fixture
def knobs(monkeypatch):
    """Shape-forcing tests: the experiment switches (MP_CLUSTER, MP_FORCE_C,
    MP_NO_TMA, MP_POOL_CAP0, ...) exist only in the ``knobs`` library variant
    (-DMP_KNOBS); the product library ignores them.  Yields the monkeypatch
    object, with every native call of the test routed to that variant."""
    from paper_1901_10084_b200 import _native
    # (a diagnostic variant selected with MP_LIB_VARIANT -- e.g. the checked
    # build -- has the switches too and stays in place)
    with _native.use_variant(os.environ.get("MP_LIB_VARIANT") or _native.KNOBS_VARIANT):
        yield monkeypatch
