"""The C-ABI library builds for sm_100a, loads, and exports every symbol the
header declares; without a GPU it fails loudly (no CPU fallback).  CPU only."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1901_10084_b200 import _native, instances

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "metricproj_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mp_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert set(syms) == set(_native.EXPORTS)
    for s in ("mp_create", "mp_run_passes", "mp_get_state", "mp_get_duals", "mp_max_violation"):
        assert s in syms


def test_library_builds_and_exports_every_symbol():
    path = _native.build()
    lib = ctypes.CDLL(path)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    L = _native.load()
    assert b"sm_100a" in L.mp_version()


def test_product_library_has_no_experiment_switches():
    """The launch-shape / timing switches live in the ``knobs`` variant only
    (-DMP_KNOBS); the product library reads MP_NCCL_LIB and MP_VERBOSE."""
    prod, knobs = _native.build_all()
    names = (b"MP_CLUSTER", b"MP_FORCE_C", b"MP_NO_TMA", b"MP_POOL_CAP0", b"MP_MIN_C", b"MP_NO_DF",
             b"MP_SLOTS", b"MP_HUB_C")
    blob = open(prod, "rb").read()
    assert not [n for n in names if n in blob]
    assert b"MP_NCCL_LIB" in blob and b"MP_VERBOSE" in blob
    kblob = open(knobs, "rb").read()
    assert all(n in kblob for n in names)
    lib = ctypes.CDLL(knobs)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    with _native.use_variant(_native.KNOBS_VARIANT):
        assert b"+knobs" in _native.load().mp_version()
    assert b"+knobs" not in _native.load().mp_version()


def test_sass_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.build()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu():
    from paper_1901_10084_b200.solver import DeviceSession
    inst = instances.random_instance(6, seed=1)
    with pytest.raises(_native.NativeError) as e:
        DeviceSession(inst)
    assert e.value.code == _native.MP_ERR_CUDA
    st = np.zeros(inst.npairs)
    from paper_1901_10084_b200 import core
    with pytest.raises(_native.NativeError):
        core.max_violation(inst, core.PrimalState(inst.n, st, st))


def test_argument_validation_before_device():
    """Bad arguments are rejected with MP_ERR_ARG (ValueError in Python)."""
    L = _native.load()
    d = np.zeros(3)
    inst = _native.MPInstance(3, _native.dptr(d), _native.dptr(d), None, None, 0.0)
    cfg = _native.MPConfig(2, 40, 0, 0)
    h = ctypes.c_void_p()
    assert L.mp_create(ctypes.byref(inst), ctypes.byref(cfg), ctypes.byref(h)) == _native.MP_ERR_ARG
    inst = _native.MPInstance(2, _native.dptr(d), _native.dptr(d), None, None, 0.5)
    assert L.mp_create(ctypes.byref(inst), ctypes.byref(cfg), ctypes.byref(h)) == _native.MP_ERR_ARG
    inst = _native.MPInstance(5, _native.dptr(np.zeros(10)), _native.dptr(np.ones(10)), None, None, 0.5)
    cfg = _native.MPConfig(7, 40, 0, 0)
    assert L.mp_create(ctypes.byref(inst), ctypes.byref(cfg), ctypes.byref(h)) == _native.MP_ERR_ARG
