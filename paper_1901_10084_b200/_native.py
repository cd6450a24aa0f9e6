"""ctypes binding of ``libmetricproj_b200.so`` (the C ABI in
``include/metricproj_b200.h``).

There is deliberately no fallback: if the shared library is missing, or the
process has no sm_100 device, every compute entry raises.  ``build()``
compiles the library in place with nvcc for ``sm_100a``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_DIR = os.path.join(PKG, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libmetricproj_b200.so")
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")

MP_OK = 0
MP_ERR_ARG = 1
MP_ERR_CUDA = 2
MP_ERR_OOM = 3
MP_ERR_NONFINITE = 4
MP_ERR_UNSUPPORTED = 5

SCHEDULE_CODES = {"serial": 0, "diagonal": 1, "tiled": 2}
MP_FLAG_TIME_ROUNDS = 1

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "-Xcompiler", "-fPIC", "-shared",
]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cuh", ".h", ".cpp")))


KNOBS_VARIANT = "knobs"  # the product library + the experiment switches (-DMP_KNOBS)


def lib_path(variant: str = "") -> str:
    return LIB_PATH if not variant else os.path.join(LIB_DIR, f"libmetricproj_b200_{variant}.so")


def _build_cmd(out, defines):
    nvcc = os.environ.get("NVCC", "nvcc")
    if not os.path.exists(nvcc) and os.path.exists("/usr/local/cuda/bin/nvcc"):
        nvcc = "/usr/local/cuda/bin/nvcc"
    return [nvcc, *NVCC_FLAGS, *(f"-D{d}" for d in defines), "-I", INCLUDE, "-I", CSRC,
            "-o", out + ".tmp", os.path.join(CSRC, "mp_solver.cu"), "-ldl"]


def _stale(out, force):
    deps = sources() + [os.path.join(INCLUDE, "metricproj_b200.h")]
    return (force or not os.path.exists(out)
            or os.path.getmtime(out) < max(os.path.getmtime(p) for p in deps))


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """Compile csrc/ into _lib/libmetricproj_b200.so (sm_100a).  A named
    ``variant`` with extra ``defines`` (e.g. MP_TRACE) builds a side library
    for diagnostics, selected at load time with MP_LIB_VARIANT or
    ``use_variant``; every variant also gets -DMP_KNOBS (the experiment
    switches the product library does not have)."""
    os.makedirs(LIB_DIR, exist_ok=True)
    out = lib_path(variant)
    if not _stale(out, force):
        return out
    if variant:
        defines = tuple(dict.fromkeys(("MP_KNOBS", *defines)))
    cmd = _build_cmd(out, defines)
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


def build_all(force: bool = False, verbose: bool = False):
    """The product library and the ``knobs`` variant (shape-forcing tests),
    compiled side by side."""
    os.makedirs(LIB_DIR, exist_ok=True)
    jobs = []
    for variant, defines in (("", ()), (KNOBS_VARIANT, ("MP_KNOBS",))):
        out = lib_path(variant)
        if _stale(out, force):
            cmd = _build_cmd(out, defines)
            if verbose:
                print(" ".join(cmd))
            jobs.append((out, subprocess.Popen(cmd)))
    for out, proc in jobs:
        if proc.wait() != 0:
            raise subprocess.CalledProcessError(proc.returncode, "nvcc")
        os.replace(out + ".tmp", out)
    return [lib_path(""), lib_path(KNOBS_VARIANT)]


class MPInstance(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64),
                ("d_flat", ctypes.POINTER(ctypes.c_double)),
                ("w_flat", ctypes.POINTER(ctypes.c_double)),
                ("reg_x", ctypes.POINTER(ctypes.c_double)),
                ("reg_f", ctypes.POINTER(ctypes.c_double)),
                ("epsilon", ctypes.c_double)]


class MPConfig(ctypes.Structure):
    _fields_ = [("schedule_kind", ctypes.c_int32),
                ("tile_b", ctypes.c_int32),
                ("device", ctypes.c_int32),
                ("flags", ctypes.c_uint32)]


class MPPassStats(ctypes.Structure):
    _fields_ = [("pass_index", ctypes.c_int64),
                ("steps", ctypes.c_int64),
                ("nnz_metric", ctypes.c_int64),
                ("primal_objective", ctypes.c_double),
                ("dual_objective", ctypes.c_double),
                ("duality_gap", ctypes.c_double),
                ("max_violation", ctypes.c_double),
                ("wall_time", ctypes.c_double)]


# every symbol include/metricproj_b200.h declares
EXPORTS = ("mp_create", "mp_run_passes", "mp_get_state", "mp_set_state", "mp_dual_count",
           "mp_get_duals", "mp_set_duals", "mp_state_max_violation", "mp_get_timing",
           "mp_trace", "mp_flush_l2", "mp_destroy", "mp_max_violation", "mp_check_division",
           "mp_get_duals_ranked", "mp_shard_plan", "mp_nccl_unique_id", "mp_shard",
           "mp_shard_volume", "mp_shard_route", "mp_group_run_passes", "mp_cc_instance", "mp_accumulate_aty", "mp_dykstra_steps",
           "mp_last_error", "mp_version")

_libs = {}                                        # variant -> loaded library
_variant = os.environ.get("MP_LIB_VARIANT", "")   # the variant load() returns


class use_variant:
    """``with use_variant("knobs"):`` -- every call inside goes to that library
    variant (sessions must be created and closed inside the block)."""

    def __init__(self, variant):
        self.variant = variant

    def __enter__(self):
        global _variant
        self.prev, _variant = _variant, self.variant
        return self

    def __exit__(self, *exc):
        global _variant
        _variant = self.prev
        return False


def load():
    """Load the shared library (raises if it has not been built)."""
    variant = _variant
    if variant in _libs:
        return _libs[variant]
    path = lib_path(variant)
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: run paper_1901_10084_b200._native.build_all() "
            "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(path)
    if variant and variant != KNOBS_VARIANT:  # a diagnostic build may predate some entry points
        class _Tolerant:
            def __init__(self, lib):
                self.__dict__["_lib"] = lib

            def __getattr__(self, name):
                try:
                    return getattr(self._lib, name)
                except AttributeError:
                    return ctypes.CFUNCTYPE(ctypes.c_int)(lambda *a: 0)

            def __setattr__(self, name, value):
                setattr(self._lib, name, value)
        L = _Tolerant(L)
    P = ctypes.c_void_p
    D = ctypes.POINTER(ctypes.c_double)
    I = ctypes.POINTER(ctypes.c_int64)
    L.mp_create.argtypes = [ctypes.POINTER(MPInstance), ctypes.POINTER(MPConfig),
                            ctypes.POINTER(P)]
    L.mp_run_passes.argtypes = [P, ctypes.c_int32, ctypes.POINTER(MPPassStats)]
    L.mp_get_state.argtypes = [P, D, D]
    L.mp_set_state.argtypes = [P, D, D]
    L.mp_dual_count.restype = ctypes.c_int64
    L.mp_dual_count.argtypes = [P]
    L.mp_get_duals.argtypes = [P, I, D, D]
    L.mp_set_duals.argtypes = [P, ctypes.c_int64, I, D, D]
    L.mp_state_max_violation.argtypes = [P, D]
    L.mp_get_timing.argtypes = [P, D, D, I]
    L.mp_flush_l2.argtypes = [P]
    L.mp_trace.argtypes = [P, ctypes.c_int32, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int32]
    L.mp_trace.restype = ctypes.c_int
    L.mp_destroy.restype = None
    L.mp_destroy.argtypes = [P]
    L.mp_max_violation.argtypes = [ctypes.c_int64, D, D, D, D]
    L.mp_accumulate_aty.argtypes = [ctypes.c_int64, ctypes.c_int64, I, D, D, D, D]
    L.mp_accumulate_aty.restype = ctypes.c_int
    L.mp_check_division.argtypes = [ctypes.c_double, ctypes.c_int64, ctypes.c_uint64, I]
    L.mp_check_division.restype = ctypes.c_int
    L.mp_get_duals_ranked.argtypes = [P, I, D, I]
    L.mp_shard_plan.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                ctypes.POINTER(ctypes.c_int32), I]
    L.mp_nccl_unique_id.argtypes = [ctypes.c_char_p]
    L.mp_shard.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.c_char_p]
    L.mp_shard_volume.argtypes = [P, I, I]
    L.mp_shard_route.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, I, I]
    L.mp_group_run_passes.argtypes = [ctypes.POINTER(P), ctypes.c_int32, ctypes.c_int32,
                                      ctypes.POINTER(MPPassStats)]
    L.mp_cc_instance.argtypes = [ctypes.c_int64, I, ctypes.POINTER(ctypes.c_int32), ctypes.c_double,
                                 ctypes.c_double, ctypes.c_double, D, D]
    L.mp_dykstra_steps.argtypes = [ctypes.c_int64, ctypes.POINTER(ctypes.c_int32), I, D, D, D, D,
                                   ctypes.c_double, ctypes.c_int64, D, D,
                                   ctypes.POINTER(ctypes.c_int32)]
    for name in ("mp_get_duals_ranked", "mp_shard_plan", "mp_nccl_unique_id", "mp_shard",
                 "mp_shard_volume", "mp_shard_route",
                 "mp_group_run_passes", "mp_cc_instance", "mp_dykstra_steps"):
        getattr(L, name).restype = ctypes.c_int
    L.mp_last_error.restype = ctypes.c_char_p
    L.mp_version.restype = ctypes.c_char_p
    for name in ("mp_create", "mp_run_passes", "mp_get_state", "mp_set_state", "mp_get_duals",
                 "mp_set_duals", "mp_state_max_violation", "mp_get_timing", "mp_flush_l2",
                 "mp_max_violation"):
        getattr(L, name).restype = ctypes.c_int
    _libs[variant] = L
    return L


def last_error() -> str:
    return load().mp_last_error().decode(errors="replace")


def dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def iptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


class NativeError(RuntimeError):
    def __init__(self, code, message):
        super().__init__(message)
        self.code = code


def check(code: int, what: str):
    if code != MP_OK:
        raise NativeError(code, f"{what}: {last_error()}")
