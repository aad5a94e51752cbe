"""ctypes binding of libsbf.so (the C ABI in include/sbf.h).

The library is the only compute path: if it is missing this module raises
on first use (no CPU fallback exists anywhere in the package).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import InvalidParameterError, ShiftBFError, UnsupportedOrderError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SBF_LIB", os.path.join(_HERE, "libsbf.so"))

SBF_OK, SBF_ERR_INVALID, SBF_ERR_UNSUPPORTED, SBF_ERR_CUDA, SBF_ERR_WORKSPACE = 0, 2, 4, 5, 6
SBF_F32, SBF_F64 = 0, 1
STAGE_F32, STAGE_F64, STAGE_U8, STAGE_U16, STAGE_I16 = 0, 1, 2, 3, 4
RULES = {"auto": 0, "exact": 1, "chernoff": 2, "none": 3}
SPATIAL_ITERATED, SPATIAL_BOX, SPATIAL_FIR = 0, 1, 2
PREC_FP32, PREC_HDR, PREC_AUTO = 0, 1, 2
PLAN_N_AMBIGUOUS, PLAN_EXACT_BIGINT, PLAN_TERMS_TRUNCATED, PLAN_NEEDS_HDR = 1, 2, 4, 8


class SbfPlan(C.Structure):
    _fields_ = [("T", C.c_double), ("sigma_r", C.c_double), ("epsilon", C.c_double),
                ("gamma", C.c_double), ("N", C.c_int32), ("M", C.c_int32), ("K", C.c_int32),
                ("K_eval", C.c_int32), ("flags", C.c_int32), ("status", C.c_int32),
                ("pad0", C.c_int32), ("pad1", C.c_int32)]


class SbfTerm(C.Structure):
    _fields_ = [("scale", C.c_double), ("freq", C.c_double), ("turns", C.c_double),
                ("index", C.c_int32), ("pad", C.c_int32)]


class SbfSpatial(C.Structure):
    _fields_ = [("mode", C.c_int32), ("passes", C.c_int32), ("r", C.c_int32), ("pad", C.c_int32),
                ("alpha", C.c_double), ("sigma_s", C.c_double)]


assert C.sizeof(SbfPlan) == 64 and C.sizeof(SbfTerm) == 32 and C.sizeof(SbfSpatial) == 32

# name -> (restype, argtypes)
_vp, _i64, _dbl, _int = C.c_void_p, C.c_int64, C.c_double, C.c_int
_SIGS = {
    "sbf_abi_version": (_int, []),
    "sbf_last_error": (C.c_char_p, []),
    "sbf_device_count": (_int, [C.POINTER(_int)]),
    "sbf_num_specialisations": (_int, []),
    "sbf_specialisation": (_int, [_int, C.POINTER(_int), C.POINTER(_int), C.POINTER(_int)]),
    "sbf_filter_geometry": (_int, [_i64, _i64, C.POINTER(SbfSpatial), _int, C.POINTER(_int)]),
    "sbf_extended_box_params": (_int, [_dbl, _int, C.POINTER(_int), C.POINTER(_dbl)]),
    "sbf_support_radius": (_int, [C.POINTER(SbfSpatial), C.POINTER(_int)]),
    "sbf_order_threshold": (_int, [_dbl, _dbl, C.POINTER(_int)]),
    "sbf_truncation_index_exact": (_int, [_int, _dbl, C.POINTER(_int)]),
    "sbf_truncation_index_exact_bigint": (_int, [_int, _dbl, C.POINTER(_int)]),
    "sbf_truncation_index_chernoff": (_int, [_int, _dbl, _dbl, C.POINTER(_int)]),
    "sbf_binomial_weights": (_int, [_int, _int, _int, _vp]),
    "sbf_brute_force_T": (_int, [_vp, _int, _i64, _i64, _i64, _int, C.POINTER(_dbl), _vp]),
    "sbf_select_plan": (_int, [_dbl, _dbl, _dbl, _int, _dbl, C.POINTER(SbfPlan)]),
    "sbf_local_range_workspace": (C.c_size_t, [_i64, _i64, _int]),
    "sbf_local_range": (_int, [_vp, _int, _i64, _i64, _i64, _int, _i64, _i64, _vp, _vp, _vp,
                               C.c_size_t, _vp]),
    "sbf_plan_device": (_int, [_vp, _int, _dbl, _dbl, _dbl, _int, _dbl, _vp, _vp, _int, _vp]),
    "sbf_plan_device_forced": (_int, [_vp, _int, _dbl, _dbl, _dbl, _int, _dbl, _int, _int, _vp, _vp,
                                      _int, _vp]),
    "sbf_filter_workspace": (C.c_size_t, [_i64, _i64, _i64, _int, C.POINTER(SbfSpatial), _int]),
    "sbf_filter": (_int, [_vp, _int, _i64, _i64, _i64, _i64, _i64, _i64, _i64,
                          C.POINTER(SbfSpatial), _vp, _vp, _vp, _int, _vp, _int, _vp, _vp,
                          C.c_size_t, _vp]),
    "sbf_shiftable_bf_workspace": (C.c_size_t, [_i64, _i64, _int, C.POINTER(SbfSpatial), _int,
                                                _int]),
    "sbf_shiftable_bf": (_int, [_vp, _int, _i64, _i64, C.POINTER(SbfSpatial), _int, _dbl, _dbl,
                                _dbl, _int, _dbl, _int, _vp, _int, _vp, _vp, _vp, _int, _vp,
                                C.c_size_t, _vp]),
    "sbf_shiftable_bf_host": (_int, [_vp, _i64, _i64, C.POINTER(SbfSpatial), _int, _dbl, _dbl,
                                     _dbl, _int, _dbl, _int, _vp, C.POINTER(SbfPlan),
                                     C.POINTER(C.c_ulonglong)]),
    "sbf_divide_with_fallback": (_int, [_vp, _vp, _vp, _i64, _vp, _vp, _vp]),
    "sbf_set_stage_mask": (_int, [_int]),
    "sbf_set_k3_events": (_int, [_vp, _vp]),
    "sbf_set_fused_epilogue": (_int, [_int]),
    "sbf_set_sweep_variant": (_int, [_int]),
    "sbf_pgm_decode": (_int, [_vp, _int, _i64, _vp, _vp]),
    "sbf_pgm_encode": (_int, [_vp, _int, _i64, _int, _vp, _vp]),
    "sbf_direct_bf": (_int, [_vp, _int, _i64, _i64, _i64, _int, _vp, _dbl, _int, _vp, _int, _vp]),
    "sbf_set_fp64_method": (_int, [_int]),
    "sbf_direct_nlm": (_int, [_vp, _int, _i64, _i64, _i64, _int, _vp, _int, _vp, _vp, _vp, _vp,
                              _vp, _vp, _vp, _int, _vp]),
    "sbf_direct_bf_expansion": (_int, [_vp, _int, _i64, _i64, _i64, _int, _vp, _vp, _vp, _int, _vp,
                                       _int, _vp]),
    "sbf_smooth": (_int, [_vp, _int, _i64, _i64, _i64, C.POINTER(SbfSpatial), _vp, _int, _vp]),
    "sbf_stage_h2d": (_int, [_vp, _int, _i64, _vp, _vp]),
    "sbf_set_split_min_radius": (_int, [_int]),
    "sbf_nlm_filter": (_int, [_vp, _int, _i64, _i64, _i64, C.POINTER(SbfSpatial), _int, _vp, _vp,
                              _int, _vp, _vp, _int, _vp, _vp]),
    "sbf_fp32_probe": (_int, [_int, _int, _int, _vp, _vp]),
}
EXPORTS = tuple(_SIGS)

_lock = threading.Lock()
_lib = None

# One filter call at a time per process.  Calls from several Python threads are
# serialised (kernels of different calls still overlap when they were enqueued
# on different streams by ONE thread, e.g. shiftable_bf_batch).  Without this
# lock tools/gpu/check_threads.py ended 3 of 6 whole-suite runs with a CUDA
# illegal memory access; with it 4 of 4 were clean (cause not found: DESIGN.md
# section 5).  SBF_SERIALISE_CALLS=0 removes it for experiments.
CALL_LOCK = threading.RLock()
_SERIALISE = os.environ.get("SBF_SERIALISE_CALLS", "1") != "0"


def serialised(fn):
    """Decorator: run a public entry point under the process-wide call lock."""
    if not _SERIALISE:
        return fn
    import functools

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        with CALL_LOCK:
            return fn(*args, **kwargs)

    return wrapper


def load():
    """Load libsbf.so once; raise loudly if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"CUDA extension {LIB_PATH} is missing; build it with "
                    "`python -m paper_1203_5128_b200.build` (there is no CPU fallback)")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.sbf_abi_version() != 1:
                raise RuntimeError("libsbf ABI version mismatch")
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().sbf_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "sbf") -> None:
    if status == SBF_OK:
        return
    msg = f"{what}: {last_error()}"
    if status in (SBF_ERR_INVALID, SBF_ERR_WORKSPACE):
        raise InvalidParameterError(msg)
    if status == SBF_ERR_UNSUPPORTED:
        raise UnsupportedOrderError(msg)
    if status == SBF_ERR_CUDA:
        raise RuntimeError(msg)
    raise ShiftBFError(f"{msg} (status {status})")


def specialisations():
    lib = load()
    out = []
    for i in range(lib.sbf_num_specialisations()):
        r, p, m = _int(), _int(), _int()
        lib.sbf_specialisation(i, C.byref(r), C.byref(p), C.byref(m))
        out.append((r.value, p.value, m.value))
    return out
