"""ctypes front end of the C oracle (oracle/sbf_oracle.c) — TEST INFRASTRUCTURE ONLY.

Same contract as `shiftbf_oracle.shiftable_bf` (reference bilateral.py:117-164):
the plan (T, N, M, folded weights and frequencies) comes from the numpy
oracle, the per-pixel work (max filter, cosine-term accumulation with the
extended-box smoother, divide with fallback) from the C restatement.  Used by
the tests (pinned against the numpy oracle and the golden vectors) and as the
timed CPU implementation in bench.py.  The product package never imports it.

    python -m oracle.coracle        # build oracle/_build/liboracle.so
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from . import shiftbf_oracle as O

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "sbf_oracle.c")
LIB = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """gcc -O2 (IEEE semantics, no fast-math) into oracle/_build/."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-o", LIB, SRC, "-lm"],
                   check=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = C.CDLL(LIB)
        P = C.c_void_p
        lib.oracle_max_filter_2d.argtypes = [P, C.c_int64, C.c_int64, C.c_int64, P]
        lib.oracle_max_filter_2d.restype = C.c_int
        lib.oracle_compute_T.argtypes = [P, C.c_int64, C.c_int64, C.c_int64]
        lib.oracle_compute_T.restype = C.c_double
        lib.oracle_accumulate.argtypes = [P, C.c_int64, C.c_int64, P, P, C.c_int, C.c_int,
                                          C.c_int64, C.c_double, C.c_int, P, P]
        lib.oracle_accumulate.restype = C.c_int
        lib.oracle_divide.argtypes = [P, P, P, C.c_int64, P]
        lib.oracle_divide.restype = C.c_int64
        _lib = lib
    return _lib


def max_filter_2d(img, radius):
    f = O.as_image(img)
    out = np.empty_like(f)
    if load().oracle_max_filter_2d(f.ctypes.data, *f.shape, int(radius), out.ctypes.data):
        raise O.OracleError("bad max-filter arguments")
    return out


def compute_T(img, radius):
    f = O.as_image(img)
    return float(load().oracle_compute_T(f.ctypes.data, *f.shape, int(radius)))


def _spatial_args(spatial):
    if spatial[0] == "box":
        return 1, int(spatial[1]), 0.0, 1
    r, alpha = O.extended_box_params(spatial[1], spatial[2])
    return 0, r, alpha, int(spatial[2])


def shiftable_bf(img, sigma_s, sigma_r, epsilon=0.0, spatial=None,
                 window_radius=None, fixed_T=None, truncation="auto"):
    """bilateral.py:117-164 — returns dict(image, T, N, M, fallback_pixels)."""
    f = O.as_image(img)
    if spatial is None:
        spatial = ("iterated", float(sigma_s), 3)
    if window_radius is not None:
        radius = int(window_radius)
    elif spatial[0] == "box":
        radius = max(1, int(spatial[1]))
    else:
        radius = max(1, O.support_radius("iterated", spatial[1], spatial[2]))
    T = float(fixed_T) if fixed_T is not None else compute_T(f, radius)
    T, N, M = O.select_plan(T, sigma_r, epsilon, truncation)
    _, scale, freq = O.folded_terms(N, M, sigma_r)
    scale = np.ascontiguousarray(scale, dtype=np.float64)
    freq = np.ascontiguousarray(freq, dtype=np.float64)
    mode, r, alpha, passes = _spatial_args(spatial)
    num = np.empty_like(f)
    den = np.empty_like(f)
    lib = load()
    rc = lib.oracle_accumulate(f.ctypes.data, *f.shape, scale.ctypes.data, freq.ctypes.data,
                               len(scale), mode, r, alpha, passes, num.ctypes.data, den.ctypes.data)
    if rc:
        raise O.OracleError(f"oracle_accumulate failed ({rc})")
    out = np.empty_like(f)
    n_bad = int(lib.oracle_divide(num.ctypes.data, den.ctypes.data, f.ctypes.data, f.size,
                                  out.ctypes.data))
    return dict(image=out, T=T, N=N, M=M, fallback_pixels=n_bad)


if __name__ == "__main__":
    print(build(force=True))
