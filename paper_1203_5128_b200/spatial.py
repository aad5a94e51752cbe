"""Spatial smoothing modes (reference spatial.py:24-57, 81-100, 185-194).

Only the parameter objects and scalar helpers live here; the smoothing
itself runs inside the fused CUDA term kernel.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Union

from . import _lib
from .errors import InvalidParameterError


@dataclass(frozen=True)
class Box:
    radius: int

    def __post_init__(self):
        if self.radius < 0:
            raise InvalidParameterError("box radius must be >= 0")


@dataclass(frozen=True)
class IteratedBox:
    sigma_s: float
    passes: int = 3

    def __post_init__(self):
        if self.sigma_s <= 0:
            raise InvalidParameterError("sigma_s must be positive")
        if self.passes < 1:
            raise InvalidParameterError("passes must be >= 1")


@dataclass(frozen=True)
class FirGaussian:
    """Accepted for API compatibility; the CUDA path rejects it (out of scope)."""

    sigma_s: float
    radius: int

    def __post_init__(self):
        if self.sigma_s <= 0:
            raise InvalidParameterError("sigma_s must be positive")
        if self.radius < 1:
            raise InvalidParameterError("radius must be >= 1")


SpatialMode = Union[Box, IteratedBox, FirGaussian]


def extended_box_params(sigma_s, passes):
    """(r, alpha) of one pass matching sigma_s^2/passes exactly (spatial.py:81-100)."""
    r, a = C.c_int(), C.c_double()
    _lib.check(_lib.load().sbf_extended_box_params(float(sigma_s), int(passes), C.byref(r),
                                                   C.byref(a)), "extended_box_params")
    return r.value, a.value


def box_radius_for_sigma(sigma_s, passes) -> int:
    return extended_box_params(sigma_s, passes)[0]


def to_c_spatial(mode: SpatialMode) -> _lib.SbfSpatial:
    sp = _lib.SbfSpatial()
    if isinstance(mode, Box):
        sp.mode, sp.passes, sp.r, sp.alpha, sp.sigma_s = _lib.SPATIAL_BOX, 1, int(mode.radius), 0.0, 0.0
    elif isinstance(mode, IteratedBox):
        r, a = extended_box_params(mode.sigma_s, mode.passes)
        sp.mode, sp.passes, sp.r, sp.alpha, sp.sigma_s = (_lib.SPATIAL_ITERATED, int(mode.passes), r,
                                                          a, float(mode.sigma_s))
    elif isinstance(mode, FirGaussian):
        raise InvalidParameterError("FirGaussian spatial mode is not supported by the CUDA path")
    else:
        raise InvalidParameterError(f"unknown spatial mode {mode!r}")
    return sp


def support_radius(mode: SpatialMode) -> int:
    """Radius beyond which the effective kernel is zero (spatial.py:185-194)."""
    if isinstance(mode, FirGaussian):
        return mode.radius
    sp = to_c_spatial(mode)
    out = C.c_int()
    _lib.check(_lib.load().sbf_support_radius(C.byref(sp), C.byref(out)), "support_radius")
    return out.value
