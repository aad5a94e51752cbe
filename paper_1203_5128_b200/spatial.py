"""Spatial smoothing modes and smoothers (reference spatial.py:24-194).

Parameter objects and scalar helpers; inside the filter the smoothing runs
in the fused CUDA term kernel, and the standalone smoothers (`box_filter`,
`iterated_box_gaussian`, `fir_gaussian`, `apply_spatial`) run `sbf_smooth`.
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
    """Sampled-Gaussian FIR mode: `fir_gaussian` / `direct_bf` weights (the
    shiftable filter itself rejects it, like the reference's per-window table)."""

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


# ---------------------------------------------------------------------------
# standalone smoothers on the GPU (reference spatial.py:65-182), float64
# ---------------------------------------------------------------------------
def _smooth(img, sp):
    import torch

    from .image import stage
    from .maxfilter import _stream_ptr

    s = stage(img)
    numpy_in = s.host and not s.torch_in
    out_f64 = numpy_in or s.dtype == _lib.SBF_F64
    out = torch.empty((s.H, s.W), dtype=torch.float64 if out_f64 else torch.float32,
                      device=s.tensor.device)
    _lib.check(_lib.load().sbf_smooth(s.tensor.data_ptr(), s.dtype, s.H, s.W, s.W, sp,
                                      out.data_ptr(), _lib.SBF_F64 if out_f64 else _lib.SBF_F32,
                                      _stream_ptr()), "smooth")
    if not bool(torch.isfinite(out).all()):
        raise InvalidParameterError("image contains non-finite samples")
    return out.cpu().numpy() if numpy_in else (out.cpu() if s.host else out)


@_lib.serialised
def box_filter(img, radius):
    """Mean over the clamped (2r+1)^2 window (spatial.py:65-78)."""
    radius = int(radius)
    if radius < 0:
        raise InvalidParameterError("radius must be >= 0")
    return _smooth(img, to_c_spatial(Box(radius)))


@_lib.serialised
def iterated_box_gaussian(img, sigma_s, passes=3):
    """`passes` extended-box passes of variance sigma_s^2/passes each (spatial.py:108-139)."""
    return _smooth(img, to_c_spatial(IteratedBox(sigma_s, passes)))


@_lib.serialised
def fir_gaussian(img, sigma_s, radius):
    """Separable sampled Gaussian, renormalised per clamped window (spatial.py:142-172)."""
    if sigma_s <= 0:
        raise InvalidParameterError("sigma_s must be positive")
    if radius < 1:
        raise InvalidParameterError("radius must be >= 1")
    sp = _lib.SbfSpatial()
    sp.mode, sp.passes, sp.r, sp.alpha, sp.sigma_s = _lib.SPATIAL_FIR, 1, int(radius), 0.0, float(sigma_s)
    return _smooth(img, sp)


@_lib.serialised
def apply_spatial(img, mode: SpatialMode):
    """spatial.py:175-182."""
    if isinstance(mode, Box):
        return box_filter(img, mode.radius)
    if isinstance(mode, IteratedBox):
        return iterated_box_gaussian(img, mode.sigma_s, mode.passes)
    if isinstance(mode, FirGaussian):
        return fir_gaussian(img, mode.sigma_s, mode.radius)
    raise InvalidParameterError(f"unknown spatial mode {mode!r}")
