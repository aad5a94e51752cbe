"""The shiftable bilateral filter — drop-in for reference bilateral.py:43-137.

`shiftable_bf(img, params)` keeps the reference signature, parameter
semantics, result type and error/warning behaviour; the work runs on the
GPU as K1 (local range) -> K2 (plan on device) -> K3 (fused term kernel)
-> K4 (divide / fallback).  Host arrays in -> float64 host array out
(like the reference); CUDA tensors in -> CUDA tensor out (input dtype).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np

from . import _lib
from .errors import InvalidParameterError
from .image import stage
from .kernels import KernelFamily, KernelPlan, log_2_over_eps, select_plan
from .maxfilter import _stream_ptr, local_range
from .spatial import IteratedBox, SpatialMode, support_radius, to_c_spatial

TERMS_CAP = 1 << 16
# |f - centre| above which the fp32 term kernel cannot hold 1e-2 absolute
# accuracy on the image's own scale; such images use the fp64-accumulating
# HDR kernel.
HDR_THRESHOLD = 4096.0
_PRECISIONS = ("auto", "fp32", "hdr")


@dataclass(frozen=True)
class FilterParams:
    """Bilateral filter configuration (bilateral.py:43-79).

    Extension (keyword, defaulted): `precision` in {"auto", "fp32", "hdr"}
    selects the term-kernel arithmetic; "auto" picks by the data range.
    """

    sigma_s: float
    sigma_r: float
    epsilon: float = 0.0
    spatial: Optional[SpatialMode] = None
    family: KernelFamily = KernelFamily.RAISED_COSINE
    window_radius: Optional[int] = None
    fixed_T: Optional[float] = None
    truncation: str = "auto"
    precision: str = "auto"

    def __post_init__(self):
        if self.sigma_s <= 0:
            raise InvalidParameterError("sigma_s must be positive")
        if self.sigma_r <= 0:
            raise InvalidParameterError("sigma_r must be positive")
        if not 0 <= self.epsilon < 1:
            raise InvalidParameterError("epsilon must lie in [0, 1)")
        if self.window_radius is not None and self.window_radius < 1:
            raise InvalidParameterError("window_radius must be >= 1")
        if self.precision not in _PRECISIONS:
            raise InvalidParameterError(f"precision must be one of {_PRECISIONS}")

    def resolved_spatial(self) -> SpatialMode:
        return self.spatial if self.spatial is not None else IteratedBox(self.sigma_s)

    def resolved_radius(self) -> int:
        if self.window_radius is not None:
            return self.window_radius
        return max(1, support_radius(self.resolved_spatial()))


class ShiftableResult(NamedTuple):
    image: object
    plan: KernelPlan
    fallback_pixels: int


def _plan_from_struct(p: _lib.SbfPlan) -> KernelPlan:
    return KernelPlan(family=KernelFamily.RAISED_COSINE, sigma_r=float(p.sigma_r), T=float(p.T),
                      N=int(p.N), M=int(p.M), epsilon=float(p.epsilon))


def _precision_code(params) -> int:
    """"auto" runs the fp32 kernels with a device-side range guard
    (SBF_PREC_AUTO): a wide-range (HDR) image is detected on the GPU and
    re-run with the fp64 path, so the common case needs no host round trip."""
    if params.precision == "fp32":
        return _lib.PREC_FP32
    if params.precision == "hdr":
        return _lib.PREC_HDR
    return _lib.PREC_AUTO


def shiftable_bf(img, params: FilterParams) -> ShiftableResult:
    """Constant-time bilateral filter; returns (image, plan, fallback count).

    Pipeline (bilateral.py:117-137): exact local range T over the spatial
    window, kernel order and truncation, one fused sweep per retained
    folded frequency, then num/den with the non-positive-normaliser
    fallback (RuntimeWarning + count).
    """
    s = stage(img)
    numpy_in = s.host and not s.torch_in
    out, plan, fallbacks = _filter_staged(s, params, out_f64=(numpy_in or s.dtype == _lib.SBF_F64),
                                          to_host=s.host)
    if fallbacks:
        warnings.warn(f"{fallbacks} pixel(s) had a non-positive normalizer; input values kept",
                      RuntimeWarning, stacklevel=2)
    # numpy in -> float64 numpy out (reference semantics); torch in -> torch
    # out in the input's float dtype, on the input's side (pinned host / CUDA)
    result = out.numpy() if numpy_in else out
    return ShiftableResult(result, plan, fallbacks)


def _filter_staged(s, params: FilterParams, out_f64: bool, to_host: bool = False):
    """K1..K4 on a staged device image; returns (output, KernelPlan, fallbacks).

    The pipeline runs without a host round trip and synchronises once at the
    end (non-finite input is rejected after the fact); "auto" resolves fp32
    vs HDR on the device and re-runs the fp64 path only for wide ranges.
    `to_host` copies the result into pinned host memory (cached allocator).
    """
    import torch

    if params.family is KernelFamily.POLYNOMIAL:
        raise InvalidParameterError("the polynomial family is not supported by the CUDA path")
    lib = _lib.load()
    mode = params.resolved_spatial()
    sp = to_c_spatial(mode)
    radius = params.resolved_radius()
    dev = s.tensor.device
    H, W = s.H, s.W
    use_fixed = params.fixed_T is not None
    # K1: T (or only the statistics when T is fixed)
    stats, _ = local_range(s, 0 if use_fixed else radius)
    prec = _precision_code(params)
    stream = _stream_ptr()
    plan_dev = torch.empty(64, dtype=torch.uint8, device=dev)
    terms = torch.empty(TERMS_CAP * 32, dtype=torch.uint8, device=dev)
    def plan_on_device(forced=None):
        args = (stats.data_ptr(), 1 if use_fixed else 0,
                float(params.fixed_T) if use_fixed else 0.0, float(params.sigma_r),
                float(params.epsilon), _lib.RULES.get(params.truncation, -1),
                log_2_over_eps(params.epsilon))
        if forced is None:
            _lib.check(lib.sbf_plan_device(*args, plan_dev.data_ptr(), terms.data_ptr(),
                                           TERMS_CAP, stream), "plan")
        else:
            _lib.check(lib.sbf_plan_device_forced(*args, forced[0], forced[1], plan_dev.data_ptr(),
                                                  terms.data_ptr(), TERMS_CAP, stream), "plan")

    plan_on_device()
    out_dtype = _lib.SBF_F64 if out_f64 else _lib.SBF_F32
    out = torch.empty((H, W), dtype=torch.float64 if out_f64 else torch.float32, device=dev)
    fb = torch.zeros(1, dtype=torch.int64, device=dev)
    ws_bytes = lib.sbf_filter_workspace(H, W, H, s.dtype, sp, prec)
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dev)
    _lib.check(lib.sbf_filter(s.tensor.data_ptr(), s.dtype, H, W, W, 0, H, 0, H, sp,
                              plan_dev.data_ptr(), terms.data_ptr(), stats.data_ptr(), prec,
                              out.data_ptr(), out_dtype, fb.data_ptr(), ws.data_ptr(), ws.numel(),
                              stream), "filter")
    out_dev = out
    if to_host:
        host = torch.empty((H, W), dtype=out.dtype, pin_memory=True)
        host.copy_(out, non_blocking=True)
        out = host
    # one small read-back for plan, fallback count and the input check
    tail = torch.cat([plan_dev, fb.view(torch.uint8), stats.view(torch.uint8)]).cpu().numpy()
    plan_c = _lib.SbfPlan.from_buffer_copy(tail[:64].tobytes())
    fallbacks = int(tail[64:72].view(np.int64)[0])
    if int(tail[72:].view(np.uint64)[7]) != 0:
        raise InvalidParameterError("image contains non-finite samples")
    _lib.check(plan_c.status, "plan")

    def rerun():
        fb.zero_()
        _lib.check(lib.sbf_filter(s.tensor.data_ptr(), s.dtype, H, W, W, 0, H, 0, H, sp,
                                  plan_dev.data_ptr(), terms.data_ptr(), stats.data_ptr(),
                                  prec, out_dev.data_ptr(), out_dtype, fb.data_ptr(),
                                  ws.data_ptr(), ws.numel(), stream), "filter")
        if to_host:
            out.copy_(out_dev)
        return (_lib.SbfPlan.from_buffer_copy(plan_dev.cpu().numpy().tobytes()),
                int(fb.item()))

    if plan_c.flags & _lib.PLAN_NEEDS_HDR:
        # the device guard found |f - centre| > 4096: fp64 path
        prec = _lib.PREC_HDR
        plan_c, fallbacks = rerun()
    if plan_c.flags & _lib.PLAN_N_AMBIGUOUS:
        # ceil(0.405 q^2) straddles an integer within 2 ulp of q^2: the host twin
        # (libm pow, bit-equal to CPython) decides, and the filter is re-run
        ph = select_plan(plan_c.T, params.sigma_r, params.epsilon, truncation=params.truncation)
        if (ph.N, ph.M) != (plan_c.N, plan_c.M):
            plan_on_device(forced=(ph.N, ph.M))
            plan_c, fallbacks = rerun()
    return out, _plan_from_struct(plan_c), fallbacks


def shiftable_bf_poly(img, params: FilterParams) -> ShiftableResult:
    """bilateral.py:167-202 — the polynomial range family is outside the CUDA path."""
    raise InvalidParameterError("the polynomial family is not supported by the CUDA path")


# backend registry of the reference (_core/__init__.py:12-71): one CUDA backend
def available_backends():
    return ["cuda"]


def backend_name() -> str:
    return "cuda"


def use_backend(name: str) -> str:
    if name != "cuda":
        raise ValueError(f"unknown backend {name!r}; choices: ['cuda']")
    return "cuda"
