"""Brute-force bilateral filter on the GPU — drop-in for reference
bilateral.py:88-99 (`gaussian_range`) and :205-239 (`direct_bf`), with the
window weights of spatial.py:155-157 / :197-213.

The O(R^2)-per-pixel accuracy oracle for the shiftable filter at full image
sizes, run by the CUDA kernel K5 (`sbf_direct_bf`).
Only the Gaussian range kernel runs on the GPU: `range_kernel` must come from
`gaussian_range`; any other callable raises InvalidParameterError rather than
running on the CPU.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InvalidParameterError
from .image import as_image, stage
from .bilateral import HDR_THRESHOLD
from .maxfilter import _nonfinite, _stream_ptr, local_range
from .spatial import Box, FirGaussian, IteratedBox


@dataclass(frozen=True)
class GaussianRange:
    """exp(-s^2 / (2 sigma_r^2)); callable on numpy arrays like the reference's closure."""

    sigma_r: float

    def __call__(self, s):
        s = np.asarray(s, dtype=np.float64)
        return np.exp(-(s * s) * (1.0 / (2.0 * self.sigma_r * self.sigma_r)))


@dataclass(frozen=True)
class ExpansionRange:
    """The truncated cosine expansion itself as a range kernel (bilateral.py:101-103)."""

    expansion: object

    def __call__(self, s):
        from .kernels import eval_truncated_kernel
        return eval_truncated_kernel(self.expansion, s)


def expansion_range(expansion) -> ExpansionRange:
    """Range kernel evaluating a truncated raised-cosine expansion (bilateral.py:101-103);
    direct_bf with it is the exact-shiftability oracle, run on the GPU in fp64."""
    return ExpansionRange(expansion)


def polynomial_range(plan):
    """(1 - s^2 / (2 N sigma_r^2))^N (bilateral.py:106-114): host-side kernel
    function only — the polynomial family is not part of the CUDA path, so
    direct_bf rejects it."""
    a = 2.0 * plan.N * plan.sigma_r ** 2

    def kernel(s):
        s = np.asarray(s, dtype=np.float64)
        return (1.0 - (s * s) / a) ** plan.N

    return kernel


def gaussian_range(sigma_r) -> GaussianRange:
    """Vectorised Gaussian range kernel of width sigma_r (bilateral.py:88-99)."""
    if sigma_r <= 0:
        raise InvalidParameterError("sigma_r must be positive")
    return GaussianRange(float(sigma_r))


def gaussian_taps(sigma_s, radius) -> np.ndarray:
    """Sampled 1-D Gaussian taps exp(-k^2 / (2 sigma_s^2)), k in [-R, R] (spatial.py:155-157)."""
    k = np.arange(-radius, radius + 1, dtype=np.float64)
    return np.exp(-(k * k) / (2.0 * sigma_s * sigma_s))


def spatial_weight_table(mode, radius=None) -> np.ndarray:
    """Explicit (2R+1)^2 window weights (spatial.py:197-213); IteratedBox is rejected."""
    if isinstance(mode, Box):
        r = mode.radius if radius is None else int(radius)
        return np.ones((2 * r + 1, 2 * r + 1))
    if isinstance(mode, FirGaussian):
        r = mode.radius if radius is None else int(radius)
        taps = gaussian_taps(mode.sigma_s, r)
        return np.outer(taps, taps)
    raise InvalidParameterError("direct filtering supports Box and FirGaussian spatial modes only")


def _taps(mode, radius):
    if isinstance(mode, Box):
        return None  # uniform window
    if isinstance(mode, FirGaussian):
        return np.ascontiguousarray(gaussian_taps(mode.sigma_s, radius))
    if isinstance(mode, IteratedBox):
        raise InvalidParameterError(
            "direct filtering supports Box and FirGaussian spatial modes only")
    raise InvalidParameterError(f"unknown spatial mode {mode!r}")


@_lib.serialised
def direct_bf(img, spatial, range_kernel, radius=None):
    """Brute-force bilateral filter over the clamped window (bilateral.py:205-239).

    Returns float64 numpy for numpy input; torch input gives a torch tensor
    in the input float dtype on the input's device.
    """
    import torch

    if not isinstance(range_kernel, (GaussianRange, ExpansionRange)):
        raise InvalidParameterError(
            "only gaussian_range() / expansion_range() kernels run on the GPU direct path")
    if radius is None:
        if isinstance(spatial, (Box, FirGaussian)):
            radius = spatial.radius
        else:
            _taps(spatial, 0)  # raises the reference's error
    radius = int(radius)
    if radius < 0:
        raise InvalidParameterError("radius must be >= 0")
    taps = _taps(spatial, radius)
    s = stage(img)
    stats, _ = local_range(s, 0)  # input statistics: non-finite samples are rejected
    st = stats.cpu().numpy()
    if _nonfinite(st):
        raise InvalidParameterError("image contains non-finite samples")
    # fp32 math unless the intensities span more than the HDR threshold
    hdr = max(abs(st[2] - st[3]), abs(st[1] - st[3])) > HDR_THRESHOLD
    numpy_in = s.host and not s.torch_in
    out_f64 = numpy_in or s.dtype == _lib.SBF_F64
    out = torch.empty((s.H, s.W), dtype=torch.float64 if out_f64 else torch.float32,
                      device=s.tensor.device)
    lib = _lib.load()
    if isinstance(range_kernel, ExpansionRange):
        e = range_kernel.expansion
        keep = 2 * np.asarray(e.indices) <= e.plan.N  # fold +-w (cos is even)
        w = np.asarray(e.weights)[keep]
        n = np.asarray(e.indices)[keep]
        scale = np.ascontiguousarray(np.where(2 * n == e.plan.N, w, 2.0 * w), dtype=np.float64)
        freq = np.ascontiguousarray(np.asarray(e.frequencies)[keep], dtype=np.float64)
        _lib.check(lib.sbf_direct_bf_expansion(
            s.tensor.data_ptr(), s.dtype, s.H, s.W, s.W, radius,
            None if taps is None else taps.ctypes.data, scale.ctypes.data, freq.ctypes.data,
            len(scale), out.data_ptr(), _lib.SBF_F64 if out_f64 else _lib.SBF_F32, _stream_ptr()),
            "direct_bf")
        return out.cpu().numpy() if numpy_in else (out.cpu() if s.host else out)
    _lib.check(lib.sbf_direct_bf(s.tensor.data_ptr(), s.dtype, s.H, s.W, s.W, radius,
                                 None if taps is None else taps.ctypes.data,
                                 float(range_kernel.sigma_r),
                                 _lib.PREC_HDR if hdr else _lib.PREC_FP32, out.data_ptr(),
                                 _lib.SBF_F64 if out_f64 else _lib.SBF_F32, _stream_ptr()),
               "direct_bf")
    return out.cpu().numpy() if numpy_in else (out.cpu() if s.host else out)


@dataclass(frozen=True)
class Metrics:
    mse: float
    mse_db: float  # 10 log10(mse); -inf when mse == 0
    max_abs: float


def metrics(a, b) -> Metrics:
    """MSE, MSE in dB and max |difference| (reference metrics.py:19-28)."""
    x = as_image(a.cpu().numpy() if hasattr(a, "cpu") else a)
    y = as_image(b.cpu().numpy() if hasattr(b, "cpu") else b)
    if x.shape != y.shape:
        raise InvalidParameterError(f"shape mismatch: {x.shape} vs {y.shape}")
    d = x - y
    mse = float(np.mean(d * d))
    return Metrics(mse=mse, mse_db=10.0 * math.log10(mse) if mse > 0 else float("-inf"),
                   max_abs=float(np.abs(d).max()))
