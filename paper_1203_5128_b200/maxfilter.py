"""Windowed maximum and exact local dynamic range on the GPU (kernel K1).

Drop-ins for reference maxfilter.py:21-61 (`max_filter_1d`, `max_filter_2d`,
`compute_T`).  Results are bit-identical to the reference: the max filter
is exact and T = max(M - f) is evaluated in float64.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import InvalidParameterError
from .image import stage


def _stream_ptr():
    import torch
    return torch.cuda.current_stream().cuda_stream


def local_range(staged, radius, want_M=False, t_rows=None):
    """Run K1; returns (stats tensor[8] float64 on device, M tensor or None)."""
    import torch

    lib = _lib.load()
    f = staged.tensor
    H, W = staged.H, staged.W
    dev = f.device
    stats = torch.empty(8, dtype=torch.float64, device=dev)
    M = torch.empty_like(f) if want_M else None
    ws_bytes = lib.sbf_local_range_workspace(H, W, staged.dtype)
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dev)
    lo, hi = t_rows if t_rows is not None else (0, H)
    _lib.check(lib.sbf_local_range(f.data_ptr(), staged.dtype, H, W, W, int(radius), lo, hi,
                                   M.data_ptr() if M is not None else None, stats.data_ptr(),
                                   ws.data_ptr(), ws.numel(), _stream_ptr()), "local_range")
    return stats, M


def _nonfinite(stats_host) -> bool:
    return int(np.asarray(stats_host[7:8]).view(np.uint64)[0]) != 0


@_lib.serialised
def max_filter_2d(img, radius):
    """Maximum over the clamped (2R+1)^2 window (maxfilter.py:41-49)."""
    if radius < 0:
        raise InvalidParameterError("radius must be >= 0")
    s = stage(img)
    stats, M = local_range(s, int(radius), want_M=True)
    st = stats.cpu().numpy()
    if _nonfinite(st):
        raise InvalidParameterError("image contains non-finite samples")
    if s.host:
        return M.cpu().numpy().astype(np.float64)
    return M


@_lib.serialised
def max_filter_1d(seq, radius):
    """Sliding maximum over the clamped window [i-R, i+R] (maxfilter.py:21-28)."""
    arr = np.asarray(seq, dtype=np.float64)
    if arr.ndim != 1 or arr.size == 0:
        raise InvalidParameterError("input must be a non-empty 1-D sequence")
    if radius < 0:
        raise InvalidParameterError("radius must be >= 0")
    return max_filter_2d(arr.reshape(1, -1), int(radius))[0]


@_lib.serialised
def compute_T(img, radius) -> float:
    """Exact max |f(x-y) - f(x)| over square windows (maxfilter.py:56-61)."""
    if radius < 0:
        raise InvalidParameterError("radius must be >= 0")
    s = stage(img)
    stats, _ = local_range(s, int(radius))
    st = stats.cpu().numpy()
    if _nonfinite(st):
        raise InvalidParameterError("image contains non-finite samples")
    if radius == 0:
        return 0.0
    return float(st[0])


@_lib.serialised
def brute_force_T(img, radius) -> float:
    """max |f(x+y) - f(x)| over all pixels and in-image offsets |y| <= R,
    evaluated directly (O(R^2) per pixel) on the GPU — reference
    maxfilter.py:64-82.  Independent of K1's separable max filter, so it
    cross-checks compute_T (Proposition 1 of the paper)."""
    import ctypes as C

    if radius < 0:
        raise InvalidParameterError("radius must be >= 0")
    s = stage(img)
    out = C.c_double(0.0)
    _lib.check(_lib.load().sbf_brute_force_T(s.tensor.data_ptr(), s.dtype, s.H, s.W, s.W,
                                             int(radius), C.byref(out), _stream_ptr()),
               "brute_force_T")
    return float(out.value)
