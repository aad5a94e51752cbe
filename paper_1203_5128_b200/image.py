"""Image validation and device staging (reference image.py:11-47).

`as_image` keeps the reference contract for host arrays (2-D, non-empty,
finite -> float64 C-contiguous).  `stage` moves an image to the GPU in the
narrowest dtype that represents it exactly (float32 for float32 and <=16-bit
integer inputs, float64 otherwise) — the reference computes in float64, and
the max filter / T must stay bit-exact, so float64 data is never rounded.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InvalidParameterError

_tls = threading.local()
_F32_EXACT = (np.float32, np.uint8, np.int8, np.uint16, np.int16, np.bool_)


def as_image(a) -> np.ndarray:
    """Validate and convert to the canonical 2-D float64 representation."""
    img = np.asarray(a, dtype=np.float64)
    if img.ndim != 2:
        raise InvalidParameterError(f"image must be 2-D, got shape {img.shape}")
    if img.size == 0:
        raise InvalidParameterError("image must be non-empty")
    if not np.isfinite(img).all():
        raise InvalidParameterError("image contains non-finite samples")
    return np.ascontiguousarray(img)


def checkerboard(height=256, width=256, square=32, low=0.0, high=255.0) -> np.ndarray:
    """Alternating squares of intensity `low` and `high` (image.py:23-29)."""
    if height < 1 or width < 1 or square < 1:
        raise InvalidParameterError("checkerboard dimensions must be positive")
    ii, jj = np.indices((height, width))
    cells = (ii // square + jj // square) % 2
    return np.where(cells == 1, float(high), float(low))


def impulse(height, width, value=1.0) -> np.ndarray:
    """Zero image with one `value` sample at the centre (image.py:32-36)."""
    img = np.zeros((height, width))
    img[height // 2, width // 2] = value
    return img


@dataclass
class Staged:
    tensor: "object"     # torch.Tensor on CUDA, C-contiguous
    dtype: int           # _lib.SBF_F32 / SBF_F64
    host: bool           # caller passed a host array
    H: int
    W: int
    torch_in: bool = False  # caller passed a torch tensor (results keep its float dtype)


def _stage_kinds():
    import torch

    kinds = {torch.float32: _lib.STAGE_F32, torch.float64: _lib.STAGE_F64,
             torch.uint8: _lib.STAGE_U8, torch.int16: _lib.STAGE_I16}
    if hasattr(torch, "uint16"):
        kinds[torch.uint16] = _lib.STAGE_U16
    return kinds


class _Kinds(dict):
    """dtype -> sbf_stage_h2d source kind, filled on first use (lazy torch)."""

    def __contains__(self, k):
        if not len(self):
            self.update(_stage_kinds())
        return dict.__contains__(self, k)


_STAGE_KINDS = _Kinds()


def _stage_pinned(t, device=None):
    """Pinned contiguous host tensor -> CUDA tensor via sbf_stage_h2d."""
    import torch

    kind = _STAGE_KINDS[t.dtype]
    out_dtype = torch.float64 if kind == _lib.STAGE_F64 else torch.float32
    # the staged copy lives only inside one (synchronising) call: reuse a
    # per-thread buffer
    d = torch.device(device or "cuda")
    d = torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())
    key = (d.index, out_dtype, tuple(t.shape))
    cache = getattr(_tls, "stage", None)
    if cache is None:
        cache = _tls.stage = {}
    dev = cache.get(key)
    if dev is None:
        if len(cache) > 8:
            cache.clear()
        dev = cache[key] = torch.empty(tuple(t.shape), dtype=out_dtype, device=d)
    lib = _lib.load()
    if dev.device.index == torch.cuda.current_device():
        rc = lib.sbf_stage_h2d(t.data_ptr(), kind, t.numel(), dev.data_ptr(),
                               torch.cuda.current_stream().cuda_stream)
    else:
        with torch.cuda.device(dev.device):
            rc = lib.sbf_stage_h2d(t.data_ptr(), kind, t.numel(), dev.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream)
    _lib.check(rc, "stage_h2d")
    # the read is stream-ordered; every public entry point synchronises on its
    # result before returning, so `t` outlives it
    return dev


def stage(img, device=None) -> Staged:
    """Put `img` (numpy array, torch tensor or nested sequence) on the GPU."""
    import torch

    if isinstance(img, torch.Tensor):
        t = img
        if t.ndim != 2:
            raise InvalidParameterError(f"image must be 2-D, got shape {tuple(t.shape)}")
        if t.numel() == 0:
            raise InvalidParameterError("image must be non-empty")
        host = not t.is_cuda
        if host and t.is_pinned() and t.is_contiguous() and t.dtype in _STAGE_KINDS:
            # pinned sources: the SMs read them over PCIe (sbf_stage_h2d),
            # stream-ordered before K1; 8/16-bit samples widen on the device
            t = _stage_pinned(t, device)
        elif t.dtype not in (torch.float32, torch.float64):
            exact32 = t.dtype in (torch.uint8, torch.int8, torch.int16, torch.bool)
            t = t.to(torch.float32 if exact32 else torch.float64)
        if host and not t.is_cuda:
            t = t.contiguous().to(device or "cuda", non_blocking=t.is_pinned())
        t = t.contiguous()
    else:
        a = np.asarray(img)
        if a.ndim != 2:
            raise InvalidParameterError(f"image must be 2-D, got shape {a.shape}")
        if a.size == 0:
            raise InvalidParameterError("image must be non-empty")
        if a.dtype.type in _F32_EXACT:
            a = np.ascontiguousarray(a, dtype=np.float32)
        else:
            a = np.ascontiguousarray(a, dtype=np.float64)
        t = torch.from_numpy(a).to(device or "cuda")
        host = True
    dt = _lib.SBF_F64 if t.dtype == torch.float64 else _lib.SBF_F32
    return Staged(t, dt, host, int(t.shape[0]), int(t.shape[1]), isinstance(img, torch.Tensor))
