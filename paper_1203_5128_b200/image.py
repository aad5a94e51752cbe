"""Image validation and device staging (reference image.py:11-47).

`as_image` keeps the reference contract for host arrays (2-D, non-empty,
finite -> float64 C-contiguous).  `stage` moves an image to the GPU in the
narrowest dtype that represents it exactly (float32 for float32 and <=16-bit
integer inputs, float64 otherwise) — the reference computes in float64, and
the max filter / T must stay bit-exact, so float64 data is never rounded.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InvalidParameterError

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
        if t.dtype not in (torch.float32, torch.float64):
            exact32 = t.dtype in (torch.uint8, torch.int8, torch.int16, torch.bool)
            t = t.to(torch.float32 if exact32 else torch.float64)
        if host:
            # pinned sources copy asynchronously, ordered before K1 on the stream
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
