"""Coarse non-local means with shiftable range kernels — drop-in for
reference nlm.py:29-137 (`PatchSpec`, `NlmResult`, `coarse_nlm_shiftable`).

SURVEY.md §8(f) rank 4: the term engine of the filter reused with
tensor-product terms.  T comes from K1 over radius + max offset norm (shared
by all components), every component gets its own plan (the reference's
per-component order cap and global multi-index budget apply, with the same
TermBudgetError), the folded multi-index table is built here and the GPU runs
it (`sbf_nlm_filter`, csrc/sbf_nlm.cu, fp64).
"""

from __future__ import annotations

import ctypes as C
import itertools
import math
import warnings
from dataclasses import dataclass
from typing import NamedTuple, Tuple

import numpy as np

from . import _lib
from .errors import InvalidParameterError, TermBudgetError
from .image import stage
from .kernels import KernelPlan, raised_cosine_expansion, select_plan
from .maxfilter import _nonfinite, _stream_ptr, local_range
from .spatial import SpatialMode, to_c_spatial

DEFAULT_COMPONENT_ORDER_CAP = 10
DEFAULT_TERM_BUDGET = 10_000


@dataclass(frozen=True)
class PatchSpec:
    """Patch offsets (first must be the origin) and per-component widths (nlm.py:29-58)."""

    offsets: Tuple[Tuple[int, int], ...]
    sigmas: Tuple[float, ...]

    def __post_init__(self):
        offsets = tuple((int(dy), int(dx)) for dy, dx in self.offsets)
        sigmas = tuple(float(s) for s in self.sigmas)
        object.__setattr__(self, "offsets", offsets)
        object.__setattr__(self, "sigmas", sigmas)
        p = len(offsets)
        if p == 0 or p > 3:
            raise InvalidParameterError("patch must have 1 to 3 offsets")
        if len(sigmas) != p:
            raise InvalidParameterError("need one sigma per patch offset")
        if offsets[0] != (0, 0):
            raise InvalidParameterError("first patch offset must be the origin")
        if len(set(offsets)) != p:
            raise InvalidParameterError("patch offsets must be distinct")
        if any(s <= 0 for s in sigmas):
            raise InvalidParameterError("patch sigmas must be positive")

    @property
    def size(self) -> int:
        return len(self.offsets)

    @property
    def max_offset_norm(self) -> int:
        return max(max(abs(dy), abs(dx)) for dy, dx in self.offsets)


class NlmResult(NamedTuple):
    image: object
    plans: Tuple[KernelPlan, ...]
    fallback_pixels: int


class _Item(C.Structure):
    _fields_ = [("weight", C.c_double), ("turns", C.c_double * 3), ("mask", C.c_int32),
                ("pad", C.c_int32)]


def _folded(plan: KernelPlan):
    """(scale, turns) of the folded terms n in [M, N/2] (cf. bilateral.py:150-154)."""
    e = raised_cosine_expansion(plan)
    out = []
    for w, om, n in zip(e.weights, e.frequencies, e.indices):
        if 2 * n > plan.N:
            break
        scale = w if 2 * n == plan.N else 2.0 * w
        out.append((float(scale), float(om) / (2.0 * math.pi)))
    return out


def build_items(plans):
    """Folded tensor-product item table (weights of exact-zero products skipped)."""
    comps = [_folded(p) for p in plans]
    p = len(plans)
    items = []
    for combo in itertools.product(*comps):
        weight = 1.0
        for s, _ in combo:
            weight *= s
        if weight == 0.0:
            continue  # contributes exactly nothing in the reference too
        turns = [t for _, t in combo] + [0.0] * (3 - p)
        for rest in range(1 << (p - 1)):
            items.append((weight, turns, rest << 1))
    arr = (_Item * max(1, len(items)))()
    for k, (w, t, m) in enumerate(items):
        arr[k].weight = w
        for j in range(3):
            arr[k].turns[j] = t[j]
        arr[k].mask = m
    return arr, len(items)


@_lib.serialised
def coarse_nlm_shiftable(img, patch: PatchSpec, spatial: SpatialMode, radius: int,
                         epsilon: float, truncation: str = "auto",
                         max_component_order: int = DEFAULT_COMPONENT_ORDER_CAP,
                         term_budget: int = DEFAULT_TERM_BUDGET) -> NlmResult:
    """Constant-time coarse non-local means (nlm.py:78-137) on the GPU.

    Returns float64 numpy for numpy input; torch input gives a torch tensor
    in the input float dtype on the input's device.
    With a single origin offset this is the bilateral filter.
    """
    import torch

    radius = int(radius)
    if radius < 0:
        raise InvalidParameterError("radius must be >= 0")
    s = stage(img)
    stats, _ = local_range(s, radius + patch.max_offset_norm)
    st = stats.cpu().numpy()
    if _nonfinite(st):
        raise InvalidParameterError("image contains non-finite samples")
    T = float(st[0])
    plans = tuple(select_plan(T, sg, epsilon, truncation=truncation) for sg in patch.sigmas)
    for j, plan in enumerate(plans):
        if plan.retained_terms > max_component_order:
            raise TermBudgetError(
                f"patch component {j} retains {plan.retained_terms} terms after "
                f"truncation, above the per-component cap of {max_component_order}")
    total = 1
    for plan in plans:
        total *= plan.retained_terms
    if total > term_budget:
        raise TermBudgetError(
            f"tensor expansion needs {total} multi-index terms, "
            f"exceeding the term budget of {term_budget}")
    items, n_items = build_items(plans)
    offs = (C.c_int32 * (2 * patch.size))(*[v for off in patch.offsets for v in off])
    numpy_in = s.host and not s.torch_in
    out_f64 = numpy_in or s.dtype == _lib.SBF_F64
    out = torch.empty((s.H, s.W), dtype=torch.float64 if out_f64 else torch.float32,
                      device=s.tensor.device)
    fb = torch.zeros(1, dtype=torch.int64, device=s.tensor.device)
    lib = _lib.load()
    _lib.check(lib.sbf_nlm_filter(s.tensor.data_ptr(), s.dtype, s.H, s.W, s.W,
                                  to_c_spatial(spatial), patch.size, offs, items, n_items,
                                  stats.data_ptr(), out.data_ptr(),
                                  _lib.SBF_F64 if out_f64 else _lib.SBF_F32, fb.data_ptr(),
                                  _stream_ptr()), "nlm")
    fallbacks = int(fb.item())
    if fallbacks:
        warnings.warn(f"{fallbacks} pixel(s) had a non-positive normalizer; input values kept",
                      RuntimeWarning, stacklevel=2)
    return NlmResult(out.cpu().numpy() if numpy_in else (out.cpu() if s.host else out), plans, fallbacks)


def expansion_range_for(plan: KernelPlan):
    """Truncated-expansion range kernel of one NLM component (nlm.py:186-189)."""
    from .direct import expansion_range
    return expansion_range(raised_cosine_expansion(plan))


@_lib.serialised
def direct_nlm(img, patch: PatchSpec, spatial: SpatialMode, radius: int,
               range_kernels="gaussian"):
    """Literal windowed coarse NLM (nlm.py:140-183), the shiftable NLM's test
    oracle, on the GPU (`sbf_direct_nlm`, float64).  `range_kernels` is
    "gaussian" or one gaussian_range / expansion_range kernel per component."""
    import torch

    from .direct import ExpansionRange, GaussianRange, _taps

    radius = int(radius)
    if range_kernels == "gaussian":
        from .direct import gaussian_range
        kernels = [gaussian_range(sg) for sg in patch.sigmas]
    else:
        kernels = list(range_kernels)
        if len(kernels) != patch.size:
            raise InvalidParameterError("need one range kernel per patch offset")
    taps = _taps(spatial, radius)
    kinds, sigmas, nterms, scales, freqs = [], [], [], [], []
    for k in kernels:
        if isinstance(k, GaussianRange):
            kinds.append(0)
            sigmas.append(k.sigma_r)
            nterms.append(0)
        elif isinstance(k, ExpansionRange):
            e = k.expansion
            keep = 2 * np.asarray(e.indices) <= e.plan.N
            w = np.asarray(e.weights)[keep]
            n = np.asarray(e.indices)[keep]
            kinds.append(1)
            sigmas.append(0.0)
            nterms.append(int(keep.sum()))
            scales.extend(np.where(2 * n == e.plan.N, w, 2.0 * w).tolist())
            freqs.extend(np.asarray(e.frequencies)[keep].tolist())
        else:
            raise InvalidParameterError(
                "only gaussian_range() / expansion_range() kernels run on the GPU direct path")
    s = stage(img)
    stats, _ = local_range(s, 0)
    if _nonfinite(stats.cpu().numpy()):
        raise InvalidParameterError("image contains non-finite samples")
    numpy_in = s.host and not s.torch_in
    out_f64 = numpy_in or s.dtype == _lib.SBF_F64
    out = torch.empty((s.H, s.W), dtype=torch.float64 if out_f64 else torch.float32,
                      device=s.tensor.device)
    i32 = lambda v: (C.c_int32 * max(1, len(v)))(*v)
    f64 = lambda v: (C.c_double * max(1, len(v)))(*v)
    _lib.check(_lib.load().sbf_direct_nlm(
        s.tensor.data_ptr(), s.dtype, s.H, s.W, s.W, radius,
        None if taps is None else taps.ctypes.data, patch.size,
        i32([v for off in patch.offsets for v in off]), i32(kinds), f64(sigmas), i32(nterms),
        f64(scales), f64(freqs), out.data_ptr(), _lib.SBF_F64 if out_f64 else _lib.SBF_F32,
        _stream_ptr()), "direct_nlm")
    return out.cpu().numpy() if numpy_in else (out.cpu() if s.host else out)
