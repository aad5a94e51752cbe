"""The shiftable bilateral filter — drop-in for reference bilateral.py:43-137.

`shiftable_bf(img, params)` keeps the reference signature, parameter
semantics, result type and error/warning behaviour; the work runs on the
GPU as K1 (local range) -> K2 (plan on device) -> K3 (fused term kernel)
-> K4 (divide / fallback).  Host arrays in -> float64 host array out
(like the reference); CUDA tensors in -> CUDA tensor out (input dtype).
"""

from __future__ import annotations

import threading
import warnings
from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np

from . import _lib
from .errors import InvalidParameterError
from .image import stage
from .kernels import KernelFamily, KernelPlan, log_2_over_eps, select_plan
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


@_lib.serialised
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


# device "meta" block of one call: plan | fallback counter | statistics, read
# back with a single copy
_META_PLAN, _META_FB, _META_STATS, _META_BYTES = 0, 64, 128, 256


_tls = threading.local()


def _read_meta(meta):
    """Copy the device meta block into a per-thread page-locked buffer and
    wait for the stream (cheaper than a pageable .cpu() round trip)."""
    import torch

    buf = getattr(_tls, "meta", None)
    if buf is None or buf.numel() != meta.numel():
        buf = _tls.meta = torch.empty(meta.numel(), dtype=torch.uint8, pin_memory=True)
    buf.copy_(meta, non_blocking=True)
    torch.cuda.current_stream(meta.device).synchronize()
    return buf.numpy().copy()


def _workspace_layout(H, W, dtype, sp_key, prec):
    """(total bytes, term-table offset, filter-workspace offset) of the
    sbf_shiftable_bf workspace: [K1 workspace | term table | K3/K4 workspace].
    Asked of the library on every call (two cheap C calls): the answer depends
    on the library's thread-local path switches (sbf_set_split_min_radius ...),
    so it must not be memoised here."""
    lib = _lib.load()
    sp = _lib.SbfSpatial(*sp_key)
    total = lib.sbf_shiftable_bf_workspace(H, W, dtype, sp, prec, TERMS_CAP)
    terms_off = lib.sbf_local_range_workspace(H, W, dtype)
    return max(total, 256), terms_off, terms_off + ((TERMS_CAP * 32 + 255) // 256) * 256


def _scratch(dev, ws_bytes):
    """Per-thread device scratch reused across calls (every call synchronises
    before it returns): the meta block and a grow-only workspace."""
    import torch

    key = dev.index if dev.index is not None else torch.cuda.current_device()
    cache = getattr(_tls, "scratch", None)
    if cache is None:
        cache = _tls.scratch = {}
    meta, ws = cache.get(key, (None, None))
    if meta is None:
        meta = torch.empty(_META_BYTES, dtype=torch.uint8, device=dev)
    if ws is None or ws.numel() < ws_bytes:
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    cache[key] = (meta, ws)
    return meta, ws


def _filter_staged(s, params: FilterParams, out_f64: bool, to_host: bool = False):
    """Runs `_filter_on_device` with the image's device current, so the
    library's per-device caches, the stream and the workspace all belong to
    the device that holds the data (a tensor on a non-current GPU)."""
    import torch

    with torch.cuda.device(s.tensor.device):
        return _filter_on_device(s, params, out_f64, to_host)


def _filter_on_device(s, params: FilterParams, out_f64: bool, to_host: bool = False):
    """K1..K4 on a staged device image; returns (output, KernelPlan, fallbacks).

    One C call (sbf_shiftable_bf) launches the whole pipeline without a host
    round trip; the call synchronises once at the end on a single read-back of
    plan, fallback count and statistics (non-finite input is rejected after
    the fact).  "auto" resolves fp32 vs HDR on the device and re-runs the fp64
    path only for wide ranges.  `to_host`: the result lands in page-locked
    host memory (cached allocator), written by the device directly.
    """
    import torch

    if params.family is KernelFamily.POLYNOMIAL:
        raise InvalidParameterError("the polynomial family is not supported by the CUDA path")
    lib = _lib.load()
    sp = to_c_spatial(params.resolved_spatial())
    radius = params.resolved_radius()
    dev = s.tensor.device
    H, W = s.H, s.W
    use_fixed = params.fixed_T is not None
    if use_fixed and not float(params.fixed_T) >= 0.0:
        raise InvalidParameterError("T must be non-negative")  # kernels.py:118-119
    prec = _precision_code(params)
    stream = torch.cuda.current_stream(dev).cuda_stream
    rule = _lib.RULES.get(params.truncation, -1)
    l2e = log_2_over_eps(params.epsilon)
    total, terms_off, fws_off = _workspace_layout(
        H, W, s.dtype, (sp.mode, sp.passes, sp.r, 0, sp.alpha, sp.sigma_s), prec)
    # the pipeline resets the fallback counter and writes plan and statistics:
    # the meta block needs no clearing
    meta, ws = _scratch(dev, total)
    plan_ptr = meta.data_ptr() + _META_PLAN
    fb_ptr = meta.data_ptr() + _META_FB
    stats_ptr = meta.data_ptr() + _META_STATS
    terms_ptr = ws.data_ptr() + terms_off
    # host results are written by the epilogue straight into page-locked
    # memory over PCIe (segment by segment, while the last terms still run)
    out = torch.empty((H, W), dtype=torch.float64 if out_f64 else torch.float32,
                      **({"pin_memory": True} if to_host else {"device": dev}))
    out_dtype = _lib.SBF_F64 if out_f64 else _lib.SBF_F32
    _lib.check(lib.sbf_shiftable_bf(s.tensor.data_ptr(), s.dtype, H, W, sp, radius,
                                    float(params.fixed_T) if use_fixed else -1.0,
                                    float(params.sigma_r), float(params.epsilon), rule, l2e, prec,
                                    out.data_ptr(), out_dtype, plan_ptr, stats_ptr, fb_ptr,
                                    TERMS_CAP, ws.data_ptr(), total, stream), "shiftable_bf")
    tail = _read_meta(meta)
    stats_host = tail[_META_STATS:_META_STATS + 64]
    if int(stats_host.view(np.uint64)[7]) != 0:
        raise InvalidParameterError("image contains non-finite samples")
    plan_c = _lib.SbfPlan.from_buffer_copy(tail[_META_PLAN:_META_PLAN + 64].tobytes())
    _lib.check(plan_c.status, "plan")
    fallbacks = int(tail[_META_FB:_META_FB + 8].view(np.int64)[0])

    def rerun():
        meta[_META_FB:_META_FB + 8].zero_()
        _lib.check(lib.sbf_filter(s.tensor.data_ptr(), s.dtype, H, W, W, 0, H, 0, H, sp, plan_ptr,
                                  terms_ptr, stats_ptr, prec, out.data_ptr(), out_dtype, fb_ptr,
                                  ws.data_ptr() + fws_off, total - fws_off, stream), "filter")
        t = _read_meta(meta)
        return (_lib.SbfPlan.from_buffer_copy(t[_META_PLAN:_META_PLAN + 64].tobytes()),
                int(t[_META_FB:_META_FB + 8].view(np.int64)[0]))

    if plan_c.flags & _lib.PLAN_NEEDS_HDR:
        # the device guard found |f - centre| > 4096: fp64 path
        prec = _lib.PREC_HDR
        plan_c, fallbacks = rerun()
    if plan_c.flags & _lib.PLAN_N_AMBIGUOUS:
        # ceil(0.405 q^2) straddles an integer within 2 ulp of q^2: the host twin
        # (libm pow, bit-equal to CPython) decides, and the filter is re-run
        ph = select_plan(plan_c.T, params.sigma_r, params.epsilon, truncation=params.truncation)
        if (ph.N, ph.M) != (plan_c.N, plan_c.M):
            _lib.check(lib.sbf_plan_device_forced(stats_ptr, 1 if use_fixed else 0,
                                                  float(params.fixed_T) if use_fixed else 0.0,
                                                  float(params.sigma_r), float(params.epsilon),
                                                  rule, l2e, ph.N, ph.M, plan_ptr, terms_ptr,
                                                  TERMS_CAP, stream), "plan")
            plan_c, fallbacks = rerun()
    return out, _plan_from_struct(plan_c), fallbacks


@_lib.serialised
def shiftable_bf_batch(imgs, params: FilterParams, lanes: int = 3, out=None, stage: str = "ce"):
    """`[shiftable_bf(img, params) for img in imgs]`, pipelined on the GPU.

    A batch of independent images (the config-4 workload) is the same call
    repeated, so each result equals the single-image call bit for bit (same
    kernels, same plan).  What changes is the schedule: images rotate over
    `lanes` CUDA streams, each with its own workspace, so one image's
    host->device copy (copy engine), another's kernels and a third's result
    write-back over PCIe (the epilogue stores straight into page-locked
    memory) overlap.  One host synchronisation for the whole batch reads
    every plan, fallback count and statistics block back.

    `imgs`: torch tensors — page-locked host tensors (float32/float64) or
    CUDA tensors; other inputs go through `shiftable_bf` one by one.
    `out`: optional list of result tensors (same shape, float dtype of the
    input, same side) to write into.  `stage`: how host images reach the
    device — "ce" (copy engine, cudaMemcpyAsync: overlaps the other lanes'
    kernels without taking SMs) or "sm" (the SMs read page-locked memory,
    sbf_stage_h2d).  Host results come back by the copy engine from a lane
    buffer, so both PCIe directions overlap the kernels.
    """
    import torch

    imgs = list(imgs)
    fast = all(isinstance(t, torch.Tensor) and t.ndim == 2 and t.numel() > 0 and
               t.dtype in (torch.float32, torch.float64) and t.is_contiguous() and
               (t.is_cuda or t.is_pinned()) for t in imgs)
    if not fast or params.family is KernelFamily.POLYNOMIAL or not imgs:
        return [shiftable_bf(t, params) for t in imgs]
    lib = _lib.load()
    sp = to_c_spatial(params.resolved_spatial())
    radius = params.resolved_radius()
    use_fixed = params.fixed_T is not None
    if use_fixed and not float(params.fixed_T) >= 0.0:
        raise InvalidParameterError("T must be non-negative")
    prec = _precision_code(params)
    rule = _lib.RULES.get(params.truncation, -1)
    l2e = log_2_over_eps(params.epsilon)
    dev = next((t.device for t in imgs if t.is_cuda), None)
    dev = dev if dev is not None else torch.device("cuda", torch.cuda.current_device())
    n = len(imgs)
    lanes = max(1, min(int(lanes), n))
    metas = torch.empty((n, _META_BYTES), dtype=torch.uint8, device=dev)
    metas_h = torch.empty((n, _META_BYTES), dtype=torch.uint8, pin_memory=True)
    outs = list(out) if out is not None else [
        torch.empty(t.shape, dtype=t.dtype, **({"device": dev} if t.is_cuda else {"pin_memory": True}))
        for t in imgs]
    with torch.cuda.device(dev):
        main = torch.cuda.current_stream(dev)
        start = torch.cuda.Event()
        start.record(main)
        lane = []
        for _ in range(lanes):
            s = torch.cuda.Stream(device=dev)
            s.wait_event(start)
            lane.append({"stream": s, "ws": None, "inp": None, "res": None})
        for i, (t, o) in enumerate(zip(imgs, outs)):
            ln = lane[i % lanes]
            H, W = int(t.shape[0]), int(t.shape[1])
            dt = _lib.SBF_F64 if t.dtype == torch.float64 else _lib.SBF_F32
            total, _, _ = _workspace_layout(H, W, dt, (sp.mode, sp.passes, sp.r, 0, sp.alpha,
                                                      sp.sigma_s), prec)
            with torch.cuda.stream(ln["stream"]):
                if ln["ws"] is None or ln["ws"].numel() < total:
                    ln["ws"] = torch.empty(total, dtype=torch.uint8, device=dev)
                src = t
                if not t.is_cuda:
                    # copy engine, stream-ordered on the lane: overlaps the
                    # other lanes' kernels without taking SMs
                    b = ln["inp"]
                    if b is None or b.shape != t.shape or b.dtype != t.dtype:
                        b = ln["inp"] = torch.empty(t.shape, dtype=t.dtype, device=dev)
                    if stage == "sm":
                        _lib.check(lib.sbf_stage_h2d(t.data_ptr(),
                                                     _lib.STAGE_F64 if dt == _lib.SBF_F64 else _lib.STAGE_F32,
                                                     t.numel(), b.data_ptr(), ln["stream"].cuda_stream),
                                   "stage_h2d")
                    else:
                        b.copy_(t, non_blocking=True)
                    src = b
                m = metas[i]
                dst = o
                if not o.is_cuda:
                    # the result lands in a lane buffer and goes back by the
                    # copy engine, overlapping the other lanes' kernels
                    r = ln["res"]
                    if r is None or r.shape != o.shape or r.dtype != o.dtype:
                        r = ln["res"] = torch.empty(o.shape, dtype=o.dtype, device=dev)
                    dst = r
                _lib.check(lib.sbf_shiftable_bf(
                    src.data_ptr(), dt, H, W, sp, radius,
                    float(params.fixed_T) if use_fixed else -1.0, float(params.sigma_r),
                    float(params.epsilon), rule, l2e, prec, dst.data_ptr(),
                    _lib.SBF_F64 if o.dtype == torch.float64 else _lib.SBF_F32,
                    m.data_ptr() + _META_PLAN, m.data_ptr() + _META_STATS,
                    m.data_ptr() + _META_FB, TERMS_CAP, ln["ws"].data_ptr(), total,
                    ln["stream"].cuda_stream), "shiftable_bf")
                if dst is not o:
                    o.copy_(dst, non_blocking=True)
                metas_h[i].copy_(m, non_blocking=True)
        for ln in lane:
            main.wait_stream(ln["stream"])
        main.synchronize()
    tails = metas_h.numpy()
    results = []
    for i, t in enumerate(imgs):
        tail = tails[i]
        if int(tail[_META_STATS:_META_STATS + 64].view(np.uint64)[7]) != 0:
            raise InvalidParameterError(f"image {i} contains non-finite samples")
        plan_c = _lib.SbfPlan.from_buffer_copy(tail[_META_PLAN:_META_PLAN + 64].tobytes())
        _lib.check(plan_c.status, "plan")
        if plan_c.flags & (_lib.PLAN_NEEDS_HDR | _lib.PLAN_N_AMBIGUOUS):
            # rare: wide range or an ambiguous order; the single-image path
            # resolves both (fp64 re-run / host twin of the plan)
            r = shiftable_bf(t, params)
            outs[i].copy_(r.image)
            results.append(ShiftableResult(outs[i], r.plan, r.fallback_pixels))
            continue
        fb = int(tail[_META_FB:_META_FB + 8].view(np.int64)[0])
        if fb:
            warnings.warn(f"image {i}: {fb} pixel(s) had a non-positive normalizer; input values kept",
                          RuntimeWarning, stacklevel=2)
        results.append(ShiftableResult(outs[i], _plan_from_struct(plan_c), fb))
    return results


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
