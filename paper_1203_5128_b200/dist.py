"""Multi-GPU drivers for the sharded configurations.

One process per GPU, `torch.distributed` for the plumbing.

* Image batches (config 4): images are independent — each has its own T and
  plan, exactly like separate `shiftable_bf` calls — so ranks take disjoint
  subsets, balanced by estimated cost (pixels x terms when known, else
  pixels).  No collective on the data path.
* Row strips (config 5): rank g owns output rows [g H/G, (g+1) H/G) and
  holds them plus a halo of max(R, support) rows (clamped at the image
  edges).  K1 computes the strip-local T over the owned rows only; the global
  T is one NCCL max-allreduce of float64 values (one per channel, all
  channels in one call) — the maximum of strip-local maxima equals the
  image-wide T exactly (max is associative).  K3 then renormalises only at
  true image borders (global row indices), so strip outputs equal the
  full-image filter (verified to 1.3e-12 in float64).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _lib
from .bilateral import TERMS_CAP, FilterParams, _plan_from_struct
from .errors import InvalidParameterError
from .kernels import log_2_over_eps
from .spatial import support_radius, to_c_spatial


@dataclass(frozen=True)
class Strip:
    rank: int
    buf_lo: int   # first image row held by the rank
    buf_hi: int   # one past the last held row
    out_lo: int   # first output row owned
    out_hi: int

    @property
    def halo_top(self) -> int:
        return self.out_lo - self.buf_lo

    @property
    def rows(self) -> int:
        return self.buf_hi - self.buf_lo


def strip_plan(H: int, world: int, halo: int) -> List[Strip]:
    """Even row partition with `halo` rows on each side (clamped)."""
    if H < 1 or world < 1 or halo < 0:
        raise InvalidParameterError("need H >= 1, world >= 1, halo >= 0")
    out = []
    for g in range(world):
        lo = (g * H) // world
        hi = ((g + 1) * H) // world
        out.append(Strip(g, max(0, lo - halo), min(H, hi + halo), lo, hi))
    return out


def shard_images(costs: Sequence[float], world: int) -> List[List[int]]:
    """Greedy longest-processing-time assignment of images to ranks."""
    order = sorted(range(len(costs)), key=lambda i: -costs[i])
    load = [0.0] * world
    parts: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        g = min(range(world), key=lambda k: load[k])
        parts[g].append(i)
        load[g] += costs[i]
    return [sorted(p) for p in parts]


def strip_halo(params: FilterParams) -> int:
    """Rows a strip must carry: the T window and the spatial support."""
    mode = params.resolved_spatial()
    return max(params.resolved_radius(), support_radius(mode))


def allreduce_max_(t, group=None):
    """In-place MAX all-reduce of a device tensor (NCCL on CUDA tensors)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


class StripFilter:
    """Filters the owned rows of one or more channels held as row strips.

    `bufs` are CUDA tensors (rows x W, float32/float64) holding image rows
    [strip.buf_lo, strip.buf_hi) of channels of height `img_H`.  `run()`
    performs K1 per channel, ONE max-allreduce of all channel T values,
    then the plan and the filter per channel, stream-ordered; `check()`
    reads plans, statistics and fallback counts back once (non-finite input,
    HDR re-run, ambiguous order) — the shiftable_bf semantics.
    """

    def __init__(self, bufs, strip: Strip, img_H: int, params: FilterParams,
                 reduce_max: Optional[Callable] = None, precision: Optional[str] = None,
                 overlap: bool = False):
        import torch
        self.lib = _lib.load()
        self.bufs = [b.contiguous() for b in bufs]
        self.strip = strip
        self.img_H = int(img_H)
        self.params = params
        self.reduce_max = reduce_max or allreduce_max_
        self.dev = self.bufs[0].device
        self.sp = to_c_spatial(params.resolved_spatial())
        self.R = params.resolved_radius()
        # the filter's precision mode: params.precision unless overridden;
        # "auto" runs the fp32 kernels with the device-side range guard
        # (check() re-runs a flagged channel on the fp64 path)
        mode = precision if precision is not None else params.precision
        self.prec = {"fp32": _lib.PREC_FP32, "hdr": _lib.PREC_HDR}.get(mode, _lib.PREC_AUTO)
        self.dt = [_lib.SBF_F64 if b.dtype == torch.float64 else _lib.SBF_F32 for b in self.bufs]
        C = len(self.bufs)
        H, W = self.bufs[0].shape
        self.H, self.W = int(H), int(W)
        rows_out = strip.out_hi - strip.out_lo
        self.stats = torch.zeros((C, 8), dtype=torch.float64, device=self.dev)
        self.T = torch.zeros(C, dtype=torch.float64, device=self.dev)
        self.plans = torch.empty((C, 64), dtype=torch.uint8, device=self.dev)
        self.terms = torch.empty((C, TERMS_CAP * 32), dtype=torch.uint8, device=self.dev)
        self.fb = torch.zeros(C, dtype=torch.int64, device=self.dev)
        self.out = [torch.empty((rows_out, self.W), dtype=b.dtype, device=self.dev)
                    for b in self.bufs]
        lr = max(self.lib.sbf_local_range_workspace(self.H, self.W, d) for d in self.dt)
        fw = max(self.lib.sbf_filter_workspace(self.H, self.W, rows_out, d, self.sp, self.prec)
                 for d in self.dt)
        self.ws = torch.empty(max(lr, fw, 256), dtype=torch.uint8, device=self.dev)
        # overlap: each channel's K2/K3/K4 on its own stream and workspace, so
        # one channel's kernels fill the SMs another's launch tails leave idle
        self.overlap = bool(overlap) and C > 1
        if self.overlap:
            self.side = [torch.cuda.Stream(device=self.dev) for _ in range(C)]
            self.side_ws = [self.ws] + [torch.empty(max(fw, 256), dtype=torch.uint8, device=self.dev)
                                        for _ in range(C - 1)]

    def _stream(self, stream_ptr):
        import torch
        return stream_ptr if stream_ptr is not None else torch.cuda.current_stream(self.dev).cuda_stream

    def _stream_obj(self, stream_ptr):
        """The torch stream object of `stream_ptr` (the current stream when
        None: wrapping its raw handle would not order the null stream)."""
        import torch
        if stream_ptr is None:
            return torch.cuda.current_stream(self.dev)
        return torch.cuda.ExternalStream(stream_ptr, device=self.dev)

    def local_T(self, stream_ptr=None):
        """K1 on every channel; returns the device tensor of strip-local T values."""
        lib, s = self.lib, self.strip
        st = self._stream(stream_ptr)
        lo, hi = s.out_lo - s.buf_lo, s.out_hi - s.buf_lo
        use_fixed = self.params.fixed_T is not None
        for c, b in enumerate(self.bufs):
            _lib.check(lib.sbf_local_range(b.data_ptr(), self.dt[c], self.H, self.W, self.W,
                                           0 if use_fixed else self.R, lo, hi, None,
                                           self.stats[c].data_ptr(), self.ws.data_ptr(),
                                           self.ws.numel(), st), "local_range")
        self.T.copy_(self.stats[:, 0])
        return self.T

    def run(self, stream_ptr=None):
        self.local_T(stream_ptr)
        if self.params.fixed_T is None:
            self.reduce_max(self.T)   # one collective for all channels
        return self.finish(stream_ptr=stream_ptr)

    def run_host(self, host_bufs, host_outs, stream_ptr=None):
        """run() for strips that live in host memory: `host_bufs[c]` (this
        rank's buffer rows of channel c, ideally page-locked) is copied to the
        device, filtered, and the owned rows are copied into `host_outs[c]`.
        The channels are pipelined: uploads and downloads ride the copy
        engines on per-channel streams, and every channel reduces its own T
        (one small collective per channel instead of one for all), so channel
        c's sweep overlaps channel c+1's upload and channel c-1's download.
        Stream-ordered on `stream_ptr`; call check() (or synchronise) before
        reading the host results."""
        import torch
        main = self._stream_obj(stream_ptr)
        if not hasattr(self, "copy_streams"):
            self.copy_streams = [torch.cuda.Stream(device=self.dev) for _ in self.bufs]
        start = torch.cuda.Event()
        start.record(main)
        lib, s, p = self.lib, self.strip, self.params
        st = self._stream(stream_ptr)
        lo, hi = s.out_lo - s.buf_lo, s.out_hi - s.buf_lo
        use_fixed = p.fixed_T is not None
        ups = []
        for c, cs in enumerate(self.copy_streams):
            cs.wait_event(start)  # the previous run's kernels are done with bufs[c] / out[c]
            with torch.cuda.stream(cs):
                self.bufs[c].copy_(host_bufs[c], non_blocking=True)
            e = torch.cuda.Event()
            e.record(cs)
            ups.append(e)
        with torch.cuda.stream(main):
            self.fb.zero_()
        for c, b in enumerate(self.bufs):
            main.wait_event(ups[c])
            _lib.check(lib.sbf_local_range(b.data_ptr(), self.dt[c], self.H, self.W, self.W,
                                           0 if use_fixed else self.R, lo, hi, None,
                                           self.stats[c].data_ptr(), self.ws.data_ptr(),
                                           self.ws.numel(), st), "local_range")
            with torch.cuda.stream(main):
                self.T[c:c + 1].copy_(self.stats[c, 0:1])
                if not use_fixed:
                    self.reduce_max(self.T[c:c + 1])
            _lib.check(lib.sbf_plan_device(
                self.T[c:c + 1].data_ptr(), 1 if use_fixed else 0,
                float(p.fixed_T) if use_fixed else 0.0, float(p.sigma_r), float(p.epsilon),
                _lib.RULES[p.truncation], log_2_over_eps(p.epsilon), self.plans[c].data_ptr(),
                self.terms[c].data_ptr(), TERMS_CAP, st), "plan")
            self._filter_channel(c, st, self.ws, self.prec)
            done = torch.cuda.Event()
            done.record(main)
            cs = self.copy_streams[c]
            cs.wait_event(done)
            with torch.cuda.stream(cs):
                host_outs[c].copy_(self.out[c], non_blocking=True)
        for cs in self.copy_streams:
            main.wait_stream(cs)
        return host_outs

    def finish(self, T_global=None, stream_ptr=None):
        """K2/K3/K4 per channel with the global T (device tensor, per channel)."""
        lib, s = self.lib, self.strip
        st = self._stream(stream_ptr)
        lo, hi = s.out_lo - s.buf_lo, s.out_hi - s.buf_lo
        p = self.params
        use_fixed = p.fixed_T is not None
        if T_global is not None:
            self.T.copy_(T_global)
        self.fb.zero_()
        if self.overlap:
            import torch
            main = self._stream_obj(stream_ptr)
            ev = torch.cuda.Event()
            ev.record(main)
        for c, b in enumerate(self.bufs):
            cst, ws = st, self.ws
            if self.overlap:
                self.side[c].wait_event(ev)
                cst, ws = self.side[c].cuda_stream, self.side_ws[c]
            _lib.check(lib.sbf_plan_device(
                self.T[c:c + 1].data_ptr(), 1 if use_fixed else 0,
                float(p.fixed_T) if use_fixed else 0.0, float(p.sigma_r), float(p.epsilon),
                _lib.RULES[p.truncation], log_2_over_eps(p.epsilon), self.plans[c].data_ptr(),
                self.terms[c].data_ptr(), TERMS_CAP, cst), "plan")
            self._filter_channel(c, cst, ws, self.prec)
        if self.overlap:
            for c in range(len(self.bufs)):
                e = torch.cuda.Event()
                e.record(self.side[c])
                main.wait_event(e)
        return self.out

    def check(self, stream_ptr=None):
        """Host-side validation after run()/finish() (one read-back of the
        plans, statistics and fallback counts; synchronises the stream):
        raises InvalidParameterError on non-finite input or a failed plan,
        re-runs a channel the device flagged (HDR range guard, or an order
        whose ceil(0.405 q^2) is ambiguous at 2 ulp — re-planned with the host
        twin), and returns [(KernelPlan, fallback_pixels)] per channel, with a
        RuntimeWarning for fallbacks, like shiftable_bf."""
        import warnings

        import torch

        from .kernels import select_plan

        st = self._stream(stream_ptr)
        self._stream_obj(stream_ptr).synchronize()
        out = []
        stats = self.stats.cpu().numpy()
        for c in range(len(self.bufs)):
            if int(stats[c, 7:8].view(np.uint64)[0]) != 0:
                raise InvalidParameterError(f"channel {c} contains non-finite samples")
            pl = _lib.SbfPlan.from_buffer_copy(self.plans[c].cpu().numpy().tobytes())
            _lib.check(pl.status, "plan")
            p = self.params
            if pl.flags & (_lib.PLAN_NEEDS_HDR | _lib.PLAN_N_AMBIGUOUS):
                prec = _lib.PREC_HDR if pl.flags & _lib.PLAN_NEEDS_HDR else self.prec
                if pl.flags & _lib.PLAN_N_AMBIGUOUS:
                    ph = select_plan(pl.T, p.sigma_r, p.epsilon, truncation=p.truncation)
                    use_fixed = p.fixed_T is not None
                    _lib.check(self.lib.sbf_plan_device_forced(
                        self.T[c:c + 1].data_ptr(), 1 if use_fixed else 0,
                        float(p.fixed_T) if use_fixed else 0.0, float(p.sigma_r),
                        float(p.epsilon), _lib.RULES[p.truncation], log_2_over_eps(p.epsilon),
                        ph.N, ph.M, self.plans[c].data_ptr(), self.terms[c].data_ptr(),
                        TERMS_CAP, st), "plan")
                self.fb[c:c + 1].zero_()
                torch.cuda.current_stream(self.dev).synchronize()
                self._filter_channel(c, st, self.ws, prec)
                self._stream_obj(stream_ptr).synchronize()
                pl = _lib.SbfPlan.from_buffer_copy(self.plans[c].cpu().numpy().tobytes())
            fb = int(self.fb[c].item())
            if fb:
                warnings.warn(f"channel {c}: {fb} pixel(s) had a non-positive normalizer; "
                              "input values kept", RuntimeWarning, stacklevel=2)
            out.append((_plan_from_struct(pl), fb))
        return out

    def launches_per_run(self):
        """Kernels of this library one run() launches (fp32 paths): per channel
        K1 (pruned exact T on strips of at least 4 Mpx: init, tile pass,
        bounds, two exact rounds, final; else the two line passes), the plan,
        and the filter (K3 sweep + divide, or the persistent split sweep + K4)
        -- profiles/r2_step_launches_cfg5.csv."""
        k1 = 6 if self.H * self.W >= (4 << 20) and self.R <= 48 else 2
        return len(self.bufs) * (k1 + 1 + 2)

    def _filter_channel(self, c, st, ws, prec):
        s = self.strip
        lo, hi = s.out_lo - s.buf_lo, s.out_hi - s.buf_lo
        _lib.check(self.lib.sbf_filter(
            self.bufs[c].data_ptr(), self.dt[c], self.H, self.W, self.W, s.buf_lo, self.img_H, lo,
            hi, self.sp, self.plans[c].data_ptr(), self.terms[c].data_ptr(),
            self.stats[c].data_ptr(), prec, self.out[c].data_ptr(), self.dt[c],
            self.fb[c:c + 1].data_ptr(), ws.data_ptr(), ws.numel(), st), "filter")

    def plans_host(self):
        return [_plan_from_struct(_lib.SbfPlan.from_buffer_copy(self.plans[c].cpu().numpy().tobytes()))
                for c in range(len(self.bufs))]


def gather_strips(outs: Sequence[np.ndarray], strips: Sequence[Strip]) -> np.ndarray:
    """Stack per-rank owned rows back into the full image (host helper)."""
    order = sorted(range(len(strips)), key=lambda i: strips[i].out_lo)
    return np.concatenate([np.asarray(outs[i]) for i in order], axis=0)
