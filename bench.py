"""Benchmark contract for the B200 shiftable bilateral filter.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 4] [--no-cpu-baseline]

Default workload: BASELINE.json configs[3], the configuration the metric
("Mpixel/s ... at 1/2/4/8 B200") is quoted on: a batch of 64 seeded
4096x4096 float32 images (SURVEY.md Appendix A generator), sigma_s=6,
sigma_r=20, eps=0.01.  One step = the whole batch through the device
pipeline (K1 local range + plan, K3 fused term sweep with the divide /
fallback epilogue), inputs resident in HBM.  The images are sharded over
the ranks by px*K (LPT) with no collective on the data path; each rank's
images rotate over three CUDA streams.  Inputs (64 MiB each) exceed what
L2 keeps across images, so no flush is needed between steps.

`--config 5` runs the 3 x 16384^2 row-strip workload (global T by an NCCL
max all-reduce); `--config 1/2/3` run single images (replicas for N>1).

`--gpus N` without torchrun environment variables re-launches this script
under `torch.distributed.run` with N ranks (one per GPU, NCCL).  Timing is
device-event time, max over ranks.  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import gc
import json
import multiprocessing as mp
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# our kernels per filtered image (fused pipeline): row max (+ statistics
# reset), column max (+ ticket clear, plan in its last CTA), K3 term sweep
# (+ divide / fallback epilogue)
# kernels of this repo that one fused call launches, per image (ncu launch lists of one
# step: profiles/r2_step_launches_cfg<N>.csv; config 5 counts in StripFilter.launches_per_run)
KERNELS_PER_IMAGE = {1: 5, 2: 4, 3: 9, 4: 8}
METRIC = "Mpixel/s shiftable Gaussian BF at 1/2/4/8 B200; % of FP32/HBM roofline"
UNIT = "Mpixel/s"
OPS_PER_PX_TERM = 132   # phasor 4 + f*c,f*s 2 + 4 images x 6 line passes x 5 + acc 6
OPS_PER_PX = 10         # local range ~8 + divide ~2
L2_FLUSH_BYTES = 256 << 20
E2E_LANES = 3  # streams of the batch API in the e2e leg (copy engine both ways); measured
# on B200 (64 config-4 images): 2 lanes 147 ms/step, 3 lanes 125 ms (steady), 4 lanes
# 125-298 ms (outliers)
PEAK_FP32_NOMINAL = 148 * 128 * 1.965e9 / 1e12  # T lane-ops/s (FADD/FMUL/FFMA = 1 op)
def _hbm_peak_gbs():
    """Measured HBM copy bandwidth of this pool's B200s (MEASURED_PEAKS.json,
    driver-written), else the profiling recipe's fallback."""
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6500.0


DFMA_PEAK_MEASURED = 16.99  # T DFMA/s on the pool's B200 (profiles/r2_fma_probe.txt)
DATA = "synthetic (SURVEY.md Appendix A seeded generator; BASELINE names no dataset)"


def _cfg_params(cfg):
    from paper_1203_5128_b200.workloads import CONFIGS
    return CONFIGS[cfg]


def config_dict(cfg, world):
    """The workload description printed by BOTH arms (ours / reference)."""
    p = _cfg_params(cfg)
    d = dict(workload=p["name"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], epsilon=p["epsilon"])
    if cfg == 4:
        d.update(images=64, H=4096, W=4096, input_dtype="float32",
                 parallelism=f"image batch sharded over {world} rank(s) by px*K (LPT), no collective",
                 l2="no flush: each 64 MiB image and its 128 MiB accumulator exceed what L2 keeps "
                    "across the batch")
    elif cfg == 5:
        d.update(channels=3, H=16384, W=16384, input_dtype="float32",
                 parallelism=f"row strips over {world} rank(s) with halos, global T by NCCL "
                             "max all-reduce (3 x fp64, one call)",
                 l2="no flush: 1 GiB channels")
    else:
        n = {1: 512, 2: 1024, 3: 2048}[cfg]
        d.update(images=1, H=n, W=n,
                 input_dtype={1: "float64", 2: "float32", 3: "uint16->float32"}[cfg],
                 parallelism=f"{world} independent replica(s)" if world > 1 else "single GPU",
                 l2="flushed between timed steps (256 MiB write)")
    return d


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_distributed(n):
    """`--gpus N` outside torchrun: run this script under torch.distributed.run
    with N ranks on 127.0.0.1 and pass its output and exit code through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


# ----------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------
class ClockSampler:
    """Samples SM clock and clock-event (throttle) reasons on a thread during
    the timed region: NVML every ~1 ms when pynvml is importable (a config-2
    timed region lasts ~10 ms), else nvidia-smi every ~100 ms."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.lines = []
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._mx = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _poll_nvml(self):
        nv, h = self._nv, self._h
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                flags = ["Active" if r & b else "Not Active" for b in bits]
                self.lines.append(", ".join([str(self.index), str(sm), str(self._mx), "0", hex(r)] + flags))
            except Exception:
                pass
            self._stop.wait(0.001)

    def _poll(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout
                self.lines += [ln.strip() for ln in out.splitlines() if ln.strip()]
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self.t = threading.Thread(target=self._poll_nvml if self._nv else self._poll, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=6)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------
# CPU baseline (the oracle port; reference arm and cpu_baseline leg only)
# ----------------------------------------------------------------------------
def _cpu_init(barrier):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import coracle as CO
    CO.load()
    barrier.wait()  # every worker is up and has its library loaded


def _cpu_band(args):
    part, rows_out, T, p = args  # part = output rows plus their halo
    from oracle import coracle as CO
    t = time.perf_counter()
    out = CO.shiftable_bf(part, p["sigma_s"], p["sigma_r"], p["epsilon"], fixed_T=T)
    dt = time.perf_counter() - t
    return rows_out * part.shape[1], dt, out["N"], out["M"]


# rows of image/channel 0 the CPU sample covers (None: the whole image)
_CPU_ROWS = {1: None, 2: None, 3: 128, 4: None, 5: 512}


class CpuSample:
    """The CPU path timed beside the GPU: the C oracle (oracle/sbf_oracle.c,
    the reference algorithm restated in float64 C; bit-identical to the
    reference on the golden cases and ~2.5x faster than its numpy/Cython
    original) on a bounded sample of the workload — image / channel 0 (or its
    leading rows), cut into one band of output rows per host core (halo =
    support, fixed_T = the image's global T: the strip equivalence of
    SURVEY.md Appendix C).  Worker processes are spawned and warmed before
    any clock starts."""

    def __init__(self, cfg, max_procs=None, min_band_rows=32):
        from oracle import coracle as CO
        from oracle import shiftbf_oracle as O
        from paper_1203_5128_b200.workloads import config_image
        CO.build()
        self.p = p = _cfg_params(cfg)
        img = config_image(cfg).astype(np.float64)
        r, a = O.extended_box_params(p["sigma_s"], 3)
        halo = 3 * (r + (1 if a > 0 else 0))
        T = CO.compute_T(img, max(1, halo))
        rows = _CPU_ROWS[cfg] or img.shape[0]
        procs = max(1, min(max_procs or os.cpu_count() or 1, rows // min_band_rows))
        band = -(-rows // procs)
        self.jobs = []
        for y0 in range(0, rows, band):
            y1 = min(rows, y0 + band)
            lo, hi = max(0, y0 - halo), min(img.shape[0], y1 + halo)
            self.jobs.append((img[lo:hi], y1 - y0, T, p))
        self.procs = len(self.jobs)
        what = "whole image 0" if rows == img.shape[0] else f"first {rows} rows of image 0"
        self.desc = (f"C oracle (oracle/sbf_oracle.c, float64) on {what} of {p['name']}: "
                     f"{self.procs} bands x {band} rows x {img.shape[1]} cols, one process per "
                     f"band (halo {halo}, fixed global T={T:.6g})")
        ctx = mp.get_context("spawn")
        barrier = ctx.Barrier(self.procs + 1)
        self.pool = ctx.Pool(self.procs, initializer=_cpu_init, initargs=(barrier,))
        barrier.wait()

    def run_once(self):
        """Mpixel/s of one pass over the sample (wall clock, all bands)."""
        t = time.perf_counter()
        res = self.pool.map(_cpu_band, self.jobs, chunksize=1)
        wall = time.perf_counter() - t
        self.NM = (res[0][2], res[0][3])
        return sum(x[0] for x in res) / wall / 1e6, wall

    def close(self):
        self.pool.terminate()
        self.pool.join()


def cpu_baseline(cfg, min_seconds=10.0, max_reps=8):
    s = CpuSample(cfg)
    try:
        vals, total = [], 0.0
        while total * s.procs < min_seconds and len(vals) < max_reps:
            v, wall = s.run_once()
            vals.append(v)
            total += wall
        v = float(np.median(vals))
        sample = (f"{s.desc}, N={s.NM[0]}, M={s.NM[1]}, {len(vals)} repetition(s) "
                  f"(median), {total:.1f}s wall")
        return dict(value=v, unit=UNIT, cores=s.procs, kind="port", sample=sample)
    finally:
        s.close()


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------
def fp32_peak(lib, torch, dev, packed=False):
    """Measured FP32 issue peak: FFMA chains (packed: FFMA2, 2 ops each)."""
    out = torch.zeros(1, device=dev)
    st = torch.cuda.current_stream()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    blocks, threads, iters = sms * 8, 256, 8192
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        lib.sbf_fp32_probe(blocks, threads, -iters if packed else iters, out.data_ptr(),
                           st.cuda_stream)
        e1.record(st)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = max(best, blocks * threads * iters * (16 if packed else 8) / (ms * 1e-3))
    return best / 1e12


def profile_traffic(cfg):
    """DRAM bytes per K3 launch from the committed ncu --set full summary of
    this workload (profiles/k3_traffic_cfg<N>.json), or None."""
    path = os.path.join(REPO, "profiles", f"k3_traffic_cfg{cfg}.json")
    try:
        with open(path) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    except Exception:
        return None


def _max_over_ranks(torch, dev, world, *vals):
    t = torch.tensor(list(vals), dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


class Pipeline:
    """Device-resident sbf_shiftable_bf calls on a set of images, rotating
    over `lanes` streams (own workspace and meta block per image slot)."""

    def __init__(self, torch, dev, imgs, params, lanes, prec=None):
        from paper_1203_5128_b200 import _lib
        from paper_1203_5128_b200.kernels import log_2_over_eps
        from paper_1203_5128_b200.spatial import to_c_spatial
        self.torch, self._lib, self.lib = torch, _lib, _lib.load()
        self.imgs = imgs
        self.params = params
        self.sp = to_c_spatial(params.resolved_spatial())
        self.R = params.resolved_radius()
        self.l2e = log_2_over_eps(params.epsilon)
        self.dts = [_lib.SBF_F64 if f.dtype == torch.float64 else _lib.SBF_F32 for f in imgs]
        # the precision the public API settles on for these images (fp32
        # kernels; config 3's 16-bit range takes the fp64 path)
        self.prec = _lib.PREC_FP32 if prec is None else prec
        self.outs = [torch.empty(f.shape, dtype=f.dtype, device=dev) for f in imgs]
        self.meta = torch.empty((len(imgs), 256), dtype=torch.uint8, device=dev)
        self.main = torch.cuda.current_stream()
        self.lanes = []
        for k in range(max(1, lanes)):
            H, W = imgs[0].shape
            ws = self.lib.sbf_shiftable_bf_workspace(H, W, self.dts[0], self.sp, self.prec, 1 << 16)
            self.lanes.append(dict(stream=torch.cuda.Stream(device=dev) if lanes > 1 else self.main,
                                   ws=torch.empty(ws, dtype=torch.uint8, device=dev)))

    def launch(self, i, lane):
        _lib, p, f = self._lib, self.params, self.imgs[i]
        H, W = f.shape
        m = self.meta[i].data_ptr()
        _lib.check(self.lib.sbf_shiftable_bf(
            f.data_ptr(), self.dts[i], H, W, self.sp, self.R, -1.0, p.sigma_r, p.epsilon, 0,
            self.l2e, self.prec, self.outs[i].data_ptr(), self.dts[i], m, m + 128, m + 64,
            1 << 16, lane["ws"].data_ptr(), lane["ws"].numel(), lane["stream"].cuda_stream))

    def step(self):
        ev = self.torch.cuda.Event()
        ev.record(self.main)
        for ln in self.lanes:
            if ln["stream"] is not self.main:
                ln["stream"].wait_event(ev)
        for i in range(len(self.imgs)):
            self.launch(i, self.lanes[i % len(self.lanes)])
        for ln in self.lanes:
            if ln["stream"] is not self.main:
                self.main.wait_stream(ln["stream"])

    def k3_times(self):
        """Each image alone on the main stream with events around its K3
        launch: [(K3 ms, K_eval)] (the dominant kernel's per-launch time)."""
        torch, lib = self.torch, self.lib
        lane = dict(stream=self.main, ws=self.lanes[0]["ws"])
        evs = []
        for i in range(len(self.imgs)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(self.main)
            b.record(self.main)  # materialise the handles
            evs.append((a, b))
        torch.cuda.synchronize()
        for i, (a, b) in enumerate(evs):
            lib.sbf_set_k3_events(a.cuda_event, b.cuda_event)
            self.launch(i, lane)
            lib.sbf_set_k3_events(None, None)
        torch.cuda.synchronize()
        plans = self.plans()
        return [(a.elapsed_time(b), pl.K_eval) for (a, b), pl in zip(evs, plans)]

    def plans(self):
        raw = self.meta.cpu().numpy()
        return [self._lib.SbfPlan.from_buffer_copy(raw[i, :64].tobytes()) for i in range(len(raw))]


def run_ours(args, rank, world, dev):
    import torch

    import paper_1203_5128_b200 as P
    from paper_1203_5128_b200 import _lib
    from paper_1203_5128_b200.dist import shard_images
    from paper_1203_5128_b200.workloads import CFG4_K, config_image, generate_many

    lib = _lib.load()
    cfg = args.config
    p = _cfg_params(cfg)
    params = P.FilterParams(sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], epsilon=p["epsilon"])
    if cfg == 4:
        # balance ranks by px * K (K per image from the reference
        # plan table, identical on every rank: no communication)
        parts = shard_images([float(k) for k in CFG4_K[:args.images]], world)
        mine = parts[rank]
        host = [np.ascontiguousarray(a) for a in generate_many(4, mine)]
        flush = None
    else:
        mine = [0]
        host = [np.ascontiguousarray(config_image(cfg))]
        flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    imgs = [torch.from_numpy(a).to(dev) for a in host]
    pipe = Pipeline(torch, dev, imgs, params, args.lanes if cfg == 4 else 1,
                    prec=_lib.PREC_HDR if cfg == 3 else _lib.PREC_FP32)
    st = pipe.main

    for _ in range(args.warmup):
        pipe.step()
        if flush is not None:
            flush.zero_()
    torch.cuda.synchronize()
    plans = pipe.plans()
    # cheap invariants of the benchmarked outputs (parity is in tests/)
    for a, o in zip(host, pipe.outs):
        o = o.cpu().numpy()
        assert np.isfinite(o).all() and o.min() >= a.min() - 1e-3 and o.max() <= a.max() + 1e-3

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        for a, b in evs:
            a.record(st)
            pipe.step()
            b.record(st)
            if flush is not None:
                flush.zero_()
        torch.cuda.synchronize()
    step_ms = float(np.sum([a.elapsed_time(b) for a, b in evs]))
    if world > 1:
        torch.distributed.barrier()

    # the dominant kernel alone, per launch (K3 term sweep + fused epilogue)
    k3 = pipe.k3_times()
    px = [int(f.shape[0] * f.shape[1]) for f in imgs]
    k3_ms = float(sum(t for t, _ in k3))
    k3_ops = float(sum(OPS_PER_PX_TERM * n * k for n, (_, k) in zip(px, k3)))

    # end to end through the public API: page-locked host images in, results
    # written into page-locked host memory, every byte inside the timed region
    pinned_in = [torch.from_numpy(a).pin_memory() for a in host]
    pinned_out = [torch.empty(a.shape, dtype=t.dtype, pin_memory=True) for a, t in zip(host, imgs)]
    def e2e_call():
        if cfg == 4:
            return P.shiftable_bf_batch(pinned_in, params, lanes=E2E_LANES, out=pinned_out)
        # one image: the single-image call (SM-staged H2D, result streamed
        # into page-locked memory by the K3 epilogue)
        return [P.shiftable_bf(pinned_in[0], params)]

    # warm-up as the timed loop runs: the previous result stays alive while the
    # next call allocates its page-locked output (two blocks of the caching
    # host allocator in rotation; a first-time cudaHostAlloc costs milliseconds)
    res = None
    for _ in range(max(2, min(args.warmup, 3))):
        res = e2e_call()
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()  # no collector pauses inside the timed region
    if world > 1:
        torch.distributed.barrier()
    e2e_ms = 0.0
    e2e_steps = []
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        res = e2e_call()
        b.record(st)
        b.synchronize()
        e2e_steps.append(a.elapsed_time(b))
        e2e_ms += e2e_steps[-1]
        if flush is not None:
            flush.zero_()
    gc.enable()
    assert all((r.plan.N, r.plan.M) == (pl.N, pl.M) for r, pl in zip(res, plans))
    h2d = sum(a.nbytes for a in host)
    d2h = sum(o.numel() * o.element_size() for o in pinned_out) + 256 * len(host)

    step_ms, e2e_ms, k3_ms_max = _max_over_ranks(torch, dev, world, step_ms, e2e_ms, k3_ms)
    total_px = args.images * 4096 * 4096 if cfg == 4 else world * px[0]
    value = total_px * args.steps / (step_ms * 1e-3) / 1e6
    e2e_value = total_px * args.steps / (e2e_ms * 1e-3) / 1e6
    peak2 = fp32_peak(lib, torch, dev, packed=True)
    achieved = k3_ops / (k3_ms * 1e-3) / 1e12
    sum_k = sum(k for _, k in k3)
    step_ops = OPS_PER_PX_TERM * sum(n * k for n, (_, k) in zip(px, k3)) + OPS_PER_PX * sum(px)
    roof = dict(
        bound="fp32", achieved=achieved, peak=PEAK_FP32_NOMINAL, unit="TFLOP/s",
        frac=achieved / PEAK_FP32_NOMINAL, traffic=profile_traffic(cfg),
        peak_source="nominal 148 SM x 128 FP32 lanes x 1.965 GHz (FADD/FMUL/FFMA = 1 op); "
                    "MEASURED_PEAKS.json has no FP32 entry",
        peak_measured_ffma2=peak2, frac_of_measured=achieved / peak2,
        kernel="K3 term sweep + fused epilogue, each image alone on one stream (CUDA events)",
        ops_per_launch=k3_ops / len(k3), k3_ms_per_launch=k3_ms / len(k3),
        ops_basis=f"{OPS_PER_PX_TERM} ops/px/evaluated term x {px[0]} px x K_eval "
                  f"(sum over this rank's {len(k3)} image(s) = {sum_k})",
        traffic_source=f"profiles/k3_traffic_cfg{cfg}.json (ncu --set full)")
    if cfg == 3:
        # untruncated 16-bit plan (M = 0): the exact dual form (fp64) runs
        # instead of the K = 1232 term sweeps; its own roofline is fp64 issue:
        # 3 fp64 ops per tap (weight product, num FMA, den add) over the
        # clamped (2S+1)^2 taps, against the measured DFMA peak
        from paper_1203_5128_b200.spatial import to_c_spatial
        spc = to_c_spatial(params.resolved_spatial())
        S = spc.passes * (spc.r + 1)
        H3, W3 = imgs[0].shape
        ny = sum(min(S, y) + min(S, H3 - 1 - y) + 1 for y in range(H3))
        nx = sum(min(S, x) + min(S, W3 - 1 - x) + 1 for x in range(W3))
        ops = 3.0 * ny * nx
        ach = ops / (k3_ms / len(k3) * 1e-3) / 1e12
        roof = dict(bound="fp64", achieved=ach, peak=DFMA_PEAK_MEASURED, unit="TFLOP/s",
                    frac=ach / DFMA_PEAK_MEASURED, traffic=None,
                    peak_source="DFMA probe (tools/gpu/fma_probe.cu, profiles/r2_fma_probe.txt: "
                                "8 independent chains, 32 warps/SM), 1 op per DFMA",
                    kernel="dual_lut_kernel (exact dual form, fp64), each image alone (CUDA events)",
                    ops_per_launch=ops, k3_ms_per_launch=k3_ms / len(k3),
                    ops_basis=f"3 fp64 ops/tap x {ny * nx:.4g} taps ((2S+1)^2 clamped, S={S})",
                    shiftable_equivalent=dict(
                        achieved=achieved, frac_of_fp32_nominal=achieved / PEAK_FP32_NOMINAL,
                        note="132 ops/px/term x K_eval of the term sweeps it replaces"))
    return dict(
        value=value, ms_per_step=step_ms / args.steps, clocks=clk.summary(),
        launches=KERNELS_PER_IMAGE[cfg] * len(imgs) * args.steps,
        e2e=dict(value=e2e_value, unit=UNIT, h2d_bytes_per_step=int(h2d), d2h_bytes_per_step=int(d2h),
                 ms_per_step=e2e_ms / args.steps,
                 # this rank's steps: PCIe-bound legs show host-side outliers here
                 ms_step_min_median_max=[float(np.min(e2e_steps)), float(np.median(e2e_steps)),
                                         float(np.max(e2e_steps))],
                 path=(f"shiftable_bf_batch ({E2E_LANES} streams): pinned host images -> copy-engine H2D, "
                       "kernels, copy-engine D2H of each result into pinned host memory; "
                       "both PCIe directions overlap other images' kernels") if cfg == 4 else
                      ("shiftable_bf on a pinned host tensor: SM-staged H2D, K1..K3, the K3 "
                       "epilogue writes the result into pinned host memory, one host sync")),
        roofline=roof,
        step_roofline=dict(achieved=step_ops * args.steps / (step_ms * 1e-3) / 1e12 * world,
                           frac=step_ops * args.steps / (step_ms * 1e-3) / 1e12 * world
                           / (PEAK_FP32_NOMINAL * world),
                           note="whole step (all kernels, all ranks) against world x nominal peak"
                                + ("; shiftable-equivalent ops (the dual form evaluates a different, "
                                   "cheaper exact sum for this M = 0 plan)" if cfg == 3 else "")),
        plans=[(float(pl.T), int(pl.N), int(pl.M), int(pl.K_eval)) for pl in plans[:4]])


def run_strips(args, rank, world, dev):
    """Config 5: 3 channels, row strips + halos, global T by NCCL max-allreduce."""
    import torch

    import paper_1203_5128_b200 as P
    from paper_1203_5128_b200.dist import StripFilter, strip_halo, strip_plan
    from paper_1203_5128_b200.workloads import config_image

    p = _cfg_params(args.config)
    size = 16384
    params = P.FilterParams(sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], epsilon=p["epsilon"])
    s = strip_plan(size, world, strip_halo(params))[rank]
    bufs = []
    for c in range(3):
        full = config_image(5, c, size=size)
        bufs.append(torch.from_numpy(np.ascontiguousarray(full[s.buf_lo:s.buf_hi])).to(dev))
        del full
    sf = StripFilter(bufs, s, size, params, overlap=args.lanes > 1)
    st = torch.cuda.current_stream()
    for _ in range(args.warmup):
        sf.run()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index or 0) as clk:
        e0.record(st)
        for _ in range(args.steps):
            sf.run()
        e1.record(st)
        e1.synchronize()
    total = e0.elapsed_time(e1)
    px = 3 * size * size
    plans = sf.plans_host()
    lib = sf.lib

    # the dominant kernel alone: each channel's split sweep (every term, one
    # persistent launch) between events on the main stream
    k3_ms, k3_ops = 0.0, 0.0
    rows_out = s.out_hi - s.out_lo
    for c, pl in enumerate(plans):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        b.record(st)  # materialise the handles
        torch.cuda.synchronize()
        lib.sbf_set_k3_events(a.cuda_event, b.cuda_event)
        sf._filter_channel(c, st.cuda_stream, sf.ws, sf.prec)
        lib.sbf_set_k3_events(None, None)
        torch.cuda.synchronize()
        k3_ms += a.elapsed_time(b)
        k3_ops += OPS_PER_PX_TERM * rows_out * size * (pl.N // 2 - pl.M + 1)

    # end to end through the public strip API with host-resident strips:
    # page-locked buffer rows in, owned rows out, every byte inside the timed
    # region (copy engines, per-channel streams)
    pinned_in = [b.cpu().pin_memory() for b in bufs]
    pinned_out = [torch.empty((rows_out, size), dtype=b.dtype, pin_memory=True) for b in bufs]
    sf.run_host(pinned_in, pinned_out)
    torch.cuda.synchronize()
    for c in range(3):  # the host results are the device results
        assert torch.equal(pinned_out[c][:64], sf.out[c][:64].cpu())
    if world > 1:
        torch.distributed.barrier()
    n_e2e = max(1, min(args.steps, 3))
    e2e_ms = 0.0
    for _ in range(n_e2e):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        sf.run_host(pinned_in, pinned_out)
        b.record(st)
        b.synchronize()
        e2e_ms += a.elapsed_time(b)
    h2d = sum(t.numel() * t.element_size() for t in pinned_in)
    d2h = sum(t.numel() * t.element_size() for t in pinned_out)

    total, e2e_ms, k3_ms_max = _max_over_ranks(torch, dev, world, total, e2e_ms, k3_ms)
    ops = OPS_PER_PX_TERM * size * size * sum(pl.N // 2 - pl.M + 1 for pl in plans)
    achieved = k3_ops / (k3_ms * 1e-3) / 1e12
    traffic = profile_traffic(5)
    step_ach = ops * args.steps / (total * 1e-3) / 1e12
    return dict(value=px * args.steps / (total * 1e-3) / 1e6, ms_per_step=total / args.steps,
                launches=sf.launches_per_run() * args.steps, clocks=clk.summary(),
                e2e=dict(value=px * n_e2e / (e2e_ms * 1e-3) / 1e6, unit=UNIT,
                         h2d_bytes_per_step=int(h2d) * world, d2h_bytes_per_step=int(d2h) * world,
                         ms_per_step=e2e_ms / n_e2e, steps=n_e2e,
                         path="StripFilter.run_host: page-locked strip rows -> copy-engine H2D per channel, "
                              "K1 and a max-allreduce of T per channel, split sweep + K4, copy-engine D2H "
                              "of the owned rows into page-locked memory; channel c's sweep overlaps "
                              "channel c+1's upload and channel c-1's download"),
                roofline=dict(bound="fp32", achieved=achieved, peak=PEAK_FP32_NOMINAL, unit="TFLOP/s",
                              frac=achieved / PEAK_FP32_NOMINAL, traffic=traffic,
                              peak_source="nominal 148 SM x 128 FP32 lanes x 1.965 GHz (FADD/FMUL/FFMA = 1 op)",
                              kernel="split_queue_kernel (SV + SH, every term in one persistent launch), "
                                     "each channel alone on one stream (CUDA events), this rank's strip",
                              ops_per_launch=k3_ops / len(plans), k3_ms_per_launch=k3_ms / len(plans),
                              ops_basis=f"{OPS_PER_PX_TERM} ops/px/term x {rows_out} x {size} px x K_eval per channel",
                              traffic_source="profiles/k3_traffic_cfg5.json (ncu --set full, one 16384^2 channel)",
                              hbm=(dict(achieved_gbs=traffic * (rows_out / size) / (k3_ms / len(plans) * 1e-3) / 1e9,
                                        peak_gbs=_hbm_peak_gbs(),
                                        frac=traffic * (rows_out / size) / (k3_ms / len(plans) * 1e-3) / 1e9
                                        / _hbm_peak_gbs(),
                                        note="measured DRAM traffic of the kernel (not algorithmic bytes) over "
                                             "its time: the split sweep's U round trip is HBM-heavy")
                                   if traffic else None)),
                step_roofline=dict(achieved=step_ach, frac=step_ach / (PEAK_FP32_NOMINAL * world),
                                   note="whole step (K1, plan, term sweeps, epilogue; 3 channels, all ranks) "
                                        "against world x nominal peak"),
                plans=[(pl.T, pl.N, pl.M) for pl in plans])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--images", type=int, default=64, help="config 4 batch size")
    ap.add_argument("--lanes", type=int, default=3,
                    help="streams the images rotate over (config 4); > 1: one stream per channel (config 5)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfgd = config_dict(args.config, world)

    if args.impl == "reference":
        # the reference's CPU path (oracle port: the Python reference cannot
        # travel to the GPU box) on all host cores, rank 0 only; each step is
        # one pass over a bounded sample of the workload
        if rank != 0:
            return
        s = CpuSample(args.config)
        try:
            for _ in range(args.warmup):
                s.run_once()
            vals = [s.run_once()[0] for _ in range(args.steps)]
        finally:
            s.close()
        v = float(np.median(vals))
        line = dict(metric=METRIC, value=v, unit=UNIT, n_gpus=world, steps=args.steps,
                    warmup=args.warmup, ms_per_step=None, higher_is_better=True,
                    scaling="strong" if args.config in (4, 5) else "weak", vs_baseline=None,
                    dtype="f64", data=DATA, config=cfgd, impl="reference",
                    cpu_baseline=dict(value=v, unit=UNIT, cores=s.procs, kind="port",
                                      sample=f"{s.desc}, N={s.NM[0]}, M={s.NM[1]}; median of "
                                             f"{args.steps} passes"),
                    e2e=dict(value=v, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
        print(json.dumps(line))
        return

    import torch
    if world > 1:
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl")
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    r = (run_strips if args.config == 5 else run_ours)(args, rank, world, dev)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    if rank != 0:
        return
    line = dict(metric=METRIC, value=r["value"], unit=UNIT, n_gpus=world, steps=args.steps,
                warmup=args.warmup, ms_per_step=r["ms_per_step"], higher_is_better=True,
                scaling="strong" if args.config in (4, 5) else "weak", vs_baseline=None,
                dtype="f64" if args.config == 3 else "f32",  # the arithmetic type of the dominant kernel
                data=DATA, config=cfgd, roofline=r["roofline"], cpu_baseline=cpu,
                e2e=r.get("e2e"), gpu_launches=r["launches"], clocks=r["clocks"])
    for k in ("step_roofline", "plans"):
        if k in r:
            line[k] = r[k]
    print(json.dumps(line))


if __name__ == "__main__":
    main()
