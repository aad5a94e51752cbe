"""Benchmark contract for the B200 shiftable bilateral filter.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 2] [--no-cpu-baseline]

One "step" = one pass of the hot path over one image of the workload:
K1 local range -> K2 device plan -> K3 fused term kernel -> K4 epilogue,
input resident in HBM, no host synchronisation inside the step.  Default
workload: BASELINE.json configs[1] (1024x1024 float32, sigma_s=5,
sigma_r=10, eps=0.01), seeded synthetic input.
L2 (126 MB) is flushed between timed steps by writing a 256 MiB buffer.
Multi-GPU (torchrun): config 2 is single-GPU by definition, so every rank
filters its own replica (weak scaling, no collective on the data path);
timing is max over ranks of device-event time.
Prints exactly one JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import gc
import json
import multiprocessing as mp
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# our kernels per filtered image (fused pipeline): row max (+ statistics
# reset), column max (+ accumulator clear; statistics and the plan in its
# last CTA), term sweep (K3), epilogue (K4)
KERNELS_PER_IMAGE = 4
# the strip path (config 5) plans all channels after the T all-reduce:
# row max, column max, plan, K3, K4
KERNELS_STRIP_IMAGE = 5
METRIC = "Mpixel/s shiftable Gaussian BF at 1/2/4/8 B200; % of FP32/HBM roofline"
UNIT = "Mpixel/s"
OPS_PER_PX_TERM = 132   # phasor 4 + f*c,f*s 2 + 4 images x 6 line passes x 5 + acc 6
OPS_PER_PX = 10         # local range ~8 + divide ~2
L2_FLUSH_BYTES = 256 << 20


def _cfg_params(cfg):
    from paper_1203_5128_b200.workloads import CONFIGS
    return CONFIGS[cfg]


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
# CPU baseline (the oracle port; reference-arm and cpu_baseline leg only)
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


def cpu_baseline(cfg=2, min_band_rows=32, max_procs=None):
    """Time the CPU oracle (float64 C restatement of the reference path,
    oracle/sbf_oracle.c — bit-identical to the reference on the golden cases
        and ~2.5x faster than its numpy/Cython original) on the whole image of
    the config, cut into one band of output rows per host core (halo =
    support, fixed_T = global T: the strip equivalence of SURVEY.md
    Appendix C).  Returns (Mpix/s, cores, sample text)."""
    from oracle import coracle as CO
    from oracle import shiftbf_oracle as O
    from paper_1203_5128_b200.workloads import config_image
    CO.build()
    p = _cfg_params(cfg)
    img = config_image(cfg).astype(np.float64)
    r, a = O.extended_box_params(p["sigma_s"], 3)
    halo = 3 * (r + (1 if a > 0 else 0))
    T = CO.compute_T(img, max(1, halo))
    # whole image when it is small (configs 1, 2), else a leading block of
    # rows holding ~8 Mpixel (configs 3-5): bounded CPU time and memory
    H = min(img.shape[0], max(min_band_rows, int(8e6) // img.shape[1]))
    procs = max(1, min(max_procs or os.cpu_count() or 1, H // min_band_rows))
    band_rows = -(-H // procs)
    jobs = []
    for y0 in range(0, H, band_rows):
        y1 = min(H, y0 + band_rows)
        a, b = max(0, y0 - halo), min(img.shape[0], y1 + halo)
        jobs.append((img[a:b], y1 - y0, T, p))
    # spawn (the caller holds CUDA threads); workers are started and warmed
    # before the clock starts, then one band per worker is timed
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(len(jobs) + 1)
    with ctx.Pool(len(jobs), initializer=_cpu_init, initargs=(barrier,)) as pool:
        barrier.wait()
        # repeat the sample until ~10 s of CPU work (all cores) have been timed
        t = time.perf_counter()
        res = pool.map(_cpu_band, jobs, chunksize=1)
        reps = 1
        while (time.perf_counter() - t) * len(jobs) < 10.0 and reps < 8:
            res = pool.map(_cpu_band, jobs, chunksize=1)
            reps += 1
        wall = time.perf_counter() - t
    px = reps * sum(x[0] for x in res)
    what = "whole image" if H == img.shape[0] else f"first {H} rows"
    sample = (f"C oracle (oracle/sbf_oracle.c, float64), {what}: {len(jobs)} bands x "
              f"{band_rows} rows x {img.shape[1]} cols of {p['name']} "
              f"(halo {halo}, fixed global T={T:.6g}, N={res[0][2]}, M={res[0][3]}), "
              f"{procs} processes, {reps} repetition(s), wall {wall:.2f}s")
    return px / wall / 1e6, procs, sample


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
    return best / 1e12, sms


def load_profile_traffic():
    """dram bytes per K3 launch from the committed ncu --set full summary."""
    path = os.path.join(REPO, "profiles", "k3_traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch")
    except Exception:
        return None


def run_ours(args, rank, world, dev):
    import torch

    import paper_1203_5128_b200 as P
    from paper_1203_5128_b200 import _lib
    from paper_1203_5128_b200.kernels import log_2_over_eps
    from paper_1203_5128_b200.spatial import to_c_spatial
    from paper_1203_5128_b200.workloads import config_image

    lib = _lib.load()
    p = _cfg_params(args.config)
    img_np = config_image(args.config)
    H, W = img_np.shape
    f = torch.from_numpy(np.ascontiguousarray(img_np)).to(dev)
    dt = _lib.SBF_F64 if f.dtype == torch.float64 else _lib.SBF_F32
    # default parameters, as a user calls it (precision "auto": fp32 kernels
    # with the device-side HDR guard); the device-resident step below passes
    # SBF_PREC_FP32 explicitly, which runs the same kernels
    params = P.FilterParams(sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], epsilon=p["epsilon"])
    sp = to_c_spatial(params.resolved_spatial())
    R = params.resolved_radius()
    prec = _lib.PREC_FP32
    cap = 1 << 16
    stats = torch.empty(8, dtype=torch.float64, device=dev)
    plan = torch.empty(64, dtype=torch.uint8, device=dev)
    out = torch.empty((H, W), dtype=torch.float32, device=dev)
    fb = torch.zeros(1, dtype=torch.int64, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    sptr = st.cuda_stream
    l2e = log_2_over_eps(p["epsilon"])

    # one step = the fused device pipeline (sbf_shiftable_bf: K1 with the plan
    # and the accumulator clear folded in, K3, K4, programmatic dependent
    # launches); events 2/3 are recorded by the library around the K3 launch
    pws = torch.empty(lib.sbf_shiftable_bf_workspace(H, W, dt, sp, prec, cap), dtype=torch.uint8,
                      device=dev)

    def step(evs=None):
        if evs is not None:
            evs[0].record(st)
            lib.sbf_set_k3_events(evs[2].cuda_event, evs[3].cuda_event)
        _lib.check(lib.sbf_shiftable_bf(f.data_ptr(), dt, H, W, sp, R, -1.0, p["sigma_r"],
                                        p["epsilon"], 0, l2e, prec, out.data_ptr(), _lib.SBF_F32,
                                        plan.data_ptr(), stats.data_ptr(), fb.data_ptr(), cap,
                                        pws.data_ptr(), pws.numel(), sptr))
        if evs is not None:
            lib.sbf_set_k3_events(None, None)
            evs[4].record(st)

    for _ in range(args.warmup):
        step()
        flush.zero_()
    torch.cuda.synchronize()
    planc = _lib.SbfPlan.from_buffer_copy(plan.cpu().numpy().tobytes())
    # parity spot check of the benchmarked output (cheap invariants)
    o = out.cpu().numpy()
    assert np.isfinite(o).all() and o.min() >= img_np.min() - 1e-3 and o.max() <= img_np.max() + 1e-3

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    evsets = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    for es in evsets:  # materialise the event handles handed to the library
        for e in es:
            e.record(st)
    torch.cuda.synchronize()
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        for k in range(args.steps):
            step(evsets[k])
            flush.zero_()
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    step_ms = [e[0].elapsed_time(e[4]) for e in evsets]
    k3_ms = [e[2].elapsed_time(e[3]) for e in evsets]
    k1_ms = [e[0].elapsed_time(e[2]) for e in evsets]  # K1 (+ fused plan / clear)
    total_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    px = H * W
    value = world * px * args.steps / (total_ms * 1e-3) / 1e6

    # e2e through the public API from pinned host memory (input H2D + result D2H)
    pinned = torch.from_numpy(np.ascontiguousarray(img_np)).pin_memory()
    res = None
    for _ in range(max(3, args.warmup)):
        # keep the previous result alive exactly like the timed loop, so the
        # pinned-host caching allocator holds both result blocks before timing
        res = P.shiftable_bf(pinned, params)
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()  # no collector pauses inside the timed region
    e2e_ms = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        res = P.shiftable_bf(pinned, params)
        e1.record(st)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
        flush.zero_()
    gc.enable()
    e2e_total = float(np.sum(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = world * px * args.steps / (e2e_total * 1e-3) / 1e6
    h2d = img_np.nbytes
    # result (the input's float dtype for torch input) + plan + stats + fallback counter
    d2h = px * res.image.element_size() + 64 + 64 + 8

    peak_meas, sms = fp32_peak(lib, torch, dev)
    peak_meas2, _ = fp32_peak(lib, torch, dev, packed=True)
    peak_nominal = sms * 128 * 1.965e9 / 1e12
    k3_avg = float(np.mean(k3_ms))
    ops = OPS_PER_PX_TERM * px * planc.K_eval
    achieved = ops / (k3_avg * 1e-3) / 1e12
    geo = ctypes_int7()
    lib.sbf_filter_geometry(H, W, sp, prec, geo)
    return dict(
        value=value, ms_per_step=ms_per_step, planc=planc, k3_avg=k3_avg, k1_avg=float(np.mean(k1_ms)),
        e2e=dict(value=e2e_value, unit=UNIT, h2d_bytes_per_step=int(h2d), d2h_bytes_per_step=int(d2h),
                 ms_per_step=e2e_total / args.steps),
        roofline=dict(bound="fp32", achieved=achieved, peak=peak_nominal, unit="TFLOP/s",
                      frac=achieved / peak_nominal, traffic=load_profile_traffic(),
                      peak_source="nominal 148 SM x 128 FP32 lanes x 1.965 GHz (ops: FADD/FMUL/FFMA = 1)",
                      peak_measured_ffma=peak_meas, peak_measured_ffma2=peak_meas2,
                      frac_of_measured=achieved / max(peak_meas, peak_meas2),
                      kernel="sbf::terms_kernel<4,3,0> (K3)",
                      ops_per_launch=ops, ops_basis=f"{OPS_PER_PX_TERM} ops/px/evaluated term x {px} px x {planc.K_eval} terms"),
        clocks=clk.summary(), geometry=list(geo), W=W, H=H, p=p)


def _device_plan_cost(lib, torch, f, params, dev):
    """(K_eval of the image's plan) — used to balance the config-4 shards."""
    import paper_1203_5128_b200 as P
    res = P.shiftable_bf(f, params)
    return res.plan.N // 2 - res.plan.M + 1


def run_batch(args, rank, world, dev):
    """Config 4: a batch of independent images sharded across ranks."""
    import torch

    import paper_1203_5128_b200 as P
    from paper_1203_5128_b200 import _lib
    from paper_1203_5128_b200.dist import shard_images
    from paper_1203_5128_b200.kernels import log_2_over_eps
    from paper_1203_5128_b200.spatial import to_c_spatial
    from paper_1203_5128_b200.workloads import config_image

    lib = _lib.load()
    p = _cfg_params(args.config)
    n_img = args.images
    params = P.FilterParams(sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], epsilon=p["epsilon"])
    sp = to_c_spatial(params.resolved_spatial())
    R = params.resolved_radius()
    # balance ranks by px * K.  Every rank plans every image
    # (K1 + host plan twin, outside the timed region) so the LPT sharding is
    # identical on all ranks without communication.
    ks_all = []
    for i in range(n_img):
        g = torch.from_numpy(np.ascontiguousarray(config_image(4, i))).to(dev)
        pl = P.select_plan(P.compute_T(g, R), p["sigma_r"], p["epsilon"])
        ks_all.append(pl.N // 2 - pl.M + 1)
        del g
    parts = shard_images([float(k) for k in ks_all], world)
    mine = parts[rank]
    imgs = [torch.from_numpy(np.ascontiguousarray(config_image(4, i))).to(dev) for i in mine]
    H, W = imgs[0].shape
    cap = 1 << 16
    st = torch.cuda.current_stream()
    l2e = log_2_over_eps(p["epsilon"])
    # images alternate between `lanes` streams (own workspace, plan, stats):
    # one image's K1 and K3 start fills the SMs the previous image's K3
    # leaves idle while its last items finish
    lanes = []
    for _ in range(max(1, args.lanes)):
        lanes.append(dict(
            stream=torch.cuda.Stream(device=dev) if args.lanes > 1 else st,
            ws=torch.empty(lib.sbf_shiftable_bf_workspace(H, W, _lib.SBF_F32, sp, _lib.PREC_FP32,
                                                          cap), dtype=torch.uint8, device=dev),
            stats=torch.empty(8, dtype=torch.float64, device=dev),
            plan=torch.empty(64, dtype=torch.uint8, device=dev),
            fb=torch.zeros(1, dtype=torch.int64, device=dev)))
    outs = [torch.empty((H, W), dtype=torch.float32, device=dev) for _ in mine]

    def step():
        for i, (f, o) in enumerate(zip(imgs, outs)):
            ln = lanes[i % len(lanes)]
            _lib.check(lib.sbf_shiftable_bf(f.data_ptr(), _lib.SBF_F32, H, W, sp, R, -1.0,
                                            p["sigma_r"], p["epsilon"], 0, l2e, _lib.PREC_FP32,
                                            o.data_ptr(), _lib.SBF_F32, ln["plan"].data_ptr(),
                                            ln["stats"].data_ptr(), ln["fb"].data_ptr(), cap,
                                            ln["ws"].data_ptr(), ln["ws"].numel(),
                                            ln["stream"].cuda_stream))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index or 0) as clk:
        e0.record(st)
        for ln in lanes:
            ln["stream"].wait_event(e0)
        for _ in range(args.steps):
            step()
        for ln in lanes:
            st.wait_stream(ln["stream"])
        e1.record(st)
        e1.synchronize()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    total = float(t.item())
    px = n_img * H * W
    # algorithmic FP32 ops of the whole batch (132 per pixel per
    # evaluated folded term); K per image from the host twin of the plan
    kt = torch.tensor([float(sum(ks_all))], dtype=torch.float64)
    ops = OPS_PER_PX_TERM * H * W * float(kt.item())
    achieved = ops * args.steps / (total * 1e-3) / 1e12
    peak = 148 * 128 * 1.965e9 / 1e12
    return dict(value=px * args.steps / (total * 1e-3) / 1e6, ms_per_step=total / args.steps,
                launches=KERNELS_PER_IMAGE * len(mine) * args.steps, clocks=clk.summary(),
                roofline=dict(bound="fp32", achieved=achieved, peak=peak * world, unit="TFLOP/s",
                              frac=achieved / (peak * world), traffic=None,
                              kernel="whole step (K1..K4 over the batch, all ranks)",
                              ops_basis=f"{OPS_PER_PX_TERM} ops/px/term x {H}x{W} px x sum K = {int(kt.item())}"),
                config=dict(workload=p["name"], images=n_img, H=H, W=W, sigma_s=p["sigma_s"],
                            sigma_r=p["sigma_r"], epsilon=p["epsilon"],
                            parallelism=f"image batch sharded over {world} rank(s) by px*K (LPT), no collective",
                            sum_K=int(sum(ks_all)), rank_K=[int(sum(ks_all[i] for i in part)) for part in parts],
                            l2="inputs (64 MiB/image) exceed what L2 keeps across images"))


def run_strips(args, rank, world, dev):
    """Config 5: 3 channels, row strips + halos, global T by NCCL max-allreduce."""
    import torch

    import paper_1203_5128_b200 as P
    from paper_1203_5128_b200.dist import StripFilter, strip_halo, strip_plan
    from paper_1203_5128_b200.workloads import config_image

    p = _cfg_params(args.config)
    size = args.size or 16384
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
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    total = float(t.item())
    px = 3 * size * size
    plans = sf.plans_host()
    # r >= 9 runs the split sweep: K1 (2) + plan + 2 kernels per term + K4
    r_sp, _ = P.extended_box_params(p["sigma_s"], 3)
    if r_sp >= 9:
        per_step = sum(3 + 2 * (pl.N // 2 - pl.M + 1) + 1 for pl in plans)
    else:
        per_step = KERNELS_STRIP_IMAGE * 3
    ops = OPS_PER_PX_TERM * size * size * sum(pl.N // 2 - pl.M + 1 for pl in plans)
    achieved = ops * args.steps / (total * 1e-3) / 1e12
    peak = 148 * 128 * 1.965e9 / 1e12 * world
    return dict(value=px * args.steps / (total * 1e-3) / 1e6, ms_per_step=total / args.steps,
                launches=per_step * args.steps, clocks=clk.summary(),
                roofline=dict(bound="fp32", achieved=achieved, peak=peak, unit="TFLOP/s",
                              frac=achieved / peak, traffic=None,
                              kernel="whole step (K1, plan, split sweep / K3, K4; 3 channels, all ranks)",
                              ops_basis=f"{OPS_PER_PX_TERM} ops/px/term x {size}^2 px x sum K over channels"),
                config=dict(workload=p["name"], channels=3, H=size, W=size, sigma_s=p["sigma_s"],
                            sigma_r=p["sigma_r"], epsilon=p["epsilon"],
                            plans=[(pl.T, pl.N, pl.M) for pl in plans],
                            parallelism=f"row strips over {world} rank(s), halo {s.out_lo - s.buf_lo or s.buf_hi - s.out_hi} rows, "
                                        "global T by NCCL max-allreduce (3 x fp64, one call)"))


def ctypes_int7():
    import ctypes
    return (ctypes.c_int * 7)()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--images", type=int, default=64, help="config 4 batch size")
    ap.add_argument("--lanes", type=int, default=3,
                    help="config 4: streams the images alternate on (1: 6043, 2: 6118, 3: 6170, 6: 6078 Mpix/s); config 5: > 1 runs each channel on its own stream")
    ap.add_argument("--size", type=int, default=None, help="config 5 side (default 16384)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    p = _cfg_params(args.config)

    if args.impl == "reference":
        # the reference's CPU path (oracle port; the Python reference cannot
        # travel to the box) on the host cores, rank 0 only
        if rank != 0:
            return
        vals = []
        for _ in range(args.warmup):
            pass  # the port has no warm-up state; warm-up steps are not timed
        for k in range(args.steps):
            v, cores, sample = cpu_baseline(args.config, max_procs=None)
            vals.append(v)
        v = float(np.median(vals))
        line = dict(metric=METRIC, value=v, unit=UNIT, n_gpus=args.gpus, steps=args.steps,
                    warmup=args.warmup, ms_per_step=None, higher_is_better=True, scaling="weak",
                    vs_baseline=None, dtype="f64", data="synthetic (SURVEY.md Appendix A generator)",
                    config=dict(workload=p["name"], sigma_s=p["sigma_s"], sigma_r=p["sigma_r"],
                                epsilon=p["epsilon"]),
                    impl="reference",
                    cpu_baseline=dict(value=v, unit=UNIT, cores=cores, kind="port", sample=sample),
                    e2e=dict(value=v, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
        print(json.dumps(line))
        return

    import torch
    if world > 1:
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl")
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    if args.config in (4, 5):
        r = (run_batch if args.config == 4 else run_strips)(args, rank, world, dev)
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        if rank == 0:
            line = dict(metric=METRIC, value=r["value"], unit=UNIT, n_gpus=world, steps=args.steps,
                        warmup=args.warmup, ms_per_step=r["ms_per_step"], higher_is_better=True,
                        scaling="strong", vs_baseline=None,
                        dtype="f32", data="synthetic (SURVEY.md Appendix A generator, seeded)",
                        config=r["config"], roofline=r.get("roofline"),
                        gpu_launches=r["launches"], clocks=r["clocks"])
            print(json.dumps(line))
        return
    r = run_ours(args, rank, world, dev)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample = cpu_baseline(args.config)
        cpu = dict(value=v, unit=UNIT, cores=cores, kind="port", sample=sample)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    if rank != 0:
        return
    pl = r["planc"]
    geo = r["geometry"]
    line = dict(
        metric=METRIC, value=r["value"], unit=UNIT, n_gpus=world, steps=args.steps,
        warmup=args.warmup, ms_per_step=r["ms_per_step"], higher_is_better=True, scaling="weak",
        vs_baseline=None, dtype="f32",
        data="synthetic (SURVEY.md Appendix A generator, seeded; BASELINE names no dataset)",
        config=dict(workload=p["name"], H=r["H"], W=r["W"], sigma_s=p["sigma_s"],
                    sigma_r=p["sigma_r"], epsilon=p["epsilon"], T=pl.T, N=pl.N, M=pl.M, K=pl.K,
                    K_eval=pl.K_eval, parallelism=("replicas" if world > 1 else "single"),
                    l2="flushed between timed steps (256 MiB write)",
                    k3_geometry=dict(halo=geo[0], out_cols_per_strip=geo[1], threads=geo[2],
                                     band_rows=geo[3], strips=geo[4], bands=geo[5], groups=geo[6]),
                    k3_ms=r["k3_avg"], k1_ms=r["k1_avg"]),
        roofline=r["roofline"], cpu_baseline=cpu, e2e=r["e2e"],
        gpu_launches=KERNELS_PER_IMAGE * args.steps, clocks=r["clocks"])
    print(json.dumps(line))


if __name__ == "__main__":
    main()
