"""Generate golden vectors from the REFERENCE implementation (run in the dev
container only; /root/reference does not exist on the GPU box).

    python tests/golden/make_golden.py [--big]

Imports the reference package `shiftbf` from /root/reference/pkg/src (its
pure-numpy line-kernel backend; the compiled backend agrees to 1e-12 per
the reference's own test_backends.py) and writes small .npz fixtures next to
this script.  `--big` also computes T/N/M of configs 2-5 (minutes).

The fixtures pin the oracle (tests/test_oracle_golden.py) and are the
known-answer vectors for the CUDA parity tests.
"""

import argparse
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import shiftbf  # noqa: E402  (reference)
from shiftbf import kernels as rk  # noqa: E402
from shiftbf import maxfilter as rm  # noqa: E402
from shiftbf import spatial as rs  # noqa: E402
from shiftbf.bilateral import FilterParams, shiftable_bf  # noqa: E402

from paper_1203_5128_b200.workloads import config_image  # noqa: E402


def plans():
    rng = np.random.default_rng(7)
    rows = []
    sigmas = [5.0, 8.0, 10.0, 10.0000001, 10.5, 15.0, 20.0, 30.0, 39.9, 40.0,
              40.5, 60.0, 100.0, 800.0]
    eps_list = [0.0, 0.005, 0.01, 0.02, 0.05, 0.25]
    Ts = [0.0, 1.0, 17.5, 100.0, 251.39522633396712, 237.54737095534801, 255.0,
          62376.0, 253.45146048069, 245.72779846191406, 236.57716369628906]
    Ts += list(rng.uniform(0, 300, 40)) + list(rng.uniform(0, 3000, 10))
    rules = ["auto", "exact", "chernoff", "none"]
    for T in Ts:
        for sr in sigmas:
            for eps in eps_list:
                for rule in rules:
                    needs_exact = rule == "exact" or (rule == "auto" and 10 < sr <= 40)
                    if needs_exact and eps > 0 and rk.order_threshold(T, sr) > 3000:
                        continue
                    p = rk.select_plan(T, sr, eps, truncation=rule)
                    rows.append((T, sr, eps, rules.index(rule), p.N, p.M))
    arr = np.array(rows, dtype=np.float64)
    # N0 table (test_kernels.py:40-45) and chernoff/exact pins
    n0 = {s: rk.order_threshold(255, s, mode="round") for s in (5, 10, 20, 30, 40, 60, 80, 100)}
    exact = [(N, e, rk.truncation_index_exact(N, e))
             for N in (1, 2, 3, 4, 5, 29, 47, 66, 101, 109, 118, 229, 263, 700, 2463)
             for e in (0.005, 0.01, 0.05, 0.5)]
    chern = [(N, e, rk.truncation_index_chernoff(N, e))
             for N in (1, 2, 29, 229, 263, 700, 2463) for e in (0.005, 0.01, 0.05)]
    np.savez_compressed(os.path.join(HERE, "plans.npz"), plans=arr,
                        n0=np.array(list(n0.items()), dtype=np.float64),
                        exact=np.array(exact, dtype=np.float64),
                        chernoff=np.array(chern, dtype=np.float64))
    # weights/frequencies for a few plans
    wts = {}
    for (N, M, sr) in ((2, 0, 1.0), (29, 7, 30.0), (229, 79, 10.0), (263, 111, 10.0), (2463, 0, 800.0)):
        e = rk.raised_cosine_expansion(rk.KernelPlan(rk.KernelFamily.RAISED_COSINE, sr, 1.0, N, M,
                                                     0.0 if M == 0 else 0.01))
        wts[f"w_{N}_{M}"] = e.weights
        wts[f"f_{N}_{M}"] = e.frequencies
    np.savez_compressed(os.path.join(HERE, "expansions.npz"), **wts)


def maxfilters():
    rng = np.random.default_rng(11)
    out = {}
    for k in range(40):
        h = int(rng.integers(1, 70))
        w = int(rng.integers(1, 70))
        R = int(rng.integers(0, 20))
        img = rng.uniform(0, 255, (h, w))
        if k % 3 == 0:
            img = np.round(img)  # ties
        if k % 5 == 0:
            img = img.astype(np.float32).astype(np.float64)
        out[f"img_{k}"] = img
        out[f"R_{k}"] = np.array(R)
        out[f"M_{k}"] = rm.max_filter_2d(img, R)
        out[f"T_{k}"] = np.array(rm.compute_T(img, R))
    for k in range(20):
        n = int(rng.integers(1, 258))
        R = int(rng.integers(0, 41))
        s = rng.uniform(-1e3, 1e3, n)
        out[f"seq_{k}"] = s
        out[f"sR_{k}"] = np.array(R)
        out[f"smax_{k}"] = rm.max_filter_1d(s, R)
    np.savez_compressed(os.path.join(HERE, "maxfilter.npz"), **out)


def smoothing():
    rng = np.random.default_rng(12)
    out = {}
    k = 0
    for sigma, passes in ((0.5, 3), (2.0, 3), (3.0, 3), (5.0, 3), (8.0, 3), (12.0, 3), (2.0, 1), (4.0, 2), (10.0, 4)):
        h = int(rng.integers(1, 60))
        w = int(rng.integers(1, 60))
        img = rng.uniform(-50, 255, (h, w))
        out[f"img_{k}"] = img
        out[f"sig_{k}"] = np.array([sigma, passes])
        out[f"out_{k}"] = rs.iterated_box_gaussian(img, sigma, passes)
        r, a = rs.extended_box_params(sigma, passes)
        out[f"ra_{k}"] = np.array([r, a])
        k += 1
    for j, radius in enumerate((0, 1, 3, 7, 30)):
        img = rng.uniform(0, 255, (int(rng.integers(1, 50)), int(rng.integers(1, 50))))
        out[f"bimg_{j}"] = img
        out[f"brad_{j}"] = np.array(radius)
        out[f"bout_{j}"] = rs.box_filter(img, radius)
    np.savez_compressed(os.path.join(HERE, "smoothing.npz"), **out)


def bf_cases():
    """Small end-to-end filter cases covering modes, borders, plans."""
    rng = np.random.default_rng(20260810)
    cases = [
        # (h, w, sigma_s, sigma_r, eps, spatial, fixed_T, truncation, lo, hi)
        (40, 40, 2.0, 40.0, 0.0, None, None, "auto", 0, 255),
        (37, 53, 3.0, 30.0, 0.01, None, None, "auto", 0, 255),
        (64, 80, 5.0, 10.0, 0.01, None, None, "auto", 0, 255),
        (33, 129, 2.0, 20.0, 0.01, None, None, "auto", 0, 255),
        (150, 70, 3.0, 25.0, 0.01, None, None, "auto", 0, 255),
        (24, 24, 2.0, 30.0, 0.01, ("box", 2), None, "auto", 0, 200),
        (32, 32, 3.0, 15.0, 0.0, ("box", 3), None, "auto", 0, 255),
        (16, 16, 2.0, 30.0, 0.0, ("box", 2), 255.0, "auto", 0, 200),
        (20, 20, 3.0, 20.0, 0.05, None, None, "chernoff", 0, 255),
        (20, 21, 3.0, 20.0, 0.05, None, None, "none", 0, 255),
        (48, 48, 8.0, 800.0, 0.01, None, None, "auto", 0, 65535),
        (45, 47, 6.0, 20.0, 0.01, None, None, "auto", 0, 255),
        (9, 7, 1.0, 50.0, 0.0, None, None, "auto", 0, 255),
        (3, 90, 4.0, 30.0, 0.01, None, None, "auto", 0, 255),
        (60, 60, 12.0, 15.0, 0.01, None, None, "auto", 0, 255),
        (64, 64, 30.0, 10.0, 0.005, ("box", 30), None, "auto", 0, 255),
    ]
    out = {}
    for k, (h, w, ss, sr, eps, sp, fT, tr, lo, hi) in enumerate(cases):
        img = rng.uniform(lo, hi, (h, w))
        if k % 2 == 1:
            img = img.astype(np.float32).astype(np.float64)
        if k == 15:
            img = shiftbf.checkerboard(h, w, 8)
        spatial = None if sp is None else rs.Box(sp[1])
        p = FilterParams(sigma_s=ss, sigma_r=sr, epsilon=eps, spatial=spatial,
                         fixed_T=fT, truncation=tr)
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = shiftable_bf(img, p)
        out[f"img_{k}"] = img
        out[f"par_{k}"] = np.array([ss, sr, eps, -1 if sp is None else sp[1],
                                    np.nan if fT is None else fT,
                                    ["auto", "exact", "chernoff", "none"].index(tr)])
        out[f"out_{k}"] = res.image
        out[f"plan_{k}"] = np.array([res.plan.T, res.plan.N, res.plan.M, res.fallback_pixels])
    np.savez_compressed(os.path.join(HERE, "bf_small.npz"), **out)


def config1():
    img = config_image(1)
    res = shiftable_bf(img, FilterParams(sigma_s=3, sigma_r=30, epsilon=0.01))
    o = res.image
    np.savez_compressed(os.path.join(HERE, "config1.npz"),
                        plan=np.array([res.plan.T, res.plan.N, res.plan.M, res.fallback_pixels]),
                        crop=o[192:320, 192:320], border=np.concatenate([o[0], o[-1], o[:, 0], o[:, -1]]),
                        stats=np.array([o.sum(), o.min(), o.max(), float((o * o).sum())]),
                        M=rm.max_filter_2d(img, 9)[::8, ::8])


def direct_cases():
    """Brute-force direct_bf (bilateral.py:205-239) with gaussian_range."""
    from shiftbf.bilateral import direct_bf, gaussian_range
    rng = np.random.default_rng(20260811)
    cases = [
        # (h, w, spatial, radius override, sigma_r, lo, hi)
        (23, 31, ("box", 2), None, 30.0, 0, 255),
        (40, 37, ("fir", 3.0, 9), None, 20.0, 0, 255),
        (17, 64, ("fir", 2.0, 6), 4, 50.0, 0, 255),
        (30, 30, ("box", 5), None, 10.0, 0, 255),
        (12, 9, ("fir", 5.0, 15), None, 25.0, 0, 255),
        (36, 28, ("fir", 4.0, 12), None, 800.0, 0, 65535),
        (1, 50, ("box", 3), None, 30.0, 0, 255),
        (45, 45, ("fir", 1.5, 5), None, 5.0, 0, 255),
    ]
    out = {}
    for k, (h, w, sp, rad, sr, lo, hi) in enumerate(cases):
        img = rng.uniform(lo, hi, (h, w))
        if k % 2 == 0:
            img = img.astype(np.float32).astype(np.float64)
        mode = rs.Box(sp[1]) if sp[0] == "box" else rs.FirGaussian(sp[1], sp[2])
        out[f"img_{k}"] = img
        out[f"par_{k}"] = np.array([0 if sp[0] == "box" else 1, sp[1],
                                    sp[1] if sp[0] == "box" else sp[2],
                                    -1 if rad is None else rad, sr])
        out[f"out_{k}"] = direct_bf(img, mode, gaussian_range(sr), radius=rad)
    np.savez_compressed(os.path.join(HERE, "direct.npz"), **out)


def nlm_cases():
    """coarse_nlm_shiftable (nlm.py:78-137) on small images."""
    from shiftbf import nlm as rn
    rng = np.random.default_rng(20260812)
    cases = [
        # (h, w, offsets, sigmas, spatial, radius, eps)
        (24, 28, [(0, 0)], [20.0], ("iter", 2.0), 6, 0.05),
        (20, 22, [(0, 0), (0, 1)], [40.0, 40.0], ("iter", 2.0), 6, 0.05),
        (18, 18, [(0, 0), (1, -1)], [50.0, 35.0], ("box", 2), 2, 0.05),
        (16, 19, [(0, 0), (0, 1), (1, 0)], [60.0, 60.0, 60.0], ("iter", 1.5), 5, 0.1),
        (22, 20, [(0, 0), (2, 0)], [80.0, 45.0], ("iter", 3.0), 9, 0.0),
    ]
    out = {}
    for k, (h, w, offs, sgs, sp, rad, eps) in enumerate(cases):
        img = rng.uniform(0, 120, (h, w))
        mode = rs.Box(sp[1]) if sp[0] == "box" else rs.IteratedBox(sp[1])
        res = rn.coarse_nlm_shiftable(img, rn.PatchSpec(tuple(offs), tuple(sgs)), mode, rad, eps)
        out[f"img_{k}"] = img
        out[f"offs_{k}"] = np.array(offs, dtype=np.int64)
        out[f"par_{k}"] = np.array(sgs + [0 if sp[0] == "box" else 1, sp[1], rad, eps])
        out[f"out_{k}"] = res.image
        out[f"plans_{k}"] = np.array([[p.T, p.N, p.M] for p in res.plans])
    np.savez_compressed(os.path.join(HERE, "nlm.npz"), **out)


def direct_nlm_cases():
    """direct_nlm (nlm.py:140-183) with Gaussian and expansion range kernels."""
    from shiftbf import nlm as rn
    rng = np.random.default_rng(20260813)
    cases = [
        # (h, w, offsets, sigmas, spatial, radius, kernels)
        (20, 23, [(0, 0), (0, 1)], [40.0, 30.0], ("box", 2), 2, "gaussian"),
        (18, 16, [(0, 0), (1, 0), (0, -1)], [50.0, 50.0, 60.0], ("fir", 1.5, 3), 3, "gaussian"),
        (16, 21, [(0, 0), (1, 1)], [40.0, 40.0], ("box", 3), 3, "expansion"),
    ]
    out = {}
    for k, (h, w, offs, sgs, sp, rad, kern) in enumerate(cases):
        img = rng.uniform(0, 120, (h, w))
        mode = rs.Box(sp[1]) if sp[0] == "box" else rs.FirGaussian(sp[1], sp[2])
        patch = rn.PatchSpec(tuple(offs), tuple(sgs))
        if kern == "gaussian":
            ref = rn.direct_nlm(img, patch, mode, rad)
        else:
            T = rm.compute_T(img, rad + patch.max_offset_norm)
            plans = [rk.select_plan(T, sg, 0.05) for sg in sgs]
            ref = rn.direct_nlm(img, patch, mode, rad, [rn.expansion_range_for(pl) for pl in plans])
        out[f"img_{k}"] = img
        out[f"offs_{k}"] = np.array(offs, dtype=np.int64)
        out[f"par_{k}"] = np.array(sgs + [0 if sp[0] == "box" else 1, sp[1],
                                          sp[1] if sp[0] == "box" else sp[2], rad,
                                          0 if kern == "gaussian" else 1])
        out[f"out_{k}"] = ref
    np.savez_compressed(os.path.join(HERE, "direct_nlm.npz"), **out)


def big_plans():
    rows = []
    specs = [(2, 0, 5.0, 10.0), (3, 0, 8.0, 800.0)] + [(4, i, 6.0, 20.0) for i in range(64)] \
        + [(5, c, 12.0, 15.0) for c in range(3)]
    for cfg, idx, ss, sr in specs:
        img = config_image(cfg, idx)
        R = max(1, rs.support_radius(rs.IteratedBox(ss)))
        T = rm.compute_T(img, R)
        p = rk.select_plan(T, sr, 0.01)
        rows.append((cfg, idx, R, T, p.N, p.M))
        print(cfg, idx, R, repr(T), p.N, p.M, flush=True)
        del img
    np.savez_compressed(os.path.join(HERE, "config_plans.npz"), rows=np.array(rows, dtype=np.float64))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--direct", action="store_true", help="only the direct_bf fixtures")
    a = ap.parse_args()
    if a.direct:
        direct_cases()
        nlm_cases()
        direct_nlm_cases()
    elif not a.big:
        plans()
        maxfilters()
        smoothing()
        bf_cases()
        config1()
        direct_cases()
        nlm_cases()
        direct_nlm_cases()
    if a.big:
        big_plans()
    print("done")
