"""Randomised parity cases for the public filter against the numpy oracle: shapes,
dtypes, spatial modes (IteratedBox with 1..4 passes, Box), sigma_s, sigma_r, epsilon,
input side (numpy / CUDA tensor).  Used by tests/test_gpu_fuzz.py and tools/gpu/fuzz.py."""
import warnings

import numpy as np


def run_cases(n, seed, variant=None, log=None):
    """Runs n seeded cases; returns the list of failure descriptions."""
    import torch

    import paper_1203_5128_b200 as P
    from oracle import shiftbf_oracle as O
    from paper_1203_5128_b200 import _lib

    lib = _lib.load()
    prev = lib.sbf_set_sweep_variant(variant) if variant is not None else None
    rng = np.random.default_rng(seed)
    fails = []
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            for i in range(n):
                H, W = int(rng.integers(1, 220)), int(rng.integers(1, 260))
                dtype = np.float32 if rng.random() < 0.6 else np.float64
                img = rng.uniform(0, 255, (H, W))
                if rng.random() < 0.5 and H > 4 and W > 4:
                    img[H // 3:, W // 2:] = np.clip(img[H // 3:, W // 2:] * 0.2 + rng.uniform(0, 200), 0, 255)
                if rng.random() < 0.3:
                    img = np.round(img)
                img = img.astype(dtype)
                sr = float(rng.choice([8.0, 12.0, 20.0, 30.0, 45.0, 60.0]))
                eps = float(rng.choice([0.0, 0.005, 0.01, 0.05]))
                kind = rng.random()
                if kind < 0.55:
                    ss = float(rng.uniform(0.6, 13.0))
                    spatial, osp = None, None
                elif kind < 0.8:
                    ss = float(rng.uniform(0.8, 9.0))
                    passes = int(rng.integers(1, 5))
                    spatial, osp = P.IteratedBox(ss, passes), ("iterated", ss, passes)
                else:
                    r = int(rng.integers(0, 15))
                    ss = float(max(r, 1))
                    spatial, osp = P.Box(r), ("box", r)
                on_device = rng.random() < 0.5
                params = P.FilterParams(sigma_s=ss, sigma_r=sr, epsilon=eps, spatial=spatial)
                tag = f"#{i} {H}x{W} {dtype.__name__} ss={ss:.4f} sr={sr} eps={eps} spatial={osp} cuda={on_device}"
                try:
                    ref = O.shiftable_bf(img.astype(np.float64), ss, sr, eps, spatial=osp)
                    if ref["N"] > 400:
                        continue
                    src = torch.from_numpy(img).cuda() if on_device else img
                    res = P.shiftable_bf(src, params)
                    out = res.image.double().cpu().numpy() if isinstance(res.image, torch.Tensor) else res.image
                    ok_plan = (res.plan.T, res.plan.N, res.plan.M) == (ref["T"], ref["N"], ref["M"])
                    d = np.abs(out - ref["image"])
                    # (a pixel whose exact normaliser is ~0 may fall back on one side only)
                    if not ok_plan or ((d <= 1e-2).mean() < 0.999 and res.fallback_pixels == ref["fallback_pixels"]):
                        fails.append(f"FAIL {tag}: plan {(res.plan.T, res.plan.N, res.plan.M)} vs "
                                     f"{(ref['T'], ref['N'], ref['M'])}, max|d| {float(d.max()):.3e}, fallbacks "
                                     f"{res.fallback_pixels} vs {ref['fallback_pixels']}")
                except Exception as e:  # noqa: BLE001 - every failure mode is reported
                    fails.append(f"ERROR {tag}: {type(e).__name__}: {str(e)[:160]}")
                if log and fails and fails[-1].split()[1] == f"#{i}":
                    log(fails[-1])
    finally:
        if prev is not None:
            lib.sbf_set_sweep_variant(prev)
    return fails
