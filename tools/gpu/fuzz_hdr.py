"""Randomised parity of the fp64 paths (precision "hdr" / "auto" on wide-range images:
dual form and generic term sweeps) against the numpy oracle."""
import os, sys, numpy as np, torch, warnings
sys.path.insert(0, os.getcwd())
import paper_1203_5128_b200 as P
from oracle import shiftbf_oracle as O
warnings.simplefilter("ignore")
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
bad = 0
for i in range(n):
    H, W = int(rng.integers(2, 120)), int(rng.integers(2, 140))
    top = float(rng.choice([255.0, 4095.0, 65535.0]))
    img = rng.uniform(0, top, (H, W))
    if rng.random() < 0.5:
        img = np.round(img)
    dtype = np.float32 if rng.random() < 0.5 else np.float64
    img = img.astype(dtype)
    sr = float(top * rng.choice([0.01, 0.03, 0.1, 0.3]))
    ss = float(rng.uniform(0.8, 9.0))
    eps = float(rng.choice([0.0, 0.01]))
    prec = str(rng.choice(["hdr", "auto"]))
    kind = rng.random()
    if kind < 0.6:
        spatial, osp = None, None
    elif kind < 0.8:
        passes = int(rng.integers(1, 5)); spatial, osp = P.IteratedBox(ss, passes), ("iterated", ss, passes)
    else:
        r = int(rng.integers(0, 20)); ss = float(max(r, 1)); spatial, osp = P.Box(r), ("box", r)
    tag = f"#{i} {H}x{W} {dtype.__name__} top={top} ss={ss:.3f} sr={sr:.1f} eps={eps} {prec} spatial={osp}"
    try:
        ref = O.shiftable_bf(img.astype(np.float64), ss, sr, eps, spatial=osp)
        if ref["N"] > 3000:
            continue
        params = P.FilterParams(sigma_s=ss, sigma_r=sr, epsilon=eps, spatial=spatial, precision=prec)
        res = P.shiftable_bf(img, params)
        ok_plan = (res.plan.T, res.plan.N, res.plan.M) == (ref["T"], ref["N"], ref["M"])
        d = np.abs(res.image - ref["image"])
        tol = 1e-2 * max(1.0, top / 255.0) if prec == "auto" and top <= 4096 else 1e-2
        if not ok_plan or ((d <= tol).mean() < 0.999 and res.fallback_pixels == ref["fallback_pixels"]):
            bad += 1
            print("FAIL", tag, "N", res.plan.N, ref["N"], "max|d|", float(d.max()), "fb", res.fallback_pixels, ref["fallback_pixels"], flush=True)
    except Exception as e:
        bad += 1
        print("ERROR", tag, type(e).__name__, str(e)[:160], flush=True)
print(f"{n} cases, {bad} failing")
