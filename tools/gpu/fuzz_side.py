"""Randomised parity of the (f) rows against the numpy oracle: direct_bf (Box / FirGaussian,
gaussian_range) and coarse_nlm_shiftable (1-2 offsets)."""
import os, sys, numpy as np, torch, warnings
sys.path.insert(0, os.getcwd())
import paper_1203_5128_b200 as P
from oracle import shiftbf_oracle as O
warnings.simplefilter("ignore")
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
bad = 0
for i in range(80):
    H, W = int(rng.integers(1, 90)), int(rng.integers(1, 110))
    dtype = np.float32 if rng.random() < 0.5 else np.float64
    img = rng.uniform(0, 255, (H, W)).astype(dtype)
    sr = float(rng.choice([5.0, 10.0, 25.0, 60.0]))
    if rng.random() < 0.5:
        r = int(rng.integers(0, 12)); mode, osp = P.Box(r), ("box", r)
    else:
        s, r = float(rng.uniform(0.7, 6.0)), int(rng.integers(1, 16)); mode, osp = P.FirGaussian(s, r), ("fir", s, r)
    try:
        src = torch.from_numpy(img).cuda() if rng.random() < 0.5 else img
        out = P.direct_bf(src, mode, P.gaussian_range(sr))
        out = out.double().cpu().numpy() if isinstance(out, torch.Tensor) else out
        ref = O.direct_bf(img.astype(np.float64), osp, sr)
        tol = 2e-3  # the direct path computes 8-bit-scale images in fp32 (tolerance of the golden-vector tests)
        d = float(np.abs(out - ref).max())
        if d > tol:
            bad += 1; print("FAIL direct", H, W, dtype.__name__, osp, sr, d, flush=True)
    except Exception as e:
        bad += 1; print("ERROR direct", H, W, dtype.__name__, osp, sr, type(e).__name__, str(e)[:140], flush=True)
print("direct_bf done", bad, flush=True)
for i in range(30):
    H, W = int(rng.integers(6, 70)), int(rng.integers(6, 80))
    img = rng.uniform(0, 255, (H, W)).astype(np.float64)
    p = int(rng.integers(1, 3))
    offs = [(0, 0)] + [(int(rng.integers(-2, 3)), int(rng.integers(-2, 3))) for _ in range(p - 1)]
    offs = [o for k, o in enumerate(offs) if o not in offs[:k]]
    sig = [float(rng.choice([40.0, 60.0, 90.0])) for _ in offs]
    ss = float(rng.uniform(1.0, 4.0)); radius = int(rng.integers(2, 10)); eps = 0.05
    try:
        res = P.coarse_nlm_shiftable(img, P.PatchSpec(tuple(offs), tuple(sig)), P.IteratedBox(ss), radius, eps)
        ref = O.coarse_nlm(img, offs, sig, ("iterated", ss, 3), radius, eps)
        d = float(np.abs(res.image - ref["image"]).max())
        if d > 1e-2:
            bad += 1; print("FAIL nlm", H, W, offs, sig, ss, radius, d, flush=True)
    except P.errors.ShiftBFError as e:
        print("skip nlm (budget)", offs, sig, str(e)[:60], flush=True)
    except Exception as e:
        bad += 1; print("ERROR nlm", H, W, offs, sig, ss, radius, type(e).__name__, str(e)[:140], flush=True)
print("all done, failing:", bad)
