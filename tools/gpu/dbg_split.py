"""Debug: split path vs the C oracle on small random cases (r >= 9)."""
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_1203_5128_b200 as P
from oracle import coracle as CO
from test_gpu_properties import _random_case
CO.build()
for seed in list(range(64)):
    img, ss, sr, eps, box, fixed = _random_case(seed)
    if box or ss < 9: continue
    res = P.shiftable_bf(img, P.FilterParams(sigma_s=ss, sigma_r=sr, epsilon=eps, fixed_T=fixed))
    ref = CO.shiftable_bf(np.asarray(img, dtype=np.float64), ss, sr, eps, fixed_T=fixed)
    d = np.abs(res.image - ref["image"])
    bad = np.argwhere(d > 1e-2)
    print(seed, img.dtype, img.shape, ss, sr, eps, "K", res.plan.N // 2 - res.plan.M + 1, "max", float(d.max()),
          "nbad", len(bad), "rows", (bad[:, 0].min(), bad[:, 0].max()) if len(bad) else None,
          "cols", (bad[:, 1].min(), bad[:, 1].max()) if len(bad) else None, flush=True)
for (h, w) in [(242, 180), (256, 180), (240, 180), (242, 256), (300, 300), (64, 500)]:
    rng = np.random.default_rng(1)
    img = rng.uniform(0, 255, (h, w)).astype(np.float32)
    for ss in (9.7, 11.6):
        res = P.shiftable_bf(img, P.FilterParams(sigma_s=ss, sigma_r=20.0, epsilon=0.01))
        ref = CO.shiftable_bf(img.astype(np.float64), ss, 20.0, 0.01)
        d = np.abs(res.image - ref["image"]); bad = np.argwhere(d > 1e-2)
        print((h, w), ss, "K", res.plan.N // 2 - res.plan.M + 1, "max", float(d.max()), "nbad", len(bad),
              "rows", (bad[:, 0].min(), bad[:, 0].max()) if len(bad) else None, flush=True)
