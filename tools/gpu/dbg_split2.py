import os, sys
import numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_1203_5128_b200 as P
from oracle import coracle as CO
from test_gpu_properties import _random_case
CO.build()
for seed in (53, 15):
    img, ss, sr, eps, box, fixed = _random_case(seed)
    ref = CO.shiftable_bf(np.asarray(img, dtype=np.float64), ss, sr, eps, fixed_T=fixed)
    outs = []
    for rep in range(6):
        res = P.shiftable_bf(img, P.FilterParams(sigma_s=ss, sigma_r=sr, epsilon=eps, fixed_T=fixed))
        d = np.abs(res.image - ref["image"]); bad = np.argwhere(d > 1e-2)
        print(seed, rep, "max", float(d.max()), "nbad", len(bad), bad[:3].tolist(), flush=True)
    # float32 copy and other widths
for w in (1, 2, 3, 4, 5, 8, 17, 33, 64, 65):
    rng = np.random.default_rng(w)
    img = rng.uniform(0, 255, (196, w))
    for sr in (45.0, 20.0):
        res = P.shiftable_bf(img, P.FilterParams(sigma_s=9.7, sigma_r=sr, epsilon=0.0))
        ref = CO.shiftable_bf(img, 9.7, sr, 0.0)
        d = np.abs(res.image - ref["image"]); bad = np.argwhere(d > 1e-2)
        print("w", w, sr, "K", res.plan.N // 2 - res.plan.M + 1, "max", float(d.max()), "nbad", len(bad), bad[:2].tolist(), flush=True)
