"""Quick GPU sanity: K3 sweep vs the C oracle on small crops of configs 1/2/4."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_1203_5128_b200 as P
from oracle import coracle as CO
from paper_1203_5128_b200.workloads import config_image, CONFIGS

for cfg, size in [(1, 96), (2, 200), (4, 300), (2, 1024), (4, 1024)]:
    p = CONFIGS[cfg]
    img = config_image(cfg, size=size)
    params = P.FilterParams(sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], epsilon=p["epsilon"])
    res = P.shiftable_bf(img, params)
    torch.cuda.synchronize()
    ref = CO.shiftable_bf(img.astype(np.float64), p["sigma_s"], p["sigma_r"], p["epsilon"])
    d = res.image - ref["image"]
    print(cfg, size, (res.plan.N, res.plan.M), (ref["N"], ref["M"]), "max", np.abs(d).max(),
          "rms", np.sqrt((d * d).mean()), "fb", res.fallback_pixels, ref["fallback_pixels"], flush=True)
    r2 = P.shiftable_bf(img, params)
    print("   deterministic:", np.array_equal(r2.image, res.image))
