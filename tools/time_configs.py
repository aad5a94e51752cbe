"""Device time of the full pipeline per config (CUDA events), for triage."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_5128_b200 as P
from paper_1203_5128_b200.workloads import CONFIGS, config_image

for cfg, size, idx in [(1, None, 0), (2, None, 0), (3, None, 0), (4, None, 0), (5, 8192, 1)]:
    p = CONFIGS[cfg]
    img = config_image(cfg, idx, size=size)
    t = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    params = P.FilterParams(sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], epsilon=p["epsilon"])
    res = P.shiftable_bf(t, params)  # warm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 3
    for _ in range(n):
        res = P.shiftable_bf(t, params)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    px = img.size
    print(f"cfg{cfg} {img.shape} N={res.plan.N} M={res.plan.M} K={res.plan.N//2-res.plan.M+1} "
          f"{ms:.2f} ms/image  {px/ms/1e3:.1f} Mpix/s", flush=True)

# SURVEY §8(f) components: brute-force direct_bf and coarse NLM (device time)
img = torch.from_numpy(config_image(2)).cuda()
for name, fn in [
    ("direct_bf cfg2 FIR R=15", lambda: P.direct_bf(img, P.FirGaussian(5.0, 15), P.gaussian_range(10.0))),
    ("coarse_nlm cfg2 p=2 sigma 60,60", lambda: P.coarse_nlm_shiftable(
        img, P.PatchSpec(((0, 0), (0, 1)), (60.0, 60.0)), P.IteratedBox(3.0), 9, 0.05)),
]:
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        r = fn()
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{name}: {ms:.2f} ms  {img.numel() / ms / 1e3:.1f} Mpix/s", flush=True)
