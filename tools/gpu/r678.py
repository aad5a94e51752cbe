"""r = 6..8: the round-1 term kernel (fp32 red.add, order-dependent) vs the split
sweep (deterministic) on a 4096^2 config-4 image: device time of the fused pipeline."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1203_5128_b200 as P
import paper_1203_5128_b200._lib as L
from paper_1203_5128_b200.workloads import config_image
lib = L.load()
img = torch.from_numpy(np.ascontiguousarray(config_image(4), dtype=np.float32)).cuda()
for ss in (7.0, 8.0, 9.5):
    params = P.FilterParams(sigma_s=ss, sigma_r=20.0, epsilon=0.01, precision="fp32")
    outs = {}
    for mr in (9, 6):
        lib.sbf_set_split_min_radius(mr)
        for _ in range(2): res = P.shiftable_bf(img, params)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): res = P.shiftable_bf(img, params)
        e1.record(); torch.cuda.synchronize()
        outs[mr] = res.image.clone()
        print(f"sigma_s={ss} split_min_r={mr}: {e0.elapsed_time(e1)/3:.3f} ms/call  K={res.plan.M}", flush=True)
    print("   max|diff|", (outs[9] - outs[6]).abs().max().item())
lib.sbf_set_split_min_radius(9)
