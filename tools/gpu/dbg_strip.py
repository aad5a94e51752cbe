import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1203_5128_b200 as P
from paper_1203_5128_b200 import _lib
from paper_1203_5128_b200.dist import StripFilter, gather_strips, strip_halo, strip_plan
from paper_1203_5128_b200.workloads import config_image
imgs = [config_image(5, c, size=384) for c in (0, 2)]
for prec in ("fp32", "auto"):
    for overlap in (False, True):
        for nstrip in (1, 2):
            params = P.FilterParams(sigma_s=12.0, sigma_r=15.0, epsilon=0.01, precision=prec)
            fulls = [P.shiftable_bf(img, params) for img in imgs]
            ts = [torch.from_numpy(img).cuda() for img in imgs]
            H = imgs[0].shape[0]
            strips = strip_plan(H, nstrip, strip_halo(params))
            fs = [StripFilter([t[s.buf_lo:s.buf_hi] for t in ts], s, H, params, overlap=overlap) for s in strips]
            Tg = torch.stack([f.local_T().clone() for f in fs]).max(dim=0).values
            outs = [[o.cpu().numpy() for o in f.finish(Tg)] for f in fs]
            torch.cuda.synchronize()
            flags = [[_lib.SbfPlan.from_buffer_copy(f.plans[c].cpu().numpy().tobytes()).flags for c in range(2)] for f in fs]
            for c, full in enumerate(fulls):
                g = gather_strips([o[c] for o in outs], strips)
                print(prec, overlap, nstrip, c, flags, float(np.abs(g - full.image).max()), flush=True)
