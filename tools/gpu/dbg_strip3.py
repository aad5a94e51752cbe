import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1203_5128_b200 as P
from paper_1203_5128_b200 import dist as D
from paper_1203_5128_b200.workloads import config_image
imgs = [config_image(5, c, size=384) for c in (0, 2)]
mode = sys.argv[1]
orig = D.StripFilter._filter_channel
def patched(self, c, st, ws, prec):
    if mode == "pre":
        torch.cuda.synchronize()
    orig(self, c, st, ws, prec)
    if mode == "post":
        torch.cuda.synchronize()
D.StripFilter._filter_channel = patched
params = P.FilterParams(sigma_s=12.0, sigma_r=15.0, epsilon=0.01, precision="fp32")
fulls = [P.shiftable_bf(img, params) for img in imgs]
ts = [torch.from_numpy(img).cuda() for img in imgs]
H = imgs[0].shape[0]
s = D.strip_plan(H, 1, D.strip_halo(params))[0]
f = D.StripFilter([t[s.buf_lo:s.buf_hi] for t in ts], s, H, params, overlap=True)
Tg = f.local_T().clone()
outs = [o.cpu().numpy() for o in f.finish(Tg)]
torch.cuda.synchronize()
outs2 = [o.cpu().numpy() for o in f.out]
for c, full in enumerate(fulls):
    print(mode, c, float(np.abs(outs[c] - full.image).max()), float(np.abs(outs2[c] - full.image).max()), flush=True)
