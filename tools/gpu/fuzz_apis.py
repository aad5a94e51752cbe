import os, sys, numpy as np, torch, warnings
sys.path.insert(0, os.getcwd())
import paper_1203_5128_b200 as P
from oracle import shiftbf_oracle as O
from paper_1203_5128_b200.dist import StripFilter, gather_strips, strip_halo, strip_plan
warnings.simplefilter("ignore")
rng = np.random.default_rng(99)
bad = 0
# 1. max filter / T bit-exact
for i in range(300):
    H, W = int(rng.integers(1, 300)), int(rng.integers(1, 300))
    R = int(rng.integers(0, 60))
    dtype = np.float32 if rng.random() < 0.5 else np.float64
    img = (rng.uniform(0, 255, (H, W)) if rng.random() < 0.7 else np.round(rng.uniform(0, 4, (H, W)))).astype(dtype)
    try:
        src = torch.from_numpy(img).cuda() if rng.random() < 0.5 else img
        M = P.max_filter_2d(src, R); T = P.compute_T(src, R)
        M = M.cpu().numpy() if isinstance(M, torch.Tensor) else M
        Mo = O.max_filter_2d(img.astype(np.float64), R); To = O.compute_T(img.astype(np.float64), R)
        if not np.array_equal(np.asarray(M, dtype=np.float64), Mo) or float(T) != To:
            bad += 1; print("FAIL maxfilter", H, W, R, dtype.__name__, float(T), To, flush=True)
    except Exception as e:
        bad += 1; print("ERROR maxfilter", H, W, R, dtype.__name__, type(e).__name__, str(e)[:120], flush=True)
print("maxfilter done", bad, flush=True)
# 2. strips vs full image
for i in range(40):
    H, W = int(rng.integers(40, 400)), int(rng.integers(8, 300))
    ss = float(rng.uniform(1.0, 12.5)); sr = float(rng.choice([15.0, 25.0, 40.0]))
    G = int(rng.integers(1, 6)); C = int(rng.integers(1, 4))
    params = P.FilterParams(sigma_s=ss, sigma_r=sr, epsilon=0.01, precision="fp32")
    try:
        chans = [rng.uniform(0, 255, (H, W)).astype(np.float32) for _ in range(C)]
        full = [P.shiftable_bf(ch, params) for ch in chans]
        strips = strip_plan(H, G, strip_halo(params))
        Ts = [f.plan.T for f in full]
        outs = [[] for _ in range(C)]
        for s in strips:
            bufs = [torch.from_numpy(np.ascontiguousarray(ch[s.buf_lo:s.buf_hi])).cuda() for ch in chans]
            sf = StripFilter(bufs, s, H, params, overlap=bool(rng.integers(0, 2)),
                             reduce_max=lambda t: t.copy_(torch.tensor(Ts, device=t.device)))
            o = sf.run(); sf.check()
            for c in range(C): outs[c].append(o[c].cpu().numpy())
        for c in range(C):
            d = np.abs(gather_strips(outs[c], strips) - full[c].image).max()
            if d > 2e-3:
                bad += 1; print("FAIL strips", H, W, ss, sr, G, C, c, float(d), flush=True)
    except Exception as e:
        bad += 1; print("ERROR strips", H, W, ss, sr, G, C, type(e).__name__, str(e)[:160], flush=True)
print("strips done", bad, flush=True)
# 3. batch API vs single calls (bit-identical)
for i in range(10):
    n = int(rng.integers(1, 7)); H, W = int(rng.integers(16, 200)), int(rng.integers(16, 200))
    ss = float(rng.uniform(1.0, 12.0))
    params = P.FilterParams(sigma_s=ss, sigma_r=20.0, epsilon=0.01)
    try:
        imgs = [torch.from_numpy(rng.uniform(0, 255, (H, W)).astype(np.float32)).pin_memory() for _ in range(n)]
        res = P.shiftable_bf_batch(imgs, params, lanes=int(rng.integers(1, 5)))
        for t, r in zip(imgs, res):
            one = P.shiftable_bf(t.cuda(), params)
            if not torch.equal(one.image.cpu(), r.image.cpu() if isinstance(r.image, torch.Tensor) else torch.from_numpy(r.image)):
                bad += 1; print("FAIL batch", n, H, W, ss, flush=True); break
    except Exception as e:
        bad += 1; print("ERROR batch", n, H, W, ss, type(e).__name__, str(e)[:160], flush=True)
print("all done, failing:", bad)
