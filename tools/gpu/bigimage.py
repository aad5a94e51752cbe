"""64-bit indexing check at sizes beyond the configs: filter one huge device-resident image
and compare windows near its far corner (and in the middle) with the same windows filtered on
their own (same fixed T, so the same plan).  Sizes: argv[1] (side, default 46400: > 2^31 px),
sigma_s argv[2] (5: K3 sweep; 12: split sweep)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_1203_5128_b200 as P
side = int(sys.argv[1]) if len(sys.argv) > 1 else 46400
ss = float(sys.argv[2]) if len(sys.argv) > 2 else 5.0
dev = torch.device("cuda")
g = torch.Generator(device=dev); g.manual_seed(1)
img = torch.empty((side, side), dtype=torch.float32, device=dev)
for y in range(0, side, 4096):  # fill in slabs (bounded temporaries)
    n = min(4096, side - y)
    img[y:y + n] = torch.rand((n, side), generator=g, device=dev) * 60.0 + 20.0
img[side // 3: side // 3 + 5000, side // 2:] += 150.0
img[side - 400:, side - 900:] += 90.0
params = P.FilterParams(sigma_s=ss, sigma_r=20.0, epsilon=0.01, fixed_T=255.0, precision="fp32")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); res = P.shiftable_bf(img, params); e1.record(); torch.cuda.synchronize()
print(f"{side}x{side} sigma_s={ss}: N={res.plan.N} M={res.plan.M} fallbacks={res.fallback_pixels} "
      f"{e0.elapsed_time(e1):.1f} ms ({side * side / e0.elapsed_time(e1) / 1e3:.0f} Mpix/s), "
      f"peak mem {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB", flush=True)
out = res.image
halo = 64
worst = 0.0
for (y0, x0, h, w) in ((side - 700, side - 800, 700, 800), (side // 2 - 300, side // 2 - 300, 600, 600),
                       (0, side - 640, 500, 640), (side - 512, 0, 512, 600)):
    ya, yb = max(0, y0 - halo), min(side, y0 + h + halo)
    xa, xb = max(0, x0 - halo), min(side, x0 + w + halo)
    sub = P.shiftable_bf(img[ya:yb, xa:xb].contiguous(), params).image
    # interior of the window: away from the cuts that are not image borders
    ty = slice(halo if ya > 0 else 0, (yb - ya) - (halo if yb < side else 0))
    tx = slice(halo if xa > 0 else 0, (xb - xa) - (halo if xb < side else 0))
    a = sub[ty, tx]
    b = out[ya + ty.start: ya + ty.stop, xa + tx.start: xa + tx.stop]
    d = float((a - b).abs().max())
    worst = max(worst, d)
    print(f"  window ({y0},{x0}) {h}x{w}: max|diff| {d:.3e}", flush=True)
print("OK" if worst <= 2e-3 else "MISMATCH", worst)
sys.exit(0 if worst <= 2e-3 else 1)
