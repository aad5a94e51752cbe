"""Warp-specialised K3 sweep vs the phase-separated sweep: output difference and
device time per sbf_filter call (K3 + divide), per variant."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1203_5128_b200.workloads import config_image, CONFIGS
import paper_1203_5128_b200._lib as L
import paper_1203_5128_b200 as P
from paper_1203_5128_b200.kernels import log_2_over_eps
from paper_1203_5128_b200.spatial import to_c_spatial

lib = L.load()
cases = []
for cfg in (2, 4, 1):
    p = CONFIGS[cfg]
    cases.append((f"cfg{cfg}", config_image(cfg), p["sigma_s"], p["sigma_r"], p["epsilon"]))
rng = np.random.default_rng(5)
for (h, w, ss) in ((300, 517, 2.0), (777, 1031, 4.0), (130, 260, 1.0), (64, 3000, 6.0)):
    cases.append((f"rnd{h}x{w}_s{ss}", (rng.random((h, w)) * 255).astype(np.float32), ss, 25.0, 0.01))
for name, img, ss, sr, eps in cases:
    f = torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32)).cuda()
    H, W = f.shape
    params = P.FilterParams(sigma_s=ss, sigma_r=sr, epsilon=eps)
    sp = to_c_spatial(params.resolved_spatial()); R = params.resolved_radius()
    stats = torch.empty(8, dtype=torch.float64, device="cuda")
    plan = torch.empty(64, dtype=torch.uint8, device="cuda")
    terms = torch.empty((1 << 16) * 32, dtype=torch.uint8, device="cuda")
    fb = torch.zeros(1, dtype=torch.int64, device="cuda")
    lr_ws = torch.empty(lib.sbf_local_range_workspace(H, W, 0), dtype=torch.uint8, device="cuda")
    f_ws = torch.empty(lib.sbf_filter_workspace(H, W, H, 0, sp, 0), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    lib.sbf_local_range(f.data_ptr(), 0, H, W, W, R, 0, H, None, stats.data_ptr(), lr_ws.data_ptr(), lr_ws.numel(), st)
    lib.sbf_plan_device(stats.data_ptr(), 0, 0.0, sr, eps, 0, log_2_over_eps(eps), plan.data_ptr(), terms.data_ptr(), 1 << 16, st)
    outs = {}
    for var in (0, 2):
        lib.sbf_set_sweep_variant(var)
        out = torch.empty((H, W), dtype=torch.float32, device="cuda")
        def run():
            L.check(lib.sbf_filter(f.data_ptr(), 0, H, W, W, 0, H, 0, H, sp, plan.data_ptr(), terms.data_ptr(), stats.data_ptr(), 0, out.data_ptr(), 0, fb.data_ptr(), f_ws.data_ptr(), f_ws.numel(), st))
        for _ in range(2): run()
        torch.cuda.synchronize()
        n = 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n): run()
        e1.record(); e1.synchronize()
        outs[var] = (out.clone(), e0.elapsed_time(e1) / n)
    d = (outs[0][0] - outs[2][0]).abs().max().item()
    print(f"{name:20s} r={sp.r} classic {outs[0][1]:.3f} ms  warp-spec {outs[2][1]:.3f} ms  max|diff| {d:.3e}", flush=True)
