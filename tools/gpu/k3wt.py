"""Device time of sbf_filter (K3 + divide) on one config-4 image and config 2 for
library builds given as arguments, sweep variant from SBF_VARIANT (default 2)."""
import os, sys, numpy as np, torch, importlib
sys.path.insert(0, os.getcwd())
from paper_1203_5128_b200.workloads import config_image, CONFIGS
libs = sys.argv[1:] or ["paper_1203_5128_b200/libsbf.so"]
var = int(os.environ.get("SBF_VARIANT", "2"))
imgs = {c: torch.from_numpy(np.ascontiguousarray(config_image(c), dtype=np.float32)).cuda() for c in (4, 2, 1)}
for path in libs:
    os.environ["SBF_LIB"] = path
    import paper_1203_5128_b200._lib as L
    importlib.reload(L)
    lib = L.load()
    import paper_1203_5128_b200 as P
    from paper_1203_5128_b200.kernels import log_2_over_eps
    from paper_1203_5128_b200.spatial import to_c_spatial
    lib.sbf_set_sweep_variant(var)
    for cfg, f in imgs.items():
        p = CONFIGS[cfg]
        H, W = f.shape
        params = P.FilterParams(sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], epsilon=p["epsilon"])
        sp = to_c_spatial(params.resolved_spatial()); R = params.resolved_radius()
        stats = torch.empty(8, dtype=torch.float64, device="cuda")
        plan = torch.empty(64, dtype=torch.uint8, device="cuda")
        terms = torch.empty((1 << 16) * 32, dtype=torch.uint8, device="cuda")
        out = torch.empty((H, W), dtype=torch.float32, device="cuda")
        fb = torch.zeros(1, dtype=torch.int64, device="cuda")
        lr_ws = torch.empty(lib.sbf_local_range_workspace(H, W, 0), dtype=torch.uint8, device="cuda")
        f_ws = torch.empty(lib.sbf_filter_workspace(H, W, H, 0, sp, 0), dtype=torch.uint8, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        lib.sbf_local_range(f.data_ptr(), 0, H, W, W, R, 0, H, None, stats.data_ptr(), lr_ws.data_ptr(), lr_ws.numel(), st)
        lib.sbf_plan_device(stats.data_ptr(), 0, 0.0, p["sigma_r"], p["epsilon"], 0, log_2_over_eps(p["epsilon"]), plan.data_ptr(), terms.data_ptr(), 1 << 16, st)
        def run():
            L.check(lib.sbf_filter(f.data_ptr(), 0, H, W, W, 0, H, 0, H, sp, plan.data_ptr(), terms.data_ptr(), stats.data_ptr(), 0, out.data_ptr(), 0, fb.data_ptr(), f_ws.data_ptr(), f_ws.numel(), st))
        for _ in range(2): run()
        torch.cuda.synchronize()
        n = 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n): run()
        e1.record(); e1.synchronize()
        print(f"{os.path.basename(path):28s} var{var} cfg{cfg} K3 ms {e0.elapsed_time(e1) / n:.3f}", flush=True)
