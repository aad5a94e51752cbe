"""Config-5 channel (16384^2, r = 11 split path): device time of the fused
entry per library build: python tools/gpu/k5ab.py lib1.so lib2.so ..."""
import os, sys, importlib
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1203_5128_b200.workloads import config_image, CONFIGS

libs = sys.argv[1:] or ["paper_1203_5128_b200/libsbf.so"]
size = int(os.environ.get("K5_SIZE", "16384"))
f = torch.from_numpy(np.ascontiguousarray(config_image(5, 0, size=size))).cuda()
H, W = f.shape
for path in libs:
    os.environ["SBF_LIB"] = path
    import paper_1203_5128_b200._lib as L
    importlib.reload(L)
    lib = L.load()
    import paper_1203_5128_b200 as P
    from paper_1203_5128_b200.kernels import log_2_over_eps
    from paper_1203_5128_b200.spatial import to_c_spatial
    p = CONFIGS[5]
    params = P.FilterParams(sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], epsilon=p["epsilon"])
    sp = to_c_spatial(params.resolved_spatial()); R = params.resolved_radius()
    cap = 1 << 16
    ws = torch.empty(lib.sbf_shiftable_bf_workspace(H, W, 0, sp, L.PREC_FP32, cap), dtype=torch.uint8, device="cuda")
    stats = torch.empty(8, dtype=torch.float64, device="cuda")
    plan = torch.empty(64, dtype=torch.uint8, device="cuda")
    out = torch.empty_like(f)
    fb = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    def run():
        L.check(lib.sbf_shiftable_bf(f.data_ptr(), 0, H, W, sp, R, -1.0, p["sigma_r"], p["epsilon"], 0,
                                     log_2_over_eps(p["epsilon"]), L.PREC_FP32, out.data_ptr(), 0,
                                     plan.data_ptr(), stats.data_ptr(), fb.data_ptr(), cap,
                                     ws.data_ptr(), ws.numel(), st))
    run(); torch.cuda.synchronize()
    ref = out.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): run()
    e1.record(); e1.synchronize()
    same = torch.equal(out, ref)
    print(f"{os.path.basename(path):22s} cfg5 channel {H}x{W} ms {e0.elapsed_time(e1) / 3:.2f} "
          f"sum {float(out.double().sum()):.6f} repeat-identical {same}", flush=True)
    del ws
    torch.cuda.empty_cache()
