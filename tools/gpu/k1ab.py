"""K1 (sbf_local_range) device time per call, A/B across library builds:
python tools/gpu/k1ab.py lib1.so lib2.so ...  (configs 2, 4 image 0, 5 channel 0)."""
import os, sys, importlib
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1203_5128_b200.workloads import config_image

libs = sys.argv[1:] or ["paper_1203_5128_b200/libsbf.so"]
cases = [(cfg, R, torch.from_numpy(np.ascontiguousarray(config_image(cfg))).cuda())
         for cfg, R in ((2, 15), (4, 18), (5, 36), (1, 9))]
for path in libs:
    os.environ["SBF_LIB"] = path
    import paper_1203_5128_b200._lib as L
    importlib.reload(L)
    lib = L.load()
    for cfg, R, f in cases:
        H, W = f.shape
        dt = L.SBF_F64 if f.dtype == torch.float64 else L.SBF_F32
        stats = torch.empty(8, dtype=torch.float64, device="cuda")
        ws = torch.empty(lib.sbf_local_range_workspace(H, W, dt), dtype=torch.uint8, device="cuda")
        M = torch.empty_like(f)
        st = torch.cuda.current_stream().cuda_stream
        def run(m=None):
            L.check(lib.sbf_local_range(f.data_ptr(), dt, H, W, W, R, 0, H, m, stats.data_ptr(),
                                        ws.data_ptr(), ws.numel(), st))
        run(M.data_ptr())
        torch.cuda.synchronize()
        T = float(stats[0].item())
        msum = float(M.double().sum().item())
        for _ in range(3): run()
        torch.cuda.synchronize()
        n = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n): run()
        e1.record(); e1.synchronize()
        us = e0.elapsed_time(e1) / n * 1e3
        T2 = float(stats[0].item())
        st2 = stats[1:3].tolist()
        gbs = H * W * f.element_size() / (us * 1e-6) / 1e9
        print(f"{os.path.basename(path):20s} cfg{cfg} {H}x{W} R={R} K1 {us:8.1f} us  ({gbs:6.0f} GB/s of f)  T={T!r} T(no M)={T2!r} min/max={st2} sumM={msum!r}", flush=True)
