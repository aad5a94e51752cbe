import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1203_5128_b200._lib as L
from paper_1203_5128_b200.workloads import config_image
lib = L.load()
for cfg, idx, R in [(4, 0, 18), (4, 5, 18), (5, 0, 36)]:
    f = torch.from_numpy(np.ascontiguousarray(config_image(cfg, idx))).cuda()
    H, W = f.shape
    stats = torch.empty(8, dtype=torch.float64, device="cuda")
    ws = torch.zeros(lib.sbf_local_range_workspace(H, W, 0), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    L.check(lib.sbf_local_range(f.data_ptr(), 0, H, W, W, R, 0, H, None, stats.data_ptr(), ws.data_ptr(), ws.numel(), st))
    torch.cuda.synchronize()
    tx, ty = (W + 31) // 32, (H + 31) // 32
    stx, sty = (W + 15) // 16, (H + 15) // 16
    off = 2 * stx * sty * 4
    off = (off + 255) // 256 * 256
    off += ((tx * ty * 8) + 255) // 256 * 256
    sl = ws[off:off + 24].cpu().numpy().view(np.uint64)
    print(cfg, idx, "T", float(stats[0]), "round1 tiles", int(sl[1]), "round2 tiles", int(sl[2]), flush=True)
