"""K3-only device time (stage mask 1, no L2 flush) for config 2; A/B with SBF_LIB=..."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1203_5128_b200 as P
from paper_1203_5128_b200 import _lib
from paper_1203_5128_b200.kernels import log_2_over_eps
from paper_1203_5128_b200.spatial import to_c_spatial
from paper_1203_5128_b200.workloads import config_image
img = config_image(2); H, W = img.shape
lib = _lib.load()
f = torch.from_numpy(np.ascontiguousarray(img)).cuda()
params = P.FilterParams(sigma_s=5, sigma_r=10, epsilon=0.01)
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
lib.sbf_plan_device(stats.data_ptr(), 0, 0.0, 10.0, 0.01, 0, log_2_over_eps(0.01), plan.data_ptr(), terms.data_ptr(), 1 << 16, st)
lib.sbf_set_stage_mask(1)
def run():
    lib.sbf_filter(f.data_ptr(), 0, H, W, W, 0, H, 0, H, sp, plan.data_ptr(), terms.data_ptr(), stats.data_ptr(), 0, out.data_ptr(), 0, fb.data_ptr(), f_ws.data_ptr(), f_ws.numel(), st)
for _ in range(5): run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): run()
e1.record(); e1.synchronize()
print(os.environ.get("SBF_LIB", "default").split("/")[-1], "K3 (+memset) ms", e0.elapsed_time(e1) / 20)
