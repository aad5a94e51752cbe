"""Per-role cycle breakdown of the warp-specialised sweep (library built with -DSBF_SWW_PROF=1):
reads the counters the kernel adds into the segment-counter area of the workspace."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1203_5128_b200.workloads import config_image, CONFIGS
import paper_1203_5128_b200._lib as L
import paper_1203_5128_b200 as P
from paper_1203_5128_b200.kernels import log_2_over_eps
from paper_1203_5128_b200.spatial import to_c_spatial
lib = L.load()
lib.sbf_set_sweep_variant(2)
cfg = int(os.environ.get("CFG", "4"))
p = CONFIGS[cfg]
f = torch.from_numpy(np.ascontiguousarray(config_image(cfg), dtype=np.float32)).cuda()
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
run(); run()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); run(); e1.record(); torch.cuda.synchronize()
c = f_ws[256:256 + 12 * 8].view(torch.int64).cpu().numpy().astype(np.float64)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
v = c[:4] / (nsm * 8); h = c[4:] / (nsm * 8)
print(f"K3 {e0.elapsed_time(e1):.3f} ms; cycles per warp (mean)")
print("V: ft_full wait %.0f  vb_empty wait %.0f  compute %.0f  item %.0f  | total %.0f" % (*v, v.sum()))
print("H: item %.0f  pairbar1 %.0f  vb_full wait %.0f  cascade %.0f  pairbar2 %.0f  af wait %.0f  accumulate %.0f  | total %.0f" % (*h[:7], h[:7].sum()))
