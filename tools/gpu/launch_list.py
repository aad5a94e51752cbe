"""One step of a config's device-resident pipeline between cudaProfilerStart/Stop, for
`ncu --profile-from-start off --metrics gpu__time_duration.sum --csv`: the list of
kernels one step launches (bench.py's gpu_launches constants come from these lists)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1203_5128_b200 as P
from paper_1203_5128_b200 import _lib
from paper_1203_5128_b200.workloads import config_image, CONFIGS
cfg = int(sys.argv[1])
p = CONFIGS[cfg]
params = P.FilterParams(sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], epsilon=p["epsilon"],
                        precision="hdr" if cfg == 3 else "fp32")
cudart = torch.cuda.cudart()
if cfg == 5:
    from paper_1203_5128_b200.dist import StripFilter, strip_halo, strip_plan
    size = 4096  # same kernels as 16384^2, one launch each
    s = strip_plan(size, 1, strip_halo(params))[0]
    bufs = [torch.from_numpy(np.ascontiguousarray(config_image(5, c, size=size))).cuda() for c in range(3)]
    sf = StripFilter(bufs, s, size, params)
    sf.run(); torch.cuda.synchronize()
    cudart.cudaProfilerStart(); sf.run(); torch.cuda.synchronize(); cudart.cudaProfilerStop()
else:
    img = torch.from_numpy(np.ascontiguousarray(config_image(cfg), dtype=np.float64 if cfg == 1 else np.float32)).cuda()
    P.shiftable_bf(img, params); torch.cuda.synchronize()
    cudart.cudaProfilerStart(); P.shiftable_bf(img, params); torch.cuda.synchronize(); cudart.cudaProfilerStop()
