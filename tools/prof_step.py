"""Minimal driver for ncu: N steps of the device pipeline on one config.

    python tools/prof_step.py [--config 2] [--steps 3]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_5128_b200 as P  # noqa: E402
from paper_1203_5128_b200 import _lib  # noqa: E402
from paper_1203_5128_b200.kernels import log_2_over_eps  # noqa: E402
from paper_1203_5128_b200.spatial import to_c_spatial  # noqa: E402
from paper_1203_5128_b200.workloads import CONFIGS, config_image  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--size", type=int, default=None)
ap.add_argument("--prec", default="fp32", choices=["fp32", "hdr", "auto"])
ap.add_argument("--fp64-method", type=int, default=None, help="sbf_set_fp64_method (0 sweeps, 1 model, 2 dual)")
a = ap.parse_args()
p = CONFIGS[a.config]
img = config_image(a.config, size=a.size)
H, W = img.shape
lib = _lib.load()
f = torch.from_numpy(np.ascontiguousarray(img)).cuda()
dt = _lib.SBF_F64 if f.dtype == torch.float64 else _lib.SBF_F32
params = P.FilterParams(sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], epsilon=p["epsilon"])
sp = to_c_spatial(params.resolved_spatial())
R = params.resolved_radius()
prec = {"fp32": _lib.PREC_FP32, "hdr": _lib.PREC_HDR, "auto": _lib.PREC_AUTO}[a.prec]
if a.fp64_method is not None:
    lib.sbf_set_fp64_method(a.fp64_method)
cap = 1 << 16
ws = torch.empty(lib.sbf_shiftable_bf_workspace(H, W, dt, sp, prec, cap), dtype=torch.uint8, device="cuda")
stats = torch.empty(8, dtype=torch.float64, device="cuda")
plan = torch.empty(64, dtype=torch.uint8, device="cuda")
out = torch.empty((H, W), dtype=torch.float32, device="cuda")
fb = torch.zeros(1, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(a.steps):
    _lib.check(lib.sbf_shiftable_bf(f.data_ptr(), dt, H, W, sp, R, -1.0, p["sigma_r"], p["epsilon"], 0,
                                    log_2_over_eps(p["epsilon"]), prec, out.data_ptr(), _lib.SBF_F32,
                                    plan.data_ptr(), stats.data_ptr(), fb.data_ptr(), cap,
                                    ws.data_ptr(), ws.numel(), st))
torch.cuda.synchronize()
pc = _lib.SbfPlan.from_buffer_copy(plan.cpu().numpy().tobytes())
print("ok", H, W, pc.N, pc.M, pc.K_eval, float(out.mean()))
