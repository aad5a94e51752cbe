"""Host-side timeline of one public shiftable_bf call (config 2, pinned input):
cProfile of the Python layer plus CUDA-event device time, for e2e triage."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_5128_b200 as P  # noqa: E402
from paper_1203_5128_b200.workloads import config_image  # noqa: E402

img = config_image(2)
pinned = torch.from_numpy(np.ascontiguousarray(img)).pin_memory()
params = P.FilterParams(sigma_s=5, sigma_r=10, epsilon=0.01)
for _ in range(5):
    P.shiftable_bf(pinned, params)
torch.cuda.synchronize()
n = 50
t = time.perf_counter()
for _ in range(n):
    P.shiftable_bf(pinned, params)
print(f"wall per call {(time.perf_counter() - t) / n * 1e3:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    P.shiftable_bf(pinned, params)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
