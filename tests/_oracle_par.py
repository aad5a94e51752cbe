"""Band-parallel C oracle for full-size parity cases (test helper).

Rows are cut into one band per host core with a halo equal to the spatial
support and the global T fixed, which reproduces the whole-image oracle
exactly (SURVEY.md Appendix C strip equivalence; checked in
test_oracle_golden.py::test_band_split_is_exact)."""

import multiprocessing as mp
import os

import numpy as np

from oracle import coracle as CO
from oracle import shiftbf_oracle as O


def _band(args):
    part, y0, y1, a, kw = args  # part = image rows [a, a + len(part))
    out = CO.shiftable_bf(part, **kw)
    return y0, y1, out["image"][y0 - a:y1 - a], out["fallback_pixels"]


def shiftable_bf_full(img, sigma_s, sigma_r, epsilon, procs=None):
    CO.build()
    f = O.as_image(img)
    r, a = O.extended_box_params(sigma_s, 3)
    halo = 3 * (r + (1 if a > 0 else 0))
    T = CO.compute_T(f, max(1, halo))
    T, N, M = O.select_plan(T, sigma_r, epsilon)
    H = f.shape[0]
    procs = max(1, min(procs or os.cpu_count() or 1, H // 32))
    rows = -(-H // procs)
    kw = dict(sigma_s=sigma_s, sigma_r=sigma_r, epsilon=epsilon, fixed_T=T)
    jobs = []
    for y in range(0, H, rows):
        a, b = max(0, y - halo), min(H, y + rows + halo)
        jobs.append((f[a:b], y, min(H, y + rows), a, kw))
    out = np.empty_like(f)
    # spawn: the caller may hold CUDA threads, where fork is unsafe
    with mp.get_context("spawn").Pool(len(jobs)) as pool:
        for y0, y1, part, _ in pool.map(_band, jobs):
            out[y0:y1] = part
    return dict(image=out, T=T, N=N, M=M)
