"""Size-independent properties of the CUDA filter at BASELINE sizes, and the
reference's own behavioural tests (test_bilateral.py:65-107) on the CUDA path.

The bilateral filter is equivariant under intensity shifts and under the
dihedral symmetries of the pixel grid (the spatial smoother and the local
range are symmetric), its untruncated output is a convex combination of the
window, and a constant image is a fixed point.  The strip decomposition of
K3 (and the split sweep) is not symmetric, so transposed / flipped runs
exercise different strip and band boundaries of the same data.
"""

import numpy as np
import pytest

from oracle import shiftbf_oracle as O
import paper_1203_5128_b200 as P
from paper_1203_5128_b200.workloads import config_image

pytestmark = pytest.mark.gpu
TOL = 1e-2  # gray levels (BASELINE north-star tolerance)


def _bf(img, **kw):
    return P.shiftable_bf(np.ascontiguousarray(img), P.FilterParams(**kw))


@pytest.mark.parametrize("cfg,size", [(2, None), (4, 2048), (5, 2048)])
def test_dihedral_equivariance_full_size(cfg, size):
    c = {2: (5.0, 10.0), 4: (6.0, 20.0), 5: (12.0, 15.0)}[cfg]
    img = config_image(cfg, size=size).astype(np.float32)
    kw = dict(sigma_s=c[0], sigma_r=c[1], epsilon=0.01)
    base = _bf(img, **kw)
    for op in (lambda a: a.T, lambda a: a[:, ::-1], lambda a: a[::-1, :]):
        res = _bf(op(img), **kw)
        assert (res.plan.T, res.plan.N, res.plan.M) == (base.plan.T, base.plan.N, base.plan.M)
        assert float(np.abs(res.image - op(base.image)).max()) <= TOL


def test_intensity_shift_equivariance_full_size():
    img = config_image(2).astype(np.float64)
    kw = dict(sigma_s=5.0, sigma_r=10.0, epsilon=0.01)
    a = _bf(img, **kw)
    b = _bf(img + 1000.0, **kw)
    assert (a.plan.T, a.plan.N, a.plan.M) == (b.plan.T, b.plan.N, b.plan.M)
    assert float(np.abs((b.image - 1000.0) - a.image).max()) <= TOL


def test_constant_image_fixed_point_full_size():
    img = np.full((1024, 1024), 77.0)
    for kw in (dict(sigma_s=3, sigma_r=20, spatial=P.Box(3)), dict(sigma_s=5, sigma_r=10, epsilon=0.01)):
        res = _bf(img, **kw)
        assert res.plan.T == 0.0 and res.plan.N == 1 and res.fallback_pixels == 0
        assert float(np.abs(res.image - 77.0).max()) <= 1e-4


@pytest.mark.parametrize("sigma_r", [15, 25, 60])
def test_exact_shiftability_against_direct_expansion(sigma_r):
    """reference test_bilateral.py:79-88: with eps = 0 the filter equals the
    brute-force filter with the (untruncated) raised-cosine kernel cos^N."""
    rng = np.random.default_rng(sigma_r)
    for _ in range(3):
        img = rng.uniform(0, 255, (32, 32))
        res = _bf(img, sigma_s=3, sigma_r=sigma_r, epsilon=0.0, spatial=P.Box(3))
        N = res.plan.N
        g = 1.0 / (np.sqrt(N) * sigma_r)
        num = np.zeros_like(img)
        den = np.zeros_like(img)
        h, w = img.shape
        for dy in range(-3, 4):
            for dx in range(-3, 4):
                ys, yd = slice(max(0, dy), h + min(0, dy)), slice(max(0, -dy), h - max(0, dy))
                xs, xd = slice(max(0, dx), w + min(0, dx)), slice(max(0, -dx), w - max(0, dx))
                nb = img[ys, xs]
                k = np.cos(g * (nb - img[yd, xd])) ** N
                num[yd, xd] += k * nb
                den[yd, xd] += k
        assert float(np.abs(res.image - num / den).max()) <= TOL


def test_output_within_local_range_when_untruncated():
    """reference test_bilateral.py:102-107 (fp32 path: a 1e-3 margin)."""
    img = np.random.default_rng(3).uniform(0, 255, (24, 24))
    out = _bf(img, sigma_s=2, sigma_r=20, epsilon=0.0, spatial=P.Box(2)).image
    assert (out <= O.max_filter_2d(img, 2) + 1e-3).all()
    assert (out >= -O.max_filter_2d(-img, 2) - 1e-3).all()


def test_plan_reflects_computed_t_and_fixed_t():
    """reference test_bilateral.py:90-100."""
    img = np.random.default_rng(4).uniform(0, 200, (24, 24))
    res = _bf(img, sigma_s=2, sigma_r=30, epsilon=0.01, spatial=P.Box(2))
    assert res.plan == P.select_plan(P.compute_T(img, 2), 30, 0.01)
    res = _bf(img[:16, :16], sigma_s=2, sigma_r=30, spatial=P.Box(2), fixed_T=255.0)
    assert res.plan.T == 255.0
