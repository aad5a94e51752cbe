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


def _random_case(seed):
    rng = np.random.default_rng(seed)
    h, w = int(rng.integers(1, 260)), int(rng.integers(1, 260))
    kind = rng.choice(["u8", "f32", "f64", "u16"])
    hi = 65535.0 if kind == "u16" else 255.0
    img = rng.uniform(0, hi, (h, w))
    if rng.random() < 0.5:  # piecewise-constant regions + noise, like the configs
        img = np.where(np.add.outer(np.arange(h), np.arange(w)) % 37 < 18, 0.2 * hi, 0.7 * hi)
        img = img + rng.normal(0, hi / 40, (h, w))
    if kind == "u8":
        img = np.clip(np.round(img), 0, 255).astype(np.uint8)
    elif kind == "u16":
        img = np.clip(np.round(img), 0, 65535).astype(np.uint16)
    elif kind == "f32":
        img = img.astype(np.float32)
    sigma_s = float(rng.choice([0.7, 1.5, 3.0, 5.0, 6.0, 9.7, 11.6]))
    sigma_r = float(rng.choice([8.0, 20.0, 45.0, 90.0])) * (257.0 if kind == "u16" else 1.0)
    eps = float(rng.choice([0.0, 0.01, 0.05]))
    box = rng.random() < 0.25
    fixed = None if rng.random() < 0.8 else float(hi)
    return img, sigma_s, sigma_r, eps, box, fixed


@pytest.mark.parametrize("seed", range(64))
def test_random_cases_vs_c_oracle(seed):
    """Seeded random shapes / dtypes / parameters (incl. 16-bit HDR, box mode,
    fixed T, the split sweep at r >= 9) against the C oracle."""
    from oracle import coracle as CO
    CO.build()
    img, ss, sr, eps, box, fixed = _random_case(seed)
    spatial = P.Box(max(1, int(round(ss)))) if box else None
    osp = ("box", max(1, int(round(ss)))) if box else None
    res = P.shiftable_bf(img, P.FilterParams(sigma_s=ss, sigma_r=sr, epsilon=eps, spatial=spatial,
                                             fixed_T=fixed))
    ref = CO.shiftable_bf(np.asarray(img, dtype=np.float64), ss, sr, eps, spatial=osp, fixed_T=fixed)
    assert (res.plan.T, res.plan.N, res.plan.M) == (ref["T"], ref["N"], ref["M"])
    d = np.abs(res.image - ref["image"])
    assert float(d.max()) <= TOL and float(np.sqrt(np.mean(d * d))) <= 1e-3, (img.dtype, img.shape, ss, sr, eps, box)
