"""The rest of the reference's public surface on the CUDA path: standalone
smoothers (spatial.py:65-182), direct_bf with expansion kernels
(bilateral.py:101-103), direct_nlm (nlm.py:140-183), backend registry and
helpers, against the reference's own golden vectors."""

import numpy as np
import pytest

from conftest import golden
from oracle import shiftbf_oracle as O
import paper_1203_5128_b200 as P

pytestmark = pytest.mark.gpu


def test_smoothers_match_reference_golden():
    g = golden("smoothing.npz")
    for k in range(9):
        sigma, passes = g[f"sig_{k}"]
        out = P.iterated_box_gaussian(g[f"img_{k}"], float(sigma), int(passes))
        np.testing.assert_allclose(out, g[f"out_{k}"], rtol=1e-11, atol=1e-9)
        out2 = P.apply_spatial(g[f"img_{k}"], P.IteratedBox(float(sigma), int(passes)))
        np.testing.assert_array_equal(out, out2)
    for j in range(5):
        out = P.box_filter(g[f"bimg_{j}"], int(g[f"brad_{j}"]))
        np.testing.assert_allclose(out, g[f"bout_{j}"], rtol=1e-11, atol=1e-9)


def test_fir_gaussian_matches_restatement():
    """spatial.py:142-172: separable sampled Gaussian, renormalised per clamped window."""
    rng = np.random.default_rng(5)
    img = rng.uniform(0, 255, (37, 53))
    for sigma, R in ((1.5, 3), (4.0, 9), (2.0, 30)):
        taps = np.exp(-(np.arange(-R, R + 1) ** 2) / (2.0 * sigma * sigma))

        def lines(a):
            n = a.shape[1]
            num = np.zeros_like(a)
            den = np.zeros(n)
            for k in range(-R, R + 1):
                if abs(k) >= n:
                    continue
                src, dst = slice(max(0, k), n + min(0, k)), slice(max(0, -k), n - max(0, k))
                num[:, dst] += taps[k + R] * a[:, src]
                den[dst] += taps[k + R]
            return num / den

        ref = lines(lines(img).T).T
        out = P.fir_gaussian(img, sigma, R)
        np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("sigma_r", [15, 25, 60])
def test_exact_shiftability_direct_expansion(sigma_r):
    """reference test_bilateral.py:79-88: shiftable_bf with eps = 0 equals
    direct_bf with expansion_range(raised_cosine_expansion(plan))."""
    rng = np.random.default_rng(sigma_r)
    for _ in range(3):
        img = rng.uniform(0, 255, (32, 32))
        res = P.shiftable_bf(img, P.FilterParams(sigma_s=3, sigma_r=sigma_r, epsilon=0.0,
                                                 spatial=P.Box(3)))
        oracle = P.direct_bf(img, P.Box(3), P.expansion_range(P.raised_cosine_expansion(res.plan)))
        assert float(np.abs(res.image - oracle).max()) <= 1e-2


def _nlm_case(g, k):
    offs = [tuple(int(v) for v in o) for o in g[f"offs_{k}"]]
    par = g[f"par_{k}"]
    p = len(offs)
    kind, a, b, rad, kern = par[p:]
    mode = P.Box(int(a)) if kind == 0 else P.FirGaussian(float(a), int(b))
    return offs, [float(v) for v in par[:p]], mode, int(rad), int(kern)


@pytest.mark.parametrize("k", range(3))
def test_direct_nlm_matches_reference_golden(k):
    g = golden("direct_nlm.npz")
    offs, sgs, mode, rad, kern = _nlm_case(g, k)
    img = g[f"img_{k}"]
    patch = P.PatchSpec(tuple(offs), tuple(sgs))
    if kern == 0:
        out = P.direct_nlm(img, patch, mode, rad)
    else:
        T = P.compute_T(img, rad + patch.max_offset_norm)
        plans = [P.select_plan(T, sg, 0.05) for sg in sgs]
        out = P.direct_nlm(img, patch, mode, rad, [P.expansion_range_for(pl) for pl in plans])
    np.testing.assert_allclose(out, g[f"out_{k}"], rtol=1e-10, atol=1e-8)


def test_shiftable_nlm_equals_direct_nlm_with_expansions():
    """The tensor-product shiftable NLM is exactly the brute-force NLM with the
    per-component truncated expansions (up to fp64 rounding)."""
    img = np.random.default_rng(11).uniform(0, 120, (30, 33))
    patch = P.PatchSpec(((0, 0), (0, 1)), (45.0, 45.0))
    res = P.coarse_nlm_shiftable(img, patch, P.Box(2), 2, 0.05)
    direct = P.direct_nlm(img, patch, P.Box(2), 2, [P.expansion_range_for(pl) for pl in res.plans])
    np.testing.assert_allclose(res.image, direct, rtol=1e-9, atol=1e-7)


def test_helpers_and_out_of_scope_entry_points():
    assert P.available_backends() == ["cuda"] and P.backend_name() == "cuda"
    assert P.use_backend("cuda") == "cuda"
    with pytest.raises(ValueError):
        P.use_backend("python")
    img = np.random.default_rng(2).uniform(0, 255, (20, 20))
    assert P.brute_force_T(img, 3) == O.brute_force_T(img, 3)
    with pytest.raises(P.InvalidParameterError):
        P.shiftable_bf_poly(img / 255.0, P.FilterParams(sigma_s=2, sigma_r=0.2))
    with pytest.raises(P.InvalidParameterError):
        P.direct_bf(img, P.Box(1), P.polynomial_range(P.select_plan(1.0, 0.2, 0.0)))
