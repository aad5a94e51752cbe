"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import math

import numpy as np
import pytest

from conftest import golden
from oracle import shiftbf_oracle as O

RULES = ["auto", "exact", "chernoff", "none"]


def test_plan_table_matches_reference():
    g = golden("plans.npz")
    for T, sr, eps, rule, N, M in g["plans"]:
        _, n, m = O.select_plan(T, sr, eps, RULES[int(rule)])
        assert (n, m) == (int(N), int(M)), (T, sr, eps, rule)


def test_n0_table_and_truncation_pins():
    g = golden("plans.npz")
    n0 = {int(s): int(n) for s, n in g["n0"]}
    assert n0 == {5: 1053, 10: 263, 20: 66, 30: 29, 40: 16, 60: 7, 80: 4, 100: 3}
    for N, e, M in g["exact"]:
        assert O.truncation_index_exact(int(N), float(e)) == int(M)
    for N, e, M in g["chernoff"]:
        assert O.truncation_index_chernoff(int(N), float(e)) == int(M)
    assert O.truncation_index_chernoff(263, 0.005) == 91


def test_expansion_weights():
    g = golden("expansions.npz")
    for key in g.files:
        if not key.startswith("w_"):
            continue
        N, M = map(int, key[2:].split("_"))
        n, w, f = O.raised_cosine_terms(N, M, {2: 1.0, 29: 30.0, 229: 10.0, 263: 10.0, 2463: 800.0}[N])
        np.testing.assert_array_equal(w, g[key])
        np.testing.assert_array_equal(f, g["f_" + key[2:]])


def test_max_filter_bit_exact():
    g = golden("maxfilter.npz")
    for k in range(40):
        img, R = g[f"img_{k}"], int(g[f"R_{k}"])
        assert np.array_equal(O.max_filter_2d(img, R), g[f"M_{k}"])
        assert O.compute_T(img, R) == float(g[f"T_{k}"])
    for k in range(20):
        assert np.array_equal(O.max_filter_1d(g[f"seq_{k}"], int(g[f"sR_{k}"])), g[f"smax_{k}"])


def test_brute_force_T_agrees():
    rng = np.random.default_rng(12)
    for _ in range(10):
        img = rng.uniform(0, 255, (int(rng.integers(2, 30)), int(rng.integers(2, 30))))
        R = int(rng.integers(1, 6))
        assert O.compute_T(img, R) == O.brute_force_T(img, R)


def test_smoothing_matches_reference():
    g = golden("smoothing.npz")
    for k in range(9):
        sigma, passes = g[f"sig_{k}"]
        r, a = O.extended_box_params(float(sigma), int(passes))
        assert (r, a) == (int(g[f"ra_{k}"][0]), float(g[f"ra_{k}"][1]))
        np.testing.assert_allclose(O.iterated_box(g[f"img_{k}"], float(sigma), int(passes)),
                                   g[f"out_{k}"], rtol=1e-12, atol=1e-9)
    for j in range(5):
        np.testing.assert_allclose(O.box_filter(g[f"bimg_{j}"], int(g[f"brad_{j}"])),
                                   g[f"bout_{j}"], rtol=1e-12, atol=1e-9)


def _run_case(g, k):
    ss, sr, eps, boxr, fT, tr = g[f"par_{k}"]
    spatial = None if boxr < 0 else ("box", int(boxr))
    return O.shiftable_bf(g[f"img_{k}"], float(ss), float(sr), float(eps), spatial=spatial,
                          fixed_T=None if math.isnan(fT) else float(fT), truncation=RULES[int(tr)])


@pytest.mark.parametrize("k", range(16))
def test_shiftable_bf_matches_reference(k):
    g = golden("bf_small.npz")
    res = _run_case(g, k)
    T, N, M, fb = g[f"plan_{k}"]
    assert (res["T"], res["N"], res["M"], res["fallback_pixels"]) == (T, int(N), int(M), int(fb))
    np.testing.assert_allclose(res["image"], g[f"out_{k}"], rtol=1e-9, atol=1e-7)


def test_config1_plan_and_crop():
    from paper_1203_5128_b200.workloads import config_image
    g = golden("config1.npz")
    img = config_image(1)
    assert O.compute_T(img, 9) == 251.39522633396712
    assert O.select_plan(251.39522633396712, 30.0, 0.01) == (251.39522633396712, 29, 7)
    np.testing.assert_array_equal(O.max_filter_2d(img, 9)[::8, ::8], g["M"])


# ---- the C restatement (oracle/sbf_oracle.c), pinned to the same vectors ----
def _coracle():
    from oracle import coracle
    coracle.build()
    return coracle


def test_c_oracle_max_filter_bit_exact():
    CO = _coracle()
    g = golden("maxfilter.npz")
    for k in range(40):
        img, R = g[f"img_{k}"], int(g[f"R_{k}"])
        assert np.array_equal(CO.max_filter_2d(img, R), g[f"M_{k}"])
        assert CO.compute_T(img, R) == float(g[f"T_{k}"])


@pytest.mark.parametrize("k", range(16))
def test_c_oracle_matches_reference(k):
    CO = _coracle()
    g = golden("bf_small.npz")
    ss, sr, eps, boxr, fT, tr = g[f"par_{k}"]
    spatial = None if boxr < 0 else ("box", int(boxr))
    res = CO.shiftable_bf(g[f"img_{k}"], float(ss), float(sr), float(eps), spatial=spatial,
                          fixed_T=None if math.isnan(fT) else float(fT), truncation=RULES[int(tr)])
    T, N, M, fb = g[f"plan_{k}"]
    assert (res["T"], res["N"], res["M"], res["fallback_pixels"]) == (T, int(N), int(M), int(fb))
    np.testing.assert_allclose(res["image"], g[f"out_{k}"], rtol=1e-9, atol=1e-7)


def test_c_oracle_agrees_with_numpy_oracle():
    CO = _coracle()
    rng = np.random.default_rng(5)
    for spatial in (None, ("box", 3), ("iterated", 2.5, 2)):
        img = rng.uniform(0, 255, (41, 67))
        a = CO.shiftable_bf(img, 2.5, 20.0, 0.01, spatial=spatial)
        b = O.shiftable_bf(img, 2.5, 20.0, 0.01, spatial=spatial)
        assert (a["T"], a["N"], a["M"]) == (b["T"], b["N"], b["M"])
        np.testing.assert_allclose(a["image"], b["image"], rtol=1e-10, atol=1e-9)


def test_band_split_is_exact():
    """The band-parallel helper used by the full-size GPU parity tests
    reproduces the whole-image oracle."""
    import _oracle_par
    CO = _coracle()
    from paper_1203_5128_b200.workloads import config_image
    img = config_image(2, size=160)
    whole = CO.shiftable_bf(img, 5.0, 10.0, 0.01)
    split = _oracle_par.shiftable_bf_full(img, 5.0, 10.0, 0.01, procs=4)
    assert (split["T"], split["N"], split["M"]) == (whole["T"], whole["N"], whole["M"])
    np.testing.assert_allclose(split["image"], whole["image"], rtol=0, atol=1e-9)


def _direct_spatial(par):
    kind, a, b, rad, sr = par
    sp = ("box", int(b)) if kind == 0 else ("fir", float(a), int(b))
    return sp, (None if rad < 0 else int(rad)), float(sr)


@pytest.mark.parametrize("k", range(8))
def test_direct_bf_matches_reference(k):
    g = golden("direct.npz")
    sp, rad, sr = _direct_spatial(g[f"par_{k}"])
    out = O.direct_bf(g[f"img_{k}"], sp, sr, radius=rad)
    np.testing.assert_allclose(out, g[f"out_{k}"], rtol=1e-12, atol=1e-9)


def _nlm_case(g, k):
    offs = [tuple(int(v) for v in o) for o in g[f"offs_{k}"]]
    par = g[f"par_{k}"]
    p = len(offs)
    sg = [float(v) for v in par[:p]]
    kind, a, rad, eps = par[p:]
    sp = ("box", int(a)) if kind == 0 else ("iterated", float(a), 3)
    return offs, sg, sp, int(rad), float(eps)


@pytest.mark.parametrize("k", range(5))
def test_coarse_nlm_matches_reference(k):
    g = golden("nlm.npz")
    offs, sg, sp, rad, eps = _nlm_case(g, k)
    res = O.coarse_nlm(g[f"img_{k}"], offs, sg, sp, rad, eps)
    assert [(res["T"], N, M) for N, M in res["plans"]] == [tuple(r) for r in g[f"plans_{k}"].tolist()]
    np.testing.assert_allclose(res["image"], g[f"out_{k}"], rtol=1e-10, atol=1e-8)


def test_nlm_item_table_folding():
    """Folding +-w per component keeps the tensor product exact."""
    from paper_1203_5128_b200 import kernels as K
    from paper_1203_5128_b200.nlm import _folded
    for N, M in ((7, 0), (15, 3), (4, 1)):
        plan = K.KernelPlan(K.KernelFamily.RAISED_COSINE, 10.0, 100.0, N, M, 0.01 if M else 0.0)
        fold = _folded(plan)
        e = K.raised_cosine_expansion(plan)
        # sum_n d_n cos(w_n s) == sum_folded scale cos(2 pi turns s) for sample s
        for s in (0.0, 1.3, 17.0, -40.5):
            full = float(np.sum(e.weights * np.cos(e.frequencies * s)))
            folded = sum(sc * math.cos(2 * math.pi * t * s) for sc, t in fold)
            assert abs(full - folded) < 1e-12
