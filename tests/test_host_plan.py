"""The plan logic compiled into libsbf.so (same source as device kernel K2)
against the reference's golden plan table and the oracle.  CPU only: the
host twin needs no GPU."""

import math
import re
import os

import numpy as np
import pytest

from conftest import golden, REPO
from oracle import shiftbf_oracle as O
import paper_1203_5128_b200 as P
from paper_1203_5128_b200 import _lib

RULES = ["auto", "exact", "chernoff", "none"]


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    header = open(os.path.join(REPO, "include", "sbf.h")).read()
    declared = set(re.findall(r"\b(sbf_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.sbf_abi_version() == 1


def test_select_plan_table():
    g = golden("plans.npz")
    for T, sr, eps, rule, N, M in g["plans"]:
        p = P.select_plan(T, sr, eps, truncation=RULES[int(rule)])
        assert (p.N, p.M) == (int(N), int(M)), (T, sr, eps, rule)


def test_pins():
    g = golden("plans.npz")
    for N, e, M in g["exact"]:
        assert P.truncation_index_exact(int(N), float(e)) == int(M)
    for N, e, M in g["chernoff"]:
        assert P.truncation_index_chernoff(int(N), float(e)) == int(M)
    assert P.truncation_index_chernoff(263, 0.005) == 91
    assert P.truncation_index_exact(4, 0.5) == 0
    p = P.select_plan(0, 10, 0.01)
    assert (p.N, p.M) == (1, 0)
    for s, n in {5: 1053, 10: 263, 20: 66, 30: 29, 40: 16, 60: 7, 80: 4, 100: 3}.items():
        assert P.order_threshold(255, s, mode="round") == n


def test_bigint_path_agrees_with_fraction_oracle():
    lib = _lib.load()
    import ctypes as C
    rng = np.random.default_rng(3)
    for _ in range(200):
        N = int(rng.integers(1, 700))
        eps = float(rng.choice([0.005, 0.01, 0.05, 0.3, 0.999, 1e-6, 1e-30]))
        m = C.c_int()
        assert lib.sbf_truncation_index_exact_bigint(N, eps, C.byref(m)) == 0
        assert m.value == O.truncation_index_exact(N, eps), (N, eps)


def test_random_plans_vs_oracle():
    rng = np.random.default_rng(5)
    for _ in range(3000):
        T = float(rng.uniform(0, 400))
        sr = float(rng.choice([rng.uniform(1, 80), 10.0, 40.0]))
        eps = float(rng.choice([0.0, 0.001, 0.01, 0.05, rng.uniform(0, 0.9)]))
        rule = RULES[int(rng.integers(0, 4))]
        N = O.order_threshold(T, sr)
        if N > 3000 and (rule == "exact" or (rule == "auto" and 10 < sr <= 40)) and eps > 0:
            continue
        p = P.select_plan(T, sr, eps, truncation=rule)
        assert (T, p.N, p.M) == O.select_plan(T, sr, eps, rule)


def test_extended_box_params_and_support():
    for sigma, passes in ((0.5, 3), (2.0, 3), (3, 3), (5, 3), (6, 3), (8, 3), (12, 3), (10.0, 4), (2.0, 1)):
        assert P.extended_box_params(sigma, passes) == O.extended_box_params(sigma, passes)
    assert [P.support_radius(P.IteratedBox(s)) for s in (3, 5, 6, 8, 12)] == [9, 15, 18, 24, 36]
    assert P.support_radius(P.Box(4)) == 4


def test_parameter_validation_errors():
    with pytest.raises(P.InvalidParameterError):
        P.FilterParams(sigma_s=0, sigma_r=1)
    with pytest.raises(P.InvalidParameterError):
        P.FilterParams(sigma_s=1, sigma_r=1, epsilon=1.0)
    with pytest.raises(P.InvalidParameterError):
        P.select_plan(10, 10, 0.01, truncation="bogus")
    with pytest.raises(P.InvalidParameterError):
        P.truncation_index_chernoff(10, 0.0)
    with pytest.raises(P.InvalidParameterError):
        P.IteratedBox(0.0)
    with pytest.raises(ValueError):  # InvalidParameterError is a ValueError
        P.Box(-1)


def test_expansion_matches_reference_golden():
    g = golden("expansions.npz")
    plan = P.KernelPlan(P.KernelFamily.RAISED_COSINE, 10.0, 1.0, 229, 79, 0.01)
    e = P.raised_cosine_expansion(plan)
    np.testing.assert_array_equal(e.weights, g["w_229_79"])
    np.testing.assert_array_equal(e.frequencies, g["f_229_79"])


def test_libm_pow_ambiguity_resolved_like_cpython():
    # (T/sigma_r)**2 via libm pow differs from q*q here and moves the ceiling
    T = 95.65885888902615
    assert O.order_threshold(T, 1.0) == 3706
    assert P.order_threshold(T, 1.0) == 3706        # host twin calls pow() like CPython


def test_cfg4_term_table_matches_reference_plans():
    """workloads.CFG4_K (bench.py's shard weights) == K of the reference's
    own plans for the 64 config-4 images."""
    from conftest import golden
    from paper_1203_5128_b200.workloads import CFG4_K
    rows = golden("config_plans.npz")["rows"]
    ks = tuple(int(r[4]) // 2 - int(r[5]) + 1 for r in rows if int(r[0]) == 4)
    assert ks == CFG4_K


def test_binomial_weights_correctly_rounded():
    """Host twin (sbf_binomial_weights) == C(N,n)/2^N rounded once, as the
    reference computes it with exact integers (kernels.py:198-212),
    subnormal tails included."""
    import math
    from fractions import Fraction
    import paper_1203_5128_b200 as P
    assert P.binomial_weights(2, 0, 2).tolist() == [0.25, 0.5, 0.25]
    for N, lo, hi in [(1, 0, 1), (29, 7, 22), (263, 111, 152), (1100, 0, 1100), (2463, 0, 60)]:
        got = P.binomial_weights(N, lo, hi)
        want = [float(Fraction(math.comb(N, n), 1 << N)) for n in range(lo, hi + 1)]
        assert got.tolist() == want, N
