"""Range-kernel plans: same public surface as reference kernels.py:39-243.

The (N, M) selection runs in the shared C/CUDA plan code (`sbf_select_plan`
on the host, kernel K2 on the device — one source, csrc/sbf_plan_logic.cuh),
so the plan the GPU filter uses is the plan these functions return.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from .errors import InvalidParameterError, UnsupportedOrderError

RC_ORDER_COEFF = 0.405      # kernels.py:31
POLY_ORDER_COEFF = 0.5      # kernels.py:32
POLYNOMIAL_ORDER_CAP = 30   # kernels.py:36


class KernelFamily(Enum):
    RAISED_COSINE = "cosine"
    POLYNOMIAL = "poly"


@dataclass(frozen=True)
class KernelPlan:
    """N: kernel order; M: terms dropped from each tail (kernels.py:44-80)."""

    family: KernelFamily
    sigma_r: float
    T: float
    N: int
    M: int
    epsilon: float

    def __post_init__(self):
        if self.sigma_r <= 0:
            raise InvalidParameterError("sigma_r must be positive")
        if self.T < 0:
            raise InvalidParameterError("T must be non-negative")
        if self.N < 1:
            raise InvalidParameterError("order N must be >= 1")
        if not 0 <= self.epsilon < 1:
            raise InvalidParameterError("epsilon must lie in [0, 1)")
        if self.M < 0 or 2 * self.M >= self.N:
            raise InvalidParameterError("need 0 <= 2M < N")
        if self.epsilon == 0 and self.M != 0:
            raise InvalidParameterError("M must be 0 when epsilon is 0")

    @property
    def retained_terms(self) -> int:
        return self.N - 2 * self.M + 1

    @property
    def dropped_fraction(self) -> float:
        return 2 * self.M / (self.N + 1)


@dataclass(frozen=True)
class ExpansionTerm:
    weight: float
    frequency: float
    index: int


@dataclass(frozen=True)
class Expansion:
    plan: KernelPlan
    weights: np.ndarray = field(repr=False)
    frequencies: np.ndarray = field(repr=False)
    indices: np.ndarray = field(repr=False)

    @property
    def terms(self):
        return [ExpansionTerm(float(w), float(f), int(n))
                for w, f, n in zip(self.weights, self.frequencies, self.indices)]

    @property
    def retained_mass(self) -> float:
        return float(self.weights.sum())


def _check_order_and_tolerance(N, epsilon):
    if N < 1:
        raise InvalidParameterError("order N must be >= 1")
    if not 0 <= epsilon < 1:
        raise InvalidParameterError("epsilon must lie in [0, 1)")


def order_threshold(T, sigma_r, family=KernelFamily.RAISED_COSINE, mode="ceil") -> int:
    """Smallest valid order for range T and width sigma_r (kernels.py:109-128)."""
    if sigma_r <= 0:
        raise InvalidParameterError("sigma_r must be positive")
    if T < 0:
        raise InvalidParameterError("T must be non-negative")
    if mode not in ("ceil", "round"):
        raise InvalidParameterError(f"unknown rounding mode {mode!r}")
    if family is KernelFamily.RAISED_COSINE and mode == "ceil":
        n = C.c_int()
        _lib.check(_lib.load().sbf_order_threshold(float(T), float(sigma_r), C.byref(n)),
                   "order_threshold")
        return n.value
    coeff = RC_ORDER_COEFF if family is KernelFamily.RAISED_COSINE else POLY_ORDER_COEFF
    x = coeff * (T / sigma_r) ** 2
    n = math.ceil(x) if mode == "ceil" else math.floor(x + 0.5)
    return max(1, n)


def truncation_index_exact(N, epsilon) -> int:
    """Exact cumulative-binomial truncation index (kernels.py:131-149)."""
    _check_order_and_tolerance(N, epsilon)
    m = C.c_int()
    _lib.check(_lib.load().sbf_truncation_index_exact(int(N), float(epsilon), C.byref(m)),
               "truncation_index_exact")
    return m.value


def truncation_index_chernoff(N, epsilon) -> int:
    """Closed-form tail-bound truncation index (kernels.py:152-163)."""
    _check_order_and_tolerance(N, epsilon)
    if epsilon == 0:
        raise InvalidParameterError(
            "epsilon must be positive for the tail-bound rule; use M=0 for epsilon=0")
    m = C.c_int()
    _lib.check(_lib.load().sbf_truncation_index_chernoff(
        int(N), float(epsilon), math.log(2.0 / epsilon), C.byref(m)), "truncation_index_chernoff")
    return m.value


def log_2_over_eps(epsilon) -> float:
    """libm log(2/eps), bit-identical to what the reference evaluates."""
    return math.log(2.0 / epsilon) if epsilon > 0 else 0.0


def select_plan(T, sigma_r, epsilon, family=KernelFamily.RAISED_COSINE,
                truncation="auto") -> KernelPlan:
    """Order and truncation for a Gaussian of width sigma_r (kernels.py:166-195)."""
    if not 0 <= epsilon < 1:
        raise InvalidParameterError("epsilon must lie in [0, 1)")
    if truncation not in _lib.RULES:
        raise InvalidParameterError(f"unknown truncation rule {truncation!r}")
    if family is KernelFamily.POLYNOMIAL:
        N = order_threshold(T, sigma_r, family)
        return KernelPlan(family=family, sigma_r=float(sigma_r), T=float(T), N=N, M=0,
                          epsilon=float(epsilon))
    if sigma_r <= 0:
        raise InvalidParameterError("sigma_r must be positive")
    if T < 0:
        raise InvalidParameterError("T must be non-negative")
    p = _lib.SbfPlan()
    _lib.check(_lib.load().sbf_select_plan(float(T), float(sigma_r), float(epsilon),
                                           _lib.RULES[truncation], log_2_over_eps(epsilon),
                                           C.byref(p)), "select_plan")
    return KernelPlan(family=family, sigma_r=float(sigma_r), T=float(T), N=p.N, M=p.M,
                      epsilon=float(epsilon))


def binomial_weights(N, lo, hi) -> np.ndarray:
    """C(N, n)/2^N for n in [lo, hi], correctly rounded to float64.

    Same contract as reference kernels.py:198-212; computed by the library's
    host twin (sbf_binomial_weights: exact multi-limb integers, round half to
    even, subnormals included)."""
    if not (isinstance(N, (int, np.integer)) and 0 <= lo <= hi <= N):
        raise InvalidParameterError("need 0 <= lo <= hi <= N")
    out = np.empty(int(hi) - int(lo) + 1, dtype=np.float64)
    _lib.check(_lib.load().sbf_binomial_weights(int(N), int(lo), int(hi), out.ctypes.data),
               "binomial_weights")
    return out


def raised_cosine_expansion(plan: KernelPlan) -> Expansion:
    """Retained terms n in [M, N-M]: weight C(N,n)/2^N, frequency
    (2n - N)/(sqrt(N) sigma_r) (reference kernels.py:215-227)."""
    if plan.family is not KernelFamily.RAISED_COSINE:
        raise InvalidParameterError("expansion defined for the raised-cosine family")
    idx = np.arange(plan.M, plan.N - plan.M + 1)
    # omega_n = (2n - N) / (sqrt(N) sigma_r): one correctly rounded division
    # per term, bit-equal to the reference's frequencies
    denom = math.sqrt(plan.N) * plan.sigma_r
    return Expansion(plan=plan, weights=binomial_weights(plan.N, plan.M, plan.N - plan.M),
                     frequencies=(2 * idx - plan.N) / denom, indices=idx)


def _as_result(values, like):
    return float(values) if np.ndim(like) == 0 else values


def eval_truncated_kernel(expansion: Expansion, s):
    """The truncated expansion sum_n d_n cos(w_n s) at s (scalar or array)."""
    s_arr = np.asarray(s, dtype=np.float64)
    total = np.zeros_like(s_arr)
    for wk, fk in zip(expansion.weights, expansion.frequencies):
        total += wk * np.cos(fk * s_arr)
    return _as_result(total, s)


def eval_gaussian(s, sigma_r):
    """The target range kernel exp(-(s/sigma_r)^2 / 2) (reference kernels.py:237-243)."""
    if not sigma_r > 0:
        raise InvalidParameterError("sigma_r must be positive")
    s_arr = np.asarray(s, dtype=np.float64)
    return _as_result(np.exp(-0.5 * np.square(s_arr / sigma_r)), s)


def polynomial_unsupported(*_a, **_k):
    raise UnsupportedOrderError("the polynomial family is not supported by the CUDA path")


def polynomial_shift_coefficients(plan, tau):
    """kernels.py:272-276 — polynomial family, outside the CUDA path."""
    polynomial_unsupported()
