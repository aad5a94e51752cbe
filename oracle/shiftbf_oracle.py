"""CPU oracle for the shiftable bilateral-filter hot path — TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference package
`shiftbf` (arXiv 1203.5128 implementation, mounted read-only at
/root/reference/pkg during development).  It is the *checker*: only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it.  The product package
(`paper_1203_5128_b200`) never imports anything from `oracle/`; its compute
path is CUDA only and fails loudly when the extension is missing.

Parity pin: every function below is checked against golden vectors produced
by the reference itself (`tests/golden/make_golden.py`, fixtures in
`tests/golden/*.npz`) in `tests/test_oracle_golden.py`.

Each function cites the reference file:line it restates (paths relative to
`/root/reference/pkg/src/shiftbf/`).
"""

from __future__ import annotations

import itertools
import math
from fractions import Fraction

import numpy as np

# kernels.py:31 — 3-digit order coefficient used by the published table.
RC_ORDER_COEFF = 0.405


class OracleError(ValueError):
    """Raised where the reference raises InvalidParameterError."""


# --------------------------------------------------------------------------
# image validation (image.py:11-20)
# --------------------------------------------------------------------------
def as_image(a) -> np.ndarray:
    x = np.asarray(a, dtype=np.float64)
    if x.ndim != 2 or x.size == 0 or not np.isfinite(x).all():
        raise OracleError("image must be 2-D, non-empty and finite")
    return np.ascontiguousarray(x)


# --------------------------------------------------------------------------
# windowed maximum / local range (maxfilter.py:21-61, _purecore.py:13-35)
# --------------------------------------------------------------------------
def _clamped_max_along(a: np.ndarray, radius: int, axis: int) -> np.ndarray:
    """max over the clamped window [i-R, i+R] along `axis`.

    Restates `_core.running_max_lines` (_fastcore.pyx:16-58): replicate
    padding makes every window full width; the partitioned left/right
    running maxima (van Herk / Gil-Werman) give each window as the max of
    one suffix and one prefix.
    """
    if radius == 0:
        return a.copy()
    a = np.moveaxis(a, axis, -1)
    n = a.shape[-1]
    w = 2 * radius + 1
    nblk = -(-(n + 2 * radius) // w)
    src = np.clip(np.arange(nblk * w) - radius, 0, n - 1)
    blocks = a[..., src].reshape(a.shape[:-1] + (nblk, w))
    prefix = np.maximum.accumulate(blocks, axis=-1).reshape(a.shape[:-1] + (nblk * w,))
    suffix = np.flip(np.maximum.accumulate(np.flip(blocks, -1), axis=-1), -1)
    suffix = suffix.reshape(a.shape[:-1] + (nblk * w,))
    out = np.maximum(suffix[..., :n], prefix[..., 2 * radius:2 * radius + n])
    return np.moveaxis(out, -1, axis)


def max_filter_1d(seq, radius) -> np.ndarray:
    """maxfilter.py:21-28."""
    s = np.asarray(seq, dtype=np.float64)
    if s.ndim != 1 or s.size == 0 or radius < 0:
        raise OracleError("bad max_filter_1d arguments")
    return _clamped_max_along(s, int(radius), 0)


def max_filter_2d(img, radius) -> np.ndarray:
    """maxfilter.py:41-49 — row pass, then column pass."""
    f = as_image(img)
    if radius < 0:
        raise OracleError("radius must be >= 0")
    rows = _clamped_max_along(f, int(radius), 1)
    return np.ascontiguousarray(_clamped_max_along(rows, int(radius), 0))


def compute_T(img, radius) -> float:
    """maxfilter.py:56-61 — T = max(M - f) in float64; 0.0 for R = 0."""
    f = as_image(img)
    if radius == 0:
        return 0.0
    return float(np.max(max_filter_2d(f, radius) - f))


def brute_force_T(img, radius) -> float:
    """maxfilter.py:64-82 — O(R^2) check of compute_T."""
    f = as_image(img)
    h, w = f.shape
    best = 0.0
    for dy in range(-radius, radius + 1):
        for dx in range(-radius, radius + 1):
            y0, y1 = max(0, -dy), min(h, h - dy)
            x0, x1 = max(0, -dx), min(w, w - dx)
            if y0 >= y1 or x0 >= x1:
                continue
            d = np.abs(f[y0 + dy:y1 + dy, x0 + dx:x1 + dx] - f[y0:y1, x0:x1])
            best = max(best, float(d.max()))
    return best


# --------------------------------------------------------------------------
# kernel plan (kernels.py:109-227)
# --------------------------------------------------------------------------
def order_threshold(T, sigma_r) -> int:
    """kernels.py:109-128, raised-cosine family, ceil mode.

    CPython `x ** 2` on floats is libm pow(x, 2.0); kept verbatim in meaning.
    """
    if sigma_r <= 0 or T < 0:
        raise OracleError("bad order_threshold arguments")
    return max(1, math.ceil(RC_ORDER_COEFF * (T / sigma_r) ** 2))


def truncation_index_exact(N, epsilon) -> int:
    """kernels.py:131-149 — exact rational cumulative binomial rule.

    Smallest M with sum_{n<=M+1} C(N, n) > (epsilon/2) 2^N, searched over
    M in [0, (N-1)//2]; epsilon is taken as its exact binary rational.
    """
    if N < 1 or not 0 <= epsilon < 1:
        raise OracleError("bad truncation arguments")
    if epsilon == 0:
        return 0
    limit = Fraction(epsilon) * (1 << N) / 2
    total = 1                     # C(N, 0)
    binom = 1
    for m in range((N - 1) // 2 + 1):
        binom = binom * (N - m) // (m + 1)   # C(N, m+1)
        if total + binom > limit:
            return m
        total += binom
    raise AssertionError("cumulative mass must pass 1/2")


def truncation_index_chernoff(N, epsilon) -> int:
    """kernels.py:152-163 — closed-form tail bound."""
    if N < 1 or not 0 < epsilon < 1:
        raise OracleError("bad chernoff arguments")
    raw = math.floor((N - math.sqrt(4.0 * N * math.log(2.0 / epsilon))) / 2.0)
    return max(0, min(raw, (N - 1) // 2))


def select_plan(T, sigma_r, epsilon, truncation="auto"):
    """kernels.py:166-195 — returns (T, N, M) for the raised-cosine family."""
    if not 0 <= epsilon < 1:
        raise OracleError("epsilon must lie in [0, 1)")
    N = order_threshold(T, sigma_r)
    if epsilon == 0 or truncation == "none":
        M = 0
    elif truncation == "auto":
        if sigma_r > 40:
            M = 0
        elif sigma_r > 10:
            M = truncation_index_exact(N, epsilon)
        else:
            M = truncation_index_chernoff(N, epsilon)
    elif truncation == "exact":
        M = truncation_index_exact(N, epsilon)
    elif truncation == "chernoff":
        M = truncation_index_chernoff(N, epsilon)
    else:
        raise OracleError(f"unknown truncation rule {truncation!r}")
    M = min(M, (N - 1) // 2)
    return float(T), N, M


def binomial_weights(N, lo, hi) -> np.ndarray:
    """kernels.py:198-212 — C(N, n)/2^N correctly rounded (exact ints)."""
    return np.array([math.comb(N, n) / (1 << N) for n in range(lo, hi + 1)],
                    dtype=np.float64)


def raised_cosine_terms(N, M, sigma_r):
    """kernels.py:215-227 — (indices, weights, frequencies) for n in [M, N-M]."""
    n = np.arange(M, N - M + 1)
    w = binomial_weights(N, M, N - M)
    freq = (2 * n - N) / (math.sqrt(N) * sigma_r)
    return n, w, freq


def folded_terms(N, M, sigma_r):
    """bilateral.py:150-154 — folded +/- pairs: (index, scale, frequency)."""
    n, w, freq = raised_cosine_terms(N, M, sigma_r)
    keep = 2 * n <= N
    scale = np.where(2 * n[keep] == N, w[keep], 2.0 * w[keep])
    return n[keep], scale, freq[keep]


# --------------------------------------------------------------------------
# spatial smoothing (spatial.py:60-139, 175-194)
# --------------------------------------------------------------------------
def extended_box_params(sigma_s, passes):
    """spatial.py:81-100."""
    v = sigma_s * sigma_s / passes
    r = int(math.floor(math.sqrt(3.0 * v + 0.25) - 0.5))
    second = r * (r + 1) * (2 * r + 1) / 3.0
    alpha = (v * (2 * r + 1) - second) / (2.0 * (r + 1) ** 2 - 2.0 * v)
    return r, alpha


def support_radius(kind, sigma_s=None, passes=3, radius=None) -> int:
    """spatial.py:185-194 for 'box' and 'iterated'."""
    if kind == "box":
        return int(radius)
    r, alpha = extended_box_params(sigma_s, passes)
    return passes * (r + (1 if alpha > 0 else 0))


def _box_pass_along(a: np.ndarray, r: int, alpha: float, axis: int) -> np.ndarray:
    """One extended-box pass along `axis` with clamped renormalisation.

    Restates `_extended_box_lines` (spatial.py:120-133) with the window sum of
    `_core.window_sum_lines` (_purecore.py:38-53): the clamped window sum plus
    alpha times each in-bounds endpoint at distance r+1, divided by the
    clamped count plus alpha per in-bounds endpoint.
    """
    a = np.moveaxis(a, axis, -1)
    n = a.shape[-1]
    pad = np.zeros(a.shape[:-1] + (1,))
    csum = np.concatenate([pad, np.cumsum(a, axis=-1)], axis=-1)  # csum[k] = sum a[:k]
    i = np.arange(n)
    hi = np.minimum(i + r, n - 1) + 1
    lo = np.maximum(i - r, 0)
    total = csum[..., hi] - csum[..., lo]
    count = (hi - lo).astype(np.float64)
    if alpha > 0.0:
        total = total.copy()
        for step in (r + 1, -(r + 1)):
            j = i + step
            ok = (j >= 0) & (j < n)
            total[..., ok] += alpha * a[..., j[ok]]
            count[ok] += alpha
    return np.moveaxis(total / count, -1, axis)


def iterated_box(img, sigma_s, passes=3) -> np.ndarray:
    """spatial.py:108-117 / 136-139 — per pass: rows then columns."""
    out = as_image(img)
    r, alpha = extended_box_params(sigma_s, passes)
    for _ in range(passes):
        out = _box_pass_along(out, r, alpha, 1)
        out = _box_pass_along(out, r, alpha, 0)
    return out


def box_filter(img, radius) -> np.ndarray:
    """spatial.py:65-78 — clamped box mean (single pass, no endpoints)."""
    f = as_image(img)
    if radius == 0:
        return f.copy()
    return _box_pass_along(_box_pass_along(f, radius, 0.0, 1), radius, 0.0, 0)


def smooth(img, spatial):
    """spatial.py:175-182 for the two modes on the hot path.

    `spatial` is ('iterated', sigma_s, passes) or ('box', radius).
    """
    if spatial[0] == "box":
        return box_filter(img, spatial[1])
    return iterated_box(img, spatial[1], spatial[2])


# --------------------------------------------------------------------------
# the filter (bilateral.py:117-164, 242-254)
# --------------------------------------------------------------------------
def divide_with_fallback(num, den, fallback):
    """bilateral.py:242-254 — returns (out, n_bad); NaN den counts as bad."""
    bad = ~(den > 0.0)
    n_bad = int(np.count_nonzero(bad))
    out = num / np.where(bad, 1.0, den)
    out[bad] = fallback[bad]
    return out, n_bad


def shiftable_bf(img, sigma_s, sigma_r, epsilon=0.0, spatial=None,
                 window_radius=None, fixed_T=None, truncation="auto"):
    """bilateral.py:117-164 — returns dict(image, T, N, M, fallback_pixels)."""
    f = as_image(img)
    if spatial is None:
        spatial = ("iterated", float(sigma_s), 3)
    if window_radius is not None:
        radius = int(window_radius)
    elif spatial[0] == "box":
        radius = max(1, int(spatial[1]))
    else:
        radius = max(1, support_radius("iterated", spatial[1], spatial[2]))
    T = float(fixed_T) if fixed_T is not None else compute_T(f, radius)
    T, N, M = select_plan(T, sigma_r, epsilon, truncation)
    num = np.zeros_like(f)
    den = np.zeros_like(f)
    for _, scale, freq in zip(*folded_terms(N, M, sigma_r)):
        theta = freq * f
        c, s = np.cos(theta), np.sin(theta)
        fc = smooth(f * c, spatial)
        fs = smooth(f * s, spatial)
        gc = smooth(c, spatial)
        gs = smooth(s, spatial)
        num += scale * (c * fc + s * fs)
        den += scale * (c * gc + s * gs)
    out, n_bad = divide_with_fallback(num, den, f)
    return dict(image=out, T=T, N=N, M=M, fallback_pixels=n_bad)


def direct_bf(img, spatial, sigma_r, radius=None):
    """bilateral.py:205-239 with gaussian_range (:88-99) and the window weights
    of spatial.py:155-157 / 197-213.  `spatial` is ('box', r) or
    ('fir', sigma_s, r)."""
    f = as_image(img)
    if radius is None:
        radius = spatial[1] if spatial[0] == "box" else spatial[2]
    R = int(radius)
    if spatial[0] == "box":
        taps = np.ones(2 * R + 1)
    else:
        k = np.arange(-R, R + 1, dtype=np.float64)
        taps = np.exp(-(k * k) / (2.0 * spatial[1] * spatial[1]))
    weights = np.outer(taps, taps)
    inv = 1.0 / (2.0 * sigma_r * sigma_r)
    h, w = f.shape
    num = np.zeros_like(f)
    den = np.zeros_like(f)
    for dy in range(-R, R + 1):
        if abs(dy) >= h:
            continue
        ys, yd = slice(max(0, dy), h + min(0, dy)), slice(max(0, -dy), h - max(0, dy))
        for dx in range(-R, R + 1):
            wsp = weights[dy + R, dx + R]
            if wsp == 0.0 or abs(dx) >= w:
                continue
            xs, xd = slice(max(0, dx), w + min(0, dx)), slice(max(0, -dx), w - max(0, dx))
            nb = f[ys, xs]
            d = nb - f[yd, xd]
            wr = wsp * np.exp(-(d * d) * inv)
            num[yd, xd] += wr * nb
            den[yd, xd] += wr
    out, _ = divide_with_fallback(num, den, f)
    return out


def _shifted_copy(f, offset):
    """nlm.py:68-75 — f(x + u) with replicate padding."""
    h, w = f.shape
    rows = np.clip(np.arange(h) + offset[0], 0, h - 1)
    cols = np.clip(np.arange(w) + offset[1], 0, w - 1)
    return f[np.ix_(rows, cols)]


def coarse_nlm(img, offsets, sigmas, spatial, radius, epsilon, truncation="auto"):
    """nlm.py:78-137 (unfolded tensor product over all 2^p masks, as the
    reference); budgets are checked by the caller.  `spatial` as in smooth().
    Returns dict(image, T, plans=[(N, M)], fallback_pixels)."""
    f = as_image(img)
    R = int(radius) + max(max(abs(dy), abs(dx)) for dy, dx in offsets)
    T = compute_T(f, R)
    plans = [select_plan(T, s, epsilon, truncation) for s in sigmas]
    comps = []
    for (T_, N, M), sg, off in zip(plans, sigmas, offsets):
        n, w, fr = raised_cosine_terms(N, M, sg)
        fj = f if tuple(off) == (0, 0) else _shifted_copy(f, off)
        comps.append([(wi, np.cos(om * fj), np.sin(om * fj)) for wi, om in zip(w, fr)])
    p = len(offsets)
    num = np.zeros_like(f)
    den = np.zeros_like(f)
    for combo in itertools.product(*comps):
        weight = 1.0
        for wi, _, _ in combo:
            weight *= wi
        cn = np.zeros_like(f)
        cd = np.zeros_like(f)
        for mask in range(1 << p):
            aux = np.ones_like(f)
            for j, (_, c, s_) in enumerate(combo):
                aux = aux * (s_ if (mask >> j) & 1 else c)
            cn += aux * smooth(f * aux, spatial)
            cd += aux * smooth(aux, spatial)
        num += weight * cn
        den += weight * cd
    out, n_bad = divide_with_fallback(num, den, f)
    return dict(image=out, T=T, plans=[(N, M) for _, N, M in plans], fallback_pixels=n_bad)


def metrics(a, b):
    """metrics.py:19-28 — (mse, mse_db, max_abs)."""
    d = as_image(a) - as_image(b)
    mse = float(np.mean(d * d))
    return mse, (10.0 * math.log10(mse) if mse > 0 else float("-inf")), float(np.abs(d).max())
