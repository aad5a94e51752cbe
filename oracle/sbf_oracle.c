/* CPU oracle, C half — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C float64 restatement of the reference's hot path (package
 * `shiftbf`, paths relative to pkg/src/shiftbf/).  It serves the tests and
 * bench.py's `cpu_baseline` / `--impl reference` legs as the checker and the
 * timed CPU implementation; the product (paper_1203_5128_b200) never links it.
 * The plan (T -> N, M, weights, frequencies) comes from the numpy oracle
 * (oracle/shiftbf_oracle.py); this file restates the per-pixel work:
 *
 *   running_max_lines    _core/_fastcore.pyx:16-58  (windowed max, clamped)
 *   max_filter_2d        maxfilter.py:41-49         (rows, then columns)
 *   window_sum_lines     _core/_fastcore.pyx:61-86  (clamped running sum)
 *   _extended_box_lines  spatial.py:120-133         (+alpha endpoints, renormalise)
 *   _extended_box_2d     spatial.py:136-139         (rows, then columns)
 *   box_filter           spatial.py:65-78           (2-D sums / outer(counts))
 *   _accumulate_cosine_terms  bilateral.py:140-164
 *   _divide_with_fallback     bilateral.py:242-254
 *
 * Column passes run as running sums over whole rows (cache friendly) with the
 * same per-element order of additions as the reference's transposed line
 * pass, so results agree with the reference to the last few ulps.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- windowed running maximum along contiguous lines (_fastcore.pyx:16-58) ---- */
static void max_lines(const double* src, int64_t m, int64_t n, int64_t R, double* out) {
  if (R == 0) {
    memcpy(out, src, (size_t)(m * n) * sizeof(double));
    return;
  }
  const int64_t w = 2 * R + 1;
  const int64_t padded = ((n + 2 * R + w - 1) / w) * w;
  double* q = malloc((size_t)padded * 3 * sizeof(double));
  double* lm = q + padded;
  double* rm = lm + padded;
  for (int64_t i = 0; i < m; ++i) {
    const double* s = src + i * n;
    for (int64_t j = 0; j < padded; ++j) {
      int64_t k = j - R;
      k = k < 0 ? 0 : (k >= n ? n - 1 : k);
      q[j] = s[k];
    }
    for (int64_t j = 0; j < padded; ++j)
      lm[j] = (j % w == 0) ? q[j] : (lm[j - 1] > q[j] ? lm[j - 1] : q[j]);
    for (int64_t j = padded - 1; j >= 0; --j)
      rm[j] = (j % w == w - 1) ? q[j] : (rm[j + 1] > q[j] ? rm[j + 1] : q[j]);
    for (int64_t j = 0; j < n; ++j) {
      const double a = rm[j], b = lm[j + 2 * R];
      out[i * n + j] = a > b ? a : b;
    }
  }
  free(q);
}

static void transpose(const double* a, int64_t m, int64_t n, double* t) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) t[j * m + i] = a[i * n + j];
}

/* maxfilter.py:41-49 */
int oracle_max_filter_2d(const double* f, int64_t H, int64_t W, int64_t R, double* out) {
  if (H < 1 || W < 1 || R < 0) return 2;
  double* a = malloc((size_t)(H * W) * sizeof(double));
  double* b = malloc((size_t)(H * W) * sizeof(double));
  max_lines(f, H, W, R, a);
  transpose(a, H, W, b);
  max_lines(b, W, H, R, a);
  transpose(a, W, H, out);
  free(a);
  free(b);
  return 0;
}

/* maxfilter.py:56-61: T = max(M - f), 0 for R = 0 */
double oracle_compute_T(const double* f, int64_t H, int64_t W, int64_t R) {
  if (R == 0) return 0.0;
  double* M = malloc((size_t)(H * W) * sizeof(double));
  oracle_max_filter_2d(f, H, W, R, M);
  double T = -INFINITY;
  for (int64_t i = 0; i < H * W; ++i) {
    const double d = M[i] - f[i];
    if (d > T) T = d;
  }
  free(M);
  return T;
}

/* clamped window count (spatial.py:60-62) */
static inline double wcount(int64_t i, int64_t n, int64_t r) {
  const int64_t hi = i + r < n - 1 ? i + r : n - 1;
  const int64_t lo = i - r > 0 ? i - r : 0;
  return (double)(hi - lo) + 1.0;
}

/* window_sum_lines (_fastcore.pyx:61-86) on one contiguous line */
static void window_sum_line(const double* s, int64_t n, int64_t r, double* out) {
  double acc = 0.0;
  const int64_t hi0 = r < n - 1 ? r : n - 1;
  for (int64_t j = 0; j <= hi0; ++j) acc += s[j];
  out[0] = acc;
  for (int64_t j = 1; j < n; ++j) {
    if (j + r < n) acc += s[j + r];
    if (j - r - 1 >= 0) acc -= s[j - r - 1];
    out[j] = acc;
  }
}

/* the same window sums down the columns of an (m, n) image, rows at a time */
static void window_sum_cols(const double* a, int64_t m, int64_t n, int64_t r, double* out,
                            double* acc) {
  const int64_t hi0 = r < m - 1 ? r : m - 1;
  for (int64_t j = 0; j < n; ++j) acc[j] = 0.0;
  for (int64_t k = 0; k <= hi0; ++k)
    for (int64_t j = 0; j < n; ++j) acc[j] += a[k * n + j];
  memcpy(out, acc, (size_t)n * sizeof(double));
  for (int64_t i = 1; i < m; ++i) {
    if (i + r < m) {
      const double* add = a + (i + r) * n;
      for (int64_t j = 0; j < n; ++j) acc[j] += add[j];
    }
    if (i - r - 1 >= 0) {
      const double* sub = a + (i - r - 1) * n;
      for (int64_t j = 0; j < n; ++j) acc[j] -= sub[j];
    }
    memcpy(out + i * n, acc, (size_t)n * sizeof(double));
  }
}

/* _extended_box_lines along rows (spatial.py:120-133) */
static void ext_box_rows(const double* a, int64_t m, int64_t n, int64_t r, double alpha,
                         double* out) {
  const int64_t e = r + 1;
  for (int64_t i = 0; i < m; ++i) {
    const double* s = a + i * n;
    double* o = out + i * n;
    window_sum_line(s, n, r, o);
    for (int64_t j = 0; j < n; ++j) {
      double num = o[j], den = wcount(j, n, r);
      if (alpha > 0.0) {
        if (j + e < n) { num += alpha * s[j + e]; den += alpha; }
        if (j - e >= 0) { num += alpha * s[j - e]; den += alpha; }
      }
      o[j] = num / den;
    }
  }
}

/* _extended_box_lines down the columns (the reference transposes first) */
static void ext_box_cols(const double* a, int64_t m, int64_t n, int64_t r, double alpha,
                         double* out, double* acc) {
  const int64_t e = r + 1;
  window_sum_cols(a, m, n, r, out, acc);
  for (int64_t i = 0; i < m; ++i) {
    double* o = out + i * n;
    double den = wcount(i, m, r);
    const double* up = (alpha > 0.0 && i + e < m) ? a + (i + e) * n : NULL;
    const double* dn = (alpha > 0.0 && i - e >= 0) ? a + (i - e) * n : NULL;
    if (up) den += alpha;
    if (dn) den += alpha;
    for (int64_t j = 0; j < n; ++j) {
      double num = o[j];
      if (up) num += alpha * up[j];
      if (dn) num += alpha * dn[j];
      o[j] = num / den;
    }
  }
}

/* apply_spatial: mode 0 = iterated extended box (spatial.py:108-117),
 * mode 1 = box_filter (spatial.py:65-78).  In place; tmp holds H*W + W. */
static void smooth(double* img, int64_t H, int64_t W, int mode, int64_t r, double alpha,
                   int passes, double* tmp) {
  double* t = tmp;
  double* acc = tmp + H * W;
  if (mode == 1) {
    if (r == 0) return;
    for (int64_t i = 0; i < H; ++i) window_sum_line(img + i * W, W, r, t + i * W);
    window_sum_cols(t, H, W, r, img, acc);
    for (int64_t i = 0; i < H; ++i) {
      const double ci = wcount(i, H, r);
      for (int64_t j = 0; j < W; ++j) img[i * W + j] /= ci * wcount(j, W, r);
    }
    return;
  }
  for (int p = 0; p < passes; ++p) {
    ext_box_rows(img, H, W, r, alpha, t);
    ext_box_cols(t, H, W, r, alpha, img, acc);
  }
}

/* _accumulate_cosine_terms (bilateral.py:140-164) over K folded terms:
 * scale[k] already includes the factor 2 of a +- pair. */
int oracle_accumulate(const double* f, int64_t H, int64_t W, const double* scale,
                      const double* freq, int K, int mode, int64_t r, double alpha, int passes,
                      double* num, double* den) {
  if (H < 1 || W < 1 || K < 0 || r < 0 || passes < 1) return 2;
  const int64_t n = H * W;
  double* buf = malloc((size_t)(6 * n + n + W) * sizeof(double));
  if (!buf) return 5;
  double *gc = buf, *gs = gc + n, *fc = gs + n, *fs = fc + n, *gcb = fs + n, *gsb = gcb + n;
  double* tmp = gsb + n;
  memset(num, 0, (size_t)n * sizeof(double));
  memset(den, 0, (size_t)n * sizeof(double));
  for (int k = 0; k < K; ++k) {
    const double w = freq[k];
    for (int64_t i = 0; i < n; ++i) {
      const double th = w * f[i];
      gc[i] = cos(th);
      gs[i] = sin(th);
      fc[i] = f[i] * gc[i];
      fs[i] = f[i] * gs[i];
    }
    memcpy(gcb, gc, (size_t)n * sizeof(double));
    memcpy(gsb, gs, (size_t)n * sizeof(double));
    smooth(fc, H, W, mode, r, alpha, passes, tmp);
    smooth(fs, H, W, mode, r, alpha, passes, tmp);
    smooth(gcb, H, W, mode, r, alpha, passes, tmp);
    smooth(gsb, H, W, mode, r, alpha, passes, tmp);
    const double s = scale[k];
    for (int64_t i = 0; i < n; ++i) {
      num[i] += s * (gc[i] * fc[i] + gs[i] * fs[i]);
      den[i] += s * (gc[i] * gcb[i] + gs[i] * gsb[i]);
    }
  }
  free(buf);
  return 0;
}

/* _divide_with_fallback (bilateral.py:242-254); returns the fallback count */
int64_t oracle_divide(const double* num, const double* den, const double* f, int64_t n,
                      double* out) {
  int64_t bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (den[i] > 0.0) {
      out[i] = num[i] / den[i];
    } else {
      out[i] = f[i];
      ++bad;
    }
  }
  return bad;
}
