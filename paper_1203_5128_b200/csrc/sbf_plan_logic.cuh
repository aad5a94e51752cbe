// Kernel-plan selection shared by the host ABI (sbf_select_plan) and the
// device kernel K2 (sbf_plan_device).  One source, two compilations: the CPU
// tests exercise exactly the arithmetic the GPU runs.
//
// Restates reference kernels.py:109-227 (order_threshold, truncation rules,
// select_plan, binomial weights, raised-cosine frequencies).
#pragma once

#include <math.h>
#include <stdint.h>

#include "../../include/sbf.h"

#ifdef __CUDACC__
#define SBF_HD __host__ __device__
#else
#define SBF_HD
#endif

namespace sbf {

// kernels.py:31
constexpr double kOrderCoeff = 0.405;
// largest order the plan supports (int32 index space, term table sizes)
constexpr double kMaxOrder = 1.0e8;
// multi-limb exact path capacity (bits of C(N, m) plus the epsilon shift)
constexpr int kLimbs = 224;  // 32-bit limbs -> 7168 bits
constexpr int kExactMaxN = 4096;

SBF_HD inline double next_up(double x) { return nextafter(x, INFINITY); }
SBF_HD inline double next_down(double x) { return nextafter(x, -INFINITY); }

// N = max(1, ceil(0.405 (T / sigma_r)^2))  (kernels.py:109-128, "ceil" mode).
// CPython evaluates `(T / sigma_r) ** 2` with libm pow(); glibc's pow is not
// correctly rounded, so on the host we call pow() exactly like CPython and on
// the device we use q*q and flag the rare inputs where a 2-ulp change of q^2
// moves the ceiling (SBF_PLAN_N_AMBIGUOUS).
SBF_HD inline int order_threshold(double T, double sigma_r, int* flags, int* status) {
  double q = T / sigma_r;
#ifdef __CUDA_ARCH__
  double q2 = q * q;
  double lo = kOrderCoeff * next_down(next_down(q2));
  double hi = kOrderCoeff * next_up(next_up(q2));
  if (ceil(lo) != ceil(hi)) *flags |= SBF_PLAN_N_AMBIGUOUS;
#else
  // a runtime exponent: compilers fold pow(q, 2.0) into q*q, CPython does not
  volatile double two = 2.0;
  double q2 = pow(q, two);
#endif
  double x = kOrderCoeff * q2;
  if (!(x <= kMaxOrder)) {
    *status = SBF_ERR_UNSUPPORTED;
    return 1;
  }
  int n = (int)ceil(x);
  return n < 1 ? 1 : n;
}

// ---------------------------------------------------------------------------
// exact truncation rule (kernels.py:131-149) — multi-limb integers.
// smallest m in [0, (N-1)//2] with sum_{n<=m+1} C(N,n) > Fraction(eps)/2 * 2^N
// ---------------------------------------------------------------------------
struct BigNat {
  uint32_t w[kLimbs];
  int n;  // used limbs
};

SBF_HD inline void big_set_small(BigNat& a, uint64_t v) {
  a.n = 0;
  while (v) {
    a.w[a.n++] = (uint32_t)v;
    v >>= 32;
  }
}
SBF_HD inline void big_mul_small(BigNat& a, uint32_t m) {
  uint64_t carry = 0;
  for (int i = 0; i < a.n; ++i) {
    uint64_t t = (uint64_t)a.w[i] * m + carry;
    a.w[i] = (uint32_t)t;
    carry = t >> 32;
  }
  if (carry) a.w[a.n++] = (uint32_t)carry;
}
SBF_HD inline void big_div_small(BigNat& a, uint32_t d) {  // exact division
  uint64_t rem = 0;
  for (int i = a.n - 1; i >= 0; --i) {
    uint64_t cur = (rem << 32) | a.w[i];
    a.w[i] = (uint32_t)(cur / d);
    rem = cur % d;
  }
  while (a.n && a.w[a.n - 1] == 0) --a.n;
}
SBF_HD inline void big_add(BigNat& out, const BigNat& a, const BigNat& b) {
  int n = a.n > b.n ? a.n : b.n;
  uint64_t carry = 0;
  for (int i = 0; i < n; ++i) {
    uint64_t t = carry + (i < a.n ? a.w[i] : 0u) + (i < b.n ? b.w[i] : 0u);
    out.w[i] = (uint32_t)t;
    carry = t >> 32;
  }
  out.n = n;
  if (carry) out.w[out.n++] = (uint32_t)carry;
}
// compare a * 2^sa with b * 2^sb  (-1, 0, 1)
SBF_HD inline int big_cmp_shifted(const BigNat& a, int sa, const BigNat& b, int sb) {
  // bit lengths
  auto bitlen = [](const BigNat& x) -> int {
    if (x.n == 0) return 0;
    uint32_t top = x.w[x.n - 1];
    int l = 0;
    while (top) {
      ++l;
      top >>= 1;
    }
    return (x.n - 1) * 32 + l;
  };
  int la = bitlen(a), lb = bitlen(b);
  if (la == 0 || lb == 0) return (la > 0) - (lb > 0);
  int ea = la + sa, eb = lb + sb;
  if (ea != eb) return ea > eb ? 1 : -1;
  // same top bit position: compare bit by bit from the top
  int total = ea;
  for (int k = total - 1; k >= 0; --k) {
    int ka = k - sa, kb = k - sb;
    int bit_a = (ka >= 0 && ka < la) ? (int)((a.w[ka >> 5] >> (ka & 31)) & 1u) : 0;
    int bit_b = (kb >= 0 && kb < lb) ? (int)((b.w[kb >> 5] >> (kb & 31)) & 1u) : 0;
    if (bit_a != bit_b) return bit_a > bit_b ? 1 : -1;
  }
  return 0;
}

SBF_HD inline int truncation_exact_bigint(int N, double eps, int* status) {
  if (N > kExactMaxN) {
    *status = SBF_ERR_UNSUPPORTED;
    return 0;
  }
  // eps = mant * 2^e exactly (53-bit integer mantissa)
  int ex;
  double fr = frexp(eps, &ex);
  uint64_t mant = (uint64_t)ldexp(fr, 53);
  int e = ex - 53;
  // threshold = mant * 2^(N + e - 1)
  int k = N + e - 1;
  BigNat thr, c, cum, s;
  big_set_small(thr, mant);
  big_set_small(c, 1);
  big_set_small(cum, 1);
  int sa = k < 0 ? -k : 0, sb = k > 0 ? k : 0;
  for (int m = 0; m <= (N - 1) / 2; ++m) {
    big_mul_small(c, (uint32_t)(N - m));
    big_div_small(c, (uint32_t)(m + 1));
    big_add(s, cum, c);
    if (big_cmp_shifted(s, sa, thr, sb) > 0) return m;
    cum = s;
  }
  *status = SBF_ERR_INVALID;  // unreachable for eps < 1
  return 0;
}

// fp64 evaluation with an ambiguity guard; exact path when it cannot decide.
SBF_HD inline int truncation_index_exact(int N, double eps, int* flags, int* status,
                                         bool force_exact = false) {
  if (eps == 0.0) return 0;
  if (force_exact) {
    *flags |= SBF_PLAN_EXACT_BIGINT;
    return truncation_exact_bigint(N, eps, status);
  }
  double c = 1.0, cum = 1.0;
  int E = 0;  // c, cum scaled by 2^-E
  const double half_eps = eps * 0.5;
  for (int m = 0; m <= (N - 1) / 2; ++m) {
    c = c * (double)(N - m) / (double)(m + 1);
    double s = cum + c;
    int pw = N - E;
    if (pw <= 1000) {
      double thr = ldexp(half_eps, pw);
      double rel = (s - thr) / thr;
      if (fabs(rel) < 1e-9) {
        *flags |= SBF_PLAN_EXACT_BIGINT;
        return truncation_exact_bigint(N, eps, status);
      }
      if (s > thr) return m;
    }
    cum = s;
    if (c > 0x1p900) {
      c *= 0x1p-900;
      cum *= 0x1p-900;
      E += 900;
    }
  }
  *status = SBF_ERR_INVALID;
  return 0;
}

// kernels.py:152-163; log(2/eps) is supplied by the caller (libm on the host,
// identical bits to CPython's math.log), sqrt/division are IEEE exact.
SBF_HD inline int truncation_index_chernoff(int N, double eps, double log_2_over_eps,
                                            int* status) {
  if (!(eps > 0.0)) {
    *status = SBF_ERR_INVALID;
    return 0;
  }
  double raw = floor(((double)N - sqrt(4.0 * (double)N * log_2_over_eps)) / 2.0);
  int lim = (N - 1) / 2;
  if (raw > (double)lim) return lim;
  if (raw < 0.0) return 0;
  return (int)raw;
}

// kernels.py:166-195
SBF_HD inline void select_plan(double T, double sigma_r, double eps, int rule,
                               double log_2_over_eps, sbf_plan* p,
                               bool force_exact = false) {
  p->T = T;
  p->sigma_r = sigma_r;
  p->epsilon = eps;
  p->flags = 0;
  p->status = SBF_OK;
  p->pad0 = p->pad1 = 0;
  if (!(sigma_r > 0.0) || !(T >= 0.0) || !(eps >= 0.0 && eps < 1.0) || rule < 0 || rule > 3) {
    p->status = SBF_ERR_INVALID;
    p->N = 1;
    p->M = 0;
    p->K = 1;
    p->K_eval = 0;
    p->gamma = 0.0;
    return;
  }
  int N = order_threshold(T, sigma_r, &p->flags, &p->status);
  int M = 0;
  if (eps == 0.0 || rule == SBF_RULE_NONE) {
    M = 0;
  } else if (rule == SBF_RULE_AUTO) {
    if (sigma_r > 40.0)
      M = 0;
    else if (sigma_r > 10.0)
      M = truncation_index_exact(N, eps, &p->flags, &p->status, force_exact);
    else
      M = truncation_index_chernoff(N, eps, log_2_over_eps, &p->status);
  } else if (rule == SBF_RULE_EXACT) {
    M = truncation_index_exact(N, eps, &p->flags, &p->status, force_exact);
  } else {
    M = truncation_index_chernoff(N, eps, log_2_over_eps, &p->status);
  }
  int lim = (N - 1) / 2;
  if (M > lim) M = lim;
  p->N = N;
  p->M = M;
  p->K = N / 2 - M + 1;
  p->K_eval = p->K;
  p->gamma = 1.0 / (sqrt((double)N) * sigma_r);
}

// spatial.py:81-100
SBF_HD inline void extended_box_params(double sigma_s, int passes, int* r, double* alpha) {
  double v = sigma_s * sigma_s / passes;
  int rr = (int)floor(sqrt(3.0 * v + 0.25) - 0.5);
  double second = rr * (rr + 1) * (2 * rr + 1) / 3.0;
  *r = rr;
  *alpha = (v * (2 * rr + 1) - second) / (2.0 * (double)(rr + 1) * (double)(rr + 1) - 2.0 * v);
}

}  // namespace sbf
