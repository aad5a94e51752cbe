// K2 — kernel plan on the device (reference kernels.py:166-227).
//
// One warp reads T from device memory (written by K1, no host round trip);
// lane 0 selects (N, M) with the same rules as the reference (shared source
// with the host ABI, sbf_plan_logic.cuh) and the warp writes the folded term
// table: for
// n = floor(N/2) down to M, scale = d_n (2 d_n for a +-pair) and
// omega_n = (2n - N) / (sqrt(N) sigma_r).  d_n = C(N,n)/2^N is evaluated by
// the centre-outward ratio recurrence (warp prefix products) normalised by
// the full binomial sum (relative error ~1e-14; weights need not be
// bit-exact, only the index set).  Exact-zero weights (float64 underflow in the reference too) are
// skipped: they contribute nothing, so skipping is arithmetic-identical.
#include <cmath>
#include <vector>

#include "sbf_common.cuh"
#include "sbf_plan_logic.cuh"
#include "sbf_plan_warp.cuh"

namespace sbf {
namespace {

__global__ void plan_kernel(const double* __restrict__ T_dev, int use_fixed, double fixed_T,
                            double sigma_r, double eps, int rule, double log_2_over_eps,
                            sbf_plan* __restrict__ plan_out, sbf_term* __restrict__ terms,
                            int cap, int forced_N, int forced_M) {
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  __shared__ sbf_plan sp;
  plan_warp(use_fixed ? fixed_T : (threadIdx.x == 0 ? T_dev[0] : 0.0), sigma_r, eps, rule,
            log_2_over_eps, plan_out, terms, cap, forced_N, forced_M, sp);
}

}  // namespace

int launch_plan(const double* T_dev, int use_fixed, double fixed_T, double sigma_r, double eps,
                int rule, double log_2_over_eps, sbf_plan* plan_dev, sbf_term* terms_dev,
                int terms_cap, cudaStream_t st, int forced_N, int forced_M) {
  SBF_REQUIRE(plan_dev && terms_dev && terms_cap > 0, SBF_ERR_INVALID, "null plan/terms buffer");
  SBF_REQUIRE(use_fixed || T_dev, SBF_ERR_INVALID, "null T");
  plan_kernel<<<1, 32, 0, st>>>(T_dev, use_fixed, fixed_T, sigma_r, eps, rule, log_2_over_eps,
                                plan_dev, terms_dev, terms_cap, forced_N, forced_M);
  SBF_CHECK_LAUNCH();
  return SBF_OK;
}

}  // namespace sbf

// ---------------------------------------------------------------------------
// host twins (same source as K2)
// ---------------------------------------------------------------------------
extern "C" {

int sbf_extended_box_params(double sigma_s, int passes, int* r, double* alpha) {
  if (!(sigma_s > 0.0) || passes < 1 || !r || !alpha) {
    sbf::set_error("sigma_s must be positive and passes >= 1");
    return SBF_ERR_INVALID;
  }
  sbf::extended_box_params(sigma_s, passes, r, alpha);
  return SBF_OK;
}

int sbf_support_radius(const sbf_spatial* sp, int* radius) {
  if (!sp || !radius) return SBF_ERR_INVALID;
  if (sp->mode == SBF_SPATIAL_BOX) {
    *radius = sp->r;
  } else {
    *radius = sp->passes * (sp->r + (sp->alpha > 0.0 ? 1 : 0));
  }
  return SBF_OK;
}

int sbf_order_threshold(double T, double sigma_r, int* N) {
  if (!(sigma_r > 0.0) || !(T >= 0.0) || !N) {
    sbf::set_error("need sigma_r > 0 and T >= 0");
    return SBF_ERR_INVALID;
  }
  int flags = 0, status = SBF_OK;
  *N = sbf::order_threshold(T, sigma_r, &flags, &status);
  return status;
}

int sbf_truncation_index_exact(int N, double epsilon, int* M) {
  if (N < 1 || !(epsilon >= 0.0 && epsilon < 1.0) || !M) {
    sbf::set_error("need N >= 1 and 0 <= epsilon < 1");
    return SBF_ERR_INVALID;
  }
  int flags = 0, status = SBF_OK;
  *M = sbf::truncation_index_exact(N, epsilon, &flags, &status, false);
  return status;
}

// force the multi-limb path (test hook for the exact arithmetic)
int sbf_truncation_index_exact_bigint(int N, double epsilon, int* M) {
  if (N < 1 || !(epsilon > 0.0 && epsilon < 1.0) || !M) return SBF_ERR_INVALID;
  int status = SBF_OK;
  *M = sbf::truncation_exact_bigint(N, epsilon, &status);
  return status;
}

int sbf_truncation_index_chernoff(int N, double epsilon, double log_2_over_eps, int* M) {
  if (N < 1 || !(epsilon > 0.0 && epsilon < 1.0) || !M) {
    sbf::set_error("epsilon must be positive for the tail-bound rule; use M=0 for epsilon=0");
    return SBF_ERR_INVALID;
  }
  int status = SBF_OK;
  *M = sbf::truncation_index_chernoff(N, epsilon, log_2_over_eps, &status);
  return status;
}

int sbf_select_plan(double T, double sigma_r, double epsilon, int rule, double log_2_over_eps,
                    sbf_plan* out) {
  if (!out) return SBF_ERR_INVALID;
  sbf::select_plan(T, sigma_r, epsilon, rule, log_2_over_eps, out);
  if (out->status != SBF_OK) sbf::set_error("select_plan failed (status %d)", out->status);
  return out->status;
}

}  // extern "C"

// Binomial weights C(N, n) / 2^N for n in [lo, hi], each correctly rounded to
// float64 (round half to even, subnormal results included) — the host twin
// of reference kernels.py:198-212.  C(N, n) is carried as an exact multi-limb
// integer (32-bit limbs) and stepped with C(N, n+1) = C(N, n) (N-n) / (n+1),
// where the division is exact.
namespace {
struct BigNat {
  std::vector<uint32_t> limb;  // little endian
  explicit BigNat(uint32_t v) : limb(1, v) {}
  void mul(uint32_t m) {
    uint64_t carry = 0;
    for (auto& x : limb) {
      const uint64_t t = (uint64_t)x * m + carry;
      x = (uint32_t)t;
      carry = t >> 32;
    }
    if (carry) limb.push_back((uint32_t)carry);
  }
  void div_exact(uint32_t d) {
    uint64_t rem = 0;
    for (size_t i = limb.size(); i-- > 0;) {
      const uint64_t cur = (rem << 32) | limb[i];
      limb[i] = (uint32_t)(cur / d);
      rem = cur % d;
    }
    while (limb.size() > 1 && limb.back() == 0) limb.pop_back();
  }
  int64_t bitlen() const {
    const uint32_t top = limb.back();
    if (top == 0) return 0;
    return (int64_t)(limb.size() - 1) * 32 + (32 - __builtin_clz(top));
  }
  bool bit(int64_t k) const {
    if (k < 0 || k / 32 >= (int64_t)limb.size()) return false;
    return (limb[k / 32] >> (k % 32)) & 1u;
  }
  bool any_below(int64_t k) const {  // any set bit at positions < k
    for (int64_t i = 0; i < k / 32 && i < (int64_t)limb.size(); ++i)
      if (limb[i]) return true;
    if (k % 32 && k / 32 < (int64_t)limb.size())
      return (limb[k / 32] & ((1u << (k % 32)) - 1u)) != 0;
    return false;
  }
  // floor(self / 2^shift) for a result below 2^64
  uint64_t shifted(int64_t shift) const {
    uint64_t r = 0;
    for (int k = 63; k >= 0; --k) r = (r << 1) | (bit(shift + k) ? 1u : 0u);
    return r;
  }
};

// self / 2^N correctly rounded to double
double ratio_pow2(const BigNat& c, int N) {
  const int64_t b = c.bitlen();
  if (b == 0) return 0.0;
  const int64_t e = b - 1 - N;  // floor(log2(result))
  // bits to drop: keep 53 significant bits, or fewer below 2^-1022
  const int64_t shift = e >= -1022 ? b - 53 : (int64_t)N - 1074;
  if (shift <= 0) return std::ldexp((double)c.shifted(0), -N);  // exact (b <= 53)
  uint64_t m = c.shifted(shift);
  const bool half = c.bit(shift - 1), sticky = c.any_below(shift - 1);
  if (half && (sticky || (m & 1u))) ++m;
  return std::ldexp((double)m, (int)(shift - N));
}
}  // namespace

extern "C" int sbf_binomial_weights(int N, int lo, int hi, double* out) {
  if (N < 0 || lo < 0 || hi < lo || hi > N || !out) {
    sbf::set_error("need 0 <= lo <= hi <= N");
    return SBF_ERR_INVALID;
  }
  BigNat c(1);
  for (int i = 1; i <= lo; ++i) {  // C(N, lo) = prod (N - lo + i) / i, exact at every step
    c.mul((uint32_t)(N - lo + i));
    c.div_exact((uint32_t)i);
  }
  for (int n = lo; n <= hi; ++n) {
    out[n - lo] = ratio_pow2(c, N);
    if (n < hi) {
      c.mul((uint32_t)(N - n));
      c.div_exact((uint32_t)(n + 1));
    }
  }
  return SBF_OK;
}
