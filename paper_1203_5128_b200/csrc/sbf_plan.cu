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
