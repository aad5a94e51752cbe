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

namespace sbf {
namespace {

// t_k = C(N, nc-k) / C(N, nc) for k = base + lane: the inclusive warp scan of
// the ratios (nc-j+1)/(N-nc+j), j = 1..k, times the carry t_{base-1}.
__device__ __forceinline__ double ratio_scan(int N, int nc, int k, double carry) {
  const int lane = threadIdx.x & 31;
  double v = (k == 0 || k > nc) ? 1.0 : (double)(nc - k + 1) / (double)(N - nc + k);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v *= u;
  }
  return carry * v;
}

// One warp.  Lane 0 selects (N, M) with the shared plan logic; the binomial
// weights (centre-outward ratio recurrence) run as warp-wide prefix products,
// 32 terms per step instead of one fp64 division chain per term.
__global__ void plan_kernel(const double* __restrict__ T_dev, int use_fixed, double fixed_T,
                            double sigma_r, double eps, int rule, double log_2_over_eps,
                            sbf_plan* __restrict__ plan_out, sbf_term* __restrict__ terms,
                            int cap, int forced_N, int forced_M) {
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  __shared__ sbf_plan sp;
  if (lane == 0) {
    const double T = use_fixed ? fixed_T : T_dev[0];
    sbf_plan p;
    select_plan(T, sigma_r, eps, rule, log_2_over_eps, &p);
    if (forced_N > 0 && p.status == SBF_OK) {
      // host-resolved (N, M) (libm pow, bit-equal to CPython) after the device
      // flagged SBF_PLAN_N_AMBIGUOUS; the term table follows from it
      p.N = forced_N;
      p.M = forced_M;
      p.K = forced_N / 2 - forced_M + 1;
      p.K_eval = p.K;
      p.gamma = 1.0 / (sqrt((double)forced_N) * sigma_r);
      p.flags &= ~SBF_PLAN_N_AMBIGUOUS;
    }
    sp = p;
  }
  __syncwarp();
  sbf_plan p = sp;
  if (p.status == SBF_OK) {
    const int N = p.N, M = p.M, nc = N / 2;
    // total = sum_{n=0}^{N} C(N,n)/C(N,nc) by symmetry from the half sum
    double half = 0.0, carry = 1.0;
    for (int base = 0; base <= nc; base += 32) {
      const int k = base + lane;
      const double t = ratio_scan(N, nc, k, carry);
      if (k <= nc) half += t;
      carry = __shfl_sync(0xffffffffu, t, 31);
      if (carry == 0.0) break;  // every later ratio product underflows too
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) half += __shfl_xor_sync(0xffffffffu, half, o);
    const double total = 2.0 * half - ((N % 2 == 0) ? 1.0 : 0.0);
    const double inv2pi = 0.15915494309189535;
    const double denom = sqrt((double)N) * sigma_r;
    int kept = 0;
    carry = 1.0;
    for (int base = 0; base <= nc - M; base += 32) {
      const int k = base + lane;
      const double t = ratio_scan(N, nc, k, carry);
      const int n = nc - k;
      const double d = t / total;
      const double scale = (2 * n == N) ? d : 2.0 * d;
      // weights only shrink away from the centre: exact zeros form a suffix
      // and contribute nothing (float64 underflow in the reference too)
      const bool keep = k <= nc - M && scale != 0.0;
      if (keep && k < cap) {
        sbf_term tm;
        tm.scale = scale;
        tm.freq = (double)(2 * n - N) / denom;
        tm.turns = tm.freq * inv2pi;
        tm.index = n;
        tm.pad = 0;
        terms[k] = tm;
      }
      const unsigned ballot = __ballot_sync(0xffffffffu, keep);
      kept += __popc(ballot);
      carry = __shfl_sync(0xffffffffu, t, 31);
      if (ballot != 0xffffffffu) break;
    }
    p.K_eval = kept;
    if (kept > cap) {
      p.flags |= SBF_PLAN_TERMS_TRUNCATED;
      p.status = SBF_ERR_UNSUPPORTED;
    }
  }
  if (lane == 0) *plan_out = p;
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
