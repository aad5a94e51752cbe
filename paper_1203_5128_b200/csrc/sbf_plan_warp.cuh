// K2 warp body shared by the plan kernel (sbf_plan.cu) and K1's last CTA
// (sbf_local_range.cu, fused pipeline): one warp selects (N, M) and writes the
// folded term table.  See sbf_plan.cu for the algorithm notes.
#pragma once

#include "sbf_common.cuh"
#include "sbf_plan_logic.cuh"

namespace sbf {

// t_k = C(N, nc-k) / C(N, nc) for k = base + lane: the inclusive warp scan of
// the ratios (nc-j+1)/(N-nc+j), j = 1..k, times the carry t_{base-1}.
__device__ __forceinline__ double plan_ratio_scan(int N, int nc, int k, double carry) {
  const int lane = threadIdx.x & 31;
  double v = (k == 0 || k > nc) ? 1.0 : (double)(nc - k + 1) / (double)(N - nc + k);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v *= u;
  }
  return carry * v;
}

// Called by all 32 lanes of one warp; T is read by lane 0 only.
__device__ __forceinline__ void plan_warp(double T, double sigma_r, double eps, int rule,
                                          double log_2_over_eps, sbf_plan* __restrict__ plan_out,
                                          sbf_term* __restrict__ terms, int cap, int forced_N,
                                          int forced_M, sbf_plan& sp) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
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
      const double t = plan_ratio_scan(N, nc, k, carry);
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
      const double t = plan_ratio_scan(N, nc, k, carry);
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


}  // namespace sbf
