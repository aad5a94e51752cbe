// Shared fp64 machinery of the generic path (sbf_generic.cu), reused by the
// coarse NLM driver (sbf_nlm.cu).
#pragma once

#include "sbf_common.cuh"

namespace sbf {

struct FusedEntry;

// Smooths four fp64 planes with the configured spatial mode (extended-box
// passes with exact clamped renormalisation, or the box filter).  When
// `fused` the caller writes the planes TRANSPOSED ([pl][W][H]) into `tmp`;
// otherwise into `planes` ([pl][H][W]).  The result is in `planes`.
struct PlaneSmoother {
  bool fused = false;
  int64_t H = 0, W = 0, row0 = 0, img_H = 0;
  int passes = 1, r = 0, pad = 0;
  double alpha = 0.0, ca = 0.0, cb = 0.0;
  const FusedEntry* fe = nullptr;
  double* gx = nullptr;
  double* gy = nullptr;
  cudaStream_t stream = nullptr;
  int init(const sbf_spatial& sp, int64_t H, int64_t W, int64_t row0, int64_t img_H,
           cudaStream_t st);
  int run(double* planes, double* tmp, cudaStream_t st, int nplanes = 4) const;
  void release(cudaStream_t st);
  PlaneSmoother() = default;
  PlaneSmoother(const PlaneSmoother&) = delete;
  PlaneSmoother& operator=(const PlaneSmoother&) = delete;
  ~PlaneSmoother() { release(stream); }  // tables freed on every exit path
};

// Dual (direct) evaluation for untruncated plans (sbf_dual.cu): picked for
// fp64 filtering when (2S+1)^2 taps per pixel cost less than K terms.
bool dual_preferred(const FilterLaunch& a, const sbf_plan& plan);
int launch_dual_direct(const FilterLaunch& a, const sbf_plan& plan);

}  // namespace sbf
