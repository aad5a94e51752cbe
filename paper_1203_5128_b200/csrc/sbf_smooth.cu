// Standalone spatial smoothers on the GPU (reference spatial.py): the
// public `box_filter` (:65-78), `iterated_box_gaussian` (:108-139) and
// `fir_gaussian` (:142-172) / `apply_spatial` (:175-182), in float64 like the
// reference.  The extended-box modes run on the plane smoother of the
// generic path (fused register-ring cascade or row/column kernels, exact
// clamped renormalisation); the FIR Gaussian is a separable window sum
// renormalised by the in-bounds taps.
#include <math.h>

#include "sbf_common.cuh"
#include "sbf_generic.h"

namespace sbf {
namespace {

// in (any float dtype, ld) -> fp64 plane [H][W] or transposed [W][H]
template <typename FT>
__global__ void load_plane(const FT* __restrict__ f, int64_t H, int64_t W, int64_t ld,
                           int transposed, double* __restrict__ out) {
  const int64_t n = H * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = i / W, x = i - y * W;
    out[transposed ? x * H + y : i] = (double)f[y * ld + x];
  }
}

template <typename OT>
__global__ void store_plane(const double* __restrict__ in, int64_t n, OT* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (OT)in[i];
}

// one FIR pass along rows (axis 1) or columns (axis 0): weighted window sum
// over in-bounds samples divided by the in-bounds weight (spatial.py:160-172)
__global__ void fir_pass(const double* __restrict__ in, double* __restrict__ out, int64_t H,
                         int64_t W, int axis, int R, double sigma) {
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t y = blockIdx.y;
  if (x >= W || y >= H) return;
  const double inv = 1.0 / (2.0 * sigma * sigma);
  const int64_t pos = axis ? x : y, n = axis ? W : H;
  double num = 0.0, den = 0.0;
  for (int k = -R; k <= R; ++k) {
    const int64_t q = pos + k;
    if (q < 0 || q >= n) continue;
    const double w = exp(-(double)(k * k) * inv);
    num += w * (axis ? in[y * W + q] : in[q * W + x]);
    den += w;
  }
  out[y * W + x] = num / den;
}

}  // namespace
}  // namespace sbf

extern "C" int sbf_smooth(const void* f, int dtype, int64_t H, int64_t W, int64_t ld,
                          const sbf_spatial* sp, void* out, int out_dtype, void* stream) {
  using namespace sbf;
  SBF_REQUIRE(f && sp && out, SBF_ERR_INVALID, "null pointer");
  SBF_REQUIRE(dtype == SBF_F32 || dtype == SBF_F64, SBF_ERR_INVALID, "bad dtype");
  SBF_REQUIRE(out_dtype == SBF_F32 || out_dtype == SBF_F64, SBF_ERR_INVALID, "bad out dtype");
  SBF_REQUIRE(H >= 1 && W >= 1 && ld >= W, SBF_ERR_INVALID, "bad image shape");
  SBF_REQUIRE(sp->r >= 0, SBF_ERR_INVALID, "radius must be >= 0");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = H * W;
  const unsigned grid = (unsigned)smin<int64_t>((n + 255) / 256, 148 * 16);
  DevBuf<double> a_b(st), b_b(st);
  SBF_CHECK_CUDA(a_b.alloc(n));
  SBF_CHECK_CUDA(b_b.alloc(n));
  double *a = a_b.p, *b = b_b.p;
  double* res = a;
  if (sp->mode == SBF_SPATIAL_FIR) {
    SBF_REQUIRE(sp->sigma_s > 0.0 && sp->r >= 1, SBF_ERR_INVALID,
                "FIR Gaussian needs sigma_s > 0 and radius >= 1");
    if (dtype == SBF_F32)
      load_plane<float><<<grid, 256, 0, st>>>(static_cast<const float*>(f), H, W, ld, 0, a);
    else
      load_plane<double><<<grid, 256, 0, st>>>(static_cast<const double*>(f), H, W, ld, 0, a);
    const dim3 g2((unsigned)((W + 255) / 256), (unsigned)H);
    fir_pass<<<g2, 256, 0, st>>>(a, b, H, W, 1, sp->r, sp->sigma_s);  // rows
    fir_pass<<<g2, 256, 0, st>>>(b, a, H, W, 0, sp->r, sp->sigma_s);  // columns
  } else {
    SBF_REQUIRE(sp->mode == SBF_SPATIAL_ITERATED || sp->mode == SBF_SPATIAL_BOX, SBF_ERR_INVALID,
                "bad spatial mode");
    PlaneSmoother sm;
    int rc = sm.init(*sp, H, W, 0, H, st);
    if (rc != SBF_OK) return rc;
    if (sp->mode == SBF_SPATIAL_BOX && sp->r == 0) {
      // spatial.py:72-73: radius 0 is the identity
      if (dtype == SBF_F32)
        load_plane<float><<<grid, 256, 0, st>>>(static_cast<const float*>(f), H, W, ld, 0, a);
      else
        load_plane<double><<<grid, 256, 0, st>>>(static_cast<const double*>(f), H, W, ld, 0, a);
    } else {
      // fused cascade expects the plane transposed in `tmp`, the others in `planes`
      double* dst = sm.fused ? b : a;
      if (dtype == SBF_F32)
        load_plane<float><<<grid, 256, 0, st>>>(static_cast<const float*>(f), H, W, ld, sm.fused,
                                                 dst);
      else
        load_plane<double><<<grid, 256, 0, st>>>(static_cast<const double*>(f), H, W, ld,
                                                  sm.fused, dst);
      rc = sm.run(a, b, st, 1);
      if (rc != SBF_OK) return rc;
    }
  }
  if (out_dtype == SBF_F64)
    store_plane<double><<<grid, 256, 0, st>>>(res, n, static_cast<double*>(out));
  else
    store_plane<float><<<grid, 256, 0, st>>>(res, n, static_cast<float*>(out));
  SBF_CHECK_LAUNCH();
  return SBF_OK;
}
