// Generic fp64 term path for spatial parameters without a specialised K3
// instantiation (large radii, unusual pass counts).  Still CUDA end to end —
// there is no CPU fallback anywhere in the library.
//
// Per term: build the four modulated planes, run each extended-box pass as a
// row kernel then a column kernel (reference order, spatial.py:114-117,
// :136-139) with exact clamped renormalisation, then accumulate num/den.
// Everything in float64, so this path is also the accuracy yardstick for
// the fast kernels.  It reads the plan back to the host once (the term count
// drives the launch loop).
#include <vector>

#include "sbf_common.cuh"
#include "sbf_generic.h"

#include "sbf_generic_fused.cuh"

namespace sbf {
namespace {

__global__ void gen_images(const void* f, int f64, int64_t H, int64_t W, int64_t ld,
                           const double* stats, double turns, double* planes) {
  const int64_t n = H * W;
  const double center = stats[3];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = i / W, x = i - y * W;
    const double fv = f64 ? static_cast<const double*>(f)[y * ld + x]
                          : (double)static_cast<const float*>(f)[y * ld + x];
    const double fc = fv - center;
    const double u = fc * turns;
    const double t = u - rint(u);
    double s, c;
    sincospi(2.0 * t, &s, &c);
    planes[i] = fc * c;
    planes[n + i] = c;
    planes[2 * n + i] = fc * s;
    planes[3 * n + i] = s;
  }
}

// same images written transposed: planes[pl][x][y]
__global__ void gen_images_T(const void* f, int f64, int64_t H, int64_t W, int64_t ld,
                             const double* stats, double turns, double* planes) {
  __shared__ double tile[4][32][33];
  const int64_t n = H * W;
  const double center = stats[3];
  const int64_t x0 = (int64_t)blockIdx.x * 32, y0 = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t y = y0 + k, x = x0 + threadIdx.x;
    if (y < H && x < W) {
      const double fv = f64 ? static_cast<const double*>(f)[y * ld + x]
                            : (double)static_cast<const float*>(f)[y * ld + x];
      const double fc = fv - center;
      const double u = fc * turns;
      const double t = u - rint(u);
      double s, c;
      sincospi(2.0 * t, &s, &c);
      tile[0][k][threadIdx.x] = fc * c;
      tile[1][k][threadIdx.x] = c;
      tile[2][k][threadIdx.x] = fc * s;
      tile[3][k][threadIdx.x] = s;
    }
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t x = x0 + k, y = y0 + threadIdx.x;
    if (x < W && y < H) {
#pragma unroll
      for (int pl = 0; pl < 4; ++pl) planes[pl * n + x * H + y] = tile[pl][threadIdx.x][k];
    }
  }
}

// one extended-box pass along rows (contiguous), 4 planes
__global__ void gen_rows(const double* __restrict__ in, double* __restrict__ out, int64_t lines,
                         int64_t W, int r, double alpha) {
  const int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (line >= lines) return;
  const double* x = in + line * W;
  double* y = out + line * W;
  double S = 0.0;
  for (int64_t k = 0; k <= r && k < W; ++k) S += x[k];
  for (int64_t i = 0; i < W; ++i) {
    if (i > 0) {
      if (i + r < W) S += x[i + r];
      if (i - r - 1 >= 0) S -= x[i - r - 1];
    }
    const int64_t lo = i - r < 0 ? 0 : i - r;
    const int64_t hi = i + r > W - 1 ? W - 1 : i + r;
    double cnt = (double)(hi - lo + 1), tot = S;
    if (alpha > 0.0) {
      if (i - r - 1 >= 0) {
        tot += alpha * x[i - r - 1];
        cnt += alpha;
      }
      if (i + r + 1 <= W - 1) {
        tot += alpha * x[i + r + 1];
        cnt += alpha;
      }
    }
    y[i] = tot / cnt;
  }
}

// one extended-box pass along columns; counts use global row positions
__global__ void gen_cols(const double* __restrict__ in, double* __restrict__ out, int nplanes,
                         int64_t H, int64_t W, int64_t row0, int64_t img_H, int r, double alpha) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= nplanes * W) return;
  const int64_t pl = id / W, xcol = id - pl * W;
  const double* x = in + pl * H * W + xcol;
  double* y = out + pl * H * W + xcol;
  double S = 0.0;
  for (int64_t k = 0; k <= r && k < H; ++k) S += x[k * W];
  for (int64_t i = 0; i < H; ++i) {
    if (i > 0) {
      if (i + r < H) S += x[(i + r) * W];
      if (i - r - 1 >= 0) S -= x[(i - r - 1) * W];
    }
    const int64_t g = row0 + i;
    const int64_t lo = g - r < 0 ? 0 : g - r;
    const int64_t hi = g + r > img_H - 1 ? img_H - 1 : g + r;
    double cnt = (double)(hi - lo + 1), tot = S;
    if (alpha > 0.0) {
      if (g - r - 1 >= 0) {
        if (i - r - 1 >= 0) tot += alpha * x[(i - r - 1) * W];
        cnt += alpha;
      }
      if (g + r + 1 <= img_H - 1) {
        if (i + r + 1 < H) tot += alpha * x[(i + r + 1) * W];
        cnt += alpha;
      }
    }
    y[i * W] = tot / cnt;
  }
}

__global__ void gen_accum(const double* __restrict__ planes, const void* f, int f64, int64_t H,
                          int64_t W, int64_t ld, int64_t out_lo, int64_t out_hi,
                          const double* stats, double turns, double scale, int first,
                          double* __restrict__ nd) {
  const int64_t n = H * W;
  const int64_t m = (out_hi - out_lo) * W;
  const double center = stats[3];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t yo = i / W, x = i - yo * W;
    const int64_t y = out_lo + yo;
    const int64_t pi = y * W + x;
    const double fv = f64 ? static_cast<const double*>(f)[y * ld + x]
                          : (double)static_cast<const float*>(f)[y * ld + x];
    const double u = (fv - center) * turns;
    const double t = u - rint(u);
    double s, c;
    sincospi(2.0 * t, &s, &c);
    const double num = scale * (c * planes[pi] + s * planes[2 * n + pi]);
    const double den = scale * (c * planes[n + pi] + s * planes[3 * n + pi]);
    if (first) {
      nd[2 * i] = num;
      nd[2 * i + 1] = den;
    } else {
      nd[2 * i] += num;
      nd[2 * i + 1] += den;
    }
  }
}

}  // namespace

// ---- reusable fp64 smoother of four planes (also used by coarse NLM) ----
int PlaneSmoother::init(const sbf_spatial& sp, int64_t H_, int64_t W_, int64_t row0_,
                        int64_t img_H_, cudaStream_t st) {
  stream = st;
  H = H_;
  W = W_;
  row0 = row0_;
  img_H = img_H_;
  passes = sp.mode == SBF_SPATIAL_BOX ? 1 : sp.passes;
  alpha = sp.mode == SBF_SPATIAL_BOX ? 0.0 : sp.alpha;
  r = sp.r;
  static const FusedEntry fused_tab[] = {
      {0, &launch_colpass<0>},   {1, &launch_colpass<1>},   {2, &launch_colpass<2>},
      {3, &launch_colpass<3>},   {4, &launch_colpass<4>},   {5, &launch_colpass<5>},
      {6, &launch_colpass<6>},   {7, &launch_colpass<7>},   {8, &launch_colpass<8>},
      {9, &launch_colpass<9>},   {10, &launch_colpass<10>}, {11, &launch_colpass<11>},
      {12, &launch_colpass<12>}};
  fe = (passes == 3 && r >= 0 && r <= 12) ? &fused_tab[r] : nullptr;
  fused = fe != nullptr;
  gx = gy = nullptr;
  if (fused) {
    pad = 3 * (r + 1) + 2 * (r + 1) + 2;
    const double cint = 2.0 * r + 1.0 + 2.0 * alpha;
    ca = (1.0 - alpha) / cint;
    cb = alpha / cint;
    SBF_CHECK_CUDA(cudaMallocAsync(&gx, sizeof(double) * (W + 2 * pad), st));
    SBF_CHECK_CUDA(cudaMallocAsync(&gy, sizeof(double) * (H + 2 * pad), st));
    gfactor_table<<<(unsigned)((W + 2 * pad + 255) / 256), 256, 0, st>>>(gx, W, 0, W, r, alpha, pad);
    gfactor_table<<<(unsigned)((H + 2 * pad + 255) / 256), 256, 0, st>>>(gy, H, row0, img_H, r,
                                                                        alpha, pad);
    SBF_CHECK_LAUNCH();
  }
  return SBF_OK;
}

int PlaneSmoother::run(double* planes, double* tmp, cudaStream_t st, int nplanes) const {
  const int bs = 256;
  const dim3 tb(32, 8);
  if (fused) {
    // input: tmp [pl][W][H] (rows as columns); output planes [pl][H][W]
    const dim3 tgridT((unsigned)((H + 31) / 32), (unsigned)((W + 31) / 32), (unsigned)nplanes);
    // segment length: the longest (least recomputed warm-up) that still gives
    // two CTAs of 128 column streams per SM.  NLM config 2 (4 planes of
    // 1024^2): 256 -> 5.9 ms of column passes, 128 -> 3.1, 96 -> 2.5,
    // 64 -> 3.6; large images keep 256.
    auto seg_for = [&](int64_t n_stream, int64_t n_cols) {
      const int64_t want = (int64_t)device_sm_count() * 2 * 128;
      int64_t seg = 64;
      for (int64_t cand : {256, 192, 128, 96}) {
        if ((int64_t)nplanes * n_cols * ((n_stream + cand - 1) / cand) >= want) {
          seg = cand;
          break;
        }
      }
      return seg;
    };
    fe->launch(tmp, planes, nplanes, W, H, seg_for(W, H), gx, 0, W, ca, cb, st);        // row passes
    transpose_planes<<<tgridT, tb, 0, st>>>(planes, tmp, W, H);                       // -> [pl][H][W]
    fe->launch(tmp, planes, nplanes, H, W, seg_for(H, W), gy, row0, img_H, ca, cb, st);  // column passes
  } else {
    // input and output: planes [pl][H][W]
    for (int ps = 0; ps < passes; ++ps) {
      gen_rows<<<(unsigned)((nplanes * H + bs - 1) / bs), bs, 0, st>>>(planes, tmp, nplanes * H, W,
                                                                       r, alpha);
      gen_cols<<<(unsigned)((nplanes * W + bs - 1) / bs), bs, 0, st>>>(tmp, planes, nplanes, H, W,
                                                                       row0, img_H, r, alpha);
    }
  }
  SBF_CHECK_LAUNCH();
  return SBF_OK;
}

void PlaneSmoother::release(cudaStream_t st) {
  if (gx) cudaFreeAsync(gx, st);
  if (gy) cudaFreeAsync(gy, st);
  gx = gy = nullptr;
}

int launch_generic_terms(const FilterLaunch& a, double* nd) {
  cudaStream_t st = a.stream;
  sbf_plan plan;
  SBF_CHECK_CUDA(cudaMemcpyAsync(&plan, a.plan, sizeof(plan), cudaMemcpyDeviceToHost, st));
  SBF_CHECK_CUDA(cudaStreamSynchronize(st));
  if (plan.status != SBF_OK) return SBF_OK;  // surfaced by the caller from the plan
  std::vector<sbf_term> terms(plan.K_eval > 0 ? plan.K_eval : 1);
  if (plan.K_eval > 0) {
    SBF_CHECK_CUDA(cudaMemcpyAsync(terms.data(), a.terms, sizeof(sbf_term) * plan.K_eval,
                                   cudaMemcpyDeviceToHost, st));
    SBF_CHECK_CUDA(cudaStreamSynchronize(st));
  }
  const int64_t H = a.H, W = a.W, n = H * W;
  DevBuf<double> planes_b(st), tmp_b(st);
  SBF_CHECK_CUDA(planes_b.alloc(4 * n));
  SBF_CHECK_CUDA(tmp_b.alloc(4 * n));
  double* planes = planes_b.p;
  double* tmp = tmp_b.p;
  const int bs = 256;
  const unsigned gpix = (unsigned)smin<int64_t>((n + bs - 1) / bs, 148 * 16);
  PlaneSmoother sm;
  int rc = sm.init(a.sp, H, W, a.row0, a.img_H, st);
  if (rc != SBF_OK) return rc;
  const dim3 tb(32, 8), tgrid((unsigned)((W + 31) / 32), (unsigned)((H + 31) / 32), 1);
  for (int k = 0; k < plan.K_eval; ++k) {
    if (sm.fused)
      gen_images_T<<<tgrid, tb, 0, st>>>(a.f, a.dtype == SBF_F64, H, W, a.ld, a.stats,
                                         terms[k].turns, tmp);  // [pl][W][H]
    else
      gen_images<<<gpix, bs, 0, st>>>(a.f, a.dtype == SBF_F64, H, W, a.ld, a.stats,
                                      terms[k].turns, planes);
    rc = sm.run(planes, tmp, st);
    if (rc != SBF_OK) return rc;
    gen_accum<<<gpix, bs, 0, st>>>(planes, a.f, a.dtype == SBF_F64, H, W, a.ld, a.out_lo,
                                   a.out_hi, a.stats, terms[k].turns, terms[k].scale, k == 0, nd);
    SBF_CHECK_LAUNCH();
  }
  return SBF_OK;
}

}  // namespace sbf
