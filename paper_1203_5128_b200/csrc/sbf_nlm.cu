// Coarse non-local means with shiftable range kernels (reference
// nlm.py:78-137) on the fp64 term engine of the
// generic path.
//
// Similarity uses p <= 3 patch samples f(x + u_j) (replicate padding,
// nlm.py:68-75), each with its own raised-cosine expansion.  The tensor
// product of the per-component expansions is evaluated item by item; an
// item is one folded multi-index (n_0..n_{p-1}) and one choice of cos/sin
// for the components j >= 1, and carries the pair
//     a1 = cos(w_0 f) R,   a2 = sin(w_0 f) R,   R = prod_{j>=1} cos|sin(w_j f(x+u_j))
// so that, exactly as in the bilateral kernel, it smooths f a1, a1, f a2, a2
// and adds weight * (a1 S[f a1] + a2 S[f a2]) to num (den likewise).  The
// 2^p sign masks of the reference are the two members of the pair times the
// 2^(p-1) items per multi-index.  Folding +-w per component is exact: every
// mask term is even in each w_j (it is bilinear in its aux image).
// Intensities are centred (mid-range) before the phases, which leaves the
// filter unchanged (it depends on differences only) and keeps fp64 phases
// small.
#include <vector>

#include "sbf_common.cuh"
#include "sbf_generic.h"

namespace sbf {
namespace {

struct NlmGeom {
  int p;
  int dy[3], dx[3];
};

__device__ __forceinline__ double load_f(const void* f, int f64, int64_t ld, int64_t y, int64_t x) {
  return f64 ? static_cast<const double*>(f)[y * ld + x]
             : (double)static_cast<const float*>(f)[y * ld + x];
}

__device__ __forceinline__ void phase(double v, double turns, double* s, double* c) {
  const double u = v * turns;
  sincospi(2.0 * (u - rint(u)), s, c);
}

__device__ __forceinline__ void nlm_aux(const void* f, int f64, int64_t H, int64_t W, int64_t ld,
                                        int64_t y, int64_t x, double center, const NlmGeom& g,
                                        const sbf_nlm_item& it, double* fc, double* a1, double* a2) {
  *fc = load_f(f, f64, ld, y, x) - center;
  double s0, c0;
  phase(*fc, it.turns[0], &s0, &c0);
  double rest = 1.0;
  for (int j = 1; j < g.p; ++j) {
    int64_t yy = y + g.dy[j], xx = x + g.dx[j];
    yy = yy < 0 ? 0 : (yy >= H ? H - 1 : yy);
    xx = xx < 0 ? 0 : (xx >= W ? W - 1 : xx);
    double s, c;
    phase(load_f(f, f64, ld, yy, xx) - center, it.turns[j], &s, &c);
    rest *= ((it.mask >> j) & 1) ? s : c;
  }
  *a1 = c0 * rest;
  *a2 = s0 * rest;
}

// planes [pl][W][H] (transposed, for the fused smoother)
__global__ void nlm_images_T(const void* f, int f64, int64_t H, int64_t W, int64_t ld,
                             const double* stats, const NlmGeom g, const sbf_nlm_item it,
                             double* planes) {
  __shared__ double tile[4][32][33];
  const int64_t n = H * W;
  const double center = stats[3];
  const int64_t x0 = (int64_t)blockIdx.x * 32, y0 = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t y = y0 + k, x = x0 + threadIdx.x;
    if (y < H && x < W) {
      double fc, a1, a2;
      nlm_aux(f, f64, H, W, ld, y, x, center, g, it, &fc, &a1, &a2);
      tile[0][k][threadIdx.x] = fc * a1;
      tile[1][k][threadIdx.x] = a1;
      tile[2][k][threadIdx.x] = fc * a2;
      tile[3][k][threadIdx.x] = a2;
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

// planes [pl][H][W]
__global__ void nlm_images(const void* f, int f64, int64_t H, int64_t W, int64_t ld,
                           const double* stats, const NlmGeom g, const sbf_nlm_item it,
                           double* planes) {
  const int64_t n = H * W;
  const double center = stats[3];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = i / W, x = i - y * W;
    double fc, a1, a2;
    nlm_aux(f, f64, H, W, ld, y, x, center, g, it, &fc, &a1, &a2);
    planes[i] = fc * a1;
    planes[n + i] = a1;
    planes[2 * n + i] = fc * a2;
    planes[3 * n + i] = a2;
  }
}

__global__ void nlm_accum(const double* __restrict__ planes, const void* f, int f64, int64_t H,
                          int64_t W, int64_t ld, const double* stats, const NlmGeom g,
                          const sbf_nlm_item it, int first, double* __restrict__ nd) {
  const int64_t n = H * W;
  const double center = stats[3];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = i / W, x = i - y * W;
    double fc, a1, a2;
    nlm_aux(f, f64, H, W, ld, y, x, center, g, it, &fc, &a1, &a2);
    const double num = it.weight * (a1 * planes[i] + a2 * planes[2 * n + i]);
    const double den = it.weight * (a1 * planes[n + i] + a2 * planes[3 * n + i]);
    if (first) {
      nd[2 * i] = num;
      nd[2 * i + 1] = den;
    } else {
      nd[2 * i] += num;
      nd[2 * i + 1] += den;
    }
  }
}

// nlm.py:137 -> bilateral.py:242-254 (centre added back)
template <typename FT, typename OT>
__global__ void nlm_epilogue(const double* __restrict__ nd, int have_terms, int64_t n, int64_t W,
                             const FT* __restrict__ f, int64_t ld, const double* stats,
                             OT* __restrict__ out, unsigned long long* __restrict__ fallback) {
  const double center = stats[3];
  unsigned long long bad_count = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double num = have_terms ? nd[2 * i] : 0.0, den = have_terms ? nd[2 * i + 1] : 0.0;
    const int64_t y = i / W, x = i - y * W;
    const bool bad = !(den > 0.0);
    out[i] = (OT)(bad ? (double)f[y * ld + x] : num / den + center);
    bad_count += bad ? 1 : 0;
  }
  for (int o = 16; o; o >>= 1) bad_count += __shfl_xor_sync(0xffffffffu, bad_count, o);
  if ((threadIdx.x & 31) == 0 && bad_count) atomicAdd(fallback, bad_count);
}

}  // namespace
}  // namespace sbf

extern "C" int sbf_nlm_filter(const void* f, int dtype, int64_t H, int64_t W, int64_t ld,
                              const sbf_spatial* sp, int p, const int32_t* offsets,
                              const sbf_nlm_item* items, int n_items, const double* stats,
                              void* out, int out_dtype, unsigned long long* fallback,
                              void* stream) {
  using namespace sbf;
  SBF_REQUIRE(f && sp && offsets && stats && out && fallback, SBF_ERR_INVALID, "null pointer");
  SBF_REQUIRE(n_items >= 0 && (n_items == 0 || items), SBF_ERR_INVALID, "bad item table");
  SBF_REQUIRE(dtype == SBF_F32 || dtype == SBF_F64, SBF_ERR_INVALID, "bad dtype");
  SBF_REQUIRE(out_dtype == SBF_F32 || out_dtype == SBF_F64, SBF_ERR_INVALID, "bad out dtype");
  SBF_REQUIRE(H >= 1 && W >= 1 && ld >= W, SBF_ERR_INVALID, "bad image shape");
  SBF_REQUIRE(p >= 1 && p <= 3, SBF_ERR_INVALID, "patch must have 1 to 3 offsets");
  SBF_REQUIRE(offsets[0] == 0 && offsets[1] == 0, SBF_ERR_INVALID,
              "first patch offset must be the origin");
  SBF_REQUIRE(sp->mode == SBF_SPATIAL_BOX || sp->mode == SBF_SPATIAL_ITERATED, SBF_ERR_INVALID,
              "bad spatial mode");
  NlmGeom g;
  memset(&g, 0, sizeof(g));
  g.p = p;
  for (int j = 0; j < p; ++j) {
    g.dy[j] = offsets[2 * j];
    g.dx[j] = offsets[2 * j + 1];
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = H * W;
  double *planes = nullptr, *tmp = nullptr, *nd = nullptr;
  SBF_CHECK_CUDA(cudaMallocAsync(&planes, sizeof(double) * 4 * n, st));
  SBF_CHECK_CUDA(cudaMallocAsync(&tmp, sizeof(double) * 4 * n, st));
  SBF_CHECK_CUDA(cudaMallocAsync(&nd, sizeof(double) * 2 * n, st));
  PlaneSmoother sm;
  int rc = sm.init(*sp, H, W, 0, H, st);
  if (rc != SBF_OK) return rc;
  const int bs = 256;
  const unsigned gpix = (unsigned)smin<int64_t>((n + bs - 1) / bs, 148 * 16);
  const dim3 tb(32, 8), tgrid((unsigned)((W + 31) / 32), (unsigned)((H + 31) / 32), 1);
  const int f64 = dtype == SBF_F64;
  for (int k = 0; k < n_items; ++k) {
    if (sm.fused)
      nlm_images_T<<<tgrid, tb, 0, st>>>(f, f64, H, W, ld, stats, g, items[k], tmp);
    else
      nlm_images<<<gpix, bs, 0, st>>>(f, f64, H, W, ld, stats, g, items[k], planes);
    rc = sm.run(planes, tmp, st);
    if (rc != SBF_OK) return rc;
    nlm_accum<<<gpix, bs, 0, st>>>(planes, f, f64, H, W, ld, stats, g, items[k], k == 0, nd);
    SBF_CHECK_LAUNCH();
  }
#define SBF_NLM_EPI(FT, OT)                                                            \
  nlm_epilogue<FT, OT><<<gpix, bs, 0, st>>>(nd, n_items > 0, n, W, static_cast<const FT*>(f), \
                                            ld, stats, static_cast<OT*>(out), fallback)
  if (!f64 && out_dtype == SBF_F32) SBF_NLM_EPI(float, float);
  else if (!f64) SBF_NLM_EPI(float, double);
  else if (out_dtype == SBF_F32) SBF_NLM_EPI(double, float);
  else SBF_NLM_EPI(double, double);
#undef SBF_NLM_EPI
  SBF_CHECK_LAUNCH();
  sm.release(st);
  SBF_CHECK_CUDA(cudaFreeAsync(planes, st));
  SBF_CHECK_CUDA(cudaFreeAsync(tmp, st));
  SBF_CHECK_CUDA(cudaFreeAsync(nd, st));
  return SBF_OK;
}
