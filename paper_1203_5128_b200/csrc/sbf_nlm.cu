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
  DevBuf<double> planes_b(st), tmp_b(st), nd_b(st);
  SBF_CHECK_CUDA(planes_b.alloc(4 * n));
  SBF_CHECK_CUDA(tmp_b.alloc(4 * n));
  SBF_CHECK_CUDA(nd_b.alloc(2 * n));
  double *planes = planes_b.p, *tmp = tmp_b.p, *nd = nd_b.p;
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
  return SBF_OK;
}

// ---------------------------------------------------------------------------
// Brute-force coarse NLM (reference nlm.py:140-183 direct_nlm): for every
// in-bounds window offset d, w = w_s(d) prod_j K_j(f_j(x+d) - f_j(x)) with
// f_j the replicate-padded copy of f shifted by u_j; out = sum w f / sum w.
// K_j is a Gaussian of width sigma_j or a truncated cosine expansion
// (expansion_range_for), float64.  The test oracle of the shiftable NLM.
// ---------------------------------------------------------------------------
namespace sbf {
namespace {

constexpr int kNlmMaxR = 128, kNlmMaxTerms = 256;
struct DirectNlmParams {
  int64_t H, W, ld;
  int R, p;
  int dy[3], dx[3];
  int kind[3];  // 0 Gaussian, 1 expansion
  double inv[3];  // 1 / (2 sigma^2)
  int K[3];
  double scale[3][kNlmMaxTerms], freq[3][kNlmMaxTerms];
  double tap[2 * kNlmMaxR + 1];
};

template <typename FT, typename OT>
__global__ void __launch_bounds__(256) direct_nlm_kernel(const FT* __restrict__ f,
                                                         OT* __restrict__ out,
                                                         const __grid_constant__ DirectNlmParams q) {
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t y = (int64_t)blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= q.W || y >= q.H) return;
  auto at = [&](int64_t yy, int64_t xx) -> double {
    yy = yy < 0 ? 0 : (yy >= q.H ? q.H - 1 : yy);
    xx = xx < 0 ? 0 : (xx >= q.W ? q.W - 1 : xx);
    return (double)f[yy * q.ld + xx];
  };
  double cj[3];
  for (int j = 0; j < q.p; ++j) cj[j] = at(y + q.dy[j], x + q.dx[j]);
  const int R = q.R;
  const int dy_lo = (int)smax<int64_t>(-R, -y), dy_hi = (int)smin<int64_t>(R, q.H - 1 - y);
  const int dx_lo = (int)smax<int64_t>(-R, -x), dx_hi = (int)smin<int64_t>(R, q.W - 1 - x);
  double num = 0.0, den = 0.0;
  for (int dy = dy_lo; dy <= dy_hi; ++dy) {
    for (int dx = dx_lo; dx <= dx_hi; ++dx) {
      double w = q.tap[dy + R] * q.tap[dx + R];
      if (w == 0.0) continue;
      for (int j = 0; j < q.p; ++j) {
        const double s = at(y + dy + q.dy[j], x + dx + q.dx[j]) - cj[j];
        if (q.kind[j] == 0) {
          w *= exp(-(s * s) * q.inv[j]);
        } else {
          double k = 0.0;
          for (int t = 0; t < q.K[j]; ++t) k += q.scale[j][t] * cos(q.freq[j][t] * s);
          w *= k;
        }
      }
      const double v = (double)f[(y + dy) * q.ld + x + dx];
      num += w * v;
      den += w;
    }
  }
  out[y * q.W + x] = (OT)(den > 0.0 ? num / den : (double)f[y * q.ld + x]);
}

}  // namespace
}  // namespace sbf

extern "C" int sbf_direct_nlm(const void* f, int dtype, int64_t H, int64_t W, int64_t ld, int R,
                              const double* taps, int p, const int32_t* offsets,
                              const int32_t* kinds, const double* sigmas, const int32_t* nterms,
                              const double* scale, const double* freq, void* out, int out_dtype,
                              void* stream) {
  using namespace sbf;
  SBF_REQUIRE(f && out && offsets && kinds, SBF_ERR_INVALID, "null pointer");
  SBF_REQUIRE(dtype == SBF_F32 || dtype == SBF_F64, SBF_ERR_INVALID, "bad dtype");
  SBF_REQUIRE(out_dtype == SBF_F32 || out_dtype == SBF_F64, SBF_ERR_INVALID, "bad out dtype");
  SBF_REQUIRE(H >= 1 && W >= 1 && ld >= W, SBF_ERR_INVALID, "bad image shape");
  SBF_REQUIRE(p >= 1 && p <= 3, SBF_ERR_INVALID, "patch must have 1 to 3 offsets");
  SBF_REQUIRE(R >= 0 && R <= kNlmMaxR, SBF_ERR_UNSUPPORTED, "radius %d outside [0, %d]", R, kNlmMaxR);
  DirectNlmParams* q = new DirectNlmParams();
  q->H = H;
  q->W = W;
  q->ld = ld;
  q->R = R;
  q->p = p;
  int off = 0;
  for (int j = 0; j < p; ++j) {
    q->dy[j] = offsets[2 * j];
    q->dx[j] = offsets[2 * j + 1];
    q->kind[j] = kinds[j];
    if (kinds[j] == 0) {
      if (!(sigmas && sigmas[j] > 0.0)) {
        delete q;
        set_error("Gaussian range kernels need sigma > 0");
        return SBF_ERR_INVALID;
      }
      q->inv[j] = 1.0 / (2.0 * sigmas[j] * sigmas[j]);
    } else {
      const int K = nterms ? nterms[j] : 0;
      if (!(K >= 1 && K <= kNlmMaxTerms && scale && freq)) {
        delete q;
        set_error("expansion range kernels need 1..%d terms", kNlmMaxTerms);
        return SBF_ERR_UNSUPPORTED;
      }
      q->K[j] = K;
      for (int t = 0; t < K; ++t) {
        q->scale[j][t] = scale[off + t];
        q->freq[j][t] = freq[off + t];
      }
      off += K;
    }
  }
  for (int k = 0; k <= 2 * R; ++k) q->tap[k] = taps ? taps[k] : 1.0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const dim3 block(32, 8), grid((unsigned)((W + 31) / 32), (unsigned)((H + 7) / 8));
#define SBF_DN(FT, OT) \
  direct_nlm_kernel<FT, OT><<<grid, block, 0, st>>>(static_cast<const FT*>(f), static_cast<OT*>(out), *q)
  if (dtype == SBF_F32 && out_dtype == SBF_F32) SBF_DN(float, float);
  else if (dtype == SBF_F32) SBF_DN(float, double);
  else if (out_dtype == SBF_F32) SBF_DN(double, float);
  else SBF_DN(double, double);
#undef SBF_DN
  delete q;
  SBF_CHECK_LAUNCH();
  return SBF_OK;
}
