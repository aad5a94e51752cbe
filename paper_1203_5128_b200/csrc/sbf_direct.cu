// K5 — brute-force bilateral filter over the clamped window (reference
// bilateral.py:205-239 `direct_bf` with `gaussian_range`, bilateral.py:88-99,
// and the window weights of spatial.py:197-213: uniform for Box, the outer
// product of sampled Gaussian taps for FirGaussian).
//
// The accuracy oracle at full sizes: O(R^2) per
// pixel, so it is an FP32/MUFU-bound kernel, not a hot path.  One thread per
// output pixel (two rows per thread for ILP); neighbours come straight from
// global memory (warp-coalesced row segments, L1-resident across dx).  The
// spatial weight is folded into the exponent in log2 domain:
//     w_s(dy, dx) exp(-d^2 / (2 sr^2)) = exp2(ly[dy] + lx[dx] - d^2 log2(e) / (2 sr^2))
// (a zero tap gives -inf, i.e. weight 0, as in the reference).  Only in-bounds
// neighbours contribute (the reference's offset_slices), num / den in fp32,
// den <= 0 (impossible with the positive Gaussian) falls back to the input.
// Wide-range (HDR) images run an fp64 twin with the reference's arithmetic.
#include <string.h>

#include "sbf_common.cuh"

namespace sbf {
namespace {

constexpr int kDirectMaxR = 255;

struct DirectParams {
  int64_t H, W, ld;
  int R;
  float c;                      // -log2(e) / (2 sigma_r^2)
  float ltap[2 * kDirectMaxR + 1];  // log2 of the 1-D taps
  double inv;                   // 1 / (2 sigma_r^2)   (fp64 variant)
  double tap[2 * kDirectMaxR + 1];  // the 1-D taps       (fp64 variant)
};

// fp64 twin for wide intensity ranges (HDR): the reference's own arithmetic,
// w = tap[dy] tap[dx] exp(-d^2 / (2 sr^2)), accumulated in float64.
template <typename FT, typename OT>
__global__ void __launch_bounds__(256) direct_kernel_f64(const FT* __restrict__ f,
                                                         OT* __restrict__ out,
                                                         const __grid_constant__ DirectParams p) {
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t y = (int64_t)blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= p.W || y >= p.H) return;
  const int R = p.R;
  const double c = (double)f[y * p.ld + x];
  const int dx_lo = (int)smax<int64_t>(-R, -x), dx_hi = (int)smin<int64_t>(R, p.W - 1 - x);
  const int dy_lo = (int)smax<int64_t>(-R, -y), dy_hi = (int)smin<int64_t>(R, p.H - 1 - y);
  double num = 0.0, den = 0.0;
  for (int dy = dy_lo; dy <= dy_hi; ++dy) {
    const FT* row = f + (y + dy) * p.ld + x;
    const double wy = p.tap[dy + R];
    if (wy == 0.0) continue;
    for (int dx = dx_lo; dx <= dx_hi; ++dx) {
      const double wsp = wy * p.tap[dx + R];
      if (wsp == 0.0) continue;
      const double v = (double)row[dx];
      const double d = v - c;
      const double w = wsp * exp(-(d * d) * p.inv);
      num += w * v;
      den += w;
    }
  }
  out[y * p.W + x] = (OT)(den > 0.0 ? num / den : c);
}

// RPT output rows per thread: every loaded neighbour serves RPT outputs (row
// s of the window serves output k at dy = s - k), 2 RPT independent
// accumulation chains; exp2 by MUFU.EX2 (ex2.approx.ftz).
#ifndef SBF_DIRECT_ROWS
#define SBF_DIRECT_ROWS 4
#endif
constexpr int kDirectRows = SBF_DIRECT_ROWS;

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <typename FT, typename OT>
__global__ void __launch_bounds__(256) direct_kernel(const FT* __restrict__ f, OT* __restrict__ out,
                                                     const __grid_constant__ DirectParams p) {
  constexpr int RPT = kDirectRows;
  __shared__ float lt[2 * kDirectMaxR + 1];
  for (int k = threadIdx.y * blockDim.x + threadIdx.x; k < 2 * p.R + 1; k += blockDim.x * blockDim.y)
    lt[k] = p.ltap[k];
  __syncthreads();
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t y0 = ((int64_t)blockIdx.y * blockDim.y + threadIdx.y) * RPT;
  if (x >= p.W || y0 >= p.H) return;
  const int nr = (int)smin<int64_t>(RPT, p.H - y0);
  const int R = p.R;
  float c[RPT], n[RPT], d[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    c[k] = k < nr ? (float)f[(y0 + k) * p.ld + x] : 0.f;
    n[k] = 0.f;
    d[k] = 0.f;
  }
  const int dx_lo = (int)smax<int64_t>(-R, -x), dx_hi = (int)smin<int64_t>(R, p.W - 1 - x);
  // rows y0 + s for s in [-R, R + RPT - 1]
  const int s_lo = (int)smax<int64_t>(-R, -y0), s_hi = (int)smin<int64_t>(R + nr - 1, p.H - 1 - y0);
  for (int s = s_lo; s <= s_hi; ++s) {
    const FT* row = f + (y0 + s) * p.ld + x;
    float ly[RPT];
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int dy = s - k;
      ly[k] = (k < nr && dy >= -R && dy <= R) ? lt[dy + R] : -INFINITY;
    }
#pragma unroll 2
    for (int dx = dx_lo; dx <= dx_hi; ++dx) {
      const float v = (float)row[dx];
      const float lx = lt[dx + R];
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        const float e = v - c[k];
        const float w = fast_exp2(fmaf(e * e, p.c, ly[k] + lx));
        n[k] = fmaf(w, v, n[k]);
        d[k] += w;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < RPT; ++k)
    if (k < nr) out[(y0 + k) * p.W + x] = (OT)(d[k] > 0.f ? n[k] / d[k] : c[k]);
}

// truncated raised-cosine expansion as the range kernel (reference
// bilateral.py:101-103 expansion_range): K(s) = sum_k scale_k cos(w_k s)
// over the folded terms, float64 (the exact-shiftability oracle)
constexpr int kDirectMaxTerms = 1024;
struct DirectTerms {
  int K;
  double scale[kDirectMaxTerms];
  double freq[kDirectMaxTerms];
};

template <typename FT, typename OT>
__global__ void __launch_bounds__(256) direct_terms_kernel(const FT* __restrict__ f,
                                                           OT* __restrict__ out,
                                                           const __grid_constant__ DirectParams p,
                                                           const DirectTerms* __restrict__ tt) {
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t y = (int64_t)blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= p.W || y >= p.H) return;
  const int R = p.R;
  const double c = (double)f[y * p.ld + x];
  const int dx_lo = (int)smax<int64_t>(-R, -x), dx_hi = (int)smin<int64_t>(R, p.W - 1 - x);
  const int dy_lo = (int)smax<int64_t>(-R, -y), dy_hi = (int)smin<int64_t>(R, p.H - 1 - y);
  const int K = tt->K;
  double num = 0.0, den = 0.0;
  for (int dy = dy_lo; dy <= dy_hi; ++dy) {
    const FT* row = f + (y + dy) * p.ld + x;
    const double wy = p.tap[dy + R];
    if (wy == 0.0) continue;
    for (int dx = dx_lo; dx <= dx_hi; ++dx) {
      const double wsp = wy * p.tap[dx + R];
      if (wsp == 0.0) continue;
      const double v = (double)row[dx];
      const double d = v - c;
      double k = 0.0;
      for (int t = 0; t < K; ++t) k += tt->scale[t] * cos(tt->freq[t] * d);
      const double w = wsp * k;
      num += w * v;
      den += w;
    }
  }
  out[y * p.W + x] = (OT)(den > 0.0 ? num / den : c);
}

template <typename FT, typename OT>
int launch_direct(const void* f, void* out, const DirectParams& p, int f64math, cudaStream_t st) {
  dim3 block(32, 8);
  if (f64math) {
    dim3 grid((unsigned)((p.W + 31) / 32), (unsigned)((p.H + 7) / 8));
    direct_kernel_f64<FT, OT><<<grid, block, 0, st>>>(static_cast<const FT*>(f),
                                                      static_cast<OT*>(out), p);
  } else {
    dim3 grid((unsigned)((p.W + 31) / 32), (unsigned)((p.H + 8 * kDirectRows - 1) / (8 * kDirectRows)));
    direct_kernel<FT, OT><<<grid, block, 0, st>>>(static_cast<const FT*>(f), static_cast<OT*>(out),
                                                  p);
  }
  SBF_CHECK_LAUNCH();
  return SBF_OK;
}

}  // namespace
}  // namespace sbf

extern "C" int sbf_direct_bf(const void* f, int dtype, int64_t H, int64_t W, int64_t ld, int R,
                             const double* taps, double sigma_r, int precision, void* out,
                             int out_dtype, void* stream) {
  using namespace sbf;
  SBF_REQUIRE(f && out, SBF_ERR_INVALID, "null pointer");
  SBF_REQUIRE(dtype == SBF_F32 || dtype == SBF_F64, SBF_ERR_INVALID, "bad dtype");
  SBF_REQUIRE(out_dtype == SBF_F32 || out_dtype == SBF_F64, SBF_ERR_INVALID, "bad out dtype");
  SBF_REQUIRE(H >= 1 && W >= 1 && ld >= W, SBF_ERR_INVALID, "bad image shape");
  SBF_REQUIRE(R >= 0 && R <= kDirectMaxR, SBF_ERR_UNSUPPORTED, "direct_bf radius %d outside [0, %d]",
              R, kDirectMaxR);
  SBF_REQUIRE(sigma_r > 0.0, SBF_ERR_INVALID, "sigma_r must be positive");
  DirectParams p;
  memset(&p, 0, sizeof(p));
  p.H = H;
  p.W = W;
  p.ld = ld;
  p.R = R;
  SBF_REQUIRE(precision == SBF_PREC_FP32 || precision == SBF_PREC_HDR, SBF_ERR_INVALID,
              "bad precision mode");
  p.c = (float)(-1.4426950408889634 / (2.0 * sigma_r * sigma_r));
  p.inv = 1.0 / (2.0 * sigma_r * sigma_r);
  for (int k = 0; k <= 2 * R; ++k) {
    const double t = taps ? taps[k] : 1.0;
    SBF_REQUIRE(t >= 0.0 && t == t, SBF_ERR_INVALID, "spatial taps must be non-negative");
    p.ltap[k] = t > 0.0 ? (float)log2(t) : -INFINITY;
    p.tap[k] = t;
  }
  const int f64math = precision == SBF_PREC_HDR;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == SBF_F32)
    return out_dtype == SBF_F32 ? launch_direct<float, float>(f, out, p, f64math, st)
                                : launch_direct<float, double>(f, out, p, f64math, st);
  return out_dtype == SBF_F32 ? launch_direct<double, float>(f, out, p, f64math, st)
                              : launch_direct<double, double>(f, out, p, f64math, st);
}

extern "C" int sbf_direct_bf_expansion(const void* f, int dtype, int64_t H, int64_t W, int64_t ld,
                                       int R, const double* taps, const double* scale,
                                       const double* freq, int K, void* out, int out_dtype,
                                       void* stream) {
  using namespace sbf;
  SBF_REQUIRE(f && out && scale && freq, SBF_ERR_INVALID, "null pointer");
  SBF_REQUIRE(dtype == SBF_F32 || dtype == SBF_F64, SBF_ERR_INVALID, "bad dtype");
  SBF_REQUIRE(out_dtype == SBF_F32 || out_dtype == SBF_F64, SBF_ERR_INVALID, "bad out dtype");
  SBF_REQUIRE(H >= 1 && W >= 1 && ld >= W, SBF_ERR_INVALID, "bad image shape");
  SBF_REQUIRE(R >= 0 && R <= kDirectMaxR, SBF_ERR_UNSUPPORTED, "direct_bf radius %d outside [0, %d]",
              R, kDirectMaxR);
  SBF_REQUIRE(K >= 1 && K <= kDirectMaxTerms, SBF_ERR_UNSUPPORTED, "expansion of %d terms", K);
  DirectParams p;
  memset(&p, 0, sizeof(p));
  p.H = H;
  p.W = W;
  p.ld = ld;
  p.R = R;
  for (int k = 0; k <= 2 * R; ++k) {
    const double t = taps ? taps[k] : 1.0;
    SBF_REQUIRE(t >= 0.0 && t == t, SBF_ERR_INVALID, "spatial taps must be non-negative");
    p.tap[k] = t;
  }
  DirectTerms ht;
  ht.K = K;
  for (int k = 0; k < K; ++k) {
    ht.scale[k] = scale[k];
    ht.freq[k] = freq[k];
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DevBuf<DirectTerms> dt_b(st);
  SBF_CHECK_CUDA(dt_b.alloc(1));
  DirectTerms* dt = dt_b.p;
  SBF_CHECK_CUDA(cudaMemcpyAsync(dt, &ht, sizeof(DirectTerms), cudaMemcpyHostToDevice, st));
  const dim3 block(32, 8), grid((unsigned)((W + 31) / 32), (unsigned)((H + 7) / 8));
#define SBF_DT(FT, OT)                                                                        \
  direct_terms_kernel<FT, OT><<<grid, block, 0, st>>>(static_cast<const FT*>(f),              \
                                                      static_cast<OT*>(out), p, dt)
  if (dtype == SBF_F32 && out_dtype == SBF_F32) SBF_DT(float, float);
  else if (dtype == SBF_F32) SBF_DT(float, double);
  else if (out_dtype == SBF_F32) SBF_DT(double, float);
  else SBF_DT(double, double);
#undef SBF_DT
  SBF_CHECK_LAUNCH();
  // the pageable source was staged by cudaMemcpyAsync before it returned
  return SBF_OK;
}

// Brute-force local range (reference maxfilter.py:64-82 `brute_force_T`):
// max over every pixel x and every offset y with |y|_inf <= R inside the image
// of |f(x+y) - f(x)|, in float64.  O(R^2) per pixel and independent of K1's
// separable max filter, so it cross-checks compute_T (the paper's
// Proposition 1 says both are equal).  One thread per pixel, block maximum,
// one 64-bit atomicMax of the order-preserving bit image per block.
namespace sbf {
template <typename T>
__global__ void brute_T_kernel(const T* __restrict__ f, int64_t H, int64_t W, int64_t ld, int R,
                               unsigned long long* __restrict__ best) {
  __shared__ unsigned long long s_best[8];
  double m = 0.0;
  const int64_t n = H * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = i / W, x = i - y * W;
    const double c = (double)f[y * ld + x];
    const int64_t y0 = y - R < 0 ? 0 : y - R, y1 = y + R >= H ? H - 1 : y + R;
    const int64_t x0 = x - R < 0 ? 0 : x - R, x1 = x + R >= W ? W - 1 : x + R;
    for (int64_t yy = y0; yy <= y1; ++yy)
      for (int64_t xx = x0; xx <= x1; ++xx) m = fmax(m, fabs((double)f[yy * ld + xx] - c));
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s_best[threadIdx.x >> 5] = ord_bits(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long b = s_best[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) b = b > s_best[w] ? b : s_best[w];
    atomicMax(best, b);
  }
}
}  // namespace sbf

extern "C" int sbf_brute_force_T(const void* f, int dtype, int64_t H, int64_t W, int64_t ld, int R,
                                 double* T_out, void* stream) {
  using namespace sbf;
  SBF_REQUIRE(f && T_out && H >= 1 && W >= 1 && ld >= W && R >= 0 &&
                  (dtype == SBF_F32 || dtype == SBF_F64),
              SBF_ERR_INVALID, "bad brute_force_T arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DevBuf<unsigned long long> best(st);
  SBF_CHECK_CUDA(best.alloc(1));
  const unsigned long long zero = 0x8000000000000000ull;  // ord_bits(+0.0)
  SBF_CHECK_CUDA(cudaMemcpyAsync(best.p, &zero, sizeof(zero), cudaMemcpyHostToDevice, st));
  const int threads = 256;
  const unsigned blocks = (unsigned)smin<int64_t>((H * W + threads - 1) / threads, 148 * 16);
  if (dtype == SBF_F32)
    brute_T_kernel<float><<<blocks, threads, 0, st>>>(static_cast<const float*>(f), H, W, ld, R, best.p);
  else
    brute_T_kernel<double><<<blocks, threads, 0, st>>>(static_cast<const double*>(f), H, W, ld, R, best.p);
  SBF_CHECK_LAUNCH();
  unsigned long long b = 0;
  SBF_CHECK_CUDA(cudaMemcpyAsync(&b, best.p, sizeof(b), cudaMemcpyDeviceToHost, st));
  SBF_CHECK_CUDA(cudaStreamSynchronize(st));
  // ord_value on the host: the maximum is >= +0.0, so the sign bit is set
  b &= 0x7fffffffffffffffull;
  double t;
  memcpy(&t, &b, sizeof(t));
  *T_out = t;
  return SBF_OK;
}
