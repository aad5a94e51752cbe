// Dual (direct) evaluation of the shiftable filter for untruncated plans.
//
// With M = 0 the retained raised-cosine expansion sums to the closed form
//     sum_n C(N,n)/2^N cos((2n-N) gamma s) = cos(gamma s)^N
// (binomial theorem; reference kernels.py:198-227 — terms whose fp64 weight
// underflows contribute < 1e-300).  By linearity of the smoother, the
// reference's num/den (bilateral.py:140-164) are then exactly
//     num(x) = sum_y A_r(x_r, y_r) A_c(x_c, y_c) cos(gamma (f(y)-f(x)))^N f(y)
// (den likewise without f(y)), where A_r / A_c are the 1-D effective weights
// of the spatial mode — `passes` extended-box passes with clamped
// renormalisation (spatial.py:108-139) or the box filter (spatial.py:65-78);
// rows and columns commute, so the 2-D weight is their product.
//
// That costs (2S+1)^2 taps per pixel instead of K terms of four smoothings,
// so for high-order plans (HDR, config 3: N = 2463, K = 1232, S = 24) it is
// the cheaper exact evaluation; the dispatcher picks it by a cost estimate.
// Everything in fp64: for integer-valued images (16-bit HDR) cos(gamma s)^N
// is tabulated per integer difference; otherwise cos(gamma s) comes from
// per-pixel phasors (cos gamma f, sin gamma f) by the angle-difference
// identity and the power by square-and-multiply (relative error ~N ulp).
#include <math.h>

#include <vector>

#include "sbf_common.cuh"

#ifndef SBF_DUAL_PARTIALS
#define SBF_DUAL_PARTIALS 8  // independent partial sums per row of taps (2: 11.65, 4: 11.56, 8: 11.42 ms)
#endif

namespace sbf {
namespace {

// per-pixel (cos gamma f, sin gamma f)
template <typename FT>
__global__ void phasor_kernel(const FT* __restrict__ f, int64_t H, int64_t W, int64_t ld,
                              const sbf_plan* __restrict__ plan, double2* __restrict__ P) {
  const double g = plan->gamma;
  const int64_t n = H * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = i / W, x = i - y * W;
    double s, c;
    sincos(g * (double)f[y * ld + x], &s, &c);
    P[i] = make_double2(c, s);
  }
}

__device__ __forceinline__ double pow_n(double c, int n) {
  double r = 1.0;
  while (n) {
    if (n & 1) r *= c;
    c *= c;
    n >>= 1;
  }
  return r;
}

template <typename FT, typename OT>
__global__ void __launch_bounds__(256) dual_kernel(const FT* __restrict__ f, int64_t H, int64_t W,
                                                   int64_t ld, int64_t out_lo, int64_t out_hi,
                                                   int S, const double* __restrict__ Wr,
                                                   const double* __restrict__ Wc,
                                                   const double2* __restrict__ P,
                                                   const sbf_plan* __restrict__ plan,
                                                   OT* __restrict__ out,
                                                   unsigned long long* __restrict__ fallback) {
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t yo = (int64_t)blockIdx.y * blockDim.y + threadIdx.y;
  const int64_t y = out_lo + yo;
  bool bad = false;
  if (x < W && y < out_hi) {
    const int N = plan->N;
    const int T = 2 * S + 1;
    const double2 px = P[y * W + x];
    const double* wr = Wr + yo * T;
    const double* wc = Wc + x * T;
    const int dy_lo = (int)smax<int64_t>(-S, -y), dy_hi = (int)smin<int64_t>(S, H - 1 - y);
    const int dx_lo = (int)smax<int64_t>(-S, -x), dx_hi = (int)smin<int64_t>(S, W - 1 - x);
    double num = 0.0, den = 0.0;
    for (int dy = dy_lo; dy <= dy_hi; ++dy) {
      const double a = wr[dy + S];
      if (a == 0.0) continue;
      const double2* prow = P + (y + dy) * W + x;
      const FT* frow = f + (y + dy) * ld + x;
      for (int dx = dx_lo; dx <= dx_hi; ++dx) {
        const double2 q = prow[dx];
        double c = fma(q.x, px.x, q.y * px.y);  // cos(gamma (f(y) - f(x)))
        c = c > 1.0 ? 1.0 : (c < -1.0 ? -1.0 : c);
        const double k = pow_n(c, N);  // odd N keeps the sign, as the expansion does
        const double w = a * wc[dx + S] * k;
        num = fma(w, (double)frow[dx], num);
        den += w;
      }
    }
    bad = !(den > 0.0);  // bilateral.py:244
    out[yo * W + x] = (OT)(bad ? (double)f[y * ld + x] : num / den);
  }
  const unsigned m = __ballot_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(fallback, (unsigned long long)__popc(m));
}

// Integer-valued images (e.g. 16-bit HDR): the kernel depends on the integer
// difference only, so cos(gamma s)^N is tabulated once for s in [0, smax]
// (even in s) and every tap is one table read.
template <typename FT>
__global__ void integral_check(const FT* __restrict__ f, int64_t H, int64_t W, int64_t ld,
                               int* __restrict__ non_integer) {
  const int64_t n = H * W;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = i / W, x = i - y * W;
    const double v = (double)f[y * ld + x];
    bad |= !(v == rint(v) && fabs(v) <= 16777216.0);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(non_integer, 1);
}

__global__ void kernel_table(const sbf_plan* __restrict__ plan, int64_t smax,
                             double* __restrict__ lut) {
  const double g = plan->gamma;
  const int N = plan->N;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s <= smax;
       s += (int64_t)gridDim.x * blockDim.x)
    lut[s] = pow_n(cos(g * (double)s), N);
}

// One CTA per 32 x 8 output tile; the (8 + 2S) x (32 + 2S) input tile and the
// tile's column / row weights are staged in shared memory, so each tap is one
// shared-memory read of f, one weight read (broadcast-free layout [dx][col])
// and one table gather.
template <typename FT, typename OT>
__global__ void __launch_bounds__(256) dual_lut_kernel(
    const FT* __restrict__ f, int64_t H, int64_t W, int64_t ld, int64_t out_lo, int64_t out_hi,
    int S, const double* __restrict__ Wr, const double* __restrict__ Wc,
    const double* __restrict__ lut, OT* __restrict__ out, unsigned long long* __restrict__ fallback) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int T = 2 * S + 1;
  const int IW = 32 + 2 * S, IH = 8 + 2 * S;
  double* wcs = reinterpret_cast<double*>(smem_raw);  // [T][32]
  double* wrs = wcs + T * 32;                           // [8][T]
  FT* fin = reinterpret_cast<FT*>(wrs + 8 * T);         // [IH][IW]
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int64_t x0 = (int64_t)blockIdx.x * 32, yo0 = (int64_t)blockIdx.y * 8;
  const int64_t y0 = out_lo + yo0;
  for (int k = tid; k < T * 32; k += 256) {
    const int d = k / 32, c = k - d * 32;
    wcs[k] = x0 + c < W ? Wc[(x0 + c) * T + d] : 0.0;
  }
  for (int k = tid; k < 8 * T; k += 256) {
    const int r = k / T, d = k - r * T;
    wrs[k] = y0 + r < out_hi ? Wr[(yo0 + r) * T + d] : 0.0;
  }
  for (int k = tid; k < IH * IW; k += 256) {
    const int iy = k / IW, ix = k - iy * IW;
    int64_t gy = y0 - S + iy, gx = x0 - S + ix;
    // outside the buffer: weight 0 there (the tables hold 0 outside the image)
    gy = gy < 0 ? 0 : (gy >= H ? H - 1 : gy);
    gx = gx < 0 ? 0 : (gx >= W ? W - 1 : gx);
    fin[k] = f[gy * ld + gx];
  }
  __syncthreads();
  const int64_t x = x0 + tx, y = y0 + ty;
  bool bad = false;
  if (x < W && y < out_hi) {
    const FT fx = fin[(ty + S) * IW + tx + S];
    const int dy_lo = (int)smax<int64_t>(-S, -y), dy_hi = (int)smin<int64_t>(S, H - 1 - y);
    const int dx_lo = (int)smax<int64_t>(-S, -x), dx_hi = (int)smin<int64_t>(S, W - 1 - x);
    double num = 0.0, den = 0.0;
    for (int dy = dy_lo; dy <= dy_hi; ++dy) {
      const double a = wrs[ty * T + dy + S];
      if (a == 0.0) continue;
      const FT* frow = fin + (ty + S + dy) * IW + tx + S;
      // independent partial sums: the fp64 accumulation chains, not the
      // gathers, bounded the loop (one chain: 12.3 ms, four: 11.5 ms, config 3)
      constexpr int NP = SBF_DUAL_PARTIALS;
      double rn[NP], rd[NP];
#pragma unroll
      for (int u = 0; u < NP; ++u) rn[u] = rd[u] = 0.0;
      int dx = dx_lo;
      for (; dx + NP - 1 <= dx_hi; dx += NP) {
#pragma unroll
        for (int u = 0; u < NP; ++u) {
          const FT v = frow[dx + u];
          const int sd = (int)(v - fx);  // exact: integer samples below 2^24
          const double w = wcs[(dx + u + S) * 32 + tx] * __ldg(lut + (sd < 0 ? -sd : sd));
          rn[u] = fma(w, (double)v, rn[u]);
          rd[u] += w;
        }
      }
      for (; dx <= dx_hi; ++dx) {
        const FT v = frow[dx];
        const int sd = (int)(v - fx);
        const double w = wcs[(dx + S) * 32 + tx] * __ldg(lut + (sd < 0 ? -sd : sd));
        rn[0] = fma(w, (double)v, rn[0]);
        rd[0] += w;
      }
#pragma unroll
      for (int u = 1; u < NP; ++u) {
        rn[0] += rn[u];
        rd[0] += rd[u];
      }
      num = fma(a, rn[0], num);
      den = fma(a, rd[0], den);
    }
    bad = !(den > 0.0);  // bilateral.py:244
    out[(y - out_lo) * W + x] = (OT)(bad ? (double)fx : num / den);
  }
  const unsigned m = __ballot_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(fallback, (unsigned long long)__popc(m));
}

// Row i of the 1-D effective smoothing matrix on an axis of length n:
// A = B^passes with B[k][j] = w(|k-j|) / cnt(k) (w = 1 inside the radius,
// alpha at r+1, samples outside the axis dropped), written as weights of
// samples i-S .. i+S.
void axis_row(int64_t n, int64_t i, int r, double alpha, int passes, int S, double* out) {
  const int T = 2 * S + 1;
  std::vector<double> u(T, 0.0), v(T, 0.0);
  u[S] = 1.0;  // index t <-> sample i - S + t
  const int e = alpha > 0.0 ? r + 1 : r;
  for (int p = 0; p < passes; ++p) {
    std::fill(v.begin(), v.end(), 0.0);
    for (int t = 0; t < T; ++t) {
      if (u[t] == 0.0) continue;
      const int64_t k = i - S + t;  // output sample of this pass
      if (k < 0 || k >= n) continue;
      double cnt = 0.0;
      for (int d = -e; d <= e; ++d) {
        const int64_t j = k + d;
        if (j < 0 || j >= n) continue;
        cnt += (d >= -r && d <= r) ? 1.0 : alpha;
      }
      for (int d = -e; d <= e; ++d) {
        const int64_t j = k + d;
        const int64_t tj = t + d;
        if (j < 0 || j >= n || tj < 0 || tj >= T) continue;
        v[tj] += u[t] * ((d >= -r && d <= r) ? 1.0 : alpha) / cnt;
      }
    }
    u.swap(v);
  }
  for (int t = 0; t < T; ++t) out[t] = u[t];
}

}  // namespace

int dual_support(const sbf_spatial& sp) {
  if (sp.mode == SBF_SPATIAL_BOX) return sp.r;
  return sp.passes * (sp.r + (sp.alpha > 0.0 ? 1 : 0));
}

// cost model (measured on B200, fp64): term sweeps ~0.17 ns per pixel-term,
// dual form ~5.5 ps per pixel-tap with the power, less with the table
bool dual_preferred(const FilterLaunch& a, const sbf_plan& plan) {
  if (plan.status != SBF_OK || plan.M != 0 || plan.K_eval < 1) return false;
  if (a.precision != SBF_PREC_HDR) return false;
  const double S = dual_support(a.sp);
  const double taps = (2 * S + 1) * (2 * S + 1);
  return taps * 5.5e-3 < (double)plan.K_eval * 0.17;
}

int launch_dual_direct(const FilterLaunch& a, const sbf_plan& plan) {
  cudaStream_t st = a.stream;
  const int S = dual_support(a.sp);
  const int T = 2 * S + 1;
  const int passes = a.sp.mode == SBF_SPATIAL_BOX ? 1 : a.sp.passes;
  const double alpha = a.sp.mode == SBF_SPATIAL_BOX ? 0.0 : a.sp.alpha;
  const int64_t rows_out = a.out_hi - a.out_lo;
  // the weights of sample j in output i depend on the global axis (row0, img_H);
  // the tables of the last geometry stay on the device (per thread): building
  // them is ~0.7 ms of host work plus two pageable copies per call
  struct WeightTables {
    int dev = -1, r = 0, passes = 0, S = 0;
    int64_t rows_out = 0, g0 = 0, img_H = 0, W = 0;
    double alpha = 0.0;
    double *Wr = nullptr, *Wc = nullptr;
  };
  static thread_local WeightTables wt;
  int dev = 0;
  SBF_CHECK_CUDA(cudaGetDevice(&dev));
  const int64_t g0 = a.row0 + a.out_lo;
  if (!(wt.Wr && wt.dev == dev && wt.r == a.sp.r && wt.passes == passes && wt.S == S &&
        wt.rows_out == rows_out && wt.g0 == g0 && wt.img_H == a.img_H && wt.W == a.W &&
        wt.alpha == alpha)) {
    // the interior row is shared by every position at least 2S from both ends
    std::vector<double> hr((size_t)rows_out * T), hc((size_t)a.W * T);
    std::vector<double> interior_r(T), interior_c(T);
    const int64_t mid_r = a.img_H / 2, mid_c = a.W / 2;
    axis_row(a.img_H, mid_r, a.sp.r, alpha, passes, S, interior_r.data());
    axis_row(a.W, mid_c, a.sp.r, alpha, passes, S, interior_c.data());
    for (int64_t yo = 0; yo < rows_out; ++yo) {
      const int64_t g = g0 + yo;
      if (g >= 2 * S && g < a.img_H - 2 * S)
        std::copy(interior_r.begin(), interior_r.end(), hr.begin() + yo * T);
      else
        axis_row(a.img_H, g, a.sp.r, alpha, passes, S, hr.data() + yo * T);
    }
    for (int64_t x = 0; x < a.W; ++x) {
      if (x >= 2 * S && x < a.W - 2 * S)
        std::copy(interior_c.begin(), interior_c.end(), hc.begin() + x * T);
      else
        axis_row(a.W, x, a.sp.r, alpha, passes, S, hc.data() + x * T);
    }
    // replacing a geometry: cudaFree waits for any kernel still reading the
    // previous tables
    if (wt.Wr) cudaFree(wt.Wr);
    if (wt.Wc) cudaFree(wt.Wc);
    wt = WeightTables();
    SBF_CHECK_CUDA(cudaMalloc(reinterpret_cast<void**>(&wt.Wr), sizeof(double) * hr.size()));
    SBF_CHECK_CUDA(cudaMalloc(reinterpret_cast<void**>(&wt.Wc), sizeof(double) * hc.size()));
    SBF_CHECK_CUDA(cudaMemcpy(wt.Wr, hr.data(), sizeof(double) * hr.size(), cudaMemcpyHostToDevice));
    SBF_CHECK_CUDA(cudaMemcpy(wt.Wc, hc.data(), sizeof(double) * hc.size(), cudaMemcpyHostToDevice));
    wt.dev = dev;
    wt.r = a.sp.r;
    wt.passes = passes;
    wt.S = S;
    wt.rows_out = rows_out;
    wt.g0 = g0;
    wt.img_H = a.img_H;
    wt.W = a.W;
    wt.alpha = alpha;
  }
  DevBuf<double2> P_b(st);
  const double *Wr = wt.Wr, *Wc = wt.Wc;
  const unsigned gpix = (unsigned)smin<int64_t>((a.H * a.W + 255) / 256, 148 * 16);
  const dim3 tb(32, 8), grid((unsigned)((a.W + 31) / 32), (unsigned)((rows_out + 7) / 8));

  // integer-valued image with a modest range: tabulated kernel
  DevBuf<int> flag_b(st);
  SBF_CHECK_CUDA(flag_b.alloc(1));
  int* flag = flag_b.p;
  SBF_CHECK_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
  if (a.dtype == SBF_F32)
    integral_check<float><<<gpix, 256, 0, st>>>(static_cast<const float*>(a.f), a.H, a.W, a.ld, flag);
  else
    integral_check<double><<<gpix, 256, 0, st>>>(static_cast<const double*>(a.f), a.H, a.W, a.ld,
                                                  flag);
  SBF_CHECK_LAUNCH();
  int non_integer = 1;
  double st_host[8];
  SBF_CHECK_CUDA(cudaMemcpyAsync(&non_integer, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  SBF_CHECK_CUDA(cudaMemcpyAsync(st_host, a.stats, sizeof(st_host), cudaMemcpyDeviceToHost, st));
  SBF_CHECK_CUDA(cudaStreamSynchronize(st));
  const double span = st_host[2] - st_host[1];
  if (!non_integer && span >= 0.0 && span <= 4194304.0) {
    const int64_t smax_v = (int64_t)span;
    DevBuf<double> lut_b(st);
    SBF_CHECK_CUDA(lut_b.alloc(smax_v + 1));
    double* lut = lut_b.p;
    kernel_table<<<(unsigned)smin<int64_t>((smax_v + 256) / 256, 148 * 8), 256, 0, st>>>(
        a.plan, smax_v, lut);
#define SBF_DUAL_LUT(FT, OT)                                                                     \
  do {                                                                                           \
    const size_t smem = sizeof(double) * (size_t)(2 * S + 1) * 40 +                              \
                        sizeof(FT) * (size_t)(8 + 2 * S) * (32 + 2 * S);                         \
    SBF_CHECK_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(dual_lut_kernel<FT, OT>), smem)); \
    dual_lut_kernel<FT, OT><<<grid, tb, smem, st>>>(static_cast<const FT*>(a.f), a.H, a.W, a.ld, \
                                               a.out_lo, a.out_hi, S, Wr, Wc, lut,               \
                                               static_cast<OT*>(a.out), a.fallback); \
  } while (0)
    if (a.dtype == SBF_F32 && a.out_dtype == SBF_F32) SBF_DUAL_LUT(float, float);
    else if (a.dtype == SBF_F32) SBF_DUAL_LUT(float, double);
    else if (a.out_dtype == SBF_F32) SBF_DUAL_LUT(double, float);
    else SBF_DUAL_LUT(double, double);
#undef SBF_DUAL_LUT
    SBF_CHECK_LAUNCH();
    return SBF_OK;
  }
  SBF_CHECK_CUDA(P_b.alloc((size_t)(a.H * a.W)));
  double2* P = P_b.p;
#define SBF_DUAL(FT, OT)                                                                         \
  do {                                                                                           \
    phasor_kernel<FT><<<gpix, 256, 0, st>>>(static_cast<const FT*>(a.f), a.H, a.W, a.ld, a.plan, \
                                            P);                                                  \
    dual_kernel<FT, OT><<<grid, tb, 0, st>>>(static_cast<const FT*>(a.f), a.H, a.W, a.ld,        \
                                             a.out_lo, a.out_hi, S, Wr, Wc, P, a.plan,           \
                                             static_cast<OT*>(a.out), a.fallback);               \
  } while (0)
  if (a.dtype == SBF_F32 && a.out_dtype == SBF_F32) SBF_DUAL(float, float);
  else if (a.dtype == SBF_F32) SBF_DUAL(float, double);
  else if (a.out_dtype == SBF_F32) SBF_DUAL(double, float);
  else SBF_DUAL(double, double);
#undef SBF_DUAL
  SBF_CHECK_LAUNCH();
  return SBF_OK;
}

}  // namespace sbf
