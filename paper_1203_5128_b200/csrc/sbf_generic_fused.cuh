// Fused fp64 extended-box cascade for the generic / HDR path.
//
// colpass_f64<R, PASSES>: one thread per (plane, column, segment) streams a
// segment of its column (plus the cascade warm-up of PASSES*(r+1) samples on
// each side) and applies all passes with the same O(1) recurrence as K3, in
// float64, ring buffers in registers.  Consecutive threads own consecutive
// columns, so every load/store is coalesced.  Normalisation uses a per-
// position factor table (cnt_int/cnt(pos), 0 outside the image) applied on
// read; the delay lines hold raw accumulators (see sbf_terms.cuh).
// The row direction is handled by running the same kernel on transposed
// planes.
#pragma once

#include "sbf_common.cuh"

namespace sbf {

template <int R, int PASSES, bool BORDER>
__device__ __forceinline__ void colpass_run(const double* __restrict__ x, double* __restrict__ y,
                                            int64_t n_stream, int64_t n_cols, int64_t o_lo,
                                            int64_t o_hi, const double* __restrict__ gt0, double a,
                                            double b) {
  constexpr int D = R + 1, L = 2 * R + 3, HALO = PASSES * D;
  double dl[PASSES][L];
  double vlast = 0.0;
#pragma unroll
  for (int p = 0; p < PASSES; ++p)
#pragma unroll
    for (int j = 0; j < L; ++j) dl[p][j] = 0.0;
  const int64_t s0 = o_lo - HALO, s1 = o_hi + HALO;
  for (int64_t base = s0; base < s1; base += L) {
#pragma unroll
    for (int J = 0; J < L; ++J) {
      const int64_t s = base + J;
      if (s >= s1) break;
      // ring slot of step s is (s - s0) mod L == J
      const double xin = (!BORDER || (s >= 0 && s < n_stream)) ? x[s * n_cols] : 0.0;
      const int JM1 = (J + L - 1) % L, JO1 = (J + 1) % L;
      double acc;
      {
        const double prev = dl[0][JM1], o1 = dl[0][JO1], o2 = dl[0][J];
        const double accp = (PASSES > 1) ? dl[PASSES > 1 ? 1 : 0][JM1] : vlast;
        dl[0][J] = xin;
        acc = fma(b, xin - o2, fma(a, prev - o1, accp));
      }
#pragma unroll
      for (int p = 1; p < PASSES; ++p) {
        double xt = acc, xp = dl[p][JM1], x1 = dl[p][JO1], x2 = dl[p][J];
        if (BORDER) {
          const double* gp = gt0 + (s - p * D);
          xt *= gp[0];
          xp *= gp[-1];
          x1 *= gp[-2 * D];
          x2 *= gp[-2 * D - 1];
        }
        const double accp = (p + 1 < PASSES) ? dl[(p + 1 < PASSES) ? p + 1 : p][JM1] : vlast;
        dl[p][J] = acc;
        acc = fma(b, xt - x2, fma(a, xp - x1, accp));
      }
      vlast = acc;
      const int64_t o = s - HALO;
      if (o >= o_lo && o < o_hi) y[o * n_cols] = BORDER ? acc * gt0[o] : acc;
    }
  }
}

template <int R, int PASSES>
__global__ void __launch_bounds__(128) colpass_f64(const double* __restrict__ in,
                                                   double* __restrict__ out, int nplanes,
                                                   int64_t n_stream, int64_t n_cols,
                                                   int64_t seg, const double* __restrict__ g,
                                                   int64_t pos0, int64_t n_global, double a,
                                                   double b) {
  constexpr int D = R + 1, HALO = PASSES * D;
  const int64_t nseg = (n_stream + seg - 1) / seg;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)nplanes * n_cols * nseg) return;
  const int64_t col = id % n_cols;
  const int64_t rest = id / n_cols;
  const int64_t sg = rest % nseg;
  const int64_t pl = rest / nseg;
  const double* x = in + pl * n_stream * n_cols + col;
  double* y = out + pl * n_stream * n_cols + col;
  const int64_t o_lo = sg * seg, o_hi = smin<int64_t>(n_stream, o_lo + seg);
  const double* gt0 = g + (HALO + 2 * D + 2);  // table index = position + pad
  // interior segment: every position the cascade touches is in the buffer
  // and has factor 1 (D away from the true image edges)
  const int64_t lo = o_lo - HALO - (PASSES + 2) * D - 2, hi = o_hi + HALO;
  const bool interior = lo >= 0 && hi <= n_stream && pos0 + lo >= D && pos0 + hi <= n_global - D;
  if (interior)
    colpass_run<R, PASSES, false>(x, y, n_stream, n_cols, o_lo, o_hi, gt0, a, b);
  else
    colpass_run<R, PASSES, true>(x, y, n_stream, n_cols, o_lo, o_hi, gt0, a, b);
}

// normalisation factor table for an axis: positions [-(HALO+2D+2), n + HALO + 2D + 2)
__global__ void gfactor_table(double* g, int64_t n_stream, int64_t pos0, int64_t n_global, int r,
                              double alpha, int pad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_stream + 2 * pad) return;
  const int64_t pos = pos0 + (i - pad);
  double v = 0.0;
  if (pos >= 0 && pos < n_global) {
    const int64_t lo = pos - r < 0 ? 0 : pos - r;
    const int64_t hi = pos + r > n_global - 1 ? n_global - 1 : pos + r;
    double cnt = (double)(hi - lo + 1);
    if (alpha > 0.0) {
      if (pos - r - 1 >= 0) cnt += alpha;
      if (pos + r + 1 <= n_global - 1) cnt += alpha;
    }
    v = (2.0 * r + 1.0 + (alpha > 0.0 ? 2.0 * alpha : 0.0)) / cnt;
  }
  g[i] = v;
}

// 4-plane tiled transpose (fp64): in [pl][H][W] -> out [pl][W][H]
__global__ void transpose_planes(const double* __restrict__ in, double* __restrict__ out,
                                 int64_t H, int64_t W) {
  __shared__ double tile[32][33];
  const int64_t pl = blockIdx.z;
  const int64_t x0 = (int64_t)blockIdx.x * 32, y0 = (int64_t)blockIdx.y * 32;
  const double* src = in + pl * H * W;
  double* dst = out + pl * H * W;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t y = y0 + k, x = x0 + threadIdx.x;
    if (y < H && x < W) tile[k][threadIdx.x] = src[y * W + x];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t x = x0 + k, y = y0 + threadIdx.x;
    if (x < W && y < H) dst[x * H + y] = tile[threadIdx.x][k];
  }
}

struct FusedEntry {
  int r;
  void (*launch)(const double*, double*, int, int64_t, int64_t, int64_t, const double*, int64_t,
                 int64_t, double, double, cudaStream_t);
};

template <int R>
void launch_colpass(const double* in, double* out, int nplanes, int64_t n_stream, int64_t n_cols,
                    int64_t seg, const double* g, int64_t pos0, int64_t n_global, double a,
                    double b, cudaStream_t st) {
  const int64_t nseg = (n_stream + seg - 1) / seg;
  const int64_t threads = (int64_t)nplanes * n_cols * nseg;
  colpass_f64<R, 3><<<(unsigned)((threads + 127) / 128), 128, 0, st>>>(
      in, out, nplanes, n_stream, n_cols, seg, g, pos0, n_global, a, b);
}

}  // namespace sbf
