// K1 — local dynamic range (reference maxfilter.py:41-61, _fastcore.pyx:16-58).
//
// Separable windowed maximum over the clamped (2R+1)^2 window, followed by
// T = max(M - f) evaluated in float64 exactly like the reference
// (`float(np.max(max_filter_2d(f, R) - f))`).  Both line passes stage a
// replicate-padded tile in shared memory (padding == clamping the window)
// and build power-of-two span maxima by doubling (log2(2R+1) fully parallel
// steps); each output is the max of two overlapping spans.  Max is exact, so
// M is bit-identical to the reference whatever the evaluation order.
//
// HBM-bound: f is read twice (row pass, column pass) and the row maxima
// once (written + read); T, min f and max f are reduced on chip and folded
// into three 64-bit atomics per CTA.
#include <cstring>
#include <type_traits>

#include "sbf_common.cuh"
#include "sbf_plan_warp.cuh"

namespace sbf {
namespace {

constexpr int kRowSeg = 1024;   // outputs per row-pass CTA
#ifndef SBF_K1_VH_ROW
#define SBF_K1_VH_ROW 0  // measured: the doubling row pass is faster (21.7 vs 24.0 us, config 2)
#endif
#ifndef SBF_K1_VH_ROWS
#define SBF_K1_VH_ROWS 8
#endif
#ifndef SBF_K1_VH_COL
#define SBF_K1_VH_COL 1
#endif
#ifndef SBF_K1_STREAM
#define SBF_K1_STREAM 1  // one-pass K1 (k1_stream_kernel) where the radius allows
#endif
constexpr bool g_k1_vh_row = SBF_K1_VH_ROW;  // van Herk blocks (else the doubling ladder)
constexpr bool g_k1_vh_col = SBF_K1_VH_COL;
constexpr int kColTile = 32;    // columns per column-pass CTA
constexpr int kColRows = 64;    // output rows per column-pass CTA
constexpr int kColThreadsY = 8;

// one FMNMX / DMNMX (the inputs are finite: non-finite images are rejected)
__device__ __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double vmax(double a, double b) { return fmax(a, b); }

// Row pass: out[y, x] = max f[y, clamp(x-R .. x+R)]
__device__ __forceinline__ void init_stats(double* stats, unsigned* done) {
  if (done) *done = 0u;
  unsigned long long* red = reinterpret_cast<unsigned long long*>(stats + 4);
  red[0] = ord_bits(0.0);
  red[1] = ord_bits(INFINITY);
  red[2] = ord_bits(-INFINITY);
  red[3] = 0ull;  // non-finite sample count (stats[7], read as uint64)
}

template <typename T>
__global__ void __launch_bounds__(256) rowmax_kernel(const T* __restrict__ f, int64_t W,
                                                     int64_t ld, int R, T* __restrict__ out,
                                                     double* __restrict__ stats,
                                                     unsigned* __restrict__ done) {
  // (PDL: the previous kernel on the stream may still read stats / f)
  pdl_wait();
  pdl_trigger();
  // the statistics accumulators are reset here (the column pass that updates
  // them runs after this kernel on the stream): one launch fewer
  if (stats && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) init_stats(stats, done);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* q = reinterpret_cast<T*>(smem_raw);
  const int64_t y = blockIdx.y;
  const int64_t x0 = (int64_t)blockIdx.x * kRowSeg;
  const int nout = (int)smin<int64_t>(kRowSeg, W - x0);
  const int win = 2 * R + 1;
  const int len = nout + 2 * R;
  const int nblk = (len + win - 1) / win;
  const int plen = nblk * win;
  T* suf = q + plen;
  const T* row = f + y * ld;
  // loads batched 4 deep per thread (independent, so they overlap in flight);
  // interior segments need no clamping
  if (x0 - R >= 0 && x0 - R + len <= W) {
    const T* src = row + (x0 - R);
#pragma unroll 4
    for (int k = threadIdx.x; k < len; k += blockDim.x) q[k] = __ldg(src + k);
  } else {
#pragma unroll 4
    for (int k = threadIdx.x; k < len; k += blockDim.x) {
      int64_t x = x0 - R + k;
      x = x < 0 ? 0 : (x >= W ? W - 1 : x);
      q[k] = __ldg(row + x);
    }
  }
  __syncthreads();
  // doubling: a[i] = max over [i, i + span) (every element in parallel,
  // log2(win) steps), then each output is the max of two overlapping spans
  T* a = q;
  T* b = suf;
  int span = 1;
  while (2 * span <= win) {
#pragma unroll 4
    for (int i = threadIdx.x; i <= len - 2 * span; i += blockDim.x) b[i] = vmax(a[i], a[i + span]);
    __syncthreads();
    T* t = a;
    a = b;
    b = t;
    span *= 2;
  }
  T* orow = out + y * W + x0;
#pragma unroll 4
  for (int j = threadIdx.x; j < nout; j += blockDim.x) orow[j] = vmax(a[j], a[j + win - span]);
}

// Suffix maxima of x[0..n) (stride `st`) into h, prefix maxima in place:
// samples are read 8 at a time ahead of the stores, so the shared-memory
// latency is paid once per chunk, not once per sample.
template <typename T>
__device__ __forceinline__ void vh_scan(T* __restrict__ x, T* __restrict__ h, int n, int st) {
  T m = x[(n - 1) * st];
  h[(n - 1) * st] = m;
  for (int i0 = n - 2; i0 >= 0; i0 -= 8) {
    T v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i0 - u >= 0) v[u] = x[(i0 - u) * st];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i0 - u >= 0) {
        m = vmax(m, v[u]);
        h[(i0 - u) * st] = m;
      }
  }
  m = x[0];
  for (int i0 = 1; i0 < n; i0 += 8) {
    T v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i0 + u < n) v[u] = x[(i0 + u) * st];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i0 + u < n) {
        m = vmax(m, v[u]);
        x[(i0 + u) * st] = m;
      }
  }
}

// Van Herk / Gil-Werman row pass: `rows` rows x one kRowSeg segment per CTA.
// The replicate-padded segment is cut into blocks of win = 2R+1 samples; per
// block one thread builds the suffix maxima (h) and, in place, the prefix
// maxima (g); output j is max(h[j], g[j + 2R]) -- 3 comparisons per sample
// whatever R (the doubling ladder took ~log2(win) passes of shared-memory
// traffic per sample and was instruction-bound).  Block strides are odd
// (win), so a warp's scan accesses are bank-conflict free.
template <typename T>
__global__ void __launch_bounds__(256) rowmax_vh_kernel(const T* __restrict__ f, int64_t H,
                                                        int64_t W, int64_t ld, int R, int rows,
                                                        T* __restrict__ out,
                                                        double* __restrict__ stats,
                                                        unsigned* __restrict__ done) {
  if (stats && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) init_stats(stats, done);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int win = 2 * R + 1;
  const int64_t x0 = (int64_t)blockIdx.x * kRowSeg;
  const int nout = (int)smin<int64_t>(kRowSeg, W - x0);
  const int len = nout + 2 * R;
  const int nblk = (len + win - 1) / win;
  const int plen = nblk * win;
  const int64_t yb = (int64_t)blockIdx.y * rows;
  const int nr = (int)smin<int64_t>(rows, H - yb);
  T* q = reinterpret_cast<T*>(smem_raw);  // [rows][plen]: samples, then prefix maxima
  T* h = q + (size_t)rows * plen;         // [rows][plen]: suffix maxima
  // one flat loop over (row, sample), 8 loads in flight per thread; the
  // padding past the segment is loaded too (clamped)
#pragma unroll 8
  for (int idx = threadIdx.x; idx < nr * plen; idx += blockDim.x) {
    const int r = idx / plen, k = idx - r * plen;
    int64_t x = x0 - R + k;
    x = x < 0 ? 0 : (x >= W ? W - 1 : x);
    q[idx] = __ldg(f + (yb + r) * ld + x);
  }
  __syncthreads();
  for (int bi = threadIdx.x; bi < nr * nblk; bi += blockDim.x) {
    const int r = bi / nblk, b = bi - r * nblk;
    vh_scan(q + r * plen + b * win, h + r * plen + b * win, win, 1);
  }
  __syncthreads();
  for (int r = 0; r < nr; ++r) {
    T* orow = out + (yb + r) * W + x0;
    const T* hr = h + r * plen;
    const T* gr = q + r * plen + 2 * R;
    for (int j = threadIdx.x; j < nout; j += blockDim.x) orow[j] = vmax(hr[j], gr[j]);
  }
}

__device__ __forceinline__ void finalize_stats(double* stats) {
  const unsigned long long* red = reinterpret_cast<const unsigned long long*>(stats + 4);
  const double T = ord_value(red[0]);
  const double mn = ord_value(red[1]), mx = ord_value(red[2]);
  stats[0] = T;
  stats[1] = mn;
  stats[2] = mx;
  // centre used by the term kernel: any constant works (BF(f + c) = BF(f) + c);
  // mid-range rounded to fp32 halves the magnitudes the fp32 sums carry.
  stats[3] = (isfinite(mn) && isfinite(mx)) ? (double)(float)(0.5 * (mn + mx)) : 0.0;
}

template <typename T>
__device__ __forceinline__ double block_reduce(double v, bool is_max, double* red) {
  for (int o = 16; o; o >>= 1) {
    double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, w) : fmin(v, w);
  }
  const int lane = (threadIdx.y * blockDim.x + threadIdx.x) & 31;
  const int warp = (threadIdx.y * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (blockDim.x * blockDim.y) >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < nwarps ? red[lane] : (is_max ? -INFINITY : INFINITY);
    for (int o = 16; o; o >>= 1) {
      double w = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_max ? fmax(v, w) : fmin(v, w);
    }
  }
  return v;
}

// Column pass fused with M - f, T, min/max.  Block = 32 columns x 8 threads.
// VH: van Herk blocks down each column (one thread per column block, see
// rowmax_vh_kernel); otherwise the doubling ladder.
template <typename T, bool VH>
__global__ void __launch_bounds__(kColTile* kColThreadsY) colmax_kernel(
    const T* __restrict__ rowmax, const T* __restrict__ f, int64_t H, int64_t W, int64_t ld,
    int R, int64_t t_lo, int64_t t_hi, T* __restrict__ M_out, unsigned long long* __restrict__ red,
    unsigned* __restrict__ done, const PlanArgs pa) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  pdl_trigger();
  pdl_wait();  // the row pass (and the statistics reset) are complete
  const int win = 2 * R + 1;
  const int64_t y0 = (int64_t)blockIdx.y * kColRows;
  const int nrows = (int)smin<int64_t>(kColRows, H - y0);
  const int len = nrows + 2 * R;
  const int nblk = (len + win - 1) / win;
  const int plen = nblk * win;
  constexpr int P = kColTile + 1;
  T* q = reinterpret_cast<T*>(smem_raw);
  T* suf = q + (size_t)plen * P;
  double* dred = reinterpret_cast<double*>(suf + (size_t)plen * P);
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t x = (int64_t)blockIdx.x * kColTile + tx;
  const bool xok = x < W;
  // fused pipeline: reset the fallback counter and clear the K3 accumulator
  // (their memset launches saved)
  if (pa.fb_reset && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && threadIdx.y == 0)
    *pa.fb_reset = 0ull;
  if (pa.zero_bytes) {
    const int64_t n16 = (int64_t)(pa.zero_bytes / 16);
    const int64_t nth = (int64_t)gridDim.x * gridDim.y * blockDim.x * blockDim.y;
    uint4* z = static_cast<uint4*>(pa.zero);
    for (int64_t i = ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x * blockDim.y +
                     threadIdx.y * blockDim.x + threadIdx.x;
         i < n16; i += nth)
      z[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  // the T phase's samples are requested first: their latency overlaps the
  // tile load and the scans instead of following them
  constexpr int FPT = kColRows / kColThreadsY;
  T fpre[FPT];
#pragma unroll
  for (int i = 0; i < FPT; ++i) {
    const int j = ty + i * kColThreadsY;
    const int64_t y = y0 + j;
    fpre[i] = (xok && j < nrows && y >= t_lo && y < t_hi) ? __ldg(f + y * ld + x) : T(0);
  }
  {
    const T* colp = rowmax + (xok ? x : 0);
    const int nload = VH ? plen : len;  // VH: the padding too (clamped)
    const int64_t ys = y0 - R;
    if (ys >= 0 && ys + nload <= H) {
      // interior tile: no clamping, the row pointer advances by a constant
      const T* pr = colp + (ys + ty) * W;
      const int64_t step = (int64_t)kColThreadsY * W;
#pragma unroll 8
      for (int k = ty; k < nload; k += kColThreadsY, pr += step) q[k * P + tx] = xok ? __ldg(pr) : T(0);
    } else {
#pragma unroll 8
      for (int k = ty; k < nload; k += kColThreadsY) {
        int64_t y = ys + k;
        y = y < 0 ? 0 : (y >= H ? H - 1 : y);
        q[k * P + tx] = xok ? __ldg(colp + y * W) : T(0);
      }
    }
  }
  __syncthreads();
  const T* a = q;
  int span = 1;  // outputs: max(a[j], a[j + win - span]) (doubling) / max(h[j], g[j + 2R]) (VH)
  const T* hh = suf;
  if (VH) {
    // suffix maxima into suf, prefix maxima in place (q)
    for (int b = ty; b < nblk; b += kColThreadsY) {
      vh_scan(q + (size_t)b * win * P + tx, suf + (size_t)b * win * P + tx, win, P);
    }
    __syncthreads();
  } else {
    // doubling along the column (see rowmax_kernel)
    T* aa = q;
    T* bb = suf;
    while (2 * span <= win) {
      for (int i = ty; i <= len - 2 * span; i += kColThreadsY)
        bb[i * P + tx] = vmax(aa[i * P + tx], aa[(i + span) * P + tx]);
      __syncthreads();
      T* t = aa;
      aa = bb;
      bb = t;
      span *= 2;
    }
    a = aa;
  }
  // min / max / finiteness in the sample type (exact); T's subtraction in fp64
  double tmax = 0.0;
  T fmn_t = T(INFINITY), fmx_t = T(-INFINITY);
  unsigned long long bad = 0;
  if (xok) {
#pragma unroll
    for (int i = 0; i < FPT; ++i) {
      const int j = ty + i * kColThreadsY;
      if (j >= nrows) break;
      const int64_t y = y0 + j;
      const T m = VH ? vmax(hh[j * P + tx], q[(j + 2 * R) * P + tx])
                     : vmax(a[j * P + tx], a[(j + win - span) * P + tx]);
      if (M_out) M_out[y * W + x] = m;
      if (y >= t_lo && y < t_hi) {
        const T fv = fpre[i];
        bad += isfinite(fv) ? 0 : 1;                 // image.py:16 (as_image finiteness)
        tmax = fmax(tmax, (double)m - (double)fv);  // maxfilter.py:61, float64 subtraction
        fmn_t = fmin(fmn_t, fv);
        fmx_t = fmax(fmx_t, fv);
      }
    }
  }
  double fmn = (double)fmn_t, fmx = (double)fmx_t;
  // one combined block reduction of (T, min, max, #non-finite)
  for (int o = 16; o; o >>= 1) {
    tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
    fmn = fmin(fmn, __shfl_xor_sync(0xffffffffu, fmn, o));
    fmx = fmax(fmx, __shfl_xor_sync(0xffffffffu, fmx, o));
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  const int tid = ty * kColTile + tx, lane = tid & 31, warp = tid >> 5;
  __shared__ int s_last;
  __shared__ sbf_plan s_plan;
  if (lane == 0) {
    dred[4 * warp] = tmax;
    dred[4 * warp + 1] = fmn;
    dred[4 * warp + 2] = fmx;
    dred[4 * warp + 3] = __longlong_as_double((long long)bad);
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kColTile * kColThreadsY / 32; ++w) {
      tmax = fmax(tmax, dred[4 * w]);
      fmn = fmin(fmn, dred[4 * w + 1]);
      fmx = fmax(fmx, dred[4 * w + 2]);
      bad += (unsigned long long)__double_as_longlong(dred[4 * w + 3]);
    }
    atomicMax(&red[0], ord_bits(tmax));
    atomicMin(&red[1], ord_bits(fmn));
    atomicMax(&red[2], ord_bits(fmx));
    if (bad) atomicAdd(&red[3], bad);
    // the last CTA folds the atomics into stats (no finalisation launch)
    __threadfence();
    s_last = 0;
    if (atomicAdd(done, 1u) == gridDim.x * gridDim.y - 1) {
      __threadfence();
      finalize_stats(reinterpret_cast<double*>(red) - 4);
      s_last = 1;
    }
  }
  if (pa.on) {
    // ... and, in the fused pipeline, builds the plan with its first warp
    // (K2 without a launch of its own)
    __syncwarp();
    if (warp == 0 && s_last)
      plan_warp(lane == 0 ? (reinterpret_cast<double*>(red) - 4)[0] : 0.0, pa.sigma_r, pa.eps, pa.rule,
                pa.log_2_over_eps, pa.plan, pa.terms, pa.cap, 0, 0, s_plan);
  }
}

// ---------------------------------------------------------------------------
// One-pass K1 ("streamed"): f is read from HBM once.
//
// A CTA of kStreamThreads threads owns a strip of TC = threads - 2R output
// columns and a band of output rows.  Thread i streams input column
// x0 - R + i down the band plus R rows above and below (samples outside the
// buffer are -inf, which is exactly the clamped window of the reference):
//  * vertical van Herk / Gil-Werman: the stream is cut into blocks of
//    w = 2R+1 rows; a running prefix maximum lives in a register, each
//    completed block is turned into suffix maxima in place in a shared-memory
//    ring of two blocks per column, and the window of output row j is
//    max(suffix[j], prefix[j + 2R]) -- 3 comparisons per sample;
//  * the vertical maxima of G output rows are staged in shared memory
//    and the same block decomposition runs along the rows (one thread per
//    (row, block)), giving M for TC columns;
//  * M - f in fp64 (maxfilter.py:61), min / max / non-finite count of f, and
//    the optional M image are produced in the same pass.
// The block reductions fold into the 64-bit order-preserving atomics of the
// two-pass kernels; the last CTA finalises the statistics and (fused
// pipeline) builds the plan.
constexpr int kStreamThreads = 256;
template <typename T>
struct StreamG {  // stream steps per group = rows of f in flight per thread = rows per horizontal batch
  static constexpr int value = sizeof(T) == 4 ? 16 : 8;
};

// suffix maxima of one column's completed vertical block, in place (stride
// st); not inlined: it runs once per block, outside the unrolled steps
template <typename T>
__device__ __noinline__ void stream_suffix(T* x, int w, int st) {
  T m = x[(w - 1) * st];
  for (int k0 = w - 2; k0 >= 0; k0 -= 8) {
    T s[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (k0 - q >= 0) s[q] = x[(k0 - q) * st];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (k0 - q >= 0) {
        m = vmax(m, s[q]);
        x[(k0 - q) * st] = m;
      }
  }
}

// one row block of the horizontal pass: suffix maxima into sr, prefix
// maxima in place (8 samples read ahead of each chain of comparisons)
template <typename T>
__device__ __forceinline__ void stream_scan_row(T* pr, T* sr, int n) {
  T m = pr[n - 1];
  sr[n - 1] = m;
  for (int k0 = n - 2; k0 >= 0; k0 -= 8) {
    T s[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (k0 - q >= 0) s[q] = pr[k0 - q];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (k0 - q >= 0) {
        m = vmax(m, s[q]);
        sr[k0 - q] = m;
      }
  }
  m = pr[0];
  for (int k0 = 1; k0 < n; k0 += 8) {
    T s[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (k0 + q < n) s[q] = pr[k0 + q];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (k0 + q < n) {
        m = vmax(m, s[q]);
        pr[k0 + q] = m;
      }
  }
}

template <typename T>
__device__ __forceinline__ T neg_inf() {
  return T(-INFINITY);
}

template <typename T>
size_t stream_smem_bytes(int R) {
  const int w = 2 * R + 1;
  return (size_t)2 * w * kStreamThreads * sizeof(T) +                    // vertical ring
         (size_t)2 * StreamG<T>::value * (kStreamThreads + 2) * sizeof(T) +  // prefix / suffix rows
         64 * sizeof(double);
}

template <typename T>
__global__ void __launch_bounds__(kStreamThreads, 2) k1_stream_kernel(
    const T* __restrict__ f, int64_t H, int64_t W, int64_t ld, int R, int band, int64_t t_lo,
    int64_t t_hi, T* __restrict__ M_out, unsigned long long* __restrict__ red,
    unsigned* __restrict__ done, const PlanArgs pa) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int NT = kStreamThreads, G = StreamG<T>::value, RB = G, HP = NT + 2;
  pdl_wait();     // the statistics reset (and f, if a kernel produced it)
  pdl_trigger();  // K3 may be scheduled; it waits for this grid itself
  const int w = 2 * R + 1;
  const int TC = NT - 2 * R;
  T* ring = reinterpret_cast<T*>(smem_raw);       // [2w][NT]
  T* hp = ring + (size_t)2 * w * NT;              // [RB][HP] vertical maxima -> prefix maxima
  T* hs = hp + (size_t)RB * HP;                   // [RB][HP] suffix maxima
  double* dred = reinterpret_cast<double*>(hs + (size_t)RB * HP);
  const int tid = threadIdx.x;
  const int64_t x0 = (int64_t)blockIdx.x * TC;
  const int64_t y0 = (int64_t)blockIdx.y * band;
  const int nout = (int)smin<int64_t>(band, H - y0);
  const int ncols = (int)smin<int64_t>(TC, W - x0);
  const int64_t xi = x0 - R + tid;  // this thread's input column
  const bool colok = xi >= 0 && xi < W;
  const int len = nout + 2 * R;     // stream length (virtual rows y0-R ..)

  if (pa.fb_reset && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) *pa.fb_reset = 0ull;
  if (pa.zero_bytes) {  // fused pipeline: clear the K3 accumulator (no memset launch)
    const int64_t n16 = (int64_t)(pa.zero_bytes / 16);
    const int64_t nth = (int64_t)gridDim.x * gridDim.y * NT;
    uint4* z = static_cast<uint4*>(pa.zero);
    for (int64_t i = ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * NT + tid; i < n16; i += nth)
      z[i] = make_uint4(0u, 0u, 0u, 0u);
  }

  double tmax = 0.0;
  T fmn = T(INFINITY), fmx = neg_inf<T>();
  unsigned long long bad = 0;

  // The stream is padded at the top with `pad` rows of -inf so that output
  // row 0's window closes on a group boundary: every group of G stream steps
  // (the unrolled register prefetch unit) then stages G whole output rows,
  // and the horizontal pass runs once per group, outside the unrolled steps.
  const int pad = (G - (2 * R) % G) % G;
  const int lenp = pad + len;
  const int first_out = pad + 2 * R;  // padded step of output row 0 (a multiple of G)
  // padded steps [tp_lo, tp_hi) are buffer rows (uniform across the CTA)
  const int tp_lo = (int)smax<int64_t>(0, R + pad - y0);
  const int tp_hi = (int)smin<int64_t>(lenp, H - (y0 - R - pad));
  const T* colp = f + (colok ? xi : 0) + (y0 - R - pad) * ld;  // row of padded step 0
  T cur[G], nxt[G];
  // G rows of f from padded step g (in flight together); groups wholly
  // inside the buffer rows load without per-step checks
  auto load_group = [&](T (&dst)[G], int g) {
    if (g >= tp_lo && g + G <= tp_hi) {
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const T v = __ldg(colp + (int64_t)(g + u) * ld);
        dst[u] = colok ? v : neg_inf<T>();
      }
    } else {
#pragma unroll
      for (int u = 0; u < G; ++u)
        dst[u] = (colok && g + u >= tp_lo && g + u < tp_hi) ? __ldg(colp + (int64_t)(g + u) * ld)
                                                            : neg_inf<T>();
    }
  };
  load_group(cur, 0);
  T P = neg_inf<T>();
  int bp = 0;    // position of the step in its vertical block (tp mod w)
  int slot = 0;  // ring slot of the step (tp mod 2w)
  // one group of G vertical steps; OUT: every step closes an output row's
  // window (groups from first_out on; steps past the stream end only stage
  // rows that are not output)
  auto vgroup = [&](auto out_tag) {
    constexpr bool OUT = decltype(out_tag)::value;
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const T v = cur[u];
      P = bp == 0 ? v : vmax(P, v);
      ring[slot * NT + tid] = v;
      if (bp == w - 1) stream_suffix(ring + (slot - (w - 1)) * NT + tid, w, NT);
      if (OUT) {
        // window of the output row: padded steps [tp - 2R, tp]
        int ss = slot - 2 * R;
        ss += ss < 0 ? 2 * w : 0;
        hp[u * HP + tid] = bp == w - 1 ? P : vmax(ring[ss * NT + tid], P);
      }
      bp = bp == w - 1 ? 0 : bp + 1;
      slot = slot == 2 * w - 1 ? 0 : slot + 1;
    }
  };
  for (int g0 = 0; g0 < lenp; g0 += G) {
    load_group(nxt, g0 + G);
    if (g0 >= first_out)
      vgroup(std::true_type{});
    else
      vgroup(std::false_type{});
    if (g0 >= first_out) {
      const int jb = min(G, lenp - g0);  // output rows staged by this group
      const int jr0 = g0 - first_out;    // band-relative row of staged row 0
      // ---- horizontal pass over the staged rows ----
      __syncthreads();
      const int nblk = (NT + w - 1) / w;
      for (int it = tid; it < jb * nblk; it += NT) {
        const int r = it % jb, b = it / jb;
        const int n = min(w, NT - b * w);
        stream_scan_row(hp + r * HP + b * w, hs + r * HP + b * w, n);
      }
      __syncthreads();
      // outputs of the group: M, M - f (fp64), statistics -- thread per
      // output column (ncols <= NT), the group's f samples requested first
      if (tid < ncols) {
        const int x = tid;
        const T* fcol = f + x0 + x + (y0 + jr0) * ld;
        T fo[G];
        const int64_t yg = y0 + jr0;
        if (jb == G && yg >= t_lo && yg + G <= t_hi) {
#pragma unroll
          for (int r = 0; r < G; ++r) fo[r] = __ldg(fcol + (int64_t)r * ld);
        } else {
#pragma unroll
          for (int r = 0; r < G; ++r)
            fo[r] = (r < jb && yg + r >= t_lo && yg + r < t_hi) ? __ldg(fcol + (int64_t)r * ld) : T(0);
        }
#pragma unroll
        for (int r = 0; r < G; ++r) {
          if (r >= jb) break;
          const T m = vmax(hs[r * HP + x], hp[r * HP + x + 2 * R]);
          const int64_t y = y0 + jr0 + r;
          if (M_out) M_out[y * W + x0 + x] = m;
          if (y >= t_lo && y < t_hi) {
            const T fv = fo[r];
            bad += isfinite(fv) ? 0 : 1;                // image.py:16
            tmax = fmax(tmax, (double)m - (double)fv);  // maxfilter.py:61
            fmn = fmin(fmn, fv);
            fmx = fmax(fmx, fv);
          }
        }
      }
      __syncthreads();  // hp / hs are restaged by the next group
    }
#pragma unroll
    for (int u = 0; u < G; ++u) cur[u] = nxt[u];
  }

  // block reduction of (T, min, max, #non-finite), then the global atomics
  double dmn = (double)fmn, dmx = (double)fmx;
  for (int o = 16; o; o >>= 1) {
    tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
    dmn = fmin(dmn, __shfl_xor_sync(0xffffffffu, dmn, o));
    dmx = fmax(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  const int lane = tid & 31, warp = tid >> 5;
  __shared__ int s_last;
  __shared__ sbf_plan s_plan;
  if (lane == 0) {
    dred[4 * warp] = tmax;
    dred[4 * warp + 1] = dmn;
    dred[4 * warp + 2] = dmx;
    dred[4 * warp + 3] = __longlong_as_double((long long)bad);
  }
  __syncthreads();
  if (tid == 0) {
    for (int wv = 1; wv < NT / 32; ++wv) {
      tmax = fmax(tmax, dred[4 * wv]);
      dmn = fmin(dmn, dred[4 * wv + 1]);
      dmx = fmax(dmx, dred[4 * wv + 2]);
      bad += (unsigned long long)__double_as_longlong(dred[4 * wv + 3]);
    }
    atomicMax(&red[0], ord_bits(tmax));
    atomicMin(&red[1], ord_bits(dmn));
    atomicMax(&red[2], ord_bits(dmx));
    if (bad) atomicAdd(&red[3], bad);
    __threadfence();
    s_last = 0;
    if (atomicAdd(done, 1u) == gridDim.x * gridDim.y - 1) {
      __threadfence();
      finalize_stats(reinterpret_cast<double*>(red) - 4);
      s_last = 1;
    }
  }
  if (pa.on) {
    __syncwarp();
    if (warp == 0 && s_last)
      plan_warp(lane == 0 ? (reinterpret_cast<double*>(red) - 4)[0] : 0.0, pa.sigma_r, pa.eps, pa.rule,
                pa.log_2_over_eps, pa.plan, pa.terms, pa.cap, 0, 0, s_plan);
  }
}

// statistics reset ahead of the one-pass K1 (programmatic dependent launch)
__global__ void stats_init_pdl_kernel(double* stats, unsigned* done) {
  pdl_wait();
  pdl_trigger();
  init_stats(stats, done);
}

// R == 0: T = 0 by definition (maxfilter.py:58-59); statistics only.
template <typename T>
__global__ void stats_only_kernel(const T* __restrict__ f, int64_t W, int64_t ld, int64_t t_lo,
                                  int64_t t_hi, T* __restrict__ M_out, int64_t H,
                                  unsigned long long* __restrict__ red) {
  __shared__ double dred[32];
  double fmn = INFINITY, fmx = -INFINITY;
  unsigned long long bad = 0;
  const int64_t n = H * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = i / W, x = i - y * W;
    const T v = f[y * ld + x];
    if (M_out) M_out[i] = v;
    if (y >= t_lo && y < t_hi) {
      bad += isfinite((double)v) ? 0 : 1;
      fmn = fmin(fmn, (double)v);
      fmx = fmax(fmx, (double)v);
    }
  }
  fmn = block_reduce<T>(fmn, false, dred);
  if (threadIdx.x == 0) atomicMin(&red[1], ord_bits(fmn));
  fmx = block_reduce<T>(fmx, true, dred);
  if (threadIdx.x == 0) atomicMax(&red[2], ord_bits(fmx));
  for (int o = 16; o; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(&red[3], bad);
}

__global__ void stats_init_kernel(double* stats, unsigned* done) { init_stats(stats, done); }

__global__ void stats_final_kernel(double* stats) { finalize_stats(stats); }

template <typename T>
size_t local_range_ws_bytes(int64_t H, int64_t W) {
  return align_up((size_t)(H * W) * sizeof(T)) + 256;  // row-max image + CTA counter
}

template <typename T>
int run(const void* fv, int64_t H, int64_t W, int64_t ld, int R, int64_t t_lo, int64_t t_hi,
        void* M_out, double* stats, void* ws, size_t ws_bytes, cudaStream_t st,
        const PlanArgs* plan) {
  PlanArgs pa;
  memset(&pa, 0, sizeof(pa));
  if (plan && R > 0) pa = *plan;
  const T* f = static_cast<const T*>(fv);
  unsigned long long* red = reinterpret_cast<unsigned long long*>(stats + 4);
  unsigned* done = nullptr;
  if (R > 0) {
    SBF_REQUIRE(ws && ws_bytes >= local_range_ws_bytes<T>(H, W), SBF_ERR_WORKSPACE,
                "local_range workspace too small");
    done = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + align_up((size_t)(H * W) * sizeof(T)));
  }
  if (R == 0) {
    stats_init_kernel<<<1, 1, 0, st>>>(stats, done);
    SBF_CHECK_LAUNCH();
  }
  // a window wider than the image equals the image-wide window (clamping)
  const int Rr = (int)smin<int64_t>(R, smax<int64_t>(W - 1, 0));
  const int Rc = (int)smin<int64_t>(R, smax<int64_t>(H - 1, 0));
  if (R == 0) {
    stats_only_kernel<T><<<2 * 148, 256, 0, st>>>(f, W, ld, t_lo, t_hi, static_cast<T*>(M_out), H,
                                                  red);
    SBF_CHECK_LAUNCH();
  } else if (SBF_K1_STREAM && sizeof(T) == 4 && R <= 24 && H * W >= (int64_t)4 << 20 &&
             stream_smem_bytes<T>(R) <= 200 * 1024) {
    // measured on B200 (K1 alone, us): config 4 (4096^2, R=18) 189 -> 157;
    // the two-pass kernels stay ahead on small images (config 2: 17 vs 20)
    // and at R = 36 (config 5, one CTA per SM: 3.09 vs 3.59 ms)
    // one pass over f (k1_stream_kernel); the statistics reset runs first
    const size_t smem = stream_smem_bytes<T>(R);
    SBF_CHECK_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(k1_stream_kernel<T>), smem));
    SBF_CHECK_CUDA(launch_pdl(stats_init_pdl_kernel, dim3(1), dim3(1), 0, st, stats, done));
    SBF_CHECK_LAUNCH();
    const int TC = kStreamThreads - 2 * R;
    const int64_t nstrips = (W + TC - 1) / TC;
    const int per_sm = (int)smax<int64_t>(1, (int64_t)(227 * 1024) / (int64_t)(smem + 1024));
    const int64_t slots = (int64_t)device_sm_count() * per_sm;
    const int64_t nb = smax<int64_t>(1, (slots + nstrips - 1) / nstrips);  // about one wave
    int64_t band = smax<int64_t>(smax<int64_t>(2 * R, 16), (H + nb - 1) / nb);
    band = smin<int64_t>(band, 1024);
    const int64_t nbands = (H + band - 1) / band;
    SBF_REQUIRE(nbands <= 65535, SBF_ERR_UNSUPPORTED, "image too tall for the K1 grid");
    SBF_CHECK_CUDA(launch_pdl(k1_stream_kernel<T>, dim3((unsigned)nstrips, (unsigned)nbands),
                              dim3(kStreamThreads), smem, st, static_cast<const T*>(f), H, W, ld, R,
                              (int)band, t_lo, t_hi, static_cast<T*>(M_out), red, done, pa));
    SBF_CHECK_LAUNCH();
    return SBF_OK;  // the last CTA wrote the final statistics
  } else {
    SBF_REQUIRE(ws_bytes >= (size_t)(H * W) * sizeof(T), SBF_ERR_WORKSPACE,
                "local_range workspace too small");
    T* rowmax = static_cast<T*>(ws);
    {
      const int win = 2 * Rr + 1;
      const int plen = ((kRowSeg + 2 * Rr + win - 1) / win) * win;
      const int64_t nseg = (W + kRowSeg - 1) / kRowSeg;
      // rows per CTA: enough CTAs for two per SM, at most 8 (4 for fp64)
      const int rmax = sizeof(T) == 4 ? SBF_K1_VH_ROWS : (SBF_K1_VH_ROWS + 1) / 2;
      const int rows = (int)smax<int64_t>(1, smin<int64_t>(rmax, (H * nseg + 295) / 296));
      const size_t smem_vh = 2 * (size_t)rows * plen * sizeof(T);
      if (g_k1_vh_row && smem_vh <= 100 * 1024) {
        SBF_CHECK_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(rowmax_vh_kernel<T>), smem_vh));
        dim3 grid((unsigned)nseg, (unsigned)((H + rows - 1) / rows));
        rowmax_vh_kernel<T><<<grid, 256, smem_vh, st>>>(f, H, W, ld, Rr, rows, rowmax, stats, done);
      } else {
        const size_t smem = 2 * (size_t)plen * sizeof(T);
        SBF_REQUIRE(smem <= 200 * 1024, SBF_ERR_UNSUPPORTED, "max-filter radius %d too large", R);
        SBF_CHECK_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(rowmax_kernel<T>), smem));
        dim3 grid((unsigned)nseg, (unsigned)H);
        SBF_CHECK_CUDA(launch_pdl(rowmax_kernel<T>, grid, dim3(256), smem, st, f, W, ld, Rr, rowmax,
                                  stats, done));
      }
      SBF_CHECK_LAUNCH();
    }
    {
      const int win = 2 * Rc + 1;
      const int plen = ((kColRows + 2 * Rc + win - 1) / win) * win;
      const size_t smem = 2 * (size_t)plen * (kColTile + 1) * sizeof(T) + 32 * sizeof(double);
      SBF_REQUIRE(smem <= 220 * 1024, SBF_ERR_UNSUPPORTED, "max-filter radius %d too large", R);
      dim3 grid((unsigned)((W + kColTile - 1) / kColTile), (unsigned)((H + kColRows - 1) / kColRows));
      dim3 block(kColTile, kColThreadsY);
      auto kern = g_k1_vh_col ? colmax_kernel<T, true> : colmax_kernel<T, false>;
      SBF_CHECK_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem));
      SBF_CHECK_CUDA(launch_pdl(kern, grid, block, smem, st, rowmax, f, H, W, ld, Rc, t_lo, t_hi,
                                static_cast<T*>(M_out), red, done, pa));
      SBF_CHECK_LAUNCH();
    }
    return SBF_OK;  // colmax's last CTA wrote the final statistics
  }
  stats_final_kernel<<<1, 1, 0, st>>>(stats);
  SBF_CHECK_LAUNCH();
  return SBF_OK;
}

}  // namespace

size_t local_range_ws(int64_t H, int64_t W, int dtype) {
  return dtype == SBF_F64 ? local_range_ws_bytes<double>(H, W) : local_range_ws_bytes<float>(H, W);
}

int launch_local_range(const void* f, int dtype, int64_t H, int64_t W, int64_t ld, int R,
                       int64_t t_lo, int64_t t_hi, void* M_out, double* stats, void* ws,
                       size_t ws_bytes, cudaStream_t st, const PlanArgs* plan) {
  // the fused plan needs the column pass (R > 0); the caller launches K2 otherwise
  SBF_REQUIRE(!plan || (R > 0 && plan->plan && plan->terms && plan->cap > 0), SBF_ERR_INVALID,
              "fused plan needs R > 0 and plan / term buffers");
  SBF_REQUIRE(f && stats, SBF_ERR_INVALID, "null pointer");
  SBF_REQUIRE(H >= 1 && W >= 1 && ld >= W, SBF_ERR_INVALID, "bad image shape %lld x %lld",
              (long long)H, (long long)W);
  SBF_REQUIRE(R >= 0, SBF_ERR_INVALID, "radius must be >= 0");
  SBF_REQUIRE(t_lo >= 0 && t_hi <= H && t_lo < t_hi, SBF_ERR_INVALID, "bad row range");
  if (dtype == SBF_F32)
    return run<float>(f, H, W, ld, R, t_lo, t_hi, M_out, stats, ws, ws_bytes, st, plan);
  if (dtype == SBF_F64)
    return run<double>(f, H, W, ld, R, t_lo, t_hi, M_out, stats, ws, ws_bytes, st, plan);
  set_error("unsupported dtype %d", dtype);
  return SBF_ERR_INVALID;
}

}  // namespace sbf
