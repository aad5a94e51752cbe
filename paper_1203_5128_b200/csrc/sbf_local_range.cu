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
#ifndef SBF_K1_PRUNE
#define SBF_K1_PRUNE 1  // T by tile bounds + exact evaluation of the tiles that can raise it
#endif
#ifndef SBF_K1P_DBG
#define SBF_K1P_DBG 0  // timing studies only: 1 = exact rounds select nothing, 2 = no exact rounds
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

// ---------------------------------------------------------------------------
// Pruned K1 (T only, no M image): exact, f read from HBM about once.
//
// T = max_x (M(x) - f(x)) with M the clamped (2R+1)^2 window maximum
// (maxfilter.py:56-61).  For 32x32 tiles, M(x) <= max over the tiles within
// n = ceil(R/32) tile steps of their maxima, and f(x) >= the tile's minimum,
// so U_t = double(that max) - double(tile min) bounds the contribution of
// every pixel of tile t (double subtraction is monotone).  Kernels:
//   tiles   one pass over f: per-tile max (all buffer rows) and min (rows in
//           [t_lo, t_hi)), the image statistics, the K3 accumulator clear;
//   bounds  U_t per tile, their maximum Umax;
//   exact 1 tiles with U_t == Umax: M - f evaluated exactly (separable window
//           maximum in shared memory, doubling ladder), T = max;
//   exact 2 tiles with T < U_t < Umax, the same; the last CTA finalises the
//           statistics and builds the plan (fused pipeline).
// Tiles whose bound cannot exceed the T already found are never evaluated:
// on the configs' 8-bit images most tiles drop out after round 1.  The
// result equals the full evaluation bit for bit (the max of the same fp64
// differences).
constexpr int kPruneTile = 32;
constexpr int kPruneSub = 16;   // bound granularity (sub-tiles of a tile)
constexpr int kPruneMaxR = 48;  // exact-tile shared memory bound ((32 + 2R)^2 samples, two buffers)

template <typename T>
__global__ void __launch_bounds__(256) k1p_tiles_kernel(
    const T* __restrict__ f, int64_t H, int64_t W, int64_t ld, int64_t t_lo, int64_t t_hi,
    int tiles_x, int stx, T* __restrict__ smax_all, T* __restrict__ smin_int,
    unsigned long long* __restrict__ red, const PlanArgs pa) {
  pdl_wait();  // statistics reset
  pdl_trigger();
  if (pa.fb_reset && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *pa.fb_reset = 0ull;
  if (pa.zero_bytes) {  // fused pipeline: clear the K3 accumulator
    const int64_t n16 = (int64_t)(pa.zero_bytes / 16);
    const int64_t nth = (int64_t)gridDim.x * gridDim.y * blockDim.x;
    uint4* z = static_cast<uint4*>(pa.zero);
    for (int64_t i = ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
         i < n16; i += nth)
      z[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  // warp w: tile (blockIdx.x * 8 + w, blockIdx.y); lane: a column, 32 rows;
  // the 8x8 sub-tile maxima (every buffer row) and minima (rows in
  // [t_lo, t_hi)) go to smax_all / smin_int
  constexpr int SUB = kPruneSub, NSG = kPruneTile / kPruneSub;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tx = blockIdx.x * 8 + w, ty = blockIdx.y;
  const int64_t x = (int64_t)tx * kPruneTile + lane;
  const int64_t y0 = (int64_t)ty * kPruneTile;
  T gmx[NSG], gmn[NSG];
  T smx = neg_inf<T>(), wmn = T(INFINITY);
  unsigned long long bad = 0;
#pragma unroll
  for (int g = 0; g < NSG; ++g) {
    gmx[g] = neg_inf<T>();
    gmn[g] = T(INFINITY);
  }
  if (tx < tiles_x && x < W) {
    const int nr = (int)smin<int64_t>(kPruneTile, H - y0);
    const T* col = f + y0 * ld + x;
    T v[kPruneTile];
#pragma unroll
    for (int r = 0; r < kPruneTile; ++r) v[r] = r < nr ? __ldg(col + (int64_t)r * ld) : T(0);
#pragma unroll
    for (int r = 0; r < kPruneTile; ++r) {
      if (r >= nr) break;
      gmx[r / SUB] = vmax(gmx[r / SUB], v[r]);  // a window may reach into halo rows
      const int64_t y = y0 + r;
      if (y >= t_lo && y < t_hi) {  // T and the statistics: interior rows only
        gmn[r / SUB] = fmin(gmn[r / SUB], v[r]);
        smx = vmax(smx, v[r]);
        bad += isfinite(v[r]) ? 0 : 1;  // image.py:16
      }
    }
  }
  // fold 8 columns (lanes) per sub-tile
#pragma unroll
  for (int g = 0; g < NSG; ++g) {
    wmn = fmin(wmn, gmn[g]);
    for (int o = 1; o < SUB; o <<= 1) {
      gmx[g] = vmax(gmx[g], __shfl_xor_sync(0xffffffffu, gmx[g], o));
      gmn[g] = fmin(gmn[g], __shfl_xor_sync(0xffffffffu, gmn[g], o));
    }
  }
  if (tx < tiles_x && (lane & (SUB - 1)) == 0) {
    const int sx = tx * NSG + lane / SUB;
    if (sx < stx) {
#pragma unroll
      for (int g = 0; g < NSG; ++g) {
        const int64_t sy = (int64_t)ty * NSG + g;
        if (sy * SUB < H) {
          smax_all[sy * stx + sx] = gmx[g];
          smin_int[sy * stx + sx] = gmn[g];
        }
      }
    }
  }
  for (int o = 16; o; o >>= 1) {
    wmn = fmin(wmn, __shfl_xor_sync(0xffffffffu, wmn, o));
    smx = vmax(smx, __shfl_xor_sync(0xffffffffu, smx, o));
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  // one atomic per CTA for each statistic (per-warp atomics on the same
  // three words serialised this pass)
  __shared__ T s_mn[8], s_mx[8];
  if (lane == 0) {
    s_mn[w] = wmn;
    s_mx[w] = smx;
    if (bad) atomicAdd(&red[3], bad);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    T a = s_mn[0], c = s_mx[0];
    for (int k = 1; k < 8; ++k) {
      a = fmin(a, s_mn[k]);
      c = vmax(c, s_mx[k]);
    }
    if (a < T(INFINITY)) atomicMin(&red[1], ord_bits((double)a));
    if (c > neg_inf<T>()) atomicMax(&red[2], ord_bits((double)c));
  }
}

__global__ void k1p_init_kernel(double* stats, unsigned* done, unsigned long long* slots) {
  pdl_wait();
  pdl_trigger();
  init_stats(stats, done);
  slots[0] = ord_bits(-INFINITY);
  slots[1] = slots[2] = 0ull;
}

// U_t for every tile with interior pixels (the max over its sub-tiles s of
// (max of the sub-tile maxima within nbs = ceil(R/8) sub-tile steps) -
// sub-tile minimum); Umax into slots[0].  Block = 256 / NS tiles of one tile row x
// their NS sub-tiles each.
template <typename T>
__global__ void __launch_bounds__(256) k1p_bounds_kernel(
    int tiles_x, int tiles_y, int stx, int sty, int nbs, const T* __restrict__ smax_all,
    const T* __restrict__ smin_int, double* __restrict__ U, unsigned long long* __restrict__ slots) {
  pdl_wait();
  pdl_trigger();
  constexpr int NSG = kPruneTile / kPruneSub, NS = NSG * NSG;  // sub-tiles per tile
  const int k = threadIdx.x / NS, sub = threadIdx.x % NS;
  const int tx = blockIdx.x * (256 / NS) + k, ty = blockIdx.y;
  const int sx = tx * NSG + (sub & (NSG - 1)), sy = ty * NSG + sub / NSG;
  double u = -INFINITY;
  if (tx < tiles_x && sx < stx && sy < sty) {
    const T mn = smin_int[(int64_t)sy * stx + sx];
    if (mn < T(INFINITY)) {
      T m = neg_inf<T>();
      const int y_lo = max(0, sy - nbs), y_hi = min(sty - 1, sy + nbs);
      const int x_lo = max(0, sx - nbs), x_hi = min(stx - 1, sx + nbs);
      for (int yy = y_lo; yy <= y_hi; ++yy) {
        const T* row = smax_all + (int64_t)yy * stx;
        for (int xx = x_lo; xx <= x_hi; ++xx) m = vmax(m, row[xx]);
      }
      u = (double)m - (double)mn;
    }
  }
  for (int o = NS / 2; o; o >>= 1) u = fmax(u, __shfl_xor_sync(0xffffffffu, u, o));
  if (sub == 0 && tx < tiles_x) U[(int64_t)ty * tiles_x + tx] = u;
  for (int o = 16; o; o >>= 1) u = fmax(u, __shfl_xor_sync(0xffffffffu, u, o));
  if ((threadIdx.x & 31) == 0 && u > -INFINITY) atomicMax(&slots[0], ord_bits(u));
}

// Exact M - f on the tiles a round selects (persistent CTAs stride over the
// tiles).  round 1: U_t == Umax; round 2: T < U_t < Umax, T = red[0] after
// round 1.  The window maximum is separable: rows then columns, each by
// power-of-two span maxima (doubling) in shared memory; samples outside the
// buffer are -inf (the clamped window).
template <typename T>
__global__ void __launch_bounds__(256) k1p_exact_kernel(
    const T* __restrict__ f, int64_t H, int64_t W, int64_t ld, int R, int64_t t_lo, int64_t t_hi,
    int tiles_x, int ntiles, int round, const double* __restrict__ U,
    const unsigned long long* __restrict__ slots, unsigned long long* __restrict__ red) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x;
  const int TS = kPruneTile, IW = TS + 2 * R, win = 2 * R + 1;
  T* a = reinterpret_cast<T*>(smem_raw);  // [IW][IW] samples / row spans
  T* b = a + IW * IW;                     // [IW][IW] ping-pong
  __shared__ double dred[8];
  const double umax = ord_value(slots[0]);
  const double tcur = ord_value(red[0]);  // T after round 1 (round 2 only)
  double tmax = 0.0;
  __shared__ int s_list[256], s_n;
  // the CTA's 256 threads test 256 tile bounds at once; the selected tiles
  // are then evaluated one after another by the whole CTA
  // (tile t goes to CTA t mod gridDim: selected tiles cluster in space, so
  // neighbours land on different CTAs)
  for (int base = 0; base * (int64_t)gridDim.x < ntiles; base += 256) {
    if (tid == 0) s_n = 0;
    __syncthreads();
    const int64_t t = (int64_t)(base + tid) * gridDim.x + blockIdx.x;
    if (t < ntiles) {
      const double u = U[t];
      const bool sel = !(SBF_K1P_DBG & 1) && (round == 1 ? (u == umax && u > 0.0) : (u > tcur && u < umax));
      if (sel) {
        s_list[atomicAdd(&s_n, 1)] = (int)t;
        atomicAdd(const_cast<unsigned long long*>(slots) + round, 1ull);  // tiles evaluated per round (diagnostic)
      }
    }
    __syncthreads();
    const int nsel = s_n;
  for (int si = 0; si < nsel; ++si) {
    const int t = s_list[si];
    const int ty = t / tiles_x, tx = t - ty * tiles_x;
    const int64_t y0 = (int64_t)ty * TS - R, x0 = (int64_t)tx * TS - R;
    // warp w takes rows w, w + 8, ...; lane takes columns lane + 32 q
    // (q < 4: IW <= 128); the loops are unrolled so that each thread's
    // shared-memory reads of a pass are in flight together
    const int lane = tid & 31, wp = tid >> 5;
    constexpr int QC = (kPruneTile + 2 * kPruneMaxR + 31) / 32;  // column slots per lane
    {
      // every load of the region issued before any store (one latency)
      constexpr int RR = (kPruneTile + 2 * kPruneMaxR + 7) / 8;  // rows per warp
      T v[RR][QC];
#pragma unroll
      for (int i = 0; i < RR; ++i) {
        const int r = wp + 8 * i;
        const int64_t y = y0 + r;
        const bool rok = r < IW && y >= 0 && y < H;
#pragma unroll
        for (int q = 0; q < QC; ++q) {
          const int c = lane + 32 * q;
          const int64_t x = x0 + c;
          v[i][q] = (rok && c < IW && x >= 0 && x < W) ? __ldg(f + y * ld + x) : neg_inf<T>();
        }
      }
#pragma unroll
      for (int i = 0; i < RR; ++i) {
        const int r = wp + 8 * i;
#pragma unroll
        for (int q = 0; q < QC; ++q) {
          const int c = lane + 32 * q;
          if (r < IW && c < IW) a[r * IW + c] = v[i][q];
        }
      }
    }
    __syncthreads();
    // the tile's own samples (for M - f) stay in registers
    T fown[kPruneTile / 8];
#pragma unroll
    for (int i = 0; i < kPruneTile / 8; ++i) fown[i] = a[(R + wp + 8 * i) * IW + R + lane];
    // row direction: a[r][c] = max over [c, c + span) by doubling
    T* src = a;
    T* dst = b;
    int span = 1;
    while (2 * span <= win) {
#pragma unroll 2
      for (int r = wp; r < IW; r += 8) {
        T* d = dst + r * IW;
        const T* sr = src + r * IW;
#pragma unroll
        for (int q = 0; q < QC; ++q) {
          const int c = lane + 32 * q;
          if (c < IW) d[c] = c + span < IW ? vmax(sr[c], sr[c + span]) : sr[c];
        }
      }
      __syncthreads();
      T* tt = src;
      src = dst;
      dst = tt;
      span *= 2;
    }
    // row maxima of the tile's output columns: rm[r][j] = max over [j, j + win)
#pragma unroll 4
    for (int r = wp; r < IW; r += 8) dst[r * IW + lane] = vmax(src[r * IW + lane], src[r * IW + lane + win - span]);
    __syncthreads();
    // column direction on rm (IW rows x TS columns, in dst)
    src = dst;
    dst = (src == a) ? b : a;
    span = 1;
    while (2 * span <= win) {
#pragma unroll 4
      for (int r = wp; r < IW; r += 8)
        dst[r * IW + lane] = r + span < IW ? vmax(src[r * IW + lane], src[(r + span) * IW + lane]) : src[r * IW + lane];
      __syncthreads();
      T* tt = src;
      src = dst;
      dst = tt;
      span *= 2;
    }
#pragma unroll
    for (int k = 0; k < kPruneTile / 8; ++k) {
      const int i = wp + 8 * k;
      const int64_t y = (int64_t)ty * TS + i, x = (int64_t)tx * TS + lane;
      if (y < t_lo || y >= t_hi || y >= H || x >= W) continue;
      const T m = vmax(src[i * IW + lane], src[(i + win - span) * IW + lane]);
      tmax = fmax(tmax, (double)m - (double)fown[k]);  // maxfilter.py:61
    }
    __syncthreads();  // a / b are reloaded for the next tile
  }
    __syncthreads();  // s_list / s_n are rewritten for the next group
  }
  for (int o = 16; o; o >>= 1) tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
  if ((tid & 31) == 0) dred[tid >> 5] = tmax;
  __syncthreads();
  if (tid == 0) {
    for (int wv = 1; wv < 8; ++wv) tmax = fmax(tmax, dred[wv]);
    atomicMax(&red[0], ord_bits(tmax));
  }
}

// statistics finalisation and (fused pipeline) the plan, after round 2: a
// one-warp kernel, so the exact-tile kernel stays small (its code is fetched
// cold by the few CTAs that evaluate a tile)
__global__ void k1p_final_kernel(unsigned long long* __restrict__ red, const PlanArgs pa) {
  __shared__ sbf_plan s_plan;
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) finalize_stats(reinterpret_cast<double*>(red) - 4);
  __syncwarp();
  if (pa.on)
    plan_warp(threadIdx.x == 0 ? (reinterpret_cast<double*>(red) - 4)[0] : 0.0, pa.sigma_r, pa.eps,
              pa.rule, pa.log_2_over_eps, pa.plan, pa.terms, pa.cap, 0, 0, s_plan);
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
  } else if (SBF_K1_PRUNE && !M_out && H * W >= ((int64_t)4 << 20) &&
             R <= (sizeof(T) == 4 ? kPruneMaxR : 24)) {
    // pruned exact T (no M image): tile bounds, then exact tiles only where
    // a tile could raise T
    const int tiles_x = (int)((W + kPruneTile - 1) / kPruneTile);
    const int tiles_y = (int)((H + kPruneTile - 1) / kPruneTile);
    const int ntiles = tiles_x * tiles_y;
    const int stx = (int)((W + kPruneSub - 1) / kPruneSub), sty = (int)((H + kPruneSub - 1) / kPruneSub);
    const size_t nsub = (size_t)stx * sty;
    char* w = static_cast<char*>(ws);
    T* smax_all = reinterpret_cast<T*>(w);
    T* smin_int = smax_all + nsub;
    double* U = reinterpret_cast<double*>(w + align_up(2 * nsub * sizeof(T)));
    unsigned long long* slots =
        reinterpret_cast<unsigned long long*>(w + align_up(2 * nsub * sizeof(T)) + align_up((size_t)ntiles * 8));
    SBF_REQUIRE(align_up(2 * nsub * sizeof(T)) + align_up((size_t)ntiles * 8) + 64 <=
                    align_up((size_t)(H * W) * sizeof(T)),
                SBF_ERR_WORKSPACE, "local_range workspace too small");
    SBF_CHECK_CUDA(launch_pdl(k1p_init_kernel, dim3(1), dim3(1), 0, st, stats, done, slots));
    SBF_CHECK_LAUNCH();
    SBF_CHECK_CUDA(launch_pdl(k1p_tiles_kernel<T>, dim3((unsigned)((tiles_x + 7) / 8), (unsigned)tiles_y),
                              dim3(256), 0, st, f, H, W, ld, t_lo, t_hi, tiles_x, stx, smax_all, smin_int,
                              red, pa));
    SBF_CHECK_LAUNCH();
    const int nbs = (R + kPruneSub - 1) / kPruneSub;
    constexpr int kTilesPerBoundsBlock = 256 / ((kPruneTile / kPruneSub) * (kPruneTile / kPruneSub));
    SBF_CHECK_CUDA(launch_pdl(k1p_bounds_kernel<T>,
                              dim3((unsigned)((tiles_x + kTilesPerBoundsBlock - 1) / kTilesPerBoundsBlock),
                                   (unsigned)tiles_y),
                              dim3(256), 0, st, tiles_x, tiles_y, stx, sty, nbs,
                              static_cast<const T*>(smax_all), static_cast<const T*>(smin_int), U, slots));
    SBF_CHECK_LAUNCH();
    const int IW = kPruneTile + 2 * R;
    const size_t smem = (size_t)2 * IW * IW * sizeof(T);
    SBF_CHECK_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(k1p_exact_kernel<T>), smem));
    const int per_sm = (int)smax<int64_t>(1, smin<int64_t>(4, (int64_t)(227 * 1024) / (int64_t)(smem + 1024)));
    const int grid = (int)smin<int64_t>(ntiles, (int64_t)device_sm_count() * per_sm);
    for (int round = 1; round <= ((SBF_K1P_DBG & 2) ? 0 : 2); ++round) {
      SBF_CHECK_CUDA(launch_pdl(k1p_exact_kernel<T>, dim3((unsigned)grid), dim3(256), smem, st, f, H, W, ld,
                                R, t_lo, t_hi, tiles_x, ntiles, round, static_cast<const double*>(U),
                                static_cast<const unsigned long long*>(slots), red));
      SBF_CHECK_LAUNCH();
    }
    SBF_CHECK_CUDA(launch_pdl(k1p_final_kernel, dim3(1), dim3(32), 0, st, red, pa));
    SBF_CHECK_LAUNCH();
    return SBF_OK;  // k1p_final_kernel wrote the final statistics (and the plan)
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
