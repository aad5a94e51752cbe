// K3 — fused per-term sweep with the divide/fallback epilogue (sm_100a).
//
// Replaces, per folded cosine term (reference bilateral.py:150-163):
//   theta = omega_n f; gc, gs = cos, sin; four apply_spatial() smoothings of
//   f*gc, gc, f*gs, gs (spatial.py:108-139: `passes` extended-box passes,
//   each renormalised over the clamped window — _extended_box_lines
//   spatial.py:120-133 over window_sum_lines _fastcore.pyx:61-86);
//   num/den += scale (gc S[f gc] + gs S[f gs]) / (gc S[gc] + gs S[gs]);
// and, after the last term, _divide_with_fallback (bilateral.py:242-254).
// Rows and columns commute (Kronecker product), so all column passes run
// first, then all row passes.
//
// One work item = one 128-column strip x one row band x one term; persistent
// CTAs (two per SM) pull items band by band from an atomic counter.
//  * f arrives by TMA: one 2-D box (128 columns x ROWS rows) per chunk of
//    ROWS = CH * L stream steps, zero-filled outside the buffer, prefetched
//    into shared memory while the previous chunk's H phase runs.
//  * V phase — one thread per column streams the band: phasor by MUFU
//    sin/cos, the four modulated images as two packed pairs
//    (f cos, cos) and (f sin, sin) (FMUL2/FADD2/FFMA2), and the column passes
//    as O(1) recurrences
//        A_t = A_{t-1} + a (x_{t-1} - x_{t-2D}) + b (x_t - x_{t-2D-1})
//    (D = r+1, a = (1-alpha)/cnt, b = alpha/cnt, cnt = 2r+1+2alpha) with
//    the 2r+3 input history of every pass in a register ring.  Blocks of
//    L = 2r+3 steps are unrolled so the ring rotates at compile time;
//    chunks hold whole blocks, so no step carries a range check.  Border
//    renormalisation (zero padding + cnt/cnt(pos)) runs only in blocks that
//    touch the image's top or bottom rows.
//  * H phase — 4 lanes per row (one per image) stream the chunk's rows with
//    the same recurrence (column renormalisation only in the two edge
//    strips) and write the smoothed values back in place.
//  * Accumulate — one thread per output column: (num, den) = cos (F_c, G_c)
//    + sin (F_s, G_s), scaled by the term weight.  Each output pixel has one
//    owner per term and the terms are applied in order: a per-row ticket
//    (terms accumulated so far) is waited for with ld.acquire and advanced
//    with st.release, so the sum order is fixed and results are
//    reproducible bit for bit.  The first term stores, the last term divides
//    (den > 0 ? num/den + centre : f, fallback count) and writes the output
//    (device or page-locked host memory) — no separate epilogue kernel.
// Intermediate images never leave the SM; only the (num, den) accumulator of
// the current band visits L2.
#pragma once

#include <cuda.h>

#include <type_traits>
#include <utility>

#include "sbf_common.cuh"

namespace sbf {

struct SweepParams {
  const float* f;  // fp32 image (centred when `centred`), ld % 4 == 0
  int64_t ld;
  int centred;
  const void* fo;  // original input (fallback values), fo_dtype
  int64_t fo_ld;
  int fo_dtype;
  void* out;
  int out_dtype;
  int H;  // buffer rows
  int W;
  int64_t row0;   // global row index of buffer row 0
  int64_t img_H;  // global image height
  int out_lo, out_hi;
  int band;
  int nstrips;
  int* ctrl;    // [0] work-queue head (zeroed before launch)
  int* seg;     // per (32-row output segment, strip): items landed (zeroed before launch)
  unsigned long long* acc;  // fixed-point (num | den) per output pixel (zeroed before launch)
  int r;
  float alpha;
  float a, b;
  const sbf_plan* plan;
  const sbf_term* terms;
  const double* stats;
  unsigned long long* fallback;
  int hdr_guard;  // SBF_PREC_AUTO: bail out (flag the plan) on wide ranges
  int fused_epi;  // 1: the item completing a segment divides it out; 0: sweep_divide_kernel follows
};

template <int R, int PASSES>
struct SweepCfg {
  static constexpr int D = R + 1;
  static constexpr int L = 2 * R + 3;
  static constexpr int HALO = PASSES * D;
  static constexpr int COLS = 128;                 // haloed columns per strip = threads
  // TMA box width: the box must start on a 16-byte boundary, so it begins at
  // the strip's first column rounded down to a multiple of 4
  static constexpr int FCOLS = COLS + 4;
  static constexpr int WC = COLS - 2 * HALO;       // output columns per strip
  static constexpr int ROWS = COLS / 4;            // stream steps (VB rows) per chunk: one H lane per (row, image)
  static constexpr int NB = (COLS + L) / L;        // H-phase blocks per row (>= COLS + 1 steps)
  static constexpr int VB_COLS = NB * L;
  static constexpr int VB_PITCH = 4 * VB_COLS + 4;  // floats; == 4 mod 32 words for 8 rows
  static constexpr int RING = ((ROWS + HALO + L - 1) / L) * L;  // phasor ring (steps)
  static constexpr int RAW_PITCH = WC + 1;
  static constexpr int GOFF = (PASSES + 2) * D + 2;
  static constexpr int THREADS = COLS;
  static constexpr int SEGR = 32;  // output rows per epilogue segment
  static_assert(WC > 0, "halo too wide for a 128-column strip");
  static constexpr size_t F_BYTES = (size_t)ROWS * FCOLS * 4;
  static constexpr size_t VB_BYTES = (size_t)ROWS * VB_PITCH * 4;
  static constexpr size_t RAW_BYTES = (size_t)RING * RAW_PITCH * 4;
};

template <class F, int... Js>
__device__ __forceinline__ void sweep_for_impl(F&& f, std::integer_sequence<int, Js...>) {
  (f(std::integral_constant<int, Js>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void sweep_for(F&& f) {
  sweep_for_impl(f, std::make_integer_sequence<int, N>{});
}

// renormalisation factor cnt_int / cnt(pos) on an axis of length n (0 outside)
__device__ __forceinline__ float axis_factor(int64_t pos, int64_t n, int r, float alpha) {
  if (pos < 0 || pos >= n) return 0.f;
  if (pos - r - 1 >= 0 && pos + r + 1 <= n - 1) return 1.f;
  const int64_t lo = pos - r < 0 ? 0 : pos - r;
  const int64_t hi = pos + r > n - 1 ? n - 1 : pos + r;
  double cnt = (double)(hi - lo + 1);
  if (alpha > 0.f) {
    if (pos - r - 1 >= 0) cnt += alpha;
    if (pos + r + 1 <= n - 1) cnt += alpha;
  }
  const double cint = 2.0 * r + 1.0 + (alpha > 0.f ? 2.0 * (double)alpha : 0.0);
  return (float)(cint / cnt);
}

__device__ __forceinline__ float2 pk(float v) { return make_float2(v, v); }

// One image pair's cascade of PASSES recurrences at ring slot J (packed).
// dl[0]: input samples; dl[p>0]: raw accumulator of pass p-1.  BORDER blocks
// normalise on read: gt[s - p*D - k] is the factor of the sample pass p reads
// at step s - k (k in {0, 1, 2D, 2D+1}); the final output is scaled by
// gt[s - PASSES*D].  gt already includes the table offset.
template <int J, int L, int D, int PASSES, bool BORDER>
__device__ __forceinline__ float2 vcascade(float2 (&dl)[PASSES][L], float2& vlast, float2 x,
                                           float2 a2, float2 nb2, float2 b2, const float* gt) {
  constexpr int JM1 = (J + L - 1) % L, JO1 = (J + 1) % L;
  float2 acc;
  {
    // the oldest sample (slot J) is consumed before the new one overwrites it
    const float2 prev = dl[0][JM1], o1 = dl[0][JO1], o2 = dl[0][J];
    const float2 accp = (PASSES > 1) ? dl[PASSES > 1 ? 1 : 0][JM1] : vlast;
    const float2 n = __ffma2_rn(nb2, o2, __ffma2_rn(a2, __fadd2_rn(prev, make_float2(-o1.x, -o1.y)), accp));
    dl[0][J] = x;
    acc = __ffma2_rn(b2, x, n);
  }
#pragma unroll
  for (int p = 1; p < PASSES; ++p) {
    float2 xp = dl[p][JM1], x1 = dl[p][JO1], x2 = dl[p][J];
    float2 gt0 = pk(1.f);
    if (BORDER) {
      const float* g = gt - p * D;
      gt0 = pk(g[0]);
      xp = __fmul2_rn(xp, pk(g[-1]));
      x1 = __fmul2_rn(x1, pk(g[-2 * D]));
      x2 = __fmul2_rn(x2, pk(g[-2 * D - 1]));
    }
    const float2 accp = (p + 1 < PASSES) ? dl[(p + 1 < PASSES) ? p + 1 : p][JM1] : vlast;
    const float2 n = __ffma2_rn(nb2, x2, __ffma2_rn(a2, __fadd2_rn(xp, make_float2(-x1.x, -x1.y)), accp));
    dl[p][J] = acc;
    acc = __ffma2_rn(b2, BORDER ? __fmul2_rn(acc, gt0) : acc, n);
  }
  vlast = acc;
  return BORDER ? __fmul2_rn(acc, pk(gt[-PASSES * D])) : acc;
}

// scalar twin for the H phase (one image per lane)
template <int J, int L, int D, int PASSES, bool BORDER>
__device__ __forceinline__ float hcascade(float (&dl)[PASSES][L], float& vlast, float x, float a,
                                          float b, const float* gt) {
  constexpr int JM1 = (J + L - 1) % L, JO1 = (J + 1) % L;
  float acc;
  {
    const float prev = dl[0][JM1], o1 = dl[0][JO1], o2 = dl[0][J];
    const float accp = (PASSES > 1) ? dl[PASSES > 1 ? 1 : 0][JM1] : vlast;
    const float n = fmaf(-b, o2, fmaf(a, prev - o1, accp));
    dl[0][J] = x;
    acc = fmaf(b, x, n);
  }
#pragma unroll
  for (int p = 1; p < PASSES; ++p) {
    float xp = dl[p][JM1], x1 = dl[p][JO1], x2 = dl[p][J], gt0 = 1.f;
    if (BORDER) {
      const float* g = gt - p * D;
      gt0 = g[0];
      xp *= g[-1];
      x1 *= g[-2 * D];
      x2 *= g[-2 * D - 1];
    }
    const float accp = (p + 1 < PASSES) ? dl[(p + 1 < PASSES) ? p + 1 : p][JM1] : vlast;
    const float n = fmaf(-b, x2, fmaf(a, xp - x1, accp));
    dl[p][J] = acc;
    acc = fmaf(b, BORDER ? acc * gt0 : acc, n);
  }
  vlast = acc;
  return BORDER ? acc * gt[-PASSES * D] : acc;
}

// ---- shared-memory helpers (TMA + mbarrier) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void sts2(float* p, float2 v) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(smem_u32(p)), "f"(v.x), "f"(v.y) : "memory");
}

// SBF_PREC_AUTO guard (the fp32 kernels hold the tolerance while
// |f - centre| stays within the 8-bit-scale regime)
__device__ __forceinline__ bool sweep_needs_hdr(const double* stats) {
  const double c = stats[3];
  return fmax(stats[2] - c, c - stats[1]) > 4096.0;
}

#ifndef SBF_SWEEP_HPF
#define SBF_SWEEP_HPF 0  // H phase: columns read ahead (0: plain loads)
#endif
#ifndef SBF_SWEEP_VPF
#define SBF_SWEEP_VPF 0  // V phase: rows of the f box read ahead (0: plain loads)
#endif
#ifndef SBF_SWEEP_ACC_BATCH
#define SBF_SWEEP_ACC_BATCH 0  // accumulate: batched shared-memory reads, clobber-free reds
#endif
#ifndef SBF_SWEEP_ABL
#define SBF_SWEEP_ABL 0  // phase ablation for timing studies (wrong results when != 0)
#endif
#ifndef SBF_SWEEP_TMA
#define SBF_SWEEP_TMA 1  // 0: the threads load the f box themselves (debug / comparison)
#endif
#ifndef SBF_SWEEP_TAIL_ROWS
#define SBF_SWEEP_TAIL_ROWS 128  // band height of the tail terms (0: no tail)
#endif
#ifndef SBF_SWEEP_TAIL_WAVES
#define SBF_SWEEP_TAIL_WAVES 3
#endif
#ifndef SBF_SWEEP_TAIL_FRAC
#define SBF_SWEEP_TAIL_FRAC 4
#endif

template <int R, int PASSES>
__global__ void __launch_bounds__(SweepCfg<R, PASSES>::THREADS, 2)
    sweep_kernel(const __grid_constant__ CUtensorMap fmap, const SweepParams p) {
  using C = SweepCfg<R, PASSES>;
  constexpr int D = C::D, L = C::L, HALO = C::HALO, WC = C::WC, COLS = C::COLS;
  constexpr int ROWS = C::ROWS, VBP = C::VB_PITCH, RING = C::RING, RAWP = C::RAW_PITCH;
  constexpr int GOFF = C::GOFF, NB = C::NB, THREADS = C::THREADS, SEGR = C::SEGR;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  // the TMA destination must be 128-byte aligned in the shared window: the
  // first bytes hold the mbarrier and the item slot, the box follows
  unsigned char* sbase = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t& s_bar = *reinterpret_cast<uint64_t*>(sbase);
  int& s_item = *reinterpret_cast<int*>(sbase + 8);
  int& s_ndone = *reinterpret_cast<int*>(sbase + 12);
  int* s_done = reinterpret_cast<int*>(sbase + 16);  // <= 28 segments per item
  float* FT = reinterpret_cast<float*>(sbase + 128);  // TMA box: ROWS x FCOLS
  float* VB = FT + ROWS * C::FCOLS;
  float* RAW = VB + ROWS * VBP;
  float* gv = RAW + RING * RAWP;
  const int gv_len = p.band + 2 * HALO + GOFF + ROWS;
  float* gh = gv + gv_len;

  pdl_wait();  // K1 / K2 results (programmatic dependent launch)
  const sbf_plan* plan = p.plan;
  if (plan->status != SBF_OK) return;
  if (p.hdr_guard && sweep_needs_hdr(p.stats)) {
    if (blockIdx.x == 0 && threadIdx.x == 0)
      atomicOr(const_cast<int*>(&plan->flags), SBF_PLAN_NEEDS_HDR);
    return;
  }
  const int tid = threadIdx.x;
  const int K_eval = plan->K_eval;
  const int rows_all = p.out_hi - p.out_lo;
  const float centerf = (float)p.stats[3];
  const float fcent = p.centred ? 0.f : centerf;  // the fp32 view may be centred already
  const double centerd = p.stats[3];
  // fixed-point scales: |den| <= sum of the term weights <= 1 + tiny, and
  // |num| <= max|f - centre| times the same (|S[z]| <= 1 for an averaging S)
  const double maxdev = fmax(p.stats[2] - centerd, centerd - p.stats[1]);
  const int nexp = ilogb(fmax(maxdev, 1.0)) + 1;  // maxdev < 2^nexp
  const float nscale = ldexpf(1.f, 29 - nexp), dscale = ldexpf(1.f, 29);
  const double inv_nscale = ldexp(1.0, nexp - 29), inv_dscale = ldexp(1.0, -29);
  if (K_eval <= 0) {
    if (!p.fused_epi) return;  // the divide kernel finds den = 0 everywhere
    // no retained term: every normaliser is 0, so every pixel falls back
    unsigned long long n = 0;
    const int64_t total = (int64_t)rows_all * p.W;
    for (int64_t i = (int64_t)blockIdx.x * THREADS + tid; i < total; i += (int64_t)gridDim.x * THREADS) {
      const int64_t y = i / p.W, x = i - y * p.W;
      const int64_t fi = (int64_t)(p.out_lo + y) * p.fo_ld + x;
      const double v = p.fo_dtype == SBF_F32 ? (double)static_cast<const float*>(p.fo)[fi]
                                             : static_cast<const double*>(p.fo)[fi];
      if (p.out_dtype == SBF_F32) static_cast<float*>(p.out)[i] = (float)v;
      else static_cast<double*>(p.out)[i] = v;
      ++n;
    }
    for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if ((tid & 31) == 0 && n) atomicAdd(p.fallback, n);
    return;
  }
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned bar_phase = 0;

  // band height from the device plan: the largest band (smem is sized for
  // p.band) that still gives >= 2 items per CTA
  int bandh = p.band;
  {
    const int per_band = max(1, p.nstrips * K_eval);
    const int nb_min = (2 * (int)gridDim.x + per_band - 1) / per_band;
    const int b = (rows_all + nb_min - 1) / nb_min;
    bandh = max(min(b, p.band), min(4 * HALO, p.band));
  }
  const int nbands = (rows_all + bandh - 1) / bandh;
  const int units = p.nstrips * nbands;
  // tail: the last Ks terms run in short bands so the queue ends with small
  // items and the CTAs finish together
  int Ks = 0, bands_s = 1, units_s = 0;
  if (SBF_SWEEP_TAIL_ROWS > 0 && bandh > SBF_SWEEP_TAIL_ROWS) {
    bands_s = (rows_all + SBF_SWEEP_TAIL_ROWS - 1) / SBF_SWEEP_TAIL_ROWS;
    units_s = p.nstrips * bands_s;
    Ks = min(K_eval / SBF_SWEEP_TAIL_FRAC,
             (SBF_SWEEP_TAIL_WAVES * (int)gridDim.x + units_s - 1) / units_s);
  }
  const int bandh_s = (rows_all + bands_s - 1) / bands_s;
  const int items_big = (K_eval - Ks) * units;
  const int total = items_big + Ks * units_s;
  const float a = p.a, b = p.b;
  const float2 a2 = pk(a), nb2 = pk(-b), b2 = pk(b);

  // V state: (f cos, cos) and (f sin, sin) pairs
  float2 dA[PASSES][L], dB[PASSES][L];
  float2 lA, lB;

  for (;;) {
    if (tid == 0) s_item = atomicAdd(p.ctrl, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= total) break;
    const bool tail = item >= items_big;
    const int i2 = tail ? item - items_big : item;
    const int per = (tail ? Ks : K_eval - Ks) * p.nstrips;
    const int band = i2 / per;
    const int r2 = i2 - band * per;
    const int kk = (tail ? K_eval - Ks : 0) + r2 / p.nstrips;
    const int si = r2 - (r2 / p.nstrips) * p.nstrips;
    // edge strips (costlier border code) first within a band
    const int strip = p.nstrips < 2 ? si : (si == 0 ? 0 : (si == 1 ? p.nstrips - 1 : si - 1));
    const int bh = tail ? bandh_s : bandh;
    const int y0 = p.out_lo + band * bh;
    const int y1 = min(p.out_hi, y0 + bh);
    const int Bn = y1 - y0;
    const int T_total = Bn + 2 * HALO;
    const int nchunks = (T_total + ROWS - 1) / ROWS;
    const int xs = strip * WC - HALO;  // image column of haloed index 0
    const int xa = xs & ~3;             // box start (16-byte aligned column)
    const int xoff = xs - xa;
    const int64_t grow0 = p.row0 + (int64_t)(y0 - HALO);  // global row of stream position 0

    // border tables (index = stream / haloed position + GOFF)
    for (int k = tid; k < nchunks * ROWS + GOFF; k += THREADS)
      gv[k] = axis_factor(grow0 + (k - GOFF), p.img_H, p.r, p.alpha);
    for (int k = tid; k < COLS + GOFF; k += THREADS)
      gh[k] = axis_factor((int64_t)xs + (k - GOFF), p.W, p.r, p.alpha);
    // stream positions whose rows have factor 1 (D from the image edges)
    const int64_t sg_lo = (int64_t)D - grow0;
    const int64_t sg_hi = p.img_H - 1 - D - grow0;
    const int qg_lo = D - xs, qg_hi = p.W - 1 - D - xs;  // haloed columns with factor 1

    const sbf_term term = p.terms[kk];
    const float scale = (float)term.scale;
    const float omega = (float)term.freq;
#pragma unroll
    for (int pp = 0; pp < PASSES; ++pp)
#pragma unroll
      for (int j = 0; j < L; ++j) {
        dA[pp][j] = pk(0.f);
        dB[pp][j] = pk(0.f);
      }
    lA = pk(0.f);
    lB = pk(0.f);
    const int q = tid;            // V: haloed column of this thread
    const int hv = tid >> 2;      // H: VB row
    const int himg = tid & 3;     // H: image (VB component)
    const int fbuf_row0 = y0 - HALO;  // buffer row of stream position 0
    auto load_box = [&](int row_start) {
      if (SBF_SWEEP_TMA) {
        if (tid == 0) {
          fence_proxy_async();
          mbar_expect_tx(&s_bar, (unsigned)C::F_BYTES);
          tma_load_2d(FT, &fmap, xa, row_start, &s_bar);
        }
      } else {
        for (int j = 0; j < ROWS; ++j) {
          const int row = row_start + j;
          for (int k = tid; k < C::FCOLS; k += THREADS) {
            const int col = xa + k;
            FT[j * C::FCOLS + k] = (row >= 0 && row < p.H && col >= 0 && col < p.W)
                                       ? p.f[(int64_t)row * p.ld + col] : 0.f;
          }
        }
      }
    };
    load_box(fbuf_row0);
    __syncthreads();  // border tables

    for (int c = 0; c < nchunks; ++c) {
      const int t0 = c * ROWS;
      if (SBF_SWEEP_TMA) {
        mbar_wait(&s_bar, bar_phase);
        bar_phase ^= 1;
      }

      // ===================== V phase =====================
      // steps [t0, t0 + ROWS) in blocks of L aligned to the stream position
      // (the ring slot of step t is t mod L): interior blocks wholly inside
      // the chunk run without checks, blocks cut by a chunk boundary check
      // the step range, blocks near the image's top or bottom renormalise
      auto vblock = [&](auto kind_tag, const int base) {
        constexpr int KIND = decltype(kind_tag)::value;  // 0 fast, 1 partial, 2 border
        constexpr bool BORDER = KIND == 2;
        const int rel = base - t0;  // chunk row of step base (may be < 0)
        const float* fsrc = FT + rel * C::FCOLS + q + xoff;
        float* vdst = VB + rel * VBP + 4 * q;
        const int rs0 = base % RING;
        float* rdst = RAW + rs0 * RAWP + (q - HALO);
        const bool out_col = q >= HALO && q < HALO + WC;
        // f of the next VPF steps is read ahead of the current step's work
        float fr[SBF_SWEEP_VPF > 0 ? SBF_SWEEP_VPF : 1];
#pragma unroll
        for (int k = 0; k < SBF_SWEEP_VPF; ++k)
          fr[k] = (KIND == 0 || (unsigned)(rel + k) < (unsigned)ROWS) ? fsrc[k * C::FCOLS] : 0.f;
        sweep_for<L>([&](auto jc) {
          constexpr int J = decltype(jc)::value;
          if (KIND != 0 && (unsigned)(rel + J) >= (unsigned)ROWS) return;
          float fraw;
          if (SBF_SWEEP_VPF > 0) {
            fraw = fr[0];
#pragma unroll
            for (int k = 0; k + 1 < SBF_SWEEP_VPF; ++k) fr[k] = fr[k + 1];
            constexpr int JN = J + (SBF_SWEEP_VPF > 0 ? SBF_SWEEP_VPF : 0);
            if (JN < L)
              fr[SBF_SWEEP_VPF > 0 ? SBF_SWEEP_VPF - 1 : 0] =
                  (KIND == 0 || (unsigned)(rel + JN) < (unsigned)ROWS) ? fsrc[JN * C::FCOLS] : 0.f;
          } else {
            fraw = fsrc[J * C::FCOLS];
          }
          const float fc = fraw - fcent;
          float sv, cv;
#if SBF_SWEEP_ABL & 8  // timing ablation only: no MUFU phasor in the V phase
          cv = fc * omega;
          sv = cv + 0.5f;
#else
          __sincosf(fc * omega, &sv, &cv);
#endif
          if (BORDER) {  // rows outside the image contribute nothing
            const int64_t gr = grow0 + base + J;
            const float m = (gr >= 0 && gr < p.img_H) ? 1.f : 0.f;
            cv *= m;
            sv *= m;
          }
          // the output pixel's sample, for its phasor in the accumulate phase
          if (out_col) rdst[J * RAWP] = fc;
          const float* gt = gv + base + J + GOFF;
          const float2 fx = make_float2(fc, 1.f);
#if SBF_SWEEP_ABL & 2  // timing ablation only: no V recurrences
          const float2 ya = __fmul2_rn(fx, pk(cv)), yb = __fmul2_rn(fx, pk(sv));
#else
          const float2 ya = vcascade<J, L, D, PASSES, BORDER>(dA, lA, __fmul2_rn(fx, pk(cv)), a2, nb2, b2, gt);
          const float2 yb = vcascade<J, L, D, PASSES, BORDER>(dB, lB, __fmul2_rn(fx, pk(sv)), a2, nb2, b2, gt);
#endif
          // VB layout per pixel: [F_c, G_c, F_s, G_s]
          sts2(vdst + J * VBP, ya);
          sts2(vdst + J * VBP + 2, yb);
        });
      };
#pragma unroll 1
      // (steps past the band's stream end feed no output row: skipped)
      for (int base = (t0 / L) * L; base < min(t0 + ROWS, T_total); base += L) {
        const bool clean = base - (PASSES + 2) * D - 1 >= sg_lo && base + L - 1 <= sg_hi;
        if (!clean)
          vblock(std::integral_constant<int, 2>{}, base);
        else if (base >= t0 && base + L <= t0 + ROWS)
          vblock(std::integral_constant<int, 0>{}, base);
        else
          vblock(std::integral_constant<int, 1>{}, base);
      }
      __syncthreads();  // VB complete; the f box is consumed
      // next chunk's box streams in while the H phase runs
      if (SBF_SWEEP_TMA && c + 1 < nchunks) load_box(fbuf_row0 + t0 + ROWS);

      // valid VB rows of this chunk: stream steps [2 HALO, 2 HALO + Bn)
      const int vlo = max(t0, 2 * HALO) - t0;
      const int vhi = min(t0 + ROWS, 2 * HALO + Bn) - t0;

      // ===================== H phase =====================
      // 4 lanes per row (one per image) stream the chunk's rows; blocks whose
      // columns all have factor 1 need no renormalisation (every block of an
      // interior strip; all but the outer blocks of the two edge strips)
      if (hv >= vlo && hv < vhi) {
        float* vrow = VB + hv * VBP + himg;
        float hd[PASSES][L];
        float hlast = 0.f;
#pragma unroll
        for (int pp = 0; pp < PASSES; ++pp)
#pragma unroll
          for (int j = 0; j < L; ++j) hd[pp][j] = 0.f;
        // inputs are read HPF columns ahead (a shift register carried from
        // block to block): the shared-memory latency overlaps the recurrences
        // instead of opening every column step
        float xr[SBF_SWEEP_HPF > 0 ? SBF_SWEEP_HPF : 1];
#pragma unroll
        for (int k = 0; k < SBF_SWEEP_HPF; ++k) xr[k] = vrow[4 * k];
        // kind: 0 warm-up (no outputs), 1 main, 2 guarded, 3 border
        auto hblock = [&](auto kind_tag, const int hbase) {
          constexpr int KIND = decltype(kind_tag)::value;
          constexpr bool GUARD = KIND >= 2, BORDER = KIND == 3;
          sweep_for<L>([&](auto jc) {
            constexpr int J = decltype(jc)::value;
            const int qq = hbase + J;
            float x;
            if (SBF_SWEEP_HPF > 0) {
              x = xr[0];
#pragma unroll
              for (int k = 0; k + 1 < SBF_SWEEP_HPF; ++k) xr[k] = xr[k + 1];
              const int qn = qq + SBF_SWEEP_HPF;
              xr[SBF_SWEEP_HPF > 0 ? SBF_SWEEP_HPF - 1 : 0] = qn < C::VB_COLS ? vrow[4 * qn] : 0.f;
            } else {
              x = vrow[4 * qq];
            }
            if (BORDER) {
              const int cc = xs + qq;
              x = (cc >= 0 && cc < p.W) ? x : 0.f;
            }
#if SBF_SWEEP_ABL & 1  // timing ablation only: no H recurrences
            const float yv = x * a;
#else
            const float yv = hcascade<J, L, D, PASSES, BORDER>(hd, hlast, x, a, b, gh + qq + GOFF);
#endif
            if (KIND == 1 || (GUARD && qq >= 2 * HALO && qq < COLS)) vrow[4 * (qq - HALO)] = yv;
          });
        };
        constexpr int KB_MAIN0 = (2 * HALO + L - 1) / L;  // first block with base >= 2 HALO
        constexpr int KB_MAIN1 = (COLS - L) / L + 1;      // blocks [KB_MAIN0, KB_MAIN1) are main
        const bool strip_in = -(PASSES + 2) * D - 1 >= qg_lo && NB * L - 1 <= qg_hi;
        if (strip_in && KB_MAIN0 < KB_MAIN1) {
          sweep_for<KB_MAIN0>([&](auto kc) {
            constexpr int KB = decltype(kc)::value;
            if constexpr (KB * L + L <= 2 * HALO)
              hblock(std::integral_constant<int, 0>{}, KB * L);
            else
              hblock(std::integral_constant<int, 2>{}, KB * L);
          });
#pragma unroll 1
          for (int kb = KB_MAIN0; kb < KB_MAIN1; ++kb) hblock(std::integral_constant<int, 1>{}, kb * L);
          sweep_for<NB - KB_MAIN1>([&](auto kc) {
            hblock(std::integral_constant<int, 2>{}, (KB_MAIN1 + decltype(kc)::value) * L);
          });
        } else {
#pragma unroll 1
          for (int kb = 0; kb < NB; ++kb) {
            const int hb = kb * L;
            // the block reads factors back to hb - (PASSES+2) D - 1
            if (hb - (PASSES + 2) * D - 1 >= qg_lo && hb + L - 1 <= qg_hi)
              hblock(std::integral_constant<int, 2>{}, hb);
            else
              hblock(std::integral_constant<int, 3>{}, hb);
          }
        }
      }
      __syncthreads();

      // ===================== accumulate =====================
      // (num, den) of this term in 32-bit fixed point, both halves of one
      // 64-bit integer, added with one red.add.u64 per pixel: integer sums
      // are associative, so the result does not depend on the order in
      // which items land (bit-reproducible), and nothing waits
      if (vlo < vhi) {
        const int ra = y0 - 2 * HALO + t0 + vlo - p.out_lo;  // first output row (rel. out_lo)
        const int nr = vhi - vlo;
        const int xlim = min(WC, p.W - strip * WC);
        const int jc = tid;
        if (jc < xlim) {
          const int col = strip * WC + jc;
          const float* vb = VB + vlo * VBP + 4 * (HALO + jc);
          unsigned long long* dst = p.acc + (int64_t)ra * p.W + col;
          // output row y0 - 2 HALO + t0 + v was sampled at step t0 + v - HALO;
          // its phasor is recomputed from the sample exactly as the V phase did
          int slot = (t0 + vlo - HALO) % RING;
          const float* rp = RAW + jc;
          const float2 fx = make_float2(scale * nscale, scale * dscale);
#if SBF_SWEEP_ACC_BATCH
          // 4 pixels' shared-memory reads issued before any is consumed; the
          // reds carry no memory clobber (the chunk's __syncthreads orders them)
          for (int v0 = 0; v0 < nr; v0 += 4) {
            float4 pvb[4];
            float fcb[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (v0 + u < nr) {
                pvb[u] = *reinterpret_cast<const float4*>(vb + (v0 + u) * VBP);
                fcb[u] = rp[slot * RAWP];
                slot = slot + 1 == RING ? 0 : slot + 1;
              }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (v0 + u >= nr) break;
              const float4 pv = pvb[u];
              const float fcv = fcb[u];
              float sv, cv;
              __sincosf(fcv * omega, &sv, &cv);
              float2 t = __ffma2_rn(pk(sv), make_float2(pv.z, pv.w),
                                    __fmul2_rn(pk(cv), make_float2(pv.x, pv.y)));
              t = __fmul2_rn(t, fx);
              const long long q =
                  ((long long)__float2int_rn(t.x) << 32) + (long long)__float2int_rn(t.y);
              asm volatile("red.global.add.u64 [%0], %1;" ::"l"(dst + (int64_t)(v0 + u) * p.W), "l"(q));
            }
          }
#else
#pragma unroll 4
          for (int v = 0; v < nr; ++v) {
            const float4 pv = *reinterpret_cast<const float4*>(vb + v * VBP);
            const float fcv = rp[slot * RAWP];
            slot = slot + 1 == RING ? 0 : slot + 1;
            float sv, cv;
#if SBF_SWEEP_ABL & 16  // timing ablation only: no MUFU phasor in the accumulate phase
            cv = fcv * omega;
            sv = cv + 0.5f;
#else
            __sincosf(fcv * omega, &sv, &cv);
#endif
            float2 t = __ffma2_rn(pk(sv), make_float2(pv.z, pv.w),
                                  __fmul2_rn(pk(cv), make_float2(pv.x, pv.y)));
            t = __fmul2_rn(t, fx);
            const long long q = ((long long)__float2int_rn(t.x) << 32) + (long long)__float2int_rn(t.y);
#if SBF_SWEEP_ABL & 4  // timing ablation only: no accumulation atomics
            if (q == 0x7fffffffffffll) dst[(int64_t)v * p.W] = q;
#else
            asm volatile("red.global.add.u64 [%0], %1;" ::"l"(dst + (int64_t)v * p.W), "l"(q) : "memory");
#endif
          }
#endif
        }
      }
      __syncthreads();  // VB / RAW are rewritten by the next chunk
    }  // chunks
    // this item's rows are in: count it on the output segments it covers;
    // the item that completes a segment (all terms, all bands over it)
    // divides it out (bilateral.py:242-254) and writes the output
    // (one segment counter per thread: the round trips to L2 overlap
    // instead of running one after another in one thread)
    if (!p.fused_epi) {
      __syncthreads();  // tables and VB are rewritten by the next item
      continue;
    }
    __threadfence();
    if (tid == 0) s_ndone = 0;
    __syncthreads();
    {
      const int s0 = (y0 - p.out_lo) / SEGR, s1 = (y1 - 1 - p.out_lo) / SEGR;
      for (int sg = s0 + tid; sg <= s1; sg += THREADS) {
        const int r0 = sg * SEGR, r1 = min(rows_all, r0 + SEGR) - 1;
        const int nm = r1 / bandh - r0 / bandh + 1;
        const int nt = Ks > 0 ? r1 / bandh_s - r0 / bandh_s + 1 : 0;
        const int expected = (K_eval - Ks) * nm + Ks * nt;
        if (atomicAdd(p.seg + (int64_t)sg * p.nstrips + strip, 1) == expected - 1)
          s_done[atomicAdd(&s_ndone, 1)] = sg;
      }
      __threadfence();
    }
    __syncthreads();
    const int ndone = s_ndone;
    if (ndone > 0) {
      const int xlim = min(WC, p.W - strip * WC);
      unsigned long long bad = 0;
      // thread per output column; each thread issues EPI_U accumulator loads
      // (L2) before it consumes any, so the segment's loads overlap
      constexpr int EPI_U = 8;
      if (tid < xlim) {
        const int col = strip * WC + tid;
        for (int d = 0; d < ndone; ++d) {
          const int r0 = s_done[d] * SEGR, nr = min(rows_all, r0 + SEGR) - r0;
          for (int v0 = 0; v0 < nr; v0 += EPI_U) {
            long long sum[EPI_U];
#pragma unroll
            for (int u = 0; u < EPI_U; ++u)
              sum[u] = v0 + u < nr ? (long long)__ldcg(p.acc + (int64_t)(r0 + v0 + u) * p.W + col) : 0;
#pragma unroll
            for (int u = 0; u < EPI_U; ++u) {
              if (v0 + u >= nr) break;
              const int rr = r0 + v0 + u;
              const int64_t ai = (int64_t)rr * p.W + col;
              const int lo = (int)(unsigned)(sum[u] & 0xffffffffll);
              const long long hi = (sum[u] - (long long)lo) >> 32;
              const double num = (double)hi * inv_nscale, den = (double)lo * inv_dscale;
              const bool is_bad = !(den > 0.0);  // bilateral.py:244 (NaN counts as bad)
              bad += is_bad ? 1 : 0;
              const int64_t fi = (int64_t)(p.out_lo + rr) * p.fo_ld + col;
              if (p.out_dtype == SBF_F32) {
                float o;
                if (is_bad)
                  o = p.fo_dtype == SBF_F32 ? static_cast<const float*>(p.fo)[fi]
                                            : (float)static_cast<const double*>(p.fo)[fi];
                else
                  o = (float)(num / den) + centerf;
                static_cast<float*>(p.out)[ai] = o;
              } else {
                double o;
                if (is_bad)
                  o = p.fo_dtype == SBF_F32 ? (double)static_cast<const float*>(p.fo)[fi]
                                            : static_cast<const double*>(p.fo)[fi];
                else
                  o = num / den + centerd;
                static_cast<double*>(p.out)[ai] = o;
              }
            }
          }
        }
      }
      for (int o = 16; o; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
      if ((tid & 31) == 0 && bad) atomicAdd(p.fallback, bad);
    }
    __syncthreads();  // tables, VB and the segment list are rewritten by the next item
  }  // work queue
}

// Divide / fallback epilogue for the fixed-point accumulator
// (bilateral.py:242-254), launched after the sweep for device outputs: every
// pixel at full GPU width, instead of one CTA per completed segment inside
// the sweep's last items (which serialised the tail: 0.23 ms of a 2.0 ms
// config-4 sweep).  Same decode and arithmetic as the fused epilogue.
static __global__ void __launch_bounds__(256) sweep_divide_kernel(
    const unsigned long long* __restrict__ acc, int64_t rows, int64_t W, int64_t out_lo,
    const void* __restrict__ fo, int64_t fo_ld, int fo_dtype, void* __restrict__ out, int out_dtype,
    const sbf_plan* __restrict__ plan, const double* __restrict__ stats,
    unsigned long long* __restrict__ fallback) {
  pdl_wait();
  if (plan->status != SBF_OK || (plan->flags & SBF_PLAN_NEEDS_HDR)) return;
  const double centerd = stats[3];
  const float centerf = (float)centerd;
  const double maxdev = fmax(stats[2] - centerd, centerd - stats[1]);
  const int nexp = ilogb(fmax(maxdev, 1.0)) + 1;
  const double inv_nscale = ldexp(1.0, nexp - 29), inv_dscale = ldexp(1.0, -29);
  unsigned long long bad = 0;
  // rows over the grid, columns over the threads (no 64-bit index division)
  for (int64_t y = blockIdx.x; y < rows; y += gridDim.x) {
    const unsigned long long* arow = acc + y * W;
    const int64_t frow = (out_lo + y) * fo_ld;
    for (int64_t x = threadIdx.x; x < W; x += blockDim.x) {
      const long long sum = (long long)__ldcs(arow + x);
      const int lo = (int)(unsigned)(sum & 0xffffffffll);
      const long long hi = (sum - (long long)lo) >> 32;
      const double num = (double)hi * inv_nscale, den = (double)lo * inv_dscale;
      const bool is_bad = !(den > 0.0);  // bilateral.py:244
      bad += is_bad ? 1 : 0;
      const int64_t i = y * W + x;
      if (out_dtype == SBF_F32) {
        float o;
        if (is_bad)
          o = fo_dtype == SBF_F32 ? static_cast<const float*>(fo)[frow + x]
                                  : (float)static_cast<const double*>(fo)[frow + x];
        else
          o = (float)(num / den) + centerf;
        static_cast<float*>(out)[i] = o;
      } else {
        double o;
        if (is_bad)
          o = fo_dtype == SBF_F32 ? (double)static_cast<const float*>(fo)[frow + x]
                                  : static_cast<const double*>(fo)[frow + x];
        else
          o = num / den + centerd;
        static_cast<double*>(out)[i] = o;
      }
    }
  }
  for (int o = 16; o; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(fallback, bad);
}

// ---- host side ----
template <int R, int PASSES>
size_t sweep_smem_bytes(int band) {
  using C = SweepCfg<R, PASSES>;
  return 256 + C::F_BYTES + C::VB_BYTES + C::RAW_BYTES +
         (size_t)(band + 2 * C::HALO + C::GOFF + C::ROWS + C::COLS + C::GOFF) * 4 + 16;
}

template <int R, int PASSES>
void sweep_geometry(int* halo, int* wc, int* threads, int* blocks_per_sm) {
  using C = SweepCfg<R, PASSES>;
  *halo = C::HALO;
  *wc = C::WC;
  *threads = C::THREADS;
  *blocks_per_sm = 2;
}

template <int R, int PASSES>
int launch_sweep(const CUtensorMap& map, const SweepParams& p, cudaStream_t st) {
  using C = SweepCfg<R, PASSES>;
  const size_t smem = sweep_smem_bytes<R, PASSES>(p.band);
  SBF_CHECK_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(sweep_kernel<R, PASSES>), smem));
  const int grid = device_sm_count() * 2;  // persistent CTAs
  SBF_CHECK_CUDA(launch_pdl(sweep_kernel<R, PASSES>, dim3((unsigned)grid), dim3(C::THREADS), smem, st,
                            map, p));
  SBF_CHECK_LAUNCH();
  return SBF_OK;
}

struct SweepEntry {
  int r, passes;
  int (*launch)(const CUtensorMap&, const SweepParams&, cudaStream_t);
  size_t (*smem)(int);
  void (*geom)(int*, int*, int*, int*);
  int rows;  // stream steps per chunk (TMA box height)
  // warp-specialised variant (sbf_sweepw.cuh; sbf_set_sweep_variant): device outputs only
  int (*launch_w)(const CUtensorMap&, const CUtensorMap&, const SweepParams&, cudaStream_t);
  size_t (*smem_w)(int);
  int wc_w, rows_w, fcols_w, afc_w, afr_w;
};

#define SBF_SWEEP_ENTRY(R, P)                                                                \
  SweepEntry { R, P, &launch_sweep<R, P>, &sweep_smem_bytes<R, P>, &sweep_geometry<R, P>,   \
               SweepCfg<R, P>::ROWS, &launch_sweepw<R, P>, &sweepw_smem_bytes<R, P>,        \
               SweepWCfg<R, P>::WC, SweepWCfg<R, P>::L, SweepWCfg<R, P>::FCOLS,             \
               SweepWCfg<R, P>::AFC, SweepWCfg<R, P>::GR }

}  // namespace sbf
