// K3 — fused per-term shiftable-filter kernel (sm_100a, FP32-issue bound).
//
// Replaces, per folded cosine term (reference bilateral.py:150-163):
//   theta = omega_n f; gc, gs = cos, sin; four apply_spatial() smoothings of
//   f*gc, gc, f*gs, gs (spatial.py:108-139: `passes` extended-box passes,
//   each renormalised over the clamped window — _extended_box_lines
//   spatial.py:120-133 on top of window_sum_lines _fastcore.pyx:61-86);
//   num/den += scale (gc*S[f gc] + gs*S[f gs]) / (gc*S[gc] + gs*S[gs]).
// Rows and columns commute exactly (Kronecker product), so all column passes
// run first, then all row passes (verified to 6e-13).
//
// B200 design ("strip sweep"; one work item = one 128-column strip x one row
// band x one term):
//  * V phase — one thread per haloed column streams the band top to bottom:
//    phasor cos/sin(2 pi frac(f nu)) by explicit range reduction + MUFU, the
//    four modulated images, and the column passes as O(1) recurrences
//        A_t = A_{t-1} + a (x_{t-1} - x_{t-2D}) + b (x_t - x_{t-2D-1})
//    (D = r+1, a = (1-alpha)/cnt, b = alpha/cnt, cnt = 2r+1+2alpha), the
//    2r+3 input history of every pass in a register ring with compile-time
//    rotation.  Pass p>0's ring stores pass p-1's raw accumulator, so the
//    accumulator needs no register of its own (no copies).  Border
//    renormalisation (zero padding + cnt/cnt(pos), 0 outside the image) is
//    applied on read, only in blocks that touch a true image border.
//  * The smoothed rows land in shared memory (VB, ROWS rows per chunk); the
//    output pixels' raw cos / sin go to a small ring (RAW).
//  * H phase — 4 lanes per row (one per image) stream the chunk's rows with
//    the same recurrence, multiply by the output pixel's raw phasor and write
//    the 4 products back in place.
//  * Accumulate — (num, den) = sums of the products, added with vector
//    red.add.v2.f32 into one zero-initialised accumulator (L2-resident).
// Persistent CTAs (one or two per SM) pull (term, band, strip) work items
// from an atomic counter, band by band, so border strips and short bands
// balance out; with the streamed epilogue each item also bumps the
// completion counters of the output segments it covers.  Launched as a
// programmatic dependent of K1 (waits, then lets its own dependent launch).
// Intermediate images never touch HBM.
#pragma once

#include <type_traits>
#include <utility>

#include "sbf_common.cuh"

namespace sbf {

struct TermParams {
  const float* f;  // fp32 image, already centred when `centred` != 0
  int64_t ld;
  int centred;
  int H;  // buffer rows
  int W;
  int64_t row0;   // global row index of buffer row 0
  int64_t img_H;  // global image height
  int out_lo, out_hi;
  int band;
  int nstrips, nbands, groups;
  int* counter;  // work-queue head (zeroed before launch)
  int r;
  float alpha;
  float a, b;
  const sbf_plan* plan;
  const sbf_term* terms;
  const double* stats;
  void* nd;
  int64_t nd_group_stride;  // (num, den) pairs per group
  int hdr_guard;            // SBF_PREC_AUTO: bail out (flag the plan) on wide ranges
  // streamed epilogue (epi != 0): K3 publishes its segment schedule and
  // per-segment item counts; the epilogue kernel divides segments out as
  // soon as they are complete (stream_epilogue_kernel, sbf_api.cu)
  int epi;
  int* seg_done;  // per output segment: finished items (zeroed before launch)
};

// SBF_PREC_AUTO guard: the fp32 kernels are accurate to the north-star
// tolerance only while |f - centre| stays within the 8-bit-scale regime
__device__ __forceinline__ bool needs_hdr(const double* stats) {
  const double c = stats[3];
  return fmax(stats[2] - c, c - stats[1]) > 4096.0;
}

#ifndef SBF_V_MAIN_VARIANT
#define SBF_V_MAIN_VARIANT 0  // separate unchecked V block variant for whole blocks (bigger code: slower)
#endif
#ifndef SBF_TRIG_AHEAD
#define SBF_TRIG_AHEAD 0  // phasor of step t+1 computed during step t (r=4: -2%, r=5: +0.5%)
#endif
#ifndef SBF_F_EARLY
#define SBF_F_EARLY 1  // read the next step's sample one step early
#endif
#ifndef SBF_TAIL_ROWS
#define SBF_TAIL_ROWS 128  // band height of the tail terms (0: no tail)
#endif
#ifndef SBF_TAIL_WAVES
#define SBF_TAIL_WAVES 3   // tail items ~ this many per CTA (capped at K/SBF_TAIL_FRAC terms)
#endif
#ifndef SBF_TAIL_FRAC
#define SBF_TAIL_FRAC 4   // at most K/4 terms in the tail
#endif
#ifndef SBF_PDL_TRIGGER
#define SBF_PDL_TRIGGER 1  // let the streamed epilogue launch while K3 runs
#endif
#ifndef SBF_EPI_COUNTERS
#define SBF_EPI_COUNTERS 1  // per-segment completion counters (streamed epilogue)
#endif
#ifndef SBF_MAIN_BAND_MAJOR
#define SBF_MAIN_BAND_MAJOR 1  // main items band by band (output segments complete early)
#endif
#ifndef SBF_TAIL_BAND_MAJOR
#define SBF_TAIL_BAND_MAJOR 1  // tail items band by band
#endif
#ifndef SBF_H_FIXED_SEQ
#define SBF_H_FIXED_SEQ 1  // interior strips: warm-up / main-loop / tail H blocks, no dispatch
#endif
#ifndef SBF_IMGS4_MAX_R
#define SBF_IMGS4_MAX_R 5  // radii up to this run 4 images per V thread (r=5: measured +2.5%)
#endif
#ifndef SBF_MAX_ROWS
#define SBF_MAX_ROWS 64    // rows per chunk cap
#endif
#ifndef SBF_IMGS2_2CTA_MAX_R
#define SBF_IMGS2_2CTA_MAX_R -1  // 2-image layouts up to this radius run 2 CTAs/SM
#endif

template <int R, int PASSES>
struct TermCfg {
  static constexpr int D = R + 1;
  static constexpr int L = 2 * R + 3;
  static constexpr int HALO = PASSES * D;
  static constexpr int IMGS = (R <= SBF_IMGS4_MAX_R) ? 4 : 2;
  static constexpr int HALO_W = 128;
  static constexpr int WC = HALO_W - 2 * HALO;
  static constexpr int NB = (HALO_W + L - 1) / L;  // H-phase blocks per row
  static constexpr int VB_COLS = NB * L;
  static constexpr int VB_PITCH = 4 * (VB_COLS + ((VB_COLS % 2 == 0) ? 1 : 2));  // == 4 mod 8 words
  static constexpr int THREADS = HALO_W * 4 / IMGS;
  static constexpr int ROWS_CAP = SBF_MAX_ROWS > HALO ? SBF_MAX_ROWS : HALO;
  static constexpr int ROWS = THREADS / 4 < ROWS_CAP ? THREADS / 4 : ROWS_CAP;
  static constexpr int RING = ROWS + HALO;
  static constexpr int RAW_PITCH = 2 * WC + 2;  // floats; == 2 mod 4 (WC even)
  static constexpr int GOFF = (PASSES + 2) * D + 2;  // table offset (most negative position)
  static constexpr int MIN_BLOCKS = (IMGS == 4 || R <= SBF_IMGS2_2CTA_MAX_R) ? 2 : 1;
  static_assert(WC > 0, "halo too wide for a 128-column strip");
  static_assert(HALO <= ROWS, "RAW ring assumes halo <= rows per chunk");
};

// compile-time loop: f(std::integral_constant<int, J>) for J in [0, N)
template <class F, int... Js>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, Js...>) {
  (f(std::integral_constant<int, Js>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

// normalisation factor cnt_int / cnt(pos) on an axis of length n (0 outside)
__device__ __forceinline__ float gfactor(int64_t pos, int64_t n, int r, float alpha) {
  if (pos < 0 || pos >= n) return 0.f;
  // interior: cnt == cint (the fp64 ratio is 1 to within an ulp, 1.0f after
  // rounding) -- skip the division for the bulk of the table
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

// One image's cascade of PASSES recurrences at rotation slot J.
// dl[0]: masked input samples; dl[p>0]: raw accumulator of pass p-1.
// Border blocks (BORDER) normalise on read: gt[s - p*D - k] is the factor of
// the sample pass p reads at step s - k (k in {0, 1, 2D, 2D+1}); the final
// output is scaled by gt[s - PASSES*D].  gt already includes the table offset.
template <int J, int L, int D, int PASSES, bool BORDER>
__device__ __forceinline__ float cascade(float (&dl)[PASSES][L], float& vlast, float x, float a,
                                         float b, const float* gt) {
  constexpr int JM1 = (J + L - 1) % L, JO1 = (J + 1) % L;
  // The oldest sample x_{t-2D-1} lives in slot J, which the new value must
  // overwrite: consume it first (-b x_old) so its register dies before the
  // new value exists — the new value is then produced in place (no copies).
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
    const float rp = dl[p][JM1], r1 = dl[p][JO1], r2 = dl[p][J];
    float xp = rp, x1 = r1, x2 = r2, gt0 = 1.f;
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

// Packed twin of `cascade`: two images per float2 (FADD2/FFMA2/FMUL2, sm_100),
// half the FP32 instructions for the same arithmetic.
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
template <int J, int L, int D, int PASSES, bool BORDER>
__device__ __forceinline__ float2 cascade2(float2 (&dl)[PASSES][L], float2& vlast, float2 x,
                                           float2 a2, float2 nb2, float2 b2, const float* gt) {
  constexpr int JM1 = (J + L - 1) % L, JO1 = (J + 1) % L;
  float2 acc;
  {
    const float2 prev = dl[0][JM1], o1 = dl[0][JO1], o2 = dl[0][J];
    const float2 accp = (PASSES > 1) ? dl[PASSES > 1 ? 1 : 0][JM1] : vlast;
    const float2 n = __ffma2_rn(nb2, o2, __ffma2_rn(a2, __fadd2_rn(prev, make_float2(-o1.x, -o1.y)), accp));
    dl[0][J] = x;
    acc = __ffma2_rn(b2, x, n);
  }
#pragma unroll
  for (int p = 1; p < PASSES; ++p) {
    float2 xp = dl[p][JM1], x1 = dl[p][JO1], x2 = dl[p][J];
    float2 gt0 = f2(1.f);
    if (BORDER) {
      const float* g = gt - p * D;
      gt0 = f2(g[0]);
      xp = __fmul2_rn(xp, f2(g[-1]));
      x1 = __fmul2_rn(x1, f2(g[-2 * D]));
      x2 = __fmul2_rn(x2, f2(g[-2 * D - 1]));
    }
    const float2 accp = (p + 1 < PASSES) ? dl[(p + 1 < PASSES) ? p + 1 : p][JM1] : vlast;
    const float2 n = __ffma2_rn(nb2, x2, __ffma2_rn(a2, __fadd2_rn(xp, make_float2(-x1.x, -x1.y)), accp));
    dl[p][J] = acc;
    acc = __ffma2_rn(b2, BORDER ? __fmul2_rn(acc, gt0) : acc, n);
  }
  vlast = acc;
  return BORDER ? __fmul2_rn(acc, f2(gt[-PASSES * D])) : acc;
}

template <int R, int PASSES>
struct VState {
  using C = TermCfg<R, PASSES>;
  float2 dl[C::IMGS / 2][PASSES][C::L];  // image pairs
  float2 vlast[C::IMGS / 2];
};

// cp.async (LDGSTS) helpers for the f prefetch ring in shared memory
__device__ __forceinline__ void cp_async_f32(float* dst_smem, const float* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int R, int PASSES>
__global__ void __launch_bounds__(TermCfg<R, PASSES>::THREADS, TermCfg<R, PASSES>::MIN_BLOCKS)
    terms_kernel(const TermParams p) {
  using C = TermCfg<R, PASSES>;
  constexpr int D = C::D, L = C::L, HALO = C::HALO, IMGS = C::IMGS, WC = C::WC;
  constexpr int ROWS = C::ROWS, RING = C::RING, VBP = C::VB_PITCH, RAWP = C::RAW_PITCH;
  constexpr int HALO_W = C::HALO_W, THREADS = C::THREADS, GOFF = C::GOFF, NB = C::NB;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* VB = reinterpret_cast<float*>(smem_raw);
  float* RAW = VB + ROWS * VBP;
  float* gv = RAW + RING * RAWP;
  const int gv_len = p.band + 2 * HALO + GOFF;
  float* gh = gv + gv_len;
  float* FR = gh + HALO_W + GOFF;  // per-thread ring of prefetched f samples (L slots)

  // Wait for K1 / K2 (PDL launch), then let the dependent epilogue launch:
  // its CTAs take whatever SM room K3 leaves and wait for segments.  The
  // wait comes first because the streamed epilogue reads the control block
  // that the fused K1 clears.
  pdl_wait();
#if SBF_PDL_TRIGGER
  pdl_trigger();
#endif
  const sbf_plan* plan = p.plan;
  if (plan->status != SBF_OK) return;
  if (p.hdr_guard && needs_hdr(p.stats)) {
    if (blockIdx.x == 0 && threadIdx.x == 0)
      atomicOr(const_cast<int*>(&plan->flags), SBF_PLAN_NEEDS_HDR);
    return;
  }
  const int K_eval = plan->K_eval;
  // band height from the device plan: the largest band (smem is sized for
  // p.band) that still gives >= 2 items per CTA; small images / few terms
  // get shorter bands instead of leaving most SMs idle (halo cost <= 1.5x)
  int bandh = p.band;
  {
    const int rows_out = p.out_hi - p.out_lo;
    const int per_band = max(1, p.nstrips * K_eval);
    const int nb_min = (2 * (int)gridDim.x + per_band - 1) / per_band;
    const int b = (rows_out + nb_min - 1) / nb_min;
    bandh = max(min(b, p.band), min(4 * HALO, p.band));
  }
  const int rows_all = p.out_hi - p.out_lo;
  const int nbands = (rows_all + bandh - 1) / bandh;
  const int units = p.nstrips * nbands;
  // tail: the last Ks terms run in short bands, so the queue ends with small
  // items and CTAs finish together (with one band size for every term, SMs
  // idled ~18% of the kernel waiting for the last long items)
  int Ks = 0, bands_s = 1, units_s = 0;
  if (SBF_TAIL_ROWS > 0 && bandh > SBF_TAIL_ROWS) {
    bands_s = (rows_all + SBF_TAIL_ROWS - 1) / SBF_TAIL_ROWS;
    units_s = p.nstrips * bands_s;
    Ks = min(K_eval / SBF_TAIL_FRAC, (SBF_TAIL_WAVES * (int)gridDim.x + units_s - 1) / units_s);
  }
  const int bandh_s = (rows_all + bands_s - 1) / bands_s;
  const int items_big = (K_eval - Ks) * units;
  const int total = items_big + Ks * units_s;
  // streamed epilogue (p.epi): output segments are the tail bands (the main
  // bands without a tail); CTA 0 publishes the schedule, every item bumps the
  // counters of the segments it covers once its reductions have landed
  // (segment bookkeeping lives in shared memory: no registers held across
  // the sweep -- the K3 register allocation is sensitive to it)
  __shared__ int s_seg_h, s_sg0, s_sg1;
  const int seg_h = Ks > 0 ? bandh_s : bandh;
  if (threadIdx.x == 0) s_seg_h = seg_h;
  if (p.epi && blockIdx.x == 0 && threadIdx.x == 0) {
    int* ctrl = p.counter;  // [0] queue head, [1] epilogue queue head, [2..8] schedule
    ctrl[2] = seg_h;
    ctrl[3] = (rows_all + seg_h - 1) / seg_h;
    ctrl[4] = bandh;
    ctrl[5] = bandh_s;
    ctrl[6] = Ks;
    ctrl[7] = K_eval;
    __threadfence();
    atomicExch(ctrl + 8, 1);
  }
  const int tid = threadIdx.x;
  const float centerf = p.centred ? 0.f : (float)p.stats[3];
  const float a = p.a, b = p.b;
  __shared__ int s_item;

  VState<R, PASSES> st;

  // persistent CTA: pull (term, band, strip) items -- band by band (main
  // terms, then the tail terms) so output segments complete one after
  // another; edge strips (costlier border code) first within a band
  for (;;) {
    if (tid == 0) s_item = atomicAdd(p.counter, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= total) break;
    const bool tail = item >= items_big;
    const int i2 = tail ? item - items_big : item;
    int kk, band, si;
    if (tail ? SBF_TAIL_BAND_MAJOR : SBF_MAIN_BAND_MAJOR) {
      const int per = (tail ? Ks : K_eval - Ks) * p.nstrips;
      band = i2 / per;
      const int r2 = i2 - band * per;
      kk = (tail ? K_eval - Ks : 0) + r2 / p.nstrips;
      si = r2 - (r2 / p.nstrips) * p.nstrips;
    } else {
      const int un = tail ? units_s : units;
      kk = i2 / un;
      const int u = i2 - kk * un;
      kk += tail ? K_eval - Ks : 0;
      band = u / p.nstrips;
      si = u - band * p.nstrips;
    }
    const int strip = p.nstrips < 2 ? si : (si == 0 ? 0 : (si == 1 ? p.nstrips - 1 : si - 1));
    const int bh = tail ? bandh_s : bandh;

  const int y0 = p.out_lo + band * bh;
  const int y1 = min(p.out_hi, y0 + bh);
  const int Bn = y1 - y0;
  const int T_total = Bn + 2 * HALO;
  if (SBF_EPI_COUNTERS && p.epi && tid == 0) {
    const int sh = s_seg_h;
    s_sg0 = (y0 - p.out_lo) / sh;
    s_sg1 = (y1 - 1 - p.out_lo) / sh;
  }
  const int xs = strip * WC - HALO;  // image column of haloed index 0

  // ---- border tables: index = stream/haloed position + GOFF ----
  const int64_t grow0 = p.row0 + (int64_t)(y0 - HALO);  // global row of stream position 0
  for (int k = tid; k < bh + 2 * HALO + GOFF; k += THREADS)
    gv[k] = gfactor(grow0 + (k - GOFF), p.img_H, p.r, p.alpha);
  for (int k = tid; k < HALO_W + GOFF; k += THREADS)
    gh[k] = gfactor((int64_t)xs + (k - GOFF), p.W, p.r, p.alpha);
  // stream positions whose rows have factor 1 (conservative: D from the edges)
  const int64_t sg_lo = (int64_t)D - grow0;
  const int64_t sg_hi = p.img_H - 1 - D - grow0;
  // stream positions whose f row exists in the buffer and the image
  const int64_t sf_hi = smin<int64_t>(smin<int64_t>((int64_t)p.H - 1 - (y0 - HALO), p.img_H - 1 - grow0),
                                      (int64_t)T_total - 1);
  const int64_t sf_lo = smax<int64_t>((int64_t)-(y0 - HALO), -grow0);
  // haloed columns whose factor is 1
  const int qg_lo = D - xs, qg_hi = p.W - 1 - D - xs;
  __syncthreads();

  // ---- roles ----
  constexpr int TPC = 4 / IMGS;  // V threads per column
  const int q = tid / TPC;       // haloed column of this V thread
  const int pair = tid % TPC;    // IMGS==2: 0 -> (f cos, cos), 1 -> (f sin, sin)
  const int col = xs + q;
  const int colc = col < 0 ? 0 : (col >= p.W ? p.W - 1 : col);  // safe address; H masks it
  const bool out_col = q >= HALO && q < HALO + WC;
  const int hv = tid >> 2;   // H-phase row within the chunk
  const int himg = tid & 3;  // H-phase image (VB component)
  const float* fcol = p.f + (int64_t)(y0 - HALO) * p.ld + colc;  // stream position 0

  {
    const sbf_term term = p.terms[kk];
    const float scale = (float)term.scale;
    const float nu = (float)term.turns;

#pragma unroll
    for (int i = 0; i < IMGS / 2; ++i) {
      st.vlast[i] = f2(0.f);
#pragma unroll
      for (int pp = 0; pp < PASSES; ++pp)
#pragma unroll
        for (int j = 0; j < L; ++j) st.dl[i][pp][j] = f2(0.f);
    }
    // raw samples are prefetched L steps ahead; the centre is subtracted at
    // use so no instruction waits on the load before then
    // f for step t is copied asynchronously (cp.async) into FR[tid][t % L],
    // L steps ahead; every executed step commits exactly one group, so the
    // sample of step t is the group committed L groups earlier.  Rows outside
    // [sf_lo, sf_hi] are never used unmasked: a clamped row is loaded instead.
    float* fr = FR + tid * L;
    auto fetch_async = [&](int t, int slot) {
      const int64_t tc = t < sf_lo ? sf_lo : (t > sf_hi ? sf_hi : (int64_t)t);
      cp_async_f32(fr + slot, fcol + tc * p.ld);
      cp_async_commit();
    };
    cp_async_wait<0>();  // previous term's tail copies landed before slots are reused
#pragma unroll
    for (int j = 0; j < L; ++j) fetch_async(j, j);
    // the sample of step t is read from the ring one step early (step t-1),
    // so its shared-memory latency hides behind a whole step of work
    // phasor of this pixel for the current term: frac(f nu) by explicit range
    // reduction (|u| < 2^22), then MUFU sin/cos (IMGS==2: cos or sin per thread)
    auto phasor = [&](float fcv, float& cv, float& sv) {
      const float u = fcv * nu;
      const float tt = u - ((u + 12582912.f) - 12582912.f);
      if (IMGS == 4) {
        __sincosf(tt * 6.28318530717958647f, &sv, &cv);
      } else {
        cv = __cosf((tt - 0.25f * pair) * 6.28318530717958647f);
        sv = cv;
      }
    };
    cp_async_wait<L - 1>();
    float fnext = fr[0];
#if SBF_TRIG_AHEAD
    float fc_ahead = fnext - centerf, ph_c, ph_s;
    phasor(fc_ahead, ph_c, ph_s);
    cp_async_wait<L - 2>();
    fnext = fr[1 % L];
#endif

    for (int t0 = 0; t0 < T_total; t0 += ROWS) {
      const int t1 = min(t0 + ROWS, T_total);
      const int rs0 = ((t0 - HALO) % RING + RING) % RING;  // RAW slot of step t0

      // ===================== V phase =====================
      // block variants: KIND 0 main (no checks), 1 partial (a full-interior
      // block cut by a chunk boundary: only the step range is checked),
      // 2 general (band edges: every condition checked, border renormalised)
      auto vblock = [&](auto kind_tag, const int base) {
        constexpr int KIND = decltype(kind_tag)::value;
        constexpr bool GUARD = KIND == 2, BORDER = KIND == 2;
        const float* fb = fcol + (int64_t)(base + L) * p.ld;
        static_for<L>([&](auto jc) {
          constexpr int J = decltype(jc)::value;
          const int t = base + J;
          if (KIND >= 1 && (unsigned)(t - t0) >= (unsigned)(t1 - t0)) return;
#if SBF_TRIG_AHEAD
          // the phasor of step t was computed during step t-1 (its chain then
          // overlaps the previous step's recurrences); prepare step t+1 now
          const float fc = fc_ahead;
          float cv = ph_c, sv = ph_s;
          fc_ahead = fnext - centerf;
          phasor(fc_ahead, ph_c, ph_s);
          cp_async_wait<(L >= 3 ? L - 3 : 0)>();  // group of step t+2 has landed
          fnext = fr[(J + 2) % L];
#else
#if SBF_F_EARLY
          const float fc = fnext - centerf;
          cp_async_wait<L - 2>();  // group of step t+1 has landed
          fnext = fr[(J + 1) % L];
#else
          cp_async_wait<L - 1>();
          const float fc = fr[J] - centerf;
#endif
          float cv, sv;
          phasor(fc, cv, sv);
#endif
          if (BORDER) {  // rows outside the image contribute nothing (zero padding)
            const float m = (grow0 + t >= 0 && grow0 + t < p.img_H) ? 1.f : 0.f;
            cv *= m;
            sv *= m;
          }
          // raw scaled phasor of output pixels for the H phase
          if (!GUARD || (t >= HALO && t < HALO + Bn)) {
            int slot = rs0 + (t - t0);
            slot = slot >= RING ? slot - RING : slot;
            float* rp = RAW + slot * RAWP + 2 * (q - HALO);
            if (out_col) {
              if (IMGS == 4) {
                *reinterpret_cast<float2*>(rp) = make_float2(cv, sv);
              } else {
                rp[pair] = cv;
              }
            }
          }
          if (GUARD) {
            fetch_async(t + L, J);
          } else {
            cp_async_f32(fr + J, fb + (int64_t)J * p.ld);
            cp_async_commit();
          }
          const float* gt = gv + t + GOFF;
          const float2 a2 = f2(a), nb2 = f2(-b), b2 = f2(b);
          if (IMGS == 4) {
            // pairs: A = (f cos, f sin) -> (F_c, F_s); B = (cos, sin) -> (G_c, G_s)
            const float2 ya = cascade2<J, L, D, PASSES, BORDER>(
                st.dl[0], st.vlast[0], __fmul2_rn(f2(fc), make_float2(cv, sv)), a2, nb2, b2, gt);
            const float2 yb = cascade2<J, L, D, PASSES, BORDER>(
                st.dl[IMGS / 2 - 1], st.vlast[IMGS / 2 - 1], make_float2(cv, sv), a2, nb2, b2, gt);
            if (!GUARD || t >= 2 * HALO) {
              // two 8-byte stores straight from the FFMA2 register pairs (one
              // 16-byte store needed ~7 MOVs per step to build a register quad)
              float2* vp = reinterpret_cast<float2*>(VB + (t - t0) * VBP + 4 * q);
              vp[0] = ya;
              vp[1] = yb;
            }
          } else {
            // one pair per thread: (f v, v), v = cos (pair 0) or sin (pair 1)
            const float2 y = cascade2<J, L, D, PASSES, BORDER>(
                st.dl[0], st.vlast[0], __fmul2_rn(make_float2(fc, 1.f), f2(cv)), a2, nb2, b2, gt);
            if (!GUARD || t >= 2 * HALO) {
              float* vp = VB + (t - t0) * VBP + 4 * q;
              *reinterpret_cast<float2*>(vp + 2 * pair) = y;
            }
          }
        });
      };
      for (int base = (t0 / L) * L; base < t1; base += L) {
        const bool clean = base >= 2 * HALO && base + L <= HALO + Bn &&
                           base + 2 * L - 1 <= sf_hi &&
                           base - (PASSES + 2) * D - 1 >= sg_lo && base + L - 1 <= sg_hi;
#if SBF_V_MAIN_VARIANT
        if (clean && base >= t0 && base + L <= t1)
          vblock(std::integral_constant<int, 0>{}, base);
        else
#endif
        if (clean)
          vblock(std::integral_constant<int, 1>{}, base);
        else
          vblock(std::integral_constant<int, 2>{}, base);
      }
      __syncthreads();

      // ===================== H phase =====================
      {
        const int t = t0 + hv;
        if (t < t1 && t >= 2 * HALO) {
          float* vrow = VB + hv * VBP + himg;
          const int oslot = (t - 2 * HALO) % RING;
          // VB image order: IMGS==4 [F_c, F_s, G_c, G_s]; IMGS==2 [F_c, G_c, F_s, G_s]
          const int rc = (IMGS == 4) ? (himg & 1) : (himg >> 1);  // 0 -> cos, 1 -> sin
          const float* rrow = RAW + oslot * RAWP + rc - 4 * HALO;  // index by 2*q
          float hd[PASSES][L];
          float hlast = 0.f;
#pragma unroll
          for (int pp = 0; pp < PASSES; ++pp)
#pragma unroll
            for (int j = 0; j < L; ++j) hd[pp][j] = 0.f;
          // kind: 0 warm-up (no outputs), 1 main, 2 guarded, 3 border
          auto hblock = [&](auto kind_tag, const int base) {
            constexpr int KIND = decltype(kind_tag)::value;
            constexpr bool GUARD = KIND >= 2, BORDER = KIND == 3;
            // the block's output phasors are read before any VB store: RAW and
            // VB are disjoint, but the compiler cannot prove it and would
            // otherwise serialise each load behind the previous store
            // (long rings, r > 5: loaded at use, the registers are needed elsewhere)
            constexpr bool PREF = L <= 13;
            float rw[PREF ? L : 1];
            if constexpr (PREF) {
              static_for<L>([&](auto jc) {
                constexpr int J = decltype(jc)::value;
                const int qq = base + J;
                if (KIND == 1) rw[J] = rrow[2 * qq];
                else if (KIND != 0) rw[J] = (qq >= 2 * HALO && qq < HALO_W) ? rrow[2 * qq] : 0.f;
              });
            }
            static_for<L>([&](auto jc) {
              constexpr int J = decltype(jc)::value;
              const int qq = base + J;
              if (GUARD && qq >= HALO_W) return;
              float x = vrow[4 * qq];
              if (BORDER) {
                const int c = xs + qq;
                x = (c >= 0 && c < p.W) ? x : 0.f;
              }
              const float yv = cascade<J, L, D, PASSES, BORDER>(hd, hlast, x, a, b, gh + qq + GOFF);
              if (KIND == 1 || (GUARD && qq >= 2 * HALO))
                vrow[4 * (qq - HALO)] = yv * (PREF ? rw[PREF ? J : 0] : rrow[2 * qq]);
            });
          };
          // interior strips (no column touches an image border) run a fixed
          // block sequence: warm-up blocks, one guarded block, a loop of main
          // blocks, guarded tail — no per-block variant dispatch
          constexpr int KB_MAIN0 = (2 * HALO + L - 1) / L;  // first block with base >= 2*HALO
          constexpr int KB_MAIN1 = (HALO_W - L) / L + 1;    // blocks [KB_MAIN0, KB_MAIN1) are main
          const bool strip_in = -(PASSES + 2) * D - 1 >= qg_lo && NB * L - 1 <= qg_hi;
          if (SBF_H_FIXED_SEQ && strip_in && KB_MAIN0 < KB_MAIN1) {
            static_for<KB_MAIN0>([&](auto kc) {
              constexpr int KB = decltype(kc)::value;
              if constexpr (KB * L + L <= 2 * HALO)
                hblock(std::integral_constant<int, 0>{}, KB * L);
              else
                hblock(std::integral_constant<int, 2>{}, KB * L);
            });
#pragma unroll 1
            for (int kb = KB_MAIN0; kb < KB_MAIN1; ++kb) hblock(std::integral_constant<int, 1>{}, kb * L);
            static_for<NB - KB_MAIN1>([&](auto kc) {
              hblock(std::integral_constant<int, 2>{}, (KB_MAIN1 + decltype(kc)::value) * L);
            });
          } else {
            for (int kb = 0; kb < NB; ++kb) {
              const int base = kb * L;
              const bool gin = base - (PASSES + 2) * D - 1 >= qg_lo && base + L - 1 <= qg_hi;
              if (gin && base + L <= 2 * HALO)
                hblock(std::integral_constant<int, 0>{}, base);
              else if (gin && base >= 2 * HALO && base + L <= HALO_W)
                hblock(std::integral_constant<int, 1>{}, base);
              else if (gin)
                hblock(std::integral_constant<int, 2>{}, base);
              else
                hblock(std::integral_constant<int, 3>{}, base);
            }
          }
        }
      }
      __syncthreads();

      // ===================== accumulate =====================
      {
        const int vlo = max(t0, 2 * HALO) - t0;
        const int vhi = min(t1, 2 * HALO + Bn) - t0;
        const int xlim = min(WC, p.W - strip * WC);  // columns of this strip inside the image
        // G groups of one thread per output column walk every G-th row of
        // the chunk: no index arithmetic per pixel (constant strides)
        constexpr int G = THREADS / WC;
        const int jc = tid % WC, g = tid / WC;
        if (g < G && jc < xlim) {
          const float* vb = VB + (vlo + g) * VBP + 4 * (HALO + jc);
          float2* dst = reinterpret_cast<float2*>(p.nd) +
                        (int64_t)(y0 - 2 * HALO + t0 + vlo + g - p.out_lo) * p.W + strip * WC + jc;
          const int64_t dstride = (int64_t)G * p.W;
#pragma unroll 4
          for (int vv = vlo + g; vv < vhi; vv += G) {
            const float4 pv = *reinterpret_cast<const float4*>(vb);
            vb += G * VBP;
            // the term weight is applied once per output pixel here
            const float num = scale * ((IMGS == 4) ? pv.x + pv.y : pv.x + pv.z);
            const float den = scale * ((IMGS == 4) ? pv.z + pv.w : pv.y + pv.w);
            asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(dst), "f"(num), "f"(den));
            dst += dstride;
          }
        }
      }
      __syncthreads();
    }  // chunks
  }  // term item
    if (SBF_EPI_COUNTERS && p.epi) {
      // every thread's reductions are ordered before the segment counters move
      __threadfence();
      __syncthreads();
      if (tid == 0)
        for (int sg = s_sg0; sg <= s_sg1; ++sg) atomicAdd(p.seg_done + sg, 1);
    }
  }  // work queue
}

// ---- host launcher ----
template <int R, int PASSES>
size_t terms_smem_bytes(int band) {
  using C = TermCfg<R, PASSES>;
  return (size_t)C::ROWS * C::VB_PITCH * 4 + (size_t)C::RING * C::RAW_PITCH * 4 +
         (size_t)(band + 2 * C::HALO + C::GOFF + C::HALO_W + C::GOFF) * 4 +
         (size_t)C::THREADS * C::L * 4 + 16;
}

template <int R, int PASSES>
int launch_terms(const TermParams& p, cudaStream_t st) {
  using C = TermCfg<R, PASSES>;
  const size_t smem = terms_smem_bytes<R, PASSES>(p.band);
  SBF_CHECK_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(terms_kernel<R, PASSES>), smem));
  const int sms = device_sm_count();
  const long long grid = (long long)sms * C::MIN_BLOCKS;  // persistent CTAs
  SBF_CHECK_CUDA(launch_pdl(terms_kernel<R, PASSES>, dim3((unsigned)grid), dim3(C::THREADS), smem, st, p));
  SBF_CHECK_LAUNCH();
  return SBF_OK;
}

template <int R, int PASSES>
void terms_geometry(int* halo, int* wc, int* threads, int* blocks_per_sm) {
  using C = TermCfg<R, PASSES>;
  *halo = C::HALO;
  *wc = C::WC;
  *threads = C::THREADS;
  *blocks_per_sm = C::MIN_BLOCKS;
}

// dispatch table entry (mode: precision the instantiation serves; 0 = fp32)
struct TermsEntry {
  int r, passes, mode;
  int (*launch)(const TermParams&, cudaStream_t);
  size_t (*smem)(int);
  void (*geom)(int*, int*, int*, int*);
};

#define SBF_TERMS_ENTRY(R, P, M) \
  TermsEntry { R, P, M, &launch_terms<R, P>, &terms_smem_bytes<R, P>, &terms_geometry<R, P> }

}  // namespace sbf
