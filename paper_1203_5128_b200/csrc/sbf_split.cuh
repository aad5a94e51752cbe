// Split term sweep for large radii (r >= 5): per term, SV smooths the four
// modulated images down whole columns and writes them to HBM (16 B/px), SH
// streams whole rows of those through a shared-memory tile ring, smooths
// them along the rows and accumulates (num, den).  Same arithmetic as K3
// (sbf_terms.cuh: extended-box recurrences, raw rings, border renormalisation
// on read); what changes is the work decomposition:
//  * K3's 128-column strips need a 2*halo column overlap (2.3x the work at
//    r=11, halo 36) and a 2*halo warm-up per strip row; SV has no column
//    halo at all and SH warms up once per image row;
//  * SV keeps only the V-phase state in registers (no VB/RAW shared memory),
//    so it runs narrow CTAs at higher occupancy; SH keeps only the H state.
// The price is 36 B/px per term of HBM traffic (U write + read, nd update),
// which at these radii is cheaper than K3's halo recomputation.
#pragma once

#include "sbf_terms.cuh"

namespace sbf {

struct SplitParams {
  const float* f;  // fp32 image (centred when `centred`)
  int64_t ld;
  int centred;
  int H, W;
  int64_t row0, img_H;
  int out_lo, out_hi;
  int r;
  float alpha, a, b;
  const sbf_plan* plan;
  const sbf_term* terms;
  const double* stats;
  float* U;    // SBF_SPLIT_TPI slots of [rows_out][W][4] column-smoothed images (term k in slot k % TPI)
  int64_t u_slot;  // floats from one slot to the next
  float2* nd;  // [rows_out][W] (num, den)
  int term;
  int band;  // SV output rows per CTA (a multiple of SH_ROWS)
  int seg;   // SH output columns per CTA
  int hdr_guard;  // SBF_PREC_AUTO: flag the plan and do nothing on wide ranges
  // device work queue of the persistent sweep (zeroed before the launch)
  int* head;
  int* sv_done;  // per band: SV tiles finished, all terms so far
  int* sh_done;  // per band: SH tiles finished, all terms so far
  int svx, svy, shx, shy;
};

#ifndef SBF_SPLIT_TPI
#define SBF_SPLIT_TPI 2  // consecutive terms per SH item (U slots in flight)
#endif

template <int R, int PASSES>
struct SplitCfg {
  static constexpr int D = R + 1;
  static constexpr int L = 2 * R + 3;
  static constexpr int HALO = PASSES * D;
  static constexpr int IMGS = (R <= 4) ? 4 : 2;
  static constexpr int SV_COLS = (IMGS == 4) ? 128 : 64;
  static constexpr int SV_THREADS = SV_COLS * 4 / IMGS;
  static constexpr int GOFF = (PASSES + 2) * D + 2;
  // SH: TPI consecutive terms per item; (32 / TPI) rows x 4 images x TPI
  // terms = 128 lanes (one recurrence each); tile = 2L stream positions,
  // ring of 3
  static constexpr int TPI = SBF_SPLIT_TPI;
  static_assert(TPI == 1 || TPI == 2 || TPI == 4, "128 SH lanes");
  static constexpr int SH_ROWS = 32 / TPI;
  static constexpr int SH_THREADS = 128;
  static constexpr int TILE = 2 * L;
  static constexpr int NTILE = 3;
  static constexpr int RINGC = NTILE * TILE;
  static constexpr int RPITCH = 4 * RINGC + 4;  // floats per row (== 4 mod 8 words)
  // border-table reach at each row end (stream positions)
  static constexpr int GEDGE = 2 * HALO + 2 * L + (PASSES + 2) * D + 4;
  static_assert(HALO < TILE, "outputs may only lag into the previous tile");
};

// ============================ SV: column sweep ============================
#ifndef SBF_SV_MINB
#define SBF_SV_MINB 1  // SV CTAs per SM the register allocation must allow
#endif

template <int R, int PASSES>
__device__ __forceinline__ void sv_tile(const SplitParams& p, const int bx, const int by) {
  using C = SplitCfg<R, PASSES>;
  constexpr int D = C::D, L = C::L, HALO = C::HALO, IMGS = C::IMGS, GOFF = C::GOFF;
  constexpr int THREADS = C::SV_THREADS, TPC = 4 / IMGS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* gv = reinterpret_cast<float*>(smem_raw);
  const int gv_len = p.band + 2 * HALO + GOFF;
  float* FR = gv + gv_len + 4;

  const int tid = threadIdx.x;
  const float centerf = p.centred ? 0.f : (float)p.stats[3];
  const float a = p.a, b = p.b;
  const float nu = (float)p.terms[p.term].turns;

  const int y0 = p.out_lo + by * p.band;
  const int y1 = min(p.out_hi, y0 + p.band);
  const int Bn = y1 - y0;
  const int T_total = Bn + 2 * HALO;
  const int64_t grow0 = p.row0 + (int64_t)(y0 - HALO);
  for (int k = tid; k < gv_len; k += THREADS) gv[k] = gfactor(grow0 + (k - GOFF), p.img_H, p.r, p.alpha);
  const int64_t sg_lo = (int64_t)D - grow0;
  const int64_t sg_hi = p.img_H - 1 - D - grow0;
  const int64_t sf_hi = smin<int64_t>(smin<int64_t>((int64_t)p.H - 1 - (y0 - HALO), p.img_H - 1 - grow0),
                                      (int64_t)T_total - 1);
  const int64_t sf_lo = smax<int64_t>((int64_t)-(y0 - HALO), -grow0);
  __syncthreads();

  const int q = tid / TPC, pair = tid % TPC;
  const int col = bx * C::SV_COLS + q;
  const bool colok = col < p.W;
  const int colc = colok ? col : p.W - 1;
  const float* fcol = p.f + (int64_t)(y0 - HALO) * p.ld + colc;
  float* urow = p.U + (int64_t)(p.term % C::TPI) * p.u_slot +
               ((int64_t)(y0 - p.out_lo - 2 * HALO) * p.W + col) * 4 + 2 * pair;

  VState<R, PASSES> st;
#pragma unroll
  for (int i = 0; i < IMGS / 2; ++i) {
    st.vlast[i] = f2(0.f);
#pragma unroll
    for (int pp = 0; pp < PASSES; ++pp)
#pragma unroll
      for (int j = 0; j < L; ++j) st.dl[i][pp][j] = f2(0.f);
  }
  float* fr = FR + tid * L;
  auto fetch_async = [&](int t, int slot) {
    const int64_t tc = t < sf_lo ? sf_lo : (t > sf_hi ? sf_hi : (int64_t)t);
    cp_async_f32(fr + slot, fcol + tc * p.ld);
    cp_async_commit();
  };
#pragma unroll
  for (int j = 0; j < L; ++j) fetch_async(j, j);
  cp_async_wait<L - 1>();
  float fnext = fr[0];

  // KIND 0: clean block, no checks; 2: band ends / image borders, all checks
  auto vblock = [&](auto kind_tag, const int base) {
    constexpr int KIND = decltype(kind_tag)::value;
    constexpr bool GUARD = KIND == 2, BORDER = KIND == 2;
    const float* fb = fcol + (int64_t)(base + L) * p.ld;
    static_for<L>([&](auto jc) {
      constexpr int J = decltype(jc)::value;
      const int t = base + J;
      if (GUARD && t >= T_total) return;
      const float fc = fnext - centerf;
      cp_async_wait<L - 2>();
      fnext = fr[(J + 1) % L];
      const float u = fc * nu;
      const float tt = u - ((u + 12582912.f) - 12582912.f);
      float cv, sv;
      if (IMGS == 4) {
        __sincosf(tt * 6.28318530717958647f, &sv, &cv);
      } else {
        cv = __cosf((tt - 0.25f * pair) * 6.28318530717958647f);
        sv = cv;
      }
      if (BORDER) {
        const float m = (grow0 + t >= 0 && grow0 + t < p.img_H) ? 1.f : 0.f;
        cv *= m;
        sv *= m;
      }
      if (GUARD) {
        fetch_async(t + L, J);
      } else {
        cp_async_f32(fr + J, fb + (int64_t)J * p.ld);
        cp_async_commit();
      }
      const float* gt = gv + t + GOFF;
      const float2 a2 = f2(a), nb2 = f2(-b), b2 = f2(b);
      const bool store = colok && (!GUARD || (t >= 2 * HALO && t < 2 * HALO + Bn));
      float* up = urow + (int64_t)t * p.W * 4;
      if (IMGS == 4) {
        const float2 ya = cascade2<J, L, D, PASSES, BORDER>(
            st.dl[0], st.vlast[0], __fmul2_rn(f2(fc), make_float2(cv, sv)), a2, nb2, b2, gt);
        const float2 yb = cascade2<J, L, D, PASSES, BORDER>(
            st.dl[IMGS / 2 - 1], st.vlast[IMGS / 2 - 1], make_float2(cv, sv), a2, nb2, b2, gt);
        if (store) *reinterpret_cast<float4*>(up) = make_float4(ya.x, ya.y, yb.x, yb.y);
      } else {
        const float2 y = cascade2<J, L, D, PASSES, BORDER>(
            st.dl[0], st.vlast[0], __fmul2_rn(make_float2(fc, 1.f), f2(cv)), a2, nb2, b2, gt);
        if (store) *reinterpret_cast<float2*>(up) = y;
      }
    });
  };
  auto clean = [&](int base) {
    return base >= 2 * HALO && base + L <= HALO + Bn && base + 2 * L - 1 <= sf_hi &&
           base - (PASSES + 2) * D - 1 >= sg_lo && base + L - 1 <= sg_hi;
  };
  for (int base = 0; base < T_total; base += L) {
    if (clean(base))
      vblock(std::integral_constant<int, 0>{}, base);
    else
      vblock(std::integral_constant<int, 2>{}, base);
  }
  cp_async_wait<0>();
}

// ============================ SH: row sweep ==============================
// Stream position s = input column + HALO; the output of step s is column
// s - 2*HALO.  A CTA owns SH_ROWS rows and the output columns [c0, c0 + seg)
// for TPI consecutive terms kA, kA + 1, ...: lane (t, row, image) streams
// term kA + t's image of that row from U slot t, from a zero state
// (exact: outputs at columns >= c0 depend only on inputs >= c0 - HALO).  The
// ring holds stream positions mod RINGC relative to the segment start; an
// output replaces its own input (position s - HALO) in place.  Both terms'
// contributions are added to (num, den) in one read-modify-write, and the
// output pixels' f samples are read once for the pair.
template <int R, int PASSES>
__device__ __forceinline__ void sh_tile(const SplitParams& p, const int bx, const int by,
                                        const int kA, const int nterms) {
  using C = SplitCfg<R, PASSES>;
  constexpr int D = C::D, L = C::L, HALO = C::HALO, IMGS = C::IMGS, GOFF = C::GOFF;
  constexpr int TILE = C::TILE, NTILE = C::NTILE, RINGC = C::RINGC, RP = C::RPITCH;
  constexpr int ROWS = C::SH_ROWS, GE = C::GEDGE, TPI = C::TPI;
  static_assert(IMGS == 2, "the U / ring order below is [F_c, G_c, F_s, G_s]");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* ring = reinterpret_cast<float*>(smem_raw);  // [TPI][ROWS][RPITCH]
  float* gL = ring + TPI * ROWS * RP;               // factors at stream positions [s0 - GOFF, s0 + GE)
  float* gR = gL + GE + GOFF;                       // factors at [sR0 - GOFF, sR0 + GE + GOFF)

  const int tid = threadIdx.x;
  const int W = p.W;
  const int c0 = by * p.seg;
  const int s0 = c0;
  const int s1 = min(c0 + p.seg + 2 * HALO, W + 2 * HALO);
  const int sR0 = max(s0, s1 - GE);
  for (int k = tid; k < GE + GOFF; k += 128) {
    gL[k] = gfactor((int64_t)(s0 + k - GOFF) - HALO, W, p.r, p.alpha);
    gR[k] = gfactor((int64_t)(sR0 + k - GOFF) - HALO, W, p.r, p.alpha);
  }
  const float a = p.a, b = p.b;
  float scale[TPI], nu[TPI];
#pragma unroll
  for (int t = 0; t < TPI; ++t) {
    const sbf_term term = p.terms[t < nterms ? kA + t : kA];
    scale[t] = t < nterms ? (float)term.scale : 0.f;
    nu[t] = (float)term.turns;
  }
  const float centerf = p.centred ? 0.f : (float)p.stats[3];
  const int r0 = p.out_lo + bx * ROWS;  // first buffer row of this CTA
  const int nrows = min(ROWS, p.out_hi - r0);
  const float* Ub = p.U + (int64_t)(r0 - p.out_lo) * W * 4;

  // tile j: stream positions s0 + [j*TILE, (j+1)*TILE), input columns s - HALO
  const int ntiles = (s1 - s0 + TILE - 1) / TILE;
  auto load_tile = [&](int j) {
    const int slot = (j % NTILE) * TILE;
    for (int k = tid; k < TPI * ROWS * TILE; k += 128) {
      const int t = k / (ROWS * TILE), k2 = k - t * (ROWS * TILE);
      const int rr = k2 / TILE, cc = k2 - rr * TILE;
      const int c = s0 + j * TILE + cc - HALO;
      float* dst = ring + (t * ROWS + rr) * RP + 4 * (slot + cc);
      if (t < nterms && rr < nrows && c >= 0 && c < W) {
        const float* src = Ub + (int64_t)t * p.u_slot + ((int64_t)rr * W + c) * 4;  // term kA + t
        const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
      } else {
        *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    cp_async_commit();
  };
  load_tile(0);
  if (ntiles > 1) load_tile(1);

  const int ht = tid / (4 * ROWS);             // term of this H lane
  const int hv = (tid >> 2) % ROWS, himg = tid & 3;
  float hd[PASSES][L];
  float hlast = 0.f;
#pragma unroll
  for (int pp = 0; pp < PASSES; ++pp)
#pragma unroll
    for (int j = 0; j < L; ++j) hd[pp][j] = 0.f;
  float* lrow = ring + (ht * ROWS + hv) * RP + himg;
  const bool hlane = hv < nrows && ht < nterms;
  // stream positions whose reach has factor 1 (cf. K3's qg_lo / qg_hi)
  const int qg_lo = D + HALO, qg_hi = W - 1 - D + HALO;

  // KIND 0 warm-up (no outputs), 1 main, 2 guarded, 3 border (tables)
  auto hblock = [&](auto kind_tag, const int base, const float* gtab, int gpos0) {
    constexpr int KIND = decltype(kind_tag)::value;
    constexpr bool GUARD = KIND >= 2, BORDER = KIND == 3;
    const int rb = (base - s0) % RINGC;  // blocks never wrap: RINGC is a multiple of L
    // inputs are read two steps ahead: the in-place output stores use a
    // wrapped (runtime) index, so the compiler cannot move later loads above
    // them; issuing each load two steps early hides its latency anyway
    float xa = lrow[4 * rb], xb = lrow[4 * (rb + 1)];
    static_for<L>([&](auto jc) {
      constexpr int J = decltype(jc)::value;
      const int s = base + J;
      if (GUARD && s >= s1) return;
      const float x = xa;  // zero outside the image (loader)
      xa = xb;
      if (J + 2 < L) xb = lrow[4 * (rb + J + 2)];
      const float yv = cascade<J, L, D, PASSES, BORDER>(
          hd, hlast, x, a, b, BORDER ? gtab + (s - gpos0) + GOFF : gtab);
      if (KIND == 1 || (GUARD && s >= s0 + 2 * HALO)) {
        int o = rb + J - HALO;
        o = o < 0 ? o + RINGC : o;
        lrow[4 * o] = yv;
      }
    });
  };

  constexpr int PX = (ROWS * TILE + 127) / 128;  // accumulate pixels per thread and tile
  for (int j = 0; j < ntiles; ++j) {
    // this tile's outputs: stream positions [s_lo, s_hi), columns s - 2*HALO.
    // Their f samples and running (num, den) are loaded now, so the global
    // latency hides behind the H phase.
    const int s_lo = max(s0 + j * TILE, s0 + 2 * HALO), s_hi = min(s0 + (j + 1) * TILE, s1);
    const int ncol = s_hi - s_lo;
    float fpx[PX];
    float2 acc_old[PX];
#pragma unroll
    for (int i = 0; i < PX; ++i) {
      const int k = tid + i * 128;
      const int rr = k / TILE, cc = k - rr * TILE;
      fpx[i] = 0.f;
      acc_old[i] = make_float2(0.f, 0.f);
      if (k < ROWS * TILE && rr < nrows && cc < ncol) {
        const int c = s_lo + cc - 2 * HALO;
        const int64_t row = r0 + rr;
        fpx[i] = __ldg(p.f + row * p.ld + c);
        // (num, den) of the previous terms, written by another CTA: from L2
        if (kA > 0) acc_old[i] = __ldcg(p.nd + (row - p.out_lo) * W + c);
      }
    }
    if (j + 1 < ntiles)
      cp_async_wait<1>();
    else
      cp_async_wait<0>();
    __syncthreads();
    // ---- H phase over this tile's blocks ----
    if (hlane) {
#pragma unroll 1
      for (int kb = 0; kb < TILE / L; ++kb) {
        const int base = s0 + j * TILE + kb * L;
        if (base >= s1) break;
        const bool left = base - (PASSES + 2) * D - 1 < qg_lo;
        const bool right = base + L - 1 > qg_hi;
        if (left)
          hblock(std::integral_constant<int, 3>{}, base, gL, s0);
        else if (right)
          hblock(std::integral_constant<int, 3>{}, base, gR, sR0);
        else if (base + L <= s0 + 2 * HALO)
          hblock(std::integral_constant<int, 0>{}, base, gL, s0);
        else if (base >= s0 + 2 * HALO && base + L <= s1)
          hblock(std::integral_constant<int, 1>{}, base, gL, s0);
        else
          hblock(std::integral_constant<int, 2>{}, base, gL, s0);
      }
    }
    __syncthreads();
    // ---- accumulate the outputs produced in this tile (both terms) ----
#pragma unroll
    for (int i = 0; i < PX; ++i) {
      const int k = tid + i * 128;
      const int rr = k / TILE, cc = k - rr * TILE;
      if (k >= ROWS * TILE || rr >= nrows || cc >= ncol) continue;
      const int s = s_lo + cc;
      const int c = s - 2 * HALO;  // output column
      const int o = (s - s0 - HALO) % RINGC;
      const float fc = fpx[i] - centerf;
      float num = acc_old[i].x, den = acc_old[i].y;
#pragma unroll
      for (int t = 0; t < TPI; ++t) {
        if (t >= nterms) break;
        // ring order [F_c, G_c, F_s, G_s]
        const float4 v = *reinterpret_cast<const float4*>(ring + (t * ROWS + rr) * RP + 4 * o);
        const float u = fc * nu[t];
        const float tt = u - ((u + 12582912.f) - 12582912.f);
        float cv, sv;
        __sincosf(tt * 6.28318530717958647f, &sv, &cv);
        num += scale[t] * (cv * v.x + sv * v.z);
        den += scale[t] * (cv * v.y + sv * v.w);
      }
      p.nd[(r0 + rr - p.out_lo) * W + c] = make_float2(num, den);
    }
    __syncthreads();
    if (j + 2 < ntiles) load_tile(j + 2);
  }
}

// ---- host side ----
template <int R, int PASSES>
size_t sv_smem_bytes(int band) {
  using C = SplitCfg<R, PASSES>;
  return (size_t)(band + 2 * C::HALO + C::GOFF + 4) * 4 + (size_t)C::SV_THREADS * C::L * 4 + 16;
}
template <int R, int PASSES>
size_t sh_smem_bytes() {
  using C = SplitCfg<R, PASSES>;
  return (size_t)C::TPI * C::SH_ROWS * C::RPITCH * 4 + (size_t)2 * (C::GEDGE + C::GOFF) * 4 + 16;
}

__device__ __forceinline__ void split_wait(const int* ctr, int target) {
  if (threadIdx.x == 0) {
    int v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
      __nanosleep(64);
    }
  }
  __syncthreads();
}

// Every term in one persistent launch with a device work queue: items are
// taken in order, per pair of terms (2j, 2j+1):
//   [SV tiles of term 2j | SV tiles of term 2j+1 | SH tiles of the pair]
// and the term count is read from the device plan (no host round trip;
// graph-capturable).  Term k's column-smoothed images go to U slot k % TPI.
// Dependencies are per row band and only ever on items taken earlier, so the
// queue cannot deadlock:
//  * SH(pair j) tiles of band b wait for all SV tiles of both terms of band b
//    (U complete) and for all SH(pair j-1) tiles of band b ((num, den)
//    updated in term order: one owner per pixel and pair, a fixed sum order);
//  * SV(2j), SV(2j+1) tiles of band b wait for all SH(pair j-1) tiles of band
//    b (their U slots have been consumed).
// (An odd K leaves the last pair with one term; its second SV block only
// counts.)
template <int R, int PASSES>
__global__ void __launch_bounds__(128) split_queue_kernel(SplitParams p) {
  using C = SplitCfg<R, PASSES>;
  static_assert(C::SV_THREADS == 128, "SV and SH tiles share the CTA shape");
  __shared__ int s_item;
  pdl_wait();
  const sbf_plan* plan = p.plan;
  if (plan->status != SBF_OK) return;
  if (p.hdr_guard && needs_hdr(p.stats)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(const_cast<int*>(&plan->flags), SBF_PLAN_NEEDS_HDR);
    return;
  }
  const int K = plan->K_eval;
  const int rows_out = p.out_hi - p.out_lo;
  if (K == 0) {  // no retained term: (num, den) = 0, every pixel falls back
    const int64_t n = (int64_t)rows_out * p.W;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
      p.nd[i] = make_float2(0.f, 0.f);
    return;
  }
  constexpr int TPI = C::TPI;
  const int npairs = (K + TPI - 1) / TPI;
  const int n_sv = p.svx * p.svy, n_sh = p.shx * p.shy;
  const int per = TPI * n_sv + n_sh;
  const long long total = (long long)npairs * per;
  const int gpb = p.band / C::SH_ROWS;  // SH row groups per band
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(p.head, 1);
    __syncthreads();
    const long long item = s_item;
    __syncthreads();  // s_item is rewritten by the next pull
    if (item >= total) break;
    const int pr = (int)(item / per), j = (int)(item - (long long)pr * per);
    if (j < TPI * n_sv) {
      const int k = pr * TPI + j / n_sv, jj = j % n_sv;
      const int bx = jj % p.svx, band = jj / p.svx;
      const int rows_b = min(p.band, rows_out - band * p.band);
      const int nsh_b = ((rows_b + C::SH_ROWS - 1) / C::SH_ROWS) * p.shy;
      // (the missing second term of an odd K only counts -- but only once the
      // previous pair's SH tiles are done: the counter is cumulative, so an
      // early count could stand in for a previous pair's unfinished SV tile)
      if (pr > 0) split_wait(p.sh_done + band, pr * nsh_b);
      if (k < K) {
        p.term = k;
        sv_tile<R, PASSES>(p, bx, band);
        __threadfence();
        __syncthreads();
      }
      if (threadIdx.x == 0) atomicAdd(p.sv_done + band, 1);
    } else {
      const int jj = j - TPI * n_sv;
      const int rx = jj / p.shy, sy = jj - rx * p.shy;
      const int band = rx / gpb;
      const int rows_b = min(p.band, rows_out - band * p.band);
      const int nsh_b = ((rows_b + C::SH_ROWS - 1) / C::SH_ROWS) * p.shy;
      split_wait(p.sv_done + band, (pr + 1) * TPI * p.svx);
      if (pr > 0) split_wait(p.sh_done + band, pr * nsh_b);
      sh_tile<R, PASSES>(p, rx, sy, pr * TPI, min(TPI, K - pr * TPI));
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) atomicAdd(p.sh_done + band, 1);
    }
  }
}

template <int R, int PASSES>
int launch_split(const SplitParams& p, cudaStream_t st) {
  const size_t smem = smax(sv_smem_bytes<R, PASSES>(p.band), sh_smem_bytes<R, PASSES>());
  SBF_CHECK_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(split_queue_kernel<R, PASSES>), smem));
  int per_sm = 0;
  SBF_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, split_queue_kernel<R, PASSES>,
                                                               128, smem));
  SBF_REQUIRE(per_sm > 0, SBF_ERR_CUDA, "split sweep: no CTA fits on an SM");
  // an ordinary launch: the queue counters are cleared by a memset just
  // before, which a programmatic (early) launch would not wait for
  split_queue_kernel<R, PASSES><<<dim3((unsigned)(per_sm * device_sm_count())), 128, smem, st>>>(p);
  SBF_CHECK_LAUNCH();
  return SBF_OK;
}

struct SplitEntry {
  int r, passes;
  int (*launch)(const SplitParams&, cudaStream_t);
  int sh_rows;  // rows per SH item
};

#define SBF_SPLIT_ENTRY(R, P) \
  SplitEntry { R, P, &launch_split<R, P>, SplitCfg<R, P>::SH_ROWS }

}  // namespace sbf
