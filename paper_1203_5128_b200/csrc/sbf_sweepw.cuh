// K3 — warp-specialised term sweep (sm_100a): the same arithmetic as
// sbf_sweep.cuh (reference bilateral.py:150-163 per folded cosine term,
// spatial.py:108-139 smoothing), organised as a producer/consumer pipeline
// inside one 512-thread CTA per SM instead of barrier-separated phases:
//
//   * two V warpgroups (256 threads, one per haloed column of a 252-column
//     strip) stream the band: phasor, the four modulated images as two packed
//     pairs and the column passes as O(1) register-ring recurrences
//     (vcascade), in whole blocks of L = 2r+3 steps (the ring rotates at
//     compile time; no step carries a range check).  f arrives by TMA, one
//     256 x L box per block, four boxes in flight.  The results go to a ring
//     of 32 VB rows in shared memory; the V warps never wait for the H phase
//     of the rows they just wrote.
//   * two H warpgroups = four pairs of warps.  Pair p owns VB rows
//     [8p, 8p+8): every fourth group of 8 stream steps.  One warp streams the
//     left half of the strip left to right, the other the right half right to
//     left (the window sums are symmetric), one lane per (row, image), each
//     warming up over 2 HALO columns; the in-place results of one half never
//     touch what the other half still reads.  Then the pair accumulates its
//     8 rows: phasor of the output pixel recomputed from f (a second TMA box
//     per group), fixed-point red.add.u64 as in sbf_sweep.cuh.
//   * mbarriers carry box-full / box-free and group-full / group-free between
//     the warpgroups; registers follow the roles (setmaxnreg): 192 per V
//     thread (156 of ring state), 64 per H thread.
// A 252-column strip has 216 output columns at r = 5 (the 128-column strips
// of sbf_sweep.cuh have 92): the V phase recomputes 1.17x instead of 1.39x.
// Device outputs only (sweep_divide_kernel follows); page-locked outputs keep
// sbf_sweep.cuh's fused epilogue.
#pragma once

#include "sbf_sweep.cuh"

#ifndef SBF_SWW_ABL
#define SBF_SWW_ABL 0  // timing ablations (wrong results): 1 no H phase, 2 no accumulate, 4 no V work
#endif

#ifndef SBF_SWW_PROF
#define SBF_SWW_PROF 0  // 1: per-role cycle counters (clock64) summed into p.seg (debug builds only)
#endif
#if SBF_SWW_PROF
#define SWW_T(k) do { const long long t__ = clock64(); prof[k] += t__ - tprev; tprev = t__; } while (0)
#else
#define SWW_T(k) do { } while (0)
#endif

namespace sbf {

template <int R, int PASSES>
struct SweepWCfg {
  static constexpr int D = R + 1;
  static constexpr int L = 2 * R + 3;
  static constexpr int HALO = PASSES * D;
  static constexpr int COLS = 252;            // haloed columns per strip
  static constexpr int FCOLS = 256;           // TMA box width (box starts 16-byte aligned)
  static constexpr int WC = COLS - 2 * HALO;  // output columns per strip
  static constexpr int WH = WC / 2;           // output columns per H half
  static constexpr int HS = WH + 2 * HALO;    // H stream steps per half
  static constexpr int GR = 8;                // stream steps (VB rows) per H group
  static constexpr int NG = 4;                // groups in the VB ring = H pairs
  static constexpr int VROWS = GR * NG;       // VB ring rows
  static constexpr int VT = 256, HT = 256, THREADS = VT + HT;
  static constexpr int VB_COLS = 256;
  static constexpr int VB_PITCH = 4 * VB_COLS + 4;  // floats; pitch / 4 odd: 8 rows x 4 images conflict-free
  static constexpr int GOFF = (PASSES + 2) * D + 2;
  static constexpr int NBH = (HS + L - 1) / L;       // H blocks per half
  static constexpr int GH_LEN = NBH * L + GOFF;
  static constexpr int NFT = 4;                       // f boxes in flight (one per V block)
  static constexpr int AFC = (WC + 3 + 3) / 4 * 4;    // accumulate-phase f box width (16-byte aligned start)
  static_assert(WC > 0 && WC % 2 == 0, "strip geometry");
  static constexpr size_t F_BYTES = (size_t)L * FCOLS * 4;
  static constexpr size_t F_STRIDE = (F_BYTES + 127) / 128 * 128;
  static constexpr size_t VB_BYTES = (size_t)VROWS * VB_PITCH * 4;
  static constexpr size_t AF_BYTES = ((size_t)GR * AFC * 4 + 127) / 128 * 128;
};

// scalar cascade for the H warps: the running sum is the last operation,
//   A_t = A_{t-1} + (b x_t + (a (x_{t-1} - x_{t-2D}) - b x_{t-2D-1})),
// so the loop-carried dependency is one FADD per pass and step (hcascade's
// nested form carries three dependent FFMAs)
template <int J, int L, int D, int PASSES, bool BORDER>
__device__ __forceinline__ float hcascade_short(float (&dl)[PASSES][L], float& vlast, float x, float a,
                                                float b, const float* gt) {
  constexpr int JM1 = (J + L - 1) % L, JO1 = (J + 1) % L;
  float acc;
  {
    const float prev = dl[0][JM1], o1 = dl[0][JO1], o2 = dl[0][J];
    const float accp = (PASSES > 1) ? dl[PASSES > 1 ? 1 : 0][JM1] : vlast;
    const float u = fmaf(a, prev - o1, -b * o2);
    dl[0][J] = x;
    acc = accp + fmaf(b, x, u);
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
    const float u = fmaf(a, xp - x1, -b * x2);
    dl[p][J] = acc;
    acc = accp + fmaf(b, BORDER ? acc * gt0 : acc, u);
  }
  vlast = acc;
  return BORDER ? acc * gt[-PASSES * D] : acc;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// wait with a safety net: a protocol error traps instead of hanging the GPU
__device__ __forceinline__ void mbar_wait_guarded(uint64_t* bar, unsigned parity) {
  unsigned ok;
  long long t0 = 0;
  for (;;) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    const long long t = clock64();
    if (t0 == 0) t0 = t;
    else if (t - t0 > 4000000000ll) __trap();
  }
}
__device__ __forceinline__ void bar_sync_named(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// geometry of one work item (every thread derives it from the item index)
struct SweepWItem {
  int item, kk, strip, y0, Bn, T_total, nblocks, ngroups, xs, pad;
  int64_t grow0;
};

template <int R, int PASSES>
__global__ void __launch_bounds__(SweepWCfg<R, PASSES>::THREADS, 1)
    sweepw_kernel(const __grid_constant__ CUtensorMap fmap, const __grid_constant__ CUtensorMap amap,
                  const SweepParams p) {
  using C = SweepWCfg<R, PASSES>;
  constexpr int D = C::D, L = C::L, HALO = C::HALO, WC = C::WC, WH = C::WH, HS = C::HS, COLS = C::COLS;
  constexpr int GR = C::GR, NG = C::NG, VBP = C::VB_PITCH, GOFF = C::GOFF, NBH = C::NBH, NFT = C::NFT;
  constexpr int FSTRIDE = (int)(C::F_STRIDE / 4), AFSTRIDE = (int)(C::AF_BYTES / 4);

  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* sbase = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* ft_full = reinterpret_cast<uint64_t*>(sbase);  // [NFT] TMA landed
  uint64_t* ft_empty = ft_full + NFT;                       // [NFT] all V warps read the box
  uint64_t* vb_full = ft_empty + NFT;                       // [NG] V warps wrote the group
  uint64_t* vb_empty = vb_full + NG;                        // [NG] the H pair consumed the group
  uint64_t* af_full = vb_empty + NG;                        // [NG] accumulate-phase f box landed
  // the current item, decoded by thread 0 (two slots: the H warps may still
  // read item i while thread 0 publishes item i + 1)
  SweepWItem* s_it = reinterpret_cast<SweepWItem*>(sbase + 160);
  float* FT = reinterpret_cast<float*>(sbase + 256);       // NFT boxes: L x FCOLS
  float* AF = FT + NFT * FSTRIDE;                           // NG boxes: GR x AFC (output pixels' f)
  float* VB = AF + NG * AFSTRIDE;                           // ring: VROWS x VB_PITCH
  float* gv = VB + C::VROWS * VBP;
  const int gv_len = p.band + 2 * HALO + GOFF + 2 * L;
  float* ghf = gv + gv_len;      // H factors by step, left-to-right half
  float* ghr = ghf + C::GH_LEN;  // right-to-left half

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
  if (K_eval <= 0) return;  // the divide kernel finds den = 0 everywhere
  const int rows_all = p.out_hi - p.out_lo;

  if (tid == 0) {
    for (int i = 0; i < NFT; ++i) {
      mbar_init(&ft_full[i], 1);
      mbar_init(&ft_empty[i], C::VT / 32);
    }
    for (int i = 0; i < NG; ++i) {
      mbar_init(&vb_full[i], C::VT / 32);
      mbar_init(&vb_empty[i], 2);
      mbar_init(&af_full[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // thread 0 draws the next item and publishes its geometry.  Band height
  // from the device plan (as sbf_sweep.cuh): the largest band that still
  // gives >= 2 items per CTA; the last Ks terms run in short bands so the
  // queue ends with small items
  auto next_item = [&](SweepWItem& it) {
    const int item = atomicAdd(p.ctrl, 1);
    int bandh = p.band;
    {
      const int per_band = max(1, p.nstrips * K_eval);
      const int nb_min = (2 * (int)gridDim.x + per_band - 1) / per_band;
      const int b = (rows_all + nb_min - 1) / nb_min;
      bandh = max(min(b, p.band), min(4 * HALO, p.band));
    }
    const int nbands = (rows_all + bandh - 1) / bandh;
    const int units = p.nstrips * nbands;
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
    if (item >= total) {
      it.item = -1;
      return;
    }
    it.item = item;
    const bool tail = item >= items_big;
    const int i2 = tail ? item - items_big : item;
    const int per = (tail ? Ks : K_eval - Ks) * p.nstrips;
    const int band = i2 / per;
    const int r2 = i2 - band * per;
    it.kk = (tail ? K_eval - Ks : 0) + r2 / p.nstrips;
    const int si = r2 - (r2 / p.nstrips) * p.nstrips;
    // edge strips (costlier border code) first within a band
    it.strip = p.nstrips < 2 ? si : (si == 0 ? 0 : (si == 1 ? p.nstrips - 1 : si - 1));
    const int bh = tail ? bandh_s : bandh;
    it.y0 = p.out_lo + band * bh;
    it.Bn = min(p.out_hi, it.y0 + bh) - it.y0;
    it.T_total = it.Bn + 2 * HALO;
    it.nblocks = (it.T_total + L - 1) / L;
    it.ngroups = (it.T_total + GR - 1) / GR;
    it.xs = it.strip * WC - HALO;                 // image column of haloed index 0
    it.grow0 = p.row0 + (int64_t)(it.y0 - HALO);  // global row of stream position 0
  };

  const int wg = tid >> 7;  // 0, 1: V warpgroups; 2, 3: H warpgroups
  // running totals over the items of this CTA (they carry the mbarrier phases):
  // V blocks (= f boxes) and groups of GR stream steps
  int B0 = 0, G0 = 0;

  if (wg < 2) {
    // =====================================================================
    // V warpgroups
    // =====================================================================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 192;");
    const float fcent = p.centred ? 0.f : (float)p.stats[3];
    const float2 a2 = pk(p.a), nb2 = pk(-p.b), b2 = pk(p.b);
    float2 dA[PASSES][L], dB[PASSES][L];
    float2 lA, lB;
    const int q = tid;  // haloed column of this thread (252..255: unused lanes)
    int g_ready = 0;    // groups whose VB rows are known to be free
#if SBF_SWW_PROF
    long long prof[4] = {0, 0, 0, 0}, tprev = clock64();
#endif
    for (int iter = 0;; ++iter) {
      if (tid == 0) next_item(s_it[iter & 1]);
      bar_sync_named(1, C::THREADS);
      const SweepWItem it = s_it[iter & 1];
      if (it.item < 0) break;
      // border tables (index = stream step + GOFF)
      for (int k = tid; k < it.nblocks * L + GOFF; k += C::VT)
        gv[k] = axis_factor(it.grow0 + (k - GOFF), p.img_H, p.r, p.alpha);
      for (int k = tid; k < C::GH_LEN; k += C::VT) {
        ghf[k] = axis_factor((int64_t)it.xs + (k - GOFF), p.W, p.r, p.alpha);
        ghr[k] = axis_factor((int64_t)it.xs + COLS - 1 - (k - GOFF), p.W, p.r, p.alpha);
      }
      const int sg_lo = (int)smax<int64_t>((int64_t)D - it.grow0, -(1 << 30));
      const int sg_hi = (int)smin<int64_t>(p.img_H - 1 - D - it.grow0, 1 << 30);
      const float omega = (float)p.terms[it.kk].freq;
#pragma unroll
      for (int pp = 0; pp < PASSES; ++pp)
#pragma unroll
        for (int j = 0; j < L; ++j) {
          dA[pp][j] = pk(0.f);
          dB[pp][j] = pk(0.f);
        }
      lA = pk(0.f);
      lB = pk(0.f);
      const int xa = it.xs & ~3;  // box start (16-byte aligned column)
      const float* fcol = FT + q + (it.xs - xa);
      auto issue_box = [&](int blk) {
        const int gb = B0 + blk, slot = gb & (NFT - 1);
        // the box's previous use (NFT blocks ago) must have been read by all V warps
        mbar_wait_guarded(&ft_empty[slot], (unsigned)(((gb / NFT) & 1) ^ 1));
        fence_proxy_async();
        mbar_expect_tx(&ft_full[slot], (unsigned)C::F_BYTES);
        tma_load_2d(FT + slot * FSTRIDE, &fmap, xa, it.y0 - HALO + blk * L, &ft_full[slot]);
      };
      if (tid == 0)
        for (int k = 0; k < min(NFT - 1, it.nblocks); ++k) issue_box(k);
      bar_sync_named(1, C::THREADS);  // tables
      SWW_T(3);

      for (int blk = 0; blk < it.nblocks; ++blk) {
        const int base = blk * L;
        const int gb = B0 + blk, slot = gb & (NFT - 1);
        mbar_wait_guarded(&ft_full[slot], (unsigned)((gb / NFT) & 1));
        SWW_T(0);
        if (tid == 0 && blk + NFT - 1 < it.nblocks) issue_box(blk + NFT - 1);
        // the VB rows this block writes: groups up to g_hi must have been consumed
        const int gsb = G0 * GR + base;  // running step index of the block's first step
        const bool last = blk + 1 == it.nblocks;
        const int g_hi = last ? G0 + it.ngroups - 1 : (gsb + L - 1) / GR;
        while (g_ready <= g_hi) {
          mbar_wait_guarded(&vb_empty[g_ready & (NG - 1)], (unsigned)(((g_ready / NG) & 1) ^ 1));
          ++g_ready;
        }
        SWW_T(1);
        const float* fsrc = fcol + slot * FSTRIDE;
        float* vcol = VB + 4 * q;
        const int r0 = gsb & (C::VROWS - 1);

        auto vblock = [&](auto kind_tag) {
          constexpr int KIND = decltype(kind_tag)::value;  // 0 fast, 1 guarded, 2 border (guarded)
          constexpr bool BORDER = KIND == 2;
          sweep_for<L>([&](auto jc) {
            constexpr int J = decltype(jc)::value;
            if (KIND != 0 && base + J >= it.T_total) return;
            const float fc = fsrc[J * C::FCOLS] - fcent;
            float sv, cv;
            __sincosf(fc * omega, &sv, &cv);
            if (BORDER) {  // rows outside the image contribute nothing
              const int64_t gr = it.grow0 + base + J;
              const float m = (gr >= 0 && gr < p.img_H) ? 1.f : 0.f;
              cv *= m;
              sv *= m;
            }
            const float* gt = gv + base + J + GOFF;
            const float2 fx = make_float2(fc, 1.f);
            const float2 ya =
                vcascade<J, L, D, PASSES, BORDER>(dA, lA, __fmul2_rn(fx, pk(cv)), a2, nb2, b2, gt);
            const float2 yb =
                vcascade<J, L, D, PASSES, BORDER>(dB, lB, __fmul2_rn(fx, pk(sv)), a2, nb2, b2, gt);
            // VB layout per pixel: [F_c, G_c, F_s, G_s]
            float* vdst = vcol + ((r0 + J) & (C::VROWS - 1)) * VBP;
            sts2(vdst, ya);
            sts2(vdst + 2, yb);
          });
        };
        if (!(SBF_SWW_ABL & 4)) {
          const bool clean = base - (PASSES + 2) * D - 1 >= sg_lo && base + L - 1 <= sg_hi;
          if (!clean)
            vblock(std::integral_constant<int, 2>{});
          else if (!last)
            vblock(std::integral_constant<int, 0>{});
          else
            vblock(std::integral_constant<int, 1>{});
        }
        __syncwarp();
        if ((tid & 31) == 0) {
          mbar_arrive(&ft_empty[slot]);
          // groups whose last step lies in this block (all the rest after the last block)
          for (int g = gsb / GR; last ? g <= g_hi : g * GR + GR <= gsb + L; ++g)
            mbar_arrive(&vb_full[g & (NG - 1)]);
        }
        SWW_T(2);
      }
      B0 += it.nblocks;
      G0 += it.ngroups;
    }
#if SBF_SWW_PROF
    if ((tid & 31) == 0)
      for (int k = 0; k < 4; ++k)
        atomicAdd(reinterpret_cast<unsigned long long*>(p.seg) + k, (unsigned long long)prof[k]);
#endif
  } else {
    // =====================================================================
    // H warpgroups: pair = two warps (left / right half) on the same 8 rows
    // =====================================================================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
    const int ht = tid - C::VT;
    const int pair = ht >> 6;
    const int half = (ht >> 5) & 1;             // 0: left to right, 1: right to left
    const int hrow = (ht & 31) >> 2;            // row of the group
    const int himg = ht & 3;                    // image (VB component)
    const int t64 = ht & 63;
    float* const VBg = VB + pair * GR * VBP;    // this pair's VB rows
    float* const AFg = AF + pair * AFSTRIDE;
    int af_uses = 0;
#if SBF_SWW_PROF
    long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tprev = clock64();
#endif
    for (int iter = 0;; ++iter) {
      bar_sync_named(1, C::THREADS);
      // (fields are re-read from shared memory where they are used: the H
      // threads have 56 registers)
      const SweepWItem& it = s_it[iter & 1];
      if (it.item < 0) break;
      // haloed columns with factor 1 (D from the image's left / right edge)
      const int qg_lo = D - it.xs, qg_hi = p.W - 1 - D - it.xs;
      const bool strip_in = -(PASSES + 2) * D - 1 >= qg_lo && COLS + (PASSES + 2) * D + 1 <= qg_hi;
      bar_sync_named(1, C::THREADS);  // tables
      SWW_T(0);

      // this pair's groups: running index n = G0 + m with n % NG == pair
      for (int m = (pair - G0) & (NG - 1); m < it.ngroups; m += NG) {
        const int n = G0 + m;
        const int t0 = m * GR;
        // valid VB rows of this group: stream steps [2 HALO, 2 HALO + Bn)
        const int vlo = max(t0, 2 * HALO) - t0;
        const int vhi = min(t0 + GR, 2 * HALO + it.Bn) - t0;
        if (vlo < vhi) {
          // both warps are past the previous accumulate: the f box is free
          bar_sync_named(2 + pair, 64);
          SWW_T(1);
          if (t64 == 0) {
            const int c0 = it.strip * WC;
            fence_proxy_async();
            mbar_expect_tx(&af_full[pair], (unsigned)(GR * C::AFC * 4));
            tma_load_2d(AFg, &amap, c0 & ~3, it.y0 - 2 * HALO + t0, &af_full[pair]);
          }
        }
        mbar_wait_guarded(&vb_full[pair], (unsigned)((n / NG) & 1));
        SWW_T(2);
        if (vlo < vhi) {
          // ===================== H phase =====================
          if (!(SBF_SWW_ABL & 1) && hrow >= vlo && hrow < vhi) {
            const float a = p.a, b = p.b;
            float hd[PASSES][L];
            float hlast = 0.f;
#pragma unroll
            for (int pp = 0; pp < PASSES; ++pp)
#pragma unroll
              for (int j = 0; j < L; ++j) hd[pp][j] = 0.f;
            // step s of the left half reads column s, of the right half
            // column COLS-1-s; the value leaving the cascade at step s belongs
            // to the column read at step s - HALO and is stored over the
            // column read at step s - 2 HALO
            float* v0 = VBg + hrow * VBP + himg + (half ? 4 * (COLS - 1) : 0);
            const float* gh = (half ? ghr : ghf) + GOFF;
            // kind: 0 warm-up (no outputs), 1 main, 2 guarded, 3 border
            auto hstep = [&](auto kind_tag, auto dir_tag, auto j_tag, const int hbase) {
              constexpr int KIND = decltype(kind_tag)::value;
              constexpr int DIR = decltype(dir_tag)::value;
              constexpr int J = decltype(j_tag)::value;
              constexpr bool GUARD = KIND >= 2, BORDER = KIND == 3;
              constexpr int SG = DIR ? -4 : 4;
              const int s = hbase + J;
              if (GUARD && s >= HS) return;
              float* vp = v0 + SG * hbase;
              float x = vp[SG * J];
              if (BORDER) {
                const int cc = it.xs + (DIR ? COLS - 1 - s : s);
                x = (cc >= 0 && cc < p.W) ? x : 0.f;
              }
              const float yv = hcascade_short<J, L, D, PASSES, BORDER>(hd, hlast, x, a, b, gh + s);
              if (KIND == 1 || (GUARD && s >= 2 * HALO)) vp[SG * (J - 2 * HALO)] = yv;
            };
            auto hblock = [&](auto kind_tag, auto dir_tag, const int hbase) {
              sweep_for<L>([&](auto jc) { hstep(kind_tag, dir_tag, jc, hbase); });
            };
            constexpr int KB_MAIN0 = (2 * HALO + L - 1) / L;  // first block with base >= 2 HALO
            constexpr int KB_MAIN1 = HS / L;                  // blocks [KB_MAIN0, KB_MAIN1) are main
            auto hrun = [&](auto dir_tag) {
              if (strip_in && KB_MAIN0 < KB_MAIN1) {
                sweep_for<KB_MAIN0>([&](auto kc) {
                  constexpr int KB = decltype(kc)::value;
                  if constexpr (KB * L + L <= 2 * HALO)
                    hblock(std::integral_constant<int, 0>{}, dir_tag, KB * L);
                  else
                    hblock(std::integral_constant<int, 2>{}, dir_tag, KB * L);
                });
#pragma unroll 1
                for (int kb = KB_MAIN0; kb < KB_MAIN1; ++kb)
                  hblock(std::integral_constant<int, 1>{}, dir_tag, kb * L);
                // the steps left over after the last whole block
                sweep_for<HS - KB_MAIN1 * L>([&](auto jc) {
                  hstep(std::integral_constant<int, 1>{}, dir_tag, jc, KB_MAIN1 * L);
                });
              } else {
#pragma unroll 1
                for (int kb = 0; kb < NBH; ++kb) {
                  const int hb = kb * L;
                  // the block reads factors back to step hb - (PASSES+2) D - 1
                  const int s_lo = hb - (PASSES + 2) * D - 1, s_hi = hb + L - 1;
                  const int c_lo = decltype(dir_tag)::value ? COLS - 1 - s_hi : s_lo;
                  const int c_hi = decltype(dir_tag)::value ? COLS - 1 - s_lo : s_hi;
                  if (c_lo >= qg_lo && c_hi <= qg_hi)
                    hblock(std::integral_constant<int, 2>{}, dir_tag, hb);
                  else
                    hblock(std::integral_constant<int, 3>{}, dir_tag, hb);
                }
              }
            };
            if (half) hrun(std::integral_constant<int, 1>{});
            else hrun(std::integral_constant<int, 0>{});
          }
          SWW_T(3);
          bar_sync_named(2 + pair, 64);
          SWW_T(4);
          mbar_wait_guarded(&af_full[pair], (unsigned)(af_uses & 1));
          ++af_uses;
          SWW_T(5);

          // ===================== accumulate =====================
          // (num, den) of this term in 32-bit fixed point, both halves of one
          // 64-bit integer, one red.add.u64 per pixel (order-independent)
          if (!(SBF_SWW_ABL & 2)) {
            const float fcent = p.centred ? 0.f : (float)p.stats[3];
            const double centerd = p.stats[3];
            const double maxdev = fmax(p.stats[2] - centerd, centerd - p.stats[1]);
            const int nexp = ilogb(fmax(maxdev, 1.0)) + 1;  // maxdev < 2^nexp
            const sbf_term term = p.terms[it.kk];
            const float scale = (float)term.scale;
            const float omega = (float)term.freq;
            const float2 fxs = make_float2(scale * ldexpf(1.f, 29 - nexp), scale * ldexpf(1.f, 29));
            const int c0 = it.strip * WC;
            const int xlim = min(WC, p.W - c0);
            const int ra = it.y0 - 2 * HALO + t0 + vlo - p.out_lo;  // first output row (rel. out_lo)
            const int nr = vhi - vlo;
            for (int jc = t64; jc < xlim; jc += 64) {
              const float* vb = VBg + vlo * VBP + 4 * (jc < WH ? jc : jc + 2 * HALO);
              unsigned long long* dst = p.acc + (int64_t)ra * p.W + (c0 + jc);
              // the output pixel's own sample, for its phasor (as the V phase formed it)
              const float* fsrc = AFg + vlo * C::AFC + (c0 & 3) + jc;
#pragma unroll 4
              for (int v = 0; v < nr; ++v) {
                const float4 pv = *reinterpret_cast<const float4*>(vb + v * VBP);
                float sv, cv;
                __sincosf((fsrc[v * C::AFC] - fcent) * omega, &sv, &cv);
                float2 t = __ffma2_rn(pk(sv), make_float2(pv.z, pv.w),
                                      __fmul2_rn(pk(cv), make_float2(pv.x, pv.y)));
                t = __fmul2_rn(t, fxs);
                const long long qv =
                    ((long long)__float2int_rn(t.x) << 32) + (long long)__float2int_rn(t.y);
                asm volatile("red.global.add.u64 [%0], %1;" ::"l"(dst + (int64_t)v * p.W), "l"(qv)
                             : "memory");
              }
            }
          }
        }
        __syncwarp();
        if ((ht & 31) == 0) mbar_arrive(&vb_empty[pair]);
        SWW_T(6);
      }
      G0 += it.ngroups;
    }
#if SBF_SWW_PROF
    if ((ht & 31) == 0)
      for (int k = 0; k < 8; ++k)
        atomicAdd(reinterpret_cast<unsigned long long*>(p.seg) + 4 + k, (unsigned long long)prof[k]);
#endif
  }
}

// ---- host side ----
template <int R, int PASSES>
size_t sweepw_smem_bytes(int band) {
  using C = SweepWCfg<R, PASSES>;
  return 512 + C::NFT * C::F_STRIDE + C::NG * C::AF_BYTES + C::VB_BYTES +
         (size_t)(band + 2 * C::HALO + C::GOFF + 2 * C::L + 2 * C::GH_LEN) * 4 + 16;
}

template <int R, int PASSES>
int launch_sweepw(const CUtensorMap& map, const CUtensorMap& amap, const SweepParams& p, cudaStream_t st) {
  using C = SweepWCfg<R, PASSES>;
  const size_t smem = sweepw_smem_bytes<R, PASSES>(p.band);
  SBF_CHECK_CUDA(ensure_dyn_smem(reinterpret_cast<const void*>(sweepw_kernel<R, PASSES>), smem));
  const int grid = device_sm_count();  // one persistent CTA per SM
  SBF_CHECK_CUDA(launch_pdl(sweepw_kernel<R, PASSES>, dim3((unsigned)grid), dim3(C::THREADS), smem, st,
                            map, amap, p));
  SBF_CHECK_LAUNCH();
  return SBF_OK;
}

}  // namespace sbf
