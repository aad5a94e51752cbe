// K3 — fused per-term shiftable-filter kernel (sm_100a, FP32-issue bound).
//
// Replaces, per folded cosine term (reference bilateral.py:150-163):
//   theta = omega_n f; gc, gs = cos, sin; four apply_spatial() smoothings of
//   f*gc, gc, f*gs, gs (spatial.py:108-139: `passes` extended-box passes,
//   rows then columns, each renormalised over the clamped window,
//   _extended_box_lines spatial.py:120-133 on top of window_sum_lines
//   _fastcore.pyx:61-86); num/den += scale (gc*S[f gc] + gs*S[f gs]) / ...
//
// B200 design ("strip sweep", one CTA = one vertical strip x one row band x
// one term group):
//  * V phase: one thread per haloed column streams the band top to bottom.
//    It builds cos/sin of 2*pi*frac(f * omega/2pi) (explicit range reduction
//    + MUFU in fp32 mode, fp64 reduction + accurate sincospi in HDR mode),
//    the 4 modulated images, and runs the `PASSES` column passes as O(1)
//    running-sum recurrences
//       V += a (x[t-1] - x[t-2D]) + b (x[t] - x[t-2D-1]),  D = r+1,
//       a = (1-alpha)/cnt, b = alpha/cnt, cnt = 2r+1+2alpha,
//    with the delay lines held in registers (compile-time rotation of a
//    2r+3 register ring; no shuffles, no shared-memory traffic).  Border
//    renormalisation is exact: zero padding plus a per-position factor
//    cnt/cnt(pos) (pos outside the image -> 0), applied only in chunks that
//    touch a true image border.
//  * The vertically smoothed rows go to shared memory in chunks of ROWS rows
//    (VB); raw scale*cos/scale*sin of the output pixels go to a small ring.
//  * H phase: 4 lanes per row (one per image) stream the chunk's rows left to
//    right with the same register recurrence, multiply by the raw phasor of
//    the output pixel and write the products back in place.
//  * Accumulate: the products are summed to (num, den) and added to this
//    CTA's exclusive slice of a partial accumulator in global memory (L2)
//    with vector red.add (first term of the group: plain store).
// Intermediate images never touch HBM.  Terms of the group are swept one
// after another; groups split the term list across CTAs (strided, largest
// weights first) and are summed by the epilogue.
#pragma once

#include <type_traits>

#include "sbf_common.cuh"

namespace sbf {

struct TermParams {
  const void* f;
  int64_t ld;
  int f64;
  int H;  // buffer rows
  int W;
  int64_t row0;   // global row index of buffer row 0
  int64_t img_H;  // global image height
  int out_lo, out_hi;
  int band;
  int nstrips, nbands, groups;
  int r;
  float alpha;
  float a, b;
  double ad, bd;
  const sbf_plan* plan;
  const sbf_term* terms;
  const double* stats;
  void* nd;
  int64_t nd_group_stride;  // (num, den) pairs per group
};

template <int R, int PASSES, int MODE>
struct TermCfg {
  static constexpr int D = R + 1;
  static constexpr int L = 2 * R + 3;
  static constexpr int HALO = PASSES * D;
  static constexpr int IMGS = (MODE == 0 && R <= 5) ? 4 : 2;
  static constexpr int HALO_W = 128;
  static constexpr int WC = HALO_W - 2 * HALO;
  static constexpr int THREADS = HALO_W * 4 / IMGS;
  static constexpr int ROWS = THREADS / 4;
  static constexpr int RING = ROWS + HALO;
  static constexpr int VB_PITCH = HALO_W * 4 + 4;  // floats; == 4 mod 32 banks
  static constexpr int RAW_PITCH = 2 * WC + 2;     // floats; == 2 mod 4 (WC even)
  static constexpr int MIN_BLOCKS = (IMGS == 4) ? 2 : 1;
  static_assert(WC > 0, "halo too wide for a 128-column strip");
  static_assert(HALO <= ROWS, "RAW ring assumes halo <= rows per chunk");
};

template <int MODE>
struct AccT;
template <>
struct AccT<0> {
  using type = float;
};
template <>
struct AccT<1> {
  using type = double;
};

// normalisation factor cnt_int / cnt(pos) on an axis of length n (0 outside)
__device__ __forceinline__ double gfactor(int64_t pos, int64_t n, int r, double alpha) {
  if (pos < 0 || pos >= n) return 0.0;
  const int64_t lo = pos - r < 0 ? 0 : pos - r;
  const int64_t hi = pos + r > n - 1 ? n - 1 : pos + r;
  double cnt = (double)(hi - lo + 1);
  if (alpha > 0.0) {
    if (pos - r - 1 >= 0) cnt += alpha;
    if (pos + r + 1 <= n - 1) cnt += alpha;
  }
  const double cint = 2.0 * r + 1.0 + (alpha > 0.0 ? 2.0 * alpha : 0.0);
  return cint / cnt;
}

template <int R, int PASSES, int MODE>
struct VState {
  using C = TermCfg<R, PASSES, MODE>;
  using acc_t = typename AccT<MODE>::type;
  float dl[PASSES][C::IMGS][C::L];
  acc_t V[PASSES][C::IMGS];
  float fq[C::L];
};

template <int R, int PASSES, int MODE>
__global__ void __launch_bounds__(TermCfg<R, PASSES, MODE>::THREADS,
                                  TermCfg<R, PASSES, MODE>::MIN_BLOCKS)
    terms_kernel(const TermParams p) {
  using C = TermCfg<R, PASSES, MODE>;
  using acc_t = typename AccT<MODE>::type;
  constexpr int D = C::D, L = C::L, HALO = C::HALO, IMGS = C::IMGS, WC = C::WC;
  constexpr int ROWS = C::ROWS, RING = C::RING, VBP = C::VB_PITCH, RAWP = C::RAW_PITCH;
  constexpr int HALO_W = C::HALO_W, THREADS = C::THREADS;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* VB = reinterpret_cast<float*>(smem_raw);
  float* RAW = VB + ROWS * VBP;
  acc_t* gv = reinterpret_cast<acc_t*>(RAW + RING * RAWP);
  const int gv_len = p.band + 2 * HALO + HALO;
  acc_t* gh = gv + gv_len;

  const sbf_plan* plan = p.plan;
  if (plan->status != SBF_OK) return;
  const int K_eval = plan->K_eval;
  int bid = blockIdx.x;
  const int grp = bid % p.groups;
  bid /= p.groups;
  const int strip = bid % p.nstrips;
  const int band = bid / p.nstrips;
  if (grp >= K_eval) return;

  const int tid = threadIdx.x;
  const int y0 = p.out_lo + band * p.band;
  const int y1 = min(p.out_hi, y0 + p.band);
  const int Bn = y1 - y0;
  const int T_total = Bn + 2 * HALO;
  const int xs = strip * WC - HALO;  // image column of haloed index 0
  const double center = p.stats[3];
  const float centerf = (float)center;

  // ---- per-CTA border tables ----
  for (int k = tid; k < gv_len; k += THREADS) {
    const int64_t grow = p.row0 + (int64_t)(y0 - HALO + (k - HALO));
    gv[k] = (acc_t)gfactor(grow, p.img_H, p.r, (double)p.alpha);
  }
  for (int k = tid; k < HALO_W + HALO; k += THREADS) {
    gh[k] = (acc_t)gfactor((int64_t)xs + (k - HALO), p.W, p.r, (double)p.alpha);
  }
  // a strip is "interior" when every column any pass touches has factor 1
  const bool strip_interior = (xs - HALO >= D) && ((int64_t)xs + HALO_W <= (int64_t)p.W - 1 - D);
  __syncthreads();

  // ---- roles ----
  constexpr int TPC = 4 / IMGS;  // V threads per column
  const int q = tid / TPC;       // haloed column of this V thread
  const int pair = tid % TPC;    // IMGS==2: 0 -> (f cos, cos), 1 -> (f sin, sin)
  const int col = xs + q;
  const bool col_ok = col >= 0 && col < p.W;
  const float colmask = col_ok ? 1.f : 0.f;
  const bool out_col = q >= HALO && q < HALO + WC;
  const int hv = tid >> 2;   // H-phase row within the chunk
  const int himg = tid & 3;  // H-phase image: 0 f*cos, 1 cos, 2 f*sin, 3 sin

  const char* fbase = static_cast<const char*>(p.f);

  VState<R, PASSES, MODE> st;

  for (int kk = grp; kk < K_eval; kk += p.groups) {
    const sbf_term term = p.terms[kk];
    const bool first = (kk == grp);
    const float scale = (float)term.scale;
    const float nu = (float)term.turns;
    const double nud = term.turns;

    // reset the recurrences; prefetch f for steps 0..L-1
#pragma unroll
    for (int pp = 0; pp < PASSES; ++pp)
#pragma unroll
      for (int i = 0; i < IMGS; ++i) {
        st.V[pp][i] = 0;
#pragma unroll
        for (int j = 0; j < L; ++j) st.dl[pp][i][j] = 0.f;
      }
    auto fetch = [&](int t) -> float {
      const int brow = y0 - HALO + t;
      const int64_t grow = p.row0 + brow;
      if (!col_ok || t >= T_total || brow < 0 || brow >= p.H || grow < 0 || grow >= p.img_H)
        return 0.f;
      const int64_t idx = (int64_t)brow * p.ld + col;
      if (p.f64) return (float)(__ldg(reinterpret_cast<const double*>(fbase) + idx) - center);
      // centre is fp32-representable: the fp32 difference is the correctly
      // rounded exact difference, identical to the fp64 route
      return __ldg(reinterpret_cast<const float*>(fbase) + idx) - centerf;
    };
#pragma unroll
    for (int j = 0; j < L; ++j) st.fq[j] = fetch(j);

    for (int t0 = 0; t0 < T_total; t0 += ROWS) {
      const int t1 = min(t0 + ROWS, T_total);
      // rows touched by this chunk's passes: stream positions [t0-HALO, t1)
      const int64_t glo = p.row0 + (y0 - HALO) + (t0 - HALO);
      const int64_t ghi = p.row0 + (y0 - HALO) + (t1 - 1);
      const bool chunk_interior = strip_interior && glo >= D && ghi <= p.img_H - 1 - D;
      // RAW ring slot of input step t0 (output rows only)
      const int rs0 = ((t0 - HALO) % RING + RING) % RING;

      // ===================== V phase =====================
      auto vphase = [&](auto border_tag) {
        constexpr bool BORDER = decltype(border_tag)::value;
        const int kb0 = t0 / L, kb1 = (t1 - 1) / L;
        for (int kb = kb0; kb <= kb1; ++kb) {
          const int base = kb * L;
#pragma unroll
          for (int J = 0; J < L; ++J) {
            const int t = base + J;
            if (t < t0 || t >= t1) continue;
            const float fc = st.fq[J];
            st.fq[J] = fetch(t + L);
            // phasor of this pixel for the current term
            float cv, sv;
            if (MODE == 0) {
              const float u = fc * nu;
              const float k = (u + 12582912.f) - 12582912.f;  // rint, |u| < 2^22
              const float tt = u - k;
              if (IMGS == 4) {
                __sincosf(tt * 6.28318530717958647f, &sv, &cv);
              } else {
                cv = __cosf((tt - 0.25f * pair) * 6.28318530717958647f);
                sv = cv;
              }
            } else {
              const double ud = (double)fc * nud;
              const float tt = (float)(ud - rint(ud));
              if (IMGS == 4) {
                sincospif(2.f * tt, &sv, &cv);
              } else {
                cv = cospif(2.f * (tt - 0.25f * pair));
                sv = cv;
              }
            }
            if (BORDER) {
              const int64_t grow = p.row0 + (y0 - HALO + t);
              const float m = (grow >= 0 && grow < p.img_H) ? colmask : 0.f;
              cv *= m;
              sv *= m;
            }
            float x[IMGS];
            if (IMGS == 4) {
              x[0] = fc * cv;
              x[1] = cv;
              x[2] = fc * sv;
              x[3] = sv;
            } else {
              x[0] = fc * cv;
              x[1] = cv;
            }
            // raw scaled phasor of output pixels for the H phase
            if (t >= HALO && t < HALO + Bn && out_col) {
              int slot = rs0 + (t - t0);
              if (slot >= RING) slot -= RING;
              float* rp = RAW + slot * RAWP + 2 * (q - HALO);
              if (IMGS == 4) {
                *reinterpret_cast<float2*>(rp) = make_float2(scale * cv, scale * sv);
              } else {
                rp[pair] = scale * cv;
              }
            }
            // column passes
            acc_t gfac[PASSES];
            if (BORDER) {
#pragma unroll
              for (int pp = 0; pp < PASSES; ++pp) gfac[pp] = gv[t - (pp + 1) * D + HALO];
            }
#pragma unroll
            for (int i = 0; i < IMGS; ++i) {
              float xin = x[i];
#pragma unroll
              for (int pp = 0; pp < PASSES; ++pp) {
                const float prev = st.dl[pp][i][(J + L - 1) % L];
                const float o1 = st.dl[pp][i][(J + 1) % L];
                const float o2 = st.dl[pp][i][J];
                st.dl[pp][i][J] = xin;
                if (MODE == 0) {
                  float v = st.V[pp][i];
                  v = fmaf(p.a, prev - o1, v);
                  v = fmaf(p.b, xin - o2, v);
                  st.V[pp][i] = v;
                  xin = BORDER ? v * (float)gfac[pp] : v;
                } else {
                  double v = st.V[pp][i];
                  v = fma(p.ad, (double)prev - (double)o1, v);
                  v = fma(p.bd, (double)xin - (double)o2, v);
                  st.V[pp][i] = v;
                  xin = (float)(BORDER ? v * (double)gfac[pp] : v);
                }
              }
              x[i] = xin;
            }
            // vertically smoothed output row -> VB
            if (t >= 2 * HALO) {
              float* vp = VB + (t - t0) * VBP + 4 * q;
              if (IMGS == 4) {
                *reinterpret_cast<float4*>(vp) = make_float4(x[0], x[1], x[2], x[3]);
              } else {
                *reinterpret_cast<float2*>(vp + 2 * pair) = make_float2(x[0], x[1]);
              }
            }
          }
        }
      };
      if (chunk_interior)
        vphase(std::integral_constant<bool, false>{});
      else
        vphase(std::integral_constant<bool, true>{});
      __syncthreads();

      // ===================== H phase =====================
      {
        const int t = t0 + hv;
        if (t < t1 && t >= 2 * HALO) {
          float* vrow = VB + hv * VBP;
          const int oslot = ((t - 2 * HALO) % RING);
          const float* rrow = RAW + oslot * RAWP + (himg >> 1);
          float hd[PASSES][L];
          acc_t hV[PASSES];
#pragma unroll
          for (int pp = 0; pp < PASSES; ++pp) {
            hV[pp] = 0;
#pragma unroll
            for (int j = 0; j < L; ++j) hd[pp][j] = 0.f;
          }
          auto hphase = [&](auto border_tag) {
            constexpr bool BORDER = decltype(border_tag)::value;
            constexpr int NB = (HALO_W + L - 1) / L;
            for (int kb = 0; kb < NB; ++kb) {
              const int base = kb * L;
              float in[L], rw[L];
#pragma unroll
              for (int J = 0; J < L; ++J) {
                const int qq = base + J;
                in[J] = (qq < HALO_W) ? vrow[4 * qq + himg] : 0.f;
                const int j = qq - 2 * HALO;
                rw[J] = (j >= 0 && j < WC) ? rrow[2 * j] : 0.f;
              }
#pragma unroll
              for (int J = 0; J < L; ++J) {
                const int qq = base + J;
                if (qq >= HALO_W) break;
                float xin = in[J];
#pragma unroll
                for (int pp = 0; pp < PASSES; ++pp) {
                  const float prev = hd[pp][(J + L - 1) % L];
                  const float o1 = hd[pp][(J + 1) % L];
                  const float o2 = hd[pp][J];
                  hd[pp][J] = xin;
                  if (MODE == 0) {
                    float v = hV[pp];
                    v = fmaf(p.a, prev - o1, v);
                    v = fmaf(p.b, xin - o2, v);
                    hV[pp] = v;
                    xin = BORDER ? v * (float)gh[qq - (pp + 1) * D + HALO] : v;
                  } else {
                    double v = hV[pp];
                    v = fma(p.ad, (double)prev - (double)o1, v);
                    v = fma(p.bd, (double)xin - (double)o2, v);
                    hV[pp] = v;
                    xin = (float)(BORDER ? v * (double)gh[qq - (pp + 1) * D + HALO] : v);
                  }
                }
                if (qq >= 2 * HALO) vrow[4 * (qq - HALO) + himg] = xin * rw[J];
              }
            }
          };
          if (strip_interior)
            hphase(std::integral_constant<bool, false>{});
          else
            hphase(std::integral_constant<bool, true>{});
        }
      }
      __syncthreads();

      // ===================== accumulate =====================
      {
        const int vlo = max(t0, 2 * HALO) - t0;
        const int vhi = min(t1, 2 * HALO + Bn) - t0;
        const int items = (vhi - vlo) * WC;
        for (int it = tid; it < items; it += THREADS) {
          const int vv = vlo + it / WC;
          const int j = it - (it / WC) * WC;
          const int x = strip * WC + j;
          if (x >= p.W) continue;
          const float4 pv = *reinterpret_cast<const float4*>(VB + vv * VBP + 4 * (HALO + j));
          const int y = y0 - 2 * HALO + t0 + vv;
          const int64_t idx = (int64_t)grp * p.nd_group_stride + (int64_t)(y - p.out_lo) * p.W + x;
          if (MODE == 0) {
            const float num = pv.x + pv.z, den = pv.y + pv.w;
            float2* dst = reinterpret_cast<float2*>(p.nd) + idx;
            if (first) {
              *dst = make_float2(num, den);
            } else {
              asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(dst), "f"(num), "f"(den)
                           : "memory");
            }
          } else {
            const double num = (double)pv.x + (double)pv.z, den = (double)pv.y + (double)pv.w;
            double* dst = reinterpret_cast<double*>(p.nd) + 2 * idx;
            if (first) {
              *reinterpret_cast<double2*>(dst) = make_double2(num, den);
            } else {
              atomicAdd(dst, num);
              atomicAdd(dst + 1, den);
            }
          }
        }
      }
      __syncthreads();
    }
  }
}

// ---- host launcher ----
template <int R, int PASSES, int MODE>
size_t terms_smem_bytes(int band) {
  using C = TermCfg<R, PASSES, MODE>;
  using acc_t = typename AccT<MODE>::type;
  return (size_t)C::ROWS * C::VB_PITCH * 4 + (size_t)C::RING * C::RAW_PITCH * 4 +
         (size_t)(band + 3 * C::HALO + C::HALO_W + C::HALO) * sizeof(acc_t) + 16;
}

template <int R, int PASSES, int MODE>
int launch_terms(const TermParams& p, cudaStream_t st) {
  using C = TermCfg<R, PASSES, MODE>;
  const size_t smem = terms_smem_bytes<R, PASSES, MODE>(p.band);
  SBF_CHECK_CUDA(cudaFuncSetAttribute(terms_kernel<R, PASSES, MODE>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const long long grid = (long long)p.nstrips * p.nbands * p.groups;
  terms_kernel<R, PASSES, MODE><<<(unsigned)grid, C::THREADS, smem, st>>>(p);
  SBF_CHECK_LAUNCH();
  return SBF_OK;
}

template <int R, int PASSES, int MODE>
void terms_geometry(int* halo, int* wc, int* threads, int* blocks_per_sm) {
  using C = TermCfg<R, PASSES, MODE>;
  *halo = C::HALO;
  *wc = C::WC;
  *threads = C::THREADS;
  *blocks_per_sm = C::MIN_BLOCKS;
}

// dispatch table entry
struct TermsEntry {
  int r, passes, mode;
  int (*launch)(const TermParams&, cudaStream_t);
  size_t (*smem)(int);
  void (*geom)(int*, int*, int*, int*);
};

#define SBF_TERMS_ENTRY(R, P, M) \
  TermsEntry { R, P, M, &launch_terms<R, P, M>, &terms_smem_bytes<R, P, M>, &terms_geometry<R, P, M> }

}  // namespace sbf
