/*
 * sbf.h — C ABI of the B200-native shiftable bilateral filter (sm_100a).
 *
 * Drop-in boundary for the hot path of the reference package `shiftbf`
 * (arXiv 1203.5128).  Plain pointers and sizes only: no torch types.  All
 * device pointers are caller-owned; the library never frees them.  Every
 * call is stream-ordered and reentrant.  Process-wide state: a thread-local
 * error string, thread-local tuning switches (sbf_set_* below, for
 * benchmarks; defaults are the measured best), per-device caches (SM count,
 * the dual form's weight tables of the last geometry) and, on first use of
 * a device, a raised release threshold of its default stream-ordered memory
 * pool (scratch blocks are kept across calls).  Status codes mirror the reference CLI exit
 * codes (reference cli.py:309-314) and map onto its exception types
 * (reference errors.py:4-25):
 *
 *   SBF_OK               0
 *   SBF_ERR_INVALID      2  -> InvalidParameterError
 *   SBF_ERR_UNSUPPORTED  4  -> UnsupportedOrderError (order/term capacity)
 *   SBF_ERR_CUDA         5  -> RuntimeError (launch or device fault)
 *   SBF_ERR_WORKSPACE    6  -> InvalidParameterError (workspace too small)
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/shiftbf):
 *   sbf_extended_box_params   spatial.py:81-100   extended_box_params
 *   sbf_support_radius        spatial.py:185-194  support_radius
 *   sbf_select_plan           kernels.py:166-195  select_plan (host twin of K2)
 *   sbf_truncation_index_exact kernels.py:131-149
 *   sbf_truncation_index_chernoff kernels.py:152-163
 *   sbf_local_range           maxfilter.py:41-61  max_filter_2d + compute_T
 *                             (_core running_max_lines, _fastcore.pyx:16-58)
 *   sbf_plan_device           kernels.py:166-227  select_plan +
 *                             raised_cosine_expansion, on the device
 *   sbf_filter                bilateral.py:140-164 _accumulate_cosine_terms
 *                             + spatial.py:108-139 iterated_box_gaussian /
 *                             :65-78 box_filter (+ _core window_sum_lines,
 *                             _fastcore.pyx:61-86) + bilateral.py:242-254
 *                             _divide_with_fallback
 *   sbf_shiftable_bf          bilateral.py:117-137 shiftable_bf (device bufs)
 *   sbf_shiftable_bf_host     bilateral.py:117-137 shiftable_bf (host bufs)
 */
#ifndef SBF_H_
#define SBF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SBF_ABI_VERSION 1

#define SBF_OK 0
#define SBF_ERR_INVALID 2
#define SBF_ERR_UNSUPPORTED 4
#define SBF_ERR_CUDA 5
#define SBF_ERR_WORKSPACE 6

/* element types of image buffers */
#define SBF_F32 0
#define SBF_F64 1

/* truncation rules (kernels.py:173-192) */
#define SBF_RULE_AUTO 0
#define SBF_RULE_EXACT 1
#define SBF_RULE_CHERNOFF 2
#define SBF_RULE_NONE 3

/* spatial modes (spatial.py:24-42) */
#define SBF_SPATIAL_ITERATED 0
#define SBF_SPATIAL_BOX 1
#define SBF_SPATIAL_FIR 2        /* sampled Gaussian taps, radius r (sbf_smooth / direct only) */

/* precision modes of the term kernel */
#define SBF_PREC_FP32 0   /* fp32 phases, sums and accumulators (8-bit-scale images) */
#define SBF_PREC_HDR 1    /* fp64 running sums and num/den accumulators (16-bit scale) */
#define SBF_PREC_AUTO 2   /* fp32 kernels, guarded on the device: if max|f - centre| > 4096
                             the term kernel does nothing and sets SBF_PLAN_NEEDS_HDR
                             (the caller re-runs with SBF_PREC_HDR); no host sync */

/* plan flags */
#define SBF_PLAN_N_AMBIGUOUS 1     /* ceil(0.405 x^2) changes within +-2 ulp of x^2 */
#define SBF_PLAN_EXACT_BIGINT 2    /* exact rule resolved by the multi-limb path */
#define SBF_PLAN_TERMS_TRUNCATED 4 /* term table capacity exceeded (status set) */
#define SBF_PLAN_NEEDS_HDR 8       /* SBF_PREC_AUTO found a wide intensity range */

typedef struct sbf_plan {
  double T;        /* dynamic range the plan was built for */
  double sigma_r;
  double epsilon;
  double gamma;    /* 1 / (sqrt(N) sigma_r) */
  int32_t N;       /* kernel order */
  int32_t M;       /* terms dropped from each tail */
  int32_t K;       /* folded terms n in [M, floor(N/2)] */
  int32_t K_eval;  /* folded terms with non-zero weight (evaluated) */
  int32_t flags;
  int32_t status;  /* SBF_OK or an error code */
  int32_t pad0, pad1;
} sbf_plan;        /* 64 bytes */

typedef struct sbf_term {
  double scale;    /* d_n, or 2 d_n for a folded +-pair (bilateral.py:154) */
  double freq;     /* omega_n = (2n - N) / (sqrt(N) sigma_r) */
  double turns;    /* omega_n / (2 pi) */
  int32_t index;   /* n */
  int32_t pad;
} sbf_term;        /* 32 bytes */

typedef struct sbf_spatial {
  int32_t mode;    /* SBF_SPATIAL_* */
  int32_t passes;  /* 1 for box */
  int32_t r;       /* per-pass integer radius */
  int32_t pad;
  double alpha;    /* endpoint weight (0 for box) */
  double sigma_s;  /* informational */
} sbf_spatial;

/* ---- library info ---- */
int sbf_abi_version(void);
const char* sbf_last_error(void);
int sbf_device_count(int* count);

/* ---- host scalar logic (identical code runs on the device in K2) ---- */
int sbf_extended_box_params(double sigma_s, int passes, int* r, double* alpha);
int sbf_support_radius(const sbf_spatial* sp, int* radius);
int sbf_truncation_index_exact(int N, double epsilon, int* M);
int sbf_truncation_index_chernoff(int N, double epsilon, double log_2_over_eps, int* M);
int sbf_order_threshold(double T, double sigma_r, int* N);
/* C(N, n) / 2^N for n in [lo, hi], correctly rounded to float64 (exact
 * multi-limb integers on the host) — replaces kernels.py:198-212
 * binomial_weights; raised_cosine_expansion builds on it. */
int sbf_binomial_weights(int N, int lo, int hi, double* out);
/* Brute-force local range (maxfilter.py:64-82 brute_force_T): O(R^2) per
 * pixel on the device, independent of the separable max filter; the result
 * is written to *T_out (host) after a stream synchronisation. */
int sbf_brute_force_T(const void* f, int dtype, int64_t H, int64_t W, int64_t ld, int R,
                      double* T_out, void* stream);
int sbf_select_plan(double T, double sigma_r, double epsilon, int rule,
                    double log_2_over_eps, sbf_plan* out);

/* ---- device entry points (all pointers device memory, stream = cudaStream_t) ---- */

/* Workspace (bytes) needed by sbf_local_range for an H x W image. */
size_t sbf_local_range_workspace(int64_t H, int64_t W, int dtype);

/* Max filter over the clamped (2R+1)^2 window and T = max(M - f) in fp64.
 * f: H x W row-major (row pitch `ld` elements), dtype SBF_F32/SBF_F64.
 * T and the image statistics are computed over buffer rows [t_lo, t_hi)
 * (row strips with halos: pass the interior rows).  M_out (nullable) gets
 * the max-filter image in the input dtype.  stats_dev (>= 4 doubles):
 * [0] = T, [1] = min f, [2] = max f, [3] = centre used by sbf_filter. */
int sbf_local_range(const void* f, int dtype, int64_t H, int64_t W, int64_t ld,
                    int R, int64_t t_lo, int64_t t_hi, void* M_out,
                    double* stats_dev, void* ws, size_t ws_bytes, void* stream);

/* Plan on the device from T = *T_dev (or fixed_T if use_fixed != 0):
 * N, M, folded term table sorted largest weight first. */
int sbf_plan_device(const double* T_dev, int use_fixed, double fixed_T,
                    double sigma_r, double epsilon, int rule,
                    double log_2_over_eps, sbf_plan* plan_dev,
                    sbf_term* terms_dev, int terms_cap, void* stream);

/* Same with (N, M) resolved on the host (sbf_select_plan, libm pow); for the
 * rare inputs the device flags SBF_PLAN_N_AMBIGUOUS. */
int sbf_plan_device_forced(const double* T_dev, int use_fixed, double fixed_T,
                           double sigma_r, double epsilon, int rule,
                           double log_2_over_eps, int N, int M, sbf_plan* plan_dev,
                           sbf_term* terms_dev, int terms_cap, void* stream);

/* Workspace (bytes) for sbf_filter on an H x W buffer producing rows_out rows. */
size_t sbf_filter_workspace(int64_t H, int64_t W, int64_t rows_out, int dtype,
                            const sbf_spatial* sp, int precision);

/* The fused shiftable filter for output rows [out_lo, out_hi) of a buffer
 * holding global image rows [row0, row0 + H) of an image of global height
 * img_H (border renormalisation only at true image borders).  The buffer
 * must include every row within the spatial support of the output rows.
 * out: (out_hi - out_lo) x W, pitch W, dtype out_dtype; device memory or
 * page-locked host memory (then written by the device over PCIe: on the K3
 * path segment by segment while the last terms run -- no separate copy).
 * stats_dev: from sbf_local_range ([3] = centre).  fallback_dev: one
 * unsigned long long counter (accumulated). */
int sbf_filter(const void* f, int dtype, int64_t H, int64_t W, int64_t ld,
               int64_t row0, int64_t img_H, int64_t out_lo, int64_t out_hi,
               const sbf_spatial* sp, const sbf_plan* plan_dev,
               const sbf_term* terms_dev, const double* stats_dev,
               int precision, void* out, int out_dtype,
               unsigned long long* fallback_dev, void* ws, size_t ws_bytes,
               void* stream);

/* Whole pipeline (K1 -> K2 -> K3 -> K4) on device buffers.  No host sync
 * and CUDA-graph capturable on the fp32 paths (the K3 sweep, r <= 5, and the
 * split sweep, 6 <= r <= 12, with SBF_PREC_FP32 / SBF_PREC_AUTO).  The fp64 paths
 * (SBF_PREC_HDR, radii without an fp32 kernel) read the plan on the host to
 * size their term loop / pick the dual form: they synchronise the stream
 * and return SBF_ERR_UNSUPPORTED under graph capture.
 * fixed_T < 0 means "compute T with window radius R".  *fallback_dev is set
 * to this call's fallback count (reset by the pipeline, not accumulated). */
size_t sbf_shiftable_bf_workspace(int64_t H, int64_t W, int dtype,
                                  const sbf_spatial* sp, int precision,
                                  int terms_cap);
int sbf_shiftable_bf(const void* f, int dtype, int64_t H, int64_t W,
                     const sbf_spatial* sp, int R, double fixed_T,
                     double sigma_r, double epsilon, int rule,
                     double log_2_over_eps, int precision, void* out,
                     int out_dtype, sbf_plan* plan_dev, double* stats_dev,
                     unsigned long long* fallback_dev, int terms_cap,
                     void* ws, size_t ws_bytes, void* stream);

/* Host-buffer convenience (copies in, runs, copies out, synchronises).
 * Output is float64 like the reference.  plan_out / fallback_out on host. */
int sbf_shiftable_bf_host(const double* f_host, int64_t H, int64_t W,
                          const sbf_spatial* sp, int R, double fixed_T,
                          double sigma_r, double epsilon, int rule,
                          double log_2_over_eps, int precision,
                          double* out_host, sbf_plan* plan_out,
                          unsigned long long* fallback_out);

/* Divide/fallback epilogue on caller buffers (bilateral.py:242-254), fp64. */
int sbf_divide_with_fallback(const double* num, const double* den,
                             const double* fallback, int64_t n, double* out,
                             unsigned long long* count_dev, void* stream);

/* ---- PGM payload codecs (pgmio.py:81-137) ---- */
/* P5 payload bytes (8-bit or big-endian 16-bit) -> fp32 samples. */
int sbf_pgm_decode(const void* payload_dev, int bytes_per_sample, int64_t n, float* out_dev,
                   void* stream);
/* clamp to [0, maxval], floor(x + 0.5), 8-bit or big-endian 16-bit bytes. */
int sbf_pgm_encode(const void* img_dev, int dtype, int64_t n, int maxval, void* out_dev,
                   void* stream);

/* ---- brute-force bilateral filter (accuracy oracle at full size) ----
 * Replaces reference bilateral.py:205-239 `direct_bf(img, spatial,
 * gaussian_range(sigma_r), radius)`: out(x) = sum_y w(y) g(f(y)-f(x)) f(y) /
 * sum_y w(y) g(...) over the in-bounds (2R+1)^2 window, g Gaussian of width
 * sigma_r, w(dy,dx) = taps[dy+R] taps[dx+R] (taps == NULL: uniform, the Box
 * mode; spatial.py:197-213).  R <= 255.  precision SBF_PREC_FP32 (fp32
 * math, log2-domain weights) or SBF_PREC_HDR (fp64, the reference's
 * arithmetic).  Device buffers, stream-ordered. */
int sbf_direct_bf(const void* f, int dtype, int64_t H, int64_t W, int64_t ld, int R,
                  const double* taps_host, double sigma_r, int precision, void* out,
                  int out_dtype, void* stream);

/* Same, with the truncated raised-cosine expansion as the range kernel
 * (bilateral.py:101-103 expansion_range): K(s) = sum_k scale[k] cos(freq[k] s)
 * over K <= 1024 folded terms (host arrays), float64. */
int sbf_direct_bf_expansion(const void* f, int dtype, int64_t H, int64_t W, int64_t ld, int R,
                            const double* taps_host, const double* scale, const double* freq,
                            int K, void* out, int out_dtype, void* stream);

/* ---- coarse non-local means (reference nlm.py:78-137) ----
 * One item = one folded multi-index of the per-component expansions and one
 * cos/sin choice for components j >= 1 (bit j of `mask`); component 0
 * supplies the (cos, sin) pair.  weight = product of the folded component
 * weights; turns[j] = w_j / (2 pi).  48 bytes. */
typedef struct sbf_nlm_item {
  double weight;
  double turns[3];
  int32_t mask;
  int32_t pad;
} sbf_nlm_item;

/* Filters f with p (1..3) patch samples at `offsets` (host, 2p ints dy,dx;
 * the first must be 0,0; replicate padding) over the host item table;
 * stats = sbf_local_range statistics (centre) of f.  fp64 throughout;
 * allocates its planes stream-ordered.  out/fallback: device. */
int sbf_nlm_filter(const void* f, int dtype, int64_t H, int64_t W, int64_t ld,
                   const sbf_spatial* sp, int p, const int32_t* offsets,
                   const sbf_nlm_item* items, int n_items, const double* stats, void* out,
                   int out_dtype, unsigned long long* fallback, void* stream);

/* Brute-force coarse NLM (nlm.py:140-183 direct_nlm): window weights taps
 * (NULL: uniform), p patch offsets (first = origin, replicate padding) and per
 * component range kernel kinds[j] = 0 Gaussian(sigmas[j]) or 1 truncated
 * expansion (nterms[j] folded terms, consecutive in scale/freq); float64. */
int sbf_direct_nlm(const void* f, int dtype, int64_t H, int64_t W, int64_t ld, int R,
                   const double* taps_host, int p, const int32_t* offsets, const int32_t* kinds,
                   const double* sigmas, const int32_t* nterms, const double* scale,
                   const double* freq, void* out, int out_dtype, void* stream);

/* ---- standalone spatial smoothers (spatial.py:65-182) ----
 * box_filter (BOX, r), iterated_box_gaussian (ITERATED: passes, r, alpha),
 * fir_gaussian (FIR: sigma_s, r); float64 arithmetic, exact clamped
 * renormalisation.  out is H x W (ld = W).  Allocates stream-ordered. */
int sbf_smooth(const void* f, int dtype, int64_t H, int64_t W, int64_t ld, const sbf_spatial* sp,
               void* out, int out_dtype, void* stream);

/* ---- host -> device staging ----
 * Copies n samples of page-locked (pinned) host memory `host_src` into device
 * memory with the SMs reading over PCIe (faster than the copy engine for
 * image-sized transfers); integer kinds are widened to float32 on the way
 * (dev_dst float32), F32/F64 copy as is.  Stream-ordered; SBF_ERR_INVALID if
 * host_src is not pinned host memory. */
#define SBF_STAGE_F32 0
#define SBF_STAGE_F64 1
#define SBF_STAGE_U8 2
#define SBF_STAGE_U16 3
#define SBF_STAGE_I16 4
int sbf_stage_h2d(const void* host_src, int src_kind, int64_t n, void* dev_dst, void* stream);

/* ---- introspection / benchmarking hooks ---- */
/* fp64 (HDR / generic) evaluation, this thread: 0 = always the K term sweeps,
 * 1 = cost model (default: the dual form cos(gamma s)^N over the (2S+1)^2
 * window when M = 0 and it is cheaper), 2 = dual whenever M = 0. */
int sbf_set_fp64_method(int mode);
/* fp32 term sweeps, this thread: radii >= r (with an instantiation) run the
 * split column/row sweep instead of the fused strip kernels (default 6: the
 * K3 sweep serves r <= 5; 0 = never the split sweep; -1 = restore the
 * default). */
int sbf_set_split_min_radius(int r);
int sbf_num_specialisations(void);
int sbf_specialisation(int i, int* r, int* passes, int* mode);
int sbf_filter_geometry(int64_t rows_out, int64_t W, const sbf_spatial* sp, int precision,
                        int* out7);
int sbf_truncation_index_exact_bigint(int N, double epsilon, int* M);
int sbf_set_stage_mask(int mask);
/* This thread: record these cudaEvent_t (NULL: none) right before and after
 * every K3 launch -- kernel-level timing inside the fused pipeline. */
int sbf_set_k3_events(void* before, void* after);
/* K3 path, this thread: the divide/fallback epilogue streamed behind the term
 * kernel (programmatic dependent launch; each output segment is divided out
 * -- and, for a page-locked host output, written over PCIe -- as soon as
 * every term has landed on it): 1 (default) = when out is host memory,
 * 2 = always, 0 = never.  Returns the previous setting (-1: bad mode). */
int sbf_set_fused_epilogue(int mode);
/* K3 sweep (r <= 5), this thread: which kernel serves device outputs --
 * 0 (default) = the phase-separated sweep (two 128-thread CTAs per SM,
 * 128-column strips), 1 = the warp-specialised sweep (one 512-thread CTA per
 * SM, 252-column strips, V / H warpgroups over mbarriers) for images of at
 * least 2^20 pixels, 2 = the warp-specialised sweep for every device output.
 * Same results within fp32 rounding of the strip geometry; measured slower
 * on B200, kept as a tested alternative.  Page-locked host
 * outputs always take the phase-separated sweep with its fused epilogue.
 * Returns the previous setting. */
int sbf_set_sweep_variant(int mode);
int sbf_fp32_probe(int blocks, int threads, int iters, float* out_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SBF_H_ */
