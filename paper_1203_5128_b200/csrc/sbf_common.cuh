// Shared helpers for the sbf CUDA library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/sbf.h"

namespace sbf {

void set_error(const char* fmt, ...);

#define SBF_CHECK_CUDA(expr)                                                  \
  do {                                                                        \
    cudaError_t e__ = (expr);                                                 \
    if (e__ != cudaSuccess) {                                                 \
      ::sbf::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e__), \
                       __FILE__, __LINE__);                                   \
      return SBF_ERR_CUDA;                                                    \
    }                                                                         \
  } while (0)

#define SBF_CHECK_LAUNCH()                                                    \
  do {                                                                        \
    cudaError_t e__ = cudaGetLastError();                                     \
    if (e__ != cudaSuccess) {                                                 \
      ::sbf::set_error("kernel launch failed: %s (%s:%d)",                    \
                       cudaGetErrorString(e__), __FILE__, __LINE__);          \
      return SBF_ERR_CUDA;                                                    \
    }                                                                         \
  } while (0)

#define SBF_REQUIRE(cond, code, ...)   \
  do {                                 \
    if (!(cond)) {                     \
      ::sbf::set_error(__VA_ARGS__);   \
      return (code);                   \
    }                                  \
  } while (0)

template <class T>
__host__ __device__ __forceinline__ T smin(T a, T b) { return a < b ? a : b; }
template <class T>
__host__ __device__ __forceinline__ T smax(T a, T b) { return a > b ? a : b; }

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Order-preserving uint64 image of a double (for atomicMax/atomicMin).
__device__ __forceinline__ unsigned long long ord_bits(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_value(unsigned long long b) {
  b = (b & 0x8000000000000000ull) ? (b & 0x7fffffffffffffffull) : ~b;
  return __longlong_as_double((long long)b);
}

// Layout of the 8-double stats block written by K1 (stats_dev):
//   [0] T   [1] min f   [2] max f   [3] centre
//   [4..6] reduction scratch (ordered-uint64 images of T, min, max)
//   [7]    number of non-finite samples (uint64 bit pattern)
constexpr int kStatsDoubles = 8;

// ---- per-launch geometry of the term kernel (host side) ----
struct TermGeom {
  int halo;      // PASSES * (r + 1)
  int halo_w;    // haloed columns per CTA
  int wc;        // output columns per CTA
  int threads;
  int rows;      // rows per chunk
  int band;      // output rows per CTA band
  int nstrips, nbands, groups;
  size_t smem;
};

// K2 fused into K1's last CTA (whole-pipeline entry): the plan arguments
struct PlanArgs {
  int on;
  int rule;
  int cap;
  double sigma_r, eps, log_2_over_eps;
  sbf_plan* plan;
  sbf_term* terms;
  void* zero;         // K3 accumulator + control block cleared by K1 (no memset launch)
  size_t zero_bytes;  // multiple of 16
  unsigned long long* fb_reset;  // fallback counter reset by K1 (nullable)
};

// Programmatic dependent launch along the pipeline (K1 row pass -> column
// pass -> K3 -> K4): a kernel launched with launch_pdl may be scheduled while
// its predecessor still runs; it calls pdl_wait() before touching anything the
// predecessor reads or writes, which returns once the predecessor grid has
// completed and flushed (a no-op for an ordinary launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#ifndef SBF_PDL_EARLY
#define SBF_PDL_EARLY 1  // 0: dependents are scheduled only when the whole primary grid exits
#endif
__device__ __forceinline__ void pdl_trigger() {
#if SBF_PDL_EARLY
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Cached device queries for the launch paths (sbf_api.cu): the SM count, and
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when it must grow.
int device_sm_count();
cudaError_t ensure_dyn_smem(const void* func, size_t bytes);

// Forward declarations of internal launchers (implemented in separate TUs).
int launch_local_range(const void* f, int dtype, int64_t H, int64_t W, int64_t ld, int R,
                       int64_t t_lo, int64_t t_hi, void* M_out, double* stats, void* ws,
                       size_t ws_bytes, cudaStream_t st, const PlanArgs* plan = nullptr);
size_t local_range_ws(int64_t H, int64_t W, int dtype);

int launch_plan(const double* T_dev, int use_fixed, double fixed_T, double sigma_r, double eps,
                int rule, double log_2_over_eps, sbf_plan* plan_dev, sbf_term* terms_dev,
                int terms_cap, cudaStream_t st, int forced_N = 0, int forced_M = 0);

// Stream-ordered device scratch that is released on every exit path
// (cudaFreeAsync on the owning stream when it goes out of scope).
// The device's default memory pool keeps freed blocks (release threshold
// raised once per device): with the default threshold of 0 every
// synchronisation handed the scratch back to the driver and the next call
// re-mapped it (milliseconds of variance on the fp64 / dual paths).
void retain_default_pool();

template <typename T>
struct DevBuf {
  T* p = nullptr;
  cudaStream_t st;
  explicit DevBuf(cudaStream_t s) : st(s) {}
  cudaError_t alloc(size_t n) {
    retain_default_pool();
    return cudaMallocAsync(reinterpret_cast<void**>(&p), n * sizeof(T), st);
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

struct FilterLaunch {
  const void* f;
  int dtype;
  int64_t H, W, ld, row0, img_H, out_lo, out_hi;
  sbf_spatial sp;
  const sbf_plan* plan;
  const sbf_term* terms;
  const double* stats;
  int precision;
  void* out;
  int out_dtype;
  unsigned long long* fallback;
  void* ws;
  size_t ws_bytes;
  cudaStream_t stream;
  int nd_zeroed = 0;  // the K3 accumulator in ws is already zero (cleared by K1)
};

int launch_filter(const FilterLaunch& a);
// bytes of ws the K3 path clears before its launch (0: another path runs)
size_t k3_zero_bytes(const FilterLaunch& a);
size_t filter_ws(int64_t H, int64_t W, int64_t rows_out, int dtype, const sbf_spatial* sp,
                 int precision);

}  // namespace sbf
