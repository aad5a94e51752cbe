// FP32 issue probe: lane-ops/s of dependent FFMA / FFMA2 chains, NC independent
// chains per thread, W warps per SM.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
template <int NC>
__global__ void k_ffma(float* out, float a, float b, int iters) {
  float x[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < NC; ++c) x[c] = fmaf(x[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c) s += x[c];
  if (s == 1234.5f) out[0] = s;
}
template <int NC>
__global__ void k_ffma2(float* out, float a, float b, int iters) {
  float2 x[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) x[c] = make_float2(threadIdx.x * 1e-3f + c, c);
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < NC; ++c) x[c] = __ffma2_rn(x[c], a2, b2);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c) s += x[c].x + x[c].y;
  if (s == 1234.5f) out[0] = s;
}
// register-operand form: b varies per thread (no uniform / immediate operand)
template <int NC>
__global__ void k_ffma_reg(float* out, float a, float b, int iters) {
  float x[NC];
  const float ar = a + threadIdx.x * 1e-9f, br = b + threadIdx.x * 1e-9f;
#pragma unroll
  for (int c = 0; c < NC; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < NC; ++c) x[c] = fmaf(x[c], ar, br);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c) s += x[c];
  if (s == 1234.5f) out[0] = s;
}
template <int NC>
__global__ void k_dfma(float* out, float a, float b, int iters) {
  double x[NC];
  const double ad = a, bd = b;
#pragma unroll
  for (int c = 0; c < NC; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < NC; ++c) x[c] = fma(x[c], ad, bd);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < NC; ++c) s += x[c];
  if (s == 1234.5) out[0] = (float)s;
}
template <typename K>
void run(const char* name, K k, int nc, int lanes_per_op, int warps_per_sm) {
  float* o;
  cudaMalloc(&o, 4);
  const int threads = 32 * warps_per_sm, blocks = 148;
  const int iters = 4096;
  k<<<blocks, threads>>>(o, 0.999f, 0.001f, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(o, 0.999f, 0.001f, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)blocks * threads * iters * 8 * nc * lanes_per_op;
  printf("%-10s chains %d warps/SM %2d : %6.2f T lane-ops/s\n", name, nc, warps_per_sm, ops / (ms * 1e-3) / 1e12);
  cudaFree(o);
}
int main() {
  for (int w : {16, 32}) {
    run("dfma", k_dfma<4>, 4, 1, w);
    run("dfma", k_dfma<8>, 8, 1, w);
  }
  for (int w : {4, 8, 16}) {
    run("ffma", k_ffma<1>, 1, 1, w);
    run("ffma", k_ffma<2>, 2, 1, w);
    run("ffma", k_ffma<4>, 4, 1, w);
    run("ffma", k_ffma<8>, 8, 1, w);
    run("ffma_reg", k_ffma_reg<4>, 4, 1, w);
    run("ffma_reg", k_ffma_reg<8>, 8, 1, w);
    run("ffma2", k_ffma2<1>, 1, 2, w);
    run("ffma2", k_ffma2<2>, 2, 2, w);
    run("ffma2", k_ffma2<4>, 4, 2, w);
    run("ffma2", k_ffma2<8>, 8, 2, w);
  }
  return 0;
}
