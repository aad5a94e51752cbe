// Standalone check of the K3 sweep's TMA + mbarrier helpers (debug tool).
// usage: tma_test <mode>; one mode per process (a fault kills the context)
//  0: grid-constant map, box 128x26 at (-18,-5)   1: map in global memory
//  2: box 32x26                                   3: coords (0,0)
//  4: cp.async.bulk (1-D, no tensor map)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cudaTypedefs.h>
#include "../../paper_1203_5128_b200/csrc/sbf_sweep.cuh"

namespace sbf {
void set_error(const char*, ...) {}
int device_sm_count() { return 148; }
cudaError_t ensure_dyn_smem(const void*, size_t) { return cudaSuccess; }
}
using namespace sbf;

__global__ void k(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, int x0, int y0,
                  float* out, int bytes, int mode, const float* src) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* sbase = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sbase);
  float* box = reinterpret_cast<float*>(sbase + 128);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar, bytes);
    if (mode == 4) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(smem_u32(box)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
    } else {
      tma_load_2d(box, mode == 1 ? gmap : &map, x0, y0, bar);
    }
  }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = box[i];
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int W = 300, H = 200;
  std::vector<float> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = (float)i;
  float *d, *o;
  CUtensorMap* gm;
  cudaMalloc(&d, W * H * 4);
  cudaMalloc(&o, 26 * 128 * 4);
  cudaMalloc(&gm, sizeof(CUtensorMap));
  cudaMemcpy(d, h.data(), W * H * 4, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  const int bw = mode == 2 ? 32 : 128, bh = 26;
  const int mode4 = mode == 4;
  int x0 = mode == 3 ? 0 : -18, y0 = mode == 3 ? 0 : -5;
  if (mode >= 5) {  // 5: (-16,0) 6: (5,0) 7: (0,-5) 8: (-18,0) 9: (4,3) 10: (290,195)
    const int xs[] = {-16, 5, 0, -18, 4, 290}, ys[] = {0, 0, -5, 0, 3, 195};
    x0 = xs[mode - 5];
    y0 = ys[mode - 5];
  }
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
  cuuint64_t strides[1] = {(cuuint64_t)W * 4};
  cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
  cuuint32_t es[2] = {1u, 1u};
  CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaMemcpy(gm, &map, sizeof(map), cudaMemcpyHostToDevice);
  printf("mode %d encode %d align %lu\n", mode, (int)cr, (unsigned long)((uintptr_t)&map % 64));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int bytes = mode == 4 ? 4096 : bw * bh * 4;
  k<<<1, 128, 64 * 1024>>>(map, gm, x0, y0, o, bytes, mode, d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("mode %d: %s\n", mode, cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<float> r(bytes / 4);
  cudaMemcpy(r.data(), o, bytes, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int j = 0; j < (mode == 4 ? 1 : bh); ++j)
    for (int i = 0; i < (mode == 4 ? 1024 : bw); ++i) {
      const int x = x0 + i, y = y0 + j;
      float want = (x >= 0 && x < W && y >= 0 && y < H) ? (float)(y * W + x) : 0.f;
      if (mode == 4) want = (float)i;
      bad += r[j * (mode == 4 ? 1024 : bw) + i] != want;
    }
  printf("  mismatches %d\n", bad);
  return 0;
}
