// PGM payload codecs on the device (reference pgmio.py:81-137).
//
// P5 pixel payloads go to the GPU as raw bytes and are decoded in place
// (8-bit or big-endian 16-bit samples -> fp32, exact for maxval <= 65535);
// results are quantised on the device exactly like the reference save_pgm:
// clamp to [0, maxval], floor(x + 0.5) (round half away from zero for
// non-negative values), then 8-bit or big-endian 16-bit.  Header parsing
// (a few dozen bytes) and the ASCII P2 form stay on the host.
#include "sbf_common.cuh"

namespace sbf {
namespace {

__global__ void pgm_decode_kernel(const unsigned char* __restrict__ in, int bytes_per,
                                  int64_t n, float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = bytes_per == 1 ? (float)in[i]
                            : (float)(((unsigned)in[2 * i] << 8) | (unsigned)in[2 * i + 1]);
  }
}

template <typename T>
__global__ void pgm_encode_kernel(const T* __restrict__ img, int64_t n, int maxval,
                                  unsigned char* __restrict__ out) {
  const double mv = (double)maxval;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = (double)img[i];
    v = v < 0.0 ? 0.0 : (v > mv ? mv : v);
    const unsigned q = (unsigned)floor(v + 0.5);
    if (maxval < 256) {
      out[i] = (unsigned char)q;
    } else {
      out[2 * i] = (unsigned char)(q >> 8);
      out[2 * i + 1] = (unsigned char)(q & 0xff);
    }
  }
}

}  // namespace
}  // namespace sbf

using namespace sbf;

extern "C" {

int sbf_pgm_decode(const void* payload_dev, int bytes_per_sample, int64_t n, float* out_dev,
                   void* stream) {
  SBF_REQUIRE(payload_dev && out_dev && n >= 0, SBF_ERR_INVALID, "null pointer");
  SBF_REQUIRE(bytes_per_sample == 1 || bytes_per_sample == 2, SBF_ERR_INVALID,
              "bytes per sample must be 1 or 2");
  if (n == 0) return SBF_OK;
  const unsigned grid = (unsigned)smin<int64_t>((n + 255) / 256, 148 * 8);
  pgm_decode_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const unsigned char*>(payload_dev), bytes_per_sample, n, out_dev);
  SBF_CHECK_LAUNCH();
  return SBF_OK;
}

int sbf_pgm_encode(const void* img_dev, int dtype, int64_t n, int maxval, void* out_dev,
                   void* stream) {
  SBF_REQUIRE(img_dev && out_dev && n >= 0, SBF_ERR_INVALID, "null pointer");
  SBF_REQUIRE(maxval >= 1 && maxval <= 65535, SBF_ERR_INVALID, "maxval must lie in [1, 65535]");
  if (n == 0) return SBF_OK;
  const unsigned grid = (unsigned)smin<int64_t>((n + 255) / 256, 148 * 8);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == SBF_F64)
    pgm_encode_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(img_dev), n, maxval,
                                                     static_cast<unsigned char*>(out_dev));
  else
    pgm_encode_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(img_dev), n, maxval,
                                                    static_cast<unsigned char*>(out_dev));
  SBF_CHECK_LAUNCH();
  return SBF_OK;
}

}  // extern "C"
