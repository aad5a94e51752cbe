/* Standalone C caller of the drop-in ABI (include/sbf.h) — what a non-Python
 * integration of the reference's shiftable_bf (bilateral.py:117-137) looks
 * like.  Reads a raw little-endian float64 image, filters it with
 * sbf_shiftable_bf_host (host buffers in and out, default AUTO precision),
 * writes the float64 result and prints the plan.
 *
 *   sbf_example in.f8 out.f8 H W sigma_s sigma_r epsilon
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "sbf.h"

int main(int argc, char** argv) {
  if (argc != 8) {
    fprintf(stderr, "usage: %s in.f8 out.f8 H W sigma_s sigma_r epsilon\n", argv[0]);
    return 2;
  }
  const long H = atol(argv[3]), W = atol(argv[4]);
  const double sigma_s = atof(argv[5]), sigma_r = atof(argv[6]), eps = atof(argv[7]);
  double* img = (double*)malloc(sizeof(double) * H * W);
  double* out = (double*)malloc(sizeof(double) * H * W);
  FILE* fi = fopen(argv[1], "rb");
  if (!fi || fread(img, sizeof(double), (size_t)(H * W), fi) != (size_t)(H * W)) {
    fprintf(stderr, "cannot read %s\n", argv[1]);
    return 3;
  }
  fclose(fi);

  sbf_spatial sp;
  int r = 0, R = 0;
  double alpha = 0.0;
  if (sbf_extended_box_params(sigma_s, 3, &r, &alpha) != SBF_OK) goto fail;
  sp.mode = SBF_SPATIAL_ITERATED;
  sp.passes = 3;
  sp.r = r;
  sp.pad = 0;
  sp.alpha = alpha;
  sp.sigma_s = sigma_s;
  if (sbf_support_radius(&sp, &R) != SBF_OK) goto fail;
  if (R < 1) R = 1; /* bilateral.py:79 resolved_radius */

  sbf_plan plan;
  unsigned long long fallback = 0;
  if (sbf_shiftable_bf_host(img, H, W, &sp, R, -1.0, sigma_r, eps, SBF_RULE_AUTO,
                            eps > 0.0 ? log(2.0 / eps) : 0.0, SBF_PREC_AUTO, out, &plan,
                            &fallback) != SBF_OK)
    goto fail;
  printf("T=%.17g N=%d M=%d K=%d fallback=%llu\n", plan.T, plan.N, plan.M, plan.K, fallback);
  FILE* fo = fopen(argv[2], "wb");
  if (!fo || fwrite(out, sizeof(double), (size_t)(H * W), fo) != (size_t)(H * W)) return 3;
  fclose(fo);
  free(img);
  free(out);
  return 0;
fail:
  fprintf(stderr, "sbf error: %s\n", sbf_last_error());
  return 4;
}
