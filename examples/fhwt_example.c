/*
 * fhwt_example.c — the C ABI (include/fhwt.h) used from plain C, no Python and no torch.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/fhwt_example.c \
 *       -L paper_1002_2184_b200 -lfhwt -L /usr/local/cuda/lib64 -lcudart -lm \
 *       -Wl,-rpath,$PWD/paper_1002_2184_b200 -o fhwt_example && ./fhwt_example
 *
 * 1. A batch of images through a plan on device buffers (fhwt_plan_2d / fhwt_plan_analyze /
 *    fhwt_plan_synthesize): perfect reconstruction within 1e-5 * max|d| (north_star bound), and
 *    LL_L(0, 0) equal to its closed form 2^L * mean of the top-left 2^L x 2^L block (SURVEY §8(c)
 *    C4; computed here in double, independently of the library).
 * 2. The same batch through the host-buffer round trip (fhwt_roundtrip_2d_host): coefficients
 *    and d_R bitwise equal to the device-buffer path.
 * 3. An invalid shape returns FHWT_ERR_INSUFFICIENT_LENGTH with a message, and nothing launches.
 * Prints one line per check and exits non-zero on the first failure.
 */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "fhwt.h"

#define CHECK(cond, ...)                   \
  do {                                     \
    if (!(cond)) {                         \
      fprintf(stderr, "FAIL: " __VA_ARGS__); \
      fprintf(stderr, "\n");               \
      return 1;                            \
    }                                      \
  } while (0)

#define FHWT(call)                                                                              \
  do {                                                                                          \
    fhwt_status st_ = (call);                                                                   \
    CHECK(st_ == FHWT_OK, "%s -> %s (%s)", #call, fhwt_status_string(st_), fhwt_last_error_message()); \
  } while (0)

#define CUDA(call)                                                                \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    CHECK(e_ == cudaSuccess, "%s -> %s", #call, cudaGetErrorString(e_));          \
  } while (0)

static uint32_t lcg(uint32_t* s) { return *s = *s * 1664525u + 1013904223u; }

int main(void) {
  const int64_t B = 3, H = 256, W = 384;
  const int L = 5;
  const size_t n = (size_t)(B * H * W), bytes = n * sizeof(float);
  float* d = (float*)malloc(bytes);
  float* c_dev = (float*)malloc(bytes);
  float* r_dev = (float*)malloc(bytes);
  float* c_host = (float*)malloc(bytes);
  float* r_host = (float*)malloc(bytes);
  CHECK(d && c_dev && r_dev && c_host && r_host, "host allocation");
  uint32_t seed = 12345u;
  float maxd = 0.f;
  for (size_t i = 0; i < n; ++i) {
    d[i] = (float)(lcg(&seed) >> 8) / 16777216.0f * 2.0f - 1.0f;   /* uniform [-1, 1) */
    if (fabsf(d[i]) > maxd) maxd = fabsf(d[i]);
  }

  /* 1. plan on device buffers */
  float *dd, *dc, *dr;
  void* ws = NULL;
  CUDA(cudaMalloc((void**)&dd, bytes));
  CUDA(cudaMalloc((void**)&dc, bytes));
  CUDA(cudaMalloc((void**)&dr, bytes));
  CUDA(cudaMemcpy(dd, d, bytes, cudaMemcpyHostToDevice));
  fhwt_plan plan;
  FHWT(fhwt_plan_2d(&plan, H, W, B, L, NULL, 0));
  const size_t wsb = fhwt_plan_workspace_bytes(plan);
  if (wsb) CUDA(cudaMalloc(&ws, wsb));
  FHWT(fhwt_plan_analyze(plan, dd, dc, ws, NULL));
  FHWT(fhwt_plan_synthesize(plan, dc, dr, ws, NULL));
  CUDA(cudaDeviceSynchronize());
  CUDA(cudaMemcpy(c_dev, dc, bytes, cudaMemcpyDeviceToHost));
  CUDA(cudaMemcpy(r_dev, dr, bytes, cudaMemcpyDeviceToHost));
  double rt = 0.0;
  for (size_t i = 0; i < n; ++i) rt = fmax(rt, fabs((double)r_dev[i] - (double)d[i]));
  CHECK(rt <= 1e-5 * maxd, "round trip error %.3e > 1e-5 * max|d|", rt);
  printf("plan round trip: max |d_R - d| = %.3e (bound %.3e)\n", rt, 1e-5 * maxd);
  for (int64_t b = 0; b < B; ++b) {   /* LL_L(0,0) = 2^L * mean of the 2^L x 2^L block */
    double sum = 0.0;
    const int blk = 1 << L;
    for (int y = 0; y < blk; ++y)
      for (int x = 0; x < blk; ++x) sum += d[(size_t)(b * H + y) * W + x];
    const double ll = sum / (double)(1 << L);   /* 2^L * sum / 4^L */
    const double got = c_dev[(size_t)b * H * W];
    CHECK(fabs(got - ll) <= 1e-5 * maxd, "image %lld LL_%d(0,0) = %.9g, closed form %.9g", (long long)b, L, got, ll);
  }
  printf("LL_%d(0,0) matches 2^L * block mean for %lld images\n", L, (long long)B);

  /* 2. host-buffer round trip: bitwise equal to the device path */
  FHWT(fhwt_roundtrip_2d_host(d, c_host, r_host, H, W, B, L, 0));
  CHECK(memcmp(c_host, c_dev, bytes) == 0, "host round trip coefficients differ from the plan path");
  CHECK(memcmp(r_host, r_dev, bytes) == 0, "host round trip d_R differs from the plan path");
  printf("fhwt_roundtrip_2d_host: coefficients and d_R bitwise equal to the plan path\n");

  /* 3. validation before any launch */
  const uint64_t launches = fhwt_launch_count();
  fhwt_plan bad;
  const fhwt_status st = fhwt_plan_2d(&bad, 100, 64, 1, 3, NULL, -1);
  CHECK(st == FHWT_ERR_INSUFFICIENT_LENGTH, "100 x 64 at L=3 gave %s", fhwt_status_string(st));
  CHECK(fhwt_launch_count() == launches, "a rejected plan launched kernels");
  printf("100 x 64, L=3 rejected: %s (%s)\n", fhwt_status_string(st), fhwt_last_error_message());

  FHWT(fhwt_plan_destroy(plan));
  cudaFree(dd);
  cudaFree(dc);
  cudaFree(dr);
  if (ws) cudaFree(ws);
  free(d), free(c_dev), free(r_dev), free(c_host), free(r_host);
  printf("OK\n");
  return 0;
}
