// Probe: does cp.async.bulk.tensor accept a 2-D box whose start column is not 16-B aligned
// (element coordinate 250 of an fp32 row)?  Loads one 8 x 64 box at (c0, r0) and compares.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap map, float* out, int c0, int r0) {
  __shared__ __align__(128) float buf[8 * 64];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)),
                 "r"(8 * 64 * 4));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(buf)),
                 "l"(&map), "r"(c0), "r"(r0), "r"((unsigned)__cvta_generic_to_shared(&bar)));
  }
  asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n" ::"r"(
      (unsigned)__cvta_generic_to_shared(&bar)));
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int W = 1000, H = 64;
  std::vector<float> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = float(i);
  float *d, *o;
  cudaMalloc(&d, W * H * 4);
  cudaMalloc(&o, 8 * 64 * 4);
  cudaMemcpy(d, h.data(), W * H * 4, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
  cuuint64_t strides[1] = {(cuuint64_t)W * 4};
  cuuint32_t box[2] = {64, 8}, es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  for (int c0 : {248, 250, 251, 125}) {
    k<<<1, 128>>>(m, o, c0, 3);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> got(8 * 64);
    cudaMemcpy(got.data(), o, 8 * 64 * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < 8; ++y)
      for (int x = 0; x < 64; ++x)
        if (got[y * 64 + x] != h[(3 + y) * W + c0 + x]) ++bad;
    printf("c0=%d err=%s mismatches=%d first=%g expect=%g\n", c0, cudaGetErrorString(e), bad, got[0], h[3 * W + c0]);
  }
  return 0;
}
