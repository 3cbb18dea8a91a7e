// Memory-pattern micro-benchmarks (not part of the library): what HBM bandwidth does each
// load/store pattern of the 2-D Haar kernels reach on B200?  Built by tools/membench.py.
//   k_linear   : grid-stride float4 copy (torch copy_-like)
//   k_tile_ldg : 32 x 256 tiles, LDG.128 loads, stores of four 16 x 128 "bands" (the level-1
//                Mallat scatter) — registers only, no smem
//   k_tile_tma : same tiles via TMA 2-stage ring, then the same band stores from smem
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ float4 ldg4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void stg4(float* p, float4 v) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w) : "memory");
}
__device__ __forceinline__ void stg2(float* p, float2 v) {
  asm volatile("st.global.L1::no_allocate.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}

__global__ void k_linear(const float* __restrict__ x, float* __restrict__ y, int64_t n4) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x)
    stg4(y + 4 * i, ldg4(x + 4 * i));
}

// One 32 x 256 tile per CTA iteration (256 threads): thread t handles rows 2r, 2r+1 (r = t/64 + 4k)
// and cols 4*(t%64)..+3; writes the 2x2-block "bands" like level 1 (LL, HL, LH, HH quadrants).
__global__ void __launch_bounds__(256) k_tile_ldg(const float* __restrict__ x, float* __restrict__ y, int64_t H,
                                                  int64_t W, int64_t batch, int unroll) {
  const int64_t tiles_c = W / 256, tiles_r = H / 32, ntiles = batch * tiles_r * tiles_c;
  const int t = threadIdx.x;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t rt = tile / tiles_c, ct = tile - rt * tiles_c;
    const int64_t b = rt / tiles_r, row0 = (rt - b * tiles_r) * 32, col0 = ct * 256;
    const float* src = x + (b * H + row0) * W + col0;
    float4 a[4], c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = (t >> 6) + 4 * k;
      a[k] = ldg4(src + int64_t(2 * r) * W + 4 * (t & 63));
      c[k] = ldg4(src + int64_t(2 * r + 1) * W + 4 * (t & 63));
    }
    float* ob = y + (b * H + (row0 >> 1)) * W + (col0 >> 1);
    const int64_t hw = (H >> 1) * W, wh = W >> 1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = (t >> 6) + 4 * k;
      float* pr = ob + int64_t(r) * W + 2 * (t & 63);
      stg2(pr, make_float2(a[k].x + c[k].x, a[k].z + c[k].z));
      stg2(pr + wh, make_float2(a[k].y + c[k].y, a[k].w + c[k].w));
      stg2(pr + hw, make_float2(a[k].x - c[k].x, a[k].z - c[k].z));
      stg2(pr + hw + wh, make_float2(a[k].y - c[k].y, a[k].w - c[k].w));
    }
  }
}

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(256) k_tile_tma(const __grid_constant__ CUtensorMap map, float* __restrict__ y,
                                                  int64_t H, int64_t W, int64_t batch, int stages, int bw, int bh,
                                                  const float* __restrict__ xsrc, int bulk, int issuers,
                                                  unsigned* ctr) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + stages * 32768);
  const int64_t tiles_c = W / 256, tiles_r = H / 32, ntiles = batch * tiles_r * tiles_c;
  const int t = threadIdx.x;
  if (t == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bars[s])), "r"(issuers));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // issuers > 1: lane 0 of warps 0..issuers-1 each arrive (expect_tx of its share) and issue
  // rows [k * 32 / issuers, (k + 1) * 32 / issuers) of the one-row boxes (bh == 1 only)
  auto issue = [&](int64_t tile, int s) {
    const int64_t rt = tile / tiles_c, ct = tile - rt * tiles_c;
    const int k = t >> 5, per = 32 / issuers;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[s])), "r"(32768 / issuers)
                 : "memory");
    if (issuers > 1) {
      for (int r = k * per; r < (k + 1) * per; ++r)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                su32(smem + s * 32768 + r * 1024)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(int(ct * 256)), "r"(int(rt * 32 + r)), "r"(su32(&bars[s]))
            : "memory");
      return;
    }
    if (bulk) {  // 32 one-row bulk copies of 1 KB (cp.async.bulk, no tensor map)
      const int64_t b = rt / tiles_r, row0 = (rt - b * tiles_r) * 32;
      for (int r = 0; r < 32; ++r)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1024, [%2];" ::"r"(
                         su32(smem + s * 32768 + r * 1024)),
                     "l"(xsrc + (b * H + row0 + r) * W + ct * 256), "r"(su32(&bars[s]))
                     : "memory");
      return;
    }
    for (int by = 0; by < 32; by += bh)
      for (int bx = 0; bx < 256; bx += bw)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                su32(smem + s * 32768 + (by * 256 + bx * bh) * 4)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(int(ct * 256 + bx)), "r"(int(rt * 32 + by)), "r"(su32(&bars[s]))
            : "memory");
  };
  const bool issuer = (t & 31) == 0 && (t >> 5) < issuers;
  // ctr != nullptr: global tile order (the counter hands out tiles; the tile index of stage s sits in
  // stile[s]; an index >= ntiles ends the loop)
  unsigned* stile = reinterpret_cast<unsigned*>(bars + stages);
  if (ctr) {
    if (t == 0)
      for (int s = 0; s < stages; ++s) {
        const unsigned tt = blockIdx.x + unsigned(s) * gridDim.x;
        stile[s] = tt;
        if (tt < ntiles) issue(tt, s);
        else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bars[s])) : "memory");
      }
  } else if (issuer)
    for (int s = 0; s < stages; ++s)
      if (blockIdx.x + int64_t(s) * gridDim.x < ntiles) issue(blockIdx.x + int64_t(s) * gridDim.x, s);
  int it = 0;
  for (int64_t tile = blockIdx.x; ctr || tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it % stages;
    const uint32_t par = (it / stages) & 1;
    asm volatile(
        "{\n.reg .pred P1;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D1;\nbra W1;\nD1:\n}\n" ::"r"(
            su32(&bars[s])),
        "r"(par)
        : "memory");
    if (ctr) {
      tile = stile[s];
      if (tile >= ntiles) break;
    }
    const int64_t rt = tile / tiles_c, ct = tile - rt * tiles_c;
    const int64_t b = rt / tiles_r, row0 = (rt - b * tiles_r) * 32, col0 = ct * 256;
    const float* st = reinterpret_cast<const float*>(smem + s * 32768);
    float* ob = y + (b * H + (row0 >> 1)) * W + (col0 >> 1);
    const int64_t hw = (H >> 1) * W, wh = W >> 1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = (t >> 6) + 4 * k;
      const float4 a = *reinterpret_cast<const float4*>(st + (2 * r) * 256 + 4 * (t & 63));
      const float4 c = *reinterpret_cast<const float4*>(st + (2 * r + 1) * 256 + 4 * (t & 63));
      float* pr = ob + int64_t(r) * W + 2 * (t & 63);
      stg2(pr, make_float2(a.x + c.x, a.z + c.z));
      stg2(pr + wh, make_float2(a.y + c.y, a.w + c.w));
      stg2(pr + hw, make_float2(a.x - c.x, a.z - c.z));
      stg2(pr + hw + wh, make_float2(a.y - c.y, a.w - c.w));
    }
    __syncthreads();
    if (ctr) {
      if (t == 0) {
        const unsigned nt = atomicAdd(ctr, 1u) + unsigned(stages) * gridDim.x;
        stile[s] = nt;
        if (nt < ntiles) issue(nt, s);
        else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bars[s])) : "memory");
      }
    } else if (issuer && tile + int64_t(stages) * gridDim.x < ntiles) {
      issue(tile + int64_t(stages) * gridDim.x, s);
    }
  }
}

}  // namespace

extern "C" {

float mb_linear(const float* x, float* y, int64_t n, int blocks, int threads, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) k_linear<<<blocks, threads>>>(x, y, n / 4);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) k_linear<<<blocks, threads>>>(x, y, n / 4);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

float mb_tile_ldg(const float* x, float* y, int64_t H, int64_t W, int64_t batch, int blocks, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) k_tile_ldg<<<blocks, 256>>>(x, y, H, W, batch, 4);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) k_tile_ldg<<<blocks, 256>>>(x, y, H, W, batch, 4);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return cudaGetLastError() == cudaSuccess ? ms / reps : -1.f;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

float mb_tile_tma(const float* x, float* y, int64_t H, int64_t W, int64_t batch, int blocks, int stages, int reps,
                  int bw, int bh, int bulk, int issuers, int order) {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {cuuint64_t(W), cuuint64_t(batch * H)};
  cuuint64_t str[1] = {cuuint64_t(W) * 4};
  cuuint32_t box[2] = {cuuint32_t(bw), cuuint32_t(bh)}, es[2] = {1, 1};
  if (reinterpret_cast<EncodeFn>(fp)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(x), dims, str, box,
                                     es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -2.f;
  const int smem = stages * 32768 + 128;
  unsigned* ctr = nullptr;
  if (order) cudaMalloc(&ctr, 16);
  cudaFuncSetAttribute(k_tile_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) {
    if (ctr) cudaMemsetAsync(ctr, 0, 16);
    k_tile_tma<<<blocks, 256, smem>>>(map, y, H, W, batch, stages, bw, bh, x, bulk, issuers, ctr);
  }
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) {
    if (ctr) cudaMemsetAsync(ctr, 0, 16);
    k_tile_tma<<<blocks, 256, smem>>>(map, y, H, W, batch, stages, bw, bh, x, bulk, issuers, ctr);
  }
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  if (ctr) cudaFree(ctr);
  return cudaGetLastError() == cudaSuccess ? ms / reps : -1.f;
}
}
