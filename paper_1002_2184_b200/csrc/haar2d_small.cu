// Batched small images (h * w <= 4096 samples, w < 128): whole-image Fast Haar analysis /
// synthesis for sm_100a.
//
// Same method and arithmetic as haar2d.cu (PAPER.md:118-124 Fig. 4, :162-176 Fig. 7, applied rows
// then columns, reading R8; folded 2 x 2 butterflies with an exact x1/2; levels >= 4 of the
// analysis in fp64, R13), organised for images too narrow for 128/256-column tiles:
// a chunk of G consecutive images is contiguous in HBM, so it moves with ONE 1-D bulk copy
// (cp.async.bulk, mbarrier complete_tx) into shared memory, all levels run there, and the chunk's
// coefficients (Mallat layout per image) leave with ONE 1-D bulk store (cp.async.bulk.global).
// Persistent CTAs, a ring of input stages, double use of the output buffer guarded by
// cp.async.bulk.wait_group.read.  Each output is produced by the same operations on the same
// operands as the tile kernels, so results are bitwise identical.
#include "fhwt_internal.cuh"

namespace fhwt {
namespace {

__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem_src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

struct Chunk {
  int64_t first;   // first image of the chunk
  int g;           // images in the chunk (the last one may be short)
};
__device__ __forceinline__ Chunk chunk_of(const Small2dParams& p, int64_t c) {
  Chunk k;
  k.first = c * p.G;
  k.g = int(p.batch - k.first < p.G ? p.batch - k.first : p.G);
  return k;
}

__device__ __forceinline__ void issue_chunk(const Small2dParams& p, const float* src, unsigned char* dst, uint64_t* bar,
                                           int64_t c) {
  const Chunk k = chunk_of(p, c);
  const uint32_t bytes = uint32_t(k.g) * uint32_t(p.H * p.W) * 4u;
  mbar_arrive_expect_tx(bar, bytes);
  bulk_load(dst, src + k.first * int64_t(p.H) * p.W, bytes, bar);
}

// One analysis level j of g images: source LL_{j-1} (per image h x w, pitch sp, image stride ss),
// bands to the output chunk O (Mallat layout, pitch W), LL_j to dst (compact per image) or, at the
// last level, to O.
template <typename TS, typename TD>
__device__ __forceinline__ void small_ana_level(const Small2dParams& p, const TS* src, int sp, int ss, float* O,
                                                TD* dst, int g, int h, int w, bool last) {
  const int h2 = h >> 1, w2 = w >> 1;
  const uint32_t per = uint32_t(h2 * w2), total = per * uint32_t(g);
  const int imgO = p.H * p.W;
  for (uint32_t u = threadIdx.x; u < total; u += blockDim.x) {
    const uint32_t gi = u / per, rem = u - gi * per, r = rem / uint32_t(w2), c = rem - r * uint32_t(w2);
    const TS* s = src + gi * ss + (2 * r) * sp + 2 * c;
    const TD a = TD(s[0]), bb = TD(s[1]), cc = TD(s[sp]), d = TD(s[sp + 1]);
    const TD s1 = a + bb, s2 = cc + d, d1 = a - bb, d2 = cc - d;
    float* o = O + gi * imgO + r * p.W + c;
    o[w2] = float((d1 + d2) * TD(0.5));
    o[h2 * p.W] = float((s1 - s2) * TD(0.5));
    o[h2 * p.W + w2] = float((d1 - d2) * TD(0.5));
    const TD ll = (s1 + s2) * TD(0.5);
    if (last)
      o[0] = float(ll);
    else
      dst[gi * per + rem] = ll;
  }
}

__global__ void __launch_bounds__(256, 2) ana2d_small_kernel(const __grid_constant__ Small2dParams p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  float* O = reinterpret_cast<float*>(smem + p.off_out);
  float* const T0 = reinterpret_cast<float*>(smem + p.off_t[0]);
  float* const T1 = reinterpret_cast<float*>(smem + p.off_t[1]);
  double* const D0 = reinterpret_cast<double*>(smem + p.off_d[0]);
  double* const D1 = reinterpret_cast<double*>(smem + p.off_d[1]);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < p.stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < p.stages; ++s) {
      const int64_t c = blockIdx.x + int64_t(s) * gridDim.x;
      if (c < p.nchunks) issue_chunk(p, p.in, smem + s * p.stage_bytes, &bars[s], c);
    }
  int it = 0;
  for (int64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x, ++it) {
    const int s = it % p.stages;
    mbar_wait(&bars[s], uint32_t(it / p.stages) & 1u);
    if (tid == 0) bulk_wait_read();   // the previous chunk's store has read O
    __syncthreads();
    const Chunk k = chunk_of(p, c);
    const float* S = reinterpret_cast<const float*>(smem + s * p.stage_bytes);
    int h = p.H, w = p.W;
    // level 1 from the stage; LL chain: T0, T1, T0 (fp32, levels 1-3), then D0, D1, ... (fp64)
    small_ana_level<float, float>(p, S, p.W, p.H * p.W, O, T0, k.g, h, w, p.L == 1);
    __syncthreads();
    if (tid == 0) {   // the stage is free: refill it
      const int64_t nc = c + int64_t(p.stages) * gridDim.x;
      if (nc < p.nchunks) issue_chunk(p, p.in, smem + s * p.stage_bytes, &bars[s], nc);
    }
    for (int j = 2; j <= p.L; ++j) {
      h >>= 1;
      w >>= 1;
      const bool last = j == p.L;
      const int hw = h * w;
      float* const Tin = (j & 1) ? T1 : T0;   // LL1 in T0, LL2 in T1, LL3 in T0
      if (j <= kFirstF64Level - 1)          // fp32 source and arithmetic (levels 2, 3)
        small_ana_level<float, float>(p, Tin, w, hw, O, (j & 1) ? T0 : T1, k.g, h, w, last);
      else if (j == kFirstF64Level)         // fp32 LL3 in, fp64 arithmetic and LL4 out
        small_ana_level<float, double>(p, Tin, w, hw, O, D0, k.g, h, w, last);
      else if (((j - kFirstF64Level) & 1) == 1)   // fp64: LL4 in D0 -> LL5 in D1, LL6 in D0, ...
        small_ana_level<double, double>(p, D0, w, hw, O, D1, k.g, h, w, last);
      else
        small_ana_level<double, double>(p, D1, w, hw, O, D0, k.g, h, w, last);
      __syncthreads();
    }
    fence_proxy_async();   // O's generic-proxy writes -> the bulk store (async proxy)
    __syncthreads();
    if (tid == 0) bulk_store(p.out + k.first * int64_t(p.H) * p.W, O, uint32_t(k.g) * uint32_t(p.H * p.W) * 4u);
  }
  if (tid == 0) bulk_wait_all();
}

// One synthesis level j of g images: LL_j (per image h2 x w2 at pitch lp, image stride ls) and the
// level-j bands of the coefficient chunk S (pitch W) -> LL_{j-1} (h x w) into dst (pitch dp,
// image stride ds).
__device__ __forceinline__ void small_syn_level(const Small2dParams& p, const float* ll, int lp, int ls,
                                                const float* S, float* dst, int dp, int ds, int g, int h, int w) {
  const int h2 = h >> 1, w2 = w >> 1;
  const uint32_t per = uint32_t(h2 * w2), total = per * uint32_t(g);
  const int imgS = p.H * p.W;
  for (uint32_t u = threadIdx.x; u < total; u += blockDim.x) {
    const uint32_t gi = u / per, rem = u - gi * per, r = rem / uint32_t(w2), c = rem - r * uint32_t(w2);
    const float* b = S + gi * imgS + r * p.W + c;
    const float vll = ll[gi * ls + r * lp + c], vhl = b[w2], vlh = b[h2 * p.W], vhh = b[h2 * p.W + w2];
    const float s = vll + vlh, t = vhl + vhh, s2 = vll - vlh, t2 = vhl - vhh;
    float* o = dst + gi * ds + (2 * r) * dp + 2 * c;
    o[0] = (s + t) * 0.5f;
    o[1] = (s - t) * 0.5f;
    o[dp] = (s2 + t2) * 0.5f;
    o[dp + 1] = (s2 - t2) * 0.5f;
  }
}

__global__ void __launch_bounds__(256, 2) syn2d_small_kernel(const __grid_constant__ Small2dParams p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  float* O = reinterpret_cast<float*>(smem + p.off_out);
  float* const T0 = reinterpret_cast<float*>(smem + p.off_t[0]);
  float* const T1 = reinterpret_cast<float*>(smem + p.off_t[1]);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < p.stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < p.stages; ++s) {
      const int64_t c = blockIdx.x + int64_t(s) * gridDim.x;
      if (c < p.nchunks) issue_chunk(p, p.in, smem + s * p.stage_bytes, &bars[s], c);
    }
  int it = 0;
  const int img = p.H * p.W;
  for (int64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x, ++it) {
    const int s = it % p.stages;
    mbar_wait(&bars[s], uint32_t(it / p.stages) & 1u);
    const Chunk k = chunk_of(p, c);
    const float* S = reinterpret_cast<const float*>(smem + s * p.stage_bytes);
    // LL_L: the top-left corner of each coefficient image (pitch W)
    const float* ll = S;
    int lp = p.W, ls = img;
    for (int j = p.L; j >= 1; --j) {
      const int h = p.H >> (j - 1), w = p.W >> (j - 1);
      if (j == 1) {
        if (tid == 0) bulk_wait_read();   // the previous chunk's store has read O
        __syncthreads();
        small_syn_level(p, ll, lp, ls, S, O, p.W, img, k.g, h, w);
      } else {
        float* dst = (j & 1) ? T1 : T0;
        small_syn_level(p, ll, lp, ls, S, dst, w, h * w, k.g, h, w);
        __syncthreads();
        ll = dst;
        lp = w;
        ls = h * w;
      }
    }
    fence_proxy_async();
    __syncthreads();   // S and O complete
    if (tid == 0) {
      bulk_store(p.out + k.first * int64_t(img), O, uint32_t(k.g) * uint32_t(img) * 4u);
      const int64_t nc = c + int64_t(p.stages) * gridDim.x;
      if (nc < p.nchunks) issue_chunk(p, p.in, smem + s * p.stage_bytes, &bars[s], nc);
    }
  }
  if (tid == 0) bulk_wait_all();
}

}  // namespace

cudaError_t small2d_occupancy(bool analysis, size_t smem, int* blocks_per_sm) {
  const void* fn = analysis ? (const void*)ana2d_small_kernel : (const void*)syn2d_small_kernel;
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fn, 256, smem);
}

cudaError_t launch_small2d(const Small2dParams& p, bool analysis, int grid, size_t smem, cudaStream_t s) {
  count_launch();
  void* args[] = {const_cast<Small2dParams*>(&p)};
  return cudaLaunchKernel(analysis ? (const void*)ana2d_small_kernel : (const void*)syn2d_small_kernel, dim3(grid),
                          dim3(256), args, smem, s);
}

}  // namespace fhwt
