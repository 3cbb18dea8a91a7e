// Warp-private level-1 synthesis of 32 x 256 output tiles, 5 levels per pass (c4, c5) — K4 v2.
//
// Method: the polyphase Fast Haar synthesis bank (§IV Eq. (19), Figs. 6-7)
// applied separably, columns then rows (reading R8), folded per 2x2 output block:
//     a = ½((LL+LH)+(HL+HH))  b = ½((LL+LH)−(HL+HH))  c = ½((LL−LH)+(HL−HH))  d = ½((LL−LH)−(HL−HH)),
// coarsest level first.  Same operations on the same operands, in the same order, as
// syn2d_warp_kernel<5> (haar2d.cu): outputs are bitwise identical (tests/test_gpu_parity.py).
//
// B200 structure ("K4"): warp w rebuilds output columns [32w, 32w + 32) of every tile
// (Haar's 2-tap support makes the 32 x 32 block independent for 5 levels), as the default kernel.
// What changes is how the level-1 bands — 3/4 of a tile's input bytes — arrive.  The default stages
// them as three 16-row TMA boxes per tile; multi-row TMA boxes stream ~10 % slower than one-row
// boxes on B200 (tools/membench.cu, profiles/r02_kernel_experiments.md: 6.0 vs 6.6-6.7 TB/s), and
// one-row boxes of the 512-B level-1 rows are more boxes than one issuing lane can feed (4.6 TB/s).
// Here every warp copies ITS OWN 16-column slice of the three level-1 bands (16 rows x 64 B each)
// with 16-B cp.async (LDGSTS) into warp-private shared memory: only that warp ever reads it, so the
// warp refills its slice for tile i + stages as soon as it has finished tile i, with no cross-warp
// hand-off; the coarse levels 2..5 + LL (1/4 of the bytes) keep the shared TMA stage, released by
// the last warp through it (shared counter), which issues the next boxes.
#include <cooperative_groups.h>

#include "fhwt_internal.cuh"
#include "haar2d_coarse.cuh"

namespace fhwt {

namespace {

constexpr int kWpThreads = 256;
constexpr int kWpSlice = 3 * 16 * 16;       // floats per warp-private level-1 slice (HL, LH, HH)
constexpr uint32_t kWpCoarseTx = 8192;      // bytes of the coarse boxes per tile (LL5 + levels 5..2)

struct WpScratch {   // per-warp LL of levels 4..1 (16 x 16 LL1, 8 x 8 LL2, 4 x 4 LL3, 2 x 2 LL4)
  float ll1[16 * 16];
  float ll2[8 * 8];
  float ll3[4 * 4];
  float ll4[2 * 2];
};

__device__ __forceinline__ unsigned atom_add_acq_rel_cta(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void cp_async_wait_n(int n) {   // n = stages - 1 pending groups allowed
  if (n >= 3) cp_async_wait<3>();
  else if (n == 2) cp_async_wait<2>();
  else if (n == 1) cp_async_wait<1>();
  else cp_async_wait<0>();
}

struct WpTile {
  uint32_t b;
  int64_t row0, col0;
};
__device__ __forceinline__ WpTile wp_tile(const Syn2dParams& p, uint32_t t) {
  const uint32_t rt = t / uint32_t(p.tiles_c), ct = t - rt * uint32_t(p.tiles_c);
  const uint32_t b = rt / uint32_t(p.tiles_r);
  return {b, int64_t(rt - b * uint32_t(p.tiles_r)) * 32, int64_t(ct) * 256};
}

// coarse boxes of tile t (LL5 + HL/LH/HH of levels 5..2) into a stage; one lane
__device__ __forceinline__ void wp_issue_coarse(const Syn2dParams& p, const TmaMaps2d& maps, unsigned char* base,
                                                uint64_t* bar, uint32_t t, uint64_t pol) {
  const WpTile x = wp_tile(p, t);
  mbar_arrive_expect_tx(bar, kWpCoarseTx);
  const int64_t llrow = p.ll_from_ws ? int64_t(x.b) * (p.Hin >> 5) + (x.row0 >> 5) : int64_t(x.b) * p.H + (x.row0 >> 5);
  tma_load_2d(base + p.box_off[0][0], &maps.ll, int(x.col0 >> 5), int(llrow), bar, pol);
#pragma unroll 1
  for (int j = 5; j >= 2; --j) {
    const int64_t hg = p.H >> j, wg = p.W >> j;
    const int64_t br = int64_t(x.b) * p.H + (x.row0 >> j), bc = x.col0 >> j;
    tma_load_2d(base + p.box_off[j][0], &maps.level[j], int(wg + bc), int(br), bar, pol);
    tma_load_2d(base + p.box_off[j][1], &maps.level[j], int(bc), int(br + hg), bar, pol);
    tma_load_2d(base + p.box_off[j][2], &maps.level[j], int(wg + bc), int(br + hg), bar, pol);
  }
}

// this warp's level-1 slice of tile t: bands q = HL, LH, HH, rows r < 16, 64 B each -> 192 x 16 B
__device__ __forceinline__ void wp_issue_slice(const Syn2dParams& p, float* slice, uint32_t t, int warp, int lane) {
  const WpTile x = wp_tile(p, t);
  const int64_t W = p.W, H = p.H;
  const float* g = p.coeffs + (int64_t(x.b) * H + (x.row0 >> 1)) * W + (x.col0 >> 1) + 16 * warp;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const int c = lane + 32 * k, q = c >> 6, r = (c >> 2) & 15, cc = (c & 3) * 4;
    const float* src = g + (q >= 1 ? (H >> 1) * W : 0) + (q != 1 ? (W >> 1) : 0) + int64_t(r) * W + cc;
    cp_async16(slice + q * 256 + r * 16 + cc, src);
  }
}

// one coarse synthesis level J (5..2) of warp w's block from the staged boxes (as haar2d.cu
// warp_syn_level, unshifted): LL_J (R x C, pitch llp) + bands -> LL_{J-1} (2R x 2C) in dst
template <int J>
__device__ __forceinline__ void wp_level(const Syn2dParams& p, const float* __restrict__ ll, int llp,
                                         const unsigned char* stage, int warp, int lane, float* __restrict__ dst) {
  constexpr int R = 32 >> J, C = 32 >> J, BP = 256 >> J;
  constexpr int V = C >= 2 ? 2 : 1, UPR = C / V, NU = R * UPR, OC = 2 * C;
  const int co = (32 * warp) >> J;
  const float* hl = reinterpret_cast<const float*>(stage + p.box_off[J][0]) + co;
  const float* lh = reinterpret_cast<const float*>(stage + p.box_off[J][1]) + co;
  const float* hh = reinterpret_cast<const float*>(stage + p.box_off[J][2]) + co;
#pragma unroll
  for (int it = 0; it < (NU + 31) / 32; ++it) {
    const int u = lane + 32 * it;
    if (NU % 32 != 0 && u >= NU) break;
    const int r = u / UPR, c = (u - r * UPR) * V;
    float vll[V], vhl[V], vlh[V], vhh[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      vll[v] = ll[r * llp + c + v];
      vhl[v] = hl[r * BP + c + v];
      vlh[v] = lh[r * BP + c + v];
      vhh[v] = hh[r * BP + c + v];
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const float s = vll[v] + vlh[v], t = vhl[v] + vhh[v];
      const float s2 = vll[v] - vlh[v], t2 = vhl[v] - vhh[v];
      float* d0 = dst + (2 * r) * OC + 2 * (c + v);
      d0[0] = (s + t) * 0.5f;
      d0[1] = (s - t) * 0.5f;
      d0[OC] = (s2 + t2) * 0.5f;
      d0[OC + 1] = (s2 - t2) * 0.5f;
    }
  }
}

__global__ void __launch_bounds__(kWpThreads, 2) syn2d_wp_kernel(const __grid_constant__ Syn2dParams p,
                                                                 const __grid_constant__ TmaMaps2d maps) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  unsigned* cnt = reinterpret_cast<unsigned*>(smem + p.bar_off + 8 * p.stages);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  WpScratch* sc = reinterpret_cast<WpScratch*>(smem + p.p_off[0] + warp * kSynScratchBytes);
  // warp-private level-1 slices: [stage][warp] after the shared coarse part of every stage
  auto slice = [&](int s) {
    return reinterpret_cast<float*>(smem + s * p.stage_bytes + p.p_off[1]) + warp * kWpSlice;
  };
  if (tid == 0) {
    for (int j = 2; j <= 5; ++j) prefetch_tmap(&maps.level[j]);
    prefetch_tmap(&maps.ll);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&bars[s], 1);
      cnt[s] = 0;
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (p.head > 0) {   // cooperative launch: coarse levels -> fp32 LL5 hand-off, then a grid barrier
    if (p.head == 1) syn_coarse<1>(p);
    else if (p.head == 2) syn_coarse<2>(p);
    else syn_coarse<3>(p);
    fence_proxy_async_global();   // generic-proxy stores, read below by TMA (async proxy)
    cooperative_groups::this_grid().sync();
    fence_proxy_async_global();
  }
  const uint32_t ntiles = uint32_t(p.ntiles), grid = gridDim.x;
  const uint64_t pol = policy_evict_first();
  for (int s = 0; s < p.stages; ++s) {
    const uint32_t t = blockIdx.x + uint32_t(s) * grid;
    if (t < ntiles) {
      if (tid == 0) wp_issue_coarse(p, maps, smem + s * p.stage_bytes, &bars[s], t, pol);
      wp_issue_slice(p, slice(s), t, warp, lane);
    }
    cp_async_commit();
  }
  int it = 0;
  for (uint32_t t = blockIdx.x; t < ntiles; t += grid, ++it) {
    const int s = it % p.stages;
    const unsigned char* stage = smem + s * p.stage_bytes;
    const WpTile x = wp_tile(p, t);
    mbar_wait(&bars[s], uint32_t(it / p.stages) & 1u);
    // ---- coarse levels 5..2 from the shared stage (LL5 box pitch 8)
    wp_level<5>(p, reinterpret_cast<const float*>(stage + p.box_off[0][0]) + warp, 8, stage, warp, lane, sc->ll4);
    __syncwarp();
    wp_level<4>(p, sc->ll4, 2, stage, warp, lane, sc->ll3);
    __syncwarp();
    wp_level<3>(p, sc->ll3, 4, stage, warp, lane, sc->ll2);
    __syncwarp();
    wp_level<2>(p, sc->ll2, 8, stage, warp, lane, sc->ll1);
    __syncwarp();
    if (lane == 0) {   // the coarse boxes of this stage are consumed: the last warp refills them
      if ((atom_add_acq_rel_cta(&cnt[s], 1u) & 7u) == 7u) {
        const uint32_t nt = t + uint32_t(p.stages) * grid;
        if (nt < ntiles) wp_issue_coarse(p, maps, smem + s * p.stage_bytes, &bars[s], nt, pol);
      }
    }
    // ---- level 1 from LL1 (scratch) and this warp's private slice, once its copies have landed
    cp_async_wait_n(p.stages - 1);
    __syncwarp();
    const float* sl = slice(s);
    float* const obase = p.out + (int64_t(x.b) * p.Hin + x.row0) * p.out_pitch + x.col0 + 32 * warp;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int u = lane + 32 * k, r = u >> 3, c = (u & 7) * 2;
      const float2 ll = *reinterpret_cast<const float2*>(sc->ll1 + r * 16 + c);
      const float2 hl = *reinterpret_cast<const float2*>(sl + r * 16 + c);
      const float2 lh = *reinterpret_cast<const float2*>(sl + 256 + r * 16 + c);
      const float2 hh = *reinterpret_cast<const float2*>(sl + 512 + r * 16 + c);
      const float vll[2] = {ll.x, ll.y}, vhl[2] = {hl.x, hl.y}, vlh[2] = {lh.x, lh.y}, vhh[2] = {hh.x, hh.y};
      float top[4], bot[4];
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const float s0 = vll[v] + vlh[v], t0 = vhl[v] + vhh[v];
        const float s2 = vll[v] - vlh[v], t2 = vhl[v] - vhh[v];
        top[2 * v] = (s0 + t0) * 0.5f;
        top[2 * v + 1] = (s0 - t0) * 0.5f;
        bot[2 * v] = (s2 + t2) * 0.5f;
        bot[2 * v + 1] = (s2 - t2) * 0.5f;
      }
      float* o = obase + int64_t(2 * r) * p.out_pitch + 2 * c;
      stg_stream4(o, make_float4(top[0], top[1], top[2], top[3]));
      stg_stream4(o + p.out_pitch, make_float4(bot[0], bot[1], bot[2], bot[3]));
    }
    __syncwarp();
    // ---- this warp's slice for tile t + stages (the slot is free: only this warp reads it)
    const uint32_t nt = t + uint32_t(p.stages) * grid;
    if (nt < ntiles) wp_issue_slice(p, slice(s), nt, warp, lane);
    cp_async_commit();
  }
  cp_async_wait<0>();
}

}  // namespace

// shared memory: stages x [coarse boxes (box_off) | 8 warp slices (p_off[1])] | 8 x scratch | bars
size_t syn2d_wp_layout(Syn2dParams* p) {
  uint32_t off = 0;
  auto box = [&](uint32_t bytes) {
    const uint32_t o = off;
    off = (off + bytes + 127) & ~127u;
    return o;
  };
  p->box_off[0][0] = box(32);
  for (int j = 5; j >= 2; --j) {
    const uint32_t bytes = uint32_t(32 >> j) * uint32_t(256 >> j) * 4u;
    for (int q = 0; q < 3; ++q) p->box_off[j][q] = box(bytes);
  }
  p->p_off[1] = off;                                   // warp slices, inside every stage
  off += 8u * kWpSlice * 4u;
  p->stage_bytes = (off + 1023) & ~1023u;
  p->p_off[0] = uint32_t(p->stages) * p->stage_bytes;  // per-warp LL scratch
  p->bar_off = p->p_off[0] + 8u * kSynScratchBytes;
  return size_t(p->bar_off) + 12 * size_t(p->stages);
}

cudaError_t syn2d_wp_occupancy(size_t smem, int* blocks_per_sm) {
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute((const void*)syn2d_wp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, (const void*)syn2d_wp_kernel, kWpThreads, smem);
}

cudaError_t launch_syn2d_wp(const Syn2dParams& p, const TmaMaps2d& maps, int grid, size_t smem, cudaStream_t s) {
  count_launch();
  void* args[] = {const_cast<Syn2dParams*>(&p), const_cast<TmaMaps2d*>(&maps)};
  if (p.head > 0)
    return cudaLaunchCooperativeKernel((const void*)syn2d_wp_kernel, dim3(grid), dim3(kWpThreads), args, smem, s);
  return cudaLaunchKernel((const void*)syn2d_wp_kernel, dim3(grid), dim3(kWpThreads), args, smem, s);
}

}  // namespace fhwt
