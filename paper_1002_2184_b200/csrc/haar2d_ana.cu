// Warp-specialised 2-D Fast Haar analysis of 32 x 256 tiles, 5 levels per pass (c4, c5) — K1 v2.
//
// Method: the polyphase Fast Haar analysis bank (§III Fig. 4) applied
// separably, rows then columns (reading R8); per 2x2 block [[a, b], [c, d]]
// the row and column butterflies fold to one exact x1/2:
//     LL = ½((a+b)+(c+d))  LH = ½((a+b)−(c+d))  HL = ½((a−b)+(c−d))  HH = ½((a−b)−(c−d)),
// iterated on LL (Mallat), levels 1-3 in fp32 and 4-5 in fp64 (reading R13), every output rounded
// once.  Same operations on the same operands, in the same order, as ana2d_kernel<float, 5, 32, 256>
// (haar2d.cu): outputs are bitwise identical (tests/test_gpu_parity.py).
//
// B200 structure ("K1"): a 32 x 256 input tile is 8 independent 32 x 32 blocks
// (Haar's 2-tap support with pairs (2k, 2k+1) closes a 2^5-aligned block under 5 levels), so
//   * warp w of the 8 compute warps owns columns [32w, 32w + 32) of every tile and runs all five
//     levels of its block alone: level 1 from the TMA stage (4 units of 2 x 4 pixels per lane),
//     levels 2+3 from its 16 x 16 LL1 in warp-private shared memory (two lanes per 4 x 4 block,
//     level 3 after a lane-pair shuffle), levels 4+5 in fp64 by warp shuffles.  No CTA barrier:
//     only __syncwarp between levels.
//   * warp 8 is the producer: one lane issues the 32 one-row TMA boxes (1 KB rows, measured faster
//     than one 32-row box) of the CTA's next tile into a stage as soon as all 8 compute warps have
//     arrived on that stage's "empty" mbarrier — which they do right after level 1, the stage's last
//     reader.  The TMA issue is off the compute warps' path.
// 2 CTAs per SM (288 threads each), `stages` 32 KB stages per CTA.
#include <cooperative_groups.h>

#include "fhwt_internal.cuh"
#include "haar2d_coarse.cuh"

namespace fhwt {

namespace {

constexpr int kWsComputeWarps = 8;
constexpr int kWsThreads = 32 * (kWsComputeWarps + 1);
constexpr int kLL1Pitch = 16;   // floats per LL1 row of a warp's 16 x 16 block

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Producer: the 32 one-row boxes of tile t (32-bit tile decode: a tile holds 8192 pixels, so tile
// counts are < 2^31 for any buffer the TMA row range admits).
__device__ __forceinline__ void ws_issue(const Ana2dParams& p, const CUtensorMap* map, unsigned char* dst,
                                         uint64_t* full, uint32_t t, uint64_t pol) {
  const uint32_t rt = t / uint32_t(p.tiles_c), ct = t - rt * uint32_t(p.tiles_c);
  mbar_arrive_expect_tx(full, 32u * 1024u);
  const int row = int(rt) * 32, col = int(ct) * 256;
  if (p.l2hint) {
#pragma unroll 1
    for (int r = 0; r < 32; ++r) tma_load_2d(dst + r * 1024, map, col, row + r, full, pol);
  } else {
#pragma unroll 1
    for (int r = 0; r < 32; ++r) tma_load_2d_nohint(dst + r * 1024, map, col, row + r, full);
  }
}

// Levels 1-5 of warp w's 32 x 32 block of one tile.  `release` is called after level 1 (the last
// read of the stage).
template <typename REL>
__device__ __forceinline__ void ws_block(const Ana2dParams& p, const float* __restrict__ st, float* __restrict__ ll1,
                                         int64_t b, int64_t row0, int64_t col0, int w, int lane, const REL& release) {
  const int64_t W = p.W, H = p.H;
  // ---- level 1: unit (orow, q) = 2 x 4 input pixels -> 1 x 2 outputs per band
  {
    const int64_t wg = W >> 1, hgW = (H >> 1) * W;
    const int q = lane & 7;
    float* const base = p.out + (b * H + (row0 >> 1)) * W + (col0 >> 1) + 16 * w + 2 * q;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int orow = (lane >> 3) + 4 * k;
      const float4 t0 = *reinterpret_cast<const float4*>(st + (2 * orow) * 256 + 32 * w + 4 * q);
      const float4 t1 = *reinterpret_cast<const float4*>(st + (2 * orow + 1) * 256 + 32 * w + 4 * q);
      float ll[2], hl[2], lh[2], hh[2];
      const float a0[2] = {t0.x, t0.z}, b0[2] = {t0.y, t0.w}, c0[2] = {t1.x, t1.z}, d0[2] = {t1.y, t1.w};
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const float s1 = a0[v] + b0[v], s2 = c0[v] + d0[v], d1 = a0[v] - b0[v], d2 = c0[v] - d0[v];
        ll[v] = (s1 + s2) * 0.5f;
        lh[v] = (s1 - s2) * 0.5f;
        hl[v] = (d1 + d2) * 0.5f;
        hh[v] = (d1 - d2) * 0.5f;
      }
      float* pr = base + int64_t(orow) * W;
      stg_stream2(pr + wg, make_float2(hl[0], hl[1]));
      stg_stream2(pr + hgW, make_float2(lh[0], lh[1]));
      stg_stream2(pr + hgW + wg, make_float2(hh[0], hh[1]));
      *reinterpret_cast<float2*>(ll1 + orow * kLL1Pitch + 2 * q) = make_float2(ll[0], ll[1]);
    }
  }
  __syncwarp();
  release();
  // ---- levels 2 + 3: two lanes per 4 x 4 LL1 block (br, bc), lane h takes LL1 columns 2h, 2h+1
  const int blk = lane >> 1, h = lane & 1, br = blk >> 2, bc = blk & 3;
  float l3;
  {
    float x[4][2];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float2 v = *reinterpret_cast<const float2*>(ll1 + (4 * br + r) * kLL1Pitch + 4 * bc + 2 * h);
      x[r][0] = v.x;
      x[r][1] = v.y;
    }
    float ll[2];
    const int64_t wg = W >> 2, hgW = (H >> 2) * W;
#pragma unroll
    for (int i = 0; i < 2; ++i) {   // level 2: row 2br + i, column 2bc + h of the warp's level-2 block
      const float a = x[2 * i][0], bb = x[2 * i][1], c = x[2 * i + 1][0], d = x[2 * i + 1][1];
      const float s1 = a + bb, s2 = c + d, d1 = a - bb, d2 = c - d;
      ll[i] = (s1 + s2) * 0.5f;
      float* pr = p.out + (b * H + (row0 >> 2) + 2 * br + i) * W + (col0 >> 2) + 8 * w + 2 * bc + h;
      stg_stream1(pr + wg, (d1 + d2) * 0.5f);
      stg_stream1(pr + hgW, (s1 - s2) * 0.5f);
      stg_stream1(pr + hgW + wg, (d1 - d2) * 0.5f);
    }
    const float o0 = __shfl_xor_sync(0xffffffffu, ll[0], 1), o1 = __shfl_xor_sync(0xffffffffu, ll[1], 1);
    // level 3 on the 2 x 2 LL2 block (lane h = 0): a = (0, 0), b = (0, 1), c = (1, 0), d = (1, 1)
    const float a = ll[0], bb = o0, c = ll[1], d = o1;
    const float s1 = a + bb, s2 = c + d, d1 = a - bb, d2 = c - d;
    l3 = (s1 + s2) * 0.5f;
    if (h == 0) {
      const int64_t wg3 = W >> 3, hgW3 = (H >> 3) * W;
      float* pr = p.out + (b * H + (row0 >> 3) + br) * W + (col0 >> 3) + 4 * w + bc;
      stg_stream1(pr + wg3, (d1 + d2) * 0.5f);
      stg_stream1(pr + hgW3, (s1 - s2) * 0.5f);
      stg_stream1(pr + hgW3 + wg3, (d1 - d2) * 0.5f);
    }
  }
  // ---- level 4 (fp64) on the 2 x 2 blocks of the warp's 4 x 4 LL3 (held by lanes 2 * (4 br + bc))
  {
    const double a = double(l3);
    const double bb = double(__shfl_down_sync(0xffffffffu, l3, 2));    // (br, bc + 1)
    const double c = double(__shfl_down_sync(0xffffffffu, l3, 8));     // (br + 1, bc)
    const double d = double(__shfl_down_sync(0xffffffffu, l3, 10));    // (br + 1, bc + 1)
    const double s1 = a + bb, s2 = c + d, d1 = a - bb, d2 = c - d;
    const double ll4 = (s1 + s2) * 0.5;
    const bool act4 = h == 0 && (br & 1) == 0 && (bc & 1) == 0;   // lanes 0, 4, 16, 20
    if (act4) {
      const int64_t wg4 = W >> 4, hgW4 = (H >> 4) * W;
      float* pr = p.out + (b * H + (row0 >> 4) + (br >> 1)) * W + (col0 >> 4) + 2 * w + (bc >> 1);
      stg_stream1(pr + wg4, float((d1 + d2) * 0.5));
      stg_stream1(pr + hgW4, float((s1 - s2) * 0.5));
      stg_stream1(pr + hgW4 + wg4, float((d1 - d2) * 0.5));
    }
    // ---- level 5 on the 2 x 2 LL4 (lanes 0, 4, 16, 20) -> lane 0
    const double a5 = ll4;
    const double b5 = __shfl_down_sync(0xffffffffu, ll4, 4);
    const double c5 = __shfl_down_sync(0xffffffffu, ll4, 16);
    const double d5 = __shfl_down_sync(0xffffffffu, ll4, 20);
    if (lane == 0) {
      const double t1 = a5 + b5, t2 = c5 + d5, e1 = a5 - b5, e2 = c5 - d5;
      const int64_t wg5 = W >> 5, hgW5 = (H >> 5) * W;
      float* pr = p.out + (b * H + (row0 >> 5)) * W + (col0 >> 5) + w;
      stg_stream1(pr + wg5, float((e1 + e2) * 0.5));
      stg_stream1(pr + hgW5, float((t1 - t2) * 0.5));
      stg_stream1(pr + hgW5 + wg5, float((e1 - e2) * 0.5));
      const double ll5 = (t1 + t2) * 0.5;
      if (p.final_pass) {
        stg_stream1(pr, float(ll5));
      } else {   // fp64 hand-off of LL5 to the coarse levels (pitch = padded Win >> 5)
        const int64_t wpitch = ((p.Win >> 5) + 3) & ~int64_t(3);
        p.ws_out[(b * (p.Hin >> 5) + (row0 >> 5)) * wpitch + (col0 >> 5) + w] = ll5;
      }
    }
  }
}

__global__ void __launch_bounds__(kWsThreads, 2) ana2d_ws_kernel(const __grid_constant__ Ana2dParams p,
                                                                 const __grid_constant__ CUtensorMap in_map) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* empty = full + p.stages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    prefetch_tmap(&in_map);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWsComputeWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t ntiles = uint32_t(p.ntiles), grid = gridDim.x;
  if (warp == kWsComputeWarps) {   // producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int it = 0;
      for (uint32_t t = blockIdx.x; t < ntiles; t += grid, ++it) {
        const int s = it % p.stages;
        if (it >= p.stages) mbar_wait(&empty[s], uint32_t(it / p.stages - 1) & 1u);
        ws_issue(p, &in_map, smem + s * p.stage_bytes, &full[s], t, pol);
      }
    }
  } else {
    float* ll1 = reinterpret_cast<float*>(smem + p.p_off[0]) + warp * (16 * kLL1Pitch);
    int it = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += grid, ++it) {
      const int s = it % p.stages;
      mbar_wait(&full[s], uint32_t(it / p.stages) & 1u);
      const uint32_t rt = t / uint32_t(p.tiles_c), ct = t - rt * uint32_t(p.tiles_c);
      const uint32_t b = rt / uint32_t(p.tiles_r);
      const int64_t row0 = int64_t(rt - b * uint32_t(p.tiles_r)) * 32, col0 = int64_t(ct) * 256;
      uint64_t* e = &empty[s];
      ws_block(p, reinterpret_cast<const float*>(smem + s * p.stage_bytes), ll1, b, row0, col0, warp, lane, [&] {
        if (lane == 0) mbar_arrive(e);
      });
    }
  }
  if (p.tail > 0) {   // cooperative launch: every CTA is resident, so the grid barrier is safe
    cooperative_groups::this_grid().sync();
    if (p.tail == 1) ana_coarse<1>(p);
    else if (p.tail == 2) ana_coarse<2>(p);
    else ana_coarse<3>(p);
  }
}

// ------------------------------------------------------------------------------------------------
// The default kernel's fused tile chain (haar2d.cu ana_fused_tile, 32 x 256 tiles, LP = 5) written
// once more for the register-load variant below: level 1 by all 256 threads (a warp stores 256-B
// row segments of every band), a barrier, levels 2+3 by warps 0-3 (one 4 x 4 LL1 block per
// thread), a barrier, levels 4+5 in fp64 by 8 lanes of warp 7, which overlap the next tile's level 1.
// level J+1 on a 2 x 2 block of level-J LL values (same operands, order and types as haar2d.cu ana_pair)
template <typename T>
__device__ __forceinline__ T fp_quad(const Ana2dParams& p, T a, T bb, T c, T d, int64_t b, int64_t row, int64_t col, int g) {
  const T s1 = a + bb, s2 = c + d, d1 = a - bb, d2 = c - d;
  const int64_t W = p.W, wg = W >> g, hgW = (p.H >> g) * W;
  float* pr = p.out + (b * p.H + row) * W + col;
  stg_stream1(pr + wg, float((d1 + d2) * T(0.5)));
  stg_stream1(pr + hgW, float((s1 - s2) * T(0.5)));
  stg_stream1(pr + hgW + wg, float((d1 - d2) * T(0.5)));
  return (s1 + s2) * T(0.5);
}

// levels J, J+1 of one thread's 4 x 4 block x of level J-1 LL (haar2d.cu ana_pair, TA -> TB)
template <typename TA, typename TB, int J>
__device__ __forceinline__ TB fp_pair(const Ana2dParams& p, const float (&x)[4][4], int64_t b, int64_t row0,
                                      int64_t col0, int br, int bc) {
  const int64_t W = p.W;
  TA ll[2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    float hl[2], lh[2], hh[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const TA a = TA(x[2 * i][2 * k]), bb = TA(x[2 * i][2 * k + 1]);
      const TA c = TA(x[2 * i + 1][2 * k]), d = TA(x[2 * i + 1][2 * k + 1]);
      const TA s1 = a + bb, s2 = c + d, d1 = a - bb, d2 = c - d;
      ll[i][k] = (s1 + s2) * TA(0.5);
      lh[k] = float((s1 - s2) * TA(0.5));
      hl[k] = float((d1 + d2) * TA(0.5));
      hh[k] = float((d1 - d2) * TA(0.5));
    }
    float* pr = p.out + (b * p.H + (row0 >> J) + 2 * br + i) * W + (col0 >> J) + 2 * bc;
    const int64_t wg = W >> J, hgW = (p.H >> J) * W;
    stg_stream2(pr + wg, make_float2(hl[0], hl[1]));
    stg_stream2(pr + hgW, make_float2(lh[0], lh[1]));
    stg_stream2(pr + hgW + wg, make_float2(hh[0], hh[1]));
  }
  return fp_quad<TB>(p, TB(ll[0][0]), TB(ll[0][1]), TB(ll[1][0]), TB(ll[1][1]), b, (row0 >> (J + 1)) + br,
                     (col0 >> (J + 1)) + bc, J + 1);
}

// The compute side of one tile of the fused chain (256 compute threads): level 1, barrier, levels
// 2+3 (warps 0-3), barrier, levels 4+5 (warp 7 lanes 0-7).  `after1` runs right after the first
// barrier (the stage has been read for the last time); BAR is the 256-thread barrier.
// Level-1 input of the fused chain from the TMA stage in shared memory.
struct SmemL1 {
  const float* st;
  __device__ __forceinline__ void operator()(int k, int orow, int oc, float4& t0, float4& t1) const {
    t0 = *reinterpret_cast<const float4*>(st + (2 * orow) * 256 + 2 * oc);
    t1 = *reinterpret_cast<const float4*>(st + (2 * orow + 1) * 256 + 2 * oc);
  }
};

template <typename BAR, typename AFTER, typename SRC = SmemL1>
__device__ __forceinline__ void fp_tile(const Ana2dParams& p, const SRC& src, float* ll1, float* ll3,
                                        uint32_t b, int64_t row0, int64_t col0, int tid, const BAR& bar,
                                        const AFTER& after1) {
  const int64_t W = p.W, H = p.H;
  {   // level 1: unit u = tid + 256 k -> (orow, oc) = (u / 64, 2 (u % 64)), a 2 x 4 input block
    const int64_t wg = W >> 1, hgW = (H >> 1) * W;
    float* const base = p.out + (int64_t(b) * H + (row0 >> 1)) * W + (col0 >> 1);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int u = tid + 256 * k, orow = u >> 6, oc = 2 * (u & 63);
      float4 t0, t1;
      src(k, orow, oc, t0, t1);
      const float a0[2] = {t0.x, t0.z}, b0[2] = {t0.y, t0.w}, c0[2] = {t1.x, t1.z}, d0[2] = {t1.y, t1.w};
      float ll[2], hl[2], lh[2], hh[2];
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const float s1 = a0[v] + b0[v], s2 = c0[v] + d0[v], d1 = a0[v] - b0[v], d2 = c0[v] - d0[v];
        ll[v] = (s1 + s2) * 0.5f;
        lh[v] = (s1 - s2) * 0.5f;
        hl[v] = (d1 + d2) * 0.5f;
        hh[v] = (d1 - d2) * 0.5f;
      }
      float* pr = base + int64_t(orow) * W + oc;
      stg_stream2(pr + wg, make_float2(hl[0], hl[1]));
      stg_stream2(pr + hgW, make_float2(lh[0], lh[1]));
      stg_stream2(pr + hgW + wg, make_float2(hh[0], hh[1]));
      *reinterpret_cast<float2*>(ll1 + orow * 128 + oc) = make_float2(ll[0], ll[1]);
    }
  }
  bar();   // LL1 complete; every compute warp is done with the stage
  after1();
  if (tid < 128) {   // levels 2 + 3: block (br, bc) of LL1, 4 x 32 blocks
    const int br = tid >> 5, bc = tid & 31;
    float x[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float4 v = *reinterpret_cast<const float4*>(ll1 + (4 * br + r) * 128 + 4 * bc);
      x[r][0] = v.x; x[r][1] = v.y; x[r][2] = v.z; x[r][3] = v.w;
    }
    ll3[br * 32 + bc] = fp_pair<float, float, 2>(p, x, b, row0, col0, br, bc);
  }
  bar();   // LL3 complete
  if (tid >= 224 && tid < 232) {   // levels 4 + 5 (fp64): block q of LL3 (4 x 32)
    const int q = tid - 224;
    float x[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float4 v = *reinterpret_cast<const float4*>(ll3 + r * 32 + 4 * q);
      x[r][0] = v.x; x[r][1] = v.y; x[r][2] = v.z; x[r][3] = v.w;
    }
    const double ll5 = fp_pair<double, double, 4>(p, x, b, row0, col0, 0, q);
    if (p.final_pass) {
      stg_stream1(p.out + (int64_t(b) * H + (row0 >> 5)) * W + (col0 >> 5) + q, float(ll5));
    } else {   // fp64 hand-off of LL5 to the coarse levels (pitch = padded Win >> 5)
      const int64_t wpitch = ((p.Win >> 5) + 3) & ~int64_t(3);
      p.ws_out[(int64_t(b) * (p.Hin >> 5) + (row0 >> 5)) * wpitch + (col0 >> 5) + q] = ll5;
    }
  }
}

__device__ __forceinline__ void ana_tail(const Ana2dParams& p) {
  if (p.tail > 0) {   // cooperative launch: every CTA is resident, so the grid barrier is safe
    cooperative_groups::this_grid().sync();
    if (p.tail == 1) ana_coarse<1>(p);
    else if (p.tail == 2) ana_coarse<2>(p);
    else ana_coarse<3>(p);
  }
}

// ------------------------------------------------------------------------------------------------
// Register loads (FHWT_ANA_FUSED=11): no input staging at all — every thread loads its four 2 x 4
// input blocks straight into registers (LDG.128, a warp reads 512 contiguous bytes per row), as
// tools/membench.cu k_tile_ldg does (6.5 TB/s at 4 CTAs/SM); latency is hidden by occupancy
// (up to 4 CTAs/SM, shared memory holds only LL1 / LL3), not by a TMA ring.
struct GlobalL1 {
  const float4 (&v)[8];
  __device__ __forceinline__ void operator()(int k, int, int, float4& t0, float4& t1) const {
    t0 = v[2 * k];
    t1 = v[2 * k + 1];
  }
};

__device__ __forceinline__ void ldg_tile_loads(const Ana2dParams& p, uint32_t t, int tid, float4 (&v)[8]) {
  const uint32_t rt = t / uint32_t(p.tiles_c), ct = t - rt * uint32_t(p.tiles_c);
  const float* src = p.in + int64_t(rt) * 32 * p.W + int64_t(ct) * 256;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int u = tid + 256 * k, orow = u >> 6, oc = 2 * (u & 63);
    v[2 * k] = ldg_stream4(src + int64_t(2 * orow) * p.W + 2 * oc);
    v[2 * k + 1] = ldg_stream4(src + int64_t(2 * orow + 1) * p.W + 2 * oc);
  }
}

// MINB: resident CTAs per SM the registers are capped for; PREFETCH: the next tile's loads are
// issued before the current tile is computed (registers double-buffered); AFTER1: the next tile's
// loads are issued right after this tile's level 1 (into the same registers, which level 1 was the
// last reader of), so they fly while levels 2-5 run — no extra registers.
template <int MINB, bool PREFETCH, bool AFTER1 = false>
__global__ void __launch_bounds__(256, MINB) ana2d_ldg_kernel(const __grid_constant__ Ana2dParams p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int tid = threadIdx.x;
  const uint32_t ntiles = uint32_t(p.ntiles), grid = gridDim.x;
  float* ll1 = reinterpret_cast<float*>(smem + p.p_off[1]);
  float* ll3 = reinterpret_cast<float*>(smem + p.p_off[0]);
  float4 v[8];
  [[maybe_unused]] float4 nv[8];
  if constexpr (PREFETCH) {
    if (blockIdx.x < ntiles) ldg_tile_loads(p, blockIdx.x, tid, nv);
  }
  if constexpr (AFTER1) {
    if (blockIdx.x < ntiles) ldg_tile_loads(p, blockIdx.x, tid, v);
  }
  for (uint32_t t = blockIdx.x; t < ntiles; t += grid) {
    const uint32_t rt = t / uint32_t(p.tiles_c), ct = t - rt * uint32_t(p.tiles_c);
    const uint32_t b = rt / uint32_t(p.tiles_r);
    const int64_t row0 = int64_t(rt - b * uint32_t(p.tiles_r)) * 32, col0 = int64_t(ct) * 256;
    if constexpr (AFTER1) {
      fp_tile(p, GlobalL1{v}, ll1, ll3, b, row0, col0, tid, [] { __syncthreads(); }, [&] {
        if (t + grid < ntiles) ldg_tile_loads(p, t + grid, tid, v);
      });
      continue;
    }
    if constexpr (PREFETCH) {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = nv[i];
      if (t + grid < ntiles) ldg_tile_loads(p, t + grid, tid, nv);
    } else {
      ldg_tile_loads(p, t, tid, v);
    }
    // (no barrier after the tile: the next tile's level 1 writes LL1 after every warp passed this
    // tile's second barrier, and warp 7's levels 4+5 read LL3 before it reaches the next first one)
    fp_tile(p, GlobalL1{v}, ll1, ll3, b, row0, col0, tid, [] { __syncthreads(); }, [] {});
  }
  ana_tail(p);
}

template <int MINB, bool PF, bool A1 = false>
static const void* ldg_fn() { return (const void*)ana2d_ldg_kernel<MINB, PF, A1>; }

// FHWT_ANA_LDG: 0 = 3 CTAs/SM, 1 = 4 CTAs/SM, 2 = prefetch at 2, 3 = next tile's loads after level 1
// at 3 CTAs/SM, 4 = the same at 2 CTAs/SM
static const void* ldg_variant(int v) {
  return v == 1   ? ldg_fn<4, false>()
         : v == 2 ? ldg_fn<2, true>()
         : v == 3 ? ldg_fn<3, false, true>()
         : v == 4 ? ldg_fn<2, false, true>()
                  : ldg_fn<3, false>();
}

}  // namespace

cudaError_t ana2d_ldg_occupancy(size_t smem, int* blocks_per_sm, int variant) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, ldg_variant(variant), 256, smem);
}

cudaError_t launch_ana2d_ldg(const Ana2dParams& p, int grid, size_t smem, cudaStream_t s, int variant) {
  count_launch();
  void* args[] = {const_cast<Ana2dParams*>(&p)};
  if (p.tail > 0) return cudaLaunchCooperativeKernel(ldg_variant(variant), dim3(grid), dim3(256), args, smem, s);
  return cudaLaunchKernel(ldg_variant(variant), dim3(grid), dim3(256), args, smem, s);
}

int ana2d_ws_threads() { return kWsThreads; }

// shared memory: stages x 32 KB | 8 x 1 KB LL1 scratch | full[stages], empty[stages]
size_t ana2d_ws_smem(int stages, uint32_t* ll1_off, uint32_t* bar_off) {
  *ll1_off = uint32_t(stages) * 32768u;
  *bar_off = *ll1_off + kWsComputeWarps * 16 * kLL1Pitch * 4;
  return size_t(*bar_off) + 16 * size_t(stages);
}

cudaError_t ana2d_ws_occupancy(size_t smem, int* blocks_per_sm) {
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute((const void*)ana2d_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, (const void*)ana2d_ws_kernel, kWsThreads, smem);
}

cudaError_t launch_ana2d_ws(const Ana2dParams& p, const CUtensorMap& in_map, int grid, size_t smem, cudaStream_t s) {
  count_launch();
  void* args[] = {const_cast<Ana2dParams*>(&p), const_cast<CUtensorMap*>(&in_map)};
  if (p.tail > 0)
    return cudaLaunchCooperativeKernel((const void*)ana2d_ws_kernel, dim3(grid), dim3(kWsThreads), args, smem, s);
  return cudaLaunchKernel((const void*)ana2d_ws_kernel, dim3(grid), dim3(kWsThreads), args, smem, s);
}

}  // namespace fhwt
