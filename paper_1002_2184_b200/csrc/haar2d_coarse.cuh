// Coarse levels 6..5+T of the 2-D first passes (analysis and synthesis), shared by haar2d.cu,
// haar2d_ana.cu and haar2d_syn.cu.
#pragma once

#include "fhwt_internal.cuh"

namespace fhwt {
namespace {

// ------------------------------------------- coarse levels 6..5+T inside the first-pass launch
// For 5 < L <= 8 the levels below LL5 (1/1024 of the samples) are computed in the same launch as
// the tiles: a grid barrier (cooperative launch, all CTAs resident), then 4^(T-1) lanes per
// 2^T x 2^T block of LL5, one lane per 2 x 2 LL5 quad (level 6), combining upwards by warp
// shuffles (levels 7, 8).  All loads are issued before any dependent arithmetic, so the phase
// costs about one L2 round trip.  Each coefficient is produced by the same operations on the same
// operands as the level-by-level fp64 pass (reading R13): results are bitwise those of the
// two-launch path (tests/test_gpu_parity.py::test_kernel_variants_bitwise_equal, FHWT_COOP).
__device__ __forceinline__ void coarse_store3(const Ana2dParams& p, int g, int64_t b, int64_t y, int64_t x, double a,
                                              double bb, double c, double d, double* ll) {
  const double s1 = a + bb, s2 = c + d, d1 = a - bb, d2 = c - d;
  const int64_t W = p.W, wg = W >> g, hgW = (p.H >> g) * W;
  float* pr = p.out + (b * p.H + y) * W + x;
  stg_stream1(pr + wg, float((d1 + d2) * 0.5));
  stg_stream1(pr + hgW, float((s1 - s2) * 0.5));
  stg_stream1(pr + hgW + wg, float((d1 - d2) * 0.5));
  *ll = (s1 + s2) * 0.5;
}

template <int T>
__device__ __forceinline__ void ana_coarse(const Ana2dParams& p) {
  constexpr int Q = 1 << (T - 1), G = Q * Q;   // lanes per block: a Q x Q grid of LL5 quads
  const int64_t hl = p.H >> 5, wl = p.W >> 5, wp = (wl + 3) & ~int64_t(3);
  const int64_t rc = wl >> T, per = (hl >> T) * rc, total = p.batch * per * G;
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) - lane; base < total; base += stride) {
    const int64_t q = base + lane;
    const bool valid = q < total;
    const int64_t r = q / G, t = q - r * G;
    const int64_t b = r / per, rem = r - b * per, by = rem / rc, bx = rem - by * rc;
    const int64_t y6 = by * Q + t / Q, x6 = bx * Q + (t % Q);   // this lane's level-6 position
    double a = 0, bb = 0, c = 0, d = 0, ll = 0;
    if (valid) {
      const double* s = p.ws_out + (b * hl + 2 * y6) * wp + 2 * x6;
      const double2 r0 = __ldcg(reinterpret_cast<const double2*>(s));
      const double2 r1 = __ldcg(reinterpret_cast<const double2*>(s + wp));
      a = r0.x; bb = r0.y; c = r1.x; d = r1.y;
      coarse_store3(p, 6, b, y6, x6, a, bb, c, d, &ll);
    }
#pragma unroll
    for (int g = 7, st = 1; g <= 5 + T; ++g, st <<= 1) {   // combine 2 x 2 lanes `st` apart
      const double vr = __shfl_down_sync(0xffffffffu, ll, st);
      const double vd = __shfl_down_sync(0xffffffffu, ll, st * Q);
      const double vdr = __shfl_down_sync(0xffffffffu, ll, st * Q + st);
      const int ty = int(t / Q), tx = int(t % Q);
      if (valid && ty % (2 * st) == 0 && tx % (2 * st) == 0)
        coarse_store3(p, g, b, y6 >> (g - 6), x6 >> (g - 6), ll, vr, vd, vdr, &ll);
    }
    if (valid && t == 0) stg_stream1(p.out + (b * p.H + by) * p.W + bx, float(ll));
  }
}

// Synthesis mirror: one lane per 2 x 2 quad of LL5; the lane walks its own path down from
// LL_{5+T} (recomputing the few shared upper butterflies instead of exchanging them) and writes
// its quad of the fp32 LL5 hand-off, the input of the tile phase.  Same fp32 operations as the
// level-by-level pass.
template <int T>
__device__ __forceinline__ void syn_coarse(const Syn2dParams& p) {
  constexpr int Q = 1 << (T - 1), G = Q * Q;
  const int64_t hl = p.H >> 5, wl = p.W >> 5, wp = (wl + 3) & ~int64_t(3);
  const int64_t rc = wl >> T, per = (hl >> T) * rc, total = p.batch * per * G;
  const int64_t W = p.W;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = q / G, t = q - r * G;
    const int64_t b = r / per, rem = r - b * per, by = rem / rc, bx = rem - by * rc;
    const int64_t y6 = by * Q + t / Q, x6 = bx * Q + (t % Q);
    float bhl[T], blh[T], bhh[T];   // bands along the path, level 5+T first (all loads up front)
#pragma unroll
    for (int i = 0; i < T; ++i) {
      const int g = 5 + T - i;
      const float* pr = p.coeffs + (b * p.H + (y6 >> (g - 6))) * W + (x6 >> (g - 6));
      bhl[i] = pr[W >> g];
      blh[i] = pr[(p.H >> g) * W];
      bhh[i] = pr[(p.H >> g) * W + (W >> g)];
    }
    float ll = p.coeffs[(b * p.H + by) * W + bx];
#pragma unroll
    for (int i = 0; i < T; ++i) {
      const int g = 5 + T - i;
      const float s = ll + blh[i], tt = bhl[i] + bhh[i], s2 = ll - blh[i], t2 = bhl[i] - bhh[i];
      const float t0 = (s + tt) * 0.5f, t1 = (s - tt) * 0.5f, b0 = (s2 + t2) * 0.5f, b1 = (s2 - t2) * 0.5f;
      if (i == T - 1) {   // level 6 -> this lane's 2 x 2 quad of LL5
        float* o = p.ll_ws_out + (b * hl + 2 * y6) * wp + 2 * x6;
        *reinterpret_cast<float2*>(o) = make_float2(t0, t1);
        *reinterpret_cast<float2*>(o + wp) = make_float2(b0, b1);
      } else {           // child of LL_g on this lane's path: position at level g - 1
        const int cy = int(y6 >> (g - 7)) & 1, cx = int(x6 >> (g - 7)) & 1;
        ll = cy ? (cx ? b1 : b0) : (cx ? t1 : t0);
      }
    }
  }
}

}  // namespace
}  // namespace fhwt
