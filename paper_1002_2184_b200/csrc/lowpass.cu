// §8(f) f1 — LL-only "lowpass image" path with uint8 input (§V, Fig. 12: the
// paper's image output is the lowpass band of the Fast Haar transform).
//
// Only the LL branch of the separable Fast Haar analysis is computed: per level
// LL_j = ½((a + b) + (c + d)) over 2x2 blocks of LL_{j-1} (rows then columns folded, reading R8).
// Input is the image's native 8-bit form (1 B/pixel), output is LL_L only (4 B per 4^L pixels), so
// the kernel is a read-dominated HBM stream: ~1 B/pixel.
//
// Stage A: one thread per 2^M x 2^M block (M = min(L, 4)) loads 2^M rows of 2^M bytes (uint4 for
// M = 4: a warp reads 512 contiguous bytes per row), runs M levels in registers (levels 1-3 in fp32,
// level 4 in fp64 — exact for uint8 either way) and writes one LL_M value.  Stage B (L > 4): one
// tiny pass per further level on the fp64 LL chain.  Outputs are rounded to fp32 once.
#include <cstdlib>

#include "fhwt_internal.cuh"

namespace fhwt {
namespace {

template <int M>
struct RowVec;
template <>
struct RowVec<4> {
  using T = uint4;
};
template <>
struct RowVec<3> {
  using T = uint2;
};
template <>
struct RowVec<2> {
  using T = uint32_t;
};
template <>
struct RowVec<1> {
  using T = uint16_t;
};

template <int M>
__device__ __forceinline__ typename RowVec<M>::T load_row(const uint8_t* p) {
  using T = typename RowVec<M>::T;
  if constexpr (M == 4) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
  } else {
    return __ldg(reinterpret_cast<const T*>(p));
  }
}

template <int M>
__device__ __forceinline__ void unpack(const typename RowVec<M>::T& t, float (&v)[1 << M]) {
  const uint8_t* b = reinterpret_cast<const uint8_t*>(&t);
#pragma unroll
  for (int i = 0; i < (1 << M); ++i) v[i] = float(b[i]);
}

// One 2^M x 2^M block -> LL_M.  Levels 1..min(M,3) fp32, level 4 fp64.
template <int M>
__global__ void __launch_bounds__(256) lowpass_stage_a(const uint8_t* __restrict__ d, float* __restrict__ out32,
                                                       double* __restrict__ out64, int64_t h, int64_t w,
                                                       int64_t batch) {
  constexpr int N = 1 << M;
  const int64_t bh = h >> M, bw = w >> M;
  const int64_t total = batch * bh * bw;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / (bh * bw), rem = i - b * bh * bw;
    const int64_t r = rem / bw, c = rem - r * bw;
    const uint8_t* src = d + (b * h + r * N) * w + c * N;
    // all 2^M row loads first (2^M x 2^M bytes in flight per thread), then the levels
    typename RowVec<M>::T raw[N];
#pragma unroll
    for (int y = 0; y < N; ++y) raw[y] = load_row<M>(src + int64_t(y) * w);
    float l1[N / 2][N / 2];
#pragma unroll
    for (int y = 0; y < N; y += 2) {
      float r0[N], r1[N];
      unpack<M>(raw[y], r0);
      unpack<M>(raw[y + 1], r1);
#pragma unroll
      for (int x = 0; x < N; x += 2) l1[y / 2][x / 2] = ((r0[x] + r0[x + 1]) + (r1[x] + r1[x + 1])) * 0.5f;
    }
    double res;
    if constexpr (M == 1) {
      res = l1[0][0];
    } else {
      float l2[N / 4][N / 4];
#pragma unroll
      for (int y = 0; y < N / 4; ++y)
#pragma unroll
        for (int x = 0; x < N / 4; ++x)
          l2[y][x] = ((l1[2 * y][2 * x] + l1[2 * y][2 * x + 1]) + (l1[2 * y + 1][2 * x] + l1[2 * y + 1][2 * x + 1])) * 0.5f;
      if constexpr (M == 2) {
        res = l2[0][0];
      } else {
        float l3[N / 8][N / 8];
#pragma unroll
        for (int y = 0; y < N / 8; ++y)
#pragma unroll
          for (int x = 0; x < N / 8; ++x)
            l3[y][x] = ((l2[2 * y][2 * x] + l2[2 * y][2 * x + 1]) + (l2[2 * y + 1][2 * x] + l2[2 * y + 1][2 * x + 1])) * 0.5f;
        if constexpr (M == 3) {
          res = l3[0][0];
        } else {  // level 4 in fp64
          res = ((double(l3[0][0]) + double(l3[0][1])) + (double(l3[1][0]) + double(l3[1][1]))) * 0.5;
        }
      }
    }
    if (out64)
      out64[i] = res;
    else
      out32[i] = float(res);
  }
}

// Wide variant (w % 16 == 0): one thread per 2^M rows x 16 columns — every row is one 16-B load,
// all issued before the arithmetic — producing 16 >> M consecutive LL_M values.
// The butterfly chain LL_j = ½((a+b)+(c+d)) is carried as the exact integer sums S_j = 2^j LL_j
// (S_j = sum of the four S_{j-1}), two 16-bit lanes per register for level 1 (SWAR: no per-byte
// int->float conversion, which is a quarter-rate pipe and bounded this kernel at ~4 TB/s), and the
// exact power-of-two scale 2^-M is applied once.  For uint8 input this is bit-identical to the
// floating-point butterflies (all values are exact dyadic rationals), which the tests assert.
__device__ __forceinline__ uint32_t pair_sums(uint32_t w) {  // bytes b0..b3 -> lanes [b0+b1, b2+b3]
  return (w & 0x00FF00FFu) + ((w >> 8) & 0x00FF00FFu);
}

template <int M>
__global__ void __launch_bounds__(256) lowpass_stage_a_wide(const uint8_t* __restrict__ d, float* __restrict__ out32,
                                                            uint32_t* __restrict__ out_s4, int64_t h, int64_t w,
                                                            int64_t batch) {
  constexpr int R = 1 << M, NO = 16 >> M;
  const int64_t bh = h >> M, bw = w >> 4;   // row blocks, 16-column groups
  const int64_t total = batch * bh * bw;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / (bh * bw), rem = i - b * bh * bw;
    const int64_t r = rem / bw, g = rem - r * bw;
    const uint8_t* src = d + (b * h + r * R) * w + g * 16;
    uint4 raw[R];
#pragma unroll
    for (int y = 0; y < R; ++y) raw[y] = load_row<4>(src + int64_t(y) * w);
    // level 1: S1 = a + b + c + d per 2x2 block, lanes [S1(2k), S1(2k+1)] of word k (<= 1020)
    uint32_t s1[R / 2][4];
#pragma unroll
    for (int y = 0; y < R / 2; ++y) {
      const uint32_t t[4] = {raw[2 * y].x, raw[2 * y].y, raw[2 * y].z, raw[2 * y].w};
      const uint32_t u[4] = {raw[2 * y + 1].x, raw[2 * y + 1].y, raw[2 * y + 1].z, raw[2 * y + 1].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) s1[y][k] = pair_sums(t[k]) + pair_sums(u[k]);
    }
    const int64_t o = (b * bh + r) * (w >> M) + g * NO;
    if constexpr (M == 1) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[2 * k] = float(s1[0][k] & 0xFFFFu) * 0.5f;
        v[2 * k + 1] = float(s1[0][k] >> 16) * 0.5f;
      }
      stg_stream4(out32 + o, make_float4(v[0], v[1], v[2], v[3]));      // o is a multiple of 8
      stg_stream4(out32 + o + 4, make_float4(v[4], v[5], v[6], v[7]));
    } else {
      // level 2: S2 = sum of a 2x2 block of S1 (lanes of one word, two row pairs)
      uint32_t s2[R / 4][4];
#pragma unroll
      for (int y = 0; y < R / 4; ++y)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          s2[y][k] = ((s1[2 * y][k] & 0xFFFFu) + (s1[2 * y][k] >> 16)) +
                     ((s1[2 * y + 1][k] & 0xFFFFu) + (s1[2 * y + 1][k] >> 16));
      if constexpr (M == 2) {
        stg_stream4(out32 + o, make_float4(float(s2[0][0]) * 0.25f, float(s2[0][1]) * 0.25f, float(s2[0][2]) * 0.25f,
                                           float(s2[0][3]) * 0.25f));
      } else {
        uint32_t s3[R / 8][2];
#pragma unroll
        for (int y = 0; y < R / 8; ++y)
#pragma unroll
          for (int k = 0; k < 2; ++k)
            s3[y][k] = (s2[2 * y][2 * k] + s2[2 * y][2 * k + 1]) + (s2[2 * y + 1][2 * k] + s2[2 * y + 1][2 * k + 1]);
        if constexpr (M == 3) {
          out32[o] = float(s3[0][0]) * 0.125f;
          out32[o + 1] = float(s3[0][1]) * 0.125f;
        } else {  // level 4 (fp64 per DESIGN.md §5; exact either way)
          const uint32_t s4 = (s3[0][0] + s3[0][1]) + (s3[1][0] + s3[1][1]);
          if (out_s4)
            out_s4[o] = s4;   // exact hand-off to the remaining levels
          else
            out32[o] = float(double(s4) * 0.0625);
        }
      }
    }
  }
}

// L = 5 in one launch (h % 32 == 0, w % 256 == 0): each thread forms the exact S4 of a 16 x 16 block
// as the wide kernel does (SWAR level 1, integer levels 2-4), and S5 = the sum of the S4 of a 2 x 2
// group of lanes by warp shuffles (lane bits: x = (b0, b2, b3, b4), y = b1: a warp covers 32 rows x
// 256 columns and lanes with equal y read one 256-B row segment per load).  LL5 = S5 / 32, exact.
__global__ void __launch_bounds__(256) lowpass_u8_warp5(const uint8_t* __restrict__ d, float* __restrict__ out,
                                                        int64_t h, int64_t w, int64_t batch) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t wr = h >> 5, wc = w >> 8, total = batch * wr * wc;
  if (wid >= total) return;
  const int64_t b = wid / (wr * wc), rem = wid - b * wr * wc;
  const int64_t tr = rem / wc, tc = rem - tr * wc;
  const int x = (lane & 1) | ((lane >> 1) & 14);   // bits 0, 2, 3, 4
  const int y = (lane >> 1) & 1;
  const uint8_t* src = d + (b * h + tr * 32 + y * 16) * w + tc * 256 + x * 16;
  uint4 raw[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) raw[r] = load_row<4>(src + int64_t(r) * w);
  uint32_t s1[8][4];
#pragma unroll
  for (int yy = 0; yy < 8; ++yy) {
    const uint32_t t[4] = {raw[2 * yy].x, raw[2 * yy].y, raw[2 * yy].z, raw[2 * yy].w};
    const uint32_t u[4] = {raw[2 * yy + 1].x, raw[2 * yy + 1].y, raw[2 * yy + 1].z, raw[2 * yy + 1].w};
#pragma unroll
    for (int k = 0; k < 4; ++k) s1[yy][k] = pair_sums(t[k]) + pair_sums(u[k]);
  }
  uint32_t s2[4][4];
#pragma unroll
  for (int yy = 0; yy < 4; ++yy)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      s2[yy][k] = ((s1[2 * yy][k] & 0xFFFFu) + (s1[2 * yy][k] >> 16)) +
                  ((s1[2 * yy + 1][k] & 0xFFFFu) + (s1[2 * yy + 1][k] >> 16));
  uint32_t s3[2][2];
#pragma unroll
  for (int yy = 0; yy < 2; ++yy)
#pragma unroll
    for (int k = 0; k < 2; ++k)
      s3[yy][k] = (s2[2 * yy][2 * k] + s2[2 * yy][2 * k + 1]) + (s2[2 * yy + 1][2 * k] + s2[2 * yy + 1][2 * k + 1]);
  const uint32_t s4 = (s3[0][0] + s3[0][1]) + (s3[1][0] + s3[1][1]);
  const uint32_t s5 = s4 + __shfl_xor_sync(0xffffffffu, s4, 1) + __shfl_xor_sync(0xffffffffu, s4, 2) +
                      __shfl_xor_sync(0xffffffffu, s4, 3);
  if ((lane & 3) != 0) return;
  out[(b * (h >> 5) + tr) * (w >> 5) + tc * 8 + (x >> 1)] = float(double(s5) * 0.03125);
}

// Levels 5..L in one launch, from the exact S4 = 16 LL_4 sums of the wide stage A: one thread per
// LL_L value sums its 2^(L-4) x 2^(L-4) block of S4 (S_L = sum of the four S_{L-1}, recursively:
// integer addition is exact, so the association order does not matter) and scales by 2^-L in fp64.
__global__ void lowpass_stage_b_s4(const uint32_t* __restrict__ s4, int64_t rows4, int64_t cols4, int64_t batch,
                                   int k, int levels, float* __restrict__ out) {
  const int64_t n = int64_t(1) << k, orow = rows4 >> k, ocol = cols4 >> k, total = batch * orow * ocol;
  const double scale = 1.0 / double(int64_t(1) << levels);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / (orow * ocol), rem = i - b * orow * ocol;
    const int64_t r = rem / ocol, c = rem - r * ocol;
    const uint32_t* p = s4 + (b * rows4 + r * n) * cols4 + c * n;
    uint64_t acc = 0;
    for (int64_t y = 0; y < n; ++y)
      for (int64_t x = 0; x < n; ++x) acc += p[y * cols4 + x];
    out[i] = float(double(acc) * scale);
  }
}

// One further level on the fp64 chain: LL_{j} (rows x cols per image) -> LL_{j+1}.
__global__ void lowpass_stage_b(const double* __restrict__ in, int64_t rows, int64_t cols, int64_t batch,
                                double* __restrict__ out64, float* __restrict__ out32) {
  const int64_t orow = rows / 2, ocol = cols / 2, total = batch * orow * ocol;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / (orow * ocol), rem = i - b * orow * ocol;
    const int64_t r = rem / ocol, c = rem - r * ocol;
    const double* p = in + (b * rows + 2 * r) * cols + 2 * c;
    const double v = ((p[0] + p[1]) + (p[cols] + p[cols + 1])) * 0.5;
    if (out32)
      out32[i] = float(v);
    else
      out64[i] = v;
  }
}

// bf16 input (§8(f) f1, "uint8/bf16 I/O"): one thread per 2^M rows x 8 columns (M = min(L, 3));
// every row is one 16-B load (8 bf16), all issued before the arithmetic.  bf16 -> fp32 is exact; the
// levels run exactly as the fused analysis kernel (levels 1-3 fp32, LL_j = ((a+b)+(c+d)) * 0.5),
// so LL_M is bitwise the fused transform's LL of the same fp32 image.  Writes 8 >> M LL_M values
// (fp32 output, or the fp64 chain when L > 3: level 4 on in fp64 by lowpass_stage_b).
__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

template <int M>
__global__ void __launch_bounds__(256) lowpass_stage_a_bf16(const uint16_t* __restrict__ d, float* __restrict__ out32,
                                                            double* __restrict__ out64, int64_t h, int64_t w,
                                                            int64_t batch) {
  constexpr int N = 1 << M, OUT = 8 >> M;
  const int64_t bh = h >> M, bw = w >> 3;   // thread blocks of N rows x 8 columns
  const int64_t total = batch * bh * bw;
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= total) return;
  const int64_t b = i / (bh * bw), rem = i - b * bh * bw;
  const int64_t r = rem / bw, c = rem - r * bw;
  const uint16_t* src = d + (b * h + r * N) * w + c * 8;
  uint4 raw[N];
#pragma unroll
  for (int y = 0; y < N; ++y)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(raw[y].x), "=r"(raw[y].y), "=r"(raw[y].z), "=r"(raw[y].w)
                 : "l"(src + int64_t(y) * w));
  float v[N][8];
#pragma unroll
  for (int y = 0; y < N; ++y) {
    const uint32_t q[4] = {raw[y].x, raw[y].y, raw[y].z, raw[y].w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[y][2 * k] = bf16lo(q[k]);
      v[y][2 * k + 1] = bf16hi(q[k]);
    }
  }
  int rows = N, cols = 8;
#pragma unroll
  for (int lev = 1; lev <= M; ++lev) {   // in place: LL_lev[y][x] into v[y][x]
#pragma unroll
    for (int y = 0; y < (N >> lev); ++y)
#pragma unroll
      for (int x = 0; x < (8 >> lev); ++x)
        v[y][x] = ((v[2 * y][2 * x] + v[2 * y][2 * x + 1]) + (v[2 * y + 1][2 * x] + v[2 * y + 1][2 * x + 1])) * 0.5f;
    rows >>= 1;
    cols >>= 1;
  }
  (void)rows;
  (void)cols;
  const int64_t orow_w = w >> M;   // LL_M row length
  const int64_t o = (b * (h >> M) + r) * orow_w + c * OUT;
#pragma unroll
  for (int x = 0; x < OUT; ++x) {
    if (out64)
      out64[o + x] = double(v[0][x]);
    else
      out32[o + x] = v[0][x];
  }
}

// L >= 4 (h % 32 == 0, w % 64 == 0): levels 1-3 per thread on an 8 x 8 block as above, then
// level 4 (fp64) over 2 x 2 blocks and level 5 over 2 x 2 of those by warp shuffles, in one launch.
// Lane bits: x = (b0, b2, b4), y = (b1, b3) -> a warp covers 32 rows x 64 columns; lanes with equal
// y read 8 consecutive 16-B chunks of a row (128 B).  LF = min(L, 5) levels; L > 5 continues on
// the fp64 chain (lowpass_stage_b) from LL_5.
template <int LF>
__global__ void __launch_bounds__(256) lowpass_bf16_warp(const uint16_t* __restrict__ d, float* __restrict__ out32,
                                                         double* __restrict__ out64, int64_t h, int64_t w,
                                                         int64_t batch) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t wr = h >> 5, wc = w >> 6, total = batch * wr * wc;   // warp tiles of 32 x 64
  if (wid >= total) return;
  const int64_t b = wid / (wr * wc), rem = wid - b * wr * wc;
  const int64_t tr = rem / wc, tc = rem - tr * wc;
  const int x = (lane & 1) | ((lane >> 1) & 2) | ((lane >> 2) & 4);   // bits 0, 2, 4
  const int y = ((lane >> 1) & 1) | ((lane >> 2) & 2);                // bits 1, 3
  const uint16_t* src = d + (b * h + tr * 32 + y * 8) * w + tc * 64 + x * 8;
  uint4 raw[8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(raw[r].x), "=r"(raw[r].y), "=r"(raw[r].z), "=r"(raw[r].w)
                 : "l"(src + int64_t(r) * w));
  float v[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const uint32_t q[4] = {raw[r].x, raw[r].y, raw[r].z, raw[r].w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[r][2 * k] = bf16lo(q[k]);
      v[r][2 * k + 1] = bf16hi(q[k]);
    }
  }
#pragma unroll
  for (int lev = 1; lev <= 3; ++lev)
#pragma unroll
    for (int yy = 0; yy < (8 >> lev); ++yy)
#pragma unroll
      for (int xx = 0; xx < (8 >> lev); ++xx)
        v[yy][xx] = ((v[2 * yy][2 * xx] + v[2 * yy][2 * xx + 1]) + (v[2 * yy + 1][2 * xx] + v[2 * yy + 1][2 * xx + 1])) *
                    0.5f;
  // level 4 (fp64): partners right (lane ^ 1), below (^ 2), diagonal (^ 3)
  double l = double(v[0][0]);
  {
    const double rr = __shfl_xor_sync(0xffffffffu, l, 1), dd = __shfl_xor_sync(0xffffffffu, l, 2),
                 dr = __shfl_xor_sync(0xffffffffu, l, 3);
    l = ((l + rr) + (dd + dr)) * 0.5;
  }
  if constexpr (LF >= 5) {   // level 5: partners lane ^ 4 (right), ^ 8 (below), ^ 12
    const double rr = __shfl_xor_sync(0xffffffffu, l, 4), dd = __shfl_xor_sync(0xffffffffu, l, 8),
                 dr = __shfl_xor_sync(0xffffffffu, l, 12);
    l = ((l + rr) + (dd + dr)) * 0.5;
  }
  const int m = LF == 4 ? 3 : 15;   // lanes holding a result: x0 = y0 = 0 (and x1 = y1 = 0 for LF = 5)
  if ((lane & m) != 0) return;
  const int64_t oc = (tc * 64 >> LF) + (x >> (LF - 3)), orr = (tr * 32 >> LF) + (y >> (LF - 3));
  const int64_t o = (b * (h >> LF) + orr) * (w >> LF) + oc;
  if (out64)
    out64[o] = l;
  else
    out32[o] = float(l);
}

int grid_lp(int64_t total) {   // grid-stride kernels: at most ~64 waves of resident CTAs
  int64_t g = (total + 255) / 256;
  if (g > 148 * 64) g = 148 * 64;
  return int(g < 1 ? 1 : g);
}

int grid_exact(int64_t total) { return int((total + 255) / 256); }

bool env_lowpass_warp() {   // A/B knob (with FHWT_TUNING=1): FHWT_LOWPASS_WARP=0 keeps the two-launch wide path
  if (!tuning_enabled()) return true;
  const char* v = std::getenv("FHWT_LOWPASS_WARP");
  return !(v && *v == '0');
}

}  // namespace

size_t lowpass_bf16_workspace_bytes(int64_t h, int64_t w, int64_t batch, int levels) {
  if (levels <= 3) return 0;
  const int64_t n3 = batch * (h >> 3) * (w >> 3);
  return size_t(n3 + n3 / 4 + 16) * sizeof(double);   // LL_3 chain + one ping-pong partner
}

cudaError_t launch_lowpass_bf16(const uint16_t* d, float* ll, int64_t h, int64_t w, int64_t batch, int levels,
                                void* ws, cudaStream_t s) {
  if (levels >= 4 && h % 32 == 0 && w % 64 == 0) {   // levels 4-5 by warp shuffles, one launch
    const int LF = levels < 5 ? levels : 5;
    double* chain = levels > 5 ? static_cast<double*>(ws) : nullptr;
    float* out_a = levels > 5 ? nullptr : ll;
    const int64_t warps = batch * (h >> 5) * (w >> 6);
    count_launch();
    if (LF == 4)
      lowpass_bf16_warp<4><<<grid_exact(warps * 32), 256, 0, s>>>(d, out_a, chain, h, w, batch);
    else
      lowpass_bf16_warp<5><<<grid_exact(warps * 32), 256, 0, s>>>(d, out_a, chain, h, w, batch);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || levels <= 5) return e;
    const int64_t n5 = batch * (h >> 5) * (w >> 5);
    double* buf[2] = {chain, chain + n5};
    int64_t rows = h >> 5, cols = w >> 5;
    int cur = 0;
    for (int j = 6; j <= levels; ++j) {
      const bool last = j == levels;
      count_launch();
      lowpass_stage_b<<<grid_lp(batch * (rows / 2) * (cols / 2)), 256, 0, s>>>(
          buf[cur], rows, cols, batch, last ? nullptr : buf[cur ^ 1], last ? ll : nullptr);
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      cur ^= 1;
      rows /= 2;
      cols /= 2;
    }
    return cudaSuccess;
  }
  const int M = levels < 3 ? levels : 3;
  const int64_t threads = batch * (h >> M) * (w >> 3);
  double* chain = levels > 3 ? static_cast<double*>(ws) : nullptr;
  float* out_a = levels > 3 ? nullptr : ll;
  count_launch();
  const int g = grid_exact(threads);
  switch (M) {
    case 1: lowpass_stage_a_bf16<1><<<g, 256, 0, s>>>(d, out_a, chain, h, w, batch); break;
    case 2: lowpass_stage_a_bf16<2><<<g, 256, 0, s>>>(d, out_a, chain, h, w, batch); break;
    default: lowpass_stage_a_bf16<3><<<g, 256, 0, s>>>(d, out_a, chain, h, w, batch); break;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || levels <= 3) return e;
  const int64_t n3 = batch * (h >> 3) * (w >> 3);
  double* buf[2] = {chain, chain + n3};
  int64_t rows = h >> 3, cols = w >> 3;
  int cur = 0;
  for (int j = 4; j <= levels; ++j) {   // levels >= 4 in fp64
    const bool last = j == levels;
    const int64_t total = batch * (rows / 2) * (cols / 2);
    count_launch();
    lowpass_stage_b<<<grid_lp(total), 256, 0, s>>>(buf[cur], rows, cols, batch, last ? nullptr : buf[cur ^ 1],
                                                    last ? ll : nullptr);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    cur ^= 1;
    rows /= 2;
    cols /= 2;
  }
  return cudaSuccess;
}

size_t lowpass_workspace_bytes(int64_t h, int64_t w, int64_t batch, int levels) {
  if (levels <= 4) return 0;
  const int64_t n4 = batch * (h >> 4) * (w >> 4);
  return size_t(n4 + n4 / 4 + 16) * sizeof(double);   // LL_4 chain + one ping-pong partner (or the S4 sums)
}

cudaError_t launch_lowpass_u8(const uint8_t* d, float* ll, int64_t h, int64_t w, int64_t batch, int levels, void* ws,
                              cudaStream_t s) {
  const int M = levels < 4 ? levels : 4;
  const int64_t n_a = batch * (h >> M) * (w >> M);
  double* chain = levels > 4 ? static_cast<double*>(ws) : nullptr;
  float* out_a = levels > 4 ? nullptr : ll;
  count_launch();
  if (levels == 5 && h % 32 == 0 && w % 256 == 0 && (reinterpret_cast<uintptr_t>(d) & 15) == 0 &&
      env_lowpass_warp()) {
    count_launch();
    lowpass_u8_warp5<<<grid_exact(batch * (h >> 5) * (w >> 8) * 32), 256, 0, s>>>(d, ll, h, w, batch);
    return cudaGetLastError();
  }
  const int64_t n_wide = batch * (h >> M) * (w >> 4);
  if (w % 16 == 0 && (reinterpret_cast<uintptr_t>(d) & 15) == 0 && (reinterpret_cast<uintptr_t>(ll) & 15) == 0 &&
      n_wide < (int64_t(1) << 31) - 256) {
    const int g = grid_exact(n_wide);
    uint32_t* s4 = levels > 4 ? static_cast<uint32_t*>(ws) : nullptr;
    switch (M) {
      case 1: lowpass_stage_a_wide<1><<<g, 256, 0, s>>>(d, out_a, s4, h, w, batch); break;
      case 2: lowpass_stage_a_wide<2><<<g, 256, 0, s>>>(d, out_a, s4, h, w, batch); break;
      case 3: lowpass_stage_a_wide<3><<<g, 256, 0, s>>>(d, out_a, s4, h, w, batch); break;
      default: lowpass_stage_a_wide<4><<<g, 256, 0, s>>>(d, out_a, s4, h, w, batch); break;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || levels <= 4) return e;
    const int64_t nL = batch * (h >> levels) * (w >> levels);
    count_launch();
    lowpass_stage_b_s4<<<grid_lp(nL), 256, 0, s>>>(s4, h >> 4, w >> 4, batch, levels - 4, levels, ll);
    return cudaGetLastError();
  } else {
    switch (M) {
      case 1: lowpass_stage_a<1><<<grid_lp(n_a), 256, 0, s>>>(d, out_a, chain, h, w, batch); break;
      case 2: lowpass_stage_a<2><<<grid_lp(n_a), 256, 0, s>>>(d, out_a, chain, h, w, batch); break;
      case 3: lowpass_stage_a<3><<<grid_lp(n_a), 256, 0, s>>>(d, out_a, chain, h, w, batch); break;
      default: lowpass_stage_a<4><<<grid_lp(n_a), 256, 0, s>>>(d, out_a, chain, h, w, batch); break;
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || levels <= 4) return e;
  // ping-pong inside the workspace: LL_4 at [0, n4), later levels alternate with [n4, n4 + n4/4)
  const int64_t n4 = n_a;
  double* buf[2] = {chain, chain + n4};
  int64_t rows = h >> 4, cols = w >> 4;
  int cur = 0;
  for (int j = 5; j <= levels; ++j) {
    const bool last = j == levels;
    const int64_t total = batch * (rows / 2) * (cols / 2);
    count_launch();
    lowpass_stage_b<<<grid_lp(total), 256, 0, s>>>(buf[cur], rows, cols, batch, last ? nullptr : buf[cur ^ 1],
                                                    last ? ll : nullptr);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    cur ^= 1;
    rows /= 2;
    cols /= 2;
  }
  return cudaSuccess;
}

}  // namespace fhwt
