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
__device__ __forceinline__ void unpack_row(const uint8_t* p, float (&v)[1 << M]) {
  using T = typename RowVec<M>::T;
  const T t = __ldg(reinterpret_cast<const T*>(p));
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
    // level 1 on row pairs as they arrive
    float l1[N / 2][N / 2];
#pragma unroll
    for (int y = 0; y < N; y += 2) {
      float r0[N], r1[N];
      unpack_row<M>(src + int64_t(y) * w, r0);
      unpack_row<M>(src + int64_t(y + 1) * w, r1);
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

int grid_lp(int64_t total) {
  int64_t g = (total + 255) / 256;
  if (g > 148 * 64) g = 148 * 64;
  return int(g < 1 ? 1 : g);
}

}  // namespace

size_t lowpass_workspace_bytes(int64_t h, int64_t w, int64_t batch, int levels) {
  if (levels <= 4) return 0;
  const int64_t n4 = batch * (h >> 4) * (w >> 4);
  return size_t(n4 + n4 / 4 + 16) * sizeof(double);   // LL_4 chain + one ping-pong partner
}

cudaError_t launch_lowpass_u8(const uint8_t* d, float* ll, int64_t h, int64_t w, int64_t batch, int levels, void* ws,
                              cudaStream_t s) {
  const int M = levels < 4 ? levels : 4;
  const int64_t n_a = batch * (h >> M) * (w >> M);
  double* chain = levels > 4 ? static_cast<double*>(ws) : nullptr;
  float* out_a = levels > 4 ? nullptr : ll;
  count_launch();
  switch (M) {
    case 1: lowpass_stage_a<1><<<grid_lp(n_a), 256, 0, s>>>(d, out_a, chain, h, w, batch); break;
    case 2: lowpass_stage_a<2><<<grid_lp(n_a), 256, 0, s>>>(d, out_a, chain, h, w, batch); break;
    case 3: lowpass_stage_a<3><<<grid_lp(n_a), 256, 0, s>>>(d, out_a, chain, h, w, batch); break;
    default: lowpass_stage_a<4><<<grid_lp(n_a), 256, 0, s>>>(d, out_a, chain, h, w, batch); break;
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
