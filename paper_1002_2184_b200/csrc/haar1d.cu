// Batched multi-level 1-D Fast Haar analysis / synthesis for sm_100a.
//
// Method: the polyphase Fast Haar analysis bank (§III Fig. 4): d0[k] =
// b00 (x[2k] + x[2k+1]), d1[k] = b00 (x[2k] − x[2k+1]), b00 = 1/√2, iterated on d0 (Mallat,
// SPEC.md:165-173); and the synthesis bank (Eq. (19), Fig. 7):
// x[2k] = a00 (d0 + d1), x[2k+1] = a00 (d0 − d1).
//
// B200 design (K5): one warp owns a 1024-sample chunk, which is
// independent for 10 levels (2-tap support, pairs (2k, 2k+1)).  Lane l loads float4 at
// 128k + 4l (k = 0..7): levels 1-2 pair in-lane; levels 3-5 pair across lanes with
// __shfl_xor_sync after a register exchange that keeps every lane busy — lane l then holds the
// values of index 32q + rotr5(l, m) — so every detail store of a warp is one contiguous segment;
// levels 6-10 run lane-per-index.  HBM traffic: one read and one write per sample.
// Precision: levels 1-3 fp32, levels >= 4 fp64 (SURVEY §8(c) C7 rule), outputs rounded once.
#include <type_traits>

#include "fhwt_internal.cuh"

namespace fhwt {

namespace {

constexpr unsigned kFull = 0xffffffffu;

template <typename T>
__device__ __forceinline__ T S_();
template <>
__device__ __forceinline__ float S_<float>() { return kS32; }
template <>
__device__ __forceinline__ double S_<double>() { return kS64; }

__device__ __forceinline__ int rotr5(int l, int m) { return ((l >> m) | (l << (5 - m))) & 31; }

// 4 consecutive input samples at idx (zero beyond the valid count m)
__device__ __forceinline__ void load4(const float* p, float* x, int idx, int m) {
  if (idx + 3 < m) {
    const float4 v = ldg_stream4(p);
    x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] = (idx + e < m) ? p[e] : 0.f;
  }
}
__device__ __forceinline__ void load4(const float* p, double* x, int idx, int m) {   // fp32 in, fp64 levels
  float t[4];
  load4(p, t, idx, m);
#pragma unroll
  for (int e = 0; e < 4; ++e) x[e] = double(t[e]);
}
__device__ __forceinline__ void load4(const double* p, double* x, int idx, int m) {
  if (idx + 3 < m) {
    const double2 v0 = *reinterpret_cast<const double2*>(p);
    const double2 v1 = *reinterpret_cast<const double2*>(p + 2);
    x[0] = v0.x; x[1] = v0.y; x[2] = v1.x; x[3] = v1.y;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] = (idx + e < m) ? p[e] : 0.0;
  }
}

// Cross-lane analysis level: lane holds K values with index 32k + rotr5(l, M); pairs differ in
// lane bit M.  After the exchange each lane owns whole pairs; outputs have index 32q + rotr5(l, M+1).
template <int K, int M, typename T>
__device__ __forceinline__ void xlevel(const T (&v)[K], T (&a)[K / 2], T (&d)[K / 2], int lane) {
  const bool bit = (lane >> M) & 1;
  const T S = S_<T>();
#pragma unroll
  for (int q = 0; q < K / 2; ++q) {
    const T send = bit ? v[2 * q] : v[2 * q + 1];
    const T r = __shfl_xor_sync(kFull, send, 1 << M);
    const T e = bit ? r : v[2 * q];
    const T o = bit ? v[2 * q + 1] : r;
    a[q] = (e + o) * S;
    d[q] = (e - o) * S;
  }
}

// Inverse of xlevel.
template <int K2, int M, typename T>
__device__ __forceinline__ void xinv(const T (&a)[K2], const T (&d)[K2], T (&v)[2 * K2], int lane) {
  const bool bit = (lane >> M) & 1;
  const T S = S_<T>();
#pragma unroll
  for (int q = 0; q < K2; ++q) {
    const T e = (a[q] + d[q]) * S;
    const T o = (a[q] - d[q]) * S;
    const T r = __shfl_xor_sync(kFull, bit ? e : o, 1 << M);
    v[2 * q] = bit ? r : e;
    v[2 * q + 1] = bit ? o : r;
  }
}

struct Ana1dCtx {
  const Haar1dParams* p;
  float* crow;      // coefficient row of this signal
  int64_t b, c;     // signal, chunk
  int m;            // valid input samples in this chunk
  __device__ __forceinline__ float* detail(int j) const {
    return crow + (p->n >> (p->g0 + j)) + c * (kChunk1d >> j);
  }
  template <typename T>
  __device__ __forceinline__ void put_detail(int j, int i, T v) const {
    if (i < (m >> j)) stg_stream1(detail(j) + i, float(v));
  }
  template <typename T>
  __device__ __forceinline__ void put_approx(int i, T v) const {
    const int j = p->Lp;
    if (i >= (m >> j)) return;
    if (p->final_pass)
      stg_stream1(crow + c * (kChunk1d >> j) + i, float(v));
    else
      static_cast<double*>(p->out)[b * p->out_pitch + c * (kChunk1d >> j) + i] = double(v);
  }
};

// Coarse levels 11..10+T of the signals a CTA holds whole (p.tail = T; chunks = 1024-sample chunks
// per signal divides the CTA's 8 warps): thread s < 8 / chunks takes signal s of the CTA from the
// chunks' fp64 LL10 values in shared memory.  Same operations, in the same order, as the fp64
// second pass (ana1d_kernel<double>): bitwise equal results.
__device__ __forceinline__ void ana1d_tail(const Haar1dParams& p, const double* ll10, int64_t cta_w0) {
  const int per = int(p.chunks), nsig = (kThreads1d / 32) / per;
  const int s = threadIdx.x;
  if (s >= nsig) return;
  const int64_t b = cta_w0 / per + s;
  float* crow = p.coeffs_out + b * p.n;
  double v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = k < per ? ll10[s * per + k] : 0.0;
  int m = per;
#pragma unroll
  for (int t = 1; t <= 3; ++t) {
    if (t > p.tail) break;
    const int j = 10 + t;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (2 * k + 1 >= m) break;
      const double e = v[2 * k], o = v[2 * k + 1];
      stg_stream1(crow + (p.n >> j) + k, float((e - o) * kS64));
      v[k] = (e + o) * kS64;
    }
    m >>= 1;
  }
  for (int k = 0; k < m; ++k) stg_stream1(crow + k, float(v[k]));
}

// F64ALL: levels 1..3 in fp64 as well (decompositions deeper than 10 levels, reading R14: the
// fp32 rounding of levels 1-3 grows by up to sqrt(2) per further level, 2^(J/2 - 1.5) x at level J).
template <typename TIn, bool F64ALL = false>
__global__ void __launch_bounds__(kThreads1d) ana1d_kernel(const __grid_constant__ Haar1dParams p) {
  using T1 = typename std::conditional<F64ALL, double, TIn>::type;  // levels 1..3; levels >= 4 are fp64
  __shared__ double tail_ll[kThreads1d / 32];
  const int lane = threadIdx.x & 31;
  const int64_t w = int64_t(blockIdx.x) * (kThreads1d / 32) + (threadIdx.x >> 5);
  if (w >= p.nwarps) return;  // warp-uniform (with p.tail, nwarps is a multiple of the CTA's warps)
  Ana1dCtx ctx;
  ctx.p = &p;
  ctx.b = w / p.chunks;
  ctx.c = w - ctx.b * p.chunks;
  const int64_t base = ctx.c * kChunk1d;
  ctx.m = int(min(int64_t(kChunk1d), p.nin - base));
  ctx.crow = p.coeffs_out + ctx.b * p.n;
  const TIn* src = static_cast<const TIn*>(p.in) + ctx.b * p.in_pitch + base;
  const int Lp = p.Lp;

  T1 x[32];
#pragma unroll
  for (int k = 0; k < 8; ++k) load4(src + 128 * k + 4 * lane, x + 4 * k, 128 * k + 4 * lane, ctx.m);

  const T1 S1 = S_<T1>();
  // ---- level 1 (in-lane): index 64k + 2l + e
  T1 a1[16];
  {
    const int mv = ctx.m >> 1;
    float* dp = ctx.detail(1);
    const bool al = (reinterpret_cast<uintptr_t>(dp) & 7) == 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      T1 dd[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const T1 xe = x[4 * k + 2 * e], xo = x[4 * k + 2 * e + 1];
        a1[2 * k + e] = (xe + xo) * S1;
        dd[e] = (xe - xo) * S1;
      }
      const int i = 64 * k + 2 * lane;
      if (al && i + 1 < mv) {
        stg_stream2(dp + i, make_float2(float(dd[0]), float(dd[1])));
      } else {
        if (i < mv) stg_stream1(dp + i, float(dd[0]));
        if (i + 1 < mv) stg_stream1(dp + i + 1, float(dd[1]));
      }
    }
    if (Lp == 1) {
      float* ap = ctx.crow + ctx.c * (kChunk1d >> 1);
      const bool aal = p.final_pass && (reinterpret_cast<uintptr_t>(ap) & 7) == 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = 64 * k + 2 * lane;
        if (aal && i + 1 < mv) {
          stg_stream2(ap + i, make_float2(float(a1[2 * k]), float(a1[2 * k + 1])));
        } else {
          ctx.put_approx(i, a1[2 * k]);
          ctx.put_approx(i + 1, a1[2 * k + 1]);
        }
      }
      return;
    }
  }
  // ---- level 2 (in-lane): index 32k + l
  T1 a2[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const T1 e = a1[2 * k], o = a1[2 * k + 1];
    a2[k] = (e + o) * S1;
    ctx.put_detail(2, 32 * k + lane, (e - o) * S1);
  }
  if (Lp == 2) {
#pragma unroll
    for (int k = 0; k < 8; ++k) ctx.put_approx(32 * k + lane, a2[k]);
    return;
  }
  // ---- level 3 (cross-lane, bit 0): index 32q + rotr5(l, 1)
  T1 a3[4], d3[4];
  xlevel<8, 0>(a2, a3, d3, lane);
  {
    const int r1 = rotr5(lane, 1);
#pragma unroll
    for (int q = 0; q < 4; ++q) ctx.put_detail(3, 32 * q + r1, d3[q]);
    if (Lp == 3) {
#pragma unroll
      for (int q = 0; q < 4; ++q) ctx.put_approx(32 * q + r1, a3[q]);
      return;
    }
  }
  // ---- level 4 (fp64 from here on), bit 1
  double v3[4], a4[2], d4[2];
#pragma unroll
  for (int q = 0; q < 4; ++q) v3[q] = double(a3[q]);
  xlevel<4, 1>(v3, a4, d4, lane);
  {
    const int r2 = rotr5(lane, 2);
#pragma unroll
    for (int q = 0; q < 2; ++q) ctx.put_detail(4, 32 * q + r2, d4[q]);
    if (Lp == 4) {
#pragma unroll
      for (int q = 0; q < 2; ++q) ctx.put_approx(32 * q + r2, a4[q]);
      return;
    }
  }
  // ---- level 5, bit 2: one value per lane, index rotr5(l, 3)
  double a5[1], d5[1];
  xlevel<2, 2>(a4, a5, d5, lane);
  const int r3 = rotr5(lane, 3);
  ctx.put_detail(5, r3, d5[0]);
  if (Lp == 5) {
    ctx.put_approx(r3, a5[0]);
    return;
  }
  // ---- levels 6..10: lane-per-index (lane l holds index l after an inverse rotation)
  double v = __shfl_sync(kFull, a5[0], ((lane << 3) | (lane >> 2)) & 31);
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const int j = 6 + t;
    const double pv = __shfl_xor_sync(kFull, v, 1 << t);
    const bool act = (lane & ((2 << t) - 1)) == 0;
    const double a = (v + pv) * kS64;
    const int i = lane >> (t + 1);
    if (act) ctx.put_detail(j, i, (v - pv) * kS64);
    v = a;
    if (j == Lp) {
      if constexpr (sizeof(TIn) == 4) {
        if (p.tail > 0) {   // Lp = 10: lane 0 holds the chunk's LL10
          if (lane == 0) tail_ll[threadIdx.x >> 5] = a;
          __syncthreads();
          ana1d_tail(p, tail_ll, int64_t(blockIdx.x) * (kThreads1d / 32));
          return;
        }
      }
      if (act) ctx.put_approx(i, a);
      return;
    }
  }
}

// -------------------------------------------------------------------------------- synthesis
struct Syn1dCtx {
  const Haar1dParams* p;
  const float* crow;
  int64_t b, c;
  int m;  // valid output samples in this chunk
  __device__ __forceinline__ const float* detail(int j) const {
    return crow + (p->n >> (p->g0 + j)) + c * (kChunk1d >> j);
  }
  __device__ __forceinline__ float ld(const float* ptr, int i, int j) const {
    return i < (m >> j) ? ldg_stream1(ptr + i) : 0.f;
  }
};

// Inverse of ana1d_tail: thread s rebuilds the fp32 LL10 values of signal s of the CTA from a_J and
// the details of levels J..11 (same operations as the fp32 coarse pass of syn1d_kernel).
__device__ __forceinline__ void syn1d_tail(const Haar1dParams& p, float* ll10, int64_t cta_w0) {
  const int per = int(p.chunks), nsig = (kThreads1d / 32) / per;
  const int s = threadIdx.x;
  if (s >= nsig) return;
  const int64_t b = cta_w0 / per + s;
  const float* crow = p.coeffs_in + b * p.n;
  float v[8];
  int m = per >> p.tail;
  for (int k = 0; k < m; ++k) v[k] = crow[k];
#pragma unroll
  for (int t = 3; t >= 1; --t) {
    if (t > p.tail) continue;
    const int j = 10 + t;
#pragma unroll
    for (int k = 3; k >= 0; --k) {
      if (k >= m) continue;
      const float a = v[k], d = crow[(p.n >> j) + k];
      v[2 * k] = (a + d) * kS32;
      v[2 * k + 1] = (a - d) * kS32;
    }
    m <<= 1;
  }
  for (int k = 0; k < per; ++k) ll10[s * per + k] = v[k];
}

// At least 3 resident CTAs (768 threads) per SM: the kernel waits on its chunk's loads (long
// scoreboard, profiles/r01_sass_hotspots.md), so occupancy is what keeps loads in flight; measured
// c2 synthesis 6711 -> 6916 GB/s, every 1-D shape +1.5-5 % (alternating processes).
__global__ void __launch_bounds__(kThreads1d, 3) syn1d_kernel(const __grid_constant__ Haar1dParams p) {
  __shared__ float tail_ll[kThreads1d / 32];
  const int lane = threadIdx.x & 31;
  const int64_t w = int64_t(blockIdx.x) * (kThreads1d / 32) + (threadIdx.x >> 5);
  if (w >= p.nwarps) return;   // with p.tail, nwarps is a multiple of the CTA's warps
  Syn1dCtx ctx;
  ctx.p = &p;
  ctx.b = w / p.chunks;
  ctx.c = w - ctx.b * p.chunks;
  const int64_t base = ctx.c * kChunk1d;
  ctx.m = int(min(int64_t(kChunk1d), p.nin - base));
  ctx.crow = p.coeffs_in + ctx.b * p.n;
  const int Lp = p.Lp;
  const float* ap = static_cast<const float*>(p.in) + ctx.b * p.in_pitch + ctx.c * (kChunk1d >> Lp);
  const float S = kS32;

  // ---- issue every coefficient load of the chunk first (memory-level parallelism)
  float d1[16], d2[8], d3[4], d4[2], d5 = 0.f, dh[5];
  {
    const float* dp = ctx.detail(1);
    const int mv = ctx.m >> 1;
    const bool al = (reinterpret_cast<uintptr_t>(dp) & 7) == 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = 64 * k + 2 * lane;
      if (al && i + 1 < mv) {
        const float2 t = ldg_stream2(dp + i);
        d1[2 * k] = t.x;
        d1[2 * k + 1] = t.y;
      } else {
        d1[2 * k] = i < mv ? dp[i] : 0.f;
        d1[2 * k + 1] = i + 1 < mv ? dp[i + 1] : 0.f;
      }
    }
  }
  if (Lp >= 2) {
#pragma unroll
    for (int k = 0; k < 8; ++k) d2[k] = ctx.ld(ctx.detail(2), 32 * k + lane, 2);
  }
  if (Lp >= 3) {
#pragma unroll
    for (int q = 0; q < 4; ++q) d3[q] = ctx.ld(ctx.detail(3), 32 * q + rotr5(lane, 1), 3);
  }
  if (Lp >= 4) {
#pragma unroll
    for (int q = 0; q < 2; ++q) d4[q] = ctx.ld(ctx.detail(4), 32 * q + rotr5(lane, 2), 4);
  }
  if (Lp >= 5) d5 = ctx.ld(ctx.detail(5), rotr5(lane, 3), 5);
#pragma unroll
  for (int t = 0; t < 5; ++t) dh[t] = (Lp >= 6 + t) ? ctx.ld(ctx.detail(6 + t), lane >> (t + 1), 6 + t) : 0.f;

  if (p.tail > 0) {   // Lp = 10: this chunk's LL10 comes from the CTA's coarse levels
    syn1d_tail(p, tail_ll, int64_t(blockIdx.x) * (kThreads1d / 32));
    __syncthreads();
  }
  auto lda = [&](int i) -> float {
    if (p.tail > 0) return tail_ll[threadIdx.x >> 5];
    return i < (ctx.m >> Lp) ? ldg_stream1(ap + i) : 0.f;
  };

  // ---- coarse levels
  float a2[8];
  if (Lp >= 3) {
    float a3[4];
    if (Lp >= 4) {
      float a4[2];
      if (Lp >= 5) {
        float a5[1];
        if (Lp >= 6) {
          // lane-per-index levels Lp..6: lane l ends with a_5[l]
          float v = lda(lane >> (Lp - 5));
#pragma unroll
          for (int t = 4; t >= 0; --t) {
            if (6 + t > Lp) continue;
            const float e = (v + dh[t]) * S, o = (v - dh[t]) * S;
            v = ((lane >> t) & 1) ? o : e;
          }
          a5[0] = __shfl_sync(kFull, v, rotr5(lane, 3));
        } else {
          a5[0] = lda(rotr5(lane, 3));
        }
        const float dd5[1] = {d5};
        xinv<1, 2>(a5, dd5, a4, lane);
      } else {
#pragma unroll
        for (int q = 0; q < 2; ++q) a4[q] = lda(32 * q + rotr5(lane, 2));
      }
      xinv<2, 1>(a4, d4, a3, lane);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) a3[q] = lda(32 * q + rotr5(lane, 1));
    }
    xinv<4, 0>(a3, d3, a2, lane);
  } else if (Lp == 2) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a2[k] = lda(32 * k + lane);
  }
  // ---- level 2 (in-lane) -> a1 at 64k + 2l + e
  float a1[16];
  if (Lp >= 2) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a1[2 * k] = (a2[k] + d2[k]) * S;
      a1[2 * k + 1] = (a2[k] - d2[k]) * S;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a1[2 * k] = lda(64 * k + 2 * lane);
      a1[2 * k + 1] = lda(64 * k + 2 * lane + 1);
    }
  }
  // ---- level 1 (in-lane) -> output float4 at 128k + 4l
  float* out = static_cast<float*>(p.out) + ctx.b * p.out_pitch + base;
  const bool oal = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float y[4];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      y[2 * e] = (a1[2 * k + e] + d1[2 * k + e]) * S;
      y[2 * e + 1] = (a1[2 * k + e] - d1[2 * k + e]) * S;
    }
    const int i = 128 * k + 4 * lane;
    if (oal && i + 3 < ctx.m) {
      stg_stream4(out + i, make_float4(y[0], y[1], y[2], y[3]));
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (i + e < ctx.m) stg_stream1(out + i + e, y[e]);
    }
  }
}

// ------------------------------------------------------------------ single-level scalar kernels
// For n % 4 != 0 (then levels == 1): one thread per pair, no vector access.
__global__ void ana1d_l1_scalar_kernel(const float* __restrict__ d, float* __restrict__ c, int64_t n, int64_t batch) {
  const int64_t half = n / 2, total = batch * half;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / half, k = i - b * half;
    const float xe = d[b * n + 2 * k], xo = d[b * n + 2 * k + 1];
    c[b * n + k] = (xe + xo) * kS32;
    c[b * n + half + k] = (xe - xo) * kS32;
  }
}

__global__ void syn1d_l1_scalar_kernel(const float* __restrict__ c, float* __restrict__ d, int64_t n, int64_t batch) {
  const int64_t half = n / 2, total = batch * half;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / half, k = i - b * half;
    const float a = c[b * n + k], dd = c[b * n + half + k];
    d[b * n + 2 * k] = (a + dd) * kS32;
    d[b * n + 2 * k + 1] = (a - dd) * kS32;
  }
}

int grid1(int64_t total) {
  int64_t g = (total + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  return int(g < 1 ? 1 : g);
}

}  // namespace

cudaError_t launch_ana1d(const Haar1dParams& p, bool in_f64, cudaStream_t s, bool f64all) {
  const int64_t blocks = (p.nwarps + (kThreads1d / 32) - 1) / (kThreads1d / 32);
  count_launch();
  if (in_f64)
    ana1d_kernel<double><<<unsigned(blocks), kThreads1d, 0, s>>>(p);
  else if (f64all)
    ana1d_kernel<float, true><<<unsigned(blocks), kThreads1d, 0, s>>>(p);
  else
    ana1d_kernel<float><<<unsigned(blocks), kThreads1d, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_syn1d(const Haar1dParams& p, cudaStream_t s) {
  const int64_t blocks = (p.nwarps + (kThreads1d / 32) - 1) / (kThreads1d / 32);
  count_launch();
  syn1d_kernel<<<unsigned(blocks), kThreads1d, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_ana1d_l1_scalar(const float* d, float* c, int64_t n, int64_t batch, cudaStream_t s) {
  count_launch();
  ana1d_l1_scalar_kernel<<<grid1(batch * (n / 2)), 256, 0, s>>>(d, c, n, batch);
  return cudaGetLastError();
}

cudaError_t launch_syn1d_l1_scalar(const float* c, float* d, int64_t n, int64_t batch, cudaStream_t s) {
  count_launch();
  syn1d_l1_scalar_kernel<<<grid1(batch * (n / 2)), 256, 0, s>>>(c, d, n, batch);
  return cudaGetLastError();
}

}  // namespace fhwt
