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
// (image, row, column) of unit u = (gi * h2 + r) * w2 + c.  POW2: h2 and w2 are powers of two
// (shifts instead of integer divisions, which dominated these kernels' issue slots).
template <bool POW2>
__device__ __forceinline__ void unit_rc(uint32_t u, uint32_t per, uint32_t w2, uint32_t& gi, uint32_t& rem,
                                        uint32_t& r, uint32_t& c) {
  if constexpr (POW2) {
    gi = u >> (__ffs(per) - 1);
    rem = u & (per - 1);
    r = rem >> (__ffs(w2) - 1);
    c = rem & (w2 - 1);
  } else {
    gi = u / per;
    rem = u - gi * per;
    r = rem / w2;
    c = rem - r * w2;
  }
}

template <typename TS, typename TD, bool POW2>
__device__ __forceinline__ void small_ana_level_t(const Small2dParams& p, const TS* src, int sp, int ss, float* O,
                                                  TD* dst, int g, int h, int w, bool last) {
  const int h2 = h >> 1, w2 = w >> 1;
  const uint32_t per = uint32_t(h2 * w2), total = per * uint32_t(g);
  const int imgO = p.H * p.W;
  for (uint32_t u = threadIdx.x; u < total; u += blockDim.x) {
    uint32_t gi, rem, r, c;
    unit_rc<POW2>(u, per, uint32_t(w2), gi, rem, r, c);
    const TS* s = src + gi * ss + (2 * r) * sp + 2 * c;   // even offset: pairs load as one 8/16-B word
    TD a, bb, cc, d;
    if constexpr (sizeof(TS) == 4) {
      const float2 r0 = *reinterpret_cast<const float2*>(s), r1 = *reinterpret_cast<const float2*>(s + sp);
      a = TD(r0.x); bb = TD(r0.y); cc = TD(r1.x); d = TD(r1.y);
    } else {
      const double2 r0 = *reinterpret_cast<const double2*>(s), r1 = *reinterpret_cast<const double2*>(s + sp);
      a = r0.x; bb = r0.y; cc = r1.x; d = r1.y;
    }
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

template <typename TS, typename TD>
__device__ __forceinline__ void small_ana_level(const Small2dParams& p, const TS* src, int sp, int ss, float* O,
                                                TD* dst, int g, int h, int w, bool last) {
  // measured (tools/generic_shapes.py SMALL=1): shifts win for L >= 4 (32x32 L=5 4.77 -> 5.74 TB/s,
  // 64x64 L=6 4.48 -> 6.14, 16x64 L=4 5.20 -> 5.43) and lose at L = 3 (64x64 5.71 -> 5.48)
  if (p.L >= 4 && ((h & (h - 1)) | (w & (w - 1))) == 0)
    small_ana_level_t<TS, TD, true>(p, src, sp, ss, O, dst, g, h, w, last);
  else
    small_ana_level_t<TS, TD, false>(p, src, sp, ss, O, dst, g, h, w, last);
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
template <bool POW2>
__device__ __forceinline__ void small_syn_level_t(const Small2dParams& p, const float* ll, int lp, int ls,
                                                  const float* S, float* dst, int dp, int ds, int g, int h, int w) {
  const int h2 = h >> 1, w2 = w >> 1;
  const uint32_t per = uint32_t(h2 * w2), total = per * uint32_t(g);
  const int imgS = p.H * p.W;
  for (uint32_t u = threadIdx.x; u < total; u += blockDim.x) {
    uint32_t gi, rem, r, c;
    unit_rc<POW2>(u, per, uint32_t(w2), gi, rem, r, c);
    const float* b = S + gi * imgS + r * p.W + c;
    const float vll = ll[gi * ls + r * lp + c], vhl = b[w2], vlh = b[h2 * p.W], vhh = b[h2 * p.W + w2];
    const float s = vll + vlh, t = vhl + vhh, s2 = vll - vlh, t2 = vhl - vhh;
    float* o = dst + gi * ds + (2 * r) * dp + 2 * c;   // even offset: one 8-B store per output row
    *reinterpret_cast<float2*>(o) = make_float2((s + t) * 0.5f, (s - t) * 0.5f);
    *reinterpret_cast<float2*>(o + dp) = make_float2((s2 + t2) * 0.5f, (s2 - t2) * 0.5f);
  }
}

__device__ __forceinline__ void small_syn_level(const Small2dParams& p, const float* ll, int lp, int ls,
                                                const float* S, float* dst, int dp, int ds, int g, int h, int w) {
  // measured: shifts win for L >= 5 (32x32 L=5 5.23 -> 5.79 TB/s, 64x64 L=6 5.01 -> 5.83) and lose
  // at L = 3, 4 (64x64 L=3 6.20 -> 5.66, 16x64 L=4 5.76 -> 5.60)
  if (p.L >= 5 && ((h & (h - 1)) | (w & (w - 1))) == 0)
    small_syn_level_t<true>(p, ll, lp, ls, S, dst, dp, ds, g, h, w);
  else
    small_syn_level_t<false>(p, ll, lp, ls, S, dst, dp, ds, g, h, w);
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

// ------------------------------------------------------------------ 1-D: batches of short signals
// Same chunk machinery for signals shorter than the 1024-sample warp chunk of haar1d.cu (which
// would leave most of a warp idle): G signals of n samples per chunk (H = 1, W = n in the params).
// Levels run in passes of up to three: one thread takes 2^K consecutive values of a signal, does
// K levels in registers, and writes each level's details as one contiguous run, so only the pass
// boundaries go through the approximation buffers.  Arithmetic exactly as haar1d.cu:
// (x_e ± x_o) * fl(1/√2) in fp32 for levels 1-3, in fp64 with the fp64 constant from level 4
// (analysis); synthesis in fp32.  Needs n % 2^min(3, J) == 0 (host check).
template <typename T>
__device__ __forceinline__ T sq();
template <>
__device__ __forceinline__ float sq<float>() { return kS32; }
template <>
__device__ __forceinline__ double sq<double>() { return kS64; }

// Analysis levels g0+1..g0+K of g signals: source a_{g0} (length m per signal, stride ss, type TS),
// details into the output chunk O (row pitch W), a_{g0+K} into dst (compact) or O (last pass).
template <int K, typename TS, typename TC>
__device__ __forceinline__ void small1d_ana_pass(const Small2dParams& p, const TS* src, int ss, float* O, TC* dst,
                                                 int g, int m, int g0, bool last) {
  constexpr int U = 1 << K;
  const int upr = m >> K;
  const uint32_t total = uint32_t(upr) * uint32_t(g);
  const TC S = sq<TC>();
  for (uint32_t u = threadIdx.x; u < total; u += blockDim.x) {
    const uint32_t gi = u / uint32_t(upr), t = u - gi * uint32_t(upr);
    TC v[U];
    const TS* sp = src + gi * ss + t * U;
    if constexpr (U == 8 && sizeof(TS) == 4) {
      if ((ss & 3) == 0) {   // 16-B aligned rows: two float4 loads, halves swapped on lanes 4-7 of
                             // each quarter-warp so every phase covers all 32 banks
        const bool sw = (threadIdx.x >> 2) & 1;
        const float4 x0 = *reinterpret_cast<const float4*>(sp + (sw ? 4 : 0));
        const float4 x1 = *reinterpret_cast<const float4*>(sp + (sw ? 0 : 4));
        const float4 lo = sw ? x1 : x0, hi = sw ? x0 : x1;
        v[0] = TC(lo.x); v[1] = TC(lo.y); v[2] = TC(lo.z); v[3] = TC(lo.w);
        v[4] = TC(hi.x); v[5] = TC(hi.y); v[6] = TC(hi.z); v[7] = TC(hi.w);
      } else {
#pragma unroll
        for (int e = 0; e < U; ++e) v[e] = TC(sp[e]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < U; ++e) v[e] = TC(sp[e]);
    }
    float* row = O + gi * p.W;
#pragma unroll
    for (int i = 1; i <= K; ++i) {   // level g0 + i: U >> i outputs
      float* dp = row + (p.W >> (g0 + i)) + t * (U >> i);
#pragma unroll
      for (int e = 0; e < (U >> i); ++e) {
        const TC a = v[2 * e], b = v[2 * e + 1];
        dp[e] = float((a - b) * S);
        v[e] = (a + b) * S;
      }
    }
    if (last)
      row[t] = float(v[0]);
    else
      dst[u] = v[0];
  }
}

// Synthesis levels lo+K-1 .. lo of g signals: a_{lo+K-1} (stride ls) and the details of those
// levels from the coefficient chunk S -> a_{lo-1} (mout per signal) into dst (stride ds).
template <int K>
__device__ __forceinline__ void small1d_syn_pass(const Small2dParams& p, const float* asrc, int ls, const float* S,
                                                 float* dst, int ds, int g, int mout, int lo) {
  constexpr int U = 1 << K;
  const int upr = mout >> K;
  const uint32_t total = uint32_t(upr) * uint32_t(g);
  for (uint32_t u = threadIdx.x; u < total; u += blockDim.x) {
    const uint32_t gi = u / uint32_t(upr), t = u - gi * uint32_t(upr);
    const float* row = S + gi * p.W;
    float v[U];
    v[0] = asrc[gi * ls + t];
#pragma unroll
    for (int i = K; i >= 1; --i) {   // level lo + i - 1: (U >> i) values -> twice as many
      const float* dp = row + (p.W >> (lo + i - 1)) + t * (U >> i);
#pragma unroll
      for (int e = (U >> i) - 1; e >= 0; --e) {
        const float a = v[e], d = dp[e];
        v[2 * e] = (a + d) * kS32;
        v[2 * e + 1] = (a - d) * kS32;
      }
    }
    float* op = dst + gi * ds + t * U;
    if (U == 8 && (ds & 3) == 0) {   // two float4 stores, halves swapped as in the analysis loads
      const bool sw = (threadIdx.x >> 2) & 1;
      const float4 lo = make_float4(v[0], v[1], v[2], v[3]), hi = make_float4(v[4 % U], v[5 % U], v[6 % U], v[7 % U]);
      *reinterpret_cast<float4*>(op + (sw ? 4 : 0)) = sw ? hi : lo;
      *reinterpret_cast<float4*>(op + (sw ? 0 : 4)) = sw ? lo : hi;
    } else {
#pragma unroll
      for (int e = 0; e < U; ++e) op[e] = v[e];
    }
  }
}

__global__ void __launch_bounds__(256, 2) ana1d_small_kernel(const __grid_constant__ Small2dParams p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  float* O = reinterpret_cast<float*>(smem + p.off_out);
  float* const A3 = reinterpret_cast<float*>(smem + p.off_t[0]);    // a_3 (fp32, n/8 per signal)
  double* const A6 = reinterpret_cast<double*>(smem + p.off_d[0]);  // a_6 (fp64, n/64 per signal)
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
  const int n = p.W, J = p.L;
  for (int64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x, ++it) {
    const int s = it % p.stages;
    mbar_wait(&bars[s], uint32_t(it / p.stages) & 1u);
    if (tid == 0) bulk_wait_read();   // the previous chunk's store has read O
    __syncthreads();
    const Chunk k = chunk_of(p, c);
    const float* S = reinterpret_cast<const float*>(smem + s * p.stage_bytes);
    // pass 1: levels 1..min(3, J), fp32, from the stage
    if (J == 1) small1d_ana_pass<1, float, float>(p, S, n, O, A3, k.g, n, 0, true);
    else if (J == 2) small1d_ana_pass<2, float, float>(p, S, n, O, A3, k.g, n, 0, true);
    else small1d_ana_pass<3, float, float>(p, S, n, O, A3, k.g, n, 0, J == 3);
    __syncthreads();
    if (tid == 0) {   // the stage is free: refill it
      const int64_t nc = c + int64_t(p.stages) * gridDim.x;
      if (nc < p.nchunks) issue_chunk(p, p.in, smem + s * p.stage_bytes, &bars[s], nc);
    }
    if (J > 3) {   // pass 2: levels 4..min(6, J), fp64, from a_3
      if (J == 4) small1d_ana_pass<1, float, double>(p, A3, n >> 3, O, A6, k.g, n >> 3, 3, true);
      else if (J == 5) small1d_ana_pass<2, float, double>(p, A3, n >> 3, O, A6, k.g, n >> 3, 3, true);
      else small1d_ana_pass<3, float, double>(p, A3, n >> 3, O, A6, k.g, n >> 3, 3, J == 6);
      __syncthreads();
    }
    if (J > 6) {   // pass 3: levels 7..J (J <= 9 for n < 1024), fp64, from a_6
      double* none = nullptr;
      if (J == 7) small1d_ana_pass<1, double, double>(p, A6, n >> 6, O, none, k.g, n >> 6, 6, true);
      else if (J == 8) small1d_ana_pass<2, double, double>(p, A6, n >> 6, O, none, k.g, n >> 6, 6, true);
      else small1d_ana_pass<3, double, double>(p, A6, n >> 6, O, none, k.g, n >> 6, 6, true);
      __syncthreads();
    }
    fence_proxy_async();   // O's generic-proxy writes -> the bulk store (async proxy)
    __syncthreads();
    if (tid == 0) bulk_store(p.out + k.first * int64_t(n), O, uint32_t(k.g) * uint32_t(n) * 4u);
  }
  if (tid == 0) bulk_wait_all();
}

__global__ void __launch_bounds__(256, 2) syn1d_small_kernel(const __grid_constant__ Small2dParams p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  float* O = reinterpret_cast<float*>(smem + p.off_out);
  float* const A3 = reinterpret_cast<float*>(smem + p.off_t[0]);   // a_3 (n/8 per signal)
  float* const A6 = reinterpret_cast<float*>(smem + p.off_t[1]);   // a_6 (n/64 per signal)
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
  const int n = p.W, J = p.L;
  for (int64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x, ++it) {
    const int s = it % p.stages;
    mbar_wait(&bars[s], uint32_t(it / p.stages) & 1u);
    const Chunk k = chunk_of(p, c);
    const float* S = reinterpret_cast<const float*>(smem + s * p.stage_bytes);
    const float* a = S;   // a_J: the first n >> J values of each coefficient row (stride n)
    int ls = n;
    if (J > 6) {   // levels J..7 -> a_6
      if (J == 7) small1d_syn_pass<1>(p, a, ls, S, A6, n >> 6, k.g, n >> 6, 7);
      else if (J == 8) small1d_syn_pass<2>(p, a, ls, S, A6, n >> 6, k.g, n >> 6, 7);
      else small1d_syn_pass<3>(p, a, ls, S, A6, n >> 6, k.g, n >> 6, 7);
      __syncthreads();
      a = A6;
      ls = n >> 6;
    }
    if (J > 3) {   // levels min(J, 6)..4 -> a_3
      if (J == 4) small1d_syn_pass<1>(p, a, ls, S, A3, n >> 3, k.g, n >> 3, 4);
      else if (J == 5) small1d_syn_pass<2>(p, a, ls, S, A3, n >> 3, k.g, n >> 3, 4);
      else small1d_syn_pass<3>(p, a, ls, S, A3, n >> 3, k.g, n >> 3, 4);
      __syncthreads();
      a = A3;
      ls = n >> 3;
    }
    if (tid == 0) bulk_wait_read();   // the previous chunk's store has read O
    __syncthreads();
    if (J == 1) small1d_syn_pass<1>(p, a, ls, S, O, n, k.g, n, 1);   // levels min(J, 3)..1 -> d_R
    else if (J == 2) small1d_syn_pass<2>(p, a, ls, S, O, n, k.g, n, 1);
    else small1d_syn_pass<3>(p, a, ls, S, O, n, k.g, n, 1);
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      bulk_store(p.out + k.first * int64_t(n), O, uint32_t(k.g) * uint32_t(n) * 4u);
      const int64_t nc = c + int64_t(p.stages) * gridDim.x;
      if (nc < p.nchunks) issue_chunk(p, p.in, smem + s * p.stage_bytes, &bars[s], nc);
    }
  }
  if (tid == 0) bulk_wait_all();
}

}  // namespace

static const void* small_fn(bool analysis, bool one_d) {
  if (one_d) return analysis ? (const void*)ana1d_small_kernel : (const void*)syn1d_small_kernel;
  return analysis ? (const void*)ana2d_small_kernel : (const void*)syn2d_small_kernel;
}

cudaError_t small2d_occupancy(bool analysis, size_t smem, int* blocks_per_sm, bool one_d) {
  const void* fn = small_fn(analysis, one_d);
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fn, 256, smem);
}

cudaError_t launch_small2d(const Small2dParams& p, bool analysis, int grid, size_t smem, cudaStream_t s, bool one_d) {
  count_launch();
  void* args[] = {const_cast<Small2dParams*>(&p)};
  return cudaLaunchKernel(small_fn(analysis, one_d), dim3(grid), dim3(256), args, smem, s);
}

}  // namespace fhwt
