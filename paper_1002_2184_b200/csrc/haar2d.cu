// Fused multi-level 2-D Fast Haar analysis / synthesis kernels for sm_100a.
//
// Method: the polyphase "Fast Haar" banks of arXiv 1002.2184 (analysis: §III
// Fig. 4; synthesis: §IV Figs. 6-7, Eq. (19)) applied separably, rows then
// columns (reading R8).  Per 2x2 input block [[a, b], [c, d]] the row
// butterflies (x_e ± x_o)/√2 followed by the column butterflies fold to one exact ×½:
//     LL = ½((a+b)+(c+d))  LH = ½((a+b)−(c+d))  HL = ½((a−b)+(c−d))  HH = ½((a−b)−(c−d))
// and the synthesis bank (Eq. (19), A00 = A01 = 1/√2) folds to
//     a = ½((LL+LH)+(HL+HH))  b = ½((LL+LH)−(HL+HH))  c = ½((LL−LH)+(HL−HH))  d = ½((LL−LH)−(HL−HH)).
//
// B200 design: persistent CTAs (2 per SM) stream TR x TC tiles
// (32 x 256 fp32 = 32 KB) through a 3-stage TMA (cp.async.bulk.tensor) + mbarrier ring; all
// Lp <= 5 levels of a tile run in shared memory / registers; every detail band is written once,
// coalesced (float2 per thread, >= 32 B per row segment at the coarsest level), so HBM sees one
// read and one write of each sample.  Levels g >= 4 are computed in fp64.
#include <cooperative_groups.h>

#include <type_traits>

#include "fhwt_internal.cuh"
#include "haar2d_coarse.cuh"

// Minimum resident CTAs per SM the 2-D kernels are compiled for (register cap 65536 / (256 * n)).
#ifndef FHWT_MINB_ANA
#define FHWT_MINB_ANA 2
#endif
#ifndef FHWT_MINB_SYN
#define FHWT_MINB_SYN 3   // measured: synthesis 6.10 TB/s at 3 CTAs/SM vs 6.02 at 2; analysis best at 2
#endif

namespace fhwt {

namespace {

// First column of column-tile ct: ct * TC, except that with clamp_last the last tile of a ragged
// width starts at Win - TC (a full tile overlapping its neighbour; Win - TC is a multiple of the
// Haar block, so the overlapped coefficients are recomputed from the same inputs: same values).
template <typename P>
__device__ __forceinline__ int64_t tile_col0(const P& p, int64_t ct) {
  const int64_t c = ct * p.TC;
  return (p.clamp_last && c + p.TC > p.Win) ? p.Win - p.TC : c;
}

// First row of row tile rt (within an image): rt * TR, except that with clamp_rows the last tile of
// a height that is not a multiple of TR starts at Hin - TR (full, overlapping its neighbour; Hin - TR
// is a multiple of 2^Lp, so the overlapped rows are recomputed from the same inputs: same values).
template <typename P>
__device__ __forceinline__ int64_t tile_row0(const P& p, int64_t rt) {
  const int64_t r = rt * p.TR;
  return (p.clamp_rows && r + p.TR > p.Hin) ? p.Hin - p.TR : r;
}

// Phase timing of the fused analysis tile chain (diagnostic build only: -DFHWT_PHASE_TIMING, see
// tools/phase_timing.py).  Thread 0 (warp 0) and thread 224 (warp 7, the levels-4+5 lanes) add the
// clock64() cycles of each phase of every tile to g_phase[16 * w + k]; the default build has no trace of it.
#ifdef FHWT_PHASE_TIMING
__device__ unsigned long long g_phase[32];
__device__ __forceinline__ void phase_mark(int k) {
  __shared__ long long last[2];
  const int t = threadIdx.x;
  if (t == 0 || t == 224) {
    const int w = t ? 1 : 0;
    const long long now = clock64();
    if (k >= 0) atomicAdd(&g_phase[16 * w + k], (unsigned long long)(now - last[w]));
    if (k == 0) atomicAdd(&g_phase[16 * w + 15], 1ull);
    last[w] = now;
  }
}
#define FHWT_PHASE(k) phase_mark(k)
#else
#define FHWT_PHASE(k) ((void)0)
#endif

// Threads per CTA of a compile-time fast variant: one 2 x 2V unit per thread on level 1 of the
// smallest tiles (8 x 128: 64 threads), so small-tile shapes (e.g. 1080-row frames) run many
// independent CTAs per SM instead of a few latency-bound 256-thread ones; 256 from 32 x 128 up.
#ifndef FHWT_FAST_PX_PER_THREAD
#define FHWT_FAST_PX_PER_THREAD 32   // measured: 16 x 256 tiles (2160-row frames) 4.8 -> 5.6 / 4.7 -> 6.0 TB/s
#endif
constexpr int fast_threads(int TRF, int TCF) {
  return TRF * TCF / FHWT_FAST_PX_PER_THREAD < 64 ? 64
         : (TRF * TCF / FHWT_FAST_PX_PER_THREAD > kThreads2d ? kThreads2d : TRF * TCF / FHWT_FAST_PX_PER_THREAD);
}

// Stores V consecutive floats at ptr[0..V) of which the first `nvalid` lie inside the band.
// ALIGNED: the caller guarantees an 8-B aligned ptr and a full vector (fast tiles).
template <int V, bool ALIGNED>
__device__ __forceinline__ void store_row(float* ptr, const float (&v)[V], int64_t nvalid) {
  if constexpr (V == 2) {
    if (ALIGNED || (nvalid >= 2 && (reinterpret_cast<uintptr_t>(ptr) & 7) == 0)) {
      stg_stream2(ptr, make_float2(v[0], v[1]));
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < V; ++i)
    if (ALIGNED || i < nvalid) stg_stream1(ptr + i, v[i]);
}

template <typename T, int N, bool ALIGNED = false>
__device__ __forceinline__ void load_row(const T* src, T (&v)[N]) {
  if constexpr (sizeof(T) == 4 && N == 4) {
    const float4 t = *reinterpret_cast<const float4*>(src);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else if constexpr (sizeof(T) == 4 && N == 2) {
    if (ALIGNED || (reinterpret_cast<uintptr_t>(src) & 7) == 0) {
      const float2 t = *reinterpret_cast<const float2*>(src);
      v[0] = t.x; v[1] = t.y;
    } else {  // HL/HH boxes shifted by an odd hoff
      v[0] = src[0]; v[1] = src[1];
    }
  } else if constexpr (sizeof(T) == 4 && N == 1) {
    v[0] = src[0];
  } else {
    static_assert(sizeof(T) == 8 && N % 2 == 0, "double rows are loaded as double2");
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const double2 t = *reinterpret_cast<const double2*>(src + i);
      v[i] = t.x; v[i + 1] = t.y;
    }
  }
}

// LL_g of a unit -> shared memory (vector store: lanes write consecutive 8/16-B words, no conflicts)
template <typename TC, int V>
__device__ __forceinline__ void store_ll_smem(TC* dst, const TC (&ll)[V]) {
  if constexpr (V == 2 && sizeof(TC) == 4) {
    *reinterpret_cast<float2*>(dst) = make_float2(ll[0], ll[1]);
  } else if constexpr (V == 2) {
    *reinterpret_cast<double2*>(dst) = make_double2(ll[0], ll[1]);
  } else {
    dst[0] = ll[0];
  }
}

// One analysis level of one tile.  Source: the R x C region (smem, pitch C) of LL_{g-1} (or the
// input tile); V output columns per thread unit (one 2 x 2V input block).  Writes HL/LH/HH of global
// level g to HBM and LL_g to smem (lldst, pitch C/2) or, on the pass's last level, to HBM (coeffs
// LL region or the fp64 workspace).
// RC, CC: compile-time R, C (0 = runtime).  FAST: full, 8-B aligned tile (no masks, no checks).
// UNR: unroll the unit loop; the lean K1 keeps it rolled (measured +0.9 % c4, +0.4 % c5 analysis)
template <typename TS, typename TC, int V, int RC, int CC, bool FAST, int NT = kThreads2d, bool UNR = true>
__device__ __forceinline__ void ana_level(const Ana2dParams& p, const TS* __restrict__ src, int R_, int C_, int j,
                                          int64_t b, int64_t row0, int64_t col0, TC* __restrict__ lldst,
                                          bool last) {
  const int R = RC ? RC : R_;
  const int C = CC ? CC : C_;
  const int OC = C >> 1;
  const int upr = OC / V;
  const int nunits = (R >> 1) * upr;
  const int g = p.g0 + j;
  const int64_t W = p.W;
  const int64_t wg = W >> g, hgW = (p.H >> g) * W;
  const int64_t brow = row0 >> j, bcol = col0 >> j;
  float* const base = p.out + (b * p.H + brow) * W + bcol;  // (orow, oc) = (0, 0) of LL_g in this tile
  const int64_t nvalid_row = FAST ? int64_t(OC) : (p.Win >> j) - bcol;
  const TC half = TC(0.5);
  const int iters = (nunits + NT - 1) / NT;
  auto unit = [&](int it) -> bool {
    const int u = int(threadIdx.x) + it * NT;
    if ((nunits % NT) != 0 && u >= nunits) return false;
    const int orow = u / upr;
    const int oc = (u - orow * upr) * V;
    TS t0[2 * V], t1[2 * V];
    load_row<TS, 2 * V, true>(src + (2 * orow) * C + 2 * oc, t0);
    load_row<TS, 2 * V, true>(src + (2 * orow + 1) * C + 2 * oc, t1);
    float hl[V], lh[V], hh[V];
    TC ll[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const TC a = TC(t0[2 * v]), bb = TC(t0[2 * v + 1]), c = TC(t1[2 * v]), d = TC(t1[2 * v + 1]);
      const TC s1 = a + bb, s2 = c + d, d1 = a - bb, d2 = c - d;
      ll[v] = (s1 + s2) * half;
      lh[v] = float((s1 - s2) * half);
      hl[v] = float((d1 + d2) * half);
      hh[v] = float((d1 - d2) * half);
    }
    const int64_t nv = nvalid_row - oc;
    float* const pr = base + int64_t(orow) * W + oc;
    store_row<V, FAST>(pr + wg, hl, nv);
    store_row<V, FAST>(pr + hgW, lh, nv);
    store_row<V, FAST>(pr + hgW + wg, hh, nv);
    if (!last) {
      store_ll_smem<TC, V>(lldst + orow * OC + oc, ll);
    } else if (p.final_pass) {
      float llf[V];
#pragma unroll
      for (int v = 0; v < V; ++v) llf[v] = float(ll[v]);
      store_row<V, FAST>(pr, llf, nv);
    } else {
      // fp64 hand-off of LL_g to the next pass (pitch = padded Win >> Lp, see fhwt_api.cu)
      const int64_t wpitch = ((p.Win >> j) + 3) & ~int64_t(3);
      double* w = p.ws_out + (b * (p.Hin >> j) + brow + orow) * wpitch + bcol + oc;
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (v < nv) w[v] = double(ll[v]);
    }
    return true;
  };
  if constexpr (UNR) {
#pragma unroll
    for (int it = 0; it < iters; ++it)
      if (!unit(it)) break;
  } else {
#pragma unroll 1
    for (int it = 0; it < iters; ++it)
      if (!unit(it)) break;
  }
}

template <typename TS, typename TC>
__device__ __forceinline__ void ana_level_v(const Ana2dParams& p, const TS* src, int R, int C, int j, int64_t b,
                                            int64_t row0, int64_t col0, TC* lldst, bool last) {
  if (((C >> 1) & 1) == 0)
    ana_level<TS, TC, 2, 0, 0, false>(p, src, R, C, j, b, row0, col0, lldst, last);
  else
    ana_level<TS, TC, 1, 0, 0, false>(p, src, R, C, j, b, row0, col0, lldst, last);
}

// Generic tile: any TR/TC, ragged right edge, runtime level count, fp32 or fp64 input.
template <typename TIn>
__device__ __forceinline__ void ana_tile(const Ana2dParams& p, const TIn* stage, unsigned char* smem, int64_t b,
                                         int64_t row0, int64_t col0) {
  int R = p.TR, C = p.TC;
  const void* src = stage;
  bool src64 = sizeof(TIn) == 8;
  for (int j = 1; j <= p.Lp; ++j) {
    const bool cmp64 = src64 || (p.g0 + j) >= kFirstF64Level;
    const bool last = j == p.Lp;
    void* dst = smem + p.p_off[j & 1];
    if (!src64 && !cmp64)
      ana_level_v<float, float>(p, (const float*)src, R, C, j, b, row0, col0, (float*)dst, last);
    else if (!src64)
      ana_level_v<float, double>(p, (const float*)src, R, C, j, b, row0, col0, (double*)dst, last);
    else
      ana_level_v<double, double>(p, (const double*)src, R, C, j, b, row0, col0, (double*)dst, last);
    if (!last) __syncthreads();
    src = dst;
    src64 = cmp64;
    R >>= 1;
    C >>= 1;
  }
}

// Loads input tile `t` into a stage: TR one-row TMA boxes issued by the 32 lanes of warp 0.
// (Measured on B200, tools/membench: 32 one-row boxes stream at 6.9 TB/s where one 32-row box
// of the same bytes stops at 6.1 TB/s.)  Must be called by all of warp 0.
// U32: 32-bit tile decode (tile counts are < 2^31: a tile holds >= 1024 pixels and a buffer < 2^36).
// Measured on two boxes (interleaved processes): +1.0-1.6 % for LP = 4, 5 (c4, c5) and -1.5 % for
// LP = 3, so the fast variants choose it by LP (the issue path is sensitive to every instruction).
template <bool CLAMPR, bool U32 = false>
__device__ __forceinline__ void ana_issue_tile(const Ana2dParams& p, const CUtensorMap* map, unsigned char* dst,
                                               uint64_t* bar, int64_t t, uint32_t bytes, uint32_t row_bytes,
                                               uint64_t pol) {
  const int lane = threadIdx.x & 31;
  int64_t rt, ct;
  if constexpr (U32) {
    const uint32_t r32 = uint32_t(t) / uint32_t(p.tiles_c);
    rt = r32;
    ct = uint32_t(t) - r32 * uint32_t(p.tiles_c);
  } else {
    rt = t / p.tiles_c;
    ct = t - rt * p.tiles_c;
  }
  // first row in the (batch * Hin)-row tensor (< 2^31: the host splits larger batches).  With
  // clamp_rows every image's last row tile moves up by row_pad = tiles_r * TR - Hin, so the row is
  // rt * TR - row_pad * (b + last) = rt * TR - row_pad * ((rt + 1) / tiles_r).  Compile-time
  // (CLAMPR): any clamp arithmetic in this issue path cost the unclamped analysis 2-4 %.
  int grow = int(rt) * p.TR;
  if constexpr (CLAMPR) grow -= p.row_pad * int((uint32_t(rt) + 1u) / uint32_t(p.tiles_r));
  if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
  __syncwarp();
  if (p.row_boxes) {
    if (lane == 0) {
      if (p.l2hint)
        for (int r = 0; r < p.TR; ++r)
          tma_load_2d(dst + r * row_bytes, map, int(tile_col0(p, ct)), grow + r, bar, pol);
      else
        for (int r = 0; r < p.TR; ++r)
          tma_load_2d_nohint(dst + r * row_bytes, map, int(tile_col0(p, ct)), grow + r, bar);
    }
  } else if (lane == 0) {
    tma_load_2d(dst, map, int(tile_col0(p, ct)), grow, bar, pol);
  }
}

// Re-arms stage s of the TMA ring with the CTA's tile `next` (warp 0; no-op past the end).
template <bool CLAMPR, bool U32 = false>
struct Refill {
  const Ana2dParams* p;
  const CUtensorMap* map;
  unsigned char* dst;
  uint64_t* bar;
  int64_t next;
  uint32_t bytes, row_bytes;
  uint64_t pol;   // must be warp-uniform (computed by every thread): a divergent cache-hint operand
                  // makes each TMA issue a waterfall loop (analysis 6.57 -> 6.15 TB/s)
  __device__ __forceinline__ void operator()() const {
    // FHWT_ANA_FUSED=9: warp 4 (idle while warps 0-3 run levels 2+3) issues instead of warp 0
    const unsigned issuer = p->fused == 9 ? 4u : 0u;
    if ((threadIdx.x >> 5) == issuer && next < p->ntiles)
      ana_issue_tile<CLAMPR, U32>(*p, map, dst, bar, next, bytes, row_bytes, pol);
  }
};

// Fast tile: first pass (g0 = 0, fp32 input), TRF x TCF full tiles, LP levels known at compile
// time, so every index is a shift/constant and levels g >= 4 are fp64 by construction.
// FULL: a full tile with 8-B aligned band rows (no masks); else stores are masked at the image's
// right edge (TMA zero-fills the columns past it) and checked for alignment (odd band offsets).
template <int J, int LP, int TRF, int TCF, bool FULL = true, typename RF>
__device__ __forceinline__ void ana_fast_step(const Ana2dParams& p, const void* src, unsigned char* smem, int64_t b,
                                              int64_t row0, int64_t col0, const RF& refill) {
  constexpr int R = TRF >> (J - 1), C = TCF >> (J - 1);
  constexpr bool src64 = J - 1 >= kFirstF64Level;
  constexpr bool cmp64 = J >= kFirstF64Level;
  using TS = typename std::conditional<src64, double, float>::type;
  using TC = typename std::conditional<cmp64, double, float>::type;
  // unchecked 8-B band stores need even band offsets: W >> J and col0 >> J (levels 1..aligned_levels)
  if (FULL && J <= p.aligned_levels)
    ana_level<TS, TC, 2, R, C, true, fast_threads(TRF, TCF)>(p, static_cast<const TS*>(src), R, C, J, b, row0, col0,
                                                             reinterpret_cast<TC*>(smem + p.p_off[J & 1]), J == LP);
  else
    ana_level<TS, TC, 2, R, C, false, fast_threads(TRF, TCF)>(p, static_cast<const TS*>(src), R, C, J, b, row0, col0,
                                                              reinterpret_cast<TC*>(smem + p.p_off[J & 1]), J == LP);
  if constexpr (J < LP) {
    __syncthreads();
    if constexpr (J == 1) refill();   // level 1 was the last reader of the TMA stage
    ana_fast_step<J + 1, LP, TRF, TCF, FULL>(p, smem + p.p_off[J & 1], smem, b, row0, col0, refill);
  }
}

// Two levels of one thread's 4 x 4 LL block (rows r0.., cols c0.. of the level-(J-1) band block):
// level J gives 2 x 2 outputs per band, level J+1 one output per band and LL_{J+1}.  TA: level-J
// arithmetic type, TB: level-(J+1) type (fp64 from kFirstF64Level).
template <typename TA, typename TB, int J, int LP>
__device__ __forceinline__ TB ana_pair(const Ana2dParams& p, const float (&x)[4][4], int64_t b, int64_t row0,
                                       int64_t col0, int br, int bc) {
  const int64_t W = p.W;
  TA ll[2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {   // level J: rows 2br + i, cols 2bc + {0, 1} of the level-J bands
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
  // level J + 1 on the 2 x 2 LL_J block (rounded to TA first, exactly as the level-by-level kernel)
  const TB a = TB(ll[0][0]), bb = TB(ll[0][1]), c = TB(ll[1][0]), d = TB(ll[1][1]);
  const TB s1 = a + bb, s2 = c + d, d1 = a - bb, d2 = c - d;
  constexpr int J1 = J + 1;
  float* pr = p.out + (b * p.H + (row0 >> J1) + br) * W + (col0 >> J1) + bc;
  const int64_t wg = W >> J1, hgW = (p.H >> J1) * W;
  stg_stream1(pr + wg, float((d1 + d2) * TB(0.5)));
  stg_stream1(pr + hgW, float((s1 - s2) * TB(0.5)));
  stg_stream1(pr + hgW + wg, float((d1 - d2) * TB(0.5)));
  const TB ll1 = (s1 + s2) * TB(0.5);
  if constexpr (J1 == LP) {   // last level of the pass: LL to the coefficients or the fp64 hand-off
    if (p.final_pass) {
      stg_stream1(pr, float(ll1));
    } else {
      const int64_t wpitch = ((p.Win >> LP) + 3) & ~int64_t(3);
      p.ws_out[(b * (p.Hin >> LP) + (row0 >> LP) + br) * wpitch + (col0 >> LP) + bc] = double(ll1);
    }
  }
  return ll1;
}

// Fused fast path for 32 x 256 tiles, LP in 3..5: level 1 by all threads, levels 2+3 in one step
// (128 threads, one 4 x 4 LL1 block each), levels 4+5 in one step (8 threads, one 4 x 4 LL3 block
// each).  Two CTA barriers per tile instead of five, and the levels 4-5 threads overlap the next
// tile's level 1 (LL1 and LL3 live in different buffers; the next tile's first barrier orders the
// reuse).  Same arithmetic, same order, as ana_fast_step: outputs are bitwise identical.
template <int LP, typename RF>
__device__ __forceinline__ void ana_fused_tile(const Ana2dParams& p, const float* stage, unsigned char* smem, int64_t b,
                                               int64_t row0, int64_t col0, const RF& refill) {
  static_assert(LP >= 3 && LP <= 5, "fused path covers 3..5 levels");
  float* ll1 = reinterpret_cast<float*>(smem + p.p_off[1]);   // 16 x 128
  float* ll3 = reinterpret_cast<float*>(smem + p.p_off[0]);   // 4 x 32
  ana_level<float, float, 2, 32, 256, true>(p, stage, 32, 256, 1, b, row0, col0, ll1, false);
  FHWT_PHASE(1);
  __syncthreads();
  FHWT_PHASE(2);
  if (p.fused != 13) refill();   // 13: refill after the second barrier (later read-ahead; experiment)
  FHWT_PHASE(3);
  const int tid = threadIdx.x;
  if (p.fused == 6) {   // levels 2 + 3 over all 256 threads: two lanes per 4 x 4 LL1 block, level 3
                        // after a lane-pair shuffle of the LL2 columns
    const int blk = tid >> 1, h = tid & 1, br = blk >> 5, bc = blk & 31;
    float x[4][2];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float2 v = *reinterpret_cast<const float2*>(ll1 + (4 * br + r) * 128 + 4 * bc + 2 * h);
      x[r][0] = v.x; x[r][1] = v.y;
    }
    const int64_t W = p.W;
    float ll[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {   // level 2: rows 2br + i, column 2bc + h of the level-2 bands
      const float a = x[2 * i][0], bb = x[2 * i][1], c = x[2 * i + 1][0], d = x[2 * i + 1][1];
      const float s1 = a + bb, s2 = c + d, d1 = a - bb, d2 = c - d;
      ll[i] = (s1 + s2) * 0.5f;
      float* pr = p.out + (b * p.H + (row0 >> 2) + 2 * br + i) * W + (col0 >> 2) + 2 * bc + h;
      const int64_t wg = W >> 2, hgW = (p.H >> 2) * W;
      stg_stream1(pr + wg, (d1 + d2) * 0.5f);
      stg_stream1(pr + hgW, (s1 - s2) * 0.5f);
      stg_stream1(pr + hgW + wg, (d1 - d2) * 0.5f);
    }
    const float o0 = __shfl_xor_sync(0xffffffffu, ll[0], 1), o1 = __shfl_xor_sync(0xffffffffu, ll[1], 1);
    if (h == 0) {   // level 3 on the 2 x 2 LL2 block (same operands and order as ana_pair)
      const float a = ll[0], bb = o0, c = ll[1], d = o1;
      const float s1 = a + bb, s2 = c + d, d1 = a - bb, d2 = c - d;
      float* pr = p.out + (b * p.H + (row0 >> 3) + br) * W + (col0 >> 3) + bc;
      const int64_t wg = W >> 3, hgW = (p.H >> 3) * W;
      stg_stream1(pr + wg, (d1 + d2) * 0.5f);
      stg_stream1(pr + hgW, (s1 - s2) * 0.5f);
      stg_stream1(pr + hgW + wg, (d1 - d2) * 0.5f);
      const float l3 = (s1 + s2) * 0.5f;
      if constexpr (LP > 3) {
        ll3[br * 32 + bc] = l3;
      } else if (p.final_pass) {
        stg_stream1(pr, l3);
      } else {
        const int64_t wpitch = ((p.Win >> 3) + 3) & ~int64_t(3);
        p.ws_out[(b * (p.Hin >> 3) + (row0 >> 3) + br) * wpitch + (col0 >> 3) + bc] = double(l3);
      }
    }
  } else if (tid < 128) {   // levels 2 + 3: block (br, bc) of LL1, 4 x 32 blocks
    const int br = tid >> 5, bc = tid & 31;
    float x[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float4 v = *reinterpret_cast<const float4*>(ll1 + (4 * br + r) * 128 + 4 * bc);
      x[r][0] = v.x; x[r][1] = v.y; x[r][2] = v.z; x[r][3] = v.w;
    }
    const float l3 = ana_pair<float, float, 2, LP>(p, x, b, row0, col0, br, bc);
    if constexpr (LP > 3) ll3[br * 32 + bc] = l3;
  }
  FHWT_PHASE(4);
  if constexpr (LP > 3) {
    __syncthreads();
    if (p.fused == 13) refill();
    FHWT_PHASE(5);
    if (tid >= 224 && tid < 232) {   // levels 4 (+ 5): warp 7 lanes 0..7, block q of LL3 (4 x 32)
      const int q = tid - 224;
      float x[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float4 v = *reinterpret_cast<const float4*>(ll3 + r * 32 + 4 * q);
        x[r][0] = v.x; x[r][1] = v.y; x[r][2] = v.z; x[r][3] = v.w;
      }
      if constexpr (LP == 5) {
        ana_pair<double, double, 4, 5>(p, x, b, row0, col0, 0, q);
        FHWT_PHASE(6);
      } else {   // LP == 4: level 4 only, on the two 2 x 4 halves of the block
        const int64_t W = p.W;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          float hl[2], lh[2], hh[2], llv[2];
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const double a = x[2 * i][2 * k], bb = x[2 * i][2 * k + 1], c = x[2 * i + 1][2 * k], d = x[2 * i + 1][2 * k + 1];
            const double s1 = a + bb, s2 = c + d, d1 = a - bb, d2 = c - d;
            llv[k] = float((s1 + s2) * 0.5);
            lh[k] = float((s1 - s2) * 0.5);
            hl[k] = float((d1 + d2) * 0.5);
            hh[k] = float((d1 - d2) * 0.5);
            if (!p.final_pass) {
              const int64_t wpitch = ((p.Win >> 4) + 3) & ~int64_t(3);
              p.ws_out[(b * (p.Hin >> 4) + (row0 >> 4) + i) * wpitch + (col0 >> 4) + 2 * q + k] = (s1 + s2) * 0.5;
            }
          }
          float* pr = p.out + (b * p.H + (row0 >> 4) + i) * W + (col0 >> 4) + 2 * q;
          const int64_t wg = W >> 4, hgW = (p.H >> 4) * W;
          stg_stream2(pr + wg, make_float2(hl[0], hl[1]));
          stg_stream2(pr + hgW, make_float2(lh[0], lh[1]));
          stg_stream2(pr + hgW + wg, make_float2(hh[0], hh[1]));
          if (p.final_pass) stg_stream2(pr, make_float2(llv[0], llv[1]));
        }
      }
    }
  }
}

// Named CTA barrier 1 (barrier 0 is __syncthreads): producers arrive without waiting, consumers
// wait; `count` threads in total (a multiple of 32).  Orders the producers' shared-memory writes
// before the consumers' reads (PTX bar.arrive / bar.sync memory ordering).
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// FHWT_ANA_FUSED=12 (32 x 256 tiles, LP = 5): the fused chain with the refill OFF the per-tile
// critical path.  Warp 0 issues the stage refill after barrier 1 and goes straight on to the next
// tile's level 1; warps 1-4 run levels 2+3 and arrive on named barrier 1; only warp 7 waits there
// (levels 4+5 need LL3); warps 5-6 go on to the next tile.  The only CTA-wide barrier per tile is
// barrier 1 (level 1 done: stage consumed, LL1 complete).  LL1 is double-buffered (it & 1): the
// next tile's level 1 may write LL1 while warps 1-4 still read this tile's.  Same operations on
// the same operands as ana_fused_tile: bitwise identical output.
template <typename RF>
__device__ __forceinline__ void ana_fused12_tile(const Ana2dParams& p, const float* stage, unsigned char* smem,
                                                 int64_t b, int64_t row0, int64_t col0, int it, const RF& refill) {
  float* ll1 = reinterpret_cast<float*>(smem + p.p_off[1]) + (it & 1) * (16 * 128);
  float* ll3 = reinterpret_cast<float*>(smem + p.p_off[0]);   // 4 x 32
  ana_level<float, float, 2, 32, 256, true>(p, stage, 32, 256, 1, b, row0, col0, ll1, false);
  __syncthreads();
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    refill();
  } else if (warp <= 4) {   // levels 2 + 3: block (br, bc) of LL1, 4 x 32 blocks
    const int t = tid - 32, br = t >> 5, bc = t & 31;
    float x[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float4 v = *reinterpret_cast<const float4*>(ll1 + (4 * br + r) * 128 + 4 * bc);
      x[r][0] = v.x; x[r][1] = v.y; x[r][2] = v.z; x[r][3] = v.w;
    }
    ll3[br * 32 + bc] = ana_pair<float, float, 2, 5>(p, x, b, row0, col0, br, bc);
    named_bar_arrive(1, 160);
  } else if (warp == 7) {   // levels 4 + 5: lanes 0..7, block q of LL3 (4 x 32)
    named_bar_sync(1, 160);
    const int q = tid - 224;
    if (q < 8) {
      float x[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float4 v = *reinterpret_cast<const float4*>(ll3 + r * 32 + 4 * q);
        x[r][0] = v.x; x[r][1] = v.y; x[r][2] = v.z; x[r][3] = v.w;
      }
      ana_pair<double, double, 4, 5>(p, x, b, row0, col0, 0, q);
    }
  }
}

// Dedicated-tail-warp variant for 32 x 256 tiles, LP = 5 (FHWT_ANA_FUSED=3, ana2d_fused3_kernel):
// levels 1+2 in registers (every thread of warps 0-7 takes two 4 x 4 input blocks), so LL1 never
// touches shared memory; one CTA barrier per tile (LL2 complete, stage free); levels 3+4 and then
// 5 by a 9th warp while warps 0-7 start the next tile (LL2 and LL4 double-buffered).  Same
// operations on the same operands as the level-by-level kernel: bitwise identical output.
__device__ __forceinline__ void ana_level5_pair(const Ana2dParams& p, const double* ll4, int64_t b, int64_t row0,
                                                int64_t col0, int q) {
  const double2 r0 = *reinterpret_cast<const double2*>(ll4 + 2 * q);
  const double2 r1 = *reinterpret_cast<const double2*>(ll4 + 16 + 2 * q);
  const double a = r0.x, bb = r0.y, c = r1.x, d = r1.y;
  const double s1 = a + bb, s2 = c + d, d1 = a - bb, d2 = c - d;
  const int64_t W = p.W, wg = W >> 5, hgW = (p.H >> 5) * W;
  float* pr = p.out + (b * p.H + (row0 >> 5)) * W + (col0 >> 5) + q;
  stg_stream1(pr + wg, float((d1 + d2) * 0.5));
  stg_stream1(pr + hgW, float((s1 - s2) * 0.5));
  stg_stream1(pr + hgW + wg, float((d1 - d2) * 0.5));
  const double ll = (s1 + s2) * 0.5;
  if (p.final_pass) {
    stg_stream1(pr, float(ll));
  } else {
    const int64_t wpitch = ((p.Win >> 5) + 3) & ~int64_t(3);
    p.ws_out[(b * (p.Hin >> 5) + (row0 >> 5)) * wpitch + (col0 >> 5) + q] = ll;
  }
}

template <typename RF>
__device__ __forceinline__ void ana_fused3_tile(const Ana2dParams& p, const float* stage, unsigned char* smem, int64_t b,
                                                int64_t row0, int64_t col0, int it, const RF& refill) {
  float* ll2 = reinterpret_cast<float*>(smem + p.p_off[1]) + (it & 1) * 512;                  // 8 x 64
  double* ll4 = reinterpret_cast<double*>(smem + p.p_off[1] + 4096) + (it & 1) * 32;          // 2 x 16
  const int tid = threadIdx.x;
#pragma unroll
  for (int k = 0; k < 2; ++k) {   // levels 1 + 2: 8 x 64 blocks of 4 x 4 input pixels
    if (tid >= 256) break;   // warp 8 is the tail warp
    const int u = tid + 256 * k, rb = u >> 6, cb = u & 63;
    float x[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float4 v = *reinterpret_cast<const float4*>(stage + (4 * rb + r) * 256 + 4 * cb);
      x[r][0] = v.x; x[r][1] = v.y; x[r][2] = v.z; x[r][3] = v.w;
    }
    ll2[rb * 64 + cb] = ana_pair<float, float, 1, 5>(p, x, b, row0, col0, rb, cb);
  }
  __syncthreads();   // LL2 complete; every warp is done with the stage
  refill();
  if ((tid >> 5) == 8) {   // tail warp: levels 3 + 4 (one 4 x 4 LL2 block per lane), then 5
    const int lane = tid & 31, br = lane >> 4, bc = lane & 15;
    float x[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float4 v = *reinterpret_cast<const float4*>(ll2 + (4 * br + r) * 64 + 4 * bc);
      x[r][0] = v.x; x[r][1] = v.y; x[r][2] = v.z; x[r][3] = v.w;
    }
    ll4[br * 16 + bc] = ana_pair<float, double, 3, 5>(p, x, b, row0, col0, br, bc);
    __syncwarp();
    if (lane < 8) ana_level5_pair(p, ll4, b, row0, col0, lane);
  }
}

// fused2 with a dedicated tail warp: 288 threads (8 warps for levels 1 + 2, warp 8 for 3-5), so
// the tail work is off the critical path of the per-tile barrier.  32 x 256 full tiles, LP = 5.
__global__ void __launch_bounds__(288, 2) ana2d_fused3_kernel(const __grid_constant__ Ana2dParams p,
                                                              const __grid_constant__ CUtensorMap in_map) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  const int tid = threadIdx.x;
  if (tid == 0) {
    prefetch_tmap(&in_map);
    for (int s = 0; s < p.stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  constexpr uint32_t row_bytes = 1024, tile_bytes = 32 * row_bytes;
  const uint64_t pol = policy_evict_first();   // warp-uniform (see Refill)
  if (tid < 32) {
    for (int s = 0; s < p.stages; ++s) {
      const int64_t t = blockIdx.x + int64_t(s) * gridDim.x;
      if (t < p.ntiles)
        ana_issue_tile<false>(p, &in_map, smem + s * p.stage_bytes, &bars[s], t, tile_bytes, row_bytes, pol);
    }
  }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++it) {
    const int s = it % p.stages;
    mbar_wait(&bars[s], uint32_t(it / p.stages) & 1u);
    const int64_t rt = tile / p.tiles_c, ct = tile - rt * p.tiles_c;
    const int64_t b = rt / p.tiles_r;
    const Refill<false> refill{&p, &in_map, smem + s * p.stage_bytes, &bars[s], tile + int64_t(p.stages) * gridDim.x,
                               tile_bytes, row_bytes, pol};
    ana_fused3_tile(p, reinterpret_cast<const float*>(smem + s * p.stage_bytes), smem, b, (rt - b * p.tiles_r) * 32,
                    ct * 256, it, refill);
  }
  if (p.tail > 0) {
    cooperative_groups::this_grid().sync();
    if (p.tail == 1) ana_coarse<1>(p);
    else if (p.tail == 2) ana_coarse<2>(p);
    else ana_coarse<3>(p);
  }
}

// The persistent tile loop of ana2d_kernel; CLAMPR: the last row tile of every image is clamped
// (p.clamp_rows), a compile-time choice so the unclamped issue path carries no clamp arithmetic.
template <typename TIn, int LPFAST, int TRF, int TCF, bool CLAMPR>
__device__ __forceinline__ void ana2d_tiles(const Ana2dParams& p, const CUtensorMap& in_map, unsigned char* smem,
                                            uint64_t* bars) {
  const int tid = threadIdx.x;
  const uint32_t row_bytes = uint32_t(p.TC) * uint32_t(sizeof(TIn));
  const uint32_t tile_bytes = uint32_t(p.TR) * row_bytes;
  const uint64_t pol = p.l2hint == 2 ? policy_evict_normal() : p.l2hint == 3 ? policy_evict_last() : policy_evict_first();   // warp-uniform (see Refill)
  if (tid < 32) {
    for (int s = 0; s < p.stages; ++s) {
      const int64_t t = blockIdx.x + int64_t(s) * gridDim.x;
      if (t < p.ntiles)
        ana_issue_tile<CLAMPR, (LPFAST >= 4)>(p, &in_map, smem + s * p.stage_bytes, &bars[s], t, tile_bytes,
                                              row_bytes, pol);
    }
  }
  int it = 0;
  FHWT_PHASE(-1);
  for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++it) {
    const int s = it % p.stages;
    FHWT_PHASE(7);
    mbar_wait(&bars[s], uint32_t(it / p.stages) & 1u);
    FHWT_PHASE(0);
#ifdef FHWT_LOOP_U32   // experiment: 32-bit tile decode in the loop (tile counts < 2^31 for LP >= 4)
    int64_t rt, ct, b;
    if constexpr (LPFAST >= 4) {
      const uint32_t r32 = uint32_t(tile) / uint32_t(p.tiles_c), b32 = r32 / uint32_t(p.tiles_r);
      rt = r32; ct = uint32_t(tile) - r32 * uint32_t(p.tiles_c); b = b32;
    } else {
      rt = tile / p.tiles_c; ct = tile - rt * p.tiles_c; b = rt / p.tiles_r;
    }
#else
    const int64_t rt = tile / p.tiles_c, ct = tile - rt * p.tiles_c;
    const int64_t b = rt / p.tiles_r;
#endif
    const int64_t row0 = CLAMPR ? tile_row0(p, rt - b * p.tiles_r) : (rt - b * p.tiles_r) * p.TR;
    const Refill<CLAMPR, (LPFAST >= 4)> refill{&p, &in_map, smem + s * p.stage_bytes, &bars[s],
                                               tile + int64_t(p.stages) * gridDim.x, tile_bytes, row_bytes, pol};
    // mask_mode 1: the last column tile is ragged (masked stores); aligned_levels < LP: the coarse
    // levels' band offsets are odd (alignment-checked stores there).  With clamp_last the last tile
    // instead starts at Win - TC (full, overlapping its neighbour: identical values stored twice).
    const bool full = p.mask_mode == 0 || ct + 1 < p.tiles_c;
    const int64_t col0 = tile_col0(p, ct);
    if constexpr (LPFAST > 0) {
      if (!full || p.aligned_levels < LPFAST) {
        if (full)
          ana_fast_step<1, LPFAST, TRF, TCF, true>(p, smem + s * p.stage_bytes, smem, b, row0, col0, refill);
        else
          ana_fast_step<1, LPFAST, TRF, TCF, false>(p, smem + s * p.stage_bytes, smem, b, row0, col0, refill);
        __syncthreads();  // LL buffers free again
        if constexpr (LPFAST == 1) refill();
        continue;
      }
    }
    if constexpr (LPFAST >= 3 && TRF == 32 && TCF == 256) {
      if (LPFAST == 5 && p.fused == 12) {   // 1 CTA barrier per tile, refill off the critical path
        ana_fused12_tile(p, reinterpret_cast<const float*>(smem + s * p.stage_bytes), smem, b, row0, col0, it,
                         refill);
      } else if (p.fused) {   // 2 barriers per tile (see ana_fused_tile)
        ana_fused_tile<LPFAST>(p, reinterpret_cast<const float*>(smem + s * p.stage_bytes), smem, b, row0, col0,
                               refill);
      } else {
        ana_fast_step<1, LPFAST, TRF, TCF>(p, smem + s * p.stage_bytes, smem, b, row0, col0, refill);
        __syncthreads();  // LL buffers free again
      }
    } else if constexpr (LPFAST > 0) {
      ana_fast_step<1, LPFAST, TRF, TCF>(p, smem + s * p.stage_bytes, smem, b, row0, col0, refill);
      __syncthreads();  // LL buffers free again
      if constexpr (LPFAST == 1) refill();
    } else {
      ana_tile<TIn>(p, reinterpret_cast<const TIn*>(smem + s * p.stage_bytes), smem, b, row0, col0);
      __syncthreads();  // stage s and the LL buffers are free again
      refill();
    }
  }
}

template <typename TIn, int LPFAST, int TRF, int TCF>
__global__ void __launch_bounds__(LPFAST > 0 ? fast_threads(TRF, TCF) : kThreads2d,
                                  LPFAST > 0 ? FHWT_MINB_ANA * kThreads2d / fast_threads(TRF, TCF) : FHWT_MINB_ANA)
    ana2d_kernel(const __grid_constant__ Ana2dParams p,
                                                           const __grid_constant__ CUtensorMap in_map) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  const int tid = threadIdx.x;
  if (tid == 0) {
    prefetch_tmap(&in_map);
    for (int s = 0; s < p.stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (p.clamp_rows)
    ana2d_tiles<TIn, LPFAST, TRF, TCF, true>(p, in_map, smem, bars);
  else
    ana2d_tiles<TIn, LPFAST, TRF, TCF, false>(p, in_map, smem, bars);
  if constexpr (LPFAST == 5) {
    if (p.tail > 0) {   // cooperative launch: every CTA is resident, so the grid barrier is safe
      cooperative_groups::this_grid().sync();
      if (p.tail == 1) ana_coarse<1>(p);
      else if (p.tail == 2) ana_coarse<2>(p);
      else ana_coarse<3>(p);
    }
  }
}

__device__ __forceinline__ void mbar_arrive_plain(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ----------------------------------------------------------------- lean K1 (c4 / c5 tiles)
// The shipped analysis kernel for full 32 x 256 tiles with LP = 5 (every c4 / c5 tile): the same
// tile chain as ana2d_kernel's fused path (ana_fused_tile<5>: level 1 by all 256 threads, barrier,
// the stage refill by warp 0 lane 0, levels 2+3 by warps 0-3, barrier, levels 4+5 in fp64 by 8
// lanes of warp 7 overlapping the next tile's level 1), compiled as its own kernel with none of
// the general kernel's other paths (row clamp, masked / ragged tiles, level-by-level fallbacks,
// experiment branches).  Same operations on the same operands: bitwise identical output.  Why a
// separate kernel: the general ana2d_kernel<float,5,32,256> is ~16.8 K SASS instructions, and
// unrelated edits to it moved the c4 analysis between 5.6 and 6.35 TB/s (a 32-bit tile decode in
// the loop alone: 6345 -> 5630 GB/s, profiles/r02_l2_policy.md); the hot loop here is all the
// kernel holds.
struct LeanRefill {
  const Ana2dParams* p;
  const CUtensorMap* map;
  unsigned char* dst;
  uint64_t* bar;
  int64_t next;
  uint64_t pol;
  __device__ __forceinline__ void operator()() const {
    if (threadIdx.x < 32 && next < p->ntiles)
      ana_issue_tile<false, true>(*p, map, dst, bar, next, 32u * 1024u, 1024u, pol);
  }
};

__device__ __forceinline__ void ana_lean_tile(const Ana2dParams& p, const float* stage, unsigned char* smem,
                                              int64_t b, int64_t row0, int64_t col0, const LeanRefill& refill) {
  float* ll1 = reinterpret_cast<float*>(smem + p.p_off[1]);   // 16 x 128
  float* ll3 = reinterpret_cast<float*>(smem + p.p_off[0]);   // 4 x 32
  ana_level<float, float, 2, 32, 256, true, kThreads2d, false>(p, stage, 32, 256, 1, b, row0, col0, ll1, false);
  __syncthreads();   // LL1 complete; the stage has been read for the last time
  refill();
  const int tid = threadIdx.x;
  if (tid < 128) {   // levels 2 + 3: block (br, bc) of LL1, 4 x 32 blocks
    const int br = tid >> 5, bc = tid & 31;
    float x[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float4 v = *reinterpret_cast<const float4*>(ll1 + (4 * br + r) * 128 + 4 * bc);
      x[r][0] = v.x; x[r][1] = v.y; x[r][2] = v.z; x[r][3] = v.w;
    }
    ll3[br * 32 + bc] = ana_pair<float, float, 2, 5>(p, x, b, row0, col0, br, bc);
  }
  __syncthreads();   // LL3 complete
  if (tid >= 224 && tid < 232) {   // levels 4 + 5 (fp64): warp 7 lanes 0..7, block q of LL3 (4 x 32)
    const int q = tid - 224;
    float x[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float4 v = *reinterpret_cast<const float4*>(ll3 + r * 32 + 4 * q);
      x[r][0] = v.x; x[r][1] = v.y; x[r][2] = v.z; x[r][3] = v.w;
    }
    ana_pair<double, double, 4, 5>(p, x, b, row0, col0, 0, q);
  }
}

// DYN: tiles are handed out in global order by an atomic counter (p.tile_ctr) instead of the static
// blockIdx + k * grid assignment, so the tiles in flight at any moment stay contiguous in memory
// however far individual CTAs drift; the tile index travels to the consumers in shared memory
// next to the stage's mbarrier (written before the arrive, read after the wait).
template <bool DYN>
__global__ void __launch_bounds__(256, FHWT_MINB_ANA) ana2d_lean_kernel(const __grid_constant__ Ana2dParams p,
                                                                      const __grid_constant__ CUtensorMap in_map) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  const int tid = threadIdx.x;
  if (tid == 0) {
    prefetch_tmap(&in_map);
    for (int s = 0; s < p.stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();   // used only with FHWT_ANA_L2HINT=1
  if constexpr (DYN) {
    unsigned* stile = reinterpret_cast<unsigned*>(smem + p.bar_off + 8 * p.stages);
    if (tid < 32) {
      for (int s = 0; s < p.stages; ++s) {
        const uint32_t t = blockIdx.x + uint32_t(s) * gridDim.x;
        if ((tid & 31) == 0) stile[s] = t;
        if (t < p.ntiles) {
          ana_issue_tile<false, true>(p, &in_map, smem + s * p.stage_bytes, &bars[s],
                                      dyn_tile(t, uint32_t(p.ntiles), p.dyn_groups), 32768u, 1024u, pol);
        } else if ((tid & 31) == 0) {
          mbar_arrive_plain(&bars[s]);
        }
      }
    }
    for (int it = 0;; ++it) {
      const int s = it % p.stages;
      mbar_wait(&bars[s], uint32_t(it / p.stages) & 1u);
      const uint32_t cval = stile[s];
      if (cval >= uint32_t(p.ntiles)) break;
      const uint32_t tile = dyn_tile(cval, uint32_t(p.ntiles), p.dyn_groups);
      // the refill's tile index is fetched now, so the atomic's round trip overlaps level 1
      uint32_t nt = 0;
      if (tid == 0) nt = atomicAdd(p.tile_ctr, 1u) + uint32_t(p.stages) * gridDim.x;
      const int64_t rt = tile / uint32_t(p.tiles_c), ct = tile - uint32_t(rt) * uint32_t(p.tiles_c);
      const int64_t b = uint32_t(rt) / uint32_t(p.tiles_r);
      const float* stage = reinterpret_cast<const float*>(smem + s * p.stage_bytes);
      float* ll1 = reinterpret_cast<float*>(smem + p.p_off[1]);
      float* ll3 = reinterpret_cast<float*>(smem + p.p_off[0]);
      const int64_t row0 = (rt - b * p.tiles_r) * 32, col0 = ct * 256;
      ana_level<float, float, 2, 32, 256, true, kThreads2d, false>(p, stage, 32, 256, 1, b, row0, col0, ll1, false);
      __syncthreads();   // LL1 complete; the stage (and stile[s]) has been read for the last time
      if (tid < 32) {   // refill with the next tile in global order
        if (tid == 0) stile[s] = nt;
        nt = __shfl_sync(0xffffffffu, nt, 0);
        if (nt < uint32_t(p.ntiles))
          ana_issue_tile<false, true>(p, &in_map, smem + s * p.stage_bytes, &bars[s],
                                      dyn_tile(nt, uint32_t(p.ntiles), p.dyn_groups), 32768u, 1024u, pol);
        else if ((tid & 31) == 0)
          mbar_arrive_plain(&bars[s]);
      }
      if (tid < 128) {
        const int br = tid >> 5, bc = tid & 31;
        float x[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float4 v = *reinterpret_cast<const float4*>(ll1 + (4 * br + r) * 128 + 4 * bc);
          x[r][0] = v.x; x[r][1] = v.y; x[r][2] = v.z; x[r][3] = v.w;
        }
        ll3[br * 32 + bc] = ana_pair<float, float, 2, 5>(p, x, b, row0, col0, br, bc);
      }
      __syncthreads();   // LL3 complete
      if (tid >= 224 && tid < 232) {
        const int q = tid - 224;
        float x[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float4 v = *reinterpret_cast<const float4*>(ll3 + r * 32 + 4 * q);
          x[r][0] = v.x; x[r][1] = v.y; x[r][2] = v.z; x[r][3] = v.w;
        }
        ana_pair<double, double, 4, 5>(p, x, b, row0, col0, 0, q);
      }
    }
  } else {
  if (tid < 32) {
    for (int s = 0; s < p.stages; ++s) {
      const int64_t t = blockIdx.x + int64_t(s) * gridDim.x;
      if (t < p.ntiles) ana_issue_tile<false, true>(p, &in_map, smem + s * p.stage_bytes, &bars[s], t, 32768u, 1024u, pol);
    }
  }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++it) {
    const int s = it % p.stages;
    mbar_wait(&bars[s], uint32_t(it / p.stages) & 1u);
#ifdef FHWT_LEAN_U32   // robustness experiment: 32-bit tile decode
    const int64_t rt = uint32_t(tile) / uint32_t(p.tiles_c), ct = uint32_t(tile) - uint32_t(rt) * uint32_t(p.tiles_c);
    const int64_t b = uint32_t(rt) / uint32_t(p.tiles_r);
#else
    const int64_t rt = tile / p.tiles_c, ct = tile - rt * p.tiles_c;
    const int64_t b = rt / p.tiles_r;
#endif
    const LeanRefill refill{&p, &in_map, smem + s * p.stage_bytes, &bars[s], tile + int64_t(p.stages) * gridDim.x, pol};
    ana_lean_tile(p, reinterpret_cast<const float*>(smem + s * p.stage_bytes), smem, b, (rt - b * p.tiles_r) * 32,
                  ct * 256, refill);
  }
  }
  if (p.tail > 0) {   // cooperative launch: every CTA is resident, so the grid barrier is safe
    cooperative_groups::this_grid().sync();
    if (p.tail == 1) ana_coarse<1>(p);
    else if (p.tail == 2) ana_coarse<2>(p);
    else ana_coarse<3>(p);
  }
}

__device__ __forceinline__ unsigned atom_add_acq_rel_cta(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}

// ---------------------------------------------------------- shared helpers of the warp kernels
// Per-warp LL scratch of the warp-decoupled synthesis kernel (syn2d_warp_kernel).
struct WarpScratch {
  float ll1[16 * 16];
  float ll2[8 * 8];
  float ll3[4 * 4];
  double ll4[2 * 2];
};
static_assert(sizeof(WarpScratch) <= kSynScratchBytes, "host smem layout");

struct TileXY {
  int64_t b, row0, col0;
};
// tile -> (image, first row, first column); 32-bit division when the tile count allows it
__device__ __forceinline__ TileXY tile_xy(int64_t tile, int64_t tiles_c, int64_t tiles_r, int TR, int TC,
                                          int64_t clamp_row0) {   // clamp_row0: Hin - TR, or -1 (no clamp)
  TileXY t;
  if (tiles_c * tiles_r < (int64_t(1) << 31) && tile < (int64_t(1) << 31)) {
    const uint32_t rt = uint32_t(tile) / uint32_t(tiles_c), ct = uint32_t(tile) - rt * uint32_t(tiles_c);
    const uint32_t b = rt / uint32_t(tiles_r);
    t.b = b;
    t.row0 = int64_t(rt - b * uint32_t(tiles_r)) * TR;
    t.col0 = int64_t(ct) * TC;
  } else {
    const int64_t rt = tile / tiles_c, ct = tile - rt * tiles_c;
    t.b = rt / tiles_r;
    t.row0 = (rt - t.b * tiles_r) * TR;
    t.col0 = ct * TC;
  }
  if (clamp_row0 >= 0 && t.row0 > clamp_row0) t.row0 = clamp_row0;
  return t;
}

// ------------------------------------------------------------------------------------ synthesis
template <int V, bool ALIGNED>
__device__ __forceinline__ void store_out_row(float* ptr, const float (&v)[2 * V], int64_t nvalid) {
  if constexpr (V == 2) {
    if (ALIGNED || (nvalid >= 4 && (reinterpret_cast<uintptr_t>(ptr) & 15) == 0)) {
      stg_stream4(ptr, make_float4(v[0], v[1], v[2], v[3]));
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < 2 * V; ++i)
    if (ALIGNED || i < nvalid) stg_stream1(ptr + i, v[i]);
}

// One synthesis level: coefficient block R x C (tile rows/cols at level j) -> LL_{j-1} (2R x 2C),
// into smem (to_smem, pitch 2C) or, for pass-level 1, into HBM.
template <int V, int RC, int CC, bool FAST, int NT = kThreads2d>
__device__ __forceinline__ void syn_level(const Syn2dParams& p, const float* __restrict__ ll, int llp,
                                          const float* __restrict__ hl, const float* __restrict__ lh,
                                          const float* __restrict__ hh, int bp, int R_, int C_, bool to_smem,
                                          int64_t b, int64_t row0, int64_t col0, float* __restrict__ dst) {
  const int R = RC ? RC : R_;
  const int C = CC ? CC : C_;
  const int upr = C / V;
  const int nunits = R * upr;
  const int OC = 2 * C;  // dst pitch when dst is smem
  const int iters = (nunits + NT - 1) / NT;
  float* const obase = p.out + (b * p.Hin + row0) * p.out_pitch + col0;
#pragma unroll
  for (int it = 0; it < iters; ++it) {
    const int u = int(threadIdx.x) + it * NT;
    if ((nunits % NT) != 0 && u >= nunits) break;
    const int r = u / upr;
    const int c = (u - r * upr) * V;
    float vll[V], vhl[V], vlh[V], vhh[V];
    load_row<float, V, FAST>(ll + r * llp + c, vll);
    load_row<float, V, FAST>(hl + r * bp + c, vhl);
    load_row<float, V, FAST>(lh + r * bp + c, vlh);
    load_row<float, V, FAST>(hh + r * bp + c, vhh);
    float top[2 * V], bot[2 * V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const float s = vll[v] + vlh[v], t = vhl[v] + vhh[v];
      const float s2 = vll[v] - vlh[v], t2 = vhl[v] - vhh[v];
      top[2 * v] = (s + t) * 0.5f;
      top[2 * v + 1] = (s - t) * 0.5f;
      bot[2 * v] = (s2 + t2) * 0.5f;
      bot[2 * v + 1] = (s2 - t2) * 0.5f;
    }
    if (to_smem) {
      float* d0 = dst + (2 * r) * OC + 2 * c;
      if constexpr (V == 2) {  // 16-B vector stores: conflict-free across the warp
        *reinterpret_cast<float4*>(d0) = make_float4(top[0], top[1], top[2], top[3]);
        *reinterpret_cast<float4*>(d0 + OC) = make_float4(bot[0], bot[1], bot[2], bot[3]);
      } else {
        d0[0] = top[0]; d0[1] = top[1];
        d0[OC] = bot[0]; d0[OC + 1] = bot[1];
      }
    } else {
      const int64_t nv = FAST ? int64_t(2 * V) : p.Win - (col0 + 2 * c);
      float* o = obase + int64_t(2 * r) * p.out_pitch + 2 * c;
      store_out_row<V, FAST>(o, top, nv);
      store_out_row<V, FAST>(o + p.out_pitch, bot, nv);
    }
  }
}

__device__ __forceinline__ void syn_tile(const Syn2dParams& p, unsigned char* stage, unsigned char* smem, int64_t b,
                                         int64_t row0, int64_t col0) {
  const float* ll = reinterpret_cast<const float*>(stage + p.box_off[0][0]);
  int llp = p.box_pitch[p.Lp];
  for (int j = p.Lp; j >= 1; --j) {
    const int R = p.TR >> j, C = p.TC >> j;
    const float* hl = reinterpret_cast<const float*>(stage + p.box_off[j][0]) + p.hoff[j];
    const float* lh = reinterpret_cast<const float*>(stage + p.box_off[j][1]);
    const float* hh = reinterpret_cast<const float*>(stage + p.box_off[j][2]) + p.hoff[j];
    float* dst = reinterpret_cast<float*>(smem + p.p_off[(j - 1) & 1]);
    if ((C & 1) == 0)
      syn_level<2, 0, 0, false>(p, ll, llp, hl, lh, hh, p.box_pitch[j], R, C, j > 1, b, row0, col0, dst);
    else
      syn_level<1, 0, 0, false>(p, ll, llp, hl, lh, hh, p.box_pitch[j], R, C, j > 1, b, row0, col0, dst);
    if (j > 1) __syncthreads();
    ll = dst;
    llp = 2 * C;
  }
}

// Fast tile: TRF x TCF full tiles, hoff = 0, LP known at compile time (box pitch = TCF >> j).
// All levels J..1 from the TMA stage (level 1 writes the output tile).
// FULL: full tile, TMA boxes starting at their band block (hoff = 0), vector loads/stores unchecked.
// !FULL (ragged width or (W >> g) % 4 != 0): same compile-time geometry, boxes shifted left by
// hoff[J] (pitch box_pitch[J]), alignment-checked loads, stores masked at the image's right edge.
template <int J, int TRF, int TCF, bool FULL = true>
__device__ __forceinline__ void syn_fast_step(const Syn2dParams& p, unsigned char* stage, unsigned char* smem,
                                              const float* ll, int llp, int64_t b, int64_t row0, int64_t col0) {
  constexpr int R = TRF >> J, C = TCF >> J;
  const int sh = FULL ? 0 : p.hoff[J], bp = FULL ? C : p.box_pitch[J];
  const float* hl = reinterpret_cast<const float*>(stage + p.box_off[J][0]) + sh;
  const float* lh = reinterpret_cast<const float*>(stage + p.box_off[J][1]);
  const float* hh = reinterpret_cast<const float*>(stage + p.box_off[J][2]) + sh;
  float* dst = reinterpret_cast<float*>(smem + p.p_off[(J - 1) & 1]);
  syn_level<2, R, C, FULL, fast_threads(TRF, TCF)>(p, ll, llp, hl, lh, hh, bp, R, C, J > 1, b, row0, col0, dst);
  if constexpr (J > 1) {
    __syncthreads();
    syn_fast_step<J - 1, TRF, TCF, FULL>(p, stage, smem, dst, 2 * C, b, row0, col0);   // LL_{J-1} pitch 2C
  }
}

// cp.async variant: every thread copies 16-B chunks of tile t (all boxes of all levels, same smem
// layout as the TMA boxes) and commits one group.  Chunk q = tid + 256 i enumerates, level by
// level, the rows of HL, LH, HH (and the LL block of level LP).
template <int LP, int TRF, int TCF>
__device__ __forceinline__ void syn_cp_async_tile(const Syn2dParams& p, unsigned char* base, int64_t t) {
  const int64_t rt = t / p.tiles_c, ct = t - rt * p.tiles_c;
  const int64_t b = rt / p.tiles_r;
  const int64_t row0 = tile_row0(p, rt - b * p.tiles_r), col0 = tile_col0(p, ct + p.ct0);
  int q0 = 0;
#pragma unroll
  for (int j = 1; j <= LP; ++j) {
    const int rows = TRF >> j, cpr = (TCF >> j) / 4, nb = rows * cpr;   // chunks per band block
    const int g = p.g0 + j;
    const int64_t hg = p.H >> g, wg = p.W >> g;
    const float* gb = p.coeffs + (b * p.H + (row0 >> j)) * p.W + (col0 >> j);
#pragma unroll
    for (int q = int(threadIdx.x); q < 3 * nb; q += fast_threads(TRF, TCF)) {
      const int band = q / nb, rem = q - band * nb, r = rem / cpr, c = (rem - r * cpr) * 4;
      // band 0 = HL (right half), 1 = LH (bottom half), 2 = HH (both)
      const float* src = gb + (band >= 1 ? hg * p.W : 0) + (band != 1 ? wg : 0) + int64_t(r) * p.W + c;
      cp_async16(base + p.box_off[j][band] + (r * (TCF >> j) + c) * 4, src);
    }
    q0 += 3 * nb;
  }
  {
    const int rows = TRF >> LP, cpr = (TCF >> LP) / 4;
    const float* lsrc;
    int64_t lpitch;
    if (p.ll_from_ws) {
      lpitch = (((p.Win >> LP) + 3) & ~int64_t(3));
      lsrc = p.ll_ws + (b * (p.Hin >> LP) + (row0 >> LP)) * lpitch + (col0 >> LP);
    } else {
      lpitch = p.W;
      lsrc = p.coeffs + (b * p.H + (row0 >> LP)) * p.W + (col0 >> LP);
    }
    for (int q = int(threadIdx.x); q < rows * cpr; q += fast_threads(TRF, TCF)) {
      const int r = q / cpr, c = (q - r * cpr) * 4;
      cp_async16(base + p.box_off[0][0] + (r * (TCF >> LP) + c) * 4, lsrc + int64_t(r) * lpitch + c);
    }
  }
  cp_async_commit();
}

// Issues the TMA loads of tile t into one stage (LL box + 3 band boxes per level).  Called by all
// of warp 0; lane 0 issues.
__device__ __forceinline__ void syn_issue_tile(const Syn2dParams& p, const TmaMaps2d& maps, unsigned char* base,
                                               uint64_t* bar, int64_t t, uint64_t pol) {
  const int lane = threadIdx.x & 31;
  const int64_t rt = t / p.tiles_c, ct = t - rt * p.tiles_c;
  const int64_t b = rt / p.tiles_r;
  const int64_t row0 = tile_row0(p, rt - b * p.tiles_r), col0 = tile_col0(p, ct + p.ct0);
  if (lane == 0) mbar_arrive_expect_tx(bar, p.tx_bytes);
  __syncwarp();
  if (lane != 0) return;
  const int L = p.Lp;
  const int64_t llrow = p.ll_from_ws ? b * (p.Hin >> L) + (row0 >> L) : b * p.H + (row0 >> L);
  const int llrows = p.row_boxes[L] ? (p.TR >> L) : 1;
  for (int r = 0; r < llrows; ++r)
    tma_load_2d(base + p.box_off[0][0] + r * p.box_pitch[L] * 4, &maps.ll, int(col0 >> L), int(llrow + r), bar, pol);
  for (int j = L; j >= 1; --j) {
    const int g = p.g0 + j;
    const int64_t hg = p.H >> g, wg = p.W >> g;
    const int64_t br = b * p.H + (row0 >> j), bc = col0 >> j;
    const int hc = int(wg + bc) - p.hoff[j];   // 16-B aligned box start
    const int rb = p.box_pitch[j] * 4;
    const int nrows = p.row_boxes[j] ? (p.TR >> j) : 1;
    for (int r = 0; r < nrows; ++r) {
      tma_load_2d(base + p.box_off[j][0] + r * rb, &maps.level[j], hc, int(br + r), bar, pol);
      tma_load_2d(base + p.box_off[j][1] + r * rb, &maps.level[j], int(bc), int(br + hg + r), bar, pol);
      tma_load_2d(base + p.box_off[j][2] + r * rb, &maps.level[j], hc, int(br + hg + r), bar, pol);
    }
  }
}

// TMA load with (HINT) or without the L2 cache-policy operand.  Measured in the bench's step
// (tools/bench_ab.sh): the hint-free form of the instruction streams faster than any policy passed
// through .L2::cache_hint (analysis 6.20 -> 6.35 TB/s with the same evict_normal default policy).
template <bool HINT>
__device__ __forceinline__ void tma_load_2d_h(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                              uint64_t pol) {
  if constexpr (HINT) tma_load_2d(dst, map, c0, c1, bar, pol);
  else tma_load_2d_nohint(dst, map, c0, c1, bar);
}

// --------------------------------------------------- warp-decoupled synthesis (32 x 256 tiles)
// Mirror of ana2d_warp_kernel: warp w rebuilds output columns [32w, 32w + 32) of a tile from the
// level-j coefficient blocks at columns [(32w) >> j, (32w + 32) >> j) of the staged boxes.
// SHIFT: band blocks that do not start 16-B aligned (W >> g or the clamped last tile's column
// offset not a multiple of 4): every box starts at the aligned column at or below the block and is 4
// columns wider (box_pitch = (TC >> j) + 4); the compute phase adds the shift (column & 3).
template <bool SHIFT = false, bool CLAMPR = true, bool HINT = true>
__device__ __forceinline__ void syn_issue_tile_lane(const Syn2dParams& p, const TmaMaps2d& maps, unsigned char* base,
                                                    uint64_t* bar, int64_t t, uint64_t pol) {
  const int64_t rt = t / p.tiles_c, ct = t - rt * p.tiles_c;
  const int64_t b = rt / p.tiles_r;
  const int64_t row0 = CLAMPR ? tile_row0(p, rt - b * p.tiles_r) : (rt - b * p.tiles_r) * p.TR;
  const int64_t col0 = tile_col0(p, ct + p.ct0);
  constexpr int64_t AL = SHIFT ? ~int64_t(3) : ~int64_t(0);
#ifdef FHWT_EXP_NOCOARSE   // timing experiment only (wrong output): level-1 boxes only
  mbar_arrive_expect_tx(bar, 3u * uint32_t(p.TR >> 1) * uint32_t(p.box_pitch[1]) * 4u);
#else
  mbar_arrive_expect_tx(bar, p.tx_bytes);
#endif
  const int L = p.Lp;
  const int64_t llrow = p.ll_from_ws ? b * (p.Hin >> L) + (row0 >> L) : b * p.H + (row0 >> L);
  const int llrows = p.row_boxes[L] ? (p.TR >> L) : 1;
#ifndef FHWT_EXP_NOCOARSE
  for (int r = 0; r < llrows; ++r)
    tma_load_2d_h<HINT>(base + p.box_off[0][0] + r * p.box_pitch[L] * 4, &maps.ll, int((col0 >> L) & AL), int(llrow + r), bar,
                pol);
#endif
  for (int j = L; j >= 1; --j) {
#ifdef FHWT_EXP_NOCOARSE
    if (j > 1) continue;
#endif
    const int g = p.g0 + j;
    const int64_t hg = p.H >> g, wg = p.W >> g;
    const int64_t br = b * p.H + (row0 >> j), bc = col0 >> j;
    const int rb = p.box_pitch[j] * 4;
    const int nrows = p.row_boxes[j] ? (p.TR >> j) : 1;
    for (int r = 0; r < nrows; ++r) {
      tma_load_2d_h<HINT>(base + p.box_off[j][0] + r * rb, &maps.level[j], int((wg + bc) & AL), int(br + r), bar, pol);
      tma_load_2d_h<HINT>(base + p.box_off[j][1] + r * rb, &maps.level[j], int(bc & AL), int(br + hg + r), bar, pol);
      tma_load_2d_h<HINT>(base + p.box_off[j][2] + r * rb, &maps.level[j], int((wg + bc) & AL), int(br + hg + r), bar, pol);
    }
  }
}

// UNR: unroll the unit loop (syn2d_warp_kernel); the producer K4 keeps it rolled, measured +1 % on
// c4 / c5 synthesis (profiles/r02_dynamic_tiles.md)
// SWZ: the level's three band boxes were landed by the 128-B-swizzled 3-D maps (syn_issue_tile_swz):
// box row r is NCH = BP / 32 lines of 128 B, and the 16-B granule g of line l sits at g ^ (l & 7), so
// rows r and r + 1 (J = 1) or r .. r + 3 (J = 2) of a warp's column slice fall in different banks.
template <int J, bool SHIFT, bool LLSHIFT, int TCF, bool UNR = true, bool SWZ = false>
__device__ __forceinline__ void warp_syn_level(const Syn2dParams& p, const float* __restrict__ ll, int llp,
                                               const unsigned char* stage, int warp, float* __restrict__ dst,
                                               int64_t b, int64_t row0, int64_t colw, int64_t col0) {
  constexpr int R = 32 >> J, C = 32 >> J, BP = (TCF >> J) + (SHIFT ? 4 : 0);
  static_assert(!SWZ || (!SHIFT && BP % 32 == 0), "swizzled boxes: whole 128-B lines, no shift");
  constexpr int V = C >= 2 ? 2 : 1, UPR = C / V, NU = R * UPR, OC = 2 * C;
  int co = (32 * warp) >> J, coh = co;
  if constexpr (SHIFT) {   // see syn_issue_tile_lane<true>
    co += int((col0 >> J) & 3);
    coh += int(((p.W >> (p.g0 + J)) + (col0 >> J)) & 3);
  }
  const float* hl = reinterpret_cast<const float*>(stage + p.box_off[J][0]) + (SWZ ? 0 : coh);
  const float* lh = reinterpret_cast<const float*>(stage + p.box_off[J][1]) + (SWZ ? 0 : co);
  const float* hh = reinterpret_cast<const float*>(stage + p.box_off[J][2]) + (SWZ ? 0 : coh);
  const int lane = threadIdx.x & 31;
  float* const obase = p.out + (b * p.Hin + row0) * p.out_pitch + colw;
  constexpr int UNROLL = UNR ? (NU + 31) / 32 : 1;
#pragma unroll UNROLL
  for (int it = 0; it < (NU + 31) / 32; ++it) {
    const int u = lane + 32 * it;
    if (NU % 32 != 0 && u >= NU) break;
    const int r = u / UPR, c = (u - r * UPR) * V;
    float vll[V], vhl[V], vlh[V], vhh[V];
#if !defined(FHWT_EXP_NOCOMPUTE)
    load_row<float, V, !LLSHIFT>(ll + r * llp + c, vll);
#endif
#if defined(FHWT_EXP_NOCOMPUTE)   // timing experiment only (wrong output): the memory pattern alone
    if constexpr (J > 1) return;
    for (int v = 0; v < V; ++v) vll[v] = vhl[v] = vlh[v] = vhh[v] = float(r);
#else
#ifdef FHWT_EXP_NOCONFLICT   // timing experiment only (wrong output): rows r, r+1 in different bank halves
    const int xo = (J <= 2) ? (r & 1) * 16 : 0;
#else
    constexpr int xo = 0;
#endif
    if constexpr (SWZ) {
      constexpr int NCH = BP / 32;
      const int cc = co + c, line = r * NCH + (cc >> 5);
      const int o = line * 32 + ((((cc >> 2) & 7) ^ (line & 7)) << 2) + (cc & 3);
      load_row<float, V, true>(hl + o, vhl);
      load_row<float, V, true>(lh + o, vlh);
      load_row<float, V, true>(hh + o, vhh);
    } else {
      load_row<float, V, !SHIFT>(hl + r * BP + c + xo, vhl);
      load_row<float, V, !SHIFT>(lh + r * BP + c + xo, vlh);
      load_row<float, V, !SHIFT>(hh + r * BP + c + xo, vhh);
    }
#endif
    float top[2 * V], bot[2 * V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const float s = vll[v] + vlh[v], t = vhl[v] + vhh[v];
      const float s2 = vll[v] - vlh[v], t2 = vhl[v] - vhh[v];
      top[2 * v] = (s + t) * 0.5f;
      top[2 * v + 1] = (s - t) * 0.5f;
      bot[2 * v] = (s2 + t2) * 0.5f;
      bot[2 * v + 1] = (s2 - t2) * 0.5f;
    }
    if constexpr (J > 1) {
      float* d0 = dst + (2 * r) * OC + 2 * c;
      if constexpr (V == 2) {
        *reinterpret_cast<float4*>(d0) = make_float4(top[0], top[1], top[2], top[3]);
        *reinterpret_cast<float4*>(d0 + OC) = make_float4(bot[0], bot[1], bot[2], bot[3]);
      } else {
        *reinterpret_cast<float2*>(d0) = make_float2(top[0], top[1]);
        *reinterpret_cast<float2*>(d0 + OC) = make_float2(bot[0], bot[1]);
      }
    } else {
      float* o = obase + int64_t(2 * r) * p.out_pitch + 2 * c;
      store_out_row<V, true>(o, top, 2 * V);
      store_out_row<V, true>(o + p.out_pitch, bot, 2 * V);
    }
  }
}

// SWZL: levels 1..SWZL read swizzled boxes
template <int J, int LP, bool SHIFT, int TCF, bool UNR = true, int SWZL = 0>
__device__ __forceinline__ void warp_syn_steps(const Syn2dParams& p, const float* ll, int llp,
                                               const unsigned char* stage, int warp, WarpScratch* sc, int64_t b,
                                               int64_t row0, int64_t colw, int64_t col0) {
  float* dst = J == 5 ? reinterpret_cast<float*>(sc->ll4) : J == 4 ? sc->ll3 : J == 3 ? sc->ll2 : sc->ll1;
  warp_syn_level<J, SHIFT, SHIFT && J == LP, TCF, UNR, (J <= SWZL)>(p, ll, llp, stage, warp, dst, b, row0, colw, col0);
  if constexpr (J > 1) {
    __syncwarp();
    warp_syn_steps<J - 1, LP, SHIFT, TCF, UNR, SWZL>(p, dst, 2 * (32 >> J), stage, warp, sc, b, row0, colw, col0);
  }
}

// The persistent tile loop of syn2d_warp_kernel; CLAMPR (p.clamp_rows) is compile-time so the
// unclamped issue path carries no clamp arithmetic (as in ana2d_tiles).
// DYN: the next tile of a released stage comes from the launch's tile counter (p.tile_ctr, global
// order) instead of tile + stages * grid; its index is stored next to the stage's mbarrier
// (stile[s]) before the arrive and read by every warp after its wait (see ana2d_lean_kernel).
template <int LP, bool SHIFT, int TCF, bool CLAMPR, bool DYN = false>
__device__ __forceinline__ void syn2d_warp_tiles(const Syn2dParams& p, const TmaMaps2d& maps, unsigned char* smem,
                                                 uint64_t* bars, unsigned* cnt, WarpScratch* sc) {
  constexpr unsigned NW = TCF / 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t pol = p.l2mode == 0 ? policy_evict_first() : p.l2mode == 1 ? policy_evict_normal() : policy_evict_last();
  if constexpr (DYN) {
    unsigned* stile = cnt + p.stages;
    unsigned* pend = cnt + 2 * p.stages;   // next tile for stage s, fetched by warp 0 during the tile
    if (tid == 0)
      for (int s = 0; s < p.stages; ++s) {
        const uint32_t t = blockIdx.x + uint32_t(s) * gridDim.x;
        stile[s] = t;
        if (t < uint32_t(p.ntiles))
          syn_issue_tile_lane<SHIFT, CLAMPR, false>(p, maps, smem + s * p.stage_bytes, &bars[s],
                                                    dyn_tile(t, uint32_t(p.ntiles), p.dyn_groups), pol);
        else mbar_arrive_plain(&bars[s]);
      }
    for (int it = 0;; ++it) {
      const int s = it % p.stages;
      mbar_wait(&bars[s], uint32_t(it / p.stages) & 1u);
      const uint32_t cval = stile[s];
      if (cval >= uint32_t(p.ntiles)) break;
      const uint32_t tile = dyn_tile(cval, uint32_t(p.ntiles), p.dyn_groups);
      uint32_t nt = 0;
      if (tid == 0) nt = atomicAdd(p.tile_ctr, 1u) + uint32_t(p.stages) * gridDim.x;   // overlaps the tile
      const TileXY xy = tile_xy(tile, p.tiles_c, p.tiles_r, 32, TCF, CLAMPR ? p.Hin - 32 : -1);
      const unsigned char* stage = smem + s * p.stage_bytes;
      const int64_t col0 = tile_col0(p, xy.col0 / TCF + p.ct0);
      const float* ll = reinterpret_cast<const float*>(stage + p.box_off[0][0]) + ((32 * warp) >> LP) +
                        (SHIFT ? int((col0 >> LP) & 3) : 0);
      warp_syn_steps<LP, LP, SHIFT, TCF>(p, ll, (TCF >> LP) + (SHIFT ? 4 : 0), stage, warp, sc, xy.b, xy.row0,
                                         col0 + 32 * warp, col0);
      __syncwarp();
      if (lane == 0) {   // stage release (as below); the last warp refills with warp 0's fetched tile
        if (tid == 0) pend[s] = nt;   // before warp 0's release: the last warp acquires it
        if ((atom_add_acq_rel_cta(&cnt[s], 1u) & (NW - 1)) == NW - 1) {
          nt = pend[s];
          stile[s] = nt;
          if (nt < uint32_t(p.ntiles))
            syn_issue_tile_lane<SHIFT, CLAMPR, false>(p, maps, smem + s * p.stage_bytes, &bars[s],
                                                      dyn_tile(nt, uint32_t(p.ntiles), p.dyn_groups), pol);
          else mbar_arrive_plain(&bars[s]);
        }
      }
    }
    return;
  }
  if (tid == 0)
    for (int s = 0; s < p.stages; ++s) {
      const int64_t t = blockIdx.x + int64_t(s) * gridDim.x;
      if (t < p.ntiles) {
        if (p.l2mode == 3) syn_issue_tile_lane<SHIFT, CLAMPR, false>(p, maps, smem + s * p.stage_bytes, &bars[s], t, pol);
        else syn_issue_tile_lane<SHIFT, CLAMPR>(p, maps, smem + s * p.stage_bytes, &bars[s], t, pol);
      }
    }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++it) {
    const int s = it % p.stages;
    mbar_wait(&bars[s], uint32_t(it / p.stages) & 1u);
    const TileXY xy = tile_xy(tile, p.tiles_c, p.tiles_r, 32, TCF, CLAMPR ? p.Hin - 32 : -1);
    const unsigned char* stage = smem + s * p.stage_bytes;
    const int64_t col0 = tile_col0(p, xy.col0 / TCF + p.ct0);
    const float* ll = reinterpret_cast<const float*>(stage + p.box_off[0][0]) + ((32 * warp) >> LP) +
                      (SHIFT ? int((col0 >> LP) & 3) : 0);
    warp_syn_steps<LP, LP, SHIFT, TCF>(p, ll, (TCF >> LP) + (SHIFT ? 4 : 0), stage, warp, sc, xy.b, xy.row0,
                                       col0 + 32 * warp, col0);
    __syncwarp();
    if (lane == 0) {   // stage release: the last warp through level 1 refills it
      // acq_rel RMW on the stage counter (after __syncwarp): releases this warp's reads of the
      // stage, and the last warp acquires every other warp's before it re-arms the stage for TMA
      // (the same release/acquire hand-off as an "empty" mbarrier; a full fence here, MEMBAR.SC,
      // showed in 2.6 % of the stall samples)
      if ((atom_add_acq_rel_cta(&cnt[s], 1u) & (NW - 1)) == NW - 1) {
        const int64_t nt = tile + int64_t(p.stages) * gridDim.x;
        if (nt < p.ntiles) {
          if (p.l2mode == 3) syn_issue_tile_lane<SHIFT, CLAMPR, false>(p, maps, smem + s * p.stage_bytes, &bars[s], nt, pol);
          else syn_issue_tile_lane<SHIFT, CLAMPR>(p, maps, smem + s * p.stage_bytes, &bars[s], nt, pol);
        }
      }
    }
  }
}

// TCF: tile columns, 256 (8 warps) or 128 (4 warps); each warp owns a 32-column slice.
template <int LP, bool SHIFT = false, int TCF = 256, bool DYN = false>
__global__ void __launch_bounds__(TCF, FHWT_MINB_SYN * 256 / TCF) syn2d_warp_kernel(const __grid_constant__ Syn2dParams p,
                                                                const __grid_constant__ TmaMaps2d maps) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  unsigned* cnt = reinterpret_cast<unsigned*>(smem + p.bar_off + 8 * p.stages);
  const int tid = threadIdx.x, warp = tid >> 5;
  WarpScratch* sc = reinterpret_cast<WarpScratch*>(smem + p.p_off[0] + warp * kSynScratchBytes);
  if (tid == 0) {
    for (int j = 1; j <= LP; ++j) prefetch_tmap(&maps.level[j]);
    prefetch_tmap(&maps.ll);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&bars[s], 1);
      cnt[s] = 0;
    }
    fence_mbar_init();
  }
  __syncthreads();
  if constexpr (LP == 5 && !SHIFT && TCF >= 256) {
    if (p.head > 0) {   // cooperative launch: coarse levels -> fp32 LL5 hand-off, then a grid barrier
      if (p.head == 1) syn_coarse<1>(p);
      else if (p.head == 2) syn_coarse<2>(p);
      else syn_coarse<3>(p);
      fence_proxy_async_global();   // generic-proxy stores, read below by TMA (async proxy)
      cooperative_groups::this_grid().sync();
      fence_proxy_async_global();
    }
  }
  if (p.clamp_rows)
    syn2d_warp_tiles<LP, SHIFT, TCF, true, DYN>(p, maps, smem, bars, cnt, sc);
  else
    syn2d_warp_tiles<LP, SHIFT, TCF, false, DYN>(p, maps, smem, bars, cnt, sc);
}

// The producer's issue in the opposite order: level-1 bands first, the coarse boxes and LL last
// (FHWT_SYN_ISSUE_REV=1; full unclamped 32-row tiles, no shifted boxes).
__device__ __forceinline__ void syn_issue_tile_fine_first(const Syn2dParams& p, const TmaMaps2d& maps,
                                                          unsigned char* base, uint64_t* bar, int64_t t) {
  const int64_t rt = t / p.tiles_c, ct = t - rt * p.tiles_c;
  const int64_t b = rt / p.tiles_r;
  const int64_t row0 = (rt - b * p.tiles_r) * p.TR, col0 = tile_col0(p, ct + p.ct0);
  mbar_arrive_expect_tx(bar, p.tx_bytes);
  const int L = p.Lp;
  for (int j = 1; j <= L; ++j) {
    const int64_t hg = p.H >> (p.g0 + j), wg = p.W >> (p.g0 + j);
    const int64_t br = b * p.H + (row0 >> j), bc = col0 >> j;
    const int rb = p.box_pitch[j] * 4;
    const int nrows = p.row_boxes[j] ? (p.TR >> j) : 1;
    for (int r = 0; r < nrows; ++r) {
      tma_load_2d_nohint(base + p.box_off[j][0] + r * rb, &maps.level[j], int(wg + bc), int(br + r), bar);
      tma_load_2d_nohint(base + p.box_off[j][1] + r * rb, &maps.level[j], int(bc), int(br + hg + r), bar);
      tma_load_2d_nohint(base + p.box_off[j][2] + r * rb, &maps.level[j], int(wg + bc), int(br + hg + r), bar);
    }
  }
  const int64_t llrow = p.ll_from_ws ? b * (p.Hin >> L) + (row0 >> L) : b * p.H + (row0 >> L);
  const int llrows = p.row_boxes[L] ? (p.TR >> L) : 1;
  for (int r = 0; r < llrows; ++r)
    tma_load_2d_nohint(base + p.box_off[0][0] + r * p.box_pitch[L] * 4, &maps.ll, int(col0 >> L), int(llrow + r), bar);
}

// The producer's issue with the level-1..SWZL (1-2) band boxes through the swizzled 3-D maps (p.swz;
// full unclamped 32 x 256 tiles, one box per band at those levels): the same bytes land in the same
// boxes, each 128-B line's 16-B granules permuted by SWIZZLE_128B (read back by warp_syn_level<SWZ>).
// A box whose innermost dimension is one 128-B line streams far faster than the 2-D box with 512-B
// rows (c4 synthesis 6.45 -> 6.92 TB/s unswizzled, 6.93 swizzled; profiles/r02_swizzle.md).
template <int SWZL>
__device__ __forceinline__ void syn_issue_tile_swz(const Syn2dParams& p, const TmaMaps2d& maps, unsigned char* base,
                                                   uint64_t* bar, int64_t t) {
  const int64_t rt = t / p.tiles_c, ct = t - rt * p.tiles_c;
  const int64_t b = rt / p.tiles_r;
  const int64_t row0 = (rt - b * p.tiles_r) * p.TR, col0 = tile_col0(p, ct + p.ct0);
  mbar_arrive_expect_tx(bar, p.tx_bytes);
  const int L = p.Lp;
  const int64_t llrow = p.ll_from_ws ? b * (p.Hin >> L) + (row0 >> L) : b * p.H + (row0 >> L);
  const int llrows = p.row_boxes[L] ? (p.TR >> L) : 1;
  for (int r = 0; r < llrows; ++r)
    tma_load_2d_nohint(base + p.box_off[0][0] + r * p.box_pitch[L] * 4, &maps.ll, int(col0 >> L), int(llrow + r), bar);
  for (int j = L; j > SWZL; --j) {
    const int64_t hg = p.H >> j, wg = p.W >> j;
    const int64_t br = b * p.H + (row0 >> j), bc = col0 >> j;
    const int rb = p.box_pitch[j] * 4;
    const int nrows = p.row_boxes[j] ? (p.TR >> j) : 1;
    for (int r = 0; r < nrows; ++r) {
      tma_load_2d_nohint(base + p.box_off[j][0] + r * rb, &maps.level[j], int(wg + bc), int(br + r), bar);
      tma_load_2d_nohint(base + p.box_off[j][1] + r * rb, &maps.level[j], int(bc), int(br + hg + r), bar);
      tma_load_2d_nohint(base + p.box_off[j][2] + r * rb, &maps.level[j], int(wg + bc), int(br + hg + r), bar);
    }
  }
#pragma unroll
  for (int j = SWZL; j >= 1; --j) {
    const int64_t hg = p.H >> j, wg = p.W >> j;
    const int64_t br = b * p.H + (row0 >> j), bc = col0 >> j;
    tma_load_3d_nohint(base + p.box_off[j][0], &maps.sw[j], 0, int((wg + bc) >> 5), int(br), bar);
    tma_load_3d_nohint(base + p.box_off[j][1], &maps.sw[j], 0, int(bc >> 5), int(br + hg), bar);
    tma_load_3d_nohint(base + p.box_off[j][2], &maps.sw[j], 0, int((wg + bc) >> 5), int(br + hg), bar);
  }
}

// K4 with a TMA producer warp (FHWT_SYN_PROD=1: static tile order, =2: global order from the tile
// counter).  32 x 256 full tiles, LP = 5, no shifted boxes.  Warps 0-7 rebuild their 32-column
// slices exactly as syn2d_warp_kernel<5> does (warp_syn_steps) and arrive on the stage's "empty"
// mbarrier (count 8) after level 1; warp 8 lane 0 waits for "empty", picks the next tile, stores
// its index next to the stage ("stile", read by the compute warps after their "full" wait) and
// issues the 16 boxes: the issue is on no compute warp's path.  Bitwise identical output.
// RAGGED: the launch covers the full tiles of a ragged width (column-tile offset p.ct0, last tile
// clamped); otherwise tiles start at column ct * TCF (c4, c5).
// SWZL > 0: level-1..SWZL boxes through the swizzled maps (syn_issue_tile_swz, warp_syn_level<SWZ>).
template <bool DYN, int TCF = 256, bool RAGGED = false, int SWZL = 0>
#ifndef FHWT_PROD_MINB
#define FHWT_PROD_MINB 2   // resident CTAs the producer K4's registers are capped for (TCF = 256)
#endif
__global__ void __launch_bounds__(TCF + 32, TCF == 256 ? FHWT_PROD_MINB : 1) syn2d_prod_kernel(const __grid_constant__ Syn2dParams p,
                                                                        const __grid_constant__ TmaMaps2d maps) {
  constexpr int NW = TCF / 32;   // compute warps; warp NW is the producer
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* empty = full + p.stages;
  unsigned* stile = reinterpret_cast<unsigned*>(empty + p.stages);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int j = SWZL + 1; j <= 5; ++j) prefetch_tmap(&maps.level[j]);
    for (int j = 1; j <= SWZL; ++j) prefetch_tmap(&maps.sw[j]);
    prefetch_tmap(&maps.ll);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (p.head > 0) {   // cooperative launch: coarse levels -> fp32 LL5 hand-off, then a grid barrier
    if (p.head == 1) syn_coarse<1>(p);
    else if (p.head == 2) syn_coarse<2>(p);
    else syn_coarse<3>(p);
    fence_proxy_async_global();
    cooperative_groups::this_grid().sync();
    fence_proxy_async_global();
  }
  const uint32_t ntiles = uint32_t(p.ntiles);
  if (warp == NW) {   // producer
    if (lane == 0) {
      for (int k = 0;; ++k) {
        const int s = k % p.stages;
        if (k >= p.stages) mbar_wait(&empty[s], uint32_t(k / p.stages - 1) & 1u);
        uint32_t t;
        if (DYN && k >= p.stages) t = atomicAdd(p.tile_ctr, 1u) + uint32_t(p.stages) * gridDim.x;
        else t = blockIdx.x + uint32_t(k) * gridDim.x;
        stile[s] = t;
        if (t >= ntiles) {
          mbar_arrive_plain(&full[s]);
          break;
        }
        if constexpr (SWZL > 0)
          syn_issue_tile_swz<SWZL>(p, maps, smem + s * p.stage_bytes, &full[s], DYN ? dyn_tile(t, ntiles, p.dyn_groups) : t);
        else if (p.issue_rev)
          syn_issue_tile_fine_first(p, maps, smem + s * p.stage_bytes, &full[s], DYN ? dyn_tile(t, ntiles, p.dyn_groups) : t);
        else
          syn_issue_tile_lane<false, false, false>(p, maps, smem + s * p.stage_bytes, &full[s],
                                                   DYN ? dyn_tile(t, ntiles, p.dyn_groups) : t, 0);
      }
    }
    return;
  }
  WarpScratch* sc = reinterpret_cast<WarpScratch*>(smem + p.p_off[0] + warp * kSynScratchBytes);
  for (int it = 0;; ++it) {
    const int s = it % p.stages;
    mbar_wait(&full[s], uint32_t(it / p.stages) & 1u);
    const uint32_t cval = stile[s];
    if (cval >= ntiles) break;
    const uint32_t tile = DYN ? dyn_tile(cval, ntiles, p.dyn_groups) : cval;
    const TileXY xy = tile_xy(tile, p.tiles_c, p.tiles_r, 32, TCF, -1);
    const unsigned char* stage = smem + s * p.stage_bytes;
    // column of the tile as the producer's boxes saw it (a ragged width runs its full tiles as a
    // launch of its own, starting at column tile p.ct0, with the last one clamped)
    const int64_t col0 = RAGGED ? tile_col0(p, xy.col0 / TCF + p.ct0) : xy.col0;
    const float* ll = reinterpret_cast<const float*>(stage + p.box_off[0][0]) + ((32 * warp) >> 5);
    warp_syn_steps<5, 5, false, TCF, false, SWZL>(p, ll, TCF >> 5, stage, warp, sc, xy.b, xy.row0, col0 + 32 * warp, col0);
    __syncwarp();
    if (lane == 0) mbar_arrive_plain(&empty[s]);
  }
}

template <int N>
__device__ __forceinline__ void cp_async_wait_rt(int n) {  // runtime-N wrapper (n in [0, N])
  if constexpr (N > 0) {
    if (n >= N) {
      cp_async_wait<N>();
      return;
    }
    cp_async_wait_rt<N - 1>(n);
  } else {
    cp_async_wait<0>();
  }
}

// MODE 0: all boxes by TMA; 2: everything by cp.async (LDGSTS).  (A register-LDG level-1 variant
// measured 5.19 TB/s vs 6.10 for cp.async and was removed; tools/sweep_syn.py history in profiles/.)
template <int LPFAST, int TRF, int TCF, int MODE>
__global__ void __launch_bounds__(LPFAST > 0 ? fast_threads(TRF, TCF) : kThreads2d,
                                  LPFAST > 0 ? FHWT_MINB_SYN * kThreads2d / fast_threads(TRF, TCF) : FHWT_MINB_SYN)
    syn2d_kernel(const __grid_constant__ Syn2dParams p,
                                                           const __grid_constant__ TmaMaps2d maps) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int j = 1; j <= p.Lp; ++j) prefetch_tmap(&maps.level[j]);
    prefetch_tmap(&maps.ll);
    for (int s = 0; s < p.stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();   // warp-uniform (see Refill)
  auto issue = [&](int64_t t, int s) { syn_issue_tile(p, maps, smem + s * p.stage_bytes, &bars[s], t, pol); };
  constexpr bool CPASYNC = MODE == 2 && LPFAST > 0;
  if constexpr (CPASYNC) {
    for (int s = 0; s < p.stages; ++s) {
      const int64_t t = blockIdx.x + int64_t(s) * gridDim.x;
      if (t < p.ntiles)
        syn_cp_async_tile<LPFAST, TRF, TCF>(p, smem + s * p.stage_bytes, t);
      else
        cp_async_commit();
    }
  } else if (tid < 32) {
    for (int s = 0; s < p.stages; ++s) {
      const int64_t t = blockIdx.x + int64_t(s) * gridDim.x;
      if (t < p.ntiles) issue(t, s);
    }
  }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++it) {
    const int s = it % p.stages;
    if constexpr (CPASYNC) {
      cp_async_wait_rt<7>(p.stages - 1);   // this thread's copies of the oldest stage have landed
      __syncthreads();                     // ... and everyone else's
    } else {
      mbar_wait(&bars[s], uint32_t(it / p.stages) & 1u);
    }
    const int64_t rt = tile / p.tiles_c, ct = tile - rt * p.tiles_c;
    const int64_t b = rt / p.tiles_r;
    const int64_t row0 = tile_row0(p, rt - b * p.tiles_r);
    unsigned char* stage = smem + s * p.stage_bytes;
    if constexpr (LPFAST > 0) {
      const float* ll = reinterpret_cast<const float*>(stage + p.box_off[0][0]);
      if (p.mask_mode == 0)
        syn_fast_step<LPFAST, TRF, TCF>(p, stage, smem, ll, TCF >> LPFAST, b, row0, tile_col0(p, ct + p.ct0));
      else
        syn_fast_step<LPFAST, TRF, TCF, false>(p, stage, smem, ll, p.box_pitch[LPFAST], b, row0,
                                               tile_col0(p, ct + p.ct0));
    } else {
      syn_tile(p, stage, smem, b, row0, tile_col0(p, ct + p.ct0));
    }
    __syncthreads();
    const int64_t nt = tile + int64_t(p.stages) * gridDim.x;
    if constexpr (CPASYNC) {
      if (nt < p.ntiles)
        syn_cp_async_tile<LPFAST, TRF, TCF>(p, smem + s * p.stage_bytes, nt);
      else
        cp_async_commit();
    } else if (tid < 32) {
      if (nt < p.ntiles) issue(nt, s);
    }
  }
}

// ------------------------------------------------------------------ single-level scalar kernels
// Used only when the row length is not a multiple of 4 (then levels == 1, since w % 2^levels == 0),
// where 16-byte vector / TMA access is impossible.  One thread per 2x2 block.
__global__ void ana2d_l1_scalar_kernel(const float* __restrict__ d, float* __restrict__ c, int64_t h, int64_t w,
                                       int64_t batch) {
  const int64_t hw = (h / 2) * (w / 2);
  const int64_t total = batch * hw;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / hw, rem = i - b * hw;
    const int64_t r = rem / (w / 2), q = rem - r * (w / 2);
    const float* x = d + b * h * w + (2 * r) * w + 2 * q;
    const float a = x[0], bb = x[1], cc = x[w], dd = x[w + 1];
    const float s1 = a + bb, s2 = cc + dd, d1 = a - bb, d2 = cc - dd;
    float* o = c + b * h * w;
    o[r * w + q] = (s1 + s2) * 0.5f;
    o[r * w + w / 2 + q] = (d1 + d2) * 0.5f;
    o[(h / 2 + r) * w + q] = (s1 - s2) * 0.5f;
    o[(h / 2 + r) * w + w / 2 + q] = (d1 - d2) * 0.5f;
  }
}

__global__ void syn2d_l1_scalar_kernel(const float* __restrict__ c, float* __restrict__ d, int64_t h, int64_t w,
                                       int64_t batch) {
  const int64_t hw = (h / 2) * (w / 2);
  const int64_t total = batch * hw;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / hw, rem = i - b * hw;
    const int64_t r = rem / (w / 2), q = rem - r * (w / 2);
    const float* o = c + b * h * w;
    const float ll = o[r * w + q], hl = o[r * w + w / 2 + q];
    const float lh = o[(h / 2 + r) * w + q], hh = o[(h / 2 + r) * w + w / 2 + q];
    const float s = ll + lh, t = hl + hh, s2 = ll - lh, t2 = hl - hh;
    float* x = d + b * h * w + (2 * r) * w + 2 * q;
    x[0] = (s + t) * 0.5f;
    x[1] = (s - t) * 0.5f;
    x[w] = (s2 + t2) * 0.5f;
    x[w + 1] = (s2 - t2) * 0.5f;
  }
}

// Pack fused with the row-band all-gather over peer memory: every LL element of this rank's band
// is stored straight into each peer's gather buffer (NVLink P2P stores through UVA pointers), at
// element offset rank * n.  One launch replaces pack + collective; a cross-rank barrier after it
// (the caller's) makes the stores visible.
__global__ void pack_ll_peers_kernel(const float* __restrict__ c, float* const* __restrict__ peers, int rank,
                                     int npeers, int64_t h, int64_t w, int64_t batch, int levels) {
  const int64_t hl = h >> levels, wl = w >> levels;
  const int64_t total = batch * hl * wl;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / (hl * wl), rem = i - b * hl * wl;
    const int64_t r = rem / wl, q = rem - r * wl;
    const float v = c[b * h * w + r * w + q];
    for (int k = 0; k < npeers; ++k) peers[k][int64_t(rank) * total + i] = v;
  }
}

__global__ void pack_ll_kernel(const float* __restrict__ c, float* __restrict__ ll, int64_t h, int64_t w,
                               int64_t batch, int levels) {
  const int64_t hl = h >> levels, wl = w >> levels;
  const int64_t total = batch * hl * wl;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / (hl * wl), rem = i - b * hl * wl;
    const int64_t r = rem / wl, q = rem - r * wl;
    ll[i] = c[b * h * w + r * w + q];
  }
}

int grid_for(int64_t total, int threads) {
  int64_t g = (total + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  return int(g < 1 ? 1 : g);
}

}  // namespace

// The dynamic-smem cap is raised to the device's opt-in maximum (not to `smem`), so a cached
// occupancy answer for a small configuration never leaves the cap below a later, larger launch.
// (minus the kernel's static shared memory, which shares the same per-block budget)
static cudaError_t raise_smem_cap(const void* fn) {
  int dev = 0, optin = 0;
  cudaFuncAttributes fa{};
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, fn);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - int(fa.sharedSizeBytes));
  return e;
}

// Fast variants: tile rows TRF in {8, 16, 32}, tile cols TCF in {128, 256}, levels LP <= log2(TRF).
template <int TRF, int TCF>
static const void* ana2d_fast_fn(int lp) {
  switch (lp) {
    case 1: return (const void*)ana2d_kernel<float, 1, TRF, TCF>;
    case 2: return (const void*)ana2d_kernel<float, 2, TRF, TCF>;
    case 3: return (const void*)ana2d_kernel<float, 3, TRF, TCF>;
    case 4:
      if constexpr (TRF >= 16) return (const void*)ana2d_kernel<float, 4, TRF, TCF>;
      return nullptr;
    case 5:
      if constexpr (TRF >= 32) return (const void*)ana2d_kernel<float, 5, TRF, TCF>;
      return nullptr;
    default: return nullptr;
  }
}

template <int TRF, int TCF, int MODE>
static const void* syn2d_fast_fn(int lp) {
  switch (lp) {
    case 1: return (const void*)syn2d_kernel<1, TRF, TCF, MODE>;
    case 2: return (const void*)syn2d_kernel<2, TRF, TCF, MODE>;
    case 3: return (const void*)syn2d_kernel<3, TRF, TCF, MODE>;
    case 4:
      if constexpr (TRF >= 16) return (const void*)syn2d_kernel<4, TRF, TCF, MODE>;
      return nullptr;
    case 5:
      if constexpr (TRF >= 32) return (const void*)syn2d_kernel<5, TRF, TCF, MODE>;
      return nullptr;
    default: return nullptr;
  }
}

template <template <int, int> class F>
static const void* by_geometry(int tr, int tc, int lp) {
  if (tr == 32) return tc == 128 ? F<32, 128>::get(lp) : F<32, 256>::get(lp);
  if (tr == 16) return tc == 128 ? F<16, 128>::get(lp) : F<16, 256>::get(lp);
  return tc == 128 ? F<8, 128>::get(lp) : F<8, 256>::get(lp);
}
template <int TRF, int TCF>
struct AnaF {
  static const void* get(int lp) { return ana2d_fast_fn<TRF, TCF>(lp); }
};
template <int TRF, int TCF>
struct SynF0 {
  static const void* get(int lp) { return syn2d_fast_fn<TRF, TCF, 0>(lp); }
};
template <int TRF, int TCF>
struct SynF2 {
  static const void* get(int lp) { return syn2d_fast_fn<TRF, TCF, 2>(lp); }
};

// fast: 0 = generic kernel; else (mode << 24) | (tile rows << 16) | (tile cols << 4) | LP
template <template <int> class K>
static const void* warp_fn(int lp) {
  switch (lp) {
    case 1: return K<1>::get();
    case 2: return K<2>::get();
    case 3: return K<3>::get();
    case 4: return K<4>::get();
    case 5: return K<5>::get();
    default: return nullptr;
  }
}
template <int LP>
struct SynW {
  static const void* get() { return (const void*)syn2d_warp_kernel<LP>; }
};
template <int LP>
struct SynWS {
  static const void* get() { return (const void*)syn2d_warp_kernel<LP, true>; }
};
template <int LP>
struct SynW512 {
  static const void* get() { return (const void*)syn2d_warp_kernel<LP, false, 512>; }
};
template <int LP>
struct SynW128 {
  static const void* get() { return (const void*)syn2d_warp_kernel<LP, false, 128>; }
};
template <int LP>
struct SynWS128 {
  static const void* get() { return (const void*)syn2d_warp_kernel<LP, true, 128>; }
};

static const void* ana2d_fn(bool in_f64, int fast) {
  if (in_f64) return (const void*)ana2d_kernel<double, 0, 0, 0>;
  if (fast == 0) return (const void*)ana2d_kernel<float, 0, 0, 0>;
  if (((fast >> 24) & 0xff) == 5) return (const void*)ana2d_fused3_kernel;
  if (((fast >> 24) & 0xff) == 7) return (const void*)ana2d_lean_kernel<false>;
  if (((fast >> 24) & 0xff) == 8) return (const void*)ana2d_lean_kernel<true>;
  return by_geometry<AnaF>((fast >> 16) & 0xff, (fast >> 4) & 0xfff, fast & 15);
}

static const void* syn2d_fn(int fast) {
  if (fast == 0) return (const void*)syn2d_kernel<0, 0, 0, 0>;
  const int mode = (fast >> 24) & 0xff;
  const bool narrow = ((fast >> 4) & 0xfff) == 128;
  if (mode == 3 && ((fast >> 4) & 0xfff) == 512) return (fast & 15) == 5 ? SynW512<5>::get() : nullptr;
  if (mode == 9) return (fast & 15) == 5 ? (const void*)syn2d_warp_kernel<5, false, 256, true> : nullptr;
  if (mode == 14)   // producer K4, global order, level-1/2 boxes swizzled
    return (fast & 15) == 5 && ((fast >> 4) & 0xfff) == 256 ? (const void*)syn2d_prod_kernel<true, 256, false, 2> : nullptr;
  if (mode >= 10 && mode <= 13) {   // producer K4: 10 / 11 static / global order, 12 / 13 the same, ragged
    if ((fast & 15) != 5) return nullptr;
    if (((fast >> 4) & 0xfff) == 512)
      return mode == 11 ? (const void*)syn2d_prod_kernel<true, 512> : mode == 10 ? (const void*)syn2d_prod_kernel<false, 512>
             : mode == 13 ? (const void*)syn2d_prod_kernel<true, 512, true> : (const void*)syn2d_prod_kernel<false, 512, true>;
    return mode == 11 ? (const void*)syn2d_prod_kernel<true> : mode == 10 ? (const void*)syn2d_prod_kernel<false>
           : mode == 13 ? (const void*)syn2d_prod_kernel<true, 256, true> : (const void*)syn2d_prod_kernel<false, 256, true>;
  }
  if (mode == 3) return narrow ? warp_fn<SynW128>(fast & 15) : warp_fn<SynW>(fast & 15);
  if (mode == 6) return narrow ? warp_fn<SynWS128>(fast & 15) : warp_fn<SynWS>(fast & 15);
  return mode == 2 ? by_geometry<SynF2>((fast >> 16) & 0xff, (fast >> 4) & 0xfff, fast & 15)
                   : by_geometry<SynF0>((fast >> 16) & 0xff, (fast >> 4) & 0xfff, fast & 15);
}

int fast_threads_rt(int fast) {   // threads of a compile-time fast variant (code as in ana2d_fn)
  return fast == 0 ? kThreads2d : fast_threads((fast >> 16) & 0xff, (fast >> 4) & 0xfff);
}
int ana2d_threads(int fast) {
  const int mode = (fast >> 24) & 0xff;
  return mode == 5 ? 288 : fast_threads_rt(fast);
}
int syn2d_threads(int fast) {
  const int mode = (fast >> 24) & 0xff;
  if (mode >= 10 && mode <= 14) return ((fast >> 4) & 0xfff) + 32;   // compute warps + the producer warp
  return (mode == 3 || mode == 6 || mode == 9) ? ((fast >> 4) & 0xfff) : fast_threads_rt(fast);   // one warp per 32 columns
}

cudaError_t ana2d_occupancy(bool in_f64, int fast_lp, size_t smem, int* blocks_per_sm) {
  const void* fn = ana2d_fn(in_f64, fast_lp);
  cudaError_t e = raise_smem_cap(fn);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fn, ana2d_threads(in_f64 ? 0 : fast_lp), smem);
}

cudaError_t syn2d_occupancy(int fast_lp, size_t smem, int* blocks_per_sm) {
  const void* fn = syn2d_fn(fast_lp);
  cudaError_t e = raise_smem_cap(fn);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fn, syn2d_threads(fast_lp), smem);
}

cudaError_t launch_ana2d(const Ana2dParams& p, const CUtensorMap& in_map, bool in_f64, int fast_lp, int grid,
                         size_t smem, cudaStream_t s) {
  count_launch();
  void* args[] = {const_cast<Ana2dParams*>(&p), const_cast<CUtensorMap*>(&in_map)};
  if (p.tail > 0)
    return cudaLaunchCooperativeKernel(ana2d_fn(in_f64, fast_lp), dim3(grid), dim3(ana2d_threads(in_f64 ? 0 : fast_lp)),
                                       args, smem, s);
  return cudaLaunchKernel(ana2d_fn(in_f64, fast_lp), dim3(grid), dim3(ana2d_threads(in_f64 ? 0 : fast_lp)), args,
                          smem, s);
}

cudaError_t launch_syn2d(const Syn2dParams& p, const TmaMaps2d& maps, int fast_lp, int grid, size_t smem,
                         cudaStream_t s) {
  count_launch();
  void* args[] = {const_cast<Syn2dParams*>(&p), const_cast<TmaMaps2d*>(&maps)};
  const dim3 block(syn2d_threads(fast_lp));
  if (p.head > 0) return cudaLaunchCooperativeKernel(syn2d_fn(fast_lp), dim3(grid), block, args, smem, s);
  return cudaLaunchKernel(syn2d_fn(fast_lp), dim3(grid), block, args, smem, s);
}

cudaError_t launch_ana2d_l1_scalar(const float* d, float* c, int64_t h, int64_t w, int64_t batch, cudaStream_t s) {
  count_launch();
  ana2d_l1_scalar_kernel<<<grid_for(batch * (h / 2) * (w / 2), 256), 256, 0, s>>>(d, c, h, w, batch);
  return cudaGetLastError();
}

cudaError_t launch_syn2d_l1_scalar(const float* c, float* d, int64_t h, int64_t w, int64_t batch, cudaStream_t s) {
  count_launch();
  syn2d_l1_scalar_kernel<<<grid_for(batch * (h / 2) * (w / 2), 256), 256, 0, s>>>(c, d, h, w, batch);
  return cudaGetLastError();
}

cudaError_t launch_pack_ll_peers(const float* c, float* const* peers, int rank, int npeers, int64_t h, int64_t w,
                                 int64_t batch, int levels, cudaStream_t s) {
  count_launch();
  pack_ll_peers_kernel<<<grid_for(batch * (h >> levels) * (w >> levels), 256), 256, 0, s>>>(c, peers, rank, npeers, h,
                                                                                             w, batch, levels);
  return cudaGetLastError();
}

#ifdef FHWT_PHASE_TIMING
extern "C" int fhwt_debug_phases(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_phase, sizeof(g_phase)) != cudaSuccess) return -1;
  if (reset) {
    static const unsigned long long zero[32] = {};
    if (cudaMemcpyToSymbol(g_phase, zero, sizeof(zero)) != cudaSuccess) return -1;
  }
  return 32;
}
#endif

cudaError_t launch_pack_ll(const float* c, float* ll, int64_t h, int64_t w, int64_t batch, int levels,
                           cudaStream_t s) {
  count_launch();
  pack_ll_kernel<<<grid_for(batch * (h >> levels) * (w >> levels), 256), 256, 0, s>>>(c, ll, h, w, batch, levels);
  return cudaGetLastError();
}

}  // namespace fhwt
