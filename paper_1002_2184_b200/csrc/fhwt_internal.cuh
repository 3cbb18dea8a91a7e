// Internal declarations shared by the fhwt CUDA translation units (not part of the C ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fhwt {

// fl(1/√2): the polyphase component b00 = a00.
constexpr float kS32 = 0.70710678118654752440f;
constexpr double kS64 = 0.70710678118654752440;

// Levels per fused pass: 2-D tiles of 32 rows cover 5 levels, 1-D warp
// chunks of 1024 samples cover 10 levels.
constexpr int kMaxLevels2dPass = 5;
constexpr int kMaxLevels1dPass = 10;
constexpr int kChunk1d = 1024;
constexpr int kThreads2d = 256;
constexpr int kThreads1d = 256;

// Warp-decoupled 2-D synthesis (haar2d.cu syn2d_warp_kernel): 32 x 256 tiles, warp w owns the
// 32 x 32 block at columns [32w, 32w + 32); per-warp LL scratch (LL1 16x16, LL2 8x8, LL3 4x4, LL4 2x2).
constexpr int kSynScratchBytes = 1408;

// First global level computed in fp64 (levels 1..3 fp32).  DESIGN.md "Precision".
constexpr int kFirstF64Level = 4;

// ------------------------------------------------------------------ 2-D pass parameters
struct Ana2dParams {
  float* out;            // Mallat coefficients, image 0, row pitch W (fp32)
  double* ws_out;        // LL_{g0+Lp} hand-off (fp64) when !final_pass; pitch Win >> Lp
  int64_t H, W;          // full image dims (output layout)
  int64_t Hin, Win;      // this pass's input dims per image (= H >> g0, W >> g0)
  int64_t batch;
  int Lp, g0;            // levels in this pass, global level offset
  int TR, TC;            // tile rows / cols (input coordinates)
  int64_t tiles_r;       // row tiles per image
  int64_t tiles_c;       // column tiles
  int64_t ntiles;
  int stages;
  uint32_t stage_bytes, p_off[2], bar_off;
  int final_pass;
  int mask_mode;         // fast variants: 0 all tiles full, 1 last column tile ragged (masked stores)
  int aligned_levels;    // levels j with even band offsets (unchecked 8-B stores): 1..aligned_levels
  int clamp_last;        // ragged width: the last column tile starts at Win - TC (see tile_col0)
  int clamp_rows;        // Hin % TR != 0: the last row tile starts at Hin - TR (see tile_row0)
  int row_pad;           // clamp_rows: tiles_r * TR - Hin (rows the last tile moves up)
  int fused;             // 32 x 256 fast tiles, LP >= 3: levels 2+3 and 4+5 fused (FHWT_ANA_FUSED, default 1)
  int tail;              // > 0: after the tiles, a grid barrier and levels 6..5+tail of the fp64 LL5
                         // hand-off in the same (cooperative) launch (ana_coarse); 0: none
  int l2hint;            // TMA loads: 0 no cache-policy operand (default), 1 evict_first, 2 evict_normal, 3 evict_last
  unsigned* tile_ctr;    // dynamic tile order (lean K1, vmode 8): next-tile counter, zeroed before the launch
  int dyn_groups;        // dynamic order: counter value c -> tile (c % G) * (ntiles / G) + c / G (G = 1: c)
  int row_boxes;         // 1: the map's box is one row and TR boxes are issued per tile (rows of
                         // 128-B multiples; TMA smem destinations must be 128-B aligned); 0: one TR-row box
  const float* in;       // first-pass input (fp32 d), read directly by the register-load kernel (haar2d_ana.cu)
};

struct Syn2dParams {
  const float* coeffs;   // Mallat coefficients (pitch W), read by the cp.async variant
  const float* ll_ws;    // LL_{g0+Lp} source in the workspace (cp.async variant; pitch pitch4(Win >> Lp))
  float* out;            // d_R (final pass, pitch W) or the LL_{g0} hand-off (pitch Win)
  int64_t out_pitch;
  int64_t H, W;          // full image dims (coefficient layout)
  int64_t Hin, Win;      // this pass's OUTPUT dims per image (= H >> g0, W >> g0)
  int64_t batch;
  int Lp, g0;
  int TR, TC;
  int64_t tiles_r, tiles_c, ntiles;
  int64_t ct0;             // first column tile of this launch (a ragged width runs as two launches)
  int clamp_last;          // ragged width: the last column tile starts at Win - TC (see tile_col0)
  int clamp_rows;          // Hin % TR != 0: the last row tile starts at Hin - TR (see tile_row0)
  int stages;
  uint32_t stage_bytes, bar_off;
  uint32_t box_off[6][3];  // per pass-level j (1..Lp): offsets of HL, LH, HH boxes; [0][0] = LL box
  int box_pitch[6];        // smem pitch (elements) of level-j boxes; [0] unused
  int hoff[6];             // HL/HH boxes start hoff[j] columns left of the band block (TMA box
                           // starts must be 16-B aligned; hoff = (W >> g) & 3)
  uint32_t p_off[2];
  uint32_t tx_bytes;       // bytes landed per stage
  int ll_from_ws;          // LL_{g0+Lp} comes from the workspace map (else from coeffs)
  int mask_mode;           // fast variants: 0 full tiles, hoff = 0; 1 ragged / shifted boxes (TMA mode only)
  int head;                // > 0: levels 5+head..6 rebuilt into the fp32 LL5 workspace first, then a grid
                           // barrier, then the tiles, in one cooperative launch (syn_coarse); 0: none
  float* ll_ws_out;        // head > 0: the LL5 workspace the head phase writes (same buffer as ll_ws)
  int row_boxes[6];        // per pass-level j: one-row boxes (1) or one (TR >> j)-row box (0); see Ana2dParams
  unsigned* tile_ctr;      // dynamic tile order (warp kernel, mode 9): next-tile counter, zeroed before the launch
  int dyn_groups;          // as Ana2dParams::dyn_groups
  int issue_rev;           // producer K4: issue level-1 boxes first (experiment knob FHWT_SYN_ISSUE_REV)
  int l2mode;              // warp kernel's TMA loads: 0 L2::evict_first, 1 evict_normal, 2 evict_last, 3 no policy (default)
  int swz;                 // producer K4: levels 1..swz (2) boxes through the 128-B-swizzled 3-D maps (TmaMaps2d::sw)
};

struct TmaMaps2d {
  CUtensorMap level[6];  // coeff view box for pass-level j = 1..Lp ([0] unused)
  CUtensorMap ll;        // LL_{g0+Lp} source box
  CUtensorMap sw[3];     // [1], [2]: level-1/2 coefficient view as {32 floats, W/32 lines, rows} with
                         // SWIZZLE_128B (producer K4, Syn2dParams::swz); [0] unused
};

// ------------------------------------------------------------------ small 2-D images
// (haar2d_small.cu) chunks of G whole images, each h * w <= 4096 samples, all levels in one pass
struct Small2dParams {
  const float* in;       // analysis: d; synthesis: coefficients (Mallat layout per image)
  float* out;            // analysis: coefficients; synthesis: d_R
  int64_t batch, nchunks;
  int H, W, L, G;        // image dims, levels, images per chunk
  int stages;
  uint32_t stage_bytes, off_out, off_t[2], off_d[2], off_bar;
};

// ------------------------------------------------------------------ 1-D pass parameters
struct Haar1dParams {
  const void* in;        // analysis: pass input (fp32 d or fp64 ws); synthesis: approx source
  int64_t in_pitch;      // elements between signals of `in`
  float* coeffs_out;     // analysis: coefficient array (pitch n)
  const float* coeffs_in;  // synthesis: coefficient array (pitch n)
  void* out;             // analysis: approx hand-off (fp64 ws) / synthesis: output (fp32)
  int64_t out_pitch;
  int64_t n;             // full signal length (coefficient pitch)
  int64_t nin;           // this pass's signal length (= n >> g0)
  int64_t batch;
  int64_t chunks;        // chunks per signal
  int64_t nwarps;
  int Lp, g0;
  int final_pass;        // analysis: approx goes to coeffs; synthesis: output is d_R
  int tail;              // > 0 (first pass, Lp = 10, chunks | 8): levels 11..10+tail run inside the
                         // CTA (its 8 warps hold whole signals) instead of a second pass
};

// launchers (return cudaError_t of the launch)
// fast_lp > 0 selects the compile-time full-tile variant: fast_lp = (tile cols << 4) | levels
cudaError_t launch_ana2d(const Ana2dParams& p, const CUtensorMap& in_map, bool in_f64, int fast_lp, int grid,
                         size_t smem, cudaStream_t s);   // cooperative launch when p.tail > 0
cudaError_t launch_syn2d(const Syn2dParams& p, const TmaMaps2d& maps, int fast_lp, int grid, size_t smem,
                         cudaStream_t s);
int syn2d_threads(int fast_lp);   // CTA size of a synthesis variant (fast code as in launch_syn2d)
cudaError_t ana2d_occupancy(bool in_f64, int fast_lp, size_t smem, int* blocks_per_sm);
// Warp-specialised analysis of full 32 x 256 tiles at LP = 5 (haar2d_ana.cu, K1 v2)
int ana2d_ws_threads();
size_t ana2d_ws_smem(int stages, uint32_t* ll1_off, uint32_t* bar_off);
cudaError_t ana2d_ws_occupancy(size_t smem, int* blocks_per_sm);
cudaError_t launch_ana2d_ws(const Ana2dParams& p, const CUtensorMap& in_map, int grid, size_t smem, cudaStream_t s);
// Synthesis with warp-private level-1 slices (haar2d_syn.cu, FHWT_SYN_MODE=7): 32 x 256 tiles, LP = 5
size_t syn2d_wp_layout(Syn2dParams* p);   // fills box_off, p_off, stage_bytes, bar_off; returns smem bytes
cudaError_t syn2d_wp_occupancy(size_t smem, int* blocks_per_sm);
cudaError_t launch_syn2d_wp(const Syn2dParams& p, const TmaMaps2d& maps, int grid, size_t smem, cudaStream_t s);
// ... and the same fused chain with register (LDG) loads, no input staging (FHWT_ANA_FUSED=11;
// variant: 0 = 3 CTAs/SM, 1 = 4 CTAs/SM, 2 = next tile prefetched into registers at 2 CTAs/SM)
cudaError_t ana2d_ldg_occupancy(size_t smem, int* blocks_per_sm, int variant);
cudaError_t launch_ana2d_ldg(const Ana2dParams& p, int grid, size_t smem, cudaStream_t s, int variant);
cudaError_t syn2d_occupancy(int fast_lp, size_t smem, int* blocks_per_sm);
// f64all (first pass of a decomposition deeper than 10 levels): levels 1-3 in fp64 too, so the only
// error left is the final rounding of each output (the 1-D reading R14)
cudaError_t launch_ana1d(const Haar1dParams& p, bool in_f64, cudaStream_t s, bool f64all = false);
cudaError_t launch_syn1d(const Haar1dParams& p, cudaStream_t s);
cudaError_t launch_ana2d_l1_scalar(const float* d, float* c, int64_t h, int64_t w, int64_t batch, cudaStream_t s);
cudaError_t launch_syn2d_l1_scalar(const float* c, float* d, int64_t h, int64_t w, int64_t batch, cudaStream_t s);
cudaError_t launch_ana1d_l1_scalar(const float* d, float* c, int64_t n, int64_t batch, cudaStream_t s);
cudaError_t launch_syn1d_l1_scalar(const float* c, float* d, int64_t n, int64_t batch, cudaStream_t s);
cudaError_t launch_pack_ll_peers(const float* c, float* const* peers, int rank, int npeers, int64_t h, int64_t w,
                                 int64_t batch, int levels, cudaStream_t s);
cudaError_t launch_pack_ll(const float* c, float* ll, int64_t h, int64_t w, int64_t batch, int levels,
                           cudaStream_t s);

// Direct-form baseline (direct.cu, §8(f) f3): `batch` groups of `count` lines of `len` samples,
// sample n of line s of group b at base[b * bstride + s * sstride + n * nstride].
struct Lines_t {
  int64_t batch, bstride, count, sstride, len, nstride;
};
cudaError_t direct_analysis_lines(const float* x, Lines_t lx, float* a, Lines_t la, float* d, Lines_t ld, float* y0,
                                  float* y1, cudaStream_t s);
cudaError_t direct_synthesis_lines(const float* a, Lines_t la, const float* d, Lines_t ld, float* r, Lines_t lr,
                                   float* u0, float* u1, cudaStream_t s);

// LL-only uint8 lowpass path (lowpass.cu, §8(f) f1)
size_t lowpass_workspace_bytes(int64_t h, int64_t w, int64_t batch, int levels);
size_t lowpass_bf16_workspace_bytes(int64_t h, int64_t w, int64_t batch, int levels);
cudaError_t launch_lowpass_bf16(const uint16_t* d, float* ll, int64_t h, int64_t w, int64_t batch, int levels,
                                void* ws, cudaStream_t s);
cudaError_t launch_lowpass_u8(const uint8_t* d, float* ll, int64_t h, int64_t w, int64_t batch, int levels, void* ws,
                              cudaStream_t s);

// one_d: the 1-D short-signal kernels (H = 1, W = n)
cudaError_t small2d_occupancy(bool analysis, size_t smem, int* blocks_per_sm, bool one_d = false);
cudaError_t launch_small2d(const Small2dParams& p, bool analysis, int grid, size_t smem, cudaStream_t s,
                           bool one_d = false);

void count_launch();
bool tuning_enabled();   // FHWT_TUNING=1: honour the FHWT_* sweep knobs (fhwt_api.cu env_int)

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_LOOP:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra WAIT_DONE;\n"
      "bra WAIT_LOOP;\n"
      "WAIT_DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// TMA 2-D tile load global -> shared, completion counted on `bar` (complete_tx bytes).
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d_nohint(void* smem_dst, const CUtensorMap* map, int c0, int c1,
                                                   uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// TMA 3-D tile load (the swizzled level-1/2 synthesis boxes: {32 floats, lines, rows}).
__device__ __forceinline__ void tma_load_3d_nohint(void* smem_dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                   uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// Ampere-style async copy (LDGSTS): 16 B global -> shared, completion tracked per thread by groups.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Dynamic tile order: counter value c -> tile index (G interleaved contiguous streams; G = 1 is the
// plain global order).  G divides ntiles (checked on the host).
__device__ __forceinline__ uint32_t dyn_tile(uint32_t c, uint32_t ntiles, int G) {
  if (G <= 1) return c;
  const uint32_t per = ntiles / uint32_t(G);
  return (c % uint32_t(G)) * per + c / uint32_t(G);
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// streaming global accesses (read once / written once: do not allocate in L1)
__device__ __forceinline__ float4 ldg_stream4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ float2 ldg_stream2(const float* p) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ float ldg_stream1(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
// Streaming stores of the transform outputs.  FHWT_STG_MODE (build-time experiment): 0 = L1 no-allocate
// (default), 1 = + L2 evict_first policy, 2 = .cs, 3 = plain st.global, 4 = + L2 evict_last policy.
#ifndef FHWT_STG_MODE
#define FHWT_STG_MODE 0
#endif
#if FHWT_STG_MODE == 1 || FHWT_STG_MODE == 4
__device__ __forceinline__ uint64_t stg_policy() {
  uint64_t p;
#if FHWT_STG_MODE == 1
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
#else
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
#endif
  return p;
}
#define FHWT_STG_PFX "st.global.L1::no_allocate.L2::cache_hint"
#define FHWT_STG_POL , "l"(stg_policy())
#define FHWT_STG_POLARG(n) ", %" #n
#else
#if FHWT_STG_MODE == 2
#define FHWT_STG_PFX "st.global.cs"
#elif FHWT_STG_MODE == 3
#define FHWT_STG_PFX "st.global"
#else
#define FHWT_STG_PFX "st.global.L1::no_allocate"
#endif
#define FHWT_STG_POL
#define FHWT_STG_POLARG(n) ""
#endif
__device__ __forceinline__ void stg_stream4(float* p, float4 v) {
  asm volatile(FHWT_STG_PFX ".v4.f32 [%0], {%1, %2, %3, %4}" FHWT_STG_POLARG(5) ";" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w) FHWT_STG_POL
               : "memory");
}
__device__ __forceinline__ void stg_stream2(float* p, float2 v) {
  asm volatile(FHWT_STG_PFX ".v2.f32 [%0], {%1, %2}" FHWT_STG_POLARG(3) ";" ::"l"(p), "f"(v.x), "f"(v.y) FHWT_STG_POL
               : "memory");
}
__device__ __forceinline__ void stg_stream1(float* p, float v) {
  asm volatile(FHWT_STG_PFX ".f32 [%0], %1" FHWT_STG_POLARG(2) ";" ::"l"(p), "f"(v) FHWT_STG_POL : "memory");
}

}  // namespace fhwt
