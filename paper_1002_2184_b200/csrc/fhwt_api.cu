// C ABI of the Fast Haar library (include/fhwt.h): validation, plans, kernel-pass scheduling,
// TMA descriptor encoding, workspace, host-buffer streaming.  No torch types cross this boundary.
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fhwt.h"
#include "fhwt_internal.cuh"

using namespace fhwt;

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

fhwt_status fail(fhwt_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

fhwt_status cuda_fail(cudaError_t e, const char* what) {
  return fail(FHWT_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define FHWT_CUDA(call, what)                 \
  do {                                        \
    cudaError_t e_ = (call);                  \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

#define FHWT_TRY(call)                   \
  do {                                   \
    fhwt_status st_ = (call);            \
    if (st_ != FHWT_OK) return st_;      \
  } while (0)

int64_t pitch4(int64_t x) { return (x + 3) & ~int64_t(3); }
size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Pass {
  int g0, Lp;
};

std::vector<Pass> make_passes(int levels, int per_pass) {
  std::vector<Pass> v;
  for (int g = 0; g < levels; g += per_pass) v.push_back({g, std::min(per_pass, levels - g)});
  return v;
}

// ------------------------------------------------------------------ device info / TMA encode
struct DevInfo {
  int sms = 0;
  int major = 0;
  bool ok = false;
};

fhwt_status device_info(DevInfo* out) {
  static std::mutex mu;
  static DevInfo cache[64];
  int dev = 0;
  FHWT_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
  if (dev < 0 || dev >= 64) return fail(FHWT_ERR_NO_DEVICE, "device index %d", dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!cache[dev].ok) {
    FHWT_CUDA(cudaDeviceGetAttribute(&cache[dev].sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
    FHWT_CUDA(cudaDeviceGetAttribute(&cache[dev].major, cudaDevAttrComputeCapabilityMajor, dev), "cc");
    cache[dev].ok = true;
  }
  if (cache[dev].major != 10)
    return fail(FHWT_ERR_NO_DEVICE, "device %d has compute capability %d.x; this library is built for sm_100a",
                dev, cache[dev].major);
  *out = cache[dev];
  return FHWT_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int env_int(const char* name, int dflt);

// L2 sector promotion of the TMA tensor maps (FHWT_TMA_L2PROMO: 0 none, 1 64 B, 2 128 B, 3 256 B;
// default 256 B)
CUtensorMapL2promotion l2_promotion() {
  switch (env_int("FHWT_TMA_L2PROMO", 3)) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

// 2-D row-major tensor view: `cols` x `rows` elements, row pitch `pitch_elems`, box bw x bh.
fhwt_status encode_2d(CUtensorMap* m, const void* base, bool f64, int64_t cols, int64_t rows, int64_t pitch_elems,
                      int bw, int bh) {
  auto fn = get_encode();
  if (!fn) return fail(FHWT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  const size_t es = f64 ? 8 : 4;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(pitch_elems) * es};
  cuuint32_t box[2] = {cuuint32_t(bw), cuuint32_t(bh)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(FHWT_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d): dims %lld x %lld pitch %lld box %d x %d", int(r),
                (long long)cols, (long long)rows, (long long)pitch_elems, bw, bh);
  return FHWT_OK;
}

// The level-j coefficient array as a 3-D view {32 floats, W / 32 lines of 128 B, rows} with
// SWIZZLE_128B, box {32, nch, bh}: one (bh)-row band box of nch * 128 B per row, landed with each
// 128-B line's 16-B granules permuted (haar2d.cu syn_issue_tile_swz / warp_syn_level<SWZ>).
fhwt_status encode_3d_swz(CUtensorMap* m, const void* base, int64_t W, int64_t rows, int nch, int bh) {
  auto fn = get_encode();
  if (!fn) return fail(FHWT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t dims[3] = {32, cuuint64_t(W / 32), cuuint64_t(rows)};
  cuuint64_t strides[2] = {128, cuuint64_t(W) * 4};
  cuuint32_t box[3] = {32, cuuint32_t(nch), cuuint32_t(bh)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, l2_promotion(),
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(FHWT_ERR_CUDA, "cuTensorMapEncodeTiled (swizzled) failed (%d): W %lld rows %lld box %d x %d", int(r),
                (long long)W, (long long)rows, nch, bh);
  return FHWT_OK;
}

// Tuning knobs (defaults chosen by measurement).  The env overrides exist
// only for the sweeps in tools/ and the A/B tests: every FHWT_* variable is ignored unless
// FHWT_TUNING=1 is set too, so a stray variable in a user's environment cannot change which
// kernel, tile or ring depth runs (results are bitwise equal either way; speed is not).
}  // namespace
namespace fhwt {
bool tuning_enabled() {
  const char* t = std::getenv("FHWT_TUNING");
  return t && t[0] == '1' && t[1] == 0;
}
}  // namespace fhwt
namespace {
int env_int(const char* name, int dflt) {
  if (!tuning_enabled()) return dflt;
  const char* v = std::getenv(name);
  return (v && *v) ? std::atoi(v) : dflt;
}

// occupancy cache: (family, fast, smem) -> blocks per SM.  family 0 = ana2d fp32, 1 = ana2d fp64,
// 2 = syn2d; fast = the variant code (0 = generic kernel).
fhwt_status occupancy(int family, int fast, size_t smem, int* bps) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int64_t, size_t>, int>> cache;
  int dev = 0;
  FHWT_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
  const int64_t key = ((int64_t(family) << 40) | (int64_t(fast) << 8)) + dev;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& e : cache)
      if (e.first.first == key && e.first.second == smem) {
        *bps = e.second;
        return FHWT_OK;
      }
  }
  cudaError_t e = family == 2 ? syn2d_occupancy(fast, smem, bps) : ana2d_occupancy(family == 1, fast, smem, bps);
  if (e != cudaSuccess) return cuda_fail(e, "occupancy query");
  if (*bps < 1) return fail(FHWT_ERR_CUDA, "kernel does not fit on an SM with %zu B shared memory", smem);
  std::lock_guard<std::mutex> lk(mu);
  cache.push_back({{key, smem}, *bps});
  return FHWT_OK;
}

// ------------------------------------------------------------------ validation
fhwt_status check_bank(const fhwt_filter_bank* fb) {
  if (!fb) return FHWT_OK;
  const double s = 1.0 / std::sqrt(2.0);
  const double ref[8] = {s, s, -s, s, s, s, s, -s};
  const double got[8] = {fb->b0[0], fb->b0[1], fb->b1[0], fb->b1[1], fb->a0[0], fb->a0[1], fb->a1[0], fb->a1[1]};
  for (int i = 0; i < 8; ++i)
    if (!(std::fabs(got[i] - ref[i]) <= 1e-12))
      return fail(FHWT_ERR_UNSUPPORTED_FILTER, "tap %d = %.17g differs from the section II Haar set", i, got[i]);
  if (fb->M != 2) return fail(FHWT_ERR_UNSUPPORTED_FILTER, "decimation factor M = %d (Haar needs M = 2)", fb->M);
  return FHWT_OK;
}

fhwt_status check_1d(int64_t n, int64_t batch, int levels) {
  if (n < 0 || batch < 0) return fail(FHWT_ERR_INVALID_ARG, "negative size n=%lld batch=%lld", (long long)n, (long long)batch);
  if (n == 0 || batch == 0) return fail(FHWT_ERR_EMPTY, "empty input n=%lld batch=%lld", (long long)n, (long long)batch);
  if (levels < 1 || levels > 62) return fail(FHWT_ERR_INVALID_LEVELS, "levels=%d", levels);
  if (n % 2) return fail(FHWT_ERR_ODD_LENGTH, "odd length n=%lld", (long long)n);
  if (n % (int64_t(1) << levels)) return fail(FHWT_ERR_INSUFFICIENT_LENGTH, "n=%lld not divisible by 2^%d", (long long)n, levels);
  return FHWT_OK;
}

fhwt_status check_2d(int64_t h, int64_t w, int64_t batch, int levels) {
  if (h < 0 || w < 0 || batch < 0) return fail(FHWT_ERR_INVALID_ARG, "negative size");
  if (h == 0 || w == 0 || batch == 0) return fail(FHWT_ERR_EMPTY, "empty input %lldx%lld batch %lld", (long long)h, (long long)w, (long long)batch);
  if (levels < 1 || levels > 62) return fail(FHWT_ERR_INVALID_LEVELS, "levels=%d", levels);
  if (h % 2 || w % 2) return fail(FHWT_ERR_ODD_LENGTH, "odd dimension %lldx%lld", (long long)h, (long long)w);
  if (h % (int64_t(1) << levels) || w % (int64_t(1) << levels))
    return fail(FHWT_ERR_INSUFFICIENT_LENGTH, "%lldx%lld not divisible by 2^%d", (long long)h, (long long)w, levels);
  if (h >= (int64_t(1) << 30) || w >= (int64_t(1) << 30))   // TMA coordinates are int32 (batches are split)
    return fail(FHWT_ERR_INVALID_ARG, "h=%lld or w=%lld exceeds the 2^30 TMA coordinate range", (long long)h,
                (long long)w);
  return FHWT_OK;
}

// Stream-ordered workspace allocations (one-shot calls) come from the device's default memory pool;
// raising its release threshold keeps freed blocks cached instead of returning them to the driver
// at every synchronisation (which made each call pay a fresh allocation).
fhwt_status ws_alloc(void** p, size_t bytes, cudaStream_t s) {
  static std::once_flag flags[64];
  int dev = 0;
  FHWT_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
  if (dev >= 0 && dev < 64)
    std::call_once(flags[dev], [dev] {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
    });
  FHWT_CUDA(cudaMallocAsync(p, bytes, s), "workspace cudaMallocAsync");
  return FHWT_OK;
}

fhwt_status check_ptrs(const void* in, const void* out, size_t bytes) {
  if (!in || !out) return fail(FHWT_ERR_INVALID_ARG, "null buffer pointer");
  const char* a = static_cast<const char*>(in);
  const char* b = static_cast<const char*>(out);
  if (a < b + bytes && b < a + bytes) return fail(FHWT_ERR_INVALID_ARG, "input and output buffers overlap (no in-place transform)");
  if ((reinterpret_cast<uintptr_t>(in) & 3) || (reinterpret_cast<uintptr_t>(out) & 3))
    return fail(FHWT_ERR_MISALIGNED, "buffers must be at least 4-byte aligned");
  return FHWT_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

namespace fhwt {
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace fhwt

// ---------------------------------------------------------------------- plan object
struct fhwt_plan_s {
  int kind;  // 1 or 2
  int device;  // CUDA device the plan runs on; -1 = the device current at each call
  int64_t n, h, w, batch;
  int levels;
  std::vector<Pass> passes;
  std::vector<size_t> ws_off;  // per pass boundary k (after pass k, k < passes-1)
  size_t ctr_off;              // 2-D: tile counters of the dynamic tile order (analysis +0, synthesis +128)
  size_t ws_bytes;
};

namespace {

constexpr size_t kCtrBytes = 256;

void plan_layout(fhwt_plan_s* p) {
  p->passes = make_passes(p->levels, p->kind == 2 ? kMaxLevels2dPass : kMaxLevels1dPass);
  p->ws_off.clear();
  size_t off = 0;
  for (size_t k = 0; k + 1 < p->passes.size(); ++k) {
    const int g = p->passes[k].g0 + p->passes[k].Lp;
    size_t elems = p->kind == 2 ? size_t(p->batch) * size_t(p->h >> g) * size_t(pitch4(p->w >> g))
                                : size_t(p->batch) * size_t(pitch4(p->n >> g));
    p->ws_off.push_back(off);
    off = align_up(off + elems * sizeof(double), 256);
  }
  // 2-D: 256 B for the tile counters of the dynamic tile order (zeroed by a stream-ordered memset
  // before each launch that uses them), so concurrent calls with distinct workspaces never share one
  p->ctr_off = off;
  if (p->kind == 2) off += kCtrBytes;
  p->ws_bytes = off;
}

int choose_tr(int64_t rows, int Lp) {
  int tr = 32;
  while (tr > 1 && rows % tr) tr >>= 1;
  return std::max(tr, 1 << Lp);
}

// First passes of heights that are not a multiple of 32 (1000, 1080, 720, ...) may keep 32-row
// tiles: the last row tile starts at H - 32 (clamp_rows; H - 32 is a multiple of 2^Lp for Lp <= 5,
// so the overlapped rows are recomputed from the same inputs and stored twice with identical bits;
// the extra traffic is (32 - H % 32) / H, allowed up to 10 %).  Measured (tools/generic_shapes.py,
// profiles/r01_generic_shapes.md): synthesis gains for every such height (1000 x 1000 3.6 -> 5.1
// TB/s, 2160 x 3840 5.9 -> 6.5); analysis gains where the height has a single factor 8 (8-row
// tiles: 1000, 1080, 600, 3000 rows) and loses where 16-row tiles were possible (720, 1200, 2160
// rows: 6.2 -> 5.4), so analysis clamps only from 8-row tiles (min_tr = 16).
int choose_tr_first(int64_t rows, int Lp, int min_tr) {
  const int tr = choose_tr(rows, Lp);
  const int64_t overlap = 32 - rows % 32;
  return (tr < min_tr && rows > 32 && overlap * 10 <= rows && Lp <= 5 && env_int("FHWT_CLAMP_ROWS", 1) != 0) ? 32
                                                                                                              : tr;
}

// Tile width of a first pass: 256 or 128 columns (full tiles when w % 128 == 0); narrower images
// use w itself (generic kernels).
int choose_tc(int64_t w, int pref) {
  if (pref < 256) return int(std::min<int64_t>(pref, w));
  if (pref == 512 && w % 512 == 0) return 512;   // synthesis sweep: 1-KB level-1 band rows (row boxes)
  if (w < 128) return env_int("FHWT_NARROW_FAST", 1) && w >= 16 && w % 16 == 0 ? 128 : int(w);   // one masked tile
  if (w % 256 == 0) return 256;
  // w % 256 == 128: 256-column tiles with the last one overlapping (clamp_last) when that repeats at
  // most 10 % of the columns; measured 1080 x 1920: synthesis 5.17 -> 6.23 TB/s (the 32 x 256
  // warp-decoupled kernel instead of 32 x 128 cp.async tiles), analysis 5.28 -> 5.43; 1280 neutral
  if (w % 128 == 0) return (128 * 10 <= w && env_int("FHWT_TC256_CLAMP", 1) != 0) ? 256 : 128;
  // ragged: 256-column tiles unless they would pad a row by more than 20 % (e.g. 800 -> 1024);
  // measured: 1600-wide rows 5.4 TB/s with 256-column tiles vs 4.6 with 128
  return ((w + 255) / 256 * 256 - w) * 5 > w ? 128 : 256;
}

// Analysis 8-row tiles (heights with a single factor 8, e.g. 1000 or 1080 rows) run faster 128
// columns wide: 1000 x 1024 images 4.7 -> 5.5 TB/s, 1000 x 1000 4.0 -> 4.5 (tools/iso_1000.py,
// tools/ab_shapes.py); synthesis is slower that way (3.65 -> 2.94) and keeps 256.

// Ring depth by stage size (tools/generic_shapes.py sweeps): analysis keeps >= 64 KB of input
// staged per CTA (2 .. 8 stages: 8 x 128 tiles 5.1 -> 6.1 TB/s at 8 stages); synthesis peaks near
// 48 KB (2 .. 4 stages; 8 stages of 8 x 128 tiles fall to 3.8 TB/s from 4.9 at 4).
int ring_stages(uint32_t stage_bytes) {
  return int(std::min<uint32_t>(8, std::max<uint32_t>(2, (65536 + stage_bytes - 1) / stage_bytes)));
}
// Analysis ring depth / CTAs-per-SM cap for the narrower first-pass tiles (tools/sweep128.sh,
// profiles/r01_generic_shapes.md; GB/s analysis, default occupancy -> table):
//   32 x 128: 2 CTAs/SM, 2 stages (3 when the last column tile overlaps): 480 x 640 5.5 -> 6.3 TB/s,
//             1152^2 5.5 -> 6.3, 1000 x 1152 (clamped rows) 5.3 -> 6.1, 600 x 800 (clamped
//             columns: 5.8 at 2 stages, 6.4 at 3) 4.6 -> 6.4
//   16 x 256: 3 CTAs/SM: 2160 x 3840 5.4 -> 6.3, 720 x 1280 5.3 -> 6.2 (at 2 stages; 4 stages as good)
//   16 x 128: 4 CTAs/SM, 4 stages: 400 x 544 4.8 -> 6.2
// 32 x 256 (c4) keeps the occupancy limit (2 CTAs/SM) and 2 stages; 8-row tiles keep the defaults.
void ana_tile_cfg(int tr, int tc, bool overlap, int* stages, int* cap_ctas) {
  if (tr == 32 && tc == 128) {
    *cap_ctas = 2;
    *stages = overlap ? 3 : 2;
  } else if (tr == 16 && tc == 256) {
    *cap_ctas = 3;
    *stages = 4;
  } else if (tr == 16 && tc == 128) {
    *cap_ctas = 4;
    *stages = 4;
  }
}

// Synthesis (cp.async variant) ring depth / CTAs-per-SM cap for the narrower tiles
// (tools/sweep_syn128.sh; GB/s synthesis, default -> table): 32 x 128 at 2 stages, 3 CTAs/SM:
// 480 x 640 5.3 -> 5.8, 600 x 800 5.0 -> 6.1, 1152^2 5.4 -> 5.8; 16 x 128 at 4 stages, 4 CTAs/SM:
// 400 x 544 5.2 -> 5.7.
void syn_tile_cfg(int mode, int tr, int tc, int* stages, int* cap_ctas) {
  if ((mode == 3 || mode == 6) && tr == 32 && tc == 128) {   // warp-decoupled kernel, 4 warps per CTA
    *stages = 2;
    *cap_ctas = 3;
  } else if (mode != 2) {
    return;
  } else if (tr == 32 && tc == 128) {
    *stages = 2;
    *cap_ctas = 3;
  } else if (tr == 16 && tc == 128) {
    *stages = 4;
    *cap_ctas = 4;
  }
}

int syn_ring_stages(uint32_t stage_bytes) {
  return int(std::min<uint32_t>(4, std::max<uint32_t>(2, (49152 + stage_bytes - 1) / stage_bytes)));
}

// Small problems (fewer tiles than SMs, e.g. one 512 x 512 image): shorter and narrower tiles so
// the work spreads over more SMs; each CTA's serial chain (load, levels, store) is what sets the
// latency there.  Only between compile-time fast geometries (rows 8/16/32, columns 128/256).
void shrink_for_small(int64_t batch, int64_t rows, int64_t cols, int Lp, int sms, int* TR, int* TC) {
  if (env_int("FHWT_SMALL_TILES", 1) == 0) return;
  auto tiles = [&] { return batch * (rows / *TR) * ((cols + *TC - 1) / *TC); };
  while (tiles() < sms && *TR > std::max(8, 1 << Lp) && rows % (*TR / 2) == 0) *TR /= 2;
  if (tiles() < sms && *TC == 256 && cols % 128 == 0) *TC = 128;
}

// ------------------------------------------------------------------ 2-D small images
// Batches of images too narrow for 128-column tiles (w < 128, h * w <= 4096, w % 4 == 0): chunks
// of whole images by 1-D bulk copies, all levels in shared memory (haar2d_small.cu).
bool small_ok(const fhwt_plan_s* pl, const void* a, const void* b) {
  return env_int("FHWT_SMALL_IMAGES", 1) != 0 && pl->w < 128 && pl->h * pl->w <= 4096 && pl->w % 4 == 0 &&
         aligned16(a) && aligned16(b);
}

fhwt_status run_small2d(const fhwt_plan_s* pl, const float* in, float* out, cudaStream_t s, bool analysis) {
  DevInfo di;
  FHWT_TRY(device_info(&di));
  Small2dParams p{};
  p.in = in;
  p.out = out;
  p.batch = pl->batch;
  p.H = int(pl->h);
  p.W = int(pl->w);
  p.L = pl->levels;
  const int img = p.H * p.W;
  p.G = std::max(1, std::min<int>(int(std::min<int64_t>(pl->batch, 1 << 20)),
                                  env_int("FHWT_SMALL_CHUNK", 8192) / img));   // ~32 KB chunks
  p.nchunks = (pl->batch + p.G - 1) / p.G;
  p.stages = env_int("FHWT_SMALL_STAGES", 2);
  p.stage_bytes = uint32_t(align_up(size_t(p.G) * img * 4, 1024));
  size_t off = size_t(p.stages) * p.stage_bytes;
  p.off_out = uint32_t(off);
  off = align_up(off + size_t(p.G) * img * 4, 128);
  for (int i = 0; i < 2; ++i) {
    p.off_t[i] = uint32_t(off);
    off = align_up(off + size_t(p.G) * (img / 4) * 4, 128);
  }
  for (int i = 0; i < 2; ++i) {
    p.off_d[i] = uint32_t(off);
    off = align_up(off + std::max<size_t>(8, size_t(p.G) * (img / 256) * 8), 128);
  }
  p.off_bar = uint32_t(off);
  const size_t smem = off + 8 * size_t(p.stages);
  int bps = 0;
  FHWT_CUDA(small2d_occupancy(analysis, smem, &bps), "small2d occupancy");
  if (bps < 1) return fail(FHWT_ERR_CUDA, "small-image kernel does not fit (%zu B shared memory)", smem);
  const int64_t grid = std::min<int64_t>(p.nchunks, int64_t(bps) * di.sms);
  FHWT_CUDA(launch_small2d(p, analysis, int(grid), smem, s), "small2d launch");
  return FHWT_OK;
}

// Batches of 1-D signals shorter than the 1024-sample warp chunk (n < 1024, n % 4 == 0): the same
// chunk machinery (haar2d_small.cu ana1d/syn1d_small_kernel).
bool small1d_ok(const fhwt_plan_s* pl, const void* a, const void* b) {
  const int64_t unit = int64_t(1) << std::min(3, pl->levels);   // values per thread in the first pass
  return env_int("FHWT_SMALL_SIGNALS", 1) != 0 && pl->n < kChunk1d && pl->n % 4 == 0 && pl->n % unit == 0 &&
         aligned16(a) && aligned16(b);
}

fhwt_status run_small1d(const fhwt_plan_s* pl, const float* in, float* out, cudaStream_t s, bool analysis) {
  DevInfo di;
  FHWT_TRY(device_info(&di));
  Small2dParams p{};
  p.in = in;
  p.out = out;
  p.batch = pl->batch;
  p.H = 1;
  p.W = int(pl->n);
  p.L = pl->levels;
  const int n = p.W;
  // Chunk size and ring depth per direction (tools/sweep_small1d.sh, GB/s for n = 256 / 512 / 128):
  // analysis 16 KB chunks x 3 stages (5544 / 5435 / 6332; 32 KB x 2: 5542 / 5505 / 5616), synthesis
  // 64 KB chunks x 2 stages (6649 / 6430 / 6517; 32 KB x 2: 5851 / 5629 / 6054).
  const int chunk = env_int("FHWT_SMALL1D_CHUNK", analysis ? 4096 : 16384);
  p.G = std::max(1, std::min<int>(int(std::min<int64_t>(pl->batch, 1 << 20)), chunk / n));
  p.nchunks = (pl->batch + p.G - 1) / p.G;
  p.stages = env_int("FHWT_SMALL_STAGES", analysis ? 3 : 2);
  p.stage_bytes = uint32_t(align_up(size_t(p.G) * n * 4, 1024));
  size_t off = size_t(p.stages) * p.stage_bytes;
  p.off_out = uint32_t(off);
  off = align_up(off + size_t(p.G) * n * 4, 128);
  // a_3 (fp32) and a_6 (analysis: fp64 in off_d[0]; synthesis: fp32 in off_t[1]) per signal
  const size_t tb[2] = {size_t(p.G) * (n / 8) * 4, size_t(p.G) * (n / 64) * 4};
  const size_t db[2] = {std::max<size_t>(8, size_t(p.G) * (n / 64) * 8), 8};
  for (int i = 0; i < 2; ++i) {
    p.off_t[i] = uint32_t(off);
    off = align_up(off + std::max<size_t>(16, tb[i]), 128);
  }
  for (int i = 0; i < 2; ++i) {
    p.off_d[i] = uint32_t(off);
    off = align_up(off + db[i], 128);
  }
  p.off_bar = uint32_t(off);
  const size_t smem = off + 8 * size_t(p.stages);
  int bps = 0;
  FHWT_CUDA(small2d_occupancy(analysis, smem, &bps, true), "small1d occupancy");
  if (bps < 1) return fail(FHWT_ERR_CUDA, "short-signal kernel does not fit (%zu B shared memory)", smem);
  if (const int cap = env_int("FHWT_SMALL_CTAS", 0)) bps = std::min(bps, cap);   // sweep knob
  const int64_t grid = std::min<int64_t>(p.nchunks, int64_t(bps) * di.sms);
  FHWT_CUDA(launch_small2d(p, analysis, int(grid), smem, s, true), "small1d launch");
  return FHWT_OK;
}

// ------------------------------------------------------------------ 2-D execution
// the workspace's tile-counter slot is usable (present and 16-B aligned: 32-bit atomics, memset)
bool ctr_ok(const char* ws, const fhwt_plan_s* pl) {
  return ws != nullptr && (reinterpret_cast<uintptr_t>(ws + pl->ctr_off) & 15) == 0;
}

fhwt_status run_ana2d(const fhwt_plan_s* pl, const float* d, float* coeffs, char* ws, cudaStream_t s) {
  const int64_t H = pl->h, W = pl->w, B = pl->batch;
  if (W % 4 != 0 || !aligned16(d) || !aligned16(coeffs)) {
    if (pl->levels != 1)
      return fail(FHWT_ERR_MISALIGNED, "multi-level 2-D transform needs 16-byte aligned buffers and w %% 4 == 0");
    FHWT_CUDA(launch_ana2d_l1_scalar(d, coeffs, H, W, B, s), "ana2d_l1_scalar launch");
    return FHWT_OK;
  }
  if (small_ok(pl, d, coeffs)) return run_small2d(pl, d, coeffs, s, true);
  DevInfo di;
  FHWT_TRY(device_info(&di));
  const size_t np = pl->passes.size();
  for (size_t k = 0; k < np; ++k) {
    const Pass ps = pl->passes[k];
    const bool in64 = k > 0;
    const bool final_pass = k + 1 == np;
    Ana2dParams p{};
    p.out = coeffs;
    p.H = H;
    p.W = W;
    p.Hin = H >> ps.g0;
    p.Win = W >> ps.g0;
    p.batch = B;
    p.Lp = ps.Lp;
    p.g0 = ps.g0;
    p.TR = in64 ? choose_tr(p.Hin, ps.Lp) : choose_tr_first(p.Hin, ps.Lp, 16);
    p.TC = in64 ? int(std::min<int64_t>(128, p.Win)) : choose_tc(p.Win, env_int("FHWT_ANA_TC", 256));
    if (!in64) shrink_for_small(B, p.Hin, p.Win, ps.Lp, di.sms, &p.TR, &p.TC);
    if (!in64 && p.TR == 8 && p.TC == 256 && env_int("FHWT_TR8_TC128", 1) != 0) p.TC = 128;   // see tr8_tc
    p.clamp_rows = p.Hin % p.TR != 0;
    p.tiles_r = (p.Hin + p.TR - 1) / p.TR;
    p.row_pad = int(p.tiles_r * p.TR - p.Hin);
    p.tiles_c = (p.Win + p.TC - 1) / p.TC;
    p.ntiles = B * p.tiles_r * p.tiles_c;
    p.final_pass = final_pass;
    p.ws_out = final_pass ? nullptr : reinterpret_cast<double*>(ws + pl->ws_off[k]);
    const void* in = k == 0 ? static_cast<const void*>(d) : static_cast<const void*>(ws + pl->ws_off[k - 1]);
    const int64_t in_pitch = k == 0 ? W : pitch4(p.Win);
    CUtensorMap map;
    // One-row boxes when a row is >= 1 KB (and a 128-B multiple): the kernel then issues TR of
    // them per tile from one thread.  B200 (tools/membench.py, tools/sweep_2d.py): 32 one-row
    // 1-KB boxes stream at 6.9 TB/s where one 32-row box stops at 6.1 TB/s; smaller row boxes
    // are request-bound and slower than multi-row boxes.
    // TMA loads without an L2 cache-policy operand (0) by default: in the bench's DWT+IDWT step the
    // hint-free instruction form streams c4 analysis at 6.35 TB/s against 6.20 with any policy
    // (evict_first / evict_normal / evict_last all 6.20; tools/bench_ab.sh, profiles/r02_l2_policy.md)
    p.l2hint = env_int("FHWT_ANA_L2HINT", 0);
    // Level-pair fusion (32 x 256 tiles), measured: LP = 5 levels 2+3 by 128 threads and 4+5 by 8 (+3 %);
    // LP = 3, 4 level by level.  Mode 6 (LP = 3: levels 2+3 by all 256 threads, two lanes per 4 x 4
    // LL1 block) won on two boxes (+1-3.5 %) and lost on two (-7 %, 2048^2 images): kept as an option.
    p.fused = env_int("FHWT_ANA_FUSED", ps.Lp == 5 ? 1 : 0);
    p.row_boxes = size_t(p.TC) * (in64 ? 8 : 4) >= 1024 && (size_t(p.TC) * (in64 ? 8 : 4)) % 128 == 0 &&
                  env_int("FHWT_ANA_ROWBOXES", 1) != 0;
    FHWT_TRY(encode_2d(&map, in, in64, p.Win, B * p.Hin, in_pitch, p.TC, p.row_boxes ? 1 : p.TR));
    // shared memory layout: stages | P[0] | P[1] | barriers
    const size_t es = in64 ? 8 : 4;
    p.stage_bytes = uint32_t(align_up(size_t(p.TR) * p.TC * es, 1024));
    // Ring depth: at least 64 KB of staged input per CTA (2 stages of 32 x 256 fp32 tiles; up to 8
    // stages of smaller tiles, e.g. 8 x 128 for 1080-row frames, where 2 stages kept too few bytes
    // in flight).
    // Narrower fast tiles: ring depth and resident CTAs per SM from a measured table (tile_cfg);
    // too many small CTAs per SM (occupancy allows 4-10) streamed 10-25 % slower.
    int cap_ctas = 0, stages = ring_stages(p.stage_bytes);
    if (!in64 && ps.g0 == 0 && env_int("FHWT_ANA_TILE_TABLE", 1) != 0)
      ana_tile_cfg(p.TR, p.TC, p.Win % p.TC != 0, &stages, &cap_ctas);
    p.stages = in64 ? 2 : env_int("FHWT_ANA_STAGES", stages);
    size_t pb[2] = {0, 0};
    for (int j = 1; j < ps.Lp; ++j) {
      const size_t sz = (in64 || ps.g0 + j >= kFirstF64Level) ? 8 : 4;
      pb[j & 1] = std::max(pb[j & 1], size_t(p.TR >> j) * size_t(p.TC >> j) * sz);
    }
    // FHWT_ANA_FUSED=12 double-buffers LL1 (haar2d.cu ana_fused12_tile)
    if (!in64 && p.fused == 12) pb[1] = std::max(pb[1], 2 * size_t(16 * 128) * 4);
    // compile-time 32 x 256 variant: first pass, full tiles (then every band offset is 8-B aligned)
    const bool fast_ok = !in64 && ps.g0 == 0 && (p.TR == 32 || p.TR == 16 || p.TR == 8) &&
                         (p.TC == 256 || p.TC == 128) && (p.Win % p.TC == 0 || env_int("FHWT_ANA_RAGGED_FAST", 1) != 0);
    // ragged widths: compile-time tile geometry with masked edge tiles (TMA zero-fills past the
    // edge); band rows are 8-B aligned when every band offset W >> j (j <= Lp) is even
    // ragged width: clamp the last tile to Win - TC (full, overlapping) when Win > TC, else masked
    p.clamp_last = p.Win % p.TC != 0 && p.Win > p.TC && env_int("FHWT_CLAMP_LAST", 1) != 0;
    p.mask_mode = (p.Win % p.TC != 0 && !p.clamp_last) ? 1 : 0;
    p.aligned_levels = 0;   // band offsets W >> j and tile starts col0 >> j even for j <= aligned_levels
    while (p.aligned_levels < ps.Lp && (W >> (p.aligned_levels + 1)) % 2 == 0 &&
           (!p.clamp_last || ((p.Win - p.TC) >> (p.aligned_levels + 1)) % 2 == 0))
      ++p.aligned_levels;
    size_t off = size_t(p.stages) * p.stage_bytes;
    p.p_off[0] = uint32_t(off);
    off = align_up(off + pb[0], 128);
    p.p_off[1] = uint32_t(off);
    off = align_up(off + pb[1], 128);
    p.bar_off = uint32_t(off);
    const size_t smem = off + 12 * size_t(p.stages);   // mbarriers + stage-release counters
    // FHWT_ANA_FUSED=3: the fused2 path with a dedicated 9th tail warp (ana2d_fused3_kernel)
    const bool fused3 = fast_ok && p.fused == 3 && ps.Lp == 5 && p.TR == 32 && p.TC == 256 && p.mask_mode == 0 &&
                        p.aligned_levels >= ps.Lp && !p.clamp_last && !p.clamp_rows;
    // FHWT_ANA_FUSED=8: warp-specialised kernel (haar2d_ana.cu): 8 compute warps, each all five
    // levels of its own 32 x 32 block, plus a TMA producer warp; no CTA barrier per tile
    const bool ws8 = fast_ok && (p.fused == 8 || p.fused == 11) && ps.Lp == 5 && p.TR == 32 &&
                     p.TC == 256 &&
                     p.mask_mode == 0 && p.aligned_levels >= ps.Lp && !p.clamp_last && !p.clamp_rows;
    // FHWT_ANA_FUSED=11: the default chain with register (LDG) loads, no input staging
    if (ws8 && p.fused == 11) {
      p.in = d;
      p.p_off[0] = 0;                                      // LL3, 4 x 32 fp32
      p.p_off[1] = 512u;                                   // LL1, 16 x 128 fp32
      const size_t lsmem = 512u + 8192u;
      int lbps = 0;
      const int lvar = env_int("FHWT_ANA_LDG", 0);
      FHWT_CUDA(ana2d_ldg_occupancy(lsmem, &lbps, lvar), "ldg occupancy");
      if (const int cap = env_int("FHWT_ANA_CTAS_PER_SM", 0)) lbps = std::min(lbps, cap);
      const int64_t lgrid = std::min<int64_t>(p.ntiles, int64_t(std::max(lbps, 1)) * di.sms);
      const bool lcoop = k == 0 && np == 2 && pl->passes[1].Lp <= 3 && env_int("FHWT_COOP", 1) != 0;
      p.tail = lcoop ? pl->passes[1].Lp : 0;
      if (env_int("FHWT_DEBUG_LAUNCH", 0))
        std::fprintf(stderr, "[fhwt] ana2d ldg11 smem %zu B ctas/SM %d grid %lld tail %d\n", lsmem, lbps,
                     (long long)lgrid, p.tail);
      FHWT_CUDA(launch_ana2d_ldg(p, int(lgrid), lsmem, s, lvar), "ana2d ldg launch");
      if (lcoop) break;
      continue;
    }
    if (ws8) {
      p.stages = env_int("FHWT_ANA_STAGES", 2);
      uint32_t ll1_off = 0, bar_off = 0;
      const size_t wsmem = ana2d_ws_smem(p.stages, &ll1_off, &bar_off);
      p.p_off[0] = ll1_off;
      p.bar_off = bar_off;
      int wbps = 0;
      FHWT_CUDA(ana2d_ws_occupancy(wsmem, &wbps), "ws occupancy");
      if (wbps < 1) return fail(FHWT_ERR_CUDA, "warp-specialised analysis does not fit (%zu B)", wsmem);
      if (const int cap = env_int("FHWT_ANA_CTAS_PER_SM", 0)) wbps = std::min(wbps, cap);
      const int64_t wgrid = std::min<int64_t>(p.ntiles, int64_t(wbps) * di.sms);
      const bool wcoop = k == 0 && np == 2 && pl->passes[1].Lp <= 3 && env_int("FHWT_COOP", 1) != 0;
      p.tail = wcoop ? pl->passes[1].Lp : 0;
      if (env_int("FHWT_DEBUG_LAUNCH", 0))
        std::fprintf(stderr, "[fhwt] ana2d ws8 stages %d smem %zu B ctas/SM %d grid %lld tail %d\n", p.stages, wsmem,
                     wbps, (long long)wgrid, p.tail);
      FHWT_CUDA(launch_ana2d_ws(p, map, int(wgrid), wsmem, s), "ana2d ws launch");
      if (wcoop) break;
      continue;
    }
    // the lean K1 (haar2d.cu ana2d_lean_kernel): full, unclamped, aligned 32 x 256 tiles at LP = 5 —
    // every c4 / c5 tile — with the default fused chain
    const bool lean = fast_ok && p.fused == 1 && ps.Lp == 5 && p.TR == 32 && p.TC == 256 && p.mask_mode == 0 &&
                      p.aligned_levels >= ps.Lp && !p.clamp_last && !p.clamp_rows &&
                      env_int("FHWT_ANA_LEAN", 1) != 0;
    // dynamic tile order (tiles handed out in global order by an atomic counter in the workspace):
    // c4 analysis 6.35 -> 6.90 TB/s, c5 6.28 -> 6.72 (profiles/r02_dynamic_tiles.md).  A workspace
    // whose counter slot is not 16-B aligned (a caller's offset pointer) keeps the static order.
    const bool dyn = lean && ctr_ok(ws, pl) && env_int("FHWT_ANA_DYN", 1) != 0;
    if (dyn) {
      const int g = env_int("FHWT_ANA_DYN_GROUPS", 1);
      p.dyn_groups = (g > 1 && p.ntiles % g == 0) ? g : 1;
      p.tile_ctr = reinterpret_cast<unsigned*>(ws + pl->ctr_off);
      FHWT_CUDA(cudaMemsetAsync(p.tile_ctr, 0, 16, s), "tile counter reset");
    }
    const int vmode = fused3 ? 5 : dyn ? 8 : lean ? 7 : 0;
    const int fast = fast_ok ? (vmode << 24) | (p.TR << 16) | (p.TC << 4) | ps.Lp : 0;
    int bps = 0;
    FHWT_TRY(occupancy(in64 ? 1 : 0, fast, smem, &bps));
    if (const int cap = env_int("FHWT_ANA_CTAS_PER_SM", env_int("FHWT_CTAS_PER_SM", cap_ctas))) bps = std::min(bps, cap);
    const int64_t grid = std::min<int64_t>(p.ntiles, int64_t(bps) * di.sms);
    // 5 < L <= 8 on the 32-row fast path: the coarse levels run after a grid barrier in the same,
    // cooperative, launch (haar2d.cu ana_coarse) instead of a second small-grid pass.
    const bool coop = k == 0 && np == 2 && pl->passes[1].Lp <= 3 && ps.Lp == 5 && fast_ok &&
                      env_int("FHWT_COOP", 1) != 0;
    p.tail = coop ? pl->passes[1].Lp : 0;
    if (env_int("FHWT_DEBUG_LAUNCH", 0))
      std::fprintf(stderr, "[fhwt] ana2d fused %d%s tile %dx%d LP %d stages %d smem %zu B ctas/SM %d grid %lld\n",
                   p.fused, lean ? " lean" : "", p.TR, p.TC, ps.Lp, p.stages, smem, bps, (long long)grid);
    FHWT_CUDA(launch_ana2d(p, map, in64, fast, int(grid), smem, s), "ana2d launch");
    if (coop) break;
  }
  return FHWT_OK;
}

fhwt_status run_syn2d(const fhwt_plan_s* pl, const float* coeffs, float* dR, char* ws, cudaStream_t s) {
  const int64_t H = pl->h, W = pl->w, B = pl->batch;
  if (W % 4 != 0 || !aligned16(coeffs) || !aligned16(dR)) {
    if (pl->levels != 1)
      return fail(FHWT_ERR_MISALIGNED, "multi-level 2-D transform needs 16-byte aligned buffers and w %% 4 == 0");
    FHWT_CUDA(launch_syn2d_l1_scalar(coeffs, dR, H, W, B, s), "syn2d_l1_scalar launch");
    return FHWT_OK;
  }
  if (small_ok(pl, coeffs, dR)) return run_small2d(pl, coeffs, dR, s, false);
  DevInfo di;
  FHWT_TRY(device_info(&di));
  const size_t np = pl->passes.size();
  // 5 < L <= 8 with 32 x 256 fine tiles: one cooperative launch of syn2d_warp_kernel<5> whose head
  // phase rebuilds LL5 from the coarse levels (haar2d.cu syn_coarse) before a grid barrier.
  bool coop = false;
  if (np == 2 && pl->passes[1].Lp <= 3 && pl->passes[0].Lp == 5 && env_int("FHWT_COOP", 1) != 0 &&
      env_int("FHWT_SYN_MODE", 3) == 3) {
    int tr = choose_tr(H, 5), tc = int(std::min<int64_t>(env_int("FHWT_SYN_TC", 256), W));
    if (tc == 256 && W % 256 && W % 128 == 0) tc = 128;
    shrink_for_small(B, H, W, 5, di.sms, &tr, &tc);
    coop = tr == 32 && ((tc == 256 && W % 256 == 0) || (tc == 512 && W % 512 == 0));
  }
  for (size_t kk = np; kk-- > 0;) {
    if (coop && kk == 1) continue;
    const Pass ps = pl->passes[kk];
    Syn2dParams p{};
    // warp-kernel TMA loads: 3 = no policy operand (default; c4 synthesis 6.34 TB/s against 6.28 with
    // evict_first, 6.30 evict_normal, 6.31 evict_last: profiles/r02_l2_policy.md)
    p.l2mode = env_int("FHWT_SYN_L2MODE", 3);
    p.H = H;
    p.W = W;
    p.Hin = H >> ps.g0;
    p.Win = W >> ps.g0;
    p.batch = B;
    p.Lp = ps.Lp;
    p.g0 = ps.g0;
    p.TR = ps.g0 == 0 ? choose_tr_first(p.Hin, ps.Lp, 32) : choose_tr(p.Hin, ps.Lp);
    p.TC = choose_tc(p.Win, env_int("FHWT_SYN_TC", 256));
    if (ps.g0 == 0) shrink_for_small(B, p.Hin, p.Win, ps.Lp, di.sms, &p.TR, &p.TC);
    p.clamp_rows = p.Hin % p.TR != 0;
    p.tiles_r = (p.Hin + p.TR - 1) / p.TR;
    p.tiles_c = (p.Win + p.TC - 1) / p.TC;
    p.ntiles = B * p.tiles_r * p.tiles_c;
    if (kk == 0) {
      p.out = dR;
      p.out_pitch = W;
    } else {
      p.out = reinterpret_cast<float*>(ws + pl->ws_off[kk - 1]);
      p.out_pitch = pitch4(p.Win);
    }
    p.coeffs = coeffs;
    TmaMaps2d maps;
    std::memset(&maps, 0, sizeof maps);
    int bw[6] = {0, 0, 0, 0, 0, 0};
    // Shifted warp-decoupled variant (mode 6, haar2d.cu syn_issue_tile_lane<true>): 32 x 256 tiles
    // whose band blocks do not all start 16-B aligned (W >> j odd or 2 mod 4, or the clamped last
    // tile's Win - 256 >> j): every box starts at the aligned column below and is 4 columns wider.
    bool shifted = false;
    // 32 x 128 tiles on the warp kernel too, for LP <= 3 and widths without an overlapping last tile
    // (tools/sweep_syn_warp128.sh, 2 stages x 3 CTAs/SM vs cp.async: 480 x 640 L=3 5866 -> 6314,
    // 1152^2 5844 -> 6305, 768 x 896 5886 -> 6305, 1000 x 1152 5938 -> 6167; but 600 x 800
    // (clamped) 6097 -> 5588, 480 x 640 L=4 6363 -> 5478, L=5 6074 -> 4878)
    const bool warp128 = env_int("FHWT_SYN_WARP128", ps.Lp <= 3 && p.Win % 128 == 0 ? 1 : 0) != 0;
    if (ps.g0 == 0 && !coop && p.TR == 32 && (p.TC == 256 || (p.TC == 128 && warp128)) && p.Win > p.TC &&
        W % 4 == 0 &&
        env_int("FHWT_SYN_SHIFT", 1) != 0 && env_int("FHWT_SYN_MODE", 3) == 3) {
      bool al = (W >> 1) % 2 == 0;
      for (int j = 1; j <= ps.Lp; ++j)
        al = al && (W >> j) % 4 == 0 && (p.Win % p.TC == 0 || ((p.Win - p.TC) >> j) % 4 == 0);
      shifted = !al;
    }
    for (int j = 1; j <= ps.Lp; ++j) {
      // TMA box starts must be 16-byte aligned: LH boxes start at col0 >> j (a multiple of 4),
      // HL/HH boxes at (W >> g) + (col0 >> j), so they start hoff = (W >> g) & 3 columns early.
      p.hoff[j] = shifted ? 0 : int((W >> (ps.g0 + j)) & 3);
      bw[j] = shifted ? (p.TC >> j) + 4 : int(pitch4((p.TC >> j) + p.hoff[j]));
      p.box_pitch[j] = bw[j];
      p.row_boxes[j] = bw[j] * 4 >= env_int("FHWT_SYN_ROWBOX_MIN", 1024) && (bw[j] * 4) % 128 == 0;   // see the analysis note
      FHWT_TRY(encode_2d(&maps.level[j], coeffs, false, W, B * H, W, bw[j], p.row_boxes[j] ? 1 : p.TR >> j));
    }
    if (kk + 1 == np) {
      p.ll_from_ws = 0;
      maps.ll = maps.level[ps.Lp];
    } else {
      p.ll_from_ws = 1;
      p.ll_ws = reinterpret_cast<const float*>(ws + pl->ws_off[kk]);
      const int64_t wl = p.Win >> ps.Lp, hl = p.Hin >> ps.Lp;
      FHWT_TRY(encode_2d(&maps.ll, ws + pl->ws_off[kk], false, wl, B * hl, pitch4(wl), bw[ps.Lp],
                         p.row_boxes[ps.Lp] ? 1 : p.TR >> ps.Lp));
    }
    // compile-time tile geometry (fast variants); full = no ragged edge and every box 16-B aligned
    const bool geom = (p.TR == 32 || p.TR == 16 || p.TR == 8) &&
                      (p.TC == 256 || p.TC == 128 || (p.TC == 512 && p.TR == 32)) && p.out_pitch % 4 == 0;
    bool aligned = geom && (W >> (ps.g0 + 1)) % 2 == 0;
    for (int j = 1; j <= ps.Lp; ++j) aligned = aligned && p.hoff[j] == 0 && bw[j] == (p.TC >> j);
    // A ragged width with aligned boxes runs as two launches: the full tiles on the fast path
    // (cp.async / warp-decoupled) and the last column of tiles on the masked TMA variant.
    const bool ragged = p.Win % p.TC != 0;
    // clamp_last: the last tile starts at Win - TC, full and on the fast path (needs those tile
    // starts 16-B aligned at every level too, or the shifted variant); otherwise the split below
    p.clamp_last = aligned && ragged && p.Win > p.TC && env_int("FHWT_CLAMP_LAST", 1) != 0;
    for (int j = 1; j <= ps.Lp && p.clamp_last; ++j) p.clamp_last = ((p.Win - p.TC) >> j) % 4 == 0;
    if (shifted) {
      aligned = true;   // every tile full, boxes widened and shifted
      p.clamp_last = ragged;
    }
    const bool split = aligned && ragged && !p.clamp_last && !coop && p.Win >= p.TC &&
                       env_int("FHWT_SYN_SPLIT", 1) != 0;
    struct Part {
      int64_t ct0, tiles_c;
      bool full;
    };
    Part parts[2] = {{0, p.tiles_c, aligned && (!ragged || p.clamp_last)}, {0, 0, false}};
    int nparts = 1;
    if (split) {
      parts[0] = {0, p.Win / p.TC, true};
      parts[1] = {p.Win / p.TC, 1, false};
      nparts = 2;
    }
    // FHWT_SYN_MODE=7 (haar2d_syn.cu): level-1 bands copied by each warp into its private slice,
    // coarse boxes by TMA; 32 x 256 full tiles of a 5-level first pass (c4, c5)
    if (env_int("FHWT_SYN_MODE", 3) == 7 && kk == 0 && ps.Lp == 5 && p.TR == 32 && p.TC == 256 && aligned &&
        !ragged && !shifted && !p.clamp_rows && p.out_pitch == W) {
      p.ct0 = 0;
      p.stages = env_int("FHWT_SYN_STAGES", 2);
      const size_t wsm = syn2d_wp_layout(&p);
      int wbps = 0;
      FHWT_CUDA(syn2d_wp_occupancy(wsm, &wbps), "syn wp occupancy");
      if (wbps < 1) return fail(FHWT_ERR_CUDA, "warp-private synthesis does not fit (%zu B)", wsm);
      if (const int cap = env_int("FHWT_CTAS_PER_SM", 0)) wbps = std::min(wbps, cap);
      const int64_t wgrid = std::min<int64_t>(p.ntiles, int64_t(wbps) * di.sms);
      if (coop) {
        p.head = pl->passes[1].Lp;
        p.ll_ws_out = reinterpret_cast<float*>(ws + pl->ws_off[0]);
      }
      if (env_int("FHWT_DEBUG_LAUNCH", 0))
        std::fprintf(stderr, "[fhwt] syn2d wp7 stages %d smem %zu B ctas/SM %d grid %lld head %d\n", p.stages, wsm,
                     wbps, (long long)wgrid, p.head);
      FHWT_CUDA(launch_syn2d_wp(p, maps, int(wgrid), wsm, s), "syn2d wp launch");
      continue;
    }
    for (int part = 0; part < nparts; ++part) {
      const bool full = parts[part].full;
      p.ct0 = parts[part].ct0;
      p.tiles_c = parts[part].tiles_c;
      p.ntiles = B * p.tiles_r * p.tiles_c;
      const bool fast = full || (geom && env_int("FHWT_SYN_RAGGED_FAST", 1) != 0);
      p.mask_mode = full ? 0 : 1;   // ragged or shifted boxes: masked variant, TMA boxes (mode 0)
      // load path of the fast variant: 0 TMA boxes, 2 cp.async (LDGSTS) for all boxes.  Measured on
      // B200 (tools/sweep_syn.py): cp.async 6.10 TB/s, TMA boxes 5.86 (register LDG of level 1: 5.19).
      int mode = full ? env_int("FHWT_SYN_MODE", 3) : 0;
      if (mode != 0 && mode != 3) mode = 2;
      // warp-decoupled variant: 32 x 256 and 32 x 128 tiles (one warp per 32 columns)
      if (mode == 3 && !(p.TR == 32 && (p.TC == 256 || p.TC == 512 || (p.TC == 128 && warp128)))) mode = 2;
      if (shifted) mode = 6;
      // dynamic tile order for the 32 x 256, LP = 5 warp kernel (c4 / c5 tiles), as in the analysis
      const bool sdyn = mode == 3 && p.TR == 32 && p.TC == 256 && ps.Lp == 5 && full && ps.g0 == 0 &&
                        ctr_ok(ws, pl) && env_int("FHWT_SYN_DYN", 0) != 0;
      // producer-warp K4 (haar2d.cu syn2d_prod_kernel; FHWT_SYN_PROD=1 static order, =2 global order,
      // the default for full 32 x 256 LP = 5 tiles, with a 3-stage ring): c4 synthesis 6.35 -> 6.41 TB/s,
      // c5 6.28 -> 6.44 (profiles/r02_dynamic_tiles.md)
      int sprod = (mode == 3 && p.TR == 32 && (p.TC == 256 || p.TC == 512) && ps.Lp == 5 && full && ps.g0 == 0 &&
                   !p.clamp_rows)
                      ? env_int("FHWT_SYN_PROD", 2) : 0;
      if (sprod == 2 && !ctr_ok(ws, pl)) sprod = 1;   // no usable counter slot: static order
      p.swz = 0;
      if (sprod > 0) {
        mode = (sprod == 2 ? 11 : 10) + ((p.ct0 != 0 || p.clamp_last) ? 2 : 0);
        // level-1/2 boxes through 128-B-swizzled 3-D maps {32 floats, lines, rows} (c4 synthesis
        // 6.45 -> 6.93 TB/s: the 128-B innermost box dimension, 7.4 %; the swizzle, which removes the
        // band reads' bank conflicts, 0.15 %; profiles/r02_swizzle.md): global order, 256-column
        // unclamped tiles, every level-1/2 band block a whole number of 128-B lines (W % 128 == 0), one
        // (TR >> j)-row box per band.  (Level 3 swizzled too measured 0.5 % slower.)
        if (mode == 11 && p.TC == 256 && W % 128 == 0 && !p.row_boxes[1] && !p.row_boxes[2] && bw[1] == 128 &&
            bw[2] == 64 && env_int("FHWT_SYN_SWZ", 1) != 0) {
          p.swz = 2;
          mode = 14;
          for (int j = 1; j <= p.swz; ++j)
            FHWT_TRY(encode_3d_swz(&maps.sw[j], coeffs, W, B * H, bw[j] / 32, p.TR >> j));
        }
        p.issue_rev = env_int("FHWT_SYN_ISSUE_REV", 0);
        const int g = env_int("FHWT_SYN_DYN_GROUPS", 1);
        p.dyn_groups = (g > 1 && p.ntiles % g == 0) ? g : 1;
        p.tile_ctr = reinterpret_cast<unsigned*>(ws + pl->ctr_off + 128);
      } else if (sdyn) {
        mode = 9;
        const int g = env_int("FHWT_SYN_DYN_GROUPS", 1);
        p.dyn_groups = (g > 1 && p.ntiles % g == 0) ? g : 1;
        p.tile_ctr = reinterpret_cast<unsigned*>(ws + pl->ctr_off + 128);
      }
      // stage layout: LL box, then per level j three boxes (128-B aligned: TMA destinations need it;
      // with cp.async a 16-B packing would admit a 3rd CTA/SM, which measured slower: 5.54 vs 6.10 TB/s)
      const size_t balign = 128;
      size_t off = 0, tx = 0;
      if (p.swz) {   // the swizzled boxes first, each 1024-B aligned (the 128-B swizzle atom is 8 lines)
        for (int j = 1; j <= p.swz; ++j) {
          const size_t bytes = size_t(p.TR >> j) * bw[j] * 4;
          for (int q = 0; q < 3; ++q) {
            p.box_off[j][q] = uint32_t(off);
            off = align_up(off + bytes, 1024);
            tx += bytes;
          }
        }
      }
      {
        const size_t bytes = size_t(p.TR >> ps.Lp) * bw[ps.Lp] * 4;
        p.box_off[0][0] = uint32_t(off);
        off = align_up(off + bytes, balign);
        tx += bytes;
      }
      for (int j = p.swz + 1; j <= ps.Lp; ++j) {
        const size_t bytes = size_t(p.TR >> j) * bw[j] * 4;
        for (int q = 0; q < 3; ++q) {
          p.box_off[j][q] = uint32_t(off);
          off = align_up(off + bytes, balign);
          tx += bytes;
        }
      }
      p.tx_bytes = uint32_t(tx);
      p.stage_bytes = uint32_t(align_up(off, 1024));
      // 2 stages for 32 x 256 tiles; the cp.async variant's narrower tiles from a measured table
      int syn_stages = syn_ring_stages(p.stage_bytes), syn_cap = 0;
      if (env_int("FHWT_SYN_TILE_TABLE", 1) != 0) syn_tile_cfg(mode, p.TR, p.TC, &syn_stages, &syn_cap);
      p.stages = env_int("FHWT_SYN_STAGES", (mode == 11 || mode == 13 || mode == 14) ? 3 : syn_stages);
      size_t pb[2] = {0, 0};
      for (int j = 2; j <= ps.Lp; ++j) {
        const int jj = j - 1;
        pb[jj & 1] = std::max(pb[jj & 1], size_t(p.TR >> jj) * size_t(p.TC >> jj) * 4);
      }
      off = size_t(p.stages) * p.stage_bytes;
      p.p_off[0] = uint32_t(off);
      if (mode == 3 || mode == 6 || mode >= 9) {
        off = align_up(off + size_t(p.TC / 32) * kSynScratchBytes, 128);
        p.p_off[1] = p.p_off[0];
      } else {
        off = align_up(off + pb[0], 128);
        p.p_off[1] = uint32_t(off);
        off = align_up(off + pb[1], 128);
      }
      p.bar_off = uint32_t(off);
      const size_t smem = off + 20 * size_t(p.stages);   // mbarriers + stage-release counters + stage tiles
      const int fast_lp = fast ? (mode << 24) | (p.TR << 16) | (p.TC << 4) | ps.Lp : 0;
      int bps = 0;
      FHWT_TRY(occupancy(2, fast_lp, smem, &bps));
      // At most 2 resident CTAs/SM: the lighter LP < 5 variants fit 3-4, which measured 2.5-6.5 %
      // slower (tools/sweep_ctas.py, profiles/r01_sweep_ctas.jsonl); LP = 5 is indifferent.
      const int cap = env_int("FHWT_CTAS_PER_SM", syn_cap);   // sweep knob; 0 = the measured default
      bps = std::min(bps, cap > 0 ? cap : (mode >= 10 ? 512 / p.TC : 2 * kThreads2d / syn2d_threads(fast_lp)));
      const int64_t grid = std::min<int64_t>(p.ntiles, int64_t(bps) * di.sms);
      if (coop) {
        if (mode != 3 && mode < 9)
          return fail(FHWT_ERR_CUDA, "internal: cooperative synthesis needs the warp-decoupled kernel");
        p.head = pl->passes[1].Lp;
        p.ll_ws_out = reinterpret_cast<float*>(ws + pl->ws_off[0]);
      }
      if (env_int("FHWT_DEBUG_LAUNCH", 0))
        std::fprintf(stderr, "[fhwt] syn2d mode %d tile %dx%d LP %d stages %d smem %zu B ctas/SM %d grid %lld\n", mode,
                     p.TR, p.TC, ps.Lp, p.stages, smem, bps, (long long)grid);
      if (mode == 9 || mode == 11 || mode == 13 || mode == 14) FHWT_CUDA(cudaMemsetAsync(p.tile_ctr, 0, 16, s), "tile counter reset");
      FHWT_CUDA(launch_syn2d(p, maps, fast_lp, int(grid), smem, s), "syn2d launch");
    }
  }
  return FHWT_OK;
}

// ------------------------------------------------------------------ 1-D execution
// Levels > 10 of signals of 1024, 2048, 4096 or 8192 samples (a full decomposition: J up to 13):
// the 8 warps of a CTA hold whole signals, so levels 11..J run inside the first-pass CTA from
// the chunks' LL10 in shared memory (haar1d.cu ana1d_tail / syn1d_tail) instead of a second pass
// whose grid has one warp per 1-8 values.  Measured 65536 x 4096, J = 12: analysis 0.371 ->
// 0.314 ms, synthesis 0.353 -> 0.311.  Returns the number of such levels, or 0.
int tail1d(const fhwt_plan_s* pl) {
  if (pl->passes.size() != 2 || pl->passes[0].Lp != 10 || env_int("FHWT_1D_TAIL", 1) == 0) return 0;
  const int64_t chunks = pl->n / kChunk1d;
  if (pl->n % kChunk1d != 0 || (chunks != 1 && chunks != 2 && chunks != 4 && chunks != 8)) return 0;
  if ((pl->batch * chunks) % 8 != 0) return 0;   // whole CTAs (8 warps) only
  return pl->passes[1].Lp;
}

fhwt_status run_ana1d(const fhwt_plan_s* pl, const float* d, float* coeffs, char* ws, cudaStream_t s) {
  const int64_t n = pl->n, B = pl->batch;
  if (n % 4 != 0 || !aligned16(d) || !aligned16(coeffs)) {
    if (pl->levels != 1)
      return fail(FHWT_ERR_MISALIGNED, "multi-level 1-D transform needs 16-byte aligned buffers and n %% 4 == 0");
    FHWT_CUDA(launch_ana1d_l1_scalar(d, coeffs, n, B, s), "ana1d_l1_scalar launch");
    return FHWT_OK;
  }
  if (small1d_ok(pl, d, coeffs)) return run_small1d(pl, d, coeffs, s, true);
  const size_t np = pl->passes.size();
  const int tail = tail1d(pl);
  for (size_t k = 0; k < np; ++k) {
    const Pass ps = pl->passes[k];
    Haar1dParams p{};
    if (tail) {   // levels 11.. inside the first pass (haar1d.cu ana1d_tail)
      p.tail = tail;
      p.final_pass = 1;
    }
    p.n = n;
    p.nin = n >> ps.g0;
    p.batch = B;
    p.Lp = ps.Lp;
    p.g0 = ps.g0;
    p.chunks = (p.nin + kChunk1d - 1) / kChunk1d;
    p.nwarps = B * p.chunks;
    p.coeffs_out = coeffs;
    p.final_pass = tail || k + 1 == np;
    p.in = k == 0 ? static_cast<const void*>(d) : static_cast<const void*>(ws + pl->ws_off[k - 1]);
    p.in_pitch = k == 0 ? n : pitch4(p.nin);
    p.out = p.final_pass ? nullptr : static_cast<void*>(ws + pl->ws_off[k]);
    p.out_pitch = p.final_pass ? 0 : pitch4(p.nin >> ps.Lp);
    FHWT_CUDA(launch_ana1d(p, k > 0, s, pl->levels > kMaxLevels1dPass), "ana1d launch");
    if (tail) break;
  }
  return FHWT_OK;
}

fhwt_status run_syn1d(const fhwt_plan_s* pl, const float* coeffs, float* dR, char* ws, cudaStream_t s) {
  const int64_t n = pl->n, B = pl->batch;
  if (n % 4 != 0 || !aligned16(coeffs) || !aligned16(dR)) {
    if (pl->levels != 1)
      return fail(FHWT_ERR_MISALIGNED, "multi-level 1-D transform needs 16-byte aligned buffers and n %% 4 == 0");
    FHWT_CUDA(launch_syn1d_l1_scalar(coeffs, dR, n, B, s), "syn1d_l1_scalar launch");
    return FHWT_OK;
  }
  if (small1d_ok(pl, coeffs, dR)) return run_small1d(pl, coeffs, dR, s, false);
  const size_t np = pl->passes.size();
  const int tail = tail1d(pl);
  for (size_t kk = np; kk-- > 0;) {
    if (tail && kk > 0) continue;   // the coarse levels run inside the fine pass (syn1d_tail)
    const Pass ps = pl->passes[kk];
    Haar1dParams p{};
    p.tail = tail;
    p.n = n;
    p.nin = n >> ps.g0;
    p.batch = B;
    p.Lp = ps.Lp;
    p.g0 = ps.g0;
    p.chunks = (p.nin + kChunk1d - 1) / kChunk1d;
    p.nwarps = B * p.chunks;
    p.coeffs_in = coeffs;
    p.final_pass = kk == 0;
    if (kk + 1 == np) {
      p.in = coeffs;
      p.in_pitch = n;
    } else {
      p.in = ws + pl->ws_off[kk];
      p.in_pitch = pitch4(p.nin >> ps.Lp);
    }
    if (kk == 0) {
      p.out = dR;
      p.out_pitch = n;
    } else {
      p.out = ws + pl->ws_off[kk - 1];
      p.out_pitch = pitch4(p.nin);
    }
    FHWT_CUDA(launch_syn1d(p, s), "syn1d launch");
  }
  return FHWT_OK;
}

size_t data_bytes(const fhwt_plan_s* p) {
  return size_t(p->batch) * (p->kind == 2 ? size_t(p->h) * size_t(p->w) : size_t(p->n)) * sizeof(float);
}

fhwt_status run_on_device(fhwt_plan p, const float* in, float* out, void* workspace, fhwt_stream_t st,
                          bool analysis);

// A plan bound to a device (fhwt_plan_1d/2d `device` >= 0) makes that device current for the
// call and restores the caller's afterwards; -1 runs on whatever device is current.
fhwt_status run(fhwt_plan p, const float* in, float* out, void* workspace, fhwt_stream_t st, bool analysis) {
  if (!p) return fail(FHWT_ERR_INVALID_ARG, "null plan");
  if (p->device < 0) return run_on_device(p, in, out, workspace, st, analysis);
  int cur = 0;
  FHWT_CUDA(cudaGetDevice(&cur), "cudaGetDevice");
  if (cur == p->device) return run_on_device(p, in, out, workspace, st, analysis);
  FHWT_CUDA(cudaSetDevice(p->device), "cudaSetDevice(plan device)");
  const fhwt_status r = run_on_device(p, in, out, workspace, st, analysis);
  cudaSetDevice(cur);
  return r;
}

fhwt_status run_on_device(fhwt_plan p, const float* in, float* out, void* workspace, fhwt_stream_t st,
                          bool analysis) {
  FHWT_TRY(check_ptrs(in, out, data_bytes(p)));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(st);
  char* ws = static_cast<char*>(workspace);
  if (ws && p->ws_bytes && (reinterpret_cast<uintptr_t>(ws) & 15) != 0)   // TMA maps and counters need it
    return fail(FHWT_ERR_MISALIGNED, "workspace must be 16-byte aligned");
  bool owned = false;
  if (p->ws_bytes && !ws) {
    void* t = nullptr;
    FHWT_TRY(ws_alloc(&t, p->ws_bytes, s));
    ws = static_cast<char*>(t);
    owned = true;
  }
  fhwt_status st_ = FHWT_OK;
  if (p->kind == 2) {
    // TMA row coordinates are int32 over the [batch * h] row view: larger batches run as
    // consecutive sub-batches (workspace needs scale with the batch, so the plan's buffer fits).
    const int64_t max_rows = env_int("FHWT_TEST_MAX_TMA_ROWS", 0) > 0 ? env_int("FHWT_TEST_MAX_TMA_ROWS", 0)
                                                                       : (int64_t(1) << 31) - 1;   // test hook
    const int64_t max_b = std::max<int64_t>(1, max_rows / p->h);
    if (p->batch <= max_b) {
      st_ = analysis ? run_ana2d(p, in, out, ws, s) : run_syn2d(p, in, out, ws, s);
    } else {
      for (int64_t b0 = 0; b0 < p->batch && st_ == FHWT_OK; b0 += max_b) {
        fhwt_plan_s sub = *p;
        sub.batch = std::min(max_b, p->batch - b0);
        plan_layout(&sub);
        const int64_t off = b0 * p->h * p->w;
        st_ = analysis ? run_ana2d(&sub, in + off, out + off, ws, s) : run_syn2d(&sub, in + off, out + off, ws, s);
      }
    }
  } else
    st_ = analysis ? run_ana1d(p, in, out, ws, s) : run_syn1d(p, in, out, ws, s);
  if (owned) {
    cudaError_t e = cudaFreeAsync(ws, s);
    if (st_ == FHWT_OK && e != cudaSuccess) return cuda_fail(e, "workspace cudaFreeAsync");
  }
  return st_;
}

}  // namespace

// ======================================================================= exported C ABI
extern "C" {

int fhwt_version(void) { return 10000; }

uint64_t fhwt_launch_count(void) { return g_launches.load(); }

const char* fhwt_last_error_message(void) { return g_last_error.c_str(); }

const char* fhwt_status_string(fhwt_status st) {
  switch (st) {
    case FHWT_OK: return "FHWT_OK";
    case FHWT_ERR_INVALID_ARG: return "FHWT_ERR_INVALID_ARG";
    case FHWT_ERR_EMPTY: return "FHWT_ERR_EMPTY";
    case FHWT_ERR_ODD_LENGTH: return "FHWT_ERR_ODD_LENGTH";
    case FHWT_ERR_INVALID_LEVELS: return "FHWT_ERR_INVALID_LEVELS";
    case FHWT_ERR_INSUFFICIENT_LENGTH: return "FHWT_ERR_INSUFFICIENT_LENGTH";
    case FHWT_ERR_SHAPE_MISMATCH: return "FHWT_ERR_SHAPE_MISMATCH";
    case FHWT_ERR_UNSUPPORTED_FILTER: return "FHWT_ERR_UNSUPPORTED_FILTER";
    case FHWT_ERR_MISALIGNED: return "FHWT_ERR_MISALIGNED";
    case FHWT_ERR_CUDA: return "FHWT_ERR_CUDA";
    case FHWT_ERR_NO_DEVICE: return "FHWT_ERR_NO_DEVICE";
  }
  return "FHWT_ERR_UNKNOWN";
}

fhwt_status fhwt_haar_filter_bank(fhwt_filter_bank* out) {
  if (!out) return fail(FHWT_ERR_INVALID_ARG, "null output");
  const double s = 1.0 / std::sqrt(2.0);
  out->b0[0] = s;  out->b0[1] = s;
  out->b1[0] = -s; out->b1[1] = s;
  out->a0[0] = s;  out->a0[1] = s;
  out->a1[0] = s;  out->a1[1] = -s;
  out->M = 2;
  return FHWT_OK;
}

// device >= 0 must name an existing CUDA device (checked once, here); -1 = current at call time
static fhwt_status check_device(int device) {
  if (device < -1) return fail(FHWT_ERR_INVALID_ARG, "device %d (use -1 for the current device)", device);
  if (device == -1) return FHWT_OK;
  int n = 0;
  FHWT_CUDA(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
  if (device >= n) return fail(FHWT_ERR_NO_DEVICE, "device %d of %d", device, n);
  return FHWT_OK;
}

fhwt_status fhwt_plan_1d(fhwt_plan* p, int64_t n, int64_t batch, int levels, const fhwt_filter_bank* fb,
                         int device) {
  if (!p) return fail(FHWT_ERR_INVALID_ARG, "null plan pointer");
  *p = nullptr;
  FHWT_TRY(check_1d(n, batch, levels));
  FHWT_TRY(check_bank(fb));
  FHWT_TRY(check_device(device));
  auto* pl = new fhwt_plan_s{};
  pl->kind = 1;
  pl->device = device;
  pl->n = n;
  pl->batch = batch;
  pl->levels = levels;
  plan_layout(pl);
  *p = pl;
  return FHWT_OK;
}

fhwt_status fhwt_plan_2d(fhwt_plan* p, int64_t h, int64_t w, int64_t batch, int levels, const fhwt_filter_bank* fb,
                         int device) {
  if (!p) return fail(FHWT_ERR_INVALID_ARG, "null plan pointer");
  *p = nullptr;
  FHWT_TRY(check_2d(h, w, batch, levels));
  FHWT_TRY(check_bank(fb));
  FHWT_TRY(check_device(device));
  auto* pl = new fhwt_plan_s{};
  pl->kind = 2;
  pl->device = device;
  pl->h = h;
  pl->w = w;
  pl->batch = batch;
  pl->levels = levels;
  plan_layout(pl);
  *p = pl;
  return FHWT_OK;
}

fhwt_status fhwt_plan_destroy(fhwt_plan p) {
  delete p;
  return FHWT_OK;
}

size_t fhwt_plan_workspace_bytes(fhwt_plan p) { return p ? p->ws_bytes : 0; }

fhwt_status fhwt_plan_analyze(fhwt_plan p, const float* d, float* coeffs, void* workspace, fhwt_stream_t s) {
  return run(p, d, coeffs, workspace, s, true);
}

fhwt_status fhwt_plan_synthesize(fhwt_plan p, const float* coeffs, float* dR, void* workspace, fhwt_stream_t s) {
  return run(p, coeffs, dR, workspace, s, false);
}

// SURVEY §8(b) names of the plan calls (same functions)
size_t fhwt_workspace_bytes(fhwt_plan p) { return fhwt_plan_workspace_bytes(p); }
fhwt_status fhwt_analyze(fhwt_plan p, const float* d, float* coeffs, void* workspace, fhwt_stream_t s) {
  return run(p, d, coeffs, workspace, s, true);
}
fhwt_status fhwt_synthesize(fhwt_plan p, const float* coeffs, float* dR, void* workspace, fhwt_stream_t s) {
  return run(p, coeffs, dR, workspace, s, false);
}

fhwt_status fhwt_analyze_1d(const float* d, float* coeffs, int64_t n, int64_t batch, int levels, fhwt_stream_t s) {
  fhwt_plan p;
  FHWT_TRY(fhwt_plan_1d(&p, n, batch, levels, nullptr, -1));
  fhwt_status st = run(p, d, coeffs, nullptr, s, true);
  delete p;
  return st;
}

fhwt_status fhwt_synthesize_1d(const float* coeffs, float* dR, int64_t n, int64_t batch, int levels, fhwt_stream_t s) {
  fhwt_plan p;
  FHWT_TRY(fhwt_plan_1d(&p, n, batch, levels, nullptr, -1));
  fhwt_status st = run(p, coeffs, dR, nullptr, s, false);
  delete p;
  return st;
}

fhwt_status fhwt_analyze_2d(const float* d, float* coeffs, int64_t h, int64_t w, int64_t batch, int levels,
                            fhwt_stream_t s) {
  fhwt_plan p;
  FHWT_TRY(fhwt_plan_2d(&p, h, w, batch, levels, nullptr, -1));
  fhwt_status st = run(p, d, coeffs, nullptr, s, true);
  delete p;
  return st;
}

fhwt_status fhwt_synthesize_2d(const float* coeffs, float* dR, int64_t h, int64_t w, int64_t batch, int levels,
                               fhwt_stream_t s) {
  fhwt_plan p;
  FHWT_TRY(fhwt_plan_2d(&p, h, w, batch, levels, nullptr, -1));
  fhwt_status st = run(p, coeffs, dR, nullptr, s, false);
  delete p;
  return st;
}

int64_t fhwt_band_offset_1d(int64_t n, int level, int band, int64_t* len) {
  if (n <= 0 || level < 1 || level > 62 || (band != 0 && band != 1) || n % (int64_t(1) << level)) return -1;
  const int64_t l = n >> level;
  if (len) *len = l;
  return band == 0 ? 0 : l;
}

int64_t fhwt_band_offset_2d(int64_t h, int64_t w, int level, int band, int64_t* rows, int64_t* cols) {
  if (h <= 0 || w <= 0 || level < 1 || level > 62 || band < 0 || band > 3) return -1;
  if (h % (int64_t(1) << level) || w % (int64_t(1) << level)) return -1;
  const int64_t hl = h >> level, wl = w >> level;
  if (rows) *rows = hl;
  if (cols) *cols = wl;
  const int64_t r = (band & 2) ? hl : 0, c = (band & 1) ? wl : 0;
  return r * w + c;
}

fhwt_status fhwt_pack_ll_2d(const float* coeffs, float* ll_packed, int64_t h, int64_t w, int64_t batch, int levels,
                            fhwt_stream_t s) {
  FHWT_TRY(check_2d(h, w, batch, levels));
  if (!coeffs || !ll_packed) return fail(FHWT_ERR_INVALID_ARG, "null buffer pointer");
  FHWT_CUDA(launch_pack_ll(coeffs, ll_packed, h, w, batch, levels, reinterpret_cast<cudaStream_t>(s)), "pack_ll launch");
  return FHWT_OK;
}

fhwt_status fhwt_pack_ll_2d_peers(const float* coeffs, float* const* peer_ll, int rank, int npeers, int64_t h,
                                  int64_t w, int64_t batch, int levels, fhwt_stream_t s) {
  FHWT_TRY(check_2d(h, w, batch, levels));
  if (!coeffs || !peer_ll) return fail(FHWT_ERR_INVALID_ARG, "null pointer");
  if (npeers < 1 || rank < 0 || rank >= npeers) return fail(FHWT_ERR_INVALID_ARG, "rank %d of %d peers", rank, npeers);
  FHWT_CUDA(launch_pack_ll_peers(coeffs, peer_ll, rank, npeers, h, w, batch, levels, reinterpret_cast<cudaStream_t>(s)),
            "pack_ll_peers launch");
  return FHWT_OK;
}

fhwt_status fhwt_plan_pack_ll_2d(fhwt_plan p, const float* coeffs, float* ll_packed, fhwt_stream_t s) {
  if (!p) return fail(FHWT_ERR_INVALID_ARG, "null plan");
  if (p->kind != 2) return fail(FHWT_ERR_INVALID_ARG, "fhwt_plan_pack_ll_2d needs a 2-D plan");
  return fhwt_pack_ll_2d(coeffs, ll_packed, p->h, p->w, p->batch, p->levels, s);
}

}  // extern "C"

// ---------------------------------------------------------------------- host-buffer streaming
namespace {

fhwt_status roundtrip_host(fhwt_plan_s* full, const float* h_d, float* h_c, float* h_r, int64_t unit_elems,
                           int64_t chunk) {
  const int64_t B = full->batch;
  if (!h_d || !h_r) return fail(FHWT_ERR_INVALID_ARG, "null host buffer");
  const int64_t unit_bytes = unit_elems * int64_t(sizeof(float));
  // Default chunk ~128 MB (pipeline fill/drain = one chunk each way), NS streams in rotation so an
  // H2D of chunk i+1 never waits behind the D2H of chunk i-1 on the same stream.
  const int64_t mb = env_int("FHWT_RT_CHUNK_MB", 128);
  if (chunk <= 0) chunk = std::max<int64_t>(1, (mb << 20) / std::max<int64_t>(unit_bytes, 1));
  chunk = std::min(chunk, B);
  constexpr int kMaxStreams = 4;
  const int NS = std::max(2, std::min(kMaxStreams, env_int("FHWT_RT_STREAMS", 3)));
  // chunk-sized plan (same shape, fewer units)
  fhwt_plan_s cp = *full;
  cp.batch = chunk;
  plan_layout(&cp);
  cudaStream_t st[kMaxStreams];
  for (int i = 0; i < NS; ++i) FHWT_CUDA(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking), "stream create");
  const size_t cbytes = size_t(chunk) * size_t(unit_bytes);
  const size_t wsb = align_up(cp.ws_bytes, 256);
  char* buf[kMaxStreams] = {nullptr, nullptr, nullptr, nullptr};
  fhwt_status rs = FHWT_OK;
  for (int i = 0; i < NS && rs == FHWT_OK; ++i) {
    void* t = nullptr;
    rs = ws_alloc(&t, 3 * align_up(cbytes, 256) + wsb, st[i]);
    buf[i] = static_cast<char*>(t);
  }
  for (int64_t u0 = 0, it = 0; u0 < B && rs == FHWT_OK; u0 += chunk, ++it) {
    const int k = int(it % NS);
    const int64_t cnt = std::min(chunk, B - u0);
    cudaStream_t s = st[k];
    float* dd = reinterpret_cast<float*>(buf[k]);
    float* dc = reinterpret_cast<float*>(buf[k] + align_up(cbytes, 256));
    float* dr = reinterpret_cast<float*>(buf[k] + 2 * align_up(cbytes, 256));
    char* ws = buf[k] + 3 * align_up(cbytes, 256);
    const size_t bytes = size_t(cnt) * size_t(unit_bytes);
    fhwt_plan_s pp = cp;
    if (cnt != chunk) {
      pp.batch = cnt;
      plan_layout(&pp);
    }
    cudaError_t e = cudaMemcpyAsync(dd, h_d + u0 * unit_elems, bytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) { rs = cuda_fail(e, "H2D copy"); break; }
    rs = run(&pp, dd, dc, ws, reinterpret_cast<fhwt_stream_t>(s), true);
    if (rs != FHWT_OK) break;
    if (h_c) {
      e = cudaMemcpyAsync(h_c + u0 * unit_elems, dc, bytes, cudaMemcpyDeviceToHost, s);
      if (e != cudaSuccess) { rs = cuda_fail(e, "D2H copy"); break; }
    }
    rs = run(&pp, dc, dr, ws, reinterpret_cast<fhwt_stream_t>(s), false);
    if (rs != FHWT_OK) break;
    e = cudaMemcpyAsync(h_r + u0 * unit_elems, dr, bytes, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) { rs = cuda_fail(e, "D2H copy"); break; }
  }
  for (int i = 0; i < NS; ++i) {
    if (buf[i]) cudaFreeAsync(buf[i], st[i]);
    cudaError_t e = cudaStreamSynchronize(st[i]);
    if (rs == FHWT_OK && e != cudaSuccess) rs = cuda_fail(e, "stream synchronize");
    cudaStreamDestroy(st[i]);
  }
  return rs;
}

}  // namespace

extern "C" fhwt_status fhwt_roundtrip_2d_host(const float* h_d, float* h_coeffs, float* h_dR, int64_t h, int64_t w,
                                              int64_t batch, int levels, int64_t chunk) {
  fhwt_plan p;
  FHWT_TRY(fhwt_plan_2d(&p, h, w, batch, levels, nullptr, -1));
  fhwt_status st = roundtrip_host(p, h_d, h_coeffs, h_dR, h * w, chunk);
  delete p;
  return st;
}

extern "C" fhwt_status fhwt_roundtrip_1d_host(const float* h_d, float* h_coeffs, float* h_dR, int64_t n, int64_t batch,
                                              int levels, int64_t chunk) {
  fhwt_plan p;
  FHWT_TRY(fhwt_plan_1d(&p, n, batch, levels, nullptr, -1));
  fhwt_status st = roundtrip_host(p, h_d, h_coeffs, h_dR, n, chunk);
  delete p;
  return st;
}

// ---------------------------------------------------------------------- direct-form baseline (f3)
namespace {

Lines_t lines(int64_t batch, int64_t bstride, int64_t count, int64_t sstride, int64_t len, int64_t nstride) {
  return Lines_t{batch, bstride, count, sstride, len, nstride};
}

fhwt_status direct_common(const void* in, const void* out, const void* ws, size_t bytes) {
  FHWT_TRY(check_ptrs(in, out, bytes));
  if (!ws) return fail(FHWT_ERR_INVALID_ARG, "the direct-form baseline needs a workspace (fhwt_direct_workspace_bytes)");
  return FHWT_OK;
}

}  // namespace

extern "C" size_t fhwt_direct_workspace_bytes(int dims, int64_t n_or_h, int64_t w, int64_t batch) {
  if (n_or_h <= 0 || batch <= 0 || (dims == 2 && w <= 0)) return 0;
  const size_t S = size_t(batch) * size_t(n_or_h) * size_t(dims == 2 ? w : 1);
  return (dims == 2 ? 4 : 3) * S * sizeof(float);
}

// 1-D: level j works on lines of len n >> (j-1); y0/y1 scratch 2*B*n, approx ping-pong 2 x B*n/2.
extern "C" fhwt_status fhwt_direct_analyze_1d(const float* d, float* coeffs, int64_t n, int64_t batch, int levels,
                                              void* workspace, fhwt_stream_t st) {
  FHWT_TRY(check_1d(n, batch, levels));
  FHWT_TRY(direct_common(d, coeffs, workspace, size_t(n) * batch * 4));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(st);
  float* y0 = static_cast<float*>(workspace);
  float* y1 = y0 + batch * n;
  float* pp[2] = {y1 + batch * n, y1 + batch * n + batch * (n / 2)};
  const float* x = d;
  int64_t xs = n;  // signal stride of the current input
  for (int j = 1; j <= levels; ++j) {
    const int64_t len = n >> (j - 1), half = len / 2;
    float* a = j == levels ? coeffs : pp[j & 1];
    const int64_t as = j == levels ? n : half;
    FHWT_CUDA(direct_analysis_lines(x, lines(1, 0, batch, xs, len, 1), a, lines(1, 0, batch, as, half, 1),
                                    coeffs + half, lines(1, 0, batch, n, half, 1), y0, y1, s),
              "direct analysis 1-D");
    x = a;
    xs = as;
  }
  return FHWT_OK;
}

extern "C" fhwt_status fhwt_direct_synthesize_1d(const float* coeffs, float* dR, int64_t n, int64_t batch, int levels,
                                                 void* workspace, fhwt_stream_t st) {
  FHWT_TRY(check_1d(n, batch, levels));
  FHWT_TRY(direct_common(coeffs, dR, workspace, size_t(n) * batch * 4));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(st);
  float* u0 = static_cast<float*>(workspace);
  float* u1 = u0 + batch * n;
  float* pp[2] = {u1 + batch * n, u1 + batch * n + batch * (n / 2)};
  const float* a = coeffs;
  int64_t as = n;
  for (int j = levels; j >= 1; --j) {
    const int64_t half = n >> j, len = 2 * half;
    float* r = j == 1 ? dR : pp[j & 1];
    const int64_t rs = j == 1 ? n : len;
    FHWT_CUDA(direct_synthesis_lines(a, lines(1, 0, batch, as, half, 1), coeffs + half, lines(1, 0, batch, n, half, 1),
                                     r, lines(1, 0, batch, rs, len, 1), u0, u1, s),
              "direct synthesis 1-D");
    a = r;
    as = rs;
  }
  return FHWT_OK;
}

// 2-D, level j on the hc x wc LL region: rows (Fig. 2 along every row) -> L, H (compact
// B x hc x wc/2); columns of L -> LL, LH and of H -> HL, HH.  Workspace: y0/y1 (2 S), L/H (S),
// LL ping-pong (2 x S/4).
extern "C" fhwt_status fhwt_direct_analyze_2d(const float* d, float* coeffs, int64_t h, int64_t w, int64_t batch,
                                              int levels, void* workspace, fhwt_stream_t st) {
  FHWT_TRY(check_2d(h, w, batch, levels));
  FHWT_TRY(direct_common(d, coeffs, workspace, size_t(h) * w * batch * 4));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(st);
  const int64_t S = batch * h * w;
  float* y0 = static_cast<float*>(workspace);
  float* y1 = y0 + S;
  float* Lb = y1 + S;
  float* Hb = Lb + S / 2;
  float* pp[2] = {Hb + S / 2, Hb + S / 2 + S / 4};
  const float* x = d;
  int64_t xb = h * w, xp = w;  // image stride, row pitch of the current LL input
  for (int j = 1; j <= levels; ++j) {
    const int64_t hc = h >> (j - 1), wc = w >> (j - 1), hh = hc / 2, wh = wc / 2;
    // rows: batch x hc lines of wc -> L, H (batch x hc x wh, compact)
    FHWT_CUDA(direct_analysis_lines(x, lines(batch, xb, hc, xp, wc, 1), Lb, lines(batch, hc * wh, hc, wh, wh, 1), Hb,
                                    lines(batch, hc * wh, hc, wh, wh, 1), y0, y1, s),
              "direct analysis 2-D rows");
    // columns of L: wh lines of hc (stride wh) -> LL (to ping-pong or coeffs), LH (coeffs)
    const bool last = j == levels;
    float* ll = last ? coeffs : pp[j & 1];
    const int64_t llb = last ? h * w : hh * wh, llp = last ? w : wh;
    FHWT_CUDA(direct_analysis_lines(Lb, lines(batch, hc * wh, wh, 1, hc, wh), ll, lines(batch, llb, wh, 1, hh, llp),
                                    coeffs + hh * w, lines(batch, h * w, wh, 1, hh, w), y0, y1, s),
              "direct analysis 2-D columns (L)");
    FHWT_CUDA(direct_analysis_lines(Hb, lines(batch, hc * wh, wh, 1, hc, wh), coeffs + wh,
                                    lines(batch, h * w, wh, 1, hh, w), coeffs + hh * w + wh,
                                    lines(batch, h * w, wh, 1, hh, w), y0, y1, s),
              "direct analysis 2-D columns (H)");
    x = ll;
    xb = llb;
    xp = llp;
  }
  return FHWT_OK;
}

extern "C" fhwt_status fhwt_direct_synthesize_2d(const float* coeffs, float* dR, int64_t h, int64_t w, int64_t batch,
                                                 int levels, void* workspace, fhwt_stream_t st) {
  FHWT_TRY(check_2d(h, w, batch, levels));
  FHWT_TRY(direct_common(coeffs, dR, workspace, size_t(h) * w * batch * 4));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(st);
  const int64_t S = batch * h * w;
  float* u0 = static_cast<float*>(workspace);
  float* u1 = u0 + S;
  float* Lb = u1 + S;
  float* Hb = Lb + S / 2;
  float* pp[2] = {Hb + S / 2, Hb + S / 2 + S / 4};
  const float* ll = coeffs;
  int64_t llb = h * w, llp = w;
  for (int j = levels; j >= 1; --j) {
    const int64_t hh = h >> j, wh = w >> j, hc = 2 * hh, wc = 2 * wh;
    // columns: (LL, LH) -> L and (HL, HH) -> H, each batch x hc x wh compact
    FHWT_CUDA(direct_synthesis_lines(ll, lines(batch, llb, wh, 1, hh, llp), coeffs + hh * w,
                                     lines(batch, h * w, wh, 1, hh, w), Lb, lines(batch, hc * wh, wh, 1, hc, wh), u0,
                                     u1, s),
              "direct synthesis 2-D columns (L)");
    FHWT_CUDA(direct_synthesis_lines(coeffs + wh, lines(batch, h * w, wh, 1, hh, w), coeffs + hh * w + wh,
                                     lines(batch, h * w, wh, 1, hh, w), Hb, lines(batch, hc * wh, wh, 1, hc, wh), u0,
                                     u1, s),
              "direct synthesis 2-D columns (H)");
    // rows: (L, H) -> LL_{j-1}
    float* r = j == 1 ? dR : pp[j & 1];
    const int64_t rb = j == 1 ? h * w : hc * wc, rp = j == 1 ? w : wc;
    FHWT_CUDA(direct_synthesis_lines(Lb, lines(batch, hc * wh, hc, wh, wh, 1), Hb, lines(batch, hc * wh, hc, wh, wh, 1),
                                     r, lines(batch, rb, hc, rp, wc, 1), u0, u1, s),
              "direct synthesis 2-D rows");
    ll = r;
    llb = rb;
    llp = rp;
  }
  return FHWT_OK;
}

// Static op counts.  Per 1-D level on N input samples (analysis) / N output samples (synthesis):
//   direct analysis  4N mul + 2N add   (2 filters x N positions x (2 mul + 1 add))
//   direct synthesis 4N mul + 3N add   (2 filters x N positions x (2 mul + 1 add) + N branch sums)
//   fast             N mul + N add     (N/2 butterflies x (2 mul + 2 add))
// 2-D separable level on hc x wc: hc lines of wc plus wc lines of hc (the L and H halves).
// This library's 2-D kernels: per 2x2 block 4 mul + 8 add (exact x1/2 folding), both directions.
extern "C" fhwt_status fhwt_op_counts(int dims, int64_t n_or_h, int64_t w, int64_t batch, int levels, int structure,
                                      int synthesis, uint64_t* mul, uint64_t* add) {
  if (!mul || !add || structure < 0 || structure > 2 || (dims != 1 && dims != 2))
    return fail(FHWT_ERR_INVALID_ARG, "bad op-count query");
  if (dims == 1)
    FHWT_TRY(check_1d(n_or_h, batch, levels));
  else
    FHWT_TRY(check_2d(n_or_h, w, batch, levels));
  auto per = [&](uint64_t N, uint64_t* m, uint64_t* a) {
    if (structure == 0) {
      *m = 4 * N;
      *a = (synthesis ? 3 : 2) * N;
    } else {
      *m = N;
      *a = N;
    }
  };
  uint64_t M = 0, A = 0;
  for (int j = 1; j <= levels; ++j) {
    if (dims == 1) {
      uint64_t m, a;
      per(uint64_t(n_or_h >> (j - 1)), &m, &a);
      M += m;
      A += a;
    } else {
      const uint64_t hc = uint64_t(n_or_h >> (j - 1)), wc = uint64_t(w >> (j - 1));
      if (structure == 2) {
        M += hc * wc;       // (hc/2)(wc/2) blocks x 4 mul
        A += 2 * hc * wc;   // x 8 add
      } else {
        uint64_t m1, a1, m2, a2;
        per(wc, &m1, &a1);
        per(hc, &m2, &a2);
        M += hc * m1 + wc * m2;
        A += hc * a1 + wc * a2;
      }
    }
  }
  *mul = M * uint64_t(batch);
  *add = A * uint64_t(batch);
  return FHWT_OK;
}

// ---------------------------------------------------------------------- LL-only lowpass (f1)
extern "C" size_t fhwt_lowpass_workspace_bytes(int64_t h, int64_t w, int64_t batch, int levels) {
  if (check_2d(h, w, batch, levels) != FHWT_OK) return 0;
  return lowpass_workspace_bytes(h, w, batch, levels);
}

extern "C" size_t fhwt_lowpass_bf16_workspace_bytes(int64_t h, int64_t w, int64_t batch, int levels) {
  if (check_2d(h, w, batch, levels) != FHWT_OK) return 0;
  return lowpass_bf16_workspace_bytes(h, w, batch, levels);
}

extern "C" fhwt_status fhwt_lowpass_2d_bf16(const uint16_t* d, float* ll, int64_t h, int64_t w, int64_t batch,
                                            int levels, void* workspace, fhwt_stream_t st) {
  FHWT_TRY(check_2d(h, w, batch, levels));
  if (!d || !ll) return fail(FHWT_ERR_INVALID_ARG, "null buffer pointer");
  if (w % 8 != 0) return fail(FHWT_ERR_MISALIGNED, "bf16 lowpass reads rows in 8-pixel (16-B) vectors: w %% 8 != 0");
  if ((reinterpret_cast<uintptr_t>(d) & 15) || (reinterpret_cast<uintptr_t>(ll) & 3))
    return fail(FHWT_ERR_MISALIGNED, "bf16 input must be 16-byte aligned");
  const char* a = reinterpret_cast<const char*>(d);
  const char* b = reinterpret_cast<const char*>(ll);
  const size_t in_bytes = size_t(batch) * h * w * 2, out_bytes = size_t(batch) * (h >> levels) * (w >> levels) * 4;
  if (a < b + out_bytes && b < a + in_bytes) return fail(FHWT_ERR_INVALID_ARG, "input and output buffers overlap");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(st);
  const size_t wsb = lowpass_bf16_workspace_bytes(h, w, batch, levels);
  void* ws = workspace;
  if (wsb && !ws) FHWT_TRY(ws_alloc(&ws, wsb, s));
  cudaError_t e = launch_lowpass_bf16(d, ll, h, w, batch, levels, ws, s);
  if (wsb && !workspace) cudaFreeAsync(ws, s);
  if (e != cudaSuccess) return cuda_fail(e, "lowpass bf16 launch");
  return FHWT_OK;
}

extern "C" fhwt_status fhwt_lowpass_2d_u8(const uint8_t* d, float* ll, int64_t h, int64_t w, int64_t batch,
                                          int levels, void* workspace, fhwt_stream_t st) {
  FHWT_TRY(check_2d(h, w, batch, levels));
  if (!d || !ll) return fail(FHWT_ERR_INVALID_ARG, "null buffer pointer");
  const int M = levels < 4 ? levels : 4;
  if ((reinterpret_cast<uintptr_t>(d) & ((uintptr_t(1) << M) - 1)) || (reinterpret_cast<uintptr_t>(ll) & 3))
    return fail(FHWT_ERR_MISALIGNED, "uint8 input must be %d-byte aligned (one vector row load per block)", 1 << M);
  const char* a = reinterpret_cast<const char*>(d);
  const char* b = reinterpret_cast<const char*>(ll);
  const size_t in_bytes = size_t(batch) * h * w, out_bytes = size_t(batch) * (h >> levels) * (w >> levels) * 4;
  if (a < b + out_bytes && b < a + in_bytes) return fail(FHWT_ERR_INVALID_ARG, "input and output buffers overlap");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(st);
  const size_t wsb = lowpass_workspace_bytes(h, w, batch, levels);
  void* ws = workspace;
  if (wsb && !ws) FHWT_TRY(ws_alloc(&ws, wsb, s));
  cudaError_t e = launch_lowpass_u8(d, ll, h, w, batch, levels, ws, s);
  if (wsb && !workspace) cudaFreeAsync(ws, s);
  if (e != cudaSuccess) return cuda_fail(e, "lowpass launch");
  return FHWT_OK;
}
