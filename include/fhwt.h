/*
 * fhwt.h — C ABI of the B200-native Fast Haar Wavelet Transform (arXiv 1002.2184).
 *
 * The library computes the paper's polyphase ("Fast Haar") two-channel analysis bank
 * (§III, Fig. 4: ↓2 moved to the input, one butterfly × b00 = 1/√2 per
 * even/odd input pair) and synthesis bank (§IV, Figs. 6-7, Eq. (19): ↑2 moved
 * to the output), iterated as a multi-level dyadic (Mallat) decomposition of batched 1-D
 * signals and applied separably (rows, then columns) to batched 2-D images.
 *
 * Conventions:
 *   R1 pairs are (x[2k], x[2k+1]): zero delay, exact PR on finite blocks, 2^L-aligned blocks
 *      are independent (no halo).
 *   R2 approx d0[k] = (x[2k] + x[2k+1]) / √2, detail d1[k] = (x[2k] − x[2k+1]) / √2 (§II taps).
 *   R3 unity-gain synthesis: r[2k] = (d0 + d1)/√2, r[2k+1] = (d0 − d1)/√2.
 *   R8 2-D: rows then columns; LH = low along rows, high along columns; quadrants [[LL,HL],[LH,HH]].
 *
 * Data layout (all buffers fp32, contiguous row-major, no padding):
 *   1-D: d is [batch][n]; coeffs is [batch][n] in Mallat order [a_J | d_J | ... | d_1],
 *        detail of level j at offsets [n/2^j, n/2^(j-1)), final approximation at [0, n/2^J).
 *   2-D: d is [batch][h][w]; coeffs is [batch][h][w]; at level j the region
 *        [0, h/2^(j-1)) x [0, w/2^(j-1)) holds [[LL_j, HL_j], [LH_j, HH_j]], recursion on LL.
 *
 * Ownership: every d / coeffs / d_R / workspace pointer is a DEVICE pointer owned by the
 * caller (except the *_host entry points, which take host pointers).  Plans hold only host
 * state and are owned by the library until fhwt_plan_destroy().  Input and output buffers
 * must not overlap (no in-place transform).
 *
 * Errors: every function returns a status; nothing aborts or throws.  Argument validation is
 * synchronous and happens before any launch; kernels run asynchronously on the given stream
 * and asynchronous faults surface at the caller's next synchronisation (or as FHWT_ERR_CUDA
 * from a later call).  fhwt_last_error_message() returns a thread-local description of the
 * last failure.  Non-finite inputs are not scanned; they propagate under IEEE rules.
 *
 * Environment: the library reads no environment variable unless FHWT_TUNING=1 is set; then the
 * FHWT_* sweep knobs of DESIGN.md §13b override the measured kernel / tile / ring-depth choices
 * (bitwise-equal alternatives kept for A/B measurement and tests).
 *
 * Precision: butterflies of levels 1-3 in fp32, from level 4 on in
 * fp64 (analysis), the hand-off between kernel passes in fp64; outputs rounded once to fp32.
 * Synthesis in fp32.
 */
#ifndef FHWT_H
#define FHWT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same object as cudaStream_t / CUstream.  NULL = the legacy default stream. */
typedef struct CUstream_st *fhwt_stream_t;

typedef enum {
  FHWT_OK = 0,
  FHWT_ERR_INVALID_ARG = 1,         /* null pointer, negative size, overlapping in/out, bad band id  */
  FHWT_ERR_EMPTY = 2,               /* SPEC EmptySignal: n == 0, h*w == 0 or batch == 0              */
  FHWT_ERR_ODD_LENGTH = 3,          /* SPEC OddLength / OddDimension                                 */
  FHWT_ERR_INVALID_LEVELS = 4,      /* SPEC InvalidLevels: levels < 1 (or > 62)                      */
  FHWT_ERR_INSUFFICIENT_LENGTH = 5, /* SPEC InsufficientLength: n (or h, w) % 2^levels != 0          */
  FHWT_ERR_SHAPE_MISMATCH = 6,      /* plan kind (1-D / 2-D) does not match the call                 */
  FHWT_ERR_UNSUPPORTED_FILTER = 7,  /* taps differ from the §II Haar set by > 1e-12, or M != 2       */
  FHWT_ERR_MISALIGNED = 8,          /* multi-level call with a device pointer not 16-B aligned       */
  FHWT_ERR_CUDA = 9,                /* CUDA runtime / driver failure (see fhwt_last_error_message)   */
  FHWT_ERR_NO_DEVICE = 10           /* no sm_100 device is current                                   */
} fhwt_status;

/* The paper's statement of the problem: analysis filters b0/b1, synthesis filters a0/a1, M = 2
 * (§II, "In Haar Wavelet M=2").  Tap k multiplies x[n-k]. */
typedef struct {
  double b0[2], b1[2], a0[2], a1[2];
  int M;
} fhwt_filter_bank;

/* Fills *out with the §II Haar set: b0 = [1/√2, 1/√2], b1 = [-1/√2, 1/√2],
 * a0 = [1/√2, 1/√2], a1 = [1/√2, -1/√2], M = 2.  INVALID_ARG if out == NULL. */
fhwt_status fhwt_haar_filter_bank(fhwt_filter_bank *out);

const char *fhwt_status_string(fhwt_status st);
const char *fhwt_last_error_message(void);
int fhwt_version(void);                    /* major*10000 + minor*100 + patch */
uint64_t fhwt_launch_count(void);          /* number of kernels this library has launched */

/* ------------------------------------------------------------------ plans
 * A plan validates and freezes (shape, levels, filter bank).  fb == NULL means the §II set; any
 * other bank must equal it within 1e-12 per tap with M == 2, else UNSUPPORTED_FILTER (the
 * polyphase reduction of PAPER.md:102/:168, B00 = B01 = A00 = A01 = 1/√2, is Haar-specific).
 * A plan is immutable: concurrent use from several streams is safe with distinct workspaces. */
typedef struct fhwt_plan_s *fhwt_plan;

/* 1-D: batch signals of n samples, `levels` dyadic levels.  Needs n % 2^levels == 0.
 * device: the CUDA device the plan's calls run on (the library makes it current for the call and
 * restores the caller's device afterwards; buffers and stream must belong to it), or -1 for the
 * device that is current at each call.
 * Errors: INVALID_ARG (p NULL, n/batch < 0, device < -1), EMPTY, INVALID_LEVELS, ODD_LENGTH,
 * INSUFFICIENT_LENGTH, UNSUPPORTED_FILTER, NO_DEVICE (device >= device count), CUDA. */
fhwt_status fhwt_plan_1d(fhwt_plan *p, int64_t n, int64_t batch, int levels, const fhwt_filter_bank *fb,
                         int device);

/* 2-D: batch images of h x w pixels, `levels` separable levels.  Needs h, w % 2^levels == 0.
 * device and errors as fhwt_plan_1d. */
fhwt_status fhwt_plan_2d(fhwt_plan *p, int64_t h, int64_t w, int64_t batch, int levels,
                         const fhwt_filter_bank *fb, int device);

fhwt_status fhwt_plan_destroy(fhwt_plan p);

/* Bytes of device workspace a call on this plan needs.  Holds the fp64 coarse-LL hand-off between
 * passes (2-D levels > 5, 1-D levels > 10) and, for 2-D plans, 256 bytes of tile counters: the
 * fused 2-D kernels hand out their tiles in global order from a counter the library zeroes with a
 * stream-ordered memset before each launch.  1-D plans with levels <= 10 need 0 bytes.  Calls that
 * may run concurrently (different streams) need distinct workspaces. */
size_t fhwt_plan_workspace_bytes(fhwt_plan p);

/* Analysis (forward DWT): d [batch][...] -> coeffs (Mallat layout, same shape).
 * workspace: 16-byte aligned device buffer of fhwt_plan_workspace_bytes(p) bytes (else
 * FHWT_ERR_MISALIGNED), or NULL (the library then
 * allocates and frees it stream-ordered on s).  Asynchronous on s. */
fhwt_status fhwt_plan_analyze(fhwt_plan p, const float *d, float *coeffs, void *workspace, fhwt_stream_t s);

/* Synthesis (inverse DWT): coeffs (Mallat layout) -> d_R.  Same workspace rules. */
fhwt_status fhwt_plan_synthesize(fhwt_plan p, const float *coeffs, float *d_R, void *workspace,
                                 fhwt_stream_t s);

/* The same three plan calls under the names of SURVEY §8(b) (fhwt_workspace_bytes, fhwt_analyze,
 * fhwt_synthesize): identical arguments, behaviour and errors. */
size_t fhwt_workspace_bytes(fhwt_plan p);
fhwt_status fhwt_analyze(fhwt_plan p, const float *d, float *coeffs, void *workspace, fhwt_stream_t s);
fhwt_status fhwt_synthesize(fhwt_plan p, const float *coeffs, float *d_R, void *workspace, fhwt_stream_t s);

/* ------------------------------------------------------------------ one-shot entry points
 * Equivalent to plan + call + destroy with the §II filter bank. */
fhwt_status fhwt_analyze_1d(const float *d, float *coeffs, int64_t n, int64_t batch, int levels, fhwt_stream_t s);
fhwt_status fhwt_synthesize_1d(const float *coeffs, float *d_R, int64_t n, int64_t batch, int levels,
                               fhwt_stream_t s);
fhwt_status fhwt_analyze_2d(const float *d, float *coeffs, int64_t h, int64_t w, int64_t batch, int levels,
                            fhwt_stream_t s);
fhwt_status fhwt_synthesize_2d(const float *coeffs, float *d_R, int64_t h, int64_t w, int64_t batch,
                               int levels, fhwt_stream_t s);

/* ------------------------------------------------------------------ layout helpers (host only)
 * 1-D: element offset of band `band` (0 = approximation a_level, 1 = detail d_level) of `level`
 * inside one signal's Mallat row; *len receives its length.  Returns -1 on bad arguments. */
int64_t fhwt_band_offset_1d(int64_t n, int level, int band, int64_t *len);
/* 2-D: element offset (row * w + col) of band (0 = LL, 1 = HL, 2 = LH, 3 = HH) of `level` inside
 * one image's Mallat layout; *rows, *cols receive the band's extent.  Returns -1 on bad args. */
int64_t fhwt_band_offset_2d(int64_t h, int64_t w, int level, int band, int64_t *rows, int64_t *cols);

/* Packs the coarsest LL_levels of every image of coeffs (row pitch w) into ll_packed,
 * contiguous [batch][h/2^levels][w/2^levels] (device).  Used before the NCCL all-gather of
 * row-band sharded images. */
fhwt_status fhwt_pack_ll_2d(const float *coeffs, float *ll_packed, int64_t h, int64_t w, int64_t batch,
                            int levels, fhwt_stream_t s);
/* The pack fused with the row-band all-gather over peer memory (NVLink P2P
 * stores instead of pack + collective): this rank's LL_levels block (as fhwt_pack_ll_2d) is stored
 * into EVERY peer's gather buffer at element offset rank * batch*(h>>levels)*(w>>levels).
 * peer_ll: DEVICE array of npeers device pointers, peer access enabled (e.g. the buffer_ptrs_dev of a
 * torch symmetric-memory rendezvous), each buffer >= npeers * batch*(h>>levels)*(w>>levels) floats;
 * rank in [0, npeers).  Asynchronous on s; the stores are visible to a peer only after a cross-rank
 * barrier that follows this call on every rank (the caller's).  Errors: INVALID_ARG, as
 * fhwt_plan_2d, CUDA. */
fhwt_status fhwt_pack_ll_2d_peers(const float *coeffs, float *const *peer_ll, int rank, int npeers, int64_t h,
                                  int64_t w, int64_t batch, int levels, fhwt_stream_t s);
/* The same pack with (h, w, batch, levels) taken from a 2-D plan (SURVEY §8(b) form).
 * Errors: INVALID_ARG (NULL plan, 1-D plan, NULL buffers). */
fhwt_status fhwt_plan_pack_ll_2d(fhwt_plan p, const float *coeffs, float *ll_packed, fhwt_stream_t s);

/* ------------------------------------------------------------------ host-buffer round trip
 * End-to-end DWT + IDWT on HOST buffers (pinned memory recommended): the batch is streamed in
 * chunks of `chunk` images (or signals) through device staging buffers owned by the call, with
 * H2D copy, analysis, synthesis and D2H copies of coeffs (if h_coeffs != NULL) and d_R
 * overlapped across 3 CUDA streams.  Blocks until the
 * results are in host memory.
 * chunk <= 0 picks a default.  Errors as the device entry points, plus CUDA for copy failures. */
fhwt_status fhwt_roundtrip_2d_host(const float *h_d, float *h_coeffs, float *h_dR, int64_t h, int64_t w,
                                   int64_t batch, int levels, int64_t chunk);
fhwt_status fhwt_roundtrip_1d_host(const float *h_d, float *h_coeffs, float *h_dR, int64_t n, int64_t batch,
                                   int levels, int64_t chunk);

/* ------------------------------------------------------------------ LL-only lowpass path (§8(f) f1)
 * The paper's image output (Fig. 12: "Lowpass output ... by applying ... Fast Haar
 * wavelet"): only the LL branch of the separable Fast Haar analysis, LL_j = ½((a+b)+(c+d)) per 2x2
 * block of LL_{j-1}, from 8-bit images.  d: [batch][h][w] uint8 (device, aligned to
 * 2^min(levels,4) bytes); ll: [batch][h/2^levels][w/2^levels] fp32 (device) = the LL_levels band of
 * fhwt_analyze_2d on the same image converted to fp32 (exact: integer sums below 2^53).
 * workspace: fhwt_lowpass_workspace_bytes bytes (0 for levels <= 4), or NULL (stream-ordered
 * allocation on s).  Errors as fhwt_plan_2d, plus MISALIGNED, INVALID_ARG, CUDA. */
size_t fhwt_lowpass_workspace_bytes(int64_t h, int64_t w, int64_t batch, int levels);
fhwt_status fhwt_lowpass_2d_u8(const uint8_t *d, float *ll, int64_t h, int64_t w, int64_t batch, int levels,
                               void *workspace, fhwt_stream_t s);

/* The same LL-only path from bfloat16 images (the "bf16 I/O" of SURVEY §8(f) f1): d is
 * [batch][h][w] bf16 bit patterns (device, 16-byte aligned, w % 8 == 0), ll fp32 as above.  bf16 ->
 * fp32 is exact and the levels are computed as fhwt_analyze_2d computes them (levels 1-3 fp32,
 * from level 4 fp64), so ll equals the LL band of fhwt_analyze_2d on the fp32 image bitwise.
 * workspace: fhwt_lowpass_bf16_workspace_bytes bytes (0 for levels <= 3), or NULL (stream-ordered
 * allocation on s).  Errors as fhwt_lowpass_2d_u8 (MISALIGNED also for w % 8 != 0). */
size_t fhwt_lowpass_bf16_workspace_bytes(int64_t h, int64_t w, int64_t batch, int levels);
fhwt_status fhwt_lowpass_2d_bf16(const uint16_t *d, float *ll, int64_t h, int64_t w, int64_t batch, int levels,
                                 void *workspace, fhwt_stream_t s);

/* ------------------------------------------------------------------ direct-form baseline (§8(f) f3)
 * The paper's ORIGINAL structure, for comparison with the Fast structure on the same hardware:
 * analysis = full-rate filtering with b0/b1 then decimation keeping n = 2k+1 (Fig. 2, Eqs. (1)-(4),
 * PAPER.md:58-74); synthesis = zero-insertion upsampling then full-rate filtering with a0/a1 and
 * summation (Fig. 5, Eq. (13)); level by level, rows then columns, every
 * intermediate materialised in device memory.  Same layouts, validation and errors as the Fast entry
 * points; workspace is REQUIRED (device, fhwt_direct_workspace_bytes bytes, caller-owned). */
size_t fhwt_direct_workspace_bytes(int dims, int64_t n_or_h, int64_t w, int64_t batch);
fhwt_status fhwt_direct_analyze_1d(const float *d, float *coeffs, int64_t n, int64_t batch, int levels,
                                   void *workspace, fhwt_stream_t s);
fhwt_status fhwt_direct_synthesize_1d(const float *coeffs, float *d_R, int64_t n, int64_t batch, int levels,
                                      void *workspace, fhwt_stream_t s);
fhwt_status fhwt_direct_analyze_2d(const float *d, float *coeffs, int64_t h, int64_t w, int64_t batch, int levels,
                                   void *workspace, fhwt_stream_t s);
fhwt_status fhwt_direct_synthesize_2d(const float *coeffs, float *d_R, int64_t h, int64_t w, int64_t batch,
                                      int levels, void *workspace, fhwt_stream_t s);

/* Static arithmetic-operation counts (multiplications, additions incl. subtractions) of one
 * multi-level transform on sample data ("less than quarter").
 * dims = 1 (n_or_h = n, w ignored) or 2; structure: 0 = direct (Figs. 2/5, full-rate, multiplies by
 * inserted zeros), 1 = Fast as drawn in the paper (separable 1-D butterflies, Figs. 4/7),
 * 2 = this library's kernels (2-D butterflies folded to one exact x1/2 per 2x2 block);
 * synthesis = 0 analysis / 1 synthesis.  INVALID_ARG on bad arguments, plus the plan errors. */
fhwt_status fhwt_op_counts(int dims, int64_t n_or_h, int64_t w, int64_t batch, int levels, int structure,
                           int synthesis, uint64_t *mul, uint64_t *add);

#ifdef __cplusplus
}
#endif
#endif /* FHWT_H */
