// §8(f) f3 — the paper's ORIGINAL (direct) Haar filter bank on B200, as a measured baseline.
//
// Analysis, Fig. 2 / Eqs. (1)-(4): full-rate filtering with the §II taps
// y_i[n] = b_i[0] x[n] + b_i[1] x[n-1] for every n, materialised, then decimation keeping n = 2k+1
// (reading R1).  Synthesis, Fig. 5 / Eq. (13): zero-insertion upsampling,
// materialised, then full-rate filtering with a0 / a1 and summation.  Level by level, rows then
// columns for 2-D, every intermediate in HBM — the structure whose cost the paper's "factor 2" and
// "less than quarter" claims are measured against.  fp32 with the taps rounded to
// fp32; the Fast kernels (haar1d.cu / haar2d.cu) are the product path.
#include "fhwt_internal.cuh"

namespace fhwt {
namespace {

// Lines_t (fhwt_internal.cuh): `batch` groups of `count` signals of `len` samples; sample n of
// signal s of group b at base[b * bstride + s * sstride + n * nstride].  Element index i ->
// (b, s, n) with n fastest when samples are contiguous (rows), s fastest otherwise (columns), so
// consecutive threads touch consecutive addresses.
struct Lines : Lines_t {
  __device__ __forceinline__ int64_t total() const { return batch * count * len; }
  __device__ __forceinline__ int64_t off(int64_t b, int64_t s, int64_t n) const {
    return b * bstride + s * sstride + n * nstride;
  }
  __device__ __forceinline__ void at(int64_t i, int64_t& b, int64_t& s, int64_t& n) const {
    const int64_t per = count * len;
    b = i / per;
    const int64_t r = i - b * per;
    if (nstride == 1) {
      s = r / len;
      n = r - s * len;
    } else {
      n = r / count;
      s = r - n * count;
    }
  }
};

struct Taps {
  float b0[2], b1[2], a0[2], a1[2];
};

#define GRID_STRIDE(i, total) \
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < (total); i += int64_t(gridDim.x) * blockDim.x)

// Fig. 2 filtering at full rate: y0/y1 (same line geometry as x, in scratch buffers).
__global__ void direct_filter_kernel(const float* __restrict__ x, Lines lx, float* __restrict__ y0,
                                     float* __restrict__ y1, Lines ly, Taps t) {
  GRID_STRIDE(i, lx.total()) {
    int64_t b, s, n;
    lx.at(i, b, s, n);
    const float xn = x[lx.off(b, s, n)];
    const float xm = n > 0 ? x[lx.off(b, s, n - 1)] : 0.f;   // x[-1] = 0
    const int64_t o = ly.off(b, s, n);
    y0[o] = t.b0[0] * xn + t.b0[1] * xm;
    y1[o] = t.b1[0] * xn + t.b1[1] * xm;
  }
}

// ↓2 keeping the odd phase: approx[k] = y0[2k+1], detail[k] = y1[2k+1].
__global__ void direct_decimate_kernel(const float* __restrict__ y0, const float* __restrict__ y1, Lines ly,
                                       float* __restrict__ a, Lines la, float* __restrict__ d, Lines ld) {
  GRID_STRIDE(i, la.total()) {
    int64_t b, s, k;
    la.at(i, b, s, k);
    const int64_t src = ly.off(b, s, 2 * k + 1);
    a[la.off(b, s, k)] = y0[src];
    d[ld.off(b, s, k)] = y1[src];
  }
}

// Fig. 5 upsampling by zero insertion: u[2k] = band[k], u[2k+1] = 0.
__global__ void direct_upsample_kernel(const float* __restrict__ a, Lines la, const float* __restrict__ d, Lines ld,
                                       float* __restrict__ u0, float* __restrict__ u1, Lines lu) {
  GRID_STRIDE(i, lu.total()) {
    int64_t b, s, n;
    lu.at(i, b, s, n);
    const int64_t o = lu.off(b, s, n);
    if (n & 1) {
      u0[o] = 0.f;
      u1[o] = 0.f;
    } else {
      u0[o] = a[la.off(b, s, n >> 1)];
      u1[o] = d[ld.off(b, s, n >> 1)];
    }
  }
}

// Fig. 5 filtering at full rate and summation: r = a0 * u0 + a1 * u1.
__global__ void direct_synth_filter_kernel(const float* __restrict__ u0, const float* __restrict__ u1, Lines lu,
                                           float* __restrict__ r, Lines lr, Taps t) {
  GRID_STRIDE(i, lu.total()) {
    int64_t b, s, n;
    lu.at(i, b, s, n);
    const int64_t o = lu.off(b, s, n);
    const float p0 = n > 0 ? u0[o - lu.nstride] : 0.f, p1 = n > 0 ? u1[o - lu.nstride] : 0.f;
    const float r0 = t.a0[0] * u0[o] + t.a0[1] * p0;
    const float r1 = t.a1[0] * u1[o] + t.a1[1] * p1;
    r[lr.off(b, s, n)] = r0 + r1;
  }
}

int grid_of(int64_t total) {
  int64_t g = (total + 255) / 256;
  if (g > 148 * 64) g = 148 * 64;
  return int(g < 1 ? 1 : g);
}

Taps make_taps() {
  const float s = float(kS64);
  return Taps{{s, s}, {-s, s}, {s, s}, {s, -s}};
}

}  // namespace

static Lines L_(const Lines_t& l) { return Lines{l}; }

// Compact full-rate scratch geometry for lines `l` (same element order as the kernels' index map).
static Lines scratch_of(const Lines_t& l) {
  Lines y{l};
  y.bstride = l.count * l.len;
  if (l.nstride == 1) {
    y.sstride = l.len;
    y.nstride = 1;
  } else {
    y.sstride = 1;
    y.nstride = l.count;
  }
  return y;
}

// One direct analysis stage (Fig. 2): x lines -> (approx a, detail d) lines of half length, via the
// full-rate scratch y0 / y1 (each batch * count * len floats).
cudaError_t direct_analysis_lines(const float* x, Lines_t lx, float* a, Lines_t la, float* d, Lines_t ld, float* y0,
                                  float* y1, cudaStream_t s) {
  const Lines X = L_(lx), Y = scratch_of(lx);
  count_launch();
  direct_filter_kernel<<<grid_of(X.batch * X.count * X.len), 256, 0, s>>>(x, X, y0, y1, Y, make_taps());
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  count_launch();
  direct_decimate_kernel<<<grid_of(la.batch * la.count * la.len), 256, 0, s>>>(y0, y1, Y, a, L_(la), d, L_(ld));
  return cudaGetLastError();
}

// One direct synthesis stage (Fig. 5): (a, d) lines of length len -> r lines of length 2 len, via
// the upsampled scratch u0 / u1.
cudaError_t direct_synthesis_lines(const float* a, Lines_t la, const float* d, Lines_t ld, float* r, Lines_t lr,
                                   float* u0, float* u1, cudaStream_t s) {
  const Lines U = scratch_of(lr);
  count_launch();
  direct_upsample_kernel<<<grid_of(U.batch * U.count * U.len), 256, 0, s>>>(a, L_(la), d, L_(ld), u0, u1, U);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  count_launch();
  direct_synth_filter_kernel<<<grid_of(U.batch * U.count * U.len), 256, 0, s>>>(u0, u1, U, r, L_(lr), make_taps());
  return cudaGetLastError();
}

}  // namespace fhwt
