// Leverage scores of a tall factor with orthonormal-ish columns
// (src/linalg.py:73-84 `leverage_scores` + the rank test of `reduced_qr`,
// :38-52), in three short kernels and two passes over the factor:
//
//   1. k_ls_gram:  G = A^T A by row chunks (fixed chunk -> CTA map, each CTA
//      sums its rows in order: deterministic), upper triangle only;
//   2. k_ls_chol:  one CTA reduces the chunk partials in a fixed order,
//      factors G = R^T R (Cholesky), applies the reference's rank test
//      |R_jj| < 1e-12 ||A||_F (||A||_F^2 = trace G) conservatively: the Gram
//      cannot resolve R_jj below ~1e-8 ||A||, so a failed pivot or
//      min R_jj < 1e-2 max R_jj (cond(A) > ~100, where the squared condition
//      number would also cost score bits) raises the "unsafe" flag and the
//      caller decides on the Householder/TSQR path instead; then inverts R;
//   3. k_ls_rows:  l_i = || a_i R^-1 ||^2, thread per row.
//
// Since Q = A R^-1 for the R of any QR of A, these are the scores the
// reference reads from its Householder Q.  Their rounding follows cond(A)^2
// instead of cond(A): exact to ~1e-16 for the orthonormal factors the
// sketched driver feeds (cond = 1).  Replaces a multi-level TSQR (latency
// bound: 0.72 ms at 2e5 x 20) with ~3 launches of a few microseconds.
#include "skx_common.cuh"

namespace skx {

constexpr int kLsMaxR = 32;
constexpr int kLsChunks = 296;  // 2 per SM
constexpr int kLsThreads = 256;

__global__ void __launch_bounds__(kLsThreads) k_ls_gram(const double* __restrict__ a, int64_t s,
                                                        int R, double* __restrict__ part) {
  __shared__ double tile[64 * kLsMaxR];
  const int nup = R * (R + 1) / 2;
  const int64_t per = (s + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = imin(s, lo + per);
  // thread t owns upper-triangle entries t, t + 256, ... (p <= q)
  double acc[3] = {0.0, 0.0, 0.0};
  int pp[3], qq[3];
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    int e = threadIdx.x + u * kLsThreads, p = 0;
    while (e >= R - p && p < R) {
      e -= R - p;
      ++p;
    }
    pp[u] = p;
    qq[u] = p + e;
  }
  for (int64_t r0 = lo; r0 < hi; r0 += 64) {
    const int rows = (int)imin(64, hi - r0);
    __syncthreads();
    for (int e = threadIdx.x; e < rows * R; e += kLsThreads) tile[e] = a[r0 * R + e];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      if (threadIdx.x + u * kLsThreads < nup) {
        const int p = pp[u], q = qq[u];
        double t = acc[u];
        for (int r = 0; r < rows; ++r) t = fma(tile[r * R + p], tile[r * R + q], t);
        acc[u] = t;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    const int e = threadIdx.x + u * kLsThreads;
    if (e < nup) part[(int64_t)blockIdx.x * nup + e] = acc[u];
  }
}

__global__ void __launch_bounds__(kLsThreads) k_ls_chol(const double* __restrict__ part, int nparts,
                                                        int R, double* __restrict__ rinv,
                                                        int* __restrict__ bad) {
  __shared__ double G[kLsMaxR * kLsMaxR];
  __shared__ double X[kLsMaxR * kLsMaxR];
  __shared__ int fail;
  const int nup = R * (R + 1) / 2;
  for (int e = threadIdx.x; e < nup; e += blockDim.x) {
    double t = 0.0;
    for (int c = 0; c < nparts; ++c) t += part[(int64_t)c * nup + e];
    int p = 0, f = e;
    while (f >= R - p) {
      f -= R - p;
      ++p;
    }
    G[p * R + p + f] = t;
  }
  if (threadIdx.x == 0) fail = 0;
  __syncthreads();
  double tr = 0.0;
  for (int j = 0; j < R; ++j) tr += G[j * R + j];
  const double tol = 1e-12 * sqrt(tr);
  // upper Cholesky in place: row j of R in G[j, j..R)
  for (int j = 0; j < R; ++j) {
    if (threadIdx.x == 0) {
      double d = G[j * R + j];
      for (int k = 0; k < j; ++k) d -= G[k * R + j] * G[k * R + j];
      if (!(d > 0.0)) {
        fail = 1;
        d = 0.0;
      }
      const double rjj = sqrt(d);
      if (!(rjj >= tol)) fail = 1;
      G[j * R + j] = rjj;
    }
    __syncthreads();
    const double rjj = G[j * R + j];
    for (int l = j + 1 + threadIdx.x; l < R; l += blockDim.x) {
      double t = G[j * R + l];
      for (int k = 0; k < j; ++k) t -= G[k * R + j] * G[k * R + l];
      G[j * R + l] = rjj > 0.0 ? t / rjj : 0.0;
    }
    __syncthreads();
  }
  // X = R^-1 (upper), column c by back substitution
  for (int c = threadIdx.x; c < R; c += blockDim.x) {
    for (int i = R - 1; i >= 0; --i) {
      double t = i == c ? 1.0 : 0.0;
      for (int k = i + 1; k <= c; ++k) t -= G[i * R + k] * X[k * R + c];
      X[i * R + c] = (i > c) ? 0.0 : (G[i * R + i] > 0.0 ? t / G[i * R + i] : 0.0);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) rinv[e] = X[e];
  if (threadIdx.x == 0) {
    double mn = G[0], mx = G[0];
    for (int j = 1; j < R; ++j) {
      mn = fmin(mn, G[j * R + j]);
      mx = fmax(mx, G[j * R + j]);
    }
    *bad = (fail || !(mn >= 1e-2 * mx)) ? 1 : 0;
  }
}

// RP = R rounded up to a multiple of 8 (X zero padded), so the row and the
// triangular product stay in registers
// (128 threads: at up to 255 registers the CTA still fits beside one CTA of
// the fitness kernel that runs next to the leverage path)
constexpr int kLsRowThreads = 128;

template <int RP>
__global__ void __launch_bounds__(kLsRowThreads) k_ls_rows(const double* __restrict__ a, int64_t s,
                                                        int R, const double* __restrict__ rinv,
                                                        double* __restrict__ scores) {
  __shared__ double X[RP * RP];
  for (int e = threadIdx.x; e < RP * RP; e += blockDim.x) {
    const int i = e / RP, c = e % RP;
    X[e] = (i < R && c < R) ? rinv[i * R + c] : 0.0;
  }
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s;
       i += (int64_t)gridDim.x * blockDim.x) {
    double row[RP];
#pragma unroll
    for (int k = 0; k < RP; ++k) row[k] = k < R ? a[i * R + k] : 0.0;
    double sum = 0.0;
#pragma unroll
    for (int c = 0; c < RP; ++c) {
      double y = 0.0;
#pragma unroll
      for (int k = 0; k <= c; ++k) y = fma(row[k], X[k * RP + c], y);
      sum = fma(y, y, sum);
    }
    scores[i] = sum;
  }
}

}  // namespace skx

using namespace skx;

extern "C" int skx_lev_scores(const double* a, int64_t s, int R, double* scores, int* bad,
                              void* ws, size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(R >= 1 && R <= kLsMaxR, "skx_lev_scores: 1 <= R <= 32");
  SKX_REQUIRE(s > R, "skx_lev_scores: leverage scores need a strictly tall matrix");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_lev_scores: ws_bytes is NULL");
  const int nup = R * (R + 1) / 2;
  const int nparts = (int)imin(kLsChunks, (s + 63) / 64);
  Arena ar(ws, *ws_bytes);
  double* part = ar.take<double>((size_t)nparts * nup);
  double* rinv = ar.take<double>((size_t)R * R);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_lev_scores: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  k_ls_gram<<<nparts, kLsThreads, 0, st>>>(a, s, R, part);
  k_ls_chol<<<1, kLsThreads, 0, st>>>(part, nparts, R, rinv, bad);
  const unsigned g = (unsigned)imin((s + kLsRowThreads - 1) / kLsRowThreads, (int64_t)num_sms() * 16);
  if (R <= 8) k_ls_rows<8><<<g, kLsRowThreads, 0, st>>>(a, s, R, rinv, scores);
  else if (R <= 16) k_ls_rows<16><<<g, kLsRowThreads, 0, st>>>(a, s, R, rinv, scores);
  else if (R <= 24) k_ls_rows<24><<<g, kLsRowThreads, 0, st>>>(a, s, R, rinv, scores);
  else k_ls_rows<32><<<g, kLsRowThreads, 0, st>>>(a, s, R, rinv, scores);
  return check_launch("skx_lev_scores", 3);
}
