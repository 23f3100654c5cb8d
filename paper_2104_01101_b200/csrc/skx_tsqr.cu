// K5/K6 helper: R factor of a tall-skinny matrix by communication-avoiding
// Householder QR (TSQR).  Used for the thin SVDs of the rank-constrained solve
// (D = Q^T X_ls is w x s_n with w <= 30; src/linalg.py:110-111), the range
// finder sketch B (s_n x k1, src/tucker.py:141) and the leverage-score QRs of
// the factors (src/linalg.py:73-84).
//
// Level 1: one CTA per block of BR rows factors its tile in shared memory with
// LAPACK-style Householder reflectors (dlarfg conventions) and writes its w x w
// R.  The stacked R's are factored again until one block remains.  Fixed order
// of every reduction: deterministic.
#include "skx_common.cuh"

namespace skx {

constexpr int kTsqrThreads = 256;

// T is column-major in shared memory: T[j * ldt + i], i < rows, j < w.
template <int BR>
__global__ void __launch_bounds__(kTsqrThreads) k_tsqr_block(const double* __restrict__ A, int64_t n,
                                                            int w, int64_t rs, int64_t cs,
                                                            double* __restrict__ Rout) {
  extern __shared__ double T[];
  __shared__ double s_tau, s_beta;
  __shared__ double s_dot[64];
  const int ldt = BR + 1;
  const int64_t r0 = blockIdx.x * (int64_t)BR;
  const int rows = (int)imin(BR, n - r0);
  for (int q = threadIdx.x; q < BR * w; q += blockDim.x) {
    const int j = q / BR, i = q - j * BR;
    T[j * ldt + i] = i < rows ? A[(r0 + i) * rs + j * cs] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int kmax = min(rows, w);
  for (int k = 0; k < kmax; ++k) {
    double* col = T + k * ldt;
    // ---- dlarfg on col[k..rows)
    if (wid == 0) {
      double sg = 0.0;
      for (int i = k + 1 + lane; i < rows; i += 32) sg = fma(col[i], col[i], sg);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sg += __shfl_xor_sync(0xffffffffu, sg, o);
      if (lane == 0) {
        const double x0 = col[k];
        if (sg == 0.0) {
          s_tau = 0.0;
          s_beta = x0;
        } else {
          const double nrm = sqrt(fma(x0, x0, sg));
          const double beta = x0 >= 0.0 ? -nrm : nrm;
          s_tau = (beta - x0) / beta;
          s_beta = beta;
        }
      }
    }
    __syncthreads();
    const double tau = s_tau, beta = s_beta;
    if (tau != 0.0) {
      const double scale = 1.0 / (col[k] - beta);
      for (int i = k + 1 + threadIdx.x; i < rows; i += blockDim.x) col[i] *= scale;
    }
    __syncthreads();
    // ---- apply H = I - tau v v^T (v_k = 1) to columns k+1..w-1
    if (tau != 0.0) {
      for (int j = k + 1 + wid; j < w; j += nw) {
        const double* cj = T + j * ldt;
        double d = 0.0;
        for (int i = k + 1 + lane; i < rows; i += 32) d = fma(col[i], cj[i], d);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        if (lane == 0) s_dot[j & 63] = tau * (cj[k] + d);
      }
      __syncthreads();
      for (int j = k + 1 + wid; j < w; j += nw) {
        double* cj = T + j * ldt;
        const double f = s_dot[j & 63];
        if (lane == 0) cj[k] -= f;
        for (int i = k + 1 + lane; i < rows; i += 32) cj[i] = fma(-f, col[i], cj[i]);
      }
    }
    if (threadIdx.x == 0) col[k] = beta;
    __syncthreads();
  }
  // R_b rows 0..w-1 (zero-padded), row-major w x w at Rout + blockIdx.x * w * w
  double* R = Rout + (int64_t)blockIdx.x * w * w;
  for (int q = threadIdx.x; q < w * w; q += blockDim.x) {
    const int i = q / w, j = q - i * w;
    R[q] = (j >= i && i < rows) ? T[j * ldt + i] : 0.0;
  }
}

}  // namespace skx

using namespace skx;

extern "C" int skx_tsqr_r(const double* a, int64_t n, int w, int64_t rs, int64_t cs, double* r,
                          void* ws, size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(w >= 1 && w <= 64, "skx_tsqr_r: 1 <= w <= 64 columns supported");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_tsqr_r: ws_bytes is NULL");
  const int BR = w <= 32 ? 256 : 128;
  // level sizes
  int64_t rows = n, total = 0;
  int levels = 0;
  while (true) {
    const int64_t nb = (rows + BR - 1) / BR;
    ++levels;
    if (nb <= 1) break;
    total += nb * w * w;
    rows = nb * w;
  }
  Arena ar(ws, *ws_bytes);
  double* buf = ar.take<double>(total > 0 ? total : 1);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_tsqr_r: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t smem = (size_t)w * (BR + 1) * sizeof(double);
  auto kern = BR == 256 ? k_tsqr_block<256> : k_tsqr_block<128>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const double* src = a;
  int64_t srs = rs, scs = cs;
  rows = n;
  double* out = buf;
  int launches = 0;
  while (true) {
    const int64_t nb = (rows + BR - 1) / BR;
    double* dst = nb <= 1 ? r : out;
    kern<<<(unsigned)(nb > 0 ? nb : 1), kTsqrThreads, smem, s>>>(src, rows, w, srs, scs, dst);
    ++launches;
    if (nb <= 1) break;
    src = out;
    srs = w;
    scs = 1;
    rows = nb * w;
    out += nb * w * w;
  }
  return check_launch("skx_tsqr_r", launches);
}
