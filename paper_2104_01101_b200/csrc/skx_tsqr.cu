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
  __shared__ double s_dot[128];
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
        if (lane == 0) s_dot[j & 127] = tau * (cj[k] + d);
      }
      __syncthreads();
      for (int j = k + 1 + wid; j < w; j += nw) {
        double* cj = T + j * ldt;
        const double f = s_dot[j & 127];
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

// ---- register variant for w <= WP <= 32: thread t of the CTA holds row t of
// the 256-row tile in registers; the step loop is unrolled (k is a compile-
// time index into the row), so the only shared-memory traffic is the three
// block reductions per reflector: ||x||^2 below the diagonal, the vector of
// dot products v^T A[:, k+1:] (warp butterfly reduce-scatter, then a fixed-
// order sum over the warps) and its broadcast.  Same reflector conventions
// (dlarfg) as k_tsqr_block, hence the same R up to rounding.
constexpr int kTsqrRows = 256;

// Butterfly reduce-scatter of NP-vectors (NP a power of two <= 32) over the
// warp: afterwards lane l holds the warp sum of component l % NP.  Stage h
// exchanges the half of the live block the partner keeps: NP - 1 shuffles,
// then 32/NP - 1 more to add the lane groups.
template <int NP>
__device__ __forceinline__ double warp_reduce_scatter(double (&p)[NP], int lane) {
#pragma unroll
  for (int h = NP / 2; h >= 1; h >>= 1) {
    const bool upper = (lane & h) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = upper ? p[i] : p[i + h];
      const double keep = upper ? p[i + h] : p[i];
      p[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  double r = p[0];
#pragma unroll
  for (int h = NP; h < 32; h <<= 1) r += __shfl_xor_sync(0xffffffffu, r, h);
  return r;
}

template <int WP>
__global__ void __launch_bounds__(kTsqrRows, 1) k_tsqr_reg(const double* __restrict__ A, int64_t n,
                                                         int w, int64_t rs, int64_t cs,
                                                         double* __restrict__ Rout) {
  constexpr int NC = WP <= 32 ? 32 : 64;  // reduction components (dot products)
  constexpr int NP = WP <= 8 ? 8 : WP <= 16 ? 16 : 32;
  __shared__ double red[kTsqrRows / 32][NC + 1];
  __shared__ double dv[NC];
  __shared__ double s_x0;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  constexpr int NW = kTsqrRows / 32;
  const int64_t r0 = blockIdx.x * (int64_t)kTsqrRows;
  const int rows = (int)imin(kTsqrRows, n - r0);
  double* R = Rout + (int64_t)blockIdx.x * w * w;
  for (int q = t; q < w * w; q += kTsqrRows) R[q] = 0.0;
  // a[j] holds column k + j of this thread's row at step k: the row shifts
  // left by one after every reflector, so the step body has static register
  // indices without unrolling the step loop (small code, no I-cache thrash)
  double a[WP];
#pragma unroll
  for (int j = 0; j < WP; ++j)
    a[j] = (t < rows && j < w) ? A[(r0 + t) * rs + (int64_t)j * cs] : 0.0;
  const int kmax = min(rows, w);
#pragma unroll 1
  for (int k = 0; k < kmax; ++k) {
    const int rem = w - k;  // live columns a[0..rem)
    // ---- dlarfg on column k, rows k..rows-1
    double sq = t > k ? a[0] * a[0] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if (lane == 0) red[wid][NC] = sq;
    if (t == k) s_x0 = a[0];
    __syncthreads();
    double sg = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) sg += red[q][NC];
    const double x0 = s_x0;
    double tau = 0.0, beta = x0;
    if (sg != 0.0) {
      const double nrm = sqrt(fma(x0, x0, sg));
      beta = x0 >= 0.0 ? -nrm : nrm;
      tau = (beta - x0) / beta;
    }
    if (tau != 0.0) {  // uniform
      const double scale = 1.0 / (x0 - beta);
      const double v = t > k ? a[0] * scale : (t == k ? 1.0 : 0.0);
      // ---- d_j = sum_t v_t a_t[j], 0 < j < rem, in blocks of NP components
#pragma unroll
      for (int j0 = 0; j0 < WP; j0 += NP) {
        if (j0 >= rem) break;
        double p[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) p[j] = (j0 + j > 0 && j0 + j < rem) ? v * a[j0 + j] : 0.0;
        const double rsum = warp_reduce_scatter<NP>(p, lane);
        if (lane < NP) red[wid][j0 + lane] = rsum;
      }
      __syncthreads();
      if (t < rem) {
        double d = 0.0;
#pragma unroll
        for (int q = 0; q < NW; ++q) d += red[q][t];
        dv[t] = tau * d;
      }
      __syncthreads();
#pragma unroll
      for (int j = 1; j < WP; ++j)
        if (j < rem) a[j] = fma(-dv[j], v, a[j]);
    }
    if (t == k) {  // row k of R is final
      a[0] = beta;
#pragma unroll
      for (int j = 0; j < WP; ++j)
        if (j < rem) R[(int64_t)k * w + k + j] = a[j];
    }
#pragma unroll
    for (int j = 0; j + 1 < WP; ++j) a[j] = a[j + 1];
    a[WP - 1] = 0.0;
    __syncthreads();  // red / dv / s_x0 reuse in the next step
  }
}

}  // namespace skx

using namespace skx;

extern "C" int skx_tsqr_r(const double* a, int64_t n, int w, int64_t rs, int64_t cs, double* r,
                          void* ws, size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(w >= 1 && w <= 96, "skx_tsqr_r: 1 <= w <= 96 columns supported");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_tsqr_r: ws_bytes is NULL");
  // 256-row tiles: every level shrinks the stack by 256 / w >= 2.7
  const int BR = kTsqrRows;
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
  size_t smem = (size_t)w * (BR + 1) * sizeof(double);
  using KF = void (*)(const double*, int64_t, int, int64_t, int64_t, double*);
  KF kern = k_tsqr_block<kTsqrRows>;  // w > 64: Householder tiles in shared memory
  if (w <= 8) kern = k_tsqr_reg<8>, smem = 0;
  else if (w <= 16) kern = k_tsqr_reg<16>, smem = 0;
  else if (w <= 24) kern = k_tsqr_reg<24>, smem = 0;
  else if (w <= 32) kern = k_tsqr_reg<32>, smem = 0;
  else if (w <= 40) kern = k_tsqr_reg<40>, smem = 0;
  else if (w <= 48) kern = k_tsqr_reg<48>, smem = 0;
  else if (w <= 64) kern = k_tsqr_reg<64>, smem = 0;
  if (smem) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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
