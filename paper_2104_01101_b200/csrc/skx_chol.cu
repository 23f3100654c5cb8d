// K5 for wide sketched systems (r = prod of the other ranks > 128: config 3
// r = 512, config 5 r = 400): the Cholesky factor R (R^T R = G) of the r x r
// Gram of Z and R^-1, in ONE CTA, replacing cuSOLVER potrf (~40 launches per
// factorisation) and the cuBLAS TRSM against the identity (src/linalg.py:44-52
// reduced_qr(z) is what they stand in for, through Cholesky QR with the same
// rank test; see linalg.sketch_qr_dev).
//
// Blocked left-looking Cholesky by 32-row panels of R, then the blocked
// inverse bottom-up.  The O(r^3) parts are FP64 tensor-core GEMMs
// (mma.sync m8n8k4): one operand panel staged in shared memory, the other
// streamed from L2 (R and R^-1 are written and re-read by the same CTA);
// the 32 x 32 diagonal blocks are factored / inverted by one warp in
// registers.  Fixed order everywhere: deterministic.
#include <math.h>

#include "skx_common.cuh"

namespace skx {

namespace {

constexpr int kCiThreads = 512;  // 16 warps
constexpr int kCiWarps = kCiThreads / 32;
constexpr int kCiMaxN = 512;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Plain (coherent) global load: R and R^-1 are written earlier in the same
// kernel by other warps of this CTA, so the non-coherent __ldg path is unsafe.
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

constexpr int kSaLd = 36;  // SA row stride (doubles): = 4 mod 16, conflict-free fragment reads

// acc[mt] += sum_k SA[k][8 mt + q] * B[k][col], k in [0, k_hi) (k_hi a multiple
// of 4), for one 8-column tile starting at global column `col0` of row-major B
// (leading dim ld); columns >= ncol and rows >= k_valid read as zero.
// SA: shared, [k][kSaLd].
__device__ __forceinline__ void panel_gemm_tile(const double* __restrict__ SA, const double* B,
                                                int64_t ld, int col0, int ncol, int k_hi,
                                                int k_valid, double (&acc)[4][2], int q, int c) {
  const int col = col0 + q;
  const bool live = col < ncol;
  int k = 0;
  // four B loads in flight per lane
  for (; k + 16 <= k_hi; k += 16) {
    double b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int kk = k + 4 * u + c;
      b[u] = (live && kk < k_valid) ? ldcg(B + (int64_t)kk * ld + col) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double* sa = SA + (k + 4 * u + c) * kSaLd + q;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) dmma(acc[mt][0], acc[mt][1], sa[8 * mt], b[u]);
    }
  }
  for (; k < k_hi; k += 4) {
    const int kk = k + c;
    const double b = (live && kk < k_valid) ? ldcg(B + (int64_t)kk * ld + col) : 0.0;
    const double* sa = SA + (k + c) * kSaLd + q;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) dmma(acc[mt][0], acc[mt][1], sa[8 * mt], b);
  }
}

}  // namespace

// G: n x n SPD (row-major, symmetric; the upper triangle is read).  R, Rinv:
// n x n row-major outputs (upper; zero below the diagonal); the block row being
// formed is kept in place in R (resp. Rinv) between the GEMM and the solve.
// info: 0, or k+1 for the first non-positive (or NaN) pivot k -- R and Rinv
// are then zero.
__global__ void __launch_bounds__(kCiThreads, 1) k_chol_inv(const double* __restrict__ G, int n,
                                                           double* R, double* Rinv,
                                                           int* __restrict__ info) {
  extern __shared__ __align__(16) double SA[];  // [K][kSaLd] panel operand
  __shared__ double Rpp[32][33];  // current diagonal block (factor, then inverse)
  __shared__ double rdiag[32];
  __shared__ int s_bad;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, q = lane >> 2, c = lane & 3;
  const int np = (n + 31) / 32;
  if (tid == 0) s_bad = 0;
  __syncthreads();

  // ---------------- Cholesky, panel p: R rows [c0, c0 + w)
  for (int p = 0; p < np; ++p) {
    const int c0 = 32 * p, w = min(32, n - c0), nc = n - c0;
    for (int e = tid; e < c0 * 32; e += kCiThreads) {
      const int k = e >> 5, m = e & 31;
      SA[k * kSaLd + m] = m < w ? ldcg(R + (int64_t)k * n + c0 + m) : 0.0;
    }
    __syncthreads();
    // block row: R[c0 + m][c0 + j] <- G[c0 + m][c0 + j] - sum_{k < c0} R[k][c0 + m] R[k][c0 + j]
    const int ntile = (nc + 7) / 8;
    for (int jt = wid; jt < ntile; jt += kCiWarps) {
      double acc[4][2] = {};
      if (c0 > 0) panel_gemm_tile(SA, R, n, c0 + 8 * jt, n, c0, c0, acc, q, c);
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int m = 8 * mt + q, j = 8 * jt + 2 * c + h;
          if (m < w && j < nc)
            R[(int64_t)(c0 + m) * n + c0 + j] = G[(int64_t)(c0 + m) * n + c0 + j] - acc[mt][h];
        }
    }
    __syncthreads();
    // diagonal block: one warp, lane j holds column j of the upper triangle
    if (wid == 0) {
      double t[32];
#pragma unroll
      for (int i = 0; i < 32; ++i)
        t[i] = (i <= lane && lane < w) ? ldcg(R + (int64_t)(c0 + i) * n + c0 + lane)
                                       : (i == lane ? 1.0 : 0.0);
      int bad = 0;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const double piv = __shfl_sync(0xffffffffu, t[k], k);
        if (!(piv > 0.0)) {  // warp-uniform; also catches NaN
          bad = k + 1;
          break;
        }
        const double d = sqrt(piv), rd = 1.0 / d;
        if (lane == k) t[k] = d;
        else if (lane > k) t[k] *= rd;  // r_kj
        const double rkj = t[k];
#pragma unroll
        for (int i = k + 1; i < 32; ++i) {
          const double rki = __shfl_sync(0xffffffffu, rkj, i);
          if (lane >= i) t[i] = fma(-rki, rkj, t[i]);
        }
      }
      if (bad && lane == 0) s_bad = c0 + bad;
#pragma unroll
      for (int i = 0; i < 32; ++i) Rpp[i][lane] = i <= lane ? t[i] : 0.0;
      if (!bad) rdiag[lane] = 1.0 / t[lane];
    }
    __syncthreads();
    if (s_bad) break;
    // the rest of the block row: R_pp^T X = T[:, 32:], one column per thread, in place
    for (int j = 32 + tid; j < nc; j += kCiThreads) {
      double* col = R + (int64_t)c0 * n + c0 + j;
      double x[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        double v = ldcg(col + (int64_t)k * n);  // w = 32 whenever nc > 32
#pragma unroll
        for (int i = 0; i < k; ++i) v = fma(-Rpp[i][k], x[i], v);
        x[k] = v * rdiag[k];
      }
#pragma unroll
      for (int k = 0; k < 32; ++k) col[(int64_t)k * n] = x[k];
    }
    // the diagonal block and the zero lower part of the block row
    for (int e = tid; e < w * c0; e += kCiThreads) R[(int64_t)(c0 + e / c0) * n + e % c0] = 0.0;
    for (int e = tid; e < w * w; e += kCiThreads) {
      const int m = e / w, j = e % w;
      R[(int64_t)(c0 + m) * n + c0 + j] = Rpp[m][j];
    }
    __syncthreads();
  }
  if (s_bad) {
    for (int64_t e = tid; e < (int64_t)n * n; e += kCiThreads) {
      R[e] = 0.0;
      Rinv[e] = 0.0;
    }
    if (tid == 0) *info = s_bad;
    return;
  }

  // ---------------- inverse X = R^-1, block rows bottom-up:
  // X[P, P] = R_pp^-1;  X[P, rest] = -R_pp^-1 (R[P, rest] X[rest, rest])
  for (int p = np - 1; p >= 0; --p) {
    const int c0 = 32 * p, w = min(32, n - c0), r0 = c0 + w, rest = n - r0;
    const int rest4 = (rest + 3) & ~3;
    for (int e = tid; e < rest4 * 32; e += kCiThreads) {  // SA[k][m] = R[c0 + m][r0 + k]
      const int k = e >> 5, m = e & 31;
      SA[k * kSaLd + m] = (m < w && k < rest) ? ldcg(R + (int64_t)(c0 + m) * n + r0 + k) : 0.0;
    }
    // diagonal block inverse: lane j back-substitutes R_pp x = e_j
    if (wid == 0) {
      double rp[32];  // rp[i] = R_pp[i][lane] (this lane's column)
#pragma unroll
      for (int i = 0; i < 32; ++i)
        rp[i] = (i < w && lane < w) ? ldcg(R + (int64_t)(c0 + i) * n + c0 + lane)
                                    : (i == lane ? 1.0 : 0.0);
      double x[32];
#pragma unroll
      for (int i = 31; i >= 0; --i) {
        double v = (i == lane) ? 1.0 : 0.0;
#pragma unroll
        for (int k = i + 1; k < 32; ++k) v = fma(-__shfl_sync(0xffffffffu, rp[i], k), x[k], v);
        const double rii = __shfl_sync(0xffffffffu, rp[i], i);
        x[i] = (i <= lane) ? v / rii : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) Rpp[i][lane] = x[i];
    }
    __syncthreads();
    if (rest > 0) {
      // Y = R[P, rest] X[rest, rest] into X's own block row (X upper
      // triangular: output column j needs rows k <= j only)
      const int ntile = (rest + 7) / 8;
      for (int jt = wid; jt < ntile; jt += kCiWarps) {
        double acc[4][2] = {};
        const int khi = min(rest4, (8 * jt + 8 + 3) & ~3);
        panel_gemm_tile(SA, Rinv + (int64_t)r0 * n, n, r0 + 8 * jt, n, khi, rest, acc, q, c);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int m = 8 * mt + q, j = 8 * jt + 2 * c + h;
            if (m < w && j < rest) Rinv[(int64_t)(c0 + m) * n + r0 + j] = acc[mt][h];
          }
      }
      __syncthreads();
      // X[P, rest] = -R_pp^-1 Y, one column per thread, in place
      for (int j = tid; j < rest; j += kCiThreads) {
        double* col = Rinv + (int64_t)c0 * n + r0 + j;
        double y[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) y[k] = k < w ? ldcg(col + (int64_t)k * n) : 0.0;
#pragma unroll
        for (int m = 0; m < 32; ++m) {
          double v = 0.0;
#pragma unroll
          for (int k = m; k < 32; ++k) v = fma(Rpp[m][k], y[k], v);
          if (m < w) col[(int64_t)m * n] = -v;
        }
      }
    }
    for (int e = tid; e < w * c0; e += kCiThreads) Rinv[(int64_t)(c0 + e / c0) * n + e % c0] = 0.0;
    for (int e = tid; e < w * w; e += kCiThreads) {
      const int m = e / w, j = e % w;
      Rinv[(int64_t)(c0 + m) * n + c0 + j] = Rpp[m][j];
    }
    __syncthreads();
  }
  if (tid == 0) *info = 0;
}

// Thin Q (r x w, w <= 32) of a tall matrix C by Householder reflections
// (LAPACK geqr2 + org2r conventions), one CTA: C in shared memory column-major,
// warp k owning column k.  Replaces torch.linalg.qr (cuSOLVER geqrf/orgqr,
// ~10 launches) in the r > 128 associated middle step of rsvd_lrls.
__global__ void __launch_bounds__(1024, 1) k_house_q(const double* __restrict__ Cg, int r, int w,
                                                     double* __restrict__ Qg) {
  extern __shared__ __align__(16) double hq[];
  double* C = hq;          // column-major, ld r
  double* Q = C + r * w;   // column-major, ld r
  __shared__ double tau[32];
  const int tid = threadIdx.x, lane = tid & 31, k = tid >> 5;
  for (int e = tid; e < r * w; e += blockDim.x) {
    const int i = e / w, j = e % w;
    C[j * r + i] = Cg[e];
  }
  __syncthreads();
  for (int j = 0; j < w; ++j) {
    if (k == j) {
      double* cj = C + j * r;
      double ss = 0.0;
      for (int i = j + 1 + lane; i < r; i += 32) ss = fma(cj[i], cj[i], ss);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      const double alpha = cj[j];
      double t = 0.0, beta = alpha, scale = 0.0;
      if (ss != 0.0) {
        beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
        t = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      __syncwarp();
      for (int i = j + 1 + lane; i < r; i += 32) cj[i] *= scale;
      if (lane == 0) {
        cj[j] = beta;
        tau[j] = t;
      }
    }
    __syncthreads();
    if (k > j && k < w) {
      const double tj = tau[j];
      const double* v = C + j * r;
      double* ck = C + k * r;
      double d = 0.0;
      for (int i = j + 1 + lane; i < r; i += 32) d = fma(v[i], ck[i], d);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      d = tj * (ck[j] + d);
      __syncwarp();
      if (lane == 0) ck[j] -= d;
      for (int i = j + 1 + lane; i < r; i += 32) ck[i] = fma(-d, v[i], ck[i]);
    }
    __syncthreads();
  }
  if (k < w) {
    double* qk = Q + k * r;
    for (int i = lane; i < r; i += 32) qk[i] = i == k ? 1.0 : 0.0;
    __syncwarp();
    for (int j = k; j >= 0; --j) {
      const double tj = tau[j];
      const double* v = C + j * r;
      double d = 0.0;
      for (int i = j + 1 + lane; i < r; i += 32) d = fma(v[i], qk[i], d);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      d = tj * (qk[j] + d);
      __syncwarp();
      if (lane == 0) qk[j] -= d;
      for (int i = j + 1 + lane; i < r; i += 32) qk[i] = fma(-d, v[i], qk[i]);
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < r * w; e += blockDim.x) {
    const int i = e / w, j = e % w;
    Qg[e] = Q[j * r + i];
  }
}

}  // namespace skx

using namespace skx;

extern "C" int skx_chol_inv_upper(const double* g, int n, double* r, double* rinv, int* info,
                                  void* stream) {
  SKX_REQUIRE(n >= 1 && n <= kCiMaxN, "skx_chol_inv_upper: 1 <= n <= %d", kCiMaxN);
  // the staged panel operand: at most n rows of kSaLd doubles
  const size_t smem = (size_t)((n + 3) & ~3) * kSaLd * 8;
  SKX_REQUIRE(smem <= (size_t)max_smem_optin(), "skx_chol_inv_upper: n = %d needs %zu B of shared memory",
              n, smem);
  cudaFuncSetAttribute(k_chol_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_chol_inv<<<1, kCiThreads, smem, (cudaStream_t)stream>>>(g, n, r, rinv, info);
  return check_launch("k_chol_inv");
}

extern "C" int skx_house_q(const double* c, int r, int w, double* q, void* stream) {
  SKX_REQUIRE(w >= 1 && w <= 32 && w <= r, "skx_house_q: need 1 <= w <= min(r, 32)");
  const size_t smem = (size_t)2 * r * w * 8;
  SKX_REQUIRE(smem <= (size_t)max_smem_optin(), "skx_house_q: %d x %d too large", r, w);
  cudaFuncSetAttribute(k_house_q, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_house_q<<<1, 32 * w, smem, (cudaStream_t)stream>>>(c, r, w, q);
  return check_launch("k_house_q");
}
