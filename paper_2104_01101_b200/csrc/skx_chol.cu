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
#include <cooperative_groups.h>
#include <math.h>
#include <stdlib.h>

#include "skx_common.cuh"

namespace skx {

namespace {

// 8 warps x 128 registers = 32K registers: the CTA fits beside one CTA of
// the fitness kernel it runs next to in the sweep pipeline (a 64K-register CTA
// has to wait until a whole SM drains)
constexpr int kCiThreads = 256;
constexpr int kCiWarps = kCiThreads / 32;
constexpr int kCiEpt = (528 + kCiThreads - 1) / kCiThreads;
constexpr int kCiMaxN = 512;
// above this order the cooperative multi-CTA form runs (kCiCoopCtas CTAs);
// up to it one CTA, which starts beside the fitness kernel of a leverage
// sweep without waiting for a whole grid's worth of free SMs (config 5: r = 400)
constexpr int kCiCoopMinN = 400;
constexpr int kCiCoopCtas = 24;
constexpr int kCiTiles = 4;  // 8 x 8 output tiles per warp step (their C loads in flight together)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Plain (coherent) global load: R and R^-1 are written earlier in the same
// kernel by other warps of this CTA, so the non-coherent __ldg path is unsafe.
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

}  // namespace

// Leading dimension (doubles) of a shared [32][*] operand block holding
// `cols` columns: >= cols and = 4 mod 16, so that the m8n8k4 fragment reads
// (lane (q, c) -> row c, column q) of a half-warp hit 16 distinct 8-byte banks.
// (cols is first rounded up to whole 8-column tiles and to the 32-wide diagonal
// block, which every panel touches)
__host__ __device__ __forceinline__ int ci_ld(int cols) {
  const int x = 8 * ((max(cols, 32) + 7) / 8);
  return x + (x % 16 == 0 ? 4 : 12);
}

// The 528 entries (i, j), i <= j, of a 32 x 32 upper triangle, kCiEpt per
// thread of the CTA (e = t, t + kCiThreads, ...): the diagonal-block steps
// below touch one entry per thread per step, with one barrier per step.
__device__ __forceinline__ void ut_entry(int e, int& i, int& j) {
  // row i holds 32 - i entries, starting at e_i = 32 i - i (i - 1) / 2
  i = 0;
  while (i < 31 && 32 * (i + 1) - (i + 1) * i / 2 <= e) ++i;
  j = i + (e - (32 * i - i * (i - 1) / 2));
}

// Factor the SPD 32 x 32 block D (shared, leading dim ld; upper triangle
// read) in place into upper R (R^T R = D) -- right-looking with the unscaled
// update a_ij -= a_ki a_kj / a_kk, rows scaled at the end -- then X = R^-1
// into Xo (leading dim 36) using V (36) as scratch.  Returns 0 or k+1 for the
// first failing pivot.  All threads of the CTA call it.
__device__ int cta_chol_inv32(double* D, int ld, double* V, double* Xo, int tid) {
  int ei[kCiEpt], ej[kCiEpt];
  bool own[kCiEpt];
#pragma unroll
  for (int u = 0; u < kCiEpt; ++u) {
    const int e = tid + u * kCiThreads;
    own[u] = e < 528;
    ut_entry(own[u] ? e : 0, ei[u], ej[u]);
  }
  int bad = 0;
  for (int k = 0; k < 32; ++k) {
    const double akk = D[k * ld + k];
    if (!(akk > 0.0)) {  // uniform (every thread reads the same pivot); NaN fails too
      bad = k + 1;
      break;
    }
    const double rp = 1.0 / akk;
#pragma unroll
    for (int u = 0; u < kCiEpt; ++u)
      if (own[u] && ei[u] > k)
        D[ei[u] * ld + ej[u]] = fma(-D[k * ld + ei[u]] * D[k * ld + ej[u]], rp, D[ei[u] * ld + ej[u]]);
    __syncthreads();
  }
  if (bad) return bad;
  // row k of R = row k / sqrt(a_kk); V = I
  double rv[kCiEpt];
#pragma unroll
  for (int u = 0; u < kCiEpt; ++u)
    rv[u] = own[u] ? D[ei[u] * ld + ej[u]] / sqrt(D[ei[u] * ld + ei[u]]) : 0.0;
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kCiEpt; ++u)
    if (own[u]) {
      const int i = ei[u], j = ej[u];
      V[i * 36 + j] = i == j ? 1.0 : 0.0;
      if (i != j) V[j * 36 + i] = 0.0;
      Xo[j * 36 + i] = 0.0;  // lower part of the inverse (diagonal rewritten below)
      D[i * ld + j] = rv[u];
    }
  __syncthreads();
  // back substitution for all columns at once: step i finalises row i of X and
  // removes it from the rows above
  for (int i = 31; i >= 0; --i) {
    const double rii = D[i * ld + i];
#pragma unroll
    for (int u = 0; u < kCiEpt; ++u)
      if (own[u]) {
        const int k = ei[u], j = ej[u];
        if (j < i) continue;
        const double xij = V[i * 36 + j] / rii;
        if (k == i) Xo[i * 36 + j] = xij;
        else if (k < i) V[k * 36 + j] = fma(-D[k * ld + i], xij, V[k * 36 + j]);
      }
    __syncthreads();
  }
  return 0;
}

// G: n x n SPD (row-major, symmetric; the upper triangle is read).  R, Rinv:
// n x n row-major outputs (upper; zero below the diagonal).  info: 0, or k+1
// for the first non-positive (or NaN) pivot k -- R and Rinv are then zero.
//
// Right-looking blocked algorithms with 32-row panels, every GEMM operand in
// shared memory (m8n8k4 FP64 tensor-core tiles, 8 x 8 outputs per warp item,
// C tiles read and written once per panel in L2):
//  Cholesky, panel p (rows P = [c0, c0 + 32) of R):  the block row of the
//   trailing matrix (kept in R's own rows) -> shared; warp 0 factors the
//   diagonal block and inverts it; the rest of the row is R_pp^-T times it (a
//   32 x 32 x (n - c0 - 32) tile GEMM); the trailing upper triangle is
//   updated A[i][j] -= sum_k R[c0+k][i] R[c0+k][j].
//  Inverse X = R^-1, block rows bottom-up: W[Q] = I_Q + (the updates already
//   subtracted), X[Q] = R_qq^-1 W[Q]; then every block row above takes its
//   rank-32 update W[0:c0, c0:] -= R[0:c0, Q] X[Q, c0:].
//
// COOP: the same algorithm on a cooperative grid of several CTAs -- every CTA
// forms the (small) block row itself, identically, and the O(n^3) tile
// updates are split over all warps of all CTAs, one grid barrier per panel;
// CTA 0 writes the block rows.  For large r with the GPU to itself (config 3,
// r = 512): one CTA is FP64-compute bound on a single SM there.
template <bool COOP>
__global__ void __launch_bounds__(kCiThreads, 2) k_chol_inv(const double* __restrict__ G, int n,
                                                           double* R, double* Rinv,
                                                           int* __restrict__ info) {
  extern __shared__ __align__(16) double cism[];
  __shared__ double Dinv[32][36];  // R_pp^-1 of the current panel
  __shared__ double Vs[32 * 36];     // scratch of the diagonal-block inverse
  __shared__ int s_bad;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, q = lane >> 2, c = lane & 3;
  const int np = (n + 31) / 32;
  const bool lead = !COOP || blockIdx.x == 0;  // writes the block rows
  const int gwid = COOP ? blockIdx.x * kCiWarps + wid : wid;
  const int gwarps = COOP ? gridDim.x * kCiWarps : kCiWarps;
  auto grid_sync = [&]() {
    if (COOP) cooperative_groups::this_grid().sync();
    else __syncthreads();
  };
  if (tid == 0) s_bad = 0;
  // the trailing matrix lives in R's own rows; panel 0 reads G directly
  __syncthreads();

  // ---------------- Cholesky
  for (int p = 0; p < np; ++p) {
    const int c0 = 32 * p, w = min(32, n - c0), nc = n - c0, ld = ci_ld(nc);
    double* BR = cism;  // [32][ld]: block row, columns c0 .. n-1 (zero beyond)
    const double* src = p == 0 ? G : R;  // first touch of the trailing matrix: G
    for (int k = wid; k < 32; k += kCiWarps)
      for (int j = lane; j < ld; j += 32)
        BR[k * ld + j] = (k < w && j < nc && j >= k) ? ldcg(src + (int64_t)(c0 + k) * n + c0 + j) : 0.0;
    __syncthreads();
    // partial last panel: identity beyond w in the diagonal block
    for (int k = w + tid; k < 32; k += kCiThreads) BR[k * ld + k] = 1.0;
    __syncthreads();
    {
      const int bad = cta_chol_inv32(BR, ld, Vs, &Dinv[0][0], tid);
      if (bad && tid == 0) s_bad = c0 + bad;
    }
    // zero the padding rows of R_pp again (identity beyond w)
    for (int e = tid; e < 32 * 32; e += kCiThreads) {
      const int i = e >> 5, j = e & 31;
      if (i >= w || j >= w || j < i) BR[i * ld + j] = 0.0;
    }
    __syncthreads();
    if (s_bad) break;
    // rest of the block row: R[P][c0+32+j] = (R_pp^-T B)[.][j], column tiles in place
    const int rest = max(nc - 32, 0), rt = (rest + 7) / 8;
    for (int jt = wid; jt < rt; jt += kCiWarps) {
      double acc[4][2] = {};
      const int j0 = 32 + 8 * jt;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const double b = BR[(4 * ks + c) * ld + j0 + q];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) dmma(acc[mt][0], acc[mt][1], Dinv[4 * ks + c][8 * mt + q], b);
      }
      __syncwarp();
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        BR[(8 * mt + q) * ld + j0 + 2 * c] = acc[mt][0];
        BR[(8 * mt + q) * ld + j0 + 2 * c + 1] = acc[mt][1];
      }
    }
    __syncthreads();
    // trailing update of the upper triangle: rows / cols r0.., 8 x 8 tiles;
    // warp per tile row (its A fragments in registers), four tiles in flight
    const int r0 = c0 + 32;
    for (int ti = gwid; ti < rt; ti += gwarps) {
      double a[8];
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) a[ks] = -BR[(4 * ks + c) * ld + 32 + 8 * ti + q];
      const int i = 8 * ti + q;
      for (int tj = ti; tj < rt; tj += kCiTiles) {
        double acc[kCiTiles][2];
#pragma unroll
        for (int v = 0; v < kCiTiles; ++v)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = 8 * (tj + v) + 2 * c + h;
            acc[v][h] = (tj + v < rt && i < rest && j < rest)
                            ? ldcg(src + (int64_t)(r0 + i) * n + r0 + j) : 0.0;
          }
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
#pragma unroll
          for (int v = 0; v < kCiTiles; ++v) {
            const double b = tj + v < rt ? BR[(4 * ks + c) * ld + 32 + 8 * (tj + v) + q] : 0.0;
            dmma(acc[v][0], acc[v][1], a[ks], b);
          }
#pragma unroll
        for (int v = 0; v < kCiTiles; ++v)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = 8 * (tj + v) + 2 * c + h;
            if (tj + v < rt && i < rest && j < rest) R[(int64_t)(r0 + i) * n + r0 + j] = acc[v][h];
          }
      }
    }
    grid_sync();
    // the final block row and R_pp^-1 to global only now: with COOP, slower
    // CTAs may read these rows' trailing values until the barrier above
    if (lead) {
      for (int i = wid; i < w; i += kCiWarps)
        if (lane < w) Rinv[(int64_t)(c0 + i) * n + c0 + lane] = Dinv[i][lane];
      for (int k = wid; k < w; k += kCiWarps)
        for (int j = lane; j < n; j += 32) R[(int64_t)(c0 + k) * n + j] = j < c0 ? 0.0 : BR[k * ld + j - c0];
    }
    __syncthreads();  // BR and Dinv are overwritten by the next panel
  }
  grid_sync();
  if (s_bad) {  // (every CTA saw the same pivot)
    if (lead) {
      for (int64_t e = tid; e < (int64_t)n * n; e += kCiThreads) {
        R[e] = 0.0;
        Rinv[e] = 0.0;
      }
      if (tid == 0) *info = s_bad;
    }
    return;
  }

  // ---------------- inverse, block rows bottom-up
  for (int Q = np - 1; Q >= 0; --Q) {
    const int c0 = 32 * Q, w = min(32, n - c0), nq = n - c0, ld = ci_ld(nq);
    double* BX = cism;             // [32][ld]: W then X block row, columns c0 ..
    double* RC = cism + 32 * ld;   // [c0][36]: R[m][c0 + k]
    // W[Q] = I_Q beside the updates accumulated in Rinv's block row (the
    // bottom block row has none)
    for (int k = wid; k < 32; k += kCiWarps)
      for (int j = lane; j < ld; j += 32) {
        double v = 0.0;
        if (k < w && j < nq)
          v = j < 32 ? (j == k ? 1.0 : 0.0) : ldcg(Rinv + (int64_t)(c0 + k) * n + c0 + j);
        BX[k * ld + j] = v;
      }
    for (int i = wid; i < 32; i += kCiWarps)
      Dinv[i][lane] = (i < w && lane < w) ? ldcg(Rinv + (int64_t)(c0 + i) * n + c0 + lane) : 0.0;
    for (int m = wid; m < c0; m += kCiWarps)
      RC[m * 36 + lane] = lane < w ? ldcg(R + (int64_t)m * n + c0 + lane) : 0.0;
    __syncthreads();
    // X[Q] = R_qq^-1 W[Q], column tiles in place
    const int nt = (nq + 7) / 8;
    for (int jt = wid; jt < nt; jt += kCiWarps) {
      double acc[4][2] = {};
      const int j0 = 8 * jt;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const double b = BX[(4 * ks + c) * ld + j0 + q];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) dmma(acc[mt][0], acc[mt][1], Dinv[8 * mt + q][4 * ks + c], b);
      }
      __syncwarp();
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        BX[(8 * mt + q) * ld + j0 + 2 * c] = acc[mt][0];
        BX[(8 * mt + q) * ld + j0 + 2 * c + 1] = acc[mt][1];
      }
    }
    __syncthreads();

    // W[0:c0, c0:] -= R[0:c0, Q] X[Q, c0:]: warp per tile row, four tiles in flight
    const int mtile = c0 / 8;
    for (int ti = gwid; ti < mtile; ti += gwarps) {
      double a[8];
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) a[ks] = -RC[(8 * ti + q) * 36 + 4 * ks + c];
      const int i = 8 * ti + q;
      for (int tj = 0; tj < nt; tj += kCiTiles) {
        double acc[kCiTiles][2];
#pragma unroll
        for (int v = 0; v < kCiTiles; ++v)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = 8 * (tj + v) + 2 * c + h;
            // first touch (the block's own 32 columns): the update starts from 0
            acc[v][h] = (tj + v < nt && j < nq && j >= 32) ? ldcg(Rinv + (int64_t)i * n + c0 + j) : 0.0;
          }
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
#pragma unroll
          for (int v = 0; v < kCiTiles; ++v) {
            const double b = tj + v < nt ? BX[(4 * ks + c) * ld + 8 * (tj + v) + q] : 0.0;
            dmma(acc[v][0], acc[v][1], a[ks], b);
          }
#pragma unroll
        for (int v = 0; v < kCiTiles; ++v)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = 8 * (tj + v) + 2 * c + h;
            if (tj + v < nt && j < nq) Rinv[(int64_t)i * n + c0 + j] = acc[v][h];
          }
      }
    }
    grid_sync();
    // X's block row replaces W's only now (slower CTAs may still be reading W)
    if (lead)
      for (int k = wid; k < w; k += kCiWarps)
        for (int j = lane; j < n; j += 32) Rinv[(int64_t)(c0 + k) * n + j] = j < c0 ? 0.0 : BX[k * ld + j - c0];
    __syncthreads();  // BX is overwritten by the next step
  }
  if (lead && tid == 0) *info = 0;
}

// Thin Q (r x w, w <= 32) of a tall matrix C by Householder reflections
// (LAPACK geqr2 + org2r conventions), one CTA: C in shared memory column-major,
// warp k owning column k.  Replaces torch.linalg.qr (cuSOLVER geqrf/orgqr,
// ~10 launches) in the r > 128 associated middle step of rsvd_lrls.
__global__ void __launch_bounds__(512) k_house_q(const double* __restrict__ Cg, int r, int w,
                                                     double* __restrict__ Qg) {
  extern __shared__ __align__(16) double hq[];
  double* C = hq;          // column-major, ld r
  double* Q = C + r * w;   // column-major, ld r
  __shared__ double tau[32];
  const int tid = threadIdx.x, lane = tid & 31, wk = tid >> 5, nwk = blockDim.x >> 5;
  for (int e = tid; e < r * w; e += blockDim.x) {
    const int i = e / w, j = e % w;
    C[j * r + i] = Cg[e];
  }
  __syncthreads();
  for (int j = 0; j < w; ++j) {
    if (wk == j % nwk) {
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
    for (int k = wk; k < w; k += nwk) {
      if (k <= j) continue;
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
      __syncwarp();
    }
    __syncthreads();
  }
  for (int k = wk; k < w; k += nwk) {
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
  // Cholesky: a 32-row block row; inverse: that plus the 32-column block of R
  size_t smem = (size_t)32 * ci_ld(n) * 8;
  for (int c0 = 0; c0 < n; c0 += 32) smem = std::max(smem, (size_t)(32 * ci_ld(n - c0) + 36 * c0) * 8);
  SKX_REQUIRE(smem <= (size_t)max_smem_optin(), "skx_chol_inv_upper: n = %d needs %zu B of shared memory",
              n, smem);
  if (n > kCiCoopMinN && getenv("SKX_CHOL_ONE_CTA") == nullptr) {
    // cooperative grid: every CTA resident at once (one per SM at this smem)
    cudaFuncSetAttribute(k_chol_inv<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chol_inv<true>, kCiThreads, smem);
    const int grid = (int)imin(kCiCoopCtas, (int64_t)imax(per_sm, 0) * num_sms());
    if (grid >= 2) {
      void* args[] = {(void*)&g, (void*)&n, (void*)&r, (void*)&rinv, (void*)&info};
      if (cudaLaunchCooperativeKernel((const void*)k_chol_inv<true>, dim3(grid), dim3(kCiThreads),
                                      args, smem, (cudaStream_t)stream) == cudaSuccess)
        return check_launch("k_chol_inv<coop>");
      cudaGetLastError();  // fall back to one CTA
    }
  }
  cudaFuncSetAttribute(k_chol_inv<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_chol_inv<false><<<1, kCiThreads, smem, (cudaStream_t)stream>>>(g, n, r, rinv, info);
  return check_launch("k_chol_inv");
}

extern "C" int skx_house_q(const double* c, int r, int w, double* q, void* stream) {
  SKX_REQUIRE(w >= 1 && w <= 32 && w <= r, "skx_house_q: need 1 <= w <= min(r, 32)");
  const size_t smem = (size_t)2 * r * w * 8;
  SKX_REQUIRE(smem <= (size_t)max_smem_optin(), "skx_house_q: %d x %d too large", r, w);
  cudaFuncSetAttribute(k_house_q, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // at most 16 warps (warp k owns columns k, k + 16): 512 x 61 registers, so the
  // CTA fits beside one CTA of the fitness kernel
  k_house_q<<<1, 32 * (w < 16 ? w : 16), smem, (cudaStream_t)stream>>>(c, r, w, q);
  return check_launch("k_house_q");
}
