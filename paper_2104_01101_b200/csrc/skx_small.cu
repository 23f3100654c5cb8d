// K5 small dense algebra in one CTA each (launch-latency scale problems):
//
//  skx_chol_upper  -- R^T R = G for an SPD n x n Gram (n <= 128); used by the
//                     CholeskyQR2 factorisation of the sketched system Z
//                     (src/linalg.py:103 reduced_qr(z); Householder QR is kept
//                     as the fallback whenever CholeskyQR2 is not safe).
//  skx_jacobi_svd  -- one-sided (Hestenes) Jacobi SVD of an n x n matrix
//                     (n <= 64): A W = U diag(s), singular values descending;
//                     replaces the LAPACK SVD of the small R factors
//                     (src/linalg.py:59 via thin_svd, src/tucker.py:141).
// Fixed iteration order everywhere: deterministic.
#include <math.h>

#include "skx_common.cuh"

namespace skx {

// Right-looking Cholesky in shared memory; row-major upper R output (zero
// lower part).  info = 0 on success, k+1 if the k-th pivot is not positive.
__global__ void __launch_bounds__(512) k_chol(const double* __restrict__ G, int n,
                                              double* __restrict__ R, int* __restrict__ info) {
  extern __shared__ double A[];  // n x ld, row-major, lower part used
  __shared__ int bad;
  const int ld = n | 1;  // odd row stride: column reads A[j*ld + k] hit distinct banks
  for (int q = threadIdx.x; q < n * n; q += blockDim.x) A[(q / n) * ld + q % n] = G[q];
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = 0; k < n; ++k) {
    // every thread reads the pivot after the previous step's barrier; thread 0
    // alone rewrites it, after its own column scaling, so no barrier is needed
    // between the read and the scaling
    const double piv = A[k * ld + k];
    if (!(piv > 0.0)) {  // also catches NaN
      if (threadIdx.x == 0 && !bad) bad = k + 1;
      __syncthreads();
      break;
    }
    const double d = sqrt(piv), inv = 1.0 / d;
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) A[i * ld + k] *= inv;
    __syncthreads();
    if (threadIdx.x == 0) A[k * ld + k] = d;
    // trailing update of the lower triangle: A[i][j] -= A[i][k] A[j][k], k < j <= i
    // (warp per row, lanes along the row: no integer division)
    for (int i = k + 1 + wid; i < n; i += nw) {
      const double lik = A[i * ld + k];
      for (int j = k + 1 + lane; j <= i; j += 32)
        A[i * ld + j] = fma(-lik, A[j * ld + k], A[i * ld + j]);
    }
    __syncthreads();
  }
  for (int q = threadIdx.x; q < n * n; q += blockDim.x) {
    const int i = q / n, j = q % n;
    R[q] = (j >= i && !bad) ? A[j * ld + i] : 0.0;  // R = L^T
  }
  if (threadIdx.x == 0) *info = bad;
}

// Register variant (n <= 128): the lower triangle is split over 1024 threads,
// entry e = t + 1024 q (q < EPT) in column-major packed order, values in
// registers.  Step k reads column k (left unscaled) from a double-buffered
// shared column, updates the owned entries right of it with
// a_ij -= c_i c_j / c_k, and the owners of column k+1 publish it for the next
// step: one barrier per step.  R row k = c / sqrt(c_k) is written as column k
// retires.  Same arithmetic as the textbook right-looking algorithm.
constexpr int kCholThreads = 1024;
constexpr int kCholEpt = 9;  // ceil(128 * 129 / 2 / 1024)

__global__ void __launch_bounds__(kCholThreads) k_chol_reg(const double* __restrict__ G, int n,
                                                           double* __restrict__ R,
                                                           int* __restrict__ info) {
  __shared__ double col[2][128];
  const int t = threadIdx.x;
  const int E = n * (n + 1) / 2;
  double a[kCholEpt];
  int ij[kCholEpt];  // i | j << 16
#pragma unroll
  for (int q = 0; q < kCholEpt; ++q) {
    const int e = t + kCholThreads * q;
    int i = 0, j = 0;
    if (e < E) {
      // column-major packed lower triangle: column j holds rows j..n-1, starts
      // at s_j = j n - j (j - 1) / 2
      j = (int)((2.0 * n + 1.0 - sqrt((2.0 * n + 1.0) * (2.0 * n + 1.0) - 8.0 * e)) * 0.5);
      while (j > 0 && j * n - j * (j - 1) / 2 > e) --j;
      while ((j + 1) * n - (j + 1) * j / 2 <= e) ++j;
      i = j + (e - (j * n - j * (j - 1) / 2));
      a[q] = G[(int64_t)i * n + j];
    } else {
      j = n;  // never active
      a[q] = 0.0;
    }
    ij[q] = i | (j << 16);
  }
  for (int q = t; q < n * n; q += kCholThreads) R[q] = 0.0;  // lower part stays zero
#pragma unroll
  for (int q = 0; q < kCholEpt; ++q)
    if ((ij[q] >> 16) == 0) col[0][ij[q] & 0xffff] = a[q];
  __syncthreads();
  int bad = 0;
  for (int k = 0; k < n; ++k) {
    const double* ck = col[k & 1];
    double* cn = col[(k + 1) & 1];
    const double piv = ck[k];
    if (!(piv > 0.0)) {  // uniform: every thread reads the same pivot
      bad = k + 1;
      break;
    }
    const double rp = 1.0 / piv, sq = sqrt(piv), rs = 1.0 / sq;
#pragma unroll
    for (int q = 0; q < kCholEpt; ++q) {
      const int i = ij[q] & 0xffff, j = ij[q] >> 16;
      if (j == k) {
        R[(int64_t)k * n + i] = i == k ? sq : a[q] * rs;
      } else if (j > k && j < n) {
        a[q] = fma(-ck[i] * ck[j], rp, a[q]);
        if (j == k + 1) cn[i] = a[q];
      }
    }
    __syncthreads();
  }
  if (bad) {
    for (int q = t; q < n * n; q += kCholThreads) R[q] = 0.0;
  }
  if (t == 0) *info = bad;
}

// 1/x from the MUFU approximation plus two Newton steps (~1 ulp), about half
// the latency of an IEEE double division on B200 (measured 114 cycles)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  return fma(r, fma(-x, r, 1.0), r);
}

// One-sided Jacobi: columns of A (n x n, shared, column-major) are rotated
// pairwise (round-robin tournament, n/2 disjoint pairs per step, one warp per
// pair) until every pair is orthogonal to eps relative; W accumulates the
// rotations.  s_j = ||a_j||, u_j = a_j / s_j, sorted descending.
__global__ void __launch_bounds__(1024, 1) k_jacobi(const double* __restrict__ Ain, int n, int rs,
                                                int cs, double* __restrict__ U,
                                                double* __restrict__ S,
                                                double* __restrict__ V) {
  extern __shared__ double sm[];
  const int np = n + (n & 1);  // even number of slots (a zero column when n is odd)
  double* A = sm;             // np columns of length n (column-major, ld = n)
  double* W = A + np * n;     // np x np rotations (column-major, ld = np)
  __shared__ int changed;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int q = threadIdx.x; q < np * n; q += blockDim.x) {
    const int j = q / n, i = q % n;
    A[q] = j < n ? Ain[i * rs + j * cs] : 0.0;
  }
  for (int q = threadIdx.x; q < np * np; q += blockDim.x) W[q] = (q / np == q % np) ? 1.0 : 0.0;
  __syncthreads();
  // round-robin (circle method): slot 0 holds column 0, slot j >= 1 holds
  // column 1 + (j - 1 + step) mod (np - 1); pairs are (slot k, slot np-1-k)
  const int nm1 = np - 1;
  const double eps = 2.220446049250313e-16;
  // rotate while |cos(a_p, a_q)| > 2 n eps: above the rounding noise of the
  // length-n dot products (a tighter threshold keeps rotating on noise and
  // runs to the sweep cap), far below what the 1e-10 parity needs
  const double tol = 2.0 * n * eps, tol2 = tol * tol;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) changed = 0;
    __syncthreads();
    for (int step = 0; step < np - 1; ++step) {
      for (int pr = wid; pr < np / 2; pr += nw) {
        // slot j >= 1 holds column 1 + (j - 1 + step) mod (np - 1); both
        // arguments are < 2 (np - 1): one conditional subtraction each
        int vp = pr - 1 + step, vq = np - 2 - pr + step;
        if (vp >= nm1) vp -= nm1;
        if (vq >= nm1) vq -= nm1;
        int p = pr == 0 ? 0 : 1 + vp;
        int q = 1 + vq;  // slot np-1-pr >= 1
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        double* ap = A + p * n;
        double* aq = A + q * n;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < n; i += 32) {
          al = fma(ap[i], ap[i], al);
          be = fma(aq[i], aq[i], be);
          ga = fma(ap[i], aq[i], ga);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        // dgesvj-style threshold: rotations below sqrt(n) * eps relative are
        // rounding noise of the dot product itself and would never settle
        // (squared test: no square root on the common no-rotation path)
        if (ga * ga > tol2 * (al * be) && ga != 0.0) {
          // the rotation only needs c^2 + s^2 = 1 to working accuracy (t's own
          // rounding merely perturbs convergence): Newton-refined reciprocals
          // instead of IEEE divisions
          const double zeta = (be - al) * (0.5 * rcp_nr(ga));
          const double t = copysign(rcp_nr(fabs(zeta) + sqrt(fma(zeta, zeta, 1.0))), zeta);
          const double c = rsqrt(fma(t, t, 1.0)), s = c * t;
          for (int i = lane; i < n; i += 32) {
            const double x = ap[i], y = aq[i];
            ap[i] = c * x - s * y;
            aq[i] = s * x + c * y;
          }
          double* wp = W + p * np;
          double* wq = W + q * np;
          for (int i = lane; i < np; i += 32) {
            const double x = wp[i], y = wq[i];
            wp[i] = c * x - s * y;
            wq[i] = s * x + c * y;
          }
          if (lane == 0) changed = 1;
        }
      }
      __syncthreads();
    }
    const int any = changed;
    __syncthreads();  // everyone has read `changed` before thread 0 resets it
    if (!any) break;
  }
  // singular values and descending order (n <= 112: one thread sorts)
  __shared__ double sv[112];
  __shared__ int ord[112];
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double s2 = 0.0;
    for (int i = 0; i < n; ++i) s2 = fma(A[j * n + i], A[j * n + i], s2);
    sv[j] = sqrt(s2);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 0; j < n; ++j) ord[j] = j;
    for (int a = 0; a < n; ++a)
      for (int b = a + 1; b < n; ++b)
        if (sv[ord[b]] > sv[ord[a]]) {
          const int t = ord[a];
          ord[a] = ord[b];
          ord[b] = t;
        }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < n * n; q += blockDim.x) {
    const int i = q / n, k = q % n;  // row i, output column k (row-major outputs)
    const int j = ord[k];
    const double s = sv[j];
    U[q] = s > 0.0 ? A[j * n + i] / s : (i == k ? 1.0 : 0.0);
    V[q] = W[j * np + i];
  }
  for (int k = threadIdx.x; k < n; k += blockDim.x) S[k] = sv[ord[k]];
}

// Middle of Algorithm 5 (rsvd_lrls, src/linalg.py:87-113) for the associated
// form used when the test width w < r:  C = R^-1 B (B = Q_z^T Y G, r x w),
// C = Q T (Householder, as LAPACK geqr2/org2r), X = R^-T Q.  One CTA of w
// warps, warp k owning column k: the triangular solves need only warp syncs;
// R sits in shared memory with an odd leading dimension so that both its
// row and its column walks are bank-conflict free.  Replaces two cuBLAS
// TRSMs and a ~25-launch cuSOLVER QR.
__global__ void __launch_bounds__(1024, 1) k_lrls_mid(const double* __restrict__ Rg,
                                                     const double* __restrict__ Bg, int r, int w,
                                                     double* __restrict__ Qg,
                                                     double* __restrict__ Xg) {
  extern __shared__ double sm[];
  const int ld = r | 1;
  double* R = sm;             // r x r upper, row-major, ld odd
  double* C = R + r * ld;     // column-major, ld r
  double* Q = C + r * w;      // column-major, ld r
  double* tau = Q + r * w;    // w
  double* rinv = tau + w;     // 1 / R_ii
  const int tid = threadIdx.x, lane = tid & 31, k = tid >> 5;
  for (int i = k; i < r; i += blockDim.x >> 5)
    for (int j = lane; j < r; j += 32) R[i * ld + j] = Rg[(int64_t)i * r + j];
  for (int i = tid; i < r; i += blockDim.x) rinv[i] = 1.0 / Rg[(int64_t)i * r + i];
  for (int i = lane; i < r; i += 32) C[k * r + i] = Bg[(int64_t)i * w + k];
  __syncthreads();
  // 1. back substitution, warp k on column k held in registers (lane l owns
  //    rows l, l + 32, ...): C <- R^-1 C
  constexpr int kSl = 4;  // r <= 128
  {
    double* ck = C + k * r;
    double c[kSl];
#pragma unroll
    for (int t = 0; t < kSl; ++t) c[t] = lane + 32 * t < r ? ck[lane + 32 * t] : 0.0;
    // row i = 32 ti + ii lives in register slot ti (static after unrolling)
#pragma unroll
    for (int ti = kSl - 1; ti >= 0; --ti) {
      for (int ii = 31; ii >= 0; --ii) {
        const int i = 32 * ti + ii;
        if (i >= r) continue;
        const double xi = __shfl_sync(0xffffffffu, c[ti], ii) * rinv[i];
#pragma unroll
        for (int t = 0; t <= ti; ++t) {
          const int l = lane + 32 * t;
          const double upd = fma(-R[min(l, r - 1) * ld + i], xi, c[t]);
          c[t] = l < i ? upd : (l == i ? xi : c[t]);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < kSl; ++t)
      if (lane + 32 * t < r) ck[lane + 32 * t] = c[t];
  }
  __syncthreads();
  // 2. Householder QR of C: v_j = [1; C[j+1:, j]], H_j = I - tau_j v v^T
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
    if (k > j) {
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
  // 3. thin Q = H_0 ... H_{w-1} [I_w; 0], warp k on column k
  {
    double* qk = Q + k * r;
    for (int i = lane; i < r; i += 32) qk[i] = i == k ? 1.0 : 0.0;
    __syncwarp();
    for (int j = k; j >= 0; --j) {  // H_j leaves column k untouched for j > k
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
    for (int i = lane; i < r; i += 32) Qg[(int64_t)i * w + k] = qk[i];
    __syncwarp();
    // 4. X = R^-T Q: forward substitution with L = R^T (L[l][i] = R[i][l]),
    //    column in registers as in step 1
    double c[kSl];
#pragma unroll
    for (int t = 0; t < kSl; ++t) c[t] = lane + 32 * t < r ? qk[lane + 32 * t] : 0.0;
#pragma unroll
    for (int ti = 0; ti < kSl; ++ti) {
      for (int ii = 0; ii < 32; ++ii) {
        const int i = 32 * ti + ii;
        if (i >= r) break;
        const double xi = __shfl_sync(0xffffffffu, c[ti], ii) * rinv[i];
#pragma unroll
        for (int t = ti; t < kSl; ++t) {
          const int l = lane + 32 * t;
          const double upd = fma(-R[i * ld + min(l, r - 1)], xi, c[t]);
          c[t] = (l > i && l < r) ? upd : (l == i ? xi : c[t]);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < kSl; ++t)
      if (lane + 32 * t < r) qk[lane + 32 * t] = c[t];
    __syncwarp();
    for (int i = lane; i < r; i += 32) Xg[(int64_t)i * w + k] = qk[i];
  }
}

// Decision flags of the Cholesky QR of the sketched system (src/linalg.py:44-52
// rank test plus the orthogonality check), in one CTA instead of ~20 small
// tensor kernels: out[0] = unsafe (Cholesky failed, or diag(R) not finite or
// spanning >= 1e6), out[1] = one pass suffices (max |Q^T Q - I| < 1e-13),
// out[2] = rank-deficient (some |R_ii| < 1e-12 ||Z||_F), out[3] = the
// speculative sweep must be replayed (out[0] | !out[1] | out[2]).  NaNs count
// as failures, as the comparisons in torch do.
__global__ void __launch_bounds__(512) k_cholqr_flags(const double* __restrict__ g1,
                                                      const double* __restrict__ r1,
                                                      const int* __restrict__ info,
                                                      const double* __restrict__ g2, int r,
                                                      int* __restrict__ out) {
  __shared__ double s_max[32], s_min[32], s_tr[32], s_dev[32];
  __shared__ int s_nan[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double dmax = -INFINITY, dmin = INFINITY, tr = 0.0, dev = 0.0;
  int nan = 0;
  for (int i = tid; i < r; i += blockDim.x) {
    const double d = r1[(int64_t)i * r + i];
    if (d != d) nan = 1;
    dmax = fmax(dmax, d);
    dmin = fmin(dmin, d);
    tr += g1[(int64_t)i * r + i];
  }
  for (int i = wid; i < r; i += blockDim.x >> 5) {  // warp per row, lanes along it
    const double* row = g2 + (int64_t)i * r;
    for (int j = lane; j < r; j += 32) {
      const double e = fabs(row[j] - (i == j ? 1.0 : 0.0));
      if (e != e) nan |= 2;
      dev = fmax(dev, e);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
    tr += __shfl_xor_sync(0xffffffffu, tr, o);
    dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
    nan |= __shfl_xor_sync(0xffffffffu, nan, o);
  }
  if (lane == 0) {
    s_max[wid] = dmax;
    s_min[wid] = dmin;
    s_tr[wid] = tr;
    s_dev[wid] = dev;
    s_nan[wid] = nan;
  }
  __syncthreads();
  if (tid == 0) {
    const int nw = blockDim.x >> 5;
    double a = -INFINITY, b = INFINITY, t = 0.0, dv = 0.0;
    int nn = 0;
    for (int w = 0; w < nw; ++w) {
      a = fmax(a, s_max[w]);
      b = fmin(b, s_min[w]);
      t += s_tr[w];
      dv = fmax(dv, s_dev[w]);
      nn |= s_nan[w];
    }
    const double tol = 1e-12 * sqrt(t);
    int bad = (t != t) ? 1 : 0;
    for (int i = 0; i < r && !bad; ++i) bad = fabs(r1[(int64_t)i * r + i]) < tol;
    const int unsafe = info[0] != 0 || (nn & 1) || !(a < 1e6 * b);
    const int one = !(nn & 2) && dv < 1e-13;
    out[0] = unsafe;
    out[1] = one;
    out[2] = bad;
    out[3] = unsafe || !one || bad;
  }
}

}  // namespace skx

using namespace skx;

extern "C" int skx_chol_upper(const double* g, int n, double* r, int* info, void* stream) {
  SKX_REQUIRE(n >= 1 && n <= 128, "skx_chol_upper: 1 <= n <= 128");
  k_chol_reg<<<1, kCholThreads, 0, (cudaStream_t)stream>>>(g, n, r, info);
  return check_launch("k_chol_reg");
}

extern "C" int skx_jacobi_svd(const double* a, int n, int64_t rs, int64_t cs, double* u,
                              double* s, double* v, void* stream) {
  SKX_REQUIRE(n >= 1 && n <= 112, "skx_jacobi_svd: 1 <= n <= 112");
  const int np = n + (n & 1);
  const size_t smem = (size_t)(np * n + np * np) * 8 + (size_t)np * 4 + 16;
  cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // one warp per column pair of a round-robin step
  k_jacobi<<<1, 32 * (np / 2 > 16 ? 32 : np / 2 < 1 ? 1 : np / 2), smem, (cudaStream_t)stream>>>(
      a, n, (int)rs, (int)cs, u, s, v);
  return check_launch("k_jacobi");
}

extern "C" int skx_lrls_mid(const double* rz, const double* b, int r, int w, double* q,
                            double* x, void* stream) {
  SKX_REQUIRE(r >= 1 && w >= 1 && w <= r && r <= 128 && w <= 32,
              "skx_lrls_mid: need 1 <= w <= min(r, 32), r <= 128");
  const size_t smem = ((size_t)r * (r | 1) + 2 * (size_t)r * w + w + r) * 8;
  cudaFuncSetAttribute(k_lrls_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_lrls_mid<<<1, 32 * w, smem, (cudaStream_t)stream>>>(rz, b, r, w, q, x);
  return check_launch("k_lrls_mid");
}

extern "C" int skx_cholqr_flags(const double* g1, const double* r1, const int* info,
                                const double* g2, int r, int* out, void* stream) {
  SKX_REQUIRE(r >= 1, "skx_cholqr_flags: empty system");
  k_cholqr_flags<<<1, r > 128 ? 512 : 256, 0, (cudaStream_t)stream>>>(g1, r1, info, g2, r, out);
  return check_launch("k_cholqr_flags");
}
