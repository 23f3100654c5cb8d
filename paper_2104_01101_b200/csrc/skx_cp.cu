// K8: CP-ALS on a small dense order-3 core in ONE CTA -- the whole second
// stage of Algorithm 6 (src/cp.py:177-224 -> cp_als(core, on_core=True),
// src/cp.py:119-174): hosvd-of-core initialisation (leading eigenvectors of
// the unfolding Grams, src/tucker.py:112-126), then per sweep and mode the
// Hadamard product of the other Grams, the core MTTKRP, pinv(rcond=1e-12)
// by a symmetric eigendecomposition, the sub-problem residual
// (src/cp.py:96-99), column normalisation into weights, the new Gram, and
// the CP fitness of the core after every sweep (src/tensors.py:339-368).
//
// Everything lives in shared memory (core 20^3 = 64 KB at config 5).  The
// symmetric eigenproblems (s_n x s_n for the init, R x R for every pinv) run
// as a parallel cyclic Jacobi: per step the n/2 disjoint rotations of a
// round-robin pairing are applied together (columns, then rows), so one CTA
// sweeps an R x R matrix in R-1 barrier-separated steps.  The two core
// contractions per sweep are shared between modes:
//   W[i,j,r] = sum_k C[i,j,k] A2[k,r]  ->  M0 = sum_j A1 W,  M1 = sum_i A0 W
//   X[j,k,r] = sum_i C[i,j,k] A0[i,r]  ->  M2 = sum_j A1 X
// and the fitness MTTKRP of sweep s (mode 0 with the final factors) is the
// mode-0 MTTKRP of sweep s+1, so each sweep costs two I*J*K*R passes.
#include "skx_common.cuh"

namespace skx {

constexpr int kCpThreads = 256;
constexpr int kCpMaxDim = 32;

struct CpBlk {
  double* red;  // kCpThreads / 32 + 1
};

__device__ __forceinline__ double cp_block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double s = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) red[32] = s;
  }
  __syncthreads();
  return red[32];
}

// Symmetric eigendecomposition a = v diag(d) v^T (n <= 32, row-major, a is
// overwritten; d = its final diagonal), parallel cyclic Jacobi with
// round-robin pairs.  cs: 2 * 16 doubles, pq: 2 * 16 ints, flag: one int.
__device__ void cp_jacobi_eig(double* a, double* v, int n, double* cs, int* pq, int* flag) {
  const int tid = threadIdx.x;
  const int nn = n + (n & 1);
  const int npair = nn / 2;
  for (int e = tid; e < n * n; e += blockDim.x) v[e] = (e / n == e % n) ? 1.0 : 0.0;
  // rotations keep ||a||_F; an off-diagonal entry below eps ||a||_F is at the
  // backward-error level of a LAPACK SVD of a (absolute criterion: a relative
  // one, |a_pq| < eps sqrt(a_pp a_qq), never settles under rounding when the
  // spectrum spans orders of magnitude)
  double fro2 = 0.0;
  for (int e = 0; e < n * n; ++e) fro2 += a[e] * a[e];
  const double tiny = 1e-16 * sqrt(fro2);
  __syncthreads();
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (tid == 0) *flag = 0;
    __syncthreads();
    for (int step = 0; step < nn - 1; ++step) {
      if (tid < npair) {
        int p, q;
        if (tid == 0) {
          p = step % (nn - 1);
          q = nn - 1;
        } else {
          p = (step + tid) % (nn - 1);
          q = (step - tid + (nn - 1)) % (nn - 1);
        }
        if (p > q) {
          int t = p;
          p = q;
          q = t;
        }
        double c = 1.0, s = 0.0;
        if (q < n) {
          const double apq = a[p * n + q];
          const double app = a[p * n + p], aqq = a[q * n + q];
          if (fabs(apq) > tiny && fabs(apq) > 1e-300) {
            const double tau = (aqq - app) / (2.0 * apq);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            *flag = 1;
          }
        }
        cs[2 * tid] = c;
        cs[2 * tid + 1] = s;
        pq[2 * tid] = p;
        pq[2 * tid + 1] = q;
      }
      __syncthreads();
      // A J (columns p, q of every row)
      for (int e = tid; e < npair * n; e += blockDim.x) {
        const int k = e / n, i = e % n;
        const int p = pq[2 * k], q = pq[2 * k + 1];
        const double s = cs[2 * k + 1];
        if (q >= n || s == 0.0) continue;
        const double c = cs[2 * k];
        const double x = a[i * n + p], y = a[i * n + q];
        a[i * n + p] = c * x - s * y;
        a[i * n + q] = s * x + c * y;
      }
      __syncthreads();
      // J^T (A J) (rows p, q) and V J
      for (int e = tid; e < npair * n; e += blockDim.x) {
        const int k = e / n, j = e % n;
        const int p = pq[2 * k], q = pq[2 * k + 1];
        const double s = cs[2 * k + 1];
        if (q >= n || s == 0.0) continue;
        const double c = cs[2 * k];
        const double x = a[p * n + j], y = a[q * n + j];
        a[p * n + j] = c * x - s * y;
        a[q * n + j] = s * x + c * y;
        const double vx = v[j * n + p], vy = v[j * n + q];
        v[j * n + p] = c * vx - s * vy;
        v[j * n + q] = s * vx + c * vy;
      }
      __syncthreads();
      if (tid < npair) {  // the annihilated pair is zero by construction
        const int p = pq[2 * tid], q = pq[2 * tid + 1];
        if (q < n && cs[2 * tid + 1] != 0.0) {
          a[p * n + q] = 0.0;
          a[q * n + p] = 0.0;
        }
      }
      __syncthreads();
    }
    if (*flag == 0) break;
    __syncthreads();
  }
  __syncthreads();
}

// order[0..n) = indices of the diagonal of a sorted descending (stable)
__device__ void cp_sort_desc(const double* a, int n, int* order) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) order[i] = i;
    for (int i = 1; i < n; ++i) {
      const int x = order[i];
      const double key = a[x * n + x];
      int j = i - 1;
      while (j >= 0 && a[order[j] * n + order[j]] < key) {
        order[j + 1] = order[j];
        --j;
      }
      order[j + 1] = x;
    }
  }
  __syncthreads();
}

struct CpDims {
  int I, J, K, R, sweeps;
};

__global__ void __launch_bounds__(kCpThreads, 2)
    k_cp_core_als(CpDims dm, const double* __restrict__ core_g, double* fac_out, double* w_out,
                  double* resid_out, double* fit_out, int* info) {
  extern __shared__ double sm[];
  const int I = dm.I, J = dm.J, K = dm.K, R = dm.R;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int dims[3] = {I, J, K};
  const int mx = max(I, max(J, K));
  // shared layout (doubles)
  double* C = sm;                                  // I*J*K
  double* Wb = C + I * J * K;                      // max(I*J, J*K) * R
  double* A[3];
  A[0] = Wb + max(I * J, J * K) * R;               // I*R
  A[1] = A[0] + I * R;                             // J*R
  A[2] = A[1] + J * R;                             // K*R
  double* G[3];
  G[0] = A[2] + K * R;                             // R*R each
  G[1] = G[0] + R * R;
  G[2] = G[1] + R * R;
  double* M = G[2] + R * R;                        // mx*R
  double* S = M + mx * R;                          // mx*R (a_scaled)
  double* E = S + mx * R;                          // mx*mx (eigen matrix)
  double* V = E + mx * mx;                         // mx*mx (eigenvectors)
  double* P = V + mx * mx;                         // R*R (pinv / Hadamard)
  double* wts = P + R * R;                         // R
  double* cs = wts + R;                            // 32
  double* red = cs + 32;                           // 33
  int* pq = (int*)(red + 34);                      // 32
  int* order = pq + 32;                            // 32
  int* flag = order + 32;                          // 1

  for (int e = tid; e < I * J * K; e += nt) C[e] = core_g[e];
  __syncthreads();
  // ||C||: np.linalg.norm of the core, squared as the reference does
  double acc = 0.0;
  for (int e = tid; e < I * J * K; e += nt) acc += C[e] * C[e];
  const double norm_t = sqrt(cp_block_sum(acc, red));
  const double norm_sq = norm_t * norm_t;
  if (norm_t == 0.0) {
    if (tid == 0) *info = 1;
    return;
  }

  // ---- hosvd-of-core init: leading eigenvectors of C_(n) C_(n)^T
  for (int n = 0; n < 3; ++n) {
    const int sn = dims[n];
    for (int e = tid; e < sn * sn; e += nt) {
      const int a = e / sn, b = e % sn;
      double g = 0.0;
      if (n == 0) {
        for (int x = 0; x < J * K; ++x) g += C[a * J * K + x] * C[b * J * K + x];
      } else if (n == 1) {
        for (int i = 0; i < I; ++i)
          for (int k = 0; k < K; ++k) g += C[(i * J + a) * K + k] * C[(i * J + b) * K + k];
      } else {
        for (int x = 0; x < I * J; ++x) g += C[x * K + a] * C[x * K + b];
      }
      E[e] = g;
    }
    __syncthreads();
    cp_jacobi_eig(E, V, sn, cs, pq, flag);
    cp_sort_desc(E, sn, order);
    for (int e = tid; e < sn * R; e += nt) {
      const int i = e / R, r = e % R;
      A[n][e] = V[i * sn + order[r]];
    }
    __syncthreads();
  }
  for (int e = tid; e < R; e += nt) wts[e] = 1.0;
  // Grams
  for (int n = 0; n < 3; ++n)
    for (int e = tid; e < R * R; e += nt) {
      const int r = e / R, s = e % R;
      double g = 0.0;
      for (int i = 0; i < dims[n]; ++i) g += A[n][i * R + r] * A[n][i * R + s];
      G[n][e] = g;
    }
  __syncthreads();

  auto build_W = [&]() {  // W[i,j,r] = sum_k C[i,j,k] A2[k,r]
    for (int e = tid; e < I * J * R; e += nt) {
      const int r = e % R, ij = e / R;
      double s = 0.0;
      for (int k = 0; k < K; ++k) s += C[ij * K + k] * A[2][k * R + r];
      Wb[e] = s;
    }
    __syncthreads();
  };
  auto m0_from_W = [&]() {  // M[i,r] = sum_j A1[j,r] W[i,j,r]
    for (int e = tid; e < I * R; e += nt) {
      const int i = e / R, r = e % R;
      double s = 0.0;
      for (int j = 0; j < J; ++j) s += Wb[(i * J + j) * R + r] * A[1][j * R + r];
      M[e] = s;
    }
    __syncthreads();
  };

  // one mode update: M holds the MTTKRP of mode n (s_n x R)
  auto update = [&](int n, double* res_slot) {
    const int sn = dims[n];
    // Hadamard of the other Grams (into E as R x R)
    for (int e = tid; e < R * R; e += nt) {
      double g = 1.0;
      for (int k = 0; k < 3; ++k)
        if (k != n) g *= G[k][e];
      E[e] = g;
      P[e] = g;  // kept for the residual
    }
    __syncthreads();
    // Fast path: when the (SPD) Hadamard Gram is well conditioned, pinv with
    // rcond = 1e-12 truncates nothing and equals the inverse; warp 0 forms it
    // by Cholesky (G = L L^T, G^-1 = L^-T L^-1) in ~3 R short serial steps
    // instead of the ~(R-1) x sweeps barrier-separated Jacobi steps, and
    // checks cond_1(G) = ||G||_1 ||G^-1||_1 < 1e4 (then the two agree to
    // ~1e-12); otherwise the eigendecomposition below runs as before.
    if (tid < 32) {
      const int lane = tid;
      for (int e = lane; e < R * R; e += 32) V[e] = P[e];
      __syncwarp();
      bool ok = true;
      for (int k = 0; k < R && ok; ++k) {
        const double dk = V[k * R + k];
        if (!(dk > 0.0)) {  // uniform
          ok = false;
          break;
        }
        const double d = sqrt(dk);
        __syncwarp();
        for (int i = k + lane; i < R; i += 32) V[i * R + k] = i == k ? d : V[i * R + k] / d;
        __syncwarp();
        const int t = R - k - 1;
        for (int e = lane; e < t * t; e += 32) {
          const int i = k + 1 + e / t, j = k + 1 + e % t;
          if (j <= i) V[i * R + j] = fma(-V[i * R + k], V[j * R + k], V[i * R + j]);
        }
        __syncwarp();
      }
      if (ok) {
        // L^-1 (lower) into E, column j by lane j
        if (lane < R) {
          const int j = lane;
          for (int i = 0; i < R; ++i) {
            double x = i == j ? 1.0 : 0.0;
            for (int k = j; k < i; ++k) x = fma(-V[i * R + k], E[k * R + j], x);
            E[i * R + j] = i < j ? 0.0 : x / V[i * R + i];
          }
        }
        __syncwarp();
        // G^-1 = L^-T L^-1 into V
        for (int e = lane; e < R * R; e += 32) {
          const int a2 = e / R, b2 = e % R;
          double x = 0.0;
          for (int k = max(a2, b2); k < R; ++k) x = fma(E[k * R + a2], E[k * R + b2], x);
          V[e] = x;
        }
        __syncwarp();
        double c1 = 0.0, c2 = 0.0;
        if (lane < R)
          for (int i = 0; i < R; ++i) {
            c1 += fabs(P[i * R + lane]);
            c2 += fabs(V[i * R + lane]);
          }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          c1 = fmax(c1, __shfl_xor_sync(0xffffffffu, c1, o));
          c2 = fmax(c2, __shfl_xor_sync(0xffffffffu, c2, o));
        }
        ok = c1 * c2 < 1e4;
      }
      if (lane == 0) *flag = ok ? 1 : 0;
    }
    __syncthreads();
    if (*flag) {
      // S = M G^-1
      for (int e = tid; e < sn * R; e += nt) {
        const int i = e / R, q = e % R;
        double s = 0.0;
        for (int r = 0; r < R; ++r) s += M[i * R + r] * V[r * R + q];
        S[e] = s;
      }
      __syncthreads();
    } else {
    for (int e = tid; e < R * R; e += nt) E[e] = P[e];
    __syncthreads();
    cp_jacobi_eig(E, V, R, cs, pq, flag);
    // pinv(G, rcond=1e-12): sum over |lambda| > 1e-12 max|lambda| of v v^T / lambda
    double* lam = cs;  // reuse: R <= 32 eigenvalues
    __syncthreads();
    if (tid == 0) {
      double smax = 0.0;
      for (int r = 0; r < R; ++r) smax = fmax(smax, fabs(E[r * R + r]));
      red[33] = 1e-12 * smax;
    }
    __syncthreads();
    for (int e = tid; e < R; e += nt) {
      const double l = E[e * R + e];
      lam[e] = fabs(l) > red[33] ? 1.0 / l : 0.0;
    }
    __syncthreads();
    // S = M @ pinv = ((M V) diag(1/lambda)) V^T ; E as scratch for M V
    for (int e = tid; e < sn * R; e += nt) {
      const int i = e / R, q = e % R;
      double s = 0.0;
      for (int r = 0; r < R; ++r) s += M[i * R + r] * V[r * R + q];
      E[e] = s * lam[q];
    }
    __syncthreads();
    for (int e = tid; e < sn * R; e += nt) {
      const int i = e / R, r = e % R;
      double s = 0.0;
      for (int q = 0; q < R; ++q) s += E[i * R + q] * V[r * R + q];
      S[e] = s;
    }
    __syncthreads();
    }
    // residual: sqrt(max(||T||^2 - 2 <S, M> + <S^T S, G_others>, 0))
    double cr = 0.0;
    for (int e = tid; e < sn * R; e += nt) cr += S[e] * M[e];
    const double cross = cp_block_sum(cr, red);
    double md = 0.0;
    for (int e = tid; e < R * R; e += nt) {
      const int r = e / R, s = e % R;
      double g = 0.0;
      for (int i = 0; i < sn; ++i) g += S[i * R + r] * S[i * R + s];
      md += g * P[e];
    }
    const double model = cp_block_sum(md, red);
    if (tid == 0) *res_slot = sqrt(fmax(norm_sq - 2.0 * cross + model, 0.0));
    // normalise the columns into the weights
    for (int r = tid; r < R; r += nt) {
      double s = 0.0;
      for (int i = 0; i < sn; ++i) s += S[i * R + r] * S[i * R + r];
      wts[r] = sqrt(s);
    }
    __syncthreads();
    for (int e = tid; e < sn * R; e += nt) {
      const double nr = wts[e % R];
      A[n][e] = S[e] / (nr > 0.0 ? nr : 1.0);
    }
    __syncthreads();
    for (int e = tid; e < R * R; e += nt) {
      const int r = e / R, s = e % R;
      double g = 0.0;
      for (int i = 0; i < sn; ++i) g += A[n][i * R + r] * A[n][i * R + s];
      G[n][e] = g;
    }
    __syncthreads();
  };

  build_W();
  m0_from_W();
  for (int sw = 0; sw < dm.sweeps; ++sw) {
    update(0, resid_out + 3 * sw);
    // M1[j,r] = sum_i A0[i,r] W[i,j,r]  (W still holds A2's contraction)
    for (int e = tid; e < J * R; e += nt) {
      const int j = e / R, r = e % R;
      double s = 0.0;
      for (int i = 0; i < I; ++i) s += Wb[(i * J + j) * R + r] * A[0][i * R + r];
      M[e] = s;
    }
    __syncthreads();
    update(1, resid_out + 3 * sw + 1);
    // X[j,k,r] = sum_i C[i,j,k] A0[i,r];  M2[k,r] = sum_j A1[j,r] X[j,k,r]
    for (int e = tid; e < J * K * R; e += nt) {
      const int r = e % R, jk = e / R;
      double s = 0.0;
      for (int i = 0; i < I; ++i) s += C[i * J * K + jk] * A[0][i * R + r];
      Wb[e] = s;
    }
    __syncthreads();
    for (int e = tid; e < K * R; e += nt) {
      const int k = e / R, r = e % R;
      double s = 0.0;
      for (int j = 0; j < J; ++j) s += Wb[(j * K + k) * R + r] * A[1][j * R + r];
      M[e] = s;
    }
    __syncthreads();
    update(2, resid_out + 3 * sw + 2);
    // fitness of CPModel(factors, weights) on the core: mttkrp mode 0 with the
    // final factors (also the next sweep's mode-0 MTTKRP)
    build_W();
    m0_from_W();
    double cr = 0.0;
    for (int e = tid; e < I * R; e += nt) cr += A[0][e] * wts[e % R] * M[e];
    const double cross = cp_block_sum(cr, red);
    double md = 0.0;
    for (int e = tid; e < R * R; e += nt) {
      const int r = e / R, s = e % R;
      md += G[0][e] * wts[r] * wts[s] * G[1][e] * G[2][e];
    }
    const double model = cp_block_sum(md, red);
    if (tid == 0) fit_out[sw] = 1.0 - sqrt(fmax(norm_sq - 2.0 * cross + model, 0.0)) / norm_t;
  }
  // outputs: factors (mode after mode), weights
  int off = 0;
  for (int n = 0; n < 3; ++n) {
    for (int e = tid; e < dims[n] * R; e += nt) fac_out[off + e] = A[n][e];
    off += dims[n] * R;
  }
  for (int e = tid; e < R; e += nt) w_out[e] = wts[e];
  if (tid == 0) *info = 0;
}

inline size_t cp_core_smem(int I, int J, int K, int R) {
  const int mx = std::max(I, std::max(J, K));
  size_t d = (size_t)I * J * K + (size_t)std::max(I * J, J * K) * R + (size_t)(I + J + K) * R +
             3 * R * R + 2 * mx * R + 2 * mx * mx + R * R + R + 32 + 34;
  return d * sizeof(double) + 32 * 2 * sizeof(int) + 16;
}

}  // namespace skx

using namespace skx;

extern "C" int skx_cp_core_als(const int64_t* dims_h, int rank, int sweeps, const double* core,
                               double* factors, double* weights, double* residuals,
                               double* fitness, int* info, void* stream) {
  SKX_REQUIRE(rank >= 1 && rank <= kCpMaxDim, "skx_cp_core_als: rank must be in 1..32");
  SKX_REQUIRE(sweeps >= 0, "skx_cp_core_als: negative sweep count");
  const int I = (int)dims_h[0], J = (int)dims_h[1], K = (int)dims_h[2];
  SKX_REQUIRE(I >= rank && J >= rank && K >= rank && I <= kCpMaxDim && J <= kCpMaxDim &&
                  K <= kCpMaxDim,
              "skx_cp_core_als: core extents must lie in [rank, 32]");
  const size_t smem = cp_core_smem(I, J, K, rank);
  SKX_REQUIRE((int64_t)smem <= (int64_t)max_smem_optin(),
              "skx_cp_core_als: core %dx%dx%d rank %d needs %zu bytes of shared memory", I, J, K,
              rank, smem);
  cudaFuncSetAttribute(k_cp_core_als, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  CpDims dm{I, J, K, rank, sweeps};
  k_cp_core_als<<<1, kCpThreads, smem, (cudaStream_t)stream>>>(dm, core, factors, weights,
                                                               residuals, fitness, info);
  return check_launch("k_cp_core_als");
}

extern "C" size_t skx_cp_core_smem_bytes(const int64_t* dims_h, int rank) {
  return cp_core_smem((int)dims_h[0], (int)dims_h[1], (int)dims_h[2], rank);
}
