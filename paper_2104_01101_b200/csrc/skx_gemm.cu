// K5: the passes over the sketched right-hand side Y in rsvd_lrls
// (src/linalg.py:103-112, associated form: Y G and W^T Y, both with a narrow
// second operand of w <= 32 columns) as FP64 tensor-core (mma.sync m8n8k4)
// streaming kernels.  Y is m x s_n and is stored either row-major (dense /
// leverage sketches) or as Y^T (TensorSketch right-hand sides), so both a
// "C = A B" (A tall, streamed by rows) and a "C = A^T B" (reduction over the
// long dimension, split over CTAs, partials summed in a fixed order) kernel
// are provided; together they cover Y G and W^T Y for either storage.
//
// The A fragments are loaded 16 bytes per lane: k-step 2j of a pair holds
// k = 8j + 2c, k-step 2j+1 holds 8j + 2c + 1 (c = lane % 4), and B is staged
// in shared memory with the same k map, so one 64-byte row piece per four
// lanes comes in per load instruction.  Deterministic: fixed tiles, fixed
// split-K partition, fixed reduction order.
#include <stdlib.h>

#include "skx_common.cuh"

namespace skx {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int kGKC = 32;      // k per staged chunk (4 k-step pairs)
constexpr int kGRows = 128;   // rows (A B) or columns (A^T B) of C per CTA

// C[M x N] = A[M x K] B[K x N]; A row-major (lda), B row-major (ldb), N <= 8 NT.
// CTA = 8 warps x 16 rows; K streamed in chunks of 32 (B chunk in shared).
// blockIdx.y = K split: k in [y kchunk, (y + 1) kchunk), written to
// C + y cstride (partials, summed in order by k_gemm_atb_sum).
template <int NT, bool VEC>
__global__ void __launch_bounds__(256) k_gemm_ab(int64_t M, int N, int64_t K,
                                                 const double* __restrict__ A, int64_t lda,
                                                 const double* __restrict__ B, int64_t ldb,
                                                 double* __restrict__ C, int64_t ldc,
                                                 int64_t kchunk, int64_t cstride) {
  __shared__ double Bs[kGKC][8 * NT + 2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, q = lane >> 2, c = lane & 3;
  const int64_t row0 = blockIdx.x * (int64_t)kGRows + wid * 16;
  const int64_t kbeg = blockIdx.y * kchunk;
  K = imin(K, kbeg + kchunk);
  C += blockIdx.y * cstride;
  double acc[2][NT][2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[t][n][0] = acc[t][n][1] = 0.0;
  const int64_t r0 = row0 + q, r1 = row0 + 8 + q;
  const double* a0 = A + (r0 < M ? r0 : 0) * lda;
  const double* a1 = A + (r1 < M ? r1 : 0) * lda;
  for (int64_t k0 = kbeg; k0 < K; k0 += kGKC) {
    __syncthreads();
    for (int e = threadIdx.x; e < kGKC * 8 * NT; e += blockDim.x) {
      const int kk = e / (8 * NT), n = e - kk * (8 * NT);
      Bs[kk][n] = (k0 + kk < K && n < N) ? B[(k0 + kk) * ldb + n] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kGKC / 8; ++j) {
      const int64_t k = k0 + 8 * j + 2 * c;
      double x0[2], x1[2];  // rows r0, r1: elements k, k+1
      if (VEC && k + 1 < K) {
        const double2 p = r0 < M ? __ldcs(reinterpret_cast<const double2*>(a0 + k)) : make_double2(0, 0);
        const double2 s = r1 < M ? __ldcs(reinterpret_cast<const double2*>(a1 + k)) : make_double2(0, 0);
        x0[0] = p.x; x0[1] = p.y; x1[0] = s.x; x1[1] = s.y;
      } else {
        x0[0] = (r0 < M && k < K) ? a0[k] : 0.0;
        x0[1] = (r0 < M && k + 1 < K) ? a0[k + 1] : 0.0;
        x1[0] = (r1 < M && k < K) ? a1[k] : 0.0;
        x1[1] = (r1 < M && k + 1 < K) ? a1[k + 1] : 0.0;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int kk = 8 * j + 2 * c + h;  // B row in the chunk for this lane's k-step
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const double bv = Bs[8 * j + 2 * c + h][n * 8 + q];
          (void)kk;
          dmma(acc[0][n][0], acc[0][n][1], x0[h], bv);
          dmma(acc[1][n][0], acc[1][n][1], x1[h], bv);
        }
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int64_t r = row0 + 8 * t + q;
    if (r >= M) continue;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int col = n * 8 + 2 * c;
      if (col < N) C[r * ldc + col] = acc[t][n][0];
      if (col + 1 < N) C[r * ldc + col + 1] = acc[t][n][1];
    }
  }
}

// Partial P[s][m][n] = sum_{k in chunk s} A[k][m] B[k][n] (A^T B); A row-major
// K x M (lda), B row-major K x N (ldb).  CTA = 8 warps x 16 columns of A.
template <int NT>
__global__ void __launch_bounds__(256) k_gemm_atb_part(int64_t M, int N, int64_t K, int64_t kchunk,
                                                       const double* __restrict__ A, int64_t lda,
                                                       const double* __restrict__ B, int64_t ldb,
                                                       double* __restrict__ P) {
  __shared__ double Bs[kGKC][8 * NT + 2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, q = lane >> 2, c = lane & 3;
  const int64_t col0 = blockIdx.x * (int64_t)kGRows + wid * 16;
  const int64_t kbeg = blockIdx.y * kchunk, kend = imin(K, kbeg + kchunk);
  double acc[2][NT][2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[t][n][0] = acc[t][n][1] = 0.0;
  const int64_t m0 = col0 + q, m1 = col0 + 8 + q;
  for (int64_t k0 = kbeg; k0 < kend; k0 += kGKC) {
    __syncthreads();
    for (int e = threadIdx.x; e < kGKC * 8 * NT; e += blockDim.x) {
      const int kk = e / (8 * NT), n = e - kk * (8 * NT);
      Bs[kk][n] = (k0 + kk < kend && n < N) ? B[(k0 + kk) * ldb + n] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < kGKC / 4; ++ks) {
      const int64_t k = k0 + 4 * ks + c;
      const double* ar = A + (k < kend ? k : kbeg) * lda;
      const double x0 = (k < kend && m0 < M) ? __ldcs(ar + m0) : 0.0;
      const double x1 = (k < kend && m1 < M) ? __ldcs(ar + m1) : 0.0;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const double bv = Bs[4 * ks + c][n * 8 + q];
        dmma(acc[0][n][0], acc[0][n][1], x0, bv);
        dmma(acc[1][n][0], acc[1][n][1], x1, bv);
      }
    }
  }
  double* Ps = P + (int64_t)blockIdx.y * M * N;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int64_t m = col0 + 8 * t + q;
    if (m >= M) continue;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int col = n * 8 + 2 * c;
      if (col < N) Ps[m * N + col] = acc[t][n][0];
      if (col + 1 < N) Ps[m * N + col + 1] = acc[t][n][1];
    }
  }
}

__global__ void k_gemm_atb_sum(const double* __restrict__ P, int64_t MN, int S, int64_t M, int N,
                               double* __restrict__ C, int64_t ldc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < MN;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int t = 0; t < S; ++t) s += P[(int64_t)t * MN + i];
    const int64_t m = i / N, n = i - m * N;
    C[m * ldc + n] = s;
  }
}

}  // namespace skx

using namespace skx;

namespace {
// K split of skx_gemm_ab: the row blocks alone can leave a last partial wave
// (config 4: 782 blocks on 592 CTA slots = 0.66 of two waves); split K into
// S <= 4 chunks (>= 256 each) when that fills the waves better, partials
// summed in a fixed order (deterministic for given shapes).
int gab_split(int64_t M, int64_t K, int NT) {
  static int occ[5] = {0, 0, 0, 0, 0};
  if (occ[NT] == 0) {
    int o = 0;
    switch (NT) {
      case 1: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_gemm_ab<1, true>, 256, 0); break;
      case 2: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_gemm_ab<2, true>, 256, 0); break;
      case 3: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_gemm_ab<3, true>, 256, 0); break;
      default: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_gemm_ab<4, true>, 256, 0); break;
    }
    occ[NT] = o > 0 ? o : 1;
  }
  const int64_t slots = (int64_t)num_sms() * occ[NT];
  const int64_t mb = (M + kGRows - 1) / kGRows;
  int best = 1;
  double best_eff = 0.0;
  for (int S = 1; S <= 4; ++S) {
    if (S > 1 && K < 256 * (int64_t)S) break;
    const int64_t tiles = mb * S, waves = (tiles + slots - 1) / slots;
    const double eff = (double)tiles / (double)(waves * slots);
    if (eff > best_eff + 0.02) {
      best = S;
      best_eff = eff;
    }
    if (S == 1 && eff >= 0.9) break;
  }
  return best;
}
}  // namespace

extern "C" int skx_gemm_ab(int64_t M, int N, int64_t K, const double* A, int64_t lda,
                           const double* B, int64_t ldb, double* C, int64_t ldc, void* ws,
                           size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(N >= 1 && N <= 32, "skx_gemm_ab: 1 <= N <= 32");
  SKX_REQUIRE(M >= 0 && K >= 0, "skx_gemm_ab: negative extent");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_gemm_ab: ws_bytes is NULL");
  const int NT = (N + 7) / 8;
  int S = (M > 0 && K > 0 && getenv("SKX_GAB_NOSPLIT") == nullptr) ? gab_split(M, K, NT) : 1;
  const int64_t kchunk = S > 1 ? ((K + S - 1) / S + kGKC - 1) / kGKC * kGKC : K;
  if (S > 1) S = (int)((K + kchunk - 1) / kchunk);
  Arena ar(ws, *ws_bytes);
  double* P = S > 1 ? ar.take<double>((size_t)S * M * N) : nullptr;
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_gemm_ab: workspace too small");
  if (M == 0) return SKX_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const bool vec = (lda % 2 == 0) && ((uintptr_t)A % 16 == 0);
  const dim3 g((unsigned)((M + kGRows - 1) / kGRows), (unsigned)S);
  double* out = S > 1 ? P : C;
  const int64_t ldo = S > 1 ? N : ldc, cs = S > 1 ? M * N : 0;
#define SKX_GAB(nt)                                                                                \
  if (NT == nt) {                                                                                  \
    if (vec) k_gemm_ab<nt, true><<<g, 256, 0, st>>>(M, N, K, A, lda, B, ldb, out, ldo, kchunk, cs); \
    else k_gemm_ab<nt, false><<<g, 256, 0, st>>>(M, N, K, A, lda, B, ldb, out, ldo, kchunk, cs);    \
  }
  SKX_GAB(1) SKX_GAB(2) SKX_GAB(3) SKX_GAB(4)
#undef SKX_GAB
  if (S > 1) {
    const int64_t MN = M * N;
    k_gemm_atb_sum<<<(unsigned)imin((MN + 255) / 256, (int64_t)num_sms() * 8), 256, 0, st>>>(
        P, MN, S, M, N, C, ldc);
  }
  return check_launch("k_gemm_ab", S > 1 ? 2 : 1);
}

extern "C" int skx_gemm_atb(int64_t M, int N, int64_t K, const double* A, int64_t lda,
                            const double* B, int64_t ldb, double* C, int64_t ldc, void* ws,
                            size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(N >= 1 && N <= 32, "skx_gemm_atb: 1 <= N <= 32");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_gemm_atb: ws_bytes is NULL");
  const int64_t mb = (M + kGRows - 1) / kGRows;
  // split K so that about four CTAs per SM stream A
  int64_t S = imax(1, imin((int64_t)num_sms() * 4 / imax(mb, 1), (K + 1023) / 1024));
  const int64_t kchunk = ((K + S - 1) / S + kGKC - 1) / kGKC * kGKC;
  S = imax(1, (K + kchunk - 1) / kchunk);
  Arena ar(ws, *ws_bytes);
  double* P = ar.take<double>((size_t)S * M * N);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_gemm_atb: workspace too small");
  if (M == 0) return SKX_OK;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((unsigned)mb, (unsigned)S);
  const int NT = (N + 7) / 8;
#define SKX_GATB(nt) \
  if (NT == nt) k_gemm_atb_part<nt><<<grid, 256, 0, st>>>(M, N, K, kchunk, A, lda, B, ldb, P);
  SKX_GATB(1) SKX_GATB(2) SKX_GATB(3) SKX_GATB(4)
#undef SKX_GATB
  const int64_t MN = M * N;
  k_gemm_atb_sum<<<(unsigned)imin((MN + 255) / 256, (int64_t)num_sms() * 8), 256, 0, st>>>(
      P, MN, (int)S, M, N, C, ldc);
  return check_launch("k_gemm_atb", 2);
}
