// K5 residual and K7 fitness passes (src/tucker.py:274; src/tensors.py:
// 339-368).  All reductions use a fixed grid and a fixed combination order,
// so results are bitwise reproducible.
#include "skx_common.cuh"

namespace skx {

constexpr int kRedBlocks = 1024;
constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
    for (int w = 0; w < nw; ++w) t += sh[w];
  }
  __syncthreads();
  return t;  // valid in thread 0
}

__global__ void k_final_sum(const double* __restrict__ part, int n, double* out) {
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += part[i];
  v = block_sum(v);
  if (threadIdx.x == 0) out[0] = v;
}

__global__ void k_sumsq(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    acc = fma(v, v, acc);
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// sum_{o,x} (sum_r U[o,r] Vt[r,x] - Y[o*ld + x])^2 -- Y's unit-stride index x
// is the inner one.  A CTA takes TO outer rows at a time (their U rows staged in
// shared memory) and sweeps x: the R values Vt[:, x] are loaded once into
// registers and reused for the TO rows, Y is streamed once, coalesced.
template <int RT, int TO>
__global__ void __launch_bounds__(256) k_resid(const double* __restrict__ U,
                                               const double* __restrict__ Vt, int64_t n_out,
                                               int64_t n_in, int R, const double* __restrict__ y,
                                               int64_t ld, double* __restrict__ part) {
  __shared__ double us[TO * RT];
  double acc = 0.0;
  for (int64_t o0 = blockIdx.x * (int64_t)TO; o0 < n_out; o0 += (int64_t)gridDim.x * TO) {
    const int nk = (int)imin(TO, n_out - o0);
    __syncthreads();
    for (int q = threadIdx.x; q < TO * RT; q += blockDim.x) {
      const int k = q / RT, r = q - k * RT;
      us[q] = (k < nk && r < R) ? U[(o0 + k) * R + r] : 0.0;
    }
    __syncthreads();
    for (int64_t x = threadIdx.x; x < n_in; x += blockDim.x) {
      double v[RT];
#pragma unroll
      for (int r = 0; r < RT; ++r) v[r] = r < R ? __ldg(Vt + (int64_t)r * n_in + x) : 0.0;
#pragma unroll
      for (int k = 0; k < TO; ++k) {
        if (k < nk) {
          double pred = 0.0;
#pragma unroll
          for (int r = 0; r < RT; ++r) pred = fma(us[k * RT + r], v[r], pred);
          const double d = pred - __ldcs(y + (o0 + k) * ld + x);
          acc = fma(d, d, acc);
        }
      }
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// Generic R (no register tile): one (o, x) pair per thread step.
__global__ void k_resid_gen(const double* __restrict__ U, const double* __restrict__ Vt,
                            int64_t n_out, int64_t n_in, int R, const double* __restrict__ y,
                            int64_t ld, double* __restrict__ part) {
  double acc = 0.0;
  for (int64_t o = blockIdx.x; o < n_out; o += gridDim.x) {
    for (int64_t x = threadIdx.x; x < n_in; x += blockDim.x) {
      double pred = 0.0;
      for (int r = 0; r < R; ++r) pred = fma(U[o * R + r], Vt[(int64_t)r * n_in + x], pred);
      const double d = pred - y[o * ld + x];
      acc = fma(d, d, acc);
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// ---- Tucker cross term, order 3, lexsorted COO grouped by i0 (colptr0).
// Warp per slice i0: W = A0[i0,:] x_0 C (R1 x R2) in shared memory, then
// each nonzero adds v * A1[i1,:] W A2[i2,:]^T.  Per-slice sums are written to
// slice_out and reduced in slice order.
// v[r2] = sum_r1 A1[i1,r1] W[r1,r2] runs R2 independent FMA chains (ILP), then
// t = v . A2[i2,:]; two nonzeros per lane share every W load.
template <int R2T>
__global__ void __launch_bounds__(256) k_tucker3(const int64_t* __restrict__ colptr, int64_t s0,
                                                 const int32_t* __restrict__ c1,
                                                 const int32_t* __restrict__ c2,
                                                 const double* __restrict__ vals,
                                                 const double* __restrict__ A0,
                                                 const double* __restrict__ A1,
                                                 const double* __restrict__ A2,
                                                 const double* __restrict__ C, int R0, int R1,
                                                 int R2, double* __restrict__ slice_out) {
  extern __shared__ double smem[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  double* W = smem + (size_t)wid * R1 * R2T;  // rows padded to R2T
  for (int64_t i0 = blockIdx.x * (int64_t)nw + wid; i0 < s0; i0 += (int64_t)gridDim.x * nw) {
    const int64_t e0 = colptr[i0], e1 = colptr[i0 + 1];
    if (e0 == e1) {
      if (lane == 0) slice_out[i0] = 0.0;
      continue;
    }
    for (int q = lane; q < R1 * R2T; q += 32) {
      const int r1 = q / R2T, r2 = q - r1 * R2T;
      double s = 0.0;
      if (r2 < R2)
        for (int r0 = 0; r0 < R0; ++r0)
          s = fma(A0[i0 * R0 + r0], C[((int64_t)r0 * R1 + r1) * R2 + r2], s);
      W[q] = s;
    }
    __syncwarp();
    double acc = 0.0;
    for (int64_t e = e0 + lane; e < e1; e += 64) {
      const int64_t f = e + 32;
      const bool has2 = f < e1;
      const double* a1 = A1 + (int64_t)c1[e] * R1;
      const double* a2 = A2 + (int64_t)c2[e] * R2;
      const double* a1b = A1 + (int64_t)c1[has2 ? f : e] * R1;
      const double* a2b = A2 + (int64_t)c2[has2 ? f : e] * R2;
      double v[R2T], w[R2T];
#pragma unroll
      for (int r = 0; r < R2T; ++r) {
        v[r] = 0.0;
        w[r] = 0.0;
      }
      for (int r1 = 0; r1 < R1; ++r1) {
        const double x = a1[r1], xb = a1b[r1];
        const double* wr = W + r1 * R2T;
#pragma unroll
        for (int r2 = 0; r2 < R2T; ++r2) {
          const double wv = wr[r2];
          v[r2] = fma(x, wv, v[r2]);
          w[r2] = fma(xb, wv, w[r2]);
        }
      }
      double t = 0.0, tb = 0.0;
#pragma unroll
      for (int r2 = 0; r2 < R2T; ++r2) {
        if (r2 < R2) {
          t = fma(v[r2], a2[r2], t);
          tb = fma(w[r2], a2b[r2], tb);
        }
      }
      acc = fma(vals[e], t, acc);
      if (has2) acc = fma(vals[f], tb, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane == 0) slice_out[i0] = acc;
    __syncwarp();
  }
}

// Generic order-N Tucker cross term: per nonzero, odometer over the core.
struct GenPack {
  int ndim;
  int64_t R[8];
  const double* A[8];
  const int32_t* c[8];
};

__global__ void k_tucker_gen(GenPack g, int64_t nnz, const double* __restrict__ vals,
                             const double* __restrict__ C, int64_t csize, double* __restrict__ part) {
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int64_t f = 0; f < csize; ++f) {
      int64_t rem = f;
      double prod = C[f];
      for (int k = g.ndim - 1; k >= 0; --k) {
        const int64_t r = rem % g.R[k];
        rem /= g.R[k];
        prod *= g.A[k][(int64_t)g.c[k][e] * g.R[k] + r];
      }
      t += prod;
    }
    acc = fma(vals[e], t, acc);
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void k_cp_cross(GenPack g, int64_t R, int64_t nnz, const double* __restrict__ vals,
                           const double* __restrict__ w, double* __restrict__ part) {
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int64_t r = 0; r < R; ++r) {
      double prod = w[r];
      for (int k = 0; k < g.ndim; ++k) prod *= g.A[k][(int64_t)g.c[k][e] * R + r];
      t += prod;
    }
    acc = fma(vals[e], t, acc);
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

}  // namespace skx

using namespace skx;

extern "C" int skx_sumsq(const double* x, int64_t n, double* out, void* ws, size_t* ws_bytes,
                         void* stream) {
  SKX_REQUIRE(ws_bytes != nullptr, "skx_sumsq: ws_bytes is NULL");
  if (ws == nullptr) {
    *ws_bytes = kRedBlocks * sizeof(double) + 256;
    return SKX_OK;
  }
  cudaStream_t s = (cudaStream_t)stream;
  double* part = (double*)ws;
  k_sumsq<<<kRedBlocks, kRedThreads, 0, s>>>(x, n, part);
  k_final_sum<<<1, 1024, 0, s>>>(part, kRedBlocks, out);
  return check_launch("skx_sumsq", 2);
}

extern "C" int skx_resid_sq(const double* u, const double* vt, int64_t n_out, int64_t n_in,
                            int64_t R, const double* y, int64_t ld, double* out, void* ws,
                            size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(ws_bytes != nullptr, "skx_resid_sq: ws_bytes is NULL");
  if (ws == nullptr) {
    *ws_bytes = kRedBlocks * sizeof(double) + 256;
    return SKX_OK;
  }
  cudaStream_t st = (cudaStream_t)stream;
  double* part = (double*)ws;
  const int r = (int)R;
  if (R <= 4)
    k_resid<4, 16><<<kRedBlocks, kRedThreads, 0, st>>>(u, vt, n_out, n_in, r, y, ld, part);
  else if (R <= 8)
    k_resid<8, 8><<<kRedBlocks, kRedThreads, 0, st>>>(u, vt, n_out, n_in, r, y, ld, part);
  else if (R <= 10)
    k_resid<10, 8><<<kRedBlocks, kRedThreads, 0, st>>>(u, vt, n_out, n_in, r, y, ld, part);
  else if (R <= 16)
    k_resid<16, 8><<<kRedBlocks, kRedThreads, 0, st>>>(u, vt, n_out, n_in, r, y, ld, part);
  else if (R <= 20)
    k_resid<20, 8><<<kRedBlocks, kRedThreads, 0, st>>>(u, vt, n_out, n_in, r, y, ld, part);
  else if (R <= 32)
    k_resid<32, 4><<<kRedBlocks, kRedThreads, 0, st>>>(u, vt, n_out, n_in, r, y, ld, part);
  else
    k_resid_gen<<<kRedBlocks, kRedThreads, 0, st>>>(u, vt, n_out, n_in, r, y, ld, part);
  k_final_sum<<<1, 1024, 0, st>>>(part, kRedBlocks, out);
  return check_launch("skx_resid_sq", 2);
}

extern "C" int skx_tucker_cross_coo(int ndim, const int64_t* shape_h, const int64_t* ranks_h,
                                    int64_t nnz, const int32_t* coords, const double* vals,
                                    const double* const* factors_h, const double* core,
                                    const int64_t* colptr0, double* out, void* ws,
                                    size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(ndim >= 1 && ndim <= 8, "skx_tucker_cross_coo: order 1..8");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_tucker_cross_coo: ws_bytes is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  const bool fast3 = (ndim == 3 && ranks_h[2] <= 32 && colptr0 != nullptr &&
                      ranks_h[1] * 32 * 8 * 8 <= 200 * 1024);
  const size_t need = fast3 ? (size_t)shape_h[0] * 8 + 256 : kRedBlocks * sizeof(double) + 256;
  if (ws == nullptr) {
    *ws_bytes = need;
    return SKX_OK;
  }
  SKX_REQUIRE(*ws_bytes >= need, "skx_tucker_cross_coo: workspace too small");
  double* part = (double*)ws;
  if (nnz == 0) {
    cudaMemsetAsync(out, 0, 8, s);
    return check_launch("tucker cross (empty)", 0);
  }
  if (fast3) {
    const int R0 = (int)ranks_h[0], R1 = (int)ranks_h[1], R2 = (int)ranks_h[2];
    const int64_t s0 = shape_h[0];
    const unsigned blocks = (unsigned)imin((s0 + 7) / 8, (int64_t)num_sms() * 8);
    const int32_t* c1 = coords + nnz;
    const int32_t* c2 = coords + 2 * nnz;
    const double* A0 = factors_h[0];
    const double* A1 = factors_h[1];
    const double* A2 = factors_h[2];
#define SKX_T3(RT)                                                                         \
  k_tucker3<RT><<<blocks, 256, (size_t)8 * R1 * RT * 8, s>>>(colptr0, s0, c1, c2, vals, A0, A1, \
                                                              A2, core, R0, R1, R2, part)
    if (R2 <= 4) SKX_T3(4);
    else if (R2 <= 8) SKX_T3(8);
    else if (R2 <= 10) SKX_T3(10);
    else if (R2 <= 16) SKX_T3(16);
    else if (R2 <= 20) SKX_T3(20);
    else SKX_T3(32);
#undef SKX_T3
    k_final_sum<<<1, 1024, 0, s>>>(part, (int)s0, out);
    return check_launch("k_tucker3", 2);
  }
  GenPack g{};
  g.ndim = ndim;
  int64_t cs = 1;
  for (int k = 0; k < ndim; ++k) {
    g.R[k] = ranks_h[k];
    g.A[k] = factors_h[k];
    g.c[k] = coords + (int64_t)k * nnz;
    cs *= ranks_h[k];
  }
  k_tucker_gen<<<kRedBlocks, kRedThreads, 0, s>>>(g, nnz, vals, core, cs, part);
  k_final_sum<<<1, 1024, 0, s>>>(part, kRedBlocks, out);
  return check_launch("k_tucker_gen", 2);
}

extern "C" int skx_cp_cross_coo(int ndim, const int64_t* shape_h, int64_t R, int64_t nnz,
                                const int32_t* coords, const double* vals,
                                const double* const* factors_h, const double* weights, double* out,
                                void* ws, size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(ndim >= 1 && ndim <= 8, "skx_cp_cross_coo: order 1..8");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_cp_cross_coo: ws_bytes is NULL");
  (void)shape_h;
  if (ws == nullptr) {
    *ws_bytes = kRedBlocks * sizeof(double) + 256;
    return SKX_OK;
  }
  cudaStream_t s = (cudaStream_t)stream;
  GenPack g{};
  g.ndim = ndim;
  for (int k = 0; k < ndim; ++k) {
    g.R[k] = R;
    g.A[k] = factors_h[k];
    g.c[k] = coords + (int64_t)k * nnz;
  }
  double* part = (double*)ws;
  k_cp_cross<<<kRedBlocks, kRedThreads, 0, s>>>(g, R, nnz, vals, weights, part);
  k_final_sum<<<1, 1024, 0, s>>>(part, kRedBlocks, out);
  return check_launch("k_cp_cross", 2);
}
