// K5 residual and K7 fitness passes (src/tucker.py:274; src/tensors.py:
// 339-368).  All reductions use a fixed grid and a fixed combination order,
// so results are bitwise reproducible.
#include <cuda.h>
#include <cstdlib>

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

// ---- residual on the FP64 tensor cores.  pred = U Vt is formed 8 x 8 at a
// time by mma.sync m8n8k4 (KS k-steps of 4 over R, zero padded): A fragment =
// 8 rows of U (lane holds U[o0 + lane/4][4ks + lane%4]), B fragment = 8
// columns of Vt (lane holds Vt[4ks + lane%4][x + lane/4]), accumulator lane
// holds pred[o0 + lane/4][x + 2(lane%4) + {0,1}] -- exactly the 16 bytes of
// Y it then loads.  A warp owns 8*NT columns (B fragments stay in registers)
// and walks row groups of 8; a CTA is 4 warps side by side (32*NT columns).
// grid = (ceil(n_in / (32*NT)), n_split).
__device__ __forceinline__ void dmma884r(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int KS, int NT>
__global__ void __launch_bounds__(128) k_resid_mma(const double* __restrict__ U,
                                                   const double* __restrict__ Vt, int64_t n_out,
                                                   int64_t n_in, int R, const double* __restrict__ y,
                                                   int64_t ld, double* __restrict__ part) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, q = lane >> 2, c = lane & 3;
  const int64_t xw = (blockIdx.x * 4 + wid) * (int64_t)(8 * NT);  // first column of the warp
  double b[NT][KS];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int64_t x = xw + nt * 8 + q;
      const int r = ks * 4 + c;
      b[nt][ks] = (x < n_in && r < R) ? __ldg(Vt + (int64_t)r * n_in + x) : 0.0;
    }
  const bool vec = (ld & 1) == 0 && ((reinterpret_cast<uintptr_t>(y) & 15) == 0);
  const int64_t per = (((n_out + gridDim.y - 1) / gridDim.y) + 7) & ~int64_t(7);
  const int64_t oa = imin(blockIdx.y * per, n_out), ob = imin(oa + per, n_out);
  double acc = 0.0;
  for (int64_t o0 = oa; o0 < ob; o0 += 8) {
    const int64_t o = o0 + q;
    const bool rok = o < ob;
    double a[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int r = ks * 4 + c;
      a[ks] = (rok && r < R) ? __ldg(U + o * R + r) : 0.0;
    }
    double yv[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int64_t x = xw + nt * 8 + 2 * c;
      const double* yp = y + o * ld + x;
      if (vec && rok && x + 1 < n_in) {
        const double2 t = __ldcs(reinterpret_cast<const double2*>(yp));
        yv[nt][0] = t.x;
        yv[nt][1] = t.y;
      } else {
        yv[nt][0] = (rok && x < n_in) ? __ldcs(yp) : 0.0;
        yv[nt][1] = (rok && x + 1 < n_in) ? __ldcs(yp + 1) : 0.0;
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) dmma884r(d0, d1, a[ks], b[nt][ks]);
      // padded rows/columns: pred = 0 and y = 0
      const double e0 = d0 - yv[nt][0], e1 = d1 - yv[nt][1];
      acc = fma(e0, e0, acc);
      acc = fma(e1, e1, acc);
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = acc;
}

// sum_{o,x} (sum_r U[o,r] Vt[r,x] - Y[o*ld + x])^2 -- Y's unit-stride index x
// is the inner one.  A CTA takes TO outer rows at a time (their U rows staged in
// shared memory) and sweeps x: the R values Vt[:, x] are loaded once into
// registers and reused for the TO rows, Y is streamed once, coalesced.
// grid = (ceil(n_in / 256), n_split): a thread owns one inner column x for the
// whole kernel (Vt[:, x] lives in registers), the CTA walks its share of outer
// rows TO at a time with their U rows staged in shared memory; the TO Y loads
// per step are independent and coalesced across the warp.
template <int RT, int TO>
__global__ void __launch_bounds__(256) k_resid(const double* __restrict__ U,
                                               const double* __restrict__ Vt, int64_t n_out,
                                               int64_t n_in, int R, const double* __restrict__ y,
                                               int64_t ld, double* __restrict__ part) {
  __shared__ double us[TO * RT];
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool xok = x < n_in;
  const int64_t xc = xok ? x : 0;
  double v[RT];
#pragma unroll
  for (int r = 0; r < RT; ++r) v[r] = (r < R) ? __ldg(Vt + (int64_t)r * n_in + xc) : 0.0;
  const int64_t per = (n_out + gridDim.y - 1) / gridDim.y;
  const int64_t oa = imin(blockIdx.y * per, n_out), ob = imin(oa + per, n_out);
  double acc = 0.0;
  for (int64_t o0 = oa; o0 < ob; o0 += TO) {
    const int nk = (int)imin(TO, ob - o0);
    __syncthreads();
    for (int q = threadIdx.x; q < TO * RT; q += blockDim.x) {
      const int k = q / RT, r = q - k * RT;
      us[q] = (k < nk && r < R) ? U[(o0 + k) * R + r] : 0.0;
    }
    __syncthreads();
    double yv[TO];
#pragma unroll
    for (int k = 0; k < TO; ++k) yv[k] = (k < nk && xok) ? __ldcs(y + (o0 + k) * ld + x) : 0.0;
#pragma unroll
    for (int k = 0; k < TO; ++k) {
      double pred = 0.0;
#pragma unroll
      for (int r = 0; r < RT; ++r) pred = fma(us[k * RT + r], v[r], pred);
      const double d = (k < nk && xok) ? pred - yv[k] : 0.0;
      acc = fma(d, d, acc);
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = acc;
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
// Per lane NP nonzeros at a time: their coordinates, values and full factor
// rows are loaded up front (one latency, many loads in flight), then
// v[r2] = sum_r1 A1[i1,r1] W[r1,r2] runs RT independent FMA chains and
// t = v . A2[i2,:].  W is shared by the NP nonzeros (one LDS per NP FMAs).
// Factor rows are gathered warp-cooperatively into shared memory (consecutive
// lanes read consecutive elements of one row, so a row costs ~3 sectors instead
// of one sector per element per lane), then each lane contracts its own NP
// nonzeros: v[r2] = sum_r1 A1[i1,r1] W[r1,r2] (RT independent FMA chains, W
// read as 16-byte broadcasts shared by the NP nonzeros), t = v . A2[i2,:].
template <int RT, int NP>
__global__ void __launch_bounds__(128) k_tucker3(const int64_t* __restrict__ colptr, int64_t s0,
                                                 const double* __restrict__ rec, uint32_t c1_mask,
                                                 const double* __restrict__ A0,
                                                 const double* __restrict__ A1,
                                                 const double* __restrict__ A2,
                                                 const double* __restrict__ C, int R0, int R1,
                                                 int R2, double* __restrict__ slice_out) {
  static_assert(RT % 2 == 0, "RT must be even");
  constexpr int LD = RT + 1;
  constexpr int PER_WARP = RT * RT + 2 * 32 * NP * LD + 1;
  extern __shared__ double smem[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  double* W = smem + (size_t)wid * (PER_WARP + 1);  // 16-byte aligned (PER_WARP + 1 even)
  double* S1 = W + RT * RT;
  double* S2 = S1 + 32 * NP * LD;
  for (int64_t i0 = blockIdx.x * (int64_t)nw + wid; i0 < s0; i0 += (int64_t)gridDim.x * nw) {
    const int64_t e0 = colptr[i0], e1 = colptr[i0 + 1];
    if (e0 == e1) {
      if (lane == 0) slice_out[i0] = 0.0;
      continue;
    }
    for (int q = lane; q < RT * RT; q += 32) {
      const int r1 = q / RT, r2 = q - r1 * RT;
      double s = 0.0;
      if (r1 < R1 && r2 < R2)
        for (int r0 = 0; r0 < R0; ++r0)
          s = fma(A0[i0 * R0 + r0], C[((int64_t)r0 * R1 + r1) * R2 + r2], s);
      W[q] = s;
    }
    __syncwarp();
    double acc = 0.0;
    for (int64_t base = e0; base < e1; base += 32 * NP) {
      int i1[NP], i2[NP];
      double x[NP];
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        const int64_t e = base + 32 * u + lane;
        const bool ok = e < e1;
        int32_t c[4];
        double xv;
        load_rec<2>(rec, ok ? e : e0, c, xv);
        i1[u] = c[0];
        i2[u] = (int)((uint32_t)c[1] & c1_mask);
        x[u] = ok ? xv : 0.0;
      }
#pragma unroll
      for (int u = 0; u < NP; ++u) {
#pragma unroll
        for (int t = 0; t < RT; ++t) {
          const int q = t * 32 + lane, j = q / RT, c = q - j * RT;
          const int r1 = __shfl_sync(0xffffffffu, i1[u], j);
          const int r2 = __shfl_sync(0xffffffffu, i2[u], j);
          S1[(u * 32 + j) * LD + c] = c < R1 ? __ldg(A1 + (int64_t)r1 * R1 + c) : 0.0;
          S2[(u * 32 + j) * LD + c] = c < R2 ? __ldg(A2 + (int64_t)r2 * R2 + c) : 0.0;
        }
      }
      __syncwarp();
      double v[NP][RT];
#pragma unroll
      for (int u = 0; u < NP; ++u)
#pragma unroll
        for (int r = 0; r < RT; ++r) v[u][r] = 0.0;
#pragma unroll
      for (int r1 = 0; r1 < RT; ++r1) {
        double a[NP];
#pragma unroll
        for (int u = 0; u < NP; ++u) a[u] = S1[(u * 32 + lane) * LD + r1];
        const double2* wr = reinterpret_cast<const double2*>(W + r1 * RT);
#pragma unroll
        for (int r2 = 0; r2 < RT; r2 += 2) {
          const double2 wv = wr[r2 / 2];
#pragma unroll
          for (int u = 0; u < NP; ++u) {
            v[u][r2] = fma(a[u], wv.x, v[u][r2]);
            v[u][r2 + 1] = fma(a[u], wv.y, v[u][r2 + 1]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        double t = 0.0;
#pragma unroll
        for (int r2 = 0; r2 < RT; ++r2) t = fma(v[u][r2], S2[(u * 32 + lane) * LD + r2], t);
        acc = fma(x[u], t, acc);
      }
      __syncwarp();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane == 0) slice_out[i0] = acc;
    __syncwarp();
  }
}

// ---- same contraction on the FP64 tensor cores (mma.sync m8n8k4 f64).
// Warp per slice i0.  W = A0[i0,:] x_0 C (R1 x R2) lives in registers as the
// B fragments (KS k-steps of 4 x NT n-tiles of 8, zero padded).  Nonzeros go
// 8 at a time: row q of the A fragment is nonzero e = base + q (lanes 4q..4q+3
// load the same 16-byte record, a broadcast), so V = A1[i1_e,:] W is one
// 8 x 8*NT tile after KS*NT DMMAs, and each lane folds its two columns per
// n-tile with A2[i2_e, cols] and v_e into a private sum.  No shared memory:
// factor rows come straight from L2 in 32-byte pieces.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int G>
struct T3Rec {
  int32_t i1[G], i2[G];
  double v[G];
};
template <int KS, int NT, int G>
struct T3Rows {
  double a[G][KS], y[G][NT][2], v[G];
};

// Three-stage software pipeline per warp: records of step s+2 (L2, after the
// slice prefetch), factor rows of step s+1, DMMAs of step s.  The buffers
// rotate by static index (body unrolled lcm(3, 2) = 6 times) so nothing is
// copied while its load is in flight.  R1T/R2T > 0 fix the ranks at compile
// time (predicates fold away); 0 reads them at run time.
// PAIR (R1 even, fixed at compile time): the A-fragment k index is permuted
// so each lane reads 16 bytes per pair of k-steps -- k-step 2j holds
// k = 8j + 2c, 2j + 1 holds 8j + 2c + 1, a last odd k-step k = 8 (KS/2) + c;
// the B fragments use the same map (the contraction over k is unchanged).
// Fewer, wider loads: 3 instead of 5 per row group at R = 20.
template <int KS, int NT, int G, int R1T, int R2T, int MB = 1, bool PAIR = false>
__global__ void __launch_bounds__(256, MB) k_tucker3_mma(const int64_t* __restrict__ colptr, int64_t s0,
                                                     const double* __restrict__ rec, uint32_t c1_mask,
                                                     const double* __restrict__ A0,
                                                     const double* __restrict__ A1,
                                                     const double* __restrict__ A2,
                                                     const double* __restrict__ C, int R0, int R1_,
                                                     int R2_, double* __restrict__ slice_out) {
  const int R1 = R1T > 0 ? R1T : R1_, R2 = R2T > 0 ? R2T : R2_;
  const int lane = threadIdx.x & 31, q = lane >> 2, c = lane & 3;
  const int64_t nw = blockDim.x >> 5, stride = (int64_t)gridDim.x * nw;
  const bool vec2 = (R2 & 1) == 0;  // A2 rows 16-byte aligned: pairs load as one LDG.128
  constexpr int STEP = 8 * G;
  auto prefetch_slice = [&](int64_t j) {  // the records of slice j into L2
    if (j >= s0) return;
    const int64_t l0 = colptr[j] * 16 / 128, l1 = (colptr[j + 1] * 16 + 127) / 128;
    for (int64_t l = l0 + lane; l < l1; l += 32)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(rec) + l * 128));
  };
  int64_t i0 = blockIdx.x * nw + (threadIdx.x >> 5);
  prefetch_slice(i0);
  for (; i0 < s0; i0 += stride) {
    prefetch_slice(i0 + stride);
    const int64_t e0 = colptr[i0], e1 = colptr[i0 + 1];
    if (e0 == e1) {
      if (lane == 0) slice_out[i0] = 0.0;
      continue;
    }
    double b[KS][NT];  // B[k][n] = W[ks*4 + c][nt*8 + q]
    constexpr int PAIRS = PAIR ? KS / 2 : 0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int k = !PAIR ? ks * 4 + c
                            : (ks < 2 * PAIRS ? 8 * (ks >> 1) + 2 * c + (ks & 1) : 8 * PAIRS + c);
        const int n = nt * 8 + q;
        double w = 0.0;
        if (k < R1 && n < R2)
          for (int r0 = 0; r0 < R0; ++r0)
            w = fma(__ldg(A0 + i0 * R0 + r0), __ldg(C + ((int64_t)r0 * R1 + k) * R2 + n), w);
        b[ks][nt] = w;
      }
    auto load_recs = [&](int64_t base, T3Rec<G>& r) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int64_t e = base + g * 8 + q;
        const bool ok = e < e1;
        int32_t cc[4];
        double xv;
        load_rec<2>(rec, ok ? e : e0, cc, xv);
        r.i1[g] = cc[0];
        r.i2[g] = (int32_t)((uint32_t)cc[1] & c1_mask);
        r.v[g] = ok ? xv : 0.0;
      }
    };
    auto load_rows = [&](const T3Rec<G>& r, T3Rows<KS, NT, G>& w) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const double* r1 = A1 + (int64_t)r.i1[g] * R1;
        const double* r2 = A2 + (int64_t)r.i2[g] * R2;
        w.v[g] = r.v[g];
        if (PAIR) {
#pragma unroll
          for (int j = 0; j < PAIRS; ++j) {
            const int k = 8 * j + 2 * c;
            const double2 p = k < R1 ? __ldg(reinterpret_cast<const double2*>(r1 + k))
                                     : make_double2(0.0, 0.0);
            w.a[g][2 * j] = p.x;
            w.a[g][2 * j + 1] = p.y;
          }
          if (KS & 1) w.a[g][KS - 1] = 8 * PAIRS + c < R1 ? __ldg(r1 + 8 * PAIRS + c) : 0.0;
        } else {
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) w.a[g][ks] = ks * 4 + c < R1 ? __ldg(r1 + ks * 4 + c) : 0.0;
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int n = nt * 8 + 2 * c;
          if (vec2) {
            const double2 p = n < R2 ? __ldg(reinterpret_cast<const double2*>(r2 + n))
                                     : make_double2(0.0, 0.0);
            w.y[g][nt][0] = p.x;
            w.y[g][nt][1] = p.y;
          } else {
            w.y[g][nt][0] = n < R2 ? __ldg(r2 + n) : 0.0;
            w.y[g][nt][1] = n + 1 < R2 ? __ldg(r2 + n + 1) : 0.0;
          }
        }
      }
    };
    double acc = 0.0;
    auto compute = [&](const T3Rows<KS, NT, G>& w) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        double t = 0.0;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) dmma884(d0, d1, w.a[g][ks], b[ks][nt]);
          t = fma(d0, w.y[g][nt][0], t);
          t = fma(d1, w.y[g][nt][1], t);
        }
        acc = fma(w.v[g], t, acc);
      }
    };
    T3Rec<G> rr[3];
    T3Rows<KS, NT, G> ww[2];
    load_recs(e0, rr[0]);
    load_recs(e0 + STEP, rr[1]);
    load_rows(rr[0], ww[0]);
    for (int64_t base = e0; base < e1; base += 6 * STEP) {
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const int64_t sb = base + s * STEP;
        if (sb >= e1) break;
        load_recs(sb + 2 * STEP, rr[(s + 2) % 3]);
        load_rows(rr[(s + 1) % 3], ww[(s + 1) % 2]);
        compute(ww[s % 2]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) slice_out[i0] = acc;
  }
}

// ---- K7 with the factor rows staged through shared memory by cp.async ----
// Same contraction as k_tucker3_mma (warp per slice, W = A0[i0,:] x_0 C in
// registers as B fragments, 8 nonzeros per m8n8k4 tile), but the random
// factor rows are gathered whole: R/2 lanes copy one 160-byte row (R = 20) in
// 16-byte cp.async pieces, 32/(R/2) rows per instruction, straight into a
// per-warp shared-memory tile (no register writeback, several batches in
// flight per SM); the DMMA fragments are then read from shared memory
// (row stride = 8 mod 16 doubles: conflict-free 16-byte fragment reads).
// Measured on B200 (tools/micro/gather.cu): whole-row 16-byte gathers move
// ~106 G rows/s, the fragment-shaped 8-byte gathers of k_tucker3_mma ~55.
// The k index of the A fragment is permuted so that each lane reads 16 bytes
// per k-step pair: k-step 2j holds k = 8j + 2c, 2j + 1 holds 8j + 2c + 1
// (c = lane % 4); B is built with the same map, so the contraction is
// unchanged.  Pipeline per warp: records of batch b+2 and rows of batch b+1
// in flight while batch b is contracted.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16_ca(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16_cg_zfill(uint32_t dst, const void* src, uint32_t n) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int R>
struct T3A {
  static constexpr int KS = (R + 3) / 4, PAIRS = KS / 2, SINGLE = KS % 2;
  static constexpr int NT = (R + 7) / 8;
  static constexpr int W1 = 8 * PAIRS + 4 * SINGLE, W2 = 8 * NT;
  static constexpr int WM = W1 > W2 ? W1 : W2;
  static constexpr int ST = ((WM + 7) / 16) * 16 + 8;  // >= WM, = 8 (mod 16) doubles
  static constexpr int LPR = R / 2;                     // 16-byte chunks per row
  static constexpr int RPI = 32 / LPR;                  // rows per copy instruction
};

// D = row lookahead (batches): rows of batch b+D and records of batch b+D+2
// are in flight while batch b is contracted (D+1 row buffers, D+3 record
// buffers per warp).
template <int R, int NB, int MB, int D>
__global__ void __launch_bounds__(256, MB) k_tucker3_async(
    const int64_t* __restrict__ colptr, int64_t s0, const double* __restrict__ rec, uint32_t c1_mask,
    const double* __restrict__ A0, const double* __restrict__ A1, const double* __restrict__ A2,
    const double* __restrict__ C, int R0, double* __restrict__ slice_out) {
  using P = T3A<R>;
  constexpr int NROWS = 2 * NB;
  constexpr int NINSTR = (NROWS + P::RPI - 1) / P::RPI;
  constexpr int ROWBUF = NROWS * P::ST;  // doubles per row buffer
  constexpr int NRB = D + 1, NRC = D + 3;
  extern __shared__ __align__(16) double t3sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, q = lane >> 2, c = lane & 3;
  double* rows = t3sm + (size_t)wid * (NRB * ROWBUF + NRC * NB * 2);
  double* recs = rows + NRB * ROWBUF;  // NRC buffers x NB records of 2 doubles
  for (int e = lane; e < NRB * ROWBUF; e += 32) rows[e] = 0.0;  // zero padding beyond R
  __syncwarp();
  const int64_t nw = blockDim.x >> 5, stride = (int64_t)gridDim.x * nw;
  const int cr = lane / P::LPR, ch = lane % P::LPR;  // copy role: row in instruction, chunk
  for (int64_t i0 = blockIdx.x * nw + wid; i0 < s0; i0 += stride) {
    {  // the next slice's records into L2
      const int64_t j = i0 + stride;
      if (j < s0) {
        const int64_t l0 = colptr[j] * 16 / 128, l1 = (colptr[j + 1] * 16 + 127) / 128;
        for (int64_t l = l0 + lane; l < l1; l += 32)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(rec) + l * 128));
      }
    }
    const int64_t e0 = colptr[i0], e1 = colptr[i0 + 1];
    if (e0 == e1) {
      if (lane == 0) slice_out[i0] = 0.0;
      continue;
    }
    const int64_t nb = (e1 - e0 + NB - 1) / NB;
    auto issue_recs = [&](int64_t b) {
      if (lane < NB) {
        const int64_t e = e0 + b * NB + lane;
        cp_async16_cg_zfill(smem_addr(recs + ((b % NRC) * NB + lane) * 2),
                            rec + 2 * (e < e1 ? e : e0), e < e1 ? 16u : 0u);
      }
    };
    auto issue_rows = [&](int64_t b) {
      const double* rb = recs + (b % NRC) * NB * 2;
      double* dst = rows + (b % NRB) * ROWBUF;
#pragma unroll
      for (int t = 0; t < NINSTR; ++t) {
        const int r = t * P::RPI + cr;
        if (cr < P::RPI && r < NROWS) {
          const bool second = r >= NB;
          const int nz = second ? r - NB : r;
          const uint32_t w = reinterpret_cast<const uint32_t*>(rb + nz * 2)[second ? 1 : 0];
          const uint32_t idx = second ? (w & c1_mask) : w;
          const double* src = (second ? A2 : A1) + (int64_t)idx * R + 2 * ch;
          cp_async16_ca(smem_addr(dst + r * P::ST + 2 * ch), src);
        }
      }
    };
    // B fragments: W[k][n] with the permuted k map
    double b[P::KS][P::NT];
#pragma unroll
    for (int ks = 0; ks < P::KS; ++ks)
#pragma unroll
      for (int nt = 0; nt < P::NT; ++nt) {
        const int k = ks < 2 * P::PAIRS ? 8 * (ks >> 1) + 2 * c + (ks & 1) : 8 * P::PAIRS + c;
        const int n = nt * 8 + q;
        double w = 0.0;
        if (k < R && n < R)
          for (int r0 = 0; r0 < R0; ++r0)
            w = fma(__ldg(A0 + i0 * R0 + r0), __ldg(C + ((int64_t)r0 * R + k) * R + n), w);
        b[ks][nt] = w;
      }
    // prologue: records of batches 0..D+1, then rows of batches 0..D-1
    for (int64_t b2 = 0; b2 < D + 2 && b2 < nb; ++b2) issue_recs(b2);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    for (int64_t b2 = 0; b2 < D && b2 < nb; ++b2) issue_rows(b2);
    cp_async_commit();
    double acc = 0.0;
    for (int64_t bi = 0; bi < nb; ++bi) {
      // rows(bi) were committed D groups ago and records(bi + D) two groups
      // ago (or in the prologue): with D >= 2 only the newest group may stay
      // in flight; with D = 1 rows(bi) are the newest group themselves
      if (bi == 0 || D < 2) cp_async_wait<0>();
      else cp_async_wait<1>();
      __syncwarp();
      if (bi + D < nb) issue_rows(bi + D);
      if (bi + D + 2 < nb) issue_recs(bi + D + 2);
      cp_async_commit();
      const double* rw = rows + (bi % NRB) * ROWBUF;
      const double* rv = recs + (bi % NRC) * NB * 2;
      constexpr int NG = NB / 8;
      // fragments of every group first, then the DMMAs k-step by k-step over
      // all (group, n-tile) accumulators: NG * NT independent chains
      double a[NG][P::KS], d[NG][P::NT][2];
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const double* ra = rw + (g * 8 + q) * P::ST;
#pragma unroll
        for (int j = 0; j < P::PAIRS; ++j) {
          const double2 p2 = *reinterpret_cast<const double2*>(ra + 8 * j + 2 * c);
          a[g][2 * j] = p2.x;
          a[g][2 * j + 1] = p2.y;
        }
        if (P::SINGLE) a[g][P::KS - 1] = ra[8 * P::PAIRS + c];
#pragma unroll
        for (int nt = 0; nt < P::NT; ++nt) d[g][nt][0] = d[g][nt][1] = 0.0;
      }
#pragma unroll
      for (int ks = 0; ks < P::KS; ++ks)
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
          for (int nt = 0; nt < P::NT; ++nt) dmma884(d[g][nt][0], d[g][nt][1], a[g][ks], b[ks][nt]);
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const double* ry = rw + (NB + g * 8 + q) * P::ST;
        double t = 0.0;
#pragma unroll
        for (int nt = 0; nt < P::NT; ++nt) {
          // the last n-tile of R = 20 holds 4 real columns: lanes c >= 2 read padding
          const bool live = nt * 8 + 2 * c < R;
          const double2 y = live ? *reinterpret_cast<const double2*>(ry + 8 * nt + 2 * c)
                                 : make_double2(0.0, 0.0);
          t = fma(d[g][nt][0], y.x, t);
          t = fma(d[g][nt][1], y.y, t);
        }
        acc = fma(rv[(g * 8 + q) * 2 + 1], t, acc);
      }
    }
    cp_async_wait<0>();
    __syncwarp();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) slice_out[i0] = acc;
  }
}

// R = 20 with the mode-2 factor rows brought in by the TMA unit
// (cp.async.bulk.tensor tile::gather4, four rows per instruction) while the
// mode-1 rows keep the 16-byte cp.async path: the two gathers then load
// different units (TMA engine vs the LSU/L1 data pipe, which the cp.async
// row copies plus the fragment reads saturate in k_tucker3_async).  The
// tensor map's box is 24 columns wide over a 20-column factor, so the four
// padding columns arrive as TMA out-of-bounds zeros: rows land at the
// conflict-free stride of 24 doubles and the last n-tile needs no masking.
// Completion of a batch's TMA rows is tracked by one mbarrier per row
// buffer (expect_tx = NB rows x 192 bytes).
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* tm, uint64_t* bar,
                                            int32_t col, int32_t r0, int32_t r1, int32_t r2,
                                            int32_t r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
      "l"(tm), "r"(smem_addr(bar)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}

constexpr int kT3tR = 20, kT3tST = 24;  // rank, smem row stride (doubles)

// LEFT: the fourth-from-last n columns of W (16..19, which a third 8-wide
// n-tile would pad to 24) go to the FP64 FMA pipe instead: each lane forms the
// partial products of its own five A-fragment k values with W[k][16..19] and
// dots them with a1[16..19]; the per-lane partials sum to the full term in
// the warp reduction at the end of the slice.  The FP64 pipe (shared by DMMA
// and DFMA) then does 10 DMMA + 29 DFMA per 8 nonzeros instead of 15 + 7:
// ~14% fewer issue slots, no padded work.
template <int NB, int MB, int D, bool LEFT = false>
__global__ void __launch_bounds__(256, MB) k_tucker3_tma(
    const __grid_constant__ CUtensorMap tmC, const int64_t* __restrict__ colptr, int64_t s0,
    const double* __restrict__ rec, uint32_t c1_mask, const double* __restrict__ A0,
    const double* __restrict__ A1, const double* __restrict__ C, int R0,
    double* __restrict__ slice_out) {
  constexpr int R = kT3tR, ST = kT3tST;
  using P = T3A<R>;
  static_assert(P::ST == ST, "row stride");
  constexpr int NINSTR = (NB + P::RPI - 1) / P::RPI;
  constexpr int ROWBUF = NB * ST;  // doubles per row buffer (one operand)
  constexpr int NRB = D + 1, NRC = D + 3;
  constexpr uint32_t TX = NB * ST * 8;
  extern __shared__ __align__(128) double t3sm[];
  __shared__ __align__(8) uint64_t bars[8][NRB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, q = lane >> 2, c = lane & 3;
  // per warp: [NRB][NB][ST] TMA rows (C), [NRB][NB][ST] cp.async rows (A1), [NRC][NB][2] records
  double* rowsC = t3sm + (size_t)wid * (2 * NRB * ROWBUF + NRC * NB * 2);
  double* rowsA = rowsC + NRB * ROWBUF;
  double* recs = rowsA + NRB * ROWBUF;
  for (int e = lane; e < NRB * ROWBUF; e += 32) rowsA[e] = 0.0;  // zero padding beyond R
  if (lane == 0)
    for (int b = 0; b < NRB; ++b) mbar_init(&bars[wid][b], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  uint32_t phase = 0;  // bit b: parity of row buffer b's next completion
  const int64_t nw = blockDim.x >> 5, stride = (int64_t)gridDim.x * nw;
  const int cr = lane / P::LPR, ch = lane % P::LPR;
  for (int64_t i0 = blockIdx.x * nw + wid; i0 < s0; i0 += stride) {
    {  // the next slice's records into L2
      const int64_t j = i0 + stride;
      if (j < s0) {
        const int64_t l0 = colptr[j] * 16 / 128, l1 = (colptr[j + 1] * 16 + 127) / 128;
        for (int64_t l = l0 + lane; l < l1; l += 32)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(rec) + l * 128));
      }
    }
    const int64_t e0 = colptr[i0], e1 = colptr[i0 + 1];
    if (e0 == e1) {
      if (lane == 0) slice_out[i0] = 0.0;
      continue;
    }
    const int64_t nb = (e1 - e0 + NB - 1) / NB;
    auto issue_recs = [&](int64_t b) {
      if (lane < NB) {
        const int64_t e = e0 + b * NB + lane;
        cp_async16_cg_zfill(smem_addr(recs + ((b % NRC) * NB + lane) * 2),
                            rec + 2 * (e < e1 ? e : e0), e < e1 ? 16u : 0u);
      }
    };
    auto issue_rows = [&](int64_t b) {
      const int slot = (int)(b % NRB);
      const uint32_t* rb = reinterpret_cast<const uint32_t*>(recs + (b % NRC) * NB * 2);
      // mode-2 rows: one gather4 per four records (padding records are zero:
      // row 0, contributing nothing)
      // order this warp's earlier generic reads of the buffer before the
      // async-proxy writes into it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (lane == 0) mbar_expect_tx(&bars[wid][slot], TX);
      __syncwarp();
      if (lane < NB / 4) {
        const int32_t i0_ = (int32_t)(rb[(4 * lane + 0) * 4 + 1] & c1_mask);
        const int32_t i1_ = (int32_t)(rb[(4 * lane + 1) * 4 + 1] & c1_mask);
        const int32_t i2_ = (int32_t)(rb[(4 * lane + 2) * 4 + 1] & c1_mask);
        const int32_t i3_ = (int32_t)(rb[(4 * lane + 3) * 4 + 1] & c1_mask);
        tma_gather4(smem_addr(rowsC + slot * ROWBUF + 4 * lane * ST), &tmC, &bars[wid][slot], 0,
                    i0_, i1_, i2_, i3_);
      }
      // mode-1 rows: R/2 lanes per row, 16-byte cp.async pieces
      double* dst = rowsA + slot * ROWBUF;
#pragma unroll
      for (int t = 0; t < NINSTR; ++t) {
        const int r = t * P::RPI + cr;
        if (cr < P::RPI && r < NB) {
          const uint32_t idx = rb[r * 4];
          cp_async16_ca(smem_addr(dst + r * ST + 2 * ch), A1 + (int64_t)idx * R + 2 * ch);
        }
      }
    };
    constexpr int NTD = LEFT ? 2 : P::NT;  // n-tiles on the tensor cores
    double b[P::KS][NTD];
#pragma unroll
    for (int ks = 0; ks < P::KS; ++ks)
#pragma unroll
      for (int nt = 0; nt < NTD; ++nt) {
        const int k = ks < 2 * P::PAIRS ? 8 * (ks >> 1) + 2 * c + (ks & 1) : 8 * P::PAIRS + c;
        const int n = nt * 8 + q;
        double w = 0.0;
        if (k < R && n < R)
          for (int r0 = 0; r0 < R0; ++r0)
            w = fma(__ldg(A0 + i0 * R0 + r0), __ldg(C + ((int64_t)r0 * R + k) * R + n), w);
        b[ks][nt] = w;
      }
    double wl[LEFT ? P::KS : 1][4];  // W[k(ks, c)][16 + j]
    if (LEFT) {
#pragma unroll
      for (int ks = 0; ks < P::KS; ++ks)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = ks < 2 * P::PAIRS ? 8 * (ks >> 1) + 2 * c + (ks & 1) : 8 * P::PAIRS + c;
          double w = 0.0;
          for (int r0 = 0; r0 < R0; ++r0)
            w = fma(__ldg(A0 + i0 * R0 + r0), __ldg(C + ((int64_t)r0 * R + k) * R + 16 + j), w);
          wl[LEFT ? ks : 0][j] = w;
        }
    }
    for (int64_t b2 = 0; b2 < D + 2 && b2 < nb; ++b2) issue_recs(b2);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    for (int64_t b2 = 0; b2 < D && b2 < nb; ++b2) issue_rows(b2);
    cp_async_commit();
    double acc = 0.0;
    for (int64_t bi = 0; bi < nb; ++bi) {
      if (bi == 0 || D < 2) cp_async_wait<0>();
      else cp_async_wait<1>();
      const int slot = (int)(bi % NRB);
      mbar_wait(&bars[wid][slot], (phase >> slot) & 1u);
      phase ^= 1u << slot;
      __syncwarp();
      if (bi + D < nb) issue_rows(bi + D);
      if (bi + D + 2 < nb) issue_recs(bi + D + 2);
      cp_async_commit();
      const double* ra0 = rowsA + slot * ROWBUF;
      const double* ry0 = rowsC + slot * ROWBUF;
      const double* rv = recs + (bi % NRC) * NB * 2;
      constexpr int NG = NB / 8;
      double a[NG][P::KS], d[NG][NTD][2];
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const double* ra = ra0 + (g * 8 + q) * ST;
#pragma unroll
        for (int j = 0; j < P::PAIRS; ++j) {
          const double2 p2 = *reinterpret_cast<const double2*>(ra + 8 * j + 2 * c);
          a[g][2 * j] = p2.x;
          a[g][2 * j + 1] = p2.y;
        }
        if (P::SINGLE) a[g][P::KS - 1] = ra[8 * P::PAIRS + c];
#pragma unroll
        for (int nt = 0; nt < NTD; ++nt) d[g][nt][0] = d[g][nt][1] = 0.0;
      }
#pragma unroll
      for (int ks = 0; ks < P::KS; ++ks)
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
          for (int nt = 0; nt < NTD; ++nt) dmma884(d[g][nt][0], d[g][nt][1], a[g][ks], b[ks][nt]);
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const double* ry = ry0 + (g * 8 + q) * ST;
        double t = 0.0;
        if (LEFT) {  // columns 16..19 on the FMA pipe: this lane's k values only
          double pl[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            double v = 0.0;
#pragma unroll
            for (int ks = 0; ks < P::KS; ++ks) v = fma(a[g][ks], wl[LEFT ? ks : 0][j], v);
            pl[j] = v;
          }
          const double2 y0 = *reinterpret_cast<const double2*>(ry + 16);
          const double2 y1 = *reinterpret_cast<const double2*>(ry + 18);
          t = fma(pl[0], y0.x, t);
          t = fma(pl[1], y0.y, t);
          t = fma(pl[2], y1.x, t);
          t = fma(pl[3], y1.y, t);
        }
#pragma unroll
        for (int nt = 0; nt < NTD; ++nt) {  // (without LEFT: columns 20..23 are TMA zero fill)
          const double2 y = *reinterpret_cast<const double2*>(ry + 8 * nt + 2 * c);
          t = fma(d[g][nt][0], y.x, t);
          t = fma(d[g][nt][1], y.y, t);
        }
        acc = fma(rv[(g * 8 + q) * 2 + 1], t, acc);
      }
    }
    cp_async_wait<0>();
    __syncwarp();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) slice_out[i0] = acc;
  }
}

template <int NB, int D>
constexpr size_t t3t_smem_bytes() {
  return (size_t)8 * (2 * (D + 1) * NB * kT3tST + (D + 3) * NB * 2) * 8;
}

// R = 20, variant 2: the mode-2 rows (the DMMA A operand) by TMA gather4 into
// shared memory as in k_tucker3_tma, but the mode-1 rows -- needed only in
// the epilogue dot t = sum_n T[e][n] a1_e[n] -- go straight from L2 into
// registers in the D-fragment layout (lane (q, c): a1_q[8 nt + 2c, +1], three
// 16-byte loads, the last for c < 2 only), issued one batch ahead.  No
// cp.async row copies and no shared-memory reads of those rows: the L1 data
// pipe (the binding unit of k_tucker3_tma: ~4.6e9 cp.async + 1e9 fragment
// wavefronts per 1e9 nonzeros) only serves the TMA rows' fragments and the
// records.  tools/micro/gather.cu: register-fragment 16-byte gathers run at
// ~72 G rows/s against ~106 for whole-row copies, but they skip the
// shared-memory write and read entirely.
template <int NB, int MB, int D, bool LEFT = false>
__global__ void __launch_bounds__(256, MB) k_tucker3_tma2(
    const __grid_constant__ CUtensorMap tmC, const int64_t* __restrict__ colptr, int64_t s0,
    const double* __restrict__ rec, uint32_t c1_mask, const double* __restrict__ A0,
    const double* __restrict__ A2, const double* __restrict__ C, int R0,
    double* __restrict__ slice_out) {
  constexpr int R = kT3tR, ST = kT3tST;
  using P = T3A<R>;
  constexpr int ROWBUF = NB * ST;  // doubles per row buffer
  constexpr int NRB = D + 1, NRC = D + 3;
  constexpr uint32_t TX = NB * ST * 8;
  constexpr int NG = NB / 8;
  extern __shared__ __align__(128) double t3sm[];
  __shared__ __align__(8) uint64_t bars[8][NRB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, q = lane >> 2, c = lane & 3;
  double* rowsC = t3sm + (size_t)wid * (NRB * ROWBUF + NRC * NB * 2);
  double* recs = rowsC + NRB * ROWBUF;
  if (lane == 0)
    for (int b = 0; b < NRB; ++b) mbar_init(&bars[wid][b], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  uint32_t phase = 0;
  const int64_t nw = blockDim.x >> 5, stride = (int64_t)gridDim.x * nw;
  for (int64_t i0 = blockIdx.x * nw + wid; i0 < s0; i0 += stride) {
    {  // the next slice's records into L2
      const int64_t j = i0 + stride;
      if (j < s0) {
        const int64_t l0 = colptr[j] * 16 / 128, l1 = (colptr[j + 1] * 16 + 127) / 128;
        for (int64_t l = l0 + lane; l < l1; l += 32)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(rec) + l * 128));
      }
    }
    const int64_t e0 = colptr[i0], e1 = colptr[i0 + 1];
    if (e0 == e1) {
      if (lane == 0) slice_out[i0] = 0.0;
      continue;
    }
    const int64_t nb = (e1 - e0 + NB - 1) / NB;
    auto issue_recs = [&](int64_t b) {
      if (lane < NB) {
        const int64_t e = e0 + b * NB + lane;
        cp_async16_cg_zfill(smem_addr(recs + ((b % NRC) * NB + lane) * 2),
                            rec + 2 * (e < e1 ? e : e0), e < e1 ? 16u : 0u);
      }
    };
    auto issue_rows = [&](int64_t b) {  // mode-1 rows (tmC maps A1): TMA, one gather4 per four records
      const int slot = (int)(b % NRB);
      const uint32_t* rb = reinterpret_cast<const uint32_t*>(recs + (b % NRC) * NB * 2);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (lane == 0) mbar_expect_tx(&bars[wid][slot], TX);
      __syncwarp();
      if (lane < NB / 4) {
        const int32_t i0_ = (int32_t)rb[(4 * lane + 0) * 4];
        const int32_t i1_ = (int32_t)rb[(4 * lane + 1) * 4];
        const int32_t i2_ = (int32_t)rb[(4 * lane + 2) * 4];
        const int32_t i3_ = (int32_t)rb[(4 * lane + 3) * 4];
        tma_gather4(smem_addr(rowsC + slot * ROWBUF + 4 * lane * ST), &tmC, &bars[wid][slot], 0,
                    i0_, i1_, i2_, i3_);
      }
    };
    // mode-2 rows of batch b straight into D-fragment registers
    constexpr int NTD = LEFT ? 2 : P::NT;  // n-tiles on the tensor cores
    double2 y[NG][LEFT ? 4 : P::NT];
    auto load_y = [&](int64_t b) {
      const uint32_t* rb = reinterpret_cast<const uint32_t*>(recs + (b % NRC) * NB * 2);
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const double2* row =
            reinterpret_cast<const double2*>(A2 + (int64_t)(rb[(g * 8 + q) * 4 + 1] & c1_mask) * R);
        if (LEFT) {  // D-fragment columns of the two DMMA n-tiles + all of cols 16..19
          y[g][0] = __ldg(row + c);
          y[g][1] = __ldg(row + 4 + c);
          y[g][2] = __ldg(row + 8);
          y[g][LEFT ? 3 : 0] = __ldg(row + 9);
        } else {
#pragma unroll
          for (int nt = 0; nt < P::NT; ++nt)
            y[g][nt] = (nt * 8 + 2 * c < R) ? __ldg(row + nt * 4 + c) : make_double2(0.0, 0.0);
        }
      }
    };
    double b[P::KS][NTD];
#pragma unroll
    for (int ks = 0; ks < P::KS; ++ks)
#pragma unroll
      for (int nt = 0; nt < NTD; ++nt) {
        const int k = ks < 2 * P::PAIRS ? 8 * (ks >> 1) + 2 * c + (ks & 1) : 8 * P::PAIRS + c;
        const int n = nt * 8 + q;
        double w = 0.0;
        if (k < R && n < R)
          for (int r0 = 0; r0 < R0; ++r0)
            w = fma(__ldg(A0 + i0 * R0 + r0), __ldg(C + ((int64_t)r0 * R + k) * R + n), w);
        b[ks][nt] = w;
      }
    double wl[LEFT ? P::KS : 1][4];  // W[k(ks, c)][16 + j]
    if (LEFT) {
#pragma unroll
      for (int ks = 0; ks < P::KS; ++ks)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = ks < 2 * P::PAIRS ? 8 * (ks >> 1) + 2 * c + (ks & 1) : 8 * P::PAIRS + c;
          double w = 0.0;
          for (int r0 = 0; r0 < R0; ++r0)
            w = fma(__ldg(A0 + i0 * R0 + r0), __ldg(C + ((int64_t)r0 * R + k) * R + 16 + j), w);
          wl[LEFT ? ks : 0][j] = w;
        }
    }
    for (int64_t b2 = 0; b2 < D + 2 && b2 < nb; ++b2) issue_recs(b2);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    for (int64_t b2 = 0; b2 < D && b2 < nb; ++b2) issue_rows(b2);
    load_y(0);
    double acc = 0.0;
    for (int64_t bi = 0; bi < nb; ++bi) {
      cp_async_wait<0>();  // records of bi + 1 .. bi + D + 1
      const int slot = (int)(bi % NRB);
      mbar_wait(&bars[wid][slot], (phase >> slot) & 1u);
      phase ^= 1u << slot;
      __syncwarp();
      if (bi + D < nb) issue_rows(bi + D);
      if (bi + D + 2 < nb) issue_recs(bi + D + 2);
      cp_async_commit();
      const double* ra0 = rowsC + slot * ROWBUF;
      const double* rv = recs + (bi % NRC) * NB * 2;
      double a[NG][P::KS], d[NG][NTD][2];
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const double* ra = ra0 + (g * 8 + q) * ST;
#pragma unroll
        for (int j = 0; j < P::PAIRS; ++j) {
          const double2 p2 = *reinterpret_cast<const double2*>(ra + 8 * j + 2 * c);
          a[g][2 * j] = p2.x;
          a[g][2 * j + 1] = p2.y;
        }
        if (P::SINGLE) a[g][P::KS - 1] = ra[8 * P::PAIRS + c];
#pragma unroll
        for (int nt = 0; nt < NTD; ++nt) d[g][nt][0] = d[g][nt][1] = 0.0;
      }
      double vq[NG];
#pragma unroll
      for (int g = 0; g < NG; ++g) vq[g] = rv[(g * 8 + q) * 2 + 1];
#pragma unroll
      for (int ks = 0; ks < P::KS; ++ks)
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
          for (int nt = 0; nt < NTD; ++nt) dmma884(d[g][nt][0], d[g][nt][1], a[g][ks], b[ks][nt]);
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        double t = 0.0;
        if (LEFT) {  // cols 16..19: this lane's five k values (partials sum in the warp reduction)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            double v = 0.0;
#pragma unroll
            for (int ks = 0; ks < P::KS; ++ks) v = fma(a[g][ks], wl[LEFT ? ks : 0][j], v);
            const double yj = j == 0 ? y[g][2].x : j == 1 ? y[g][2].y : j == 2 ? y[g][LEFT ? 3 : 0].x
                                                                                 : y[g][LEFT ? 3 : 0].y;
            t = fma(v, yj, t);
          }
        }
#pragma unroll
        for (int nt = 0; nt < NTD; ++nt) {
          t = fma(d[g][nt][0], y[g][nt].x, t);
          t = fma(d[g][nt][1], y[g][nt].y, t);
        }
        acc = fma(vq[g], t, acc);
      }
      if (bi + 1 < nb) load_y(bi + 1);  // consumed at the end of the next batch
    }
    cp_async_wait<0>();
    __syncwarp();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) slice_out[i0] = acc;
  }
}

template <int NB, int D>
constexpr size_t t3t2_smem_bytes() {
  return (size_t)8 * ((D + 1) * NB * kT3tST + (D + 3) * NB * 2) * 8;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*SkxEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static bool skx_factor_tmap(CUtensorMap* tm, const double* A, int64_t rows, int R, int box_cols) {
  static SkxEncodeTiled enc = nullptr;
  if (enc == nullptr) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      enc = nullptr;
    if (enc == nullptr) return false;
  }
  if (rows >= (int64_t(1) << 31) || ((uintptr_t)A % 16) != 0 || (R * 8) % 16 != 0) return false;
  cuuint64_t dims[2] = {(cuuint64_t)R, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)R * 8};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, 1};
  cuuint32_t es[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)A, dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---- full TTMc of an order-3 COO at ranks 20 x 20 (modes 1, 2) -------------
// For Algorithm 6's last Tucker fitness pass: per mode-0 slice i0,
// M(i0) = sum_e v_e a1_e a2_e^T (20 x 20) on FP64 tensor cores with the
// nonzeros as the K dimension (m8n8k4: A = a1 rows (b), B = v a2 rows (c),
// 4 nonzeros per k-step, 3 x 3 tiles of the 24 x 24 padded M), both factor
// rows gathered by TMA gather4 into shared memory (box 24 over 20 columns:
// zero padding, conflict-free stride) as k_tucker3_tma2 does for one of them.
// Then P = sum_i0 A0[i0] (x) M(i0) (skx_gemm_atb) is the whole core-sized
// TTMc X x_0 A0^T x_1 A1^T x_2 A2^T, and ANY model on these factors has its
// cross term as one dot with P: the Tucker core's (the fitness) and the CP
// model's (G' = [[lambda; B_0, B_1, B_2]], Alg. 6's final fitness), so one
// pass replaces the last Tucker fitness pass plus the CP fitness pass.
template <int NB, int MB, int D>
__global__ void __launch_bounds__(256, MB) k_ttmc3_tma(
    const __grid_constant__ CUtensorMap tm1, const __grid_constant__ CUtensorMap tm2,
    const int64_t* __restrict__ colptr, int64_t s0, const double* __restrict__ rec,
    uint32_t c1_mask, double* __restrict__ mout) {
  constexpr int ST = kT3tST;
  constexpr int ROWBUF = NB * ST;
  constexpr int NRB = D + 1, NRC = D + 3;
  constexpr uint32_t TX = 2 * NB * ST * 8;  // both row sets of a batch
  extern __shared__ __align__(128) double t3sm[];
  __shared__ __align__(8) uint64_t bars[8][NRB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  double* rows1 = t3sm + (size_t)wid * (2 * NRB * ROWBUF + NRC * NB * 2);
  double* rows2 = rows1 + NRB * ROWBUF;
  double* recs = rows2 + NRB * ROWBUF;
  if (lane == 0)
    for (int b = 0; b < NRB; ++b) mbar_init(&bars[wid][b], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  uint32_t phase = 0;
  const int64_t nw = blockDim.x >> 5, stride = (int64_t)gridDim.x * nw;
  for (int64_t i0 = blockIdx.x * nw + wid; i0 < s0; i0 += stride) {
    const int64_t e0 = colptr[i0], e1 = colptr[i0 + 1];
    double* mo = mout + i0 * 400;
    if (e0 == e1) {
      for (int k = lane; k < 400; k += 32) mo[k] = 0.0;
      continue;
    }
    const int64_t nb = (e1 - e0 + NB - 1) / NB;
    auto issue_recs = [&](int64_t b) {
      if (lane < NB) {
        const int64_t e = e0 + b * NB + lane;
        cp_async16_cg_zfill(smem_addr(recs + ((b % NRC) * NB + lane) * 2),
                            rec + 2 * (e < e1 ? e : e0), e < e1 ? 16u : 0u);
      }
    };
    auto issue_rows = [&](int64_t b) {  // records {i1, i2 | bits, v}: both rows by TMA
      const int slot = (int)(b % NRB);
      const uint32_t* rb = reinterpret_cast<const uint32_t*>(recs + (b % NRC) * NB * 2);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (lane == 0) mbar_expect_tx(&bars[wid][slot], TX);
      __syncwarp();
      if (lane < NB / 4) {
        const uint32_t* r4 = rb + 16 * lane;
        tma_gather4(smem_addr(rows1 + slot * ROWBUF + 4 * lane * ST), &tm1, &bars[wid][slot], 0,
                    (int32_t)r4[0], (int32_t)r4[4], (int32_t)r4[8], (int32_t)r4[12]);
        tma_gather4(smem_addr(rows2 + slot * ROWBUF + 4 * lane * ST), &tm2, &bars[wid][slot], 0,
                    (int32_t)(r4[1] & c1_mask), (int32_t)(r4[5] & c1_mask),
                    (int32_t)(r4[9] & c1_mask), (int32_t)(r4[13] & c1_mask));
      }
    };
    double d[3][3][2];
#pragma unroll
    for (int mt = 0; mt < 3; ++mt)
#pragma unroll
      for (int nt = 0; nt < 3; ++nt) d[mt][nt][0] = d[mt][nt][1] = 0.0;
    for (int64_t b2 = 0; b2 < D + 2 && b2 < nb; ++b2) issue_recs(b2);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    for (int64_t b2 = 0; b2 < D && b2 < nb; ++b2) issue_rows(b2);
    for (int64_t bi = 0; bi < nb; ++bi) {
      cp_async_wait<0>();
      const int slot = (int)(bi % NRB);
      mbar_wait(&bars[wid][slot], (phase >> slot) & 1u);
      phase ^= 1u << slot;
      __syncwarp();
      if (bi + D < nb) issue_rows(bi + D);
      if (bi + D + 2 < nb) issue_recs(bi + D + 2);
      cp_async_commit();
      const double* r1 = rows1 + slot * ROWBUF;
      const double* r2 = rows2 + slot * ROWBUF;
      const double* rv = recs + (bi % NRC) * NB * 2;
#pragma unroll
      for (int ks = 0; ks < NB / 4; ++ks) {
        const int e = 4 * ks + t;
        const double x = rv[e * 2 + 1];
        double a[3], bv[3];
#pragma unroll
        for (int mt = 0; mt < 3; ++mt) a[mt] = r1[e * ST + 8 * mt + g];
#pragma unroll
        for (int nt = 0; nt < 3; ++nt) bv[nt] = x * r2[e * ST + 8 * nt + g];
#pragma unroll
        for (int mt = 0; mt < 3; ++mt)
#pragma unroll
          for (int nt = 0; nt < 3; ++nt) dmma884(d[mt][nt][0], d[mt][nt][1], a[mt], bv[nt]);
      }
      __syncwarp();  // every lane's reads of this slot before it is refilled
    }
    cp_async_wait<0>();
    __syncwarp();
    // D fragment: lane (g, t) holds M[b = 8 mt + g][c = 8 nt + 2 t, +1]
#pragma unroll
    for (int mt = 0; mt < 3; ++mt)
#pragma unroll
      for (int nt = 0; nt < 3; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int b = 8 * mt + g, c = 8 * nt + 2 * t + j;
          if (b < 20 && c < 20) mo[b * 20 + c] = d[mt][nt][j];
        }
  }
}

template <int NB, int D>
constexpr size_t ttmc3_smem_bytes() {
  return (size_t)8 * (2 * (D + 1) * NB * kT3tST + (D + 3) * NB * 2) * 8;
}

template <int R, int NB, int D>
constexpr size_t t3a_smem_bytes() {
  return (size_t)8 * ((D + 1) * 2 * NB * T3A<R>::ST + (D + 3) * NB * 2) * 8;
}

// Skip-mode sparse TTMc for order 3 (src/tensors.py:261-277): row i_n of the
// s_n x (R1 R2) unfolding is sum_e (v_e A1[i1_e, k1]) A2[i2_e, k2] over the
// column's records in layout order (= the reference's mode_sort order), with
// the products and sums unfused so the rounding follows numpy's.  Warp per
// column; lane owns output entries k = lane + 32 t (k1 = k / R2, k2 = k % R2)
// and accumulates them in registers; the column's records are loaded 32 at a
// time and broadcast by shuffles.
template <int T>
__global__ void __launch_bounds__(256) k_ttmc3_skip(int64_t s_n, const int64_t* __restrict__ colptr,
                                                    const double* __restrict__ rec, uint32_t c1_mask,
                                                    const double* __restrict__ A1, int R1,
                                                    const double* __restrict__ A2, int R2,
                                                    double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t tw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int RR = R1 * R2;
  int o1[T], o2[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int k = lane + 32 * t;
    o1[t] = k < RR ? k / R2 : 0;
    o2[t] = k < RR ? k % R2 : 0;
  }
  for (int64_t col = gw; col < s_n; col += tw) {
    double acc[T];
#pragma unroll
    for (int t = 0; t < T; ++t) acc[t] = 0.0;
    const int64_t e0 = colptr[col], e1 = colptr[col + 1];
    for (int64_t base = e0; base < e1; base += 32) {
      const int64_t e = base + lane;
      int32_t ca = 0, cb = 0;
      double v = 0.0;
      if (e < e1) {
        int32_t cc[4];
        load_rec<2>(rec, e, cc, v);
        ca = cc[0];
        cb = (int32_t)((uint32_t)cc[1] & c1_mask);
      }
      const int n = (int)imin(32, e1 - base);
      for (int q = 0; q < n; ++q) {
        const int64_t ia = __shfl_sync(0xffffffffu, ca, q);
        const int64_t ib = __shfl_sync(0xffffffffu, cb, q);
        const double vv = __shfl_sync(0xffffffffu, v, q);
        const double* a1 = A1 + ia * R1;
        const double* a2 = A2 + ib * R2;
#pragma unroll
        for (int t = 0; t < T; ++t)
          acc[t] = __dadd_rn(acc[t], __dmul_rn(__dmul_rn(vv, __ldg(a1 + o1[t])), __ldg(a2 + o2[t])));
      }
    }
    double* dst = out + col * (int64_t)RR;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int k = lane + 32 * t;
      if (k < RR) dst[k] = acc[t];
    }
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

// CP cross term <T, [[w; A0, A1, A2]]> for an order-3 tensor over its mode-0
// fibre layout (src/tensors.py:354-361: mttkrp(T, factors, 0) contracted
// with w * A0).  Warp per slice i0, u = w * A0[i0, :] once.  The warp reads
// 32 records at a time, one 16-byte record per lane (coalesced), and hands
// the coordinates / values out by shuffles; every nonzero is then served by
// LPR = ceil(R/2) lanes, lane c loading the 16-byte chunk c of both of its
// random rows A1[i1] and A2[i2] (L2-resident) and accumulating
// v * sum_{r in chunk} u_r a1_r a2_r.  Each load instruction covers 32/LPR
// whole rows, so it touches only their lines (the L1 wavefront count, not
// the bytes, limits this kernel).  Deterministic: fixed lane / slice
// partition, per-slice partials summed by k_final_sum.
template <int LPR, bool VEC2>
__global__ void __launch_bounds__(256) k_cp3_fibre(const int64_t* __restrict__ colptr, int64_t s0,
                                                   const double* __restrict__ rec, uint32_t c1_mask,
                                                   const double* __restrict__ A0,
                                                   const double* __restrict__ A1,
                                                   const double* __restrict__ A2,
                                                   const double* __restrict__ w, int R,
                                                   double* __restrict__ slice_out) {
  constexpr int NPI = 32 / LPR;                      // nonzeros per load instruction
  constexpr int STEPS = (32 + NPI - 1) / NPI;        // to cover a 32-record batch
  constexpr int U = STEPS >= 4 ? 4 : STEPS;          // steps with loads in flight
  const int lane = threadIdx.x & 31, grp = lane / LPR, ch = lane % LPR, c0 = 2 * ch;
  const bool act = grp < NPI;
  const int64_t nw = blockDim.x >> 5, stride = (int64_t)gridDim.x * nw;
  for (int64_t i0 = blockIdx.x * nw + (threadIdx.x >> 5); i0 < s0; i0 += stride) {
    const int64_t e0 = colptr[i0], e1 = colptr[i0 + 1];
    {  // the next slice's records into L2
      const int64_t j = i0 + stride;
      if (j < s0) {
        const int64_t l0 = colptr[j] * 16 / 128, l1 = (colptr[j + 1] * 16 + 127) / 128;
        for (int64_t l = l0 + lane; l < l1; l += 32)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(rec) + l * 128));
      }
    }
    const double u0 = c0 < R ? w[c0] * A0[i0 * R + c0] : 0.0;
    const double u1 = c0 + 1 < R ? w[c0 + 1] * A0[i0 * R + c0 + 1] : 0.0;
    double acc = 0.0;
    for (int64_t base = e0; base < e1; base += 32) {
      int32_t rc1 = 0, rc2 = 0;
      double rv = 0.0;
      if (base + lane < e1) {
        int32_t cc[4];
        load_rec<2>(rec, base + lane, cc, rv);
        rc1 = cc[0];
        rc2 = (int32_t)((uint32_t)cc[1] & c1_mask);
      }
#pragma unroll
      for (int s = 0; s < STEPS; s += U) {
        int32_t i1[U], i2[U];
        double vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = (s + u) * NPI + grp;
          const int src = idx < 32 ? idx : 31;
          i1[u] = __shfl_sync(0xffffffffu, rc1, src);
          i2[u] = __shfl_sync(0xffffffffu, rc2, src);
          vv[u] = __shfl_sync(0xffffffffu, rv, src);
          if (!act || idx >= 32 || s + u >= STEPS) vv[u] = 0.0;
        }
        double x0[U], x1[U], y0[U], y1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const double* ra = A1 + (int64_t)i1[u] * R;
          const double* rb = A2 + (int64_t)i2[u] * R;
          if (VEC2) {
            const double2 p = c0 < R ? __ldg(reinterpret_cast<const double2*>(ra + c0))
                                     : make_double2(0.0, 0.0);
            const double2 q = c0 < R ? __ldg(reinterpret_cast<const double2*>(rb + c0))
                                     : make_double2(0.0, 0.0);
            x0[u] = p.x;
            x1[u] = p.y;
            y0[u] = q.x;
            y1[u] = q.y;
          } else {
            x0[u] = c0 < R ? __ldg(ra + c0) : 0.0;
            x1[u] = c0 + 1 < R ? __ldg(ra + c0 + 1) : 0.0;
            y0[u] = c0 < R ? __ldg(rb + c0) : 0.0;
            y1[u] = c0 + 1 < R ? __ldg(rb + c0 + 1) : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc = fma(vv[u], fma(u0 * x0[u], y0[u], u1 * x1[u] * y1[u]), acc);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) slice_out[i0] = acc;
  }
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
  int nparts = 0;
  if (R >= 5 && R <= 32) {
    // 4 warps x 8*NT columns per CTA (NT = 4 up to 3 k-steps, else 2: fewer
    // registers, more rows in flight); row splits so that CTAs <= kRedBlocks
    const int KS = (int)((R + 3) / 4);
    const int NT = KS <= 3 ? 4 : 2;
    const int64_t xb = (n_in + 32 * NT - 1) / (32 * NT);
    const int64_t ys = imax(1, imin(kRedBlocks / imax(xb, 1), (n_out + 63) / 64));
    dim3 grid((unsigned)xb, (unsigned)ys);
    nparts = (int)(xb * ys);
#define SKX_RM(ks, nt)                                                                       \
  if (KS == ks) k_resid_mma<ks, nt><<<grid, 128, 0, st>>>(u, vt, n_out, n_in, r, y, ld, part);
    SKX_RM(2, 4) SKX_RM(3, 4) SKX_RM(4, 2) SKX_RM(5, 2) SKX_RM(6, 2) SKX_RM(7, 2) SKX_RM(8, 2)
#undef SKX_RM
  } else {
    // (x-blocks) x (row splits) <= kRedBlocks CTAs, fixed for given shapes
    const int64_t xb = (n_in + kRedThreads - 1) / kRedThreads;
    const int64_t ys = imax(1, imin(kRedBlocks / imax(xb, 1), (n_out + 15) / 16));
    dim3 grid((unsigned)xb, (unsigned)ys);
    nparts = (int)(xb * ys);
    if (xb > kRedBlocks || R > 32) {
      k_resid_gen<<<kRedBlocks, kRedThreads, 0, st>>>(u, vt, n_out, n_in, r, y, ld, part);
      nparts = kRedBlocks;
    } else {
      k_resid<4, 16><<<grid, kRedThreads, 0, st>>>(u, vt, n_out, n_in, r, y, ld, part);
    }
  }
  k_final_sum<<<1, 1024, 0, st>>>(part, nparts, out);
  return check_launch("skx_resid_sq", 2);
}

// Full TTMc P = X x_0 A0^T x_1 A1^T x_2 A2^T of an order-3 COO with ranks
// (R0 <= 32, 20, 20), from its mode-0 fibre layout: per-slice 20 x 20 sums by
// k_ttmc3_tma into the workspace, then P[(b, c), a] = sum_i0 M(i0)[b][c]
// A0[i0][a] (skx_gemm_atb).  P is 400 x R0 row-major.  <P, C> is the Tucker
// cross term of any core C on these factors (src/tensors.py:339-353).
extern "C" int skx_tucker_ttmc3_r20(const int64_t* shape_h, int R0, const int64_t* colptr0,
                                    const void* rec0, uint32_t c1_mask, const double* A0,
                                    const double* A1, const double* A2, double* P, void* ws,
                                    size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(ws_bytes != nullptr, "skx_tucker_ttmc3_r20: ws_bytes is NULL");
  SKX_REQUIRE(R0 >= 1 && R0 <= 32, "skx_tucker_ttmc3_r20: R0 in 1..32");
  const int64_t s0 = shape_h[0];
  size_t gws = 0;
  SKX_TRY(skx_gemm_atb(400, R0, s0, nullptr, 400, nullptr, R0, nullptr, R0, nullptr, &gws, stream));
  Arena ar(ws, *ws_bytes);
  double* mslice = ar.take<double>((size_t)s0 * 400);
  char* gw = ar.take<char>(gws);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_tucker_ttmc3_r20: workspace too small");
  CUtensorMap tm1, tm2;
  SKX_REQUIRE(skx_factor_tmap(&tm1, A1, shape_h[1], 20, kT3tST) &&
                  skx_factor_tmap(&tm2, A2, shape_h[2], 20, kT3tST),
              "skx_tucker_ttmc3_r20: tensor maps unavailable");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t sm = ttmc3_smem_bytes<16, 1>();
  cudaFuncSetAttribute(k_ttmc3_tma<16, 2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const unsigned mb = (unsigned)imax(1, (s0 + 7) / 8);
  k_ttmc3_tma<16, 2, 1><<<mb, 256, sm, s>>>(tm1, tm2, colptr0, s0, (const double*)rec0, c1_mask,
                                             mslice);
  SKX_TRY(check_launch("k_ttmc3_tma"));
  size_t b = gws;
  return skx_gemm_atb(400, R0, s0, mslice, 400, A0, R0, P, R0, gw, &b, stream);
}

extern "C" int skx_tucker_cross_coo(int ndim, const int64_t* shape_h, const int64_t* ranks_h,
                                    int64_t nnz, const int32_t* coords, const double* vals,
                                    const double* const* factors_h, const double* core,
                                    const int64_t* colptr0, const void* rec0, uint32_t c1_mask,
                                    double* out, void* ws, size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(ndim >= 1 && ndim <= 8, "skx_tucker_cross_coo: order 1..8");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_tucker_cross_coo: ws_bytes is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  const bool fast3 = (ndim == 3 && ranks_h[1] <= 32 && ranks_h[2] <= 32 && colptr0 != nullptr &&
                      rec0 != nullptr);
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
    const unsigned blocks = (unsigned)imin((s0 + 3) / 4, (int64_t)num_sms() * 16);
    const double* rec = (const double*)rec0;
    const double* A0 = factors_h[0];
    const double* A1 = factors_h[1];
    const double* A2 = factors_h[2];
    const int RM = R1 > R2 ? R1 : R2;
#define SKX_T3(RT, NP)                                                                    \
  do {                                                                                    \
    const size_t sm = (size_t)4 * (RT * RT + 2 * 32 * NP * (RT + 1) + 2) * 8;             \
    cudaFuncSetAttribute(k_tucker3<RT, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                         (int)sm);                                                        \
    k_tucker3<RT, NP><<<blocks, 128, sm, s>>>(colptr0, s0, rec, c1_mask, A0, A1, A2, core, R0, R1,  \
                                              R2, part);                                  \
  } while (0)
    // ranks <= 4: too little work per row for the 8x8x4 tiles (SIMT kernel is faster)
    if (RM <= 4) {
      if (RM <= 4) SKX_T3(4, 4);
      else if (RM <= 8) SKX_T3(8, 2);
      else if (RM <= 10) SKX_T3(10, 2);
      else if (RM <= 16) SKX_T3(16, 1);
      else if (RM <= 20) SKX_T3(20, 1);
      else SKX_T3(32, 1);
    } else {
      // k-steps of 4 over R1, n-tiles of 8 over R2
      const int KS = (R1 + 3) / 4, NT = (R2 + 7) / 8;
      // short CTAs (one slice per warp): when the fitness runs on a
      // low-priority stream beside a sweep, SMs free up every few tens of
      // microseconds for the sweep's kernels instead of once per wave
      // (persistent grids measured 2-6 ms slower per config-4 call)
      const unsigned mb = (unsigned)imax(1, (s0 + 7) / 8);
#define SKX_T3M(ks, nt)                                                                    \
  if (KS <= ks && NT == nt) {                                                              \
    k_tucker3_mma<ks, nt, 2, 0, 0><<<mb, 256, 0, s>>>(colptr0, s0, rec, c1_mask, A0, A1, A2, core, R0, \
                                                     R1, R2, part);                         \
  } else
      // two 8-warp CTAs per SM (128 registers, no spills): twice the warps to
      // hide the L2 latency of the factor-row gathers (R = 20: 13.3 -> 10.3 ms
      // per 2e8 nonzeros; R = 10 unchanged or better)
      // R = 20 (config 5): rows staged through shared memory by cp.async --
      // in the pipeline, beside the sweeps, it measures 57 ms per 1e9-nonzero
      // pass against 70 ms for the register-pipelined kernel (which is faster
      // alone, 9.9 vs 11.9 ms per 2e8: its 128 registers per thread crowd out
      // the sweeps' kernels).  Other even ranks: register pipeline with 16-byte
      // A-fragment loads (config 4: 4.0 ms per pass in the pipeline).
#define SKX_T3A(RR, NB, MBB, DD)                                                                \
  do {                                                                                          \
    const size_t sm = t3a_smem_bytes<RR, NB, DD>();                                             \
    cudaFuncSetAttribute(k_tucker3_async<RR, NB, MBB, DD>,                                      \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);                 \
    k_tucker3_async<RR, NB, MBB, DD><<<mb, 256, sm, s>>>(colptr0, s0, rec, c1_mask, A0, A1, A2, \
                                                         core, R0, part);                       \
  } while (0)
      // (row lookahead D = 2 with NB = 8 or one CTA per SM measured slower
      // in the pipeline: 592 / 610 vs 538 ms per config-5 call)
      CUtensorMap tmC;
      // SKX_K7_ASYNC set: the all-cp.async kernel (A/B and test hook; read per call)
      const bool force_async = getenv("SKX_K7_ASYNC") != nullptr;
      if (R1 == 20 && R2 == 20 && !force_async &&
          skx_factor_tmap(&tmC, A2, shape_h[2], 20, kT3tST)) {
        // (variants measured at config 5, alone: NB = 16 / 2 CTAs per SM /
        // lookahead 1 = 45.0 ms; NB = 8 with 3 or 4 CTAs 46.5 / 51.2; lookahead
        // 2 59-67; epilogue of batch b-1 deferred behind batch b's DMMAs 56-82
        // (register spills))
        const size_t sm = t3t_smem_bytes<16, 1>();
        // default: k_tucker3_tma2 (mode-1 rows by TMA, mode-2 rows into
        // registers; config 5 alone: 36.9 ms per 1e9-nonzero pass against 43.4
        // for k_tucker3_tma with the FMA-pipe tail and 45.1 padded).
        // SKX_K7=1: k_tucker3_tma (A/B); SKX_K7=2[D][MB]: tma2 variants
        const char* k7v = getenv("SKX_K7");
        if ((k7v == nullptr || k7v[0] == '2') &&
            skx_factor_tmap(&tmC, A1, shape_h[1], 20, kT3tST)) {  // mode-2 rows into registers
          const int dd = (k7v != nullptr && k7v[1] == '2') ? 2 : 1;
          const int mbb = (k7v != nullptr && k7v[1] != 0 && k7v[2] == '3') ? 3 : 2;
#define SKX_T3T2(MBB, DD)                                                                     \
  do {                                                                                        \
    const size_t sm2 = t3t2_smem_bytes<16, DD>();                                             \
    cudaFuncSetAttribute(k_tucker3_tma2<16, MBB, DD>,                                         \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);              \
    k_tucker3_tma2<16, MBB, DD><<<mb, 256, sm2, s>>>(tmC, colptr0, s0, rec, c1_mask, A0, A2,  \
                                                     core, R0, part);                         \
  } while (0)
          // (A/B) FMA-pipe tail, NB = 16 or 8: 43.5 ms (spills at 128 registers);
          // with one 255-register CTA per SM instead: 60.5 ms (half the warps)
          if (k7v != nullptr && k7v[1] == 'L') {
            const bool nb8 = k7v[2] == '8';
            if (nb8) {
              const size_t sm2 = t3t2_smem_bytes<8, 1>();
              cudaFuncSetAttribute(k_tucker3_tma2<8, 2, 1, true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
              k_tucker3_tma2<8, 2, 1, true><<<mb, 256, sm2, s>>>(tmC, colptr0, s0, rec, c1_mask, A0,
                                                                   A2, core, R0, part);
            } else {
              const size_t sm2 = t3t2_smem_bytes<16, 1>();
              cudaFuncSetAttribute(k_tucker3_tma2<16, 2, 1, true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
              k_tucker3_tma2<16, 2, 1, true><<<mb, 256, sm2, s>>>(tmC, colptr0, s0, rec, c1_mask, A0,
                                                                    A2, core, R0, part);
            }
          } else if (dd == 1 && mbb == 2) SKX_T3T2(2, 1);
          else if (dd == 2 && mbb == 2) SKX_T3T2(2, 2);
          else if (dd == 1) SKX_T3T2(3, 1);
          else SKX_T3T2(3, 2);
#undef SKX_T3T2
        } else if (getenv("SKX_K7_PAD") == nullptr &&
                   skx_factor_tmap(&tmC, A2, shape_h[2], 20, kT3tST)) {  // 16..19 on the FMA pipe
          cudaFuncSetAttribute(k_tucker3_tma<16, 2, 1, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
          k_tucker3_tma<16, 2, 1, true><<<mb, 256, sm, s>>>(tmC, colptr0, s0, rec, c1_mask, A0, A1,
                                                             core, R0, part);
        } else {  // (A/B: padded third n-tile on the tensor cores)
          cudaFuncSetAttribute(k_tucker3_tma<16, 2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)sm);
          k_tucker3_tma<16, 2, 1><<<mb, 256, sm, s>>>(tmC, colptr0, s0, rec, c1_mask, A0, A1, core,
                                                       R0, part);
        }
      } else if (R1 == 20 && R2 == 20) {
        SKX_T3A(20, 16, 2, 1);
      } else if (R1 == 10 && R2 == 10) {
        k_tucker3_mma<3, 2, 2, 10, 10, 2, true><<<mb, 256, 0, s>>>(colptr0, s0, rec, c1_mask, A0, A1,
                                                                   A2, core, R0, R1, R2, part);
      } else
      SKX_T3M(2, 1) SKX_T3M(3, 1) SKX_T3M(5, 1) SKX_T3M(8, 1)
      SKX_T3M(2, 2) SKX_T3M(3, 2) SKX_T3M(5, 2) SKX_T3M(8, 2)
      SKX_T3M(2, 3) SKX_T3M(3, 3) SKX_T3M(5, 3) SKX_T3M(8, 3)
      SKX_T3M(2, 4) SKX_T3M(3, 4) SKX_T3M(5, 4) SKX_T3M(8, 4) {
        SKX_REQUIRE(false, "skx_tucker_cross_coo: no kernel for ranks %d x %d", R1, R2);
      }
#undef SKX_T3M
    }
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

extern "C" int skx_cp_cross_fibre3(int64_t s0, const int64_t* colptr0, const void* rec0,
                                   uint32_t c1_mask, int R, const double* const* factors_h,
                                   const double* weights, double* out, void* ws, size_t* ws_bytes,
                                   void* stream) {
  SKX_REQUIRE(R >= 1 && R <= 32, "skx_cp_cross_fibre3: 1 <= R <= 32");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_cp_cross_fibre3: ws_bytes is NULL");
  const size_t need = (size_t)imax(s0, 1) * 8 + 256;
  if (ws == nullptr) {
    *ws_bytes = need;
    return SKX_OK;
  }
  SKX_REQUIRE(*ws_bytes >= need, "skx_cp_cross_fibre3: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  double* part = (double*)ws;
  const unsigned mb = (unsigned)imax(1, (s0 + 7) / 8);
  const double* rec = (const double*)rec0;
  const double *A0 = factors_h[0], *A1 = factors_h[1], *A2 = factors_h[2];
  const int half = (R + 1) / 2;
  const bool v2 = (R & 1) == 0;
#define SKX_CP3(lp)                                                                            \
  case lp:                                                                                     \
    if (v2)                                                                                    \
      k_cp3_fibre<lp, true><<<mb, 256, 0, s>>>(colptr0, s0, rec, c1_mask, A0, A1, A2, weights, \
                                               R, part);                                       \
    else                                                                                       \
      k_cp3_fibre<lp, false><<<mb, 256, 0, s>>>(colptr0, s0, rec, c1_mask, A0, A1, A2,         \
                                                weights, R, part);                             \
    break;
  switch (half) {
    SKX_CP3(1) SKX_CP3(2) SKX_CP3(3) SKX_CP3(4) SKX_CP3(5) SKX_CP3(6) SKX_CP3(7) SKX_CP3(8)
    SKX_CP3(9) SKX_CP3(10) SKX_CP3(11) SKX_CP3(12) SKX_CP3(13) SKX_CP3(14) SKX_CP3(15)
    SKX_CP3(16)
    default: break;
  }
#undef SKX_CP3
  k_final_sum<<<1, 1024, 0, s>>>(part, (int)s0, out);
  return check_launch("k_cp3_fibre", 2);
}

extern "C" int skx_ttmc3_skip_coo(int64_t s_n, const int64_t* colptr, const void* rec,
                                  uint32_t c1_mask, const double* a1, int r1, const double* a2,
                                  int r2, double* out, void* stream) {
  SKX_REQUIRE(r1 >= 1 && r2 >= 1 && r1 * r2 <= 1024,
              "skx_ttmc3_skip_coo: need 1 <= R1 R2 <= 1024");
  if (s_n == 0) return SKX_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int rr = r1 * r2;
  const int64_t blocks = imin((s_n + 7) / 8, (int64_t)num_sms() * 16);
  const double* rc = (const double*)rec;
#define SKX_TT(T) k_ttmc3_skip<T><<<(unsigned)blocks, 256, 0, s>>>(s_n, colptr, rc, c1_mask, a1, r1, \
                                                                  a2, r2, out)
  if (rr <= 32) SKX_TT(1);
  else if (rr <= 64) SKX_TT(2);
  else if (rr <= 128) SKX_TT(4);
  else if (rr <= 256) SKX_TT(8);
  else if (rr <= 512) SKX_TT(16);
  else SKX_TT(32);
#undef SKX_TT
  return check_launch("k_ttmc3_skip");
}

// ---- dense TTM chain for the Tucker fitness of a dense tensor -------------
// out[b, r, p] = sum_i A[i, r] T[b, i, p] for T viewed as (B, s, P) in C
// order: the mode-n product with A^T of a tensor whose modes before n are
// folded into B and after n into P (src/tensors.py:217-247, ttmc with every
// mode, as the fitness needs: src/tensors.py:349-353).  Applied mode after
// mode, the first pass streams the whole tensor once (HBM-bound: R FMAs per
// 8-byte element on the FP64 pipe) and the later ones touch tensors smaller
// by R_n / s_n.  Thread per output column p; A's rows are staged through
// shared memory in tiles of 64; the R accumulators live in registers.
namespace skx {
template <int RT>
__global__ void __launch_bounds__(256) k_ttm_lead(const double* __restrict__ T, int64_t B, int64_t s,
                                                  int64_t P, const double* __restrict__ A, int R,
                                                  double* __restrict__ out) {
  __shared__ double At[64 * RT];
  const int64_t nblk_p = (P + blockDim.x - 1) / blockDim.x;
  for (int64_t blk = blockIdx.x; blk < B * nblk_p; blk += gridDim.x) {
    const int64_t b = blk / nblk_p;
    const int64_t p = (blk - b * nblk_p) * blockDim.x + threadIdx.x;
    double acc[RT];
#pragma unroll
    for (int r = 0; r < RT; ++r) acc[r] = 0.0;
    const double* tb = T + b * s * P;
    for (int64_t i0 = 0; i0 < s; i0 += 64) {
      const int ni = (int)imin(64, s - i0);
      __syncthreads();
      for (int e = threadIdx.x; e < ni * RT; e += blockDim.x) {
        const int ii = e / RT, r = e - ii * RT;
        At[e] = r < R ? A[(i0 + ii) * R + r] : 0.0;
      }
      __syncthreads();
      if (p < P) {
        for (int ii = 0; ii < ni; ++ii) {
          const double x = __ldcs(tb + (i0 + ii) * P + p);
#pragma unroll
          for (int r = 0; r < RT; ++r) acc[r] = fma(At[ii * RT + r], x, acc[r]);
        }
      }
    }
    if (p < P) {
      double* ob = out + b * (int64_t)R * P + p;
      for (int r = 0; r < R; ++r) ob[(int64_t)r * P] = acc[r < RT ? r : 0];
    }
  }
}
}  // namespace skx

extern "C" int skx_ttm_lead(const double* t, int64_t B, int64_t s, int64_t P, const double* a,
                            int R, double* out, void* stream) {
  SKX_REQUIRE(R >= 1 && R <= 32, "skx_ttm_lead: 1 <= R <= 32");
  SKX_REQUIRE(B >= 1 && s >= 1 && P >= 1, "skx_ttm_lead: empty operand");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t work = B * ((P + 255) / 256);
  const unsigned g = (unsigned)imin(work, (int64_t)num_sms() * 8);
#define SKX_TL(rt) k_ttm_lead<rt><<<g, 256, 0, st>>>(t, B, s, P, a, R, out)
  if (R <= 4) SKX_TL(4);
  else if (R <= 8) SKX_TL(8);
  else if (R <= 12) SKX_TL(12);
  else if (R <= 16) SKX_TL(16);
  else if (R <= 24) SKX_TL(24);
  else SKX_TL(32);
#undef SKX_TL
  return check_launch("k_ttm_lead");
}
