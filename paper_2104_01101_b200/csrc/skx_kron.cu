// K2: TensorSketch of a Kronecker chain, Z = S (A_1 kron ... kron A_k)
// (src/sketching.py:113-147), as exact circular convolutions of the per-mode
// CountSketches -- no FFT.
//
//  plan  (once per TensorSketchOp; its tables never change across sweeps):
//        rows of every mode bucket-sorted (cub radix sort, stable, so rows stay
//        ascending inside a bucket) and run-length encoded: run r = bucket rb[r]
//        holding rows[rs[r] .. rs[r+1]).
//  apply (every sub-problem):
//        CS of mode k, per run and column: ascending-row sequential sums (the
//        order numpy's add.at uses, src/sketching.py:62);
//        Z_1 = dense CountSketch of A_1; Z_{k} = Z_{k-1} (*) CS_k column by
//        column: z_new[h, (q,p)] = sum_runs cs_k[r,p] z[(h - rb[r]) mod m, q],
//        cost m x #runs per output column (#runs <= min(m, s_k)), runs split
//        across CTAs into fixed-order partial sums (deterministic).
// Z is produced column-major (ld = m), the layout the QR consumes.
#include <cub/cub.cuh>

#include "skx_common.cuh"

namespace skx {

struct KronModePlan {
  uint32_t* rows;  // s_k, bit 31 = sign of the row
  uint32_t* rb;    // run buckets (<= s_k)
  int64_t* rs;     // run starts (<= s_k + 1)
  int* nrun;       // device scalar
};

__global__ void k_kp_keys(const uint32_t* __restrict__ tab, int64_t s, uint32_t* keys,
                          uint32_t* vals) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= s) return;
  const uint32_t t = tab[i];
  keys[i] = pk_bucket(t);
  vals[i] = (uint32_t)i | (t & 0x80000000u);
}

// cs[r*R + p] = sum over the run's rows (ascending) of sign * A[row, p]
__global__ void k_kp_cs(const double* __restrict__ A, int64_t R, KronModePlan pl,
                        double* __restrict__ cs) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nr = *pl.nrun;
  if (idx >= nr * R) return;
  const int64_t r = idx / R, p = idx - r * R;
  const int64_t e0 = pl.rs[r], e1 = pl.rs[r + 1];
  double s = 0.0;
  int64_t e = e0;
  for (; e + 8 <= e1; e += 8) {  // 8 independent loads in flight, summed in order
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t w = pl.rows[e + u];
      const double v = A[(int64_t)(w & 0x7fffffffu) * R + p];
      x[u] = (w >> 31) ? -v : v;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) s += x[u];
  }
  for (; e < e1; ++e) {
    const uint32_t w = pl.rows[e];
    const double v = A[(int64_t)(w & 0x7fffffffu) * R + p];
    s += (w >> 31) ? -v : v;
  }
  cs[idx] = s;
}

__global__ void k_kp_dense(const double* __restrict__ cs, KronModePlan pl, int64_t R, int64_t m,
                           double* __restrict__ zt) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nr = *pl.nrun;
  if (idx >= nr * R) return;
  const int64_t r = idx / R, p = idx - r * R;
  zt[p * m + pl.rb[r]] = cs[idx];
}

// grid (h-blocks, q, run-split).  Partial sums part[split][q*R+p][h].  Each
// thread owns KH output buckets (h, h + 256, ...) so every run's CountSketch
// row (PC values, a broadcast load) is reused KH times from registers.
constexpr int kKpKH = 4;

template <int PC>
__global__ void __launch_bounds__(256) k_kp_conv(const double* __restrict__ zc, int64_t m,
                                                 const double* __restrict__ cs, KronModePlan pl,
                                                 int64_t R, int nsplit, double* __restrict__ part,
                                                 int64_t rnew) {
  extern __shared__ double zs[];
  const int64_t q = blockIdx.y;
  for (int64_t h = threadIdx.x; h < m; h += blockDim.x) zs[h] = zc[q * m + h];
  __syncthreads();
  const int64_t hb = blockIdx.x * (int64_t)blockDim.x * kKpKH + threadIdx.x;
  if (hb >= m) return;
  const int64_t nr = *pl.nrun;
  const int64_t per = (nr + nsplit - 1) / nsplit;
  const int64_t r0 = imin(blockIdx.z * per, nr), r1 = imin(r0 + per, nr);
  for (int64_t p0 = 0; p0 < R; p0 += PC) {
    double acc[kKpKH][PC];
#pragma unroll
    for (int j = 0; j < kKpKH; ++j)
#pragma unroll
      for (int u = 0; u < PC; ++u) acc[j][u] = 0.0;
    for (int64_t r = r0; r < r1; ++r) {
      const double* y = cs + r * R + p0;
      double yv[PC];
#pragma unroll
      for (int u = 0; u < PC; ++u) yv[u] = p0 + u < R ? __ldg(y + u) : 0.0;
      const int64_t b = (int64_t)pl.rb[r];
#pragma unroll
      for (int j = 0; j < kKpKH; ++j) {
        int64_t src = hb + j * (int64_t)blockDim.x - b;
        if (src < 0) src += m;
        const double zv = src < m ? zs[src] : 0.0;
#pragma unroll
        for (int u = 0; u < PC; ++u) acc[j][u] = fma(yv[u], zv, acc[j][u]);
      }
    }
#pragma unroll
    for (int j = 0; j < kKpKH; ++j) {
      const int64_t h = hb + j * (int64_t)blockDim.x;
      if (h >= m) continue;
#pragma unroll
      for (int u = 0; u < PC; ++u)
        if (p0 + u < R) part[((int64_t)blockIdx.z * rnew + q * R + p0 + u) * m + h] = acc[j][u];
    }
  }
}

__global__ void k_kp_sum(const double* __restrict__ part, int nsplit, int64_t n,
                         double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int k = 0; k < nsplit; ++k) s += part[(int64_t)k * n + i];
  out[i] = s;
}

// plan buffer layout per mode: rows[s] u32 | rb[s] u32 | rs[s+1] i64 | nrun i32
struct PlanLayout {
  size_t off[15][4];
  size_t total;
};

static PlanLayout plan_layout(int n, const int64_t* ext) {
  PlanLayout L{};
  size_t o = 0;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  for (int k = 0; k < n; ++k) {
    const size_t s = (size_t)ext[k];
    L.off[k][0] = o; o = al(o + 4 * s);
    L.off[k][1] = o; o = al(o + 4 * s);
    L.off[k][2] = o; o = al(o + 8 * (s + 1));
    L.off[k][3] = o; o = al(o + 8);
  }
  L.total = o;
  return L;
}

static KronModePlan mode_plan(void* plan, const PlanLayout& L, int k) {
  char* b = (char*)plan;
  KronModePlan p;
  p.rows = (uint32_t*)(b + L.off[k][0]);
  p.rb = (uint32_t*)(b + L.off[k][1]);
  p.rs = (int64_t*)(b + L.off[k][2]);
  p.nrun = (int*)(b + L.off[k][3]);
  return p;
}

}  // namespace skx

using namespace skx;

extern "C" int skx_ts_kron_plan(int n_other, const int64_t* ext_h, const uint32_t* tab,
                                const int64_t* tab_off_h, int64_t m, void* plan, size_t* plan_bytes,
                                void* ws, size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(n_other >= 1 && n_other <= 15, "skx_ts_kron_plan: 1..15 factors supported");
  SKX_REQUIRE(plan_bytes != nullptr && ws_bytes != nullptr, "skx_ts_kron_plan: size pointers NULL");
  const PlanLayout L = plan_layout(n_other, ext_h);
  int64_t smax = 1;
  for (int k = 0; k < n_other; ++k) smax = imax(smax, ext_h[k]);
  Arena ar(ws, *ws_bytes);
  uint32_t* k_in = ar.take<uint32_t>(smax);
  uint32_t* k_out = ar.take<uint32_t>(smax);
  uint32_t* v_in = ar.take<uint32_t>(smax);
  int64_t* cnt = ar.take<int64_t>(smax + 1);
  size_t b1 = 0, b2 = 0, b3 = 0;
  cudaStream_t s = (cudaStream_t)stream;
  cub::DeviceRadixSort::SortPairs(nullptr, b1, k_in, k_out, v_in, v_in, (int)smax, 0, 32, s);
  cub::DeviceRunLengthEncode::Encode(nullptr, b2, k_out, k_in, cnt, (int*)nullptr, (int)smax, s);
  cub::DeviceScan::ExclusiveSum(nullptr, b3, cnt, (int64_t*)nullptr, (int)smax + 1, s);
  const size_t cb = std::max(b1, std::max(b2, b3));
  void* tmp = ar.take<char>(cb);
  if (plan == nullptr || ws == nullptr) {
    *plan_bytes = L.total;
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok() && *plan_bytes >= L.total, "skx_ts_kron_plan: buffers too small");
  int bits = 1;
  while ((int64_t(1) << bits) < m) ++bits;
  for (int k = 0; k < n_other; ++k) {
    const int64_t sk = ext_h[k];
    KronModePlan p = mode_plan(plan, L, k);
    k_kp_keys<<<(unsigned)((sk + 255) / 256), 256, 0, s>>>(tab + tab_off_h[k], sk, k_in, v_in);
    size_t c1 = cb;
    cub::DeviceRadixSort::SortPairs(tmp, c1, k_in, k_out, v_in, p.rows, (int)sk, 0, bits, s);
    cudaMemsetAsync(cnt, 0, (sk + 1) * sizeof(int64_t), s);
    c1 = cb;
    cub::DeviceRunLengthEncode::Encode(tmp, c1, k_out, p.rb, cnt, p.nrun, (int)sk, s);
    c1 = cb;
    cub::DeviceScan::ExclusiveSum(tmp, c1, cnt, p.rs, (int)sk + 1, s);
  }
  return check_launch("skx_ts_kron_plan", 4 * n_other);
}

extern "C" int skx_ts_kron_apply(int n_other, const int64_t* ext_h, const int64_t* ranks_h,
                                 const double* const* factors_h, const void* plan, int64_t m,
                                 double* z, void* ws, size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(n_other >= 1 && n_other <= 15, "skx_ts_kron_apply: 1..15 factors supported");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_ts_kron_apply: ws_bytes is NULL");
  const PlanLayout L = plan_layout(n_other, ext_h);
  int64_t smax = 1, rmax = 1, rtot = 1, rmid = 1;
  for (int k = 0; k < n_other; ++k) {
    smax = imax(smax, ext_h[k]);
    rmax = imax(rmax, ranks_h[k]);
    rtot *= ranks_h[k];
  }
  for (int k = 0; k + 1 < n_other; ++k) rmid *= ranks_h[k];
  const int nsms = num_sms();
  // run split chosen so the largest step has >= 2 CTAs per SM
  const int64_t hblk = (m + 256 * kKpKH - 1) / (256 * kKpKH);
  int nsplit = (int)imax(1, imin(32, (2 * nsms + hblk * rmid - 1) / imax(1, hblk * rmid)));
  Arena ar(ws, *ws_bytes);
  double* cs = ar.take<double>(smax * rmax);
  double* zbuf = ar.take<double>(rmid * m);
  double* part = ar.take<double>((size_t)nsplit * rtot * m);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_ts_kron_apply: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  int launches = 0;
  int64_t rcur = 1;
  for (int k = 0; k < n_other; ++k) {
    const int64_t sk = ext_h[k], R = ranks_h[k];
    KronModePlan p = mode_plan(const_cast<void*>(plan), L, k);
    k_kp_cs<<<(unsigned)((sk * R + 255) / 256), 256, 0, s>>>(factors_h[k], R, p, cs);
    // destination: z for the last mode, ping-pong before (so the last lands in z)
    double* dst = ((n_other - 1 - k) % 2 == 0) ? z : zbuf;
    if (k == 0) {
      cudaMemsetAsync(dst, 0, (size_t)R * m * sizeof(double), s);
      k_kp_dense<<<(unsigned)((sk * R + 255) / 256), 256, 0, s>>>(cs, p, R, m, dst);
      launches += 2;
    } else {
      const double* src = (dst == z) ? zbuf : z;
      const int64_t rnew = rcur * R;
      dim3 grid((unsigned)hblk, (unsigned)rcur, (unsigned)nsplit);
      if (R <= 4)
        k_kp_conv<4><<<grid, 256, (size_t)m * 8, s>>>(src, m, cs, p, R, nsplit, part, rnew);
      else if (R <= 8)
        k_kp_conv<8><<<grid, 256, (size_t)m * 8, s>>>(src, m, cs, p, R, nsplit, part, rnew);
      else if (R <= 10)
        k_kp_conv<10><<<grid, 256, (size_t)m * 8, s>>>(src, m, cs, p, R, nsplit, part, rnew);
      else
        k_kp_conv<16><<<grid, 256, (size_t)m * 8, s>>>(src, m, cs, p, R, nsplit, part, rnew);
      const int64_t n = rnew * m;
      k_kp_sum<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(part, nsplit, n, dst);
      launches += 3;
    }
    rcur *= R;
  }
  return check_launch("skx_ts_kron_apply", launches);
}
