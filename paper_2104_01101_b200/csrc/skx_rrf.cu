// K4: randomized range finder, CountSketch stage (src/sketching.py:54-56,
// 305-341; src/tucker.py:129-144).
//
// numpy draws hash = integers(0, k2, P) then sign = integers(0, 2, P) from
// rng_init.  Column j's hash is the j-th *accepted* Lemire draw: with the
// sorted rejection positions r_0 < r_1 < ... (skx_lemire_scan) and
// d_i = r_i - i, its u32 index is q(j) = j + #{i : d_i <= j}.  k = 2 never
// rejects, so sign j sits at u32 index sign_q0 + j.  The P_n-long tables of
// the reference (160-640 GB at configs 4-5) are never materialised for COO
// inputs: each nonzero evaluates its two Philox blocks on the fly.
#include <cub/cub.cuh>

#include "skx_common.cuh"

namespace skx {

// Map the sorted absolute rejection positions onto run indices of an
// integers() call that starts at raw word p0 (optionally preceded by the
// buffered high half of raw word pend_raw): q = 0 for that half, else
// q = has + (A - 2 p0); positions outside the run are dropped.  Then
// d_j = q_j - j and n_le = #{d_j <= P-1}.  Single thread: there are O(cap)
// (~1e3) entries and the order must be preserved.
__global__ void k_rej_to_d(const uint64_t* __restrict__ sorted, const unsigned long long* count,
                           int64_t cap, uint64_t p0, uint32_t has, uint64_t pend_raw, uint64_t P,
                           uint64_t* __restrict__ d, unsigned long long* n_le) {
  const int64_t n = (int64_t)umin64(*count, (unsigned long long)cap);
  int64_t j = 0;
  unsigned long long le = 0;
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t A = sorted[i];
    uint64_t q;
    if (has && A == 2 * pend_raw + 1) q = 0;
    else if (A >= 2 * p0) q = (uint64_t)has + (A - 2 * p0);
    else continue;
    const uint64_t dj = q - (uint64_t)j;
    d[j++] = dj;
    if (dj <= P - 1) ++le;
  }
  for (; j < cap; ++j) d[j] = ~0ULL;
  *n_le = le;
}

__global__ void k_fill_max(uint64_t* a, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = ~0ULL;
}

__device__ __forceinline__ uint64_t count_le(const uint64_t* d, int64_t n, uint64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (d[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return (uint64_t)lo;
}


struct RrfRng {
  U32Stream st;
  uint64_t sign_q0;
  const uint64_t* d;
  int64_t nd;
  uint32_t k2;
};

// q(j) from a shared-memory bucket table: cnt[b] = #{d_i < b << shift}
// (kRrfBuckets buckets over the column range), then the few d entries inside
// j's bucket (usually none: ~1e2 rejections over 4096 buckets).
constexpr int kRrfBuckets = 4096;

__device__ __forceinline__ uint64_t count_le_tab(const RrfRng& r, const uint32_t* cnt, int shift,
                                                uint64_t j) {
  const uint64_t b = j >> shift;
  uint32_t i = cnt[b];
  const uint32_t e = cnt[b + 1];
  while (i < e && r.d[i] <= j) ++i;
  return i;
}

__device__ __forceinline__ uint32_t rrf_entry_q(const RrfRng& r, uint64_t j, uint64_t q) {
  const uint32_t hu = r.st.at(q);
  const uint32_t h = (uint32_t)(((uint64_t)hu * r.k2) >> 32);
  const uint32_t su = r.st.at(r.sign_q0 + j);
  return h | (su & 0x80000000u);  // integers(0,2) = u >> 31; sign = 1 - 2g
}

__device__ __forceinline__ uint32_t rrf_entry(const RrfRng& r, uint64_t j) {
  const uint64_t q = j + count_le(r.d, r.nd, j);
  const uint32_t hu = r.st.at(q);
  const uint32_t h = (uint32_t)(((uint64_t)hu * r.k2) >> 32);
  const uint32_t su = r.st.at(r.sign_q0 + j);
  return h | (su & 0x80000000u);  // integers(0,2) = u >> 31; sign = 1 - 2g
}

__global__ void k_rrf_table(RrfRng r, int64_t P, uint32_t* __restrict__ tab) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; j < P; j += stride) tab[j] = rrf_entry(r, (uint64_t)j);
}

// Fibre-major COO: warp per column i_n, warp-private k2 accumulator; ordered.
struct OthExt {
  int n;
  int64_t ext[15];
};

// c1_mask: the last other coordinate is rec word & c1_mask (layouts from
// skx_coo_fibre_ts keep sketch bits above it).
template <int U, int NO>
__global__ void __launch_bounds__(256) k_rrf_coo(RrfRng r, OthExt oe, int64_t s_n,
                                                 const int64_t* __restrict__ colptr,
                                                 const double* __restrict__ rec, uint32_t c1_mask,
                                                 double* __restrict__ st1) {
  extern __shared__ double smem[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int64_t k2 = r.k2;
  double* acc = smem + (size_t)wid * (k2 + 32);
  double* stage = acc + k2;
  // bucket table of the sorted rejection offsets (after the accumulators)
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + (size_t)nw * (k2 + 32));
  uint64_t P = 1;
  for (int k = 0; k < NO; ++k) P *= (uint64_t)oe.ext[k];
  int shift = 0;
  while ((P >> shift) >= (uint64_t)kRrfBuckets) ++shift;
  for (int b = threadIdx.x; b <= kRrfBuckets; b += blockDim.x) {
    const uint64_t v = (uint64_t)b << shift;  // count d_i < v
    int64_t lo = 0, hi = r.nd;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (r.d[mid] < v) lo = mid + 1; else hi = mid;
    }
    cnt[b] = (uint32_t)lo;
  }
  __syncthreads();
  const int64_t gw = blockIdx.x * (int64_t)nw + wid;
  const int64_t tw = (int64_t)gridDim.x * nw;
  for (int64_t col = gw; col < s_n; col += tw) {
    for (int64_t h = lane; h < k2; h += 32) acc[h] = 0.0;
    __syncwarp();
    const int64_t e0 = colptr[col], e1 = colptr[col + 1];
    for (int64_t base = e0; base < e1; base += 32 * U) {
      uint32_t bk[U];
      double v[U];
      int32_t c[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = base + u * 32 + lane;
        load_rec<NO>(rec, e < e1 ? e : e0, c[u], v[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = base + u * 32 + lane < e1;
        uint64_t j = 0;
#pragma unroll
        for (int k = 0; k < NO; ++k)
          j = j * (uint64_t)oe.ext[k] +
              (uint64_t)((uint32_t)c[u][k] & (k == NO - 1 ? c1_mask : 0xffffffffu));
        const uint32_t t = rrf_entry_q(r, j, j + count_le_tab(r, cnt, shift, j));
        bk[u] = ok ? pk_bucket(t) : kNoBucket;
        v[u] = pk_neg(t) ? -v[u] : v[u];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) warp_ordered_add(acc, bk[u], v[u], stage);
    }
    double* dst = st1 + col * k2;
    for (int64_t h = lane; h < k2; h += 32) dst[h] = acc[h];
    __syncwarp();
  }
}

}  // namespace skx

using namespace skx;

// Sort the scan output and turn it into the d-array of a run (p0, has,
// pend_raw) (length cap, padded with UINT64_MAX); *n_le receives
// #{d_i <= P-1} = rejections among the P hash draws, i.e. the sign run starts
// at u32 index P + *n_le.
extern "C" int skx_lemire_finish(uint64_t* rej, const unsigned long long* count, int64_t cap,
                                 uint64_t p0, uint32_t has, uint64_t pend_raw, uint64_t P,
                                 uint64_t* d, unsigned long long* n_le, void* ws, size_t* ws_bytes,
                                 void* stream) {
  SKX_REQUIRE(ws_bytes != nullptr, "skx_lemire_finish: ws_bytes is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  Arena ar(ws, *ws_bytes);
  uint64_t* sorted = ar.take<uint64_t>(cap);
  size_t cb = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, cb, rej, sorted, (int)cap, 0, 64, s);
  void* tmp = ar.take<char>(cb);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_lemire_finish: workspace too small");
  // entries beyond count were never written: neutralise them before sorting
  // (the caller pre-fills rej with UINT64_MAX via skx_fill_u64max).
  cub::DeviceRadixSort::SortKeys(tmp, cb, rej, sorted, (int)cap, 0, 64, s);
  k_rej_to_d<<<1, 1, 0, s>>>(sorted, count, cap, p0, has, pend_raw, P, d, n_le);
  return check_launch("skx_lemire_finish", 2);
}

extern "C" int skx_fill_u64max(uint64_t* a, int64_t n, void* stream) {
  if (n <= 0) return SKX_OK;
  k_fill_max<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(a, n);
  return check_launch("k_fill_max");
}

static RrfRng make_rng(uint64_t k0, uint64_t k1, uint64_t p0, uint32_t has_pending, uint32_t pending,
                       uint64_t sign_q0, const uint64_t* d, int64_t nd, int64_t k2) {
  RrfRng r;
  r.st.k0 = k0;
  r.st.k1 = k1;
  r.st.p0 = p0;
  r.st.has_pending = has_pending;
  r.st.pending = pending;
  r.sign_q0 = sign_q0;
  r.d = d;
  r.nd = nd;
  r.k2 = (uint32_t)k2;
  return r;
}

extern "C" int skx_rrf_table(uint64_t k0, uint64_t k1, uint64_t p0, uint32_t has_pending,
                             uint32_t pending, uint64_t sign_q0, const uint64_t* rej, int64_t nrej,
                             int64_t P, int64_t k2, uint32_t* tab, void* stream) {
  SKX_REQUIRE(k2 >= 1 && k2 < (int64_t(1) << 31), "skx_rrf_table: k2 out of range");
  if (P == 0) return SKX_OK;
  RrfRng r = make_rng(k0, k1, p0, has_pending, pending, sign_q0, rej, nrej, k2);
  int blocks = (int)imin((P + 255) / 256, (int64_t)num_sms() * 16);
  k_rrf_table<<<blocks, 256, 0, (cudaStream_t)stream>>>(r, P, tab);
  return check_launch("k_rrf_table");
}

extern "C" int skx_rrf_stage1_coo(int n_other, const int64_t* ext_h, int64_t s_n,
                                  const int64_t* colptr, const void* rec, uint64_t k0, uint64_t k1,
                                  uint64_t p0, uint32_t has_pending, uint32_t pending,
                                  uint64_t sign_q0, const uint64_t* rej, int64_t nrej, int64_t k2,
                                  uint32_t c1_mask, double* stage1, void* stream) {
  SKX_REQUIRE(n_other >= 1 && n_other <= 4, "skx_rrf_stage1_coo: 1..4 other modes");
  const int64_t per = (k2 + 32) * 8;
  const int64_t tab_bytes = (kRrfBuckets + 1) * 4;
  int nw = (int)imin(8, (int64_t)(max_smem_optin() - 1024 - tab_bytes) / per);
  SKX_REQUIRE(nw >= 1, "skx_rrf_stage1_coo: k2 too large for shared memory");
  SKX_REQUIRE(nrej < (int64_t(1) << 32), "skx_rrf_stage1_coo: rejection list too long");
  if (s_n == 0) return SKX_OK;
  RrfRng r = make_rng(k0, k1, p0, has_pending, pending, sign_q0, rej, nrej, k2);
  OthExt oe{};
  oe.n = n_other;
  for (int k = 0; k < n_other; ++k) oe.ext[k] = ext_h[k];
  const size_t smem = (size_t)nw * per + tab_bytes;
  auto kern = n_other == 1 ? k_rrf_coo<4, 1>
            : n_other == 2 ? k_rrf_coo<4, 2>
            : n_other == 3 ? k_rrf_coo<4, 3>
                           : k_rrf_coo<4, 4>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t blocks = imin((int64_t)num_sms() * per_sm, (s_n + nw - 1) / nw);
  kern<<<(unsigned)blocks, nw * 32, smem, (cudaStream_t)stream>>>(
      r, oe, s_n, colptr, (const double*)rec, c1_mask, stage1);
  return check_launch("k_rrf_coo");
}
