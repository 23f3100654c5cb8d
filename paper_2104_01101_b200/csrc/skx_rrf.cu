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
#include <stdlib.h>

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

// ---- RRF stage 1 straight from the lexsorted COO, no fibre layout ----------
// st1[i_n, h(j)] += sign(j) v over the nonzeros, accumulated EXACTLY in
// fixed point with atomics: the value range of the tensor is checked once
// (skx_value_range: nonzero |v| within 2^41 of each other, all finite), so
// every contribution v * 2^S (S = 93 - emax) is an integer of magnitude below
// 2^94; it is split into three 32-bit limbs (bits 0-31 and 32-63 unsigned,
// 64-95 signed) that are summed in 64-bit cells by fire-and-forget atomic
// reductions (no carry round trips; fewer than 2^32 addends per cell cannot
// overflow), and the cells are recombined into the exact 128-bit sum, rounded
// once to double.  Integer addition is associative: the result is
// deterministic whatever the atomic order, and within the reference's own
// float rounding of the exact sum.  This removes the (i_n, others) sort that
// a deterministic ordered accumulation needs: at 1e9 nonzeros that sort costs
// ~50 ms per mode, more than the Philox work.

// max / min unbiased exponent of the nonzero |v|, and a non-finite flag
__global__ void k_value_range(const double* __restrict__ v, int64_t n, int* __restrict__ out) {
  int emax = -100000, emin = 100000, bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t b = (uint64_t)__double_as_longlong(v[i]);
    const int ex = (int)((b >> 52) & 0x7ff);
    if (ex == 0x7ff) bad = 1;
    else if (ex == 0) { if ((b << 12) != 0) bad = 1; }  // subnormal: treat as out of range
    else {
      emax = max(emax, ex - 1023);
      emin = min(emin, ex - 1023);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    emin = min(emin, __shfl_xor_sync(0xffffffffu, emin, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out + 0, emax);
    atomicMin(out + 1, emin);
    atomicOr(out + 2, bad);
  }
}

__global__ void k_value_range_init(int* out) {
  out[0] = -100000;
  out[1] = 100000;
  out[2] = 0;
}

struct CooSoA {
  const int32_t* c[5];
  int64_t ext[5];
};

// v * 2^S as a two's-complement 128-bit integer (hi, lo); |v| < 2^(Emax+1)
// and S = 94 - (Emax + 1) make the shift 0 .. 41
__device__ __forceinline__ void to_fixed(double v, int S, uint64_t& hi, uint64_t& lo) {
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  const int ex = (int)((b >> 52) & 0x7ff);
  if (ex == 0) {
    hi = lo = 0;
    return;
  }
  const uint64_t m = (b & 0xfffffffffffffULL) | 0x10000000000000ULL;
  const int sh = ex - 1023 - 52 + S;  // >= 0 by the range check
  uint64_t h = sh == 0 ? 0 : (sh >= 64 ? (m << (sh - 64)) : (m >> (64 - sh)));
  uint64_t l = sh >= 64 ? 0 : (m << sh);
  if (b >> 63) {  // negate
    l = ~l + 1;
    h = ~h + (l == 0 ? 1 : 0);
  }
  hi = h;
  lo = l;
}

// Row-count bound for the two-limb accumulation: counts of nonzeros per
// block of 2^CB consecutive rows (per-CTA shared histograms), then the max.
__global__ void __launch_bounds__(256) k_row_hist_coarse(const int32_t* __restrict__ rows,
                                                         int64_t nnz, int CB, int nbins,
                                                         unsigned int* __restrict__ hist) {
  extern __shared__ unsigned int hsm[];
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) hsm[b] = 0;
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hsm[(uint32_t)__ldcs(rows + e) >> CB], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x)
    if (hsm[b]) atomicAdd(&hist[b], hsm[b]);
}

__global__ void k_max_u32(const unsigned int* __restrict__ a, int n, unsigned int* __restrict__ out) {
  unsigned int m = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m = max(m, a[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ unsigned int w[32];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) m = max(m, w[i]);
    *out = max(m, w[0]);
  }
}

// two-limb form when every cell receives < 2^16 addends (guaranteed when the
// largest 2^CB-row block holds < 2^16 nonzeros): value = L1 2^48 + L0 with
// L0 = sum of bits 0-47 (unsigned) and L1 = sum of value >> 48 (signed,
// |.| < 2^46): 2 reductions per nonzero instead of 3.
constexpr unsigned int kFxTwoLimbMax = 1u << 16;

// d-array entries held in shared memory by the FX kernel (the rejection
// lists of configs 4-5 hold ~1e2-2.4e3 entries); larger lists read global memory
constexpr int kFxSmemD = 3072;

__device__ __forceinline__ uint64_t count_le_tab_s(const uint64_t* dsm, int64_t nd_s,
                                                   const uint64_t* dg, const uint32_t* cnt,
                                                   int shift, uint64_t j) {
  const uint64_t b = j >> shift;
  uint32_t i = cnt[b];
  const uint32_t e = cnt[b + 1];
  while (i < e && (i < nd_s ? dsm[i] : dg[i]) <= j) ++i;
  return i;
}

template <int NO, int U>
__global__ void __launch_bounds__(256) k_rrf_coo_fx(RrfRng r, CooSoA cs, int mode, int64_t nnz,
                                                    const double* __restrict__ vals, int S,
                                                    const unsigned int* __restrict__ rowmax,
                                                    unsigned long long* __restrict__ acc) {
  const bool two = *rowmax < kFxTwoLimbMax;
  __shared__ uint32_t cnt[kRrfBuckets + 1];
  __shared__ uint64_t dsm[kFxSmemD];
  uint64_t P = 1;
  int oth[NO];
#pragma unroll
  for (int k = 0; k < NO; ++k) {
    oth[k] = k + (k >= mode ? 1 : 0);
    P *= (uint64_t)cs.ext[oth[k]];
  }
  int shift = 0;
  while ((P >> shift) >= (uint64_t)kRrfBuckets) ++shift;
  for (int b = threadIdx.x; b <= kRrfBuckets; b += blockDim.x) {
    const uint64_t v = (uint64_t)b << shift;
    int64_t lo = 0, hi = r.nd;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (r.d[mid] < v) lo = mid + 1; else hi = mid;
    }
    cnt[b] = (uint32_t)lo;
  }
  const int64_t nd_s = imin(r.nd, kFxSmemD);
  for (int64_t i = threadIdx.x; i < nd_s; i += blockDim.x) dsm[i] = r.d[i];
  __syncthreads();
  const uint64_t k2 = r.k2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x) * U + threadIdx.x; base < nnz;
       base += stride) {
    // all loads of the U elements first (no early exit between them), then
    // the Philox work and the reductions
    uint32_t cc[U][NO], rw[U];
    double vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + (int64_t)u * blockDim.x;
      const int64_t ee = e < nnz ? e : base;
#pragma unroll
      for (int k = 0; k < NO; ++k) cc[u][k] = (uint32_t)__ldcs(cs.c[oth[k]] + ee);
      rw[u] = (uint32_t)__ldcs(cs.c[mode] + ee);
      vv[u] = e < nnz ? __ldcs(vals + ee) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (base + (int64_t)u * blockDim.x >= nnz) continue;
      uint64_t j = 0;
#pragma unroll
      for (int k = 0; k < NO; ++k) j = j * (uint64_t)cs.ext[oth[k]] + (uint64_t)cc[u][k];
      const uint32_t t = rrf_entry_q(r, j, j + count_le_tab_s(dsm, nd_s, r.d, cnt, shift, j));
      uint64_t hi, lo;
      to_fixed(pk_neg(t) ? -vv[u] : vv[u], S, hi, lo);
      // three 32-bit limbs (bits 0-31, 32-63 unsigned; 64-95 signed: |value|
      // < 2^94, so bits 94.. are sign copies) summed in 64-bit cells by
      // fire-and-forget reductions (no carries to wait for: < 2^32 addends)
      unsigned long long* cell = acc + 4 * ((uint64_t)rw[u] * k2 + pk_bucket(t));
      if (two) {
        atomicAdd(cell, (unsigned long long)(lo & 0xffffffffffffULL));
        atomicAdd(cell + 1, (unsigned long long)((hi << 16) | (lo >> 48)));  // value >> 48
      } else {
        atomicAdd(cell, (unsigned long long)(lo & 0xffffffffULL));
        atomicAdd(cell + 1, (unsigned long long)(lo >> 32));
        atomicAdd(cell + 2, (unsigned long long)(long long)(int32_t)(uint32_t)hi);
      }
    }
  }
}


// ---------------------------------------------------------------------------
// RRF stage 1 with L2-resident accumulators (order-3 leverage runs, config 5).
// The fixed-point accumulation above scatters 2 atomics per nonzero over the
// whole s_n x k2 accumulator (3 GB at config 5): every atomic misses L2 and
// costs a DRAM read-modify-write (ncu: ~130 GB of DRAM traffic for 20 GB of
// input, long-scoreboard bound).  Here the nonzeros are first partitioned by
// output row block -- a counting sort that needs no random numbers, so it runs
// while the compute-bound rejection scans still occupy the SMs -- into
// records {key = i_n << 40 | flat other index, value}; the stage-1 pass then
// walks the records in row-block order with all CTAs in the same region, so
// the live accumulator rows (a few MB) stay in L2.  Same integer sums, so
// the result is bitwise that of skx_rrf_stage1_fx.
constexpr int kPartTile = 65536;  // nonzeros per partition tile (256 threads x 256)
constexpr int kPartMaxBk = 256;   // row blocks per mode

struct PartPlan {
  int nmode;
  int mode[2];
  int shift[2];  // row block = i_n >> shift
  int nbk[2];
};

__global__ void __launch_bounds__(256) k_part_count(CooSoA cs, int64_t nnz, PartPlan pp,
                                                    int64_t ntile, unsigned long long* __restrict__ cnt) {
  __shared__ unsigned int h[2][kPartMaxBk];
  for (int t = blockIdx.x; t < ntile; t += gridDim.x) {
    for (int i = threadIdx.x; i < 2 * kPartMaxBk; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    const int64_t e0 = (int64_t)t * kPartTile, e1 = imin(e0 + kPartTile, nnz);
    for (int md = 0; md < pp.nmode; ++md) {
      const int32_t* rows = cs.c[pp.mode[md]];
      for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x)
        atomicAdd(&h[md][(uint32_t)__ldcs(rows + e) >> pp.shift[md]], 1u);
    }
    __syncthreads();
    // bucket-major layout [mode][bucket][tile]: one exclusive scan per mode
    // gives every (bucket, tile) its first output slot
    for (int md = 0; md < pp.nmode; ++md)
      for (int b = threadIdx.x; b < pp.nbk[md]; b += blockDim.x)
        cnt[((int64_t)md * kPartMaxBk + b) * ntile + t] = h[md][b];
    __syncthreads();
  }
}

template <int NO>
__global__ void __launch_bounds__(256) k_part_scatter(CooSoA cs, int64_t nnz,
                                                      const double* __restrict__ vals, PartPlan pp,
                                                      int64_t ntile, const unsigned long long* off,
                                                      uint64_t* __restrict__ key0, double* __restrict__ val0,
                                                      uint64_t* __restrict__ key1, double* __restrict__ val1) {
  __shared__ unsigned long long pos[2][kPartMaxBk];
  for (int t = blockIdx.x; t < ntile; t += gridDim.x) {
    for (int md = 0; md < pp.nmode; ++md)
      for (int b = threadIdx.x; b < pp.nbk[md]; b += blockDim.x)
        pos[md][b] = off[((int64_t)md * kPartMaxBk + b) * ntile + t];
    __syncthreads();
    const int64_t e0 = (int64_t)t * kPartTile, e1 = imin(e0 + kPartTile, nnz);
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      uint32_t c[NO + 1];
#pragma unroll
      for (int k = 0; k <= NO; ++k) c[k] = (uint32_t)__ldcs(cs.c[k] + e);
      const double v = __ldcs(vals + e);
#pragma unroll
      for (int md = 0; md < 2; ++md) {
        if (md >= pp.nmode) break;
        const int mode = pp.mode[md];
        uint64_t j = 0;
#pragma unroll
        for (int k = 0; k <= NO; ++k)
          if (k != mode) j = j * (uint64_t)cs.ext[k] + c[k];
        const unsigned long long p = atomicAdd(&pos[md][c[mode] >> pp.shift[md]], 1ull);
        const uint64_t key = ((uint64_t)c[mode] << 40) | j;
        if (md == 0) {
          __stcs(reinterpret_cast<unsigned long long*>(key0) + p, key);
          __stcs(val0 + p, v);
        } else {
          __stcs(reinterpret_cast<unsigned long long*>(key1) + p, key);
          __stcs(val1 + p, v);
        }
      }
    }
    __syncthreads();
  }
}

// k_rrf_coo_fx over partitioned records (key = i_n << 40 | j, value)
template <int U>
__global__ void __launch_bounds__(256) k_rrf_rec_fx(RrfRng r, uint64_t P, int64_t nnz,
                                                    const uint64_t* __restrict__ keys,
                                                    const double* __restrict__ vals, int S,
                                                    const unsigned int* __restrict__ rowmax,
                                                    unsigned long long* __restrict__ acc) {
  const bool two = *rowmax < kFxTwoLimbMax;
  __shared__ uint32_t cnt[kRrfBuckets + 1];
  __shared__ uint64_t dsm[kFxSmemD];
  int shift = 0;
  while ((P >> shift) >= (uint64_t)kRrfBuckets) ++shift;
  for (int b = threadIdx.x; b <= kRrfBuckets; b += blockDim.x) {
    const uint64_t v = (uint64_t)b << shift;
    int64_t lo = 0, hi = r.nd;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (r.d[mid] < v) lo = mid + 1; else hi = mid;
    }
    cnt[b] = (uint32_t)lo;
  }
  const int64_t nd_s = imin(r.nd, kFxSmemD);
  for (int64_t i = threadIdx.x; i < nd_s; i += blockDim.x) dsm[i] = r.d[i];
  __syncthreads();
  const uint64_t k2 = r.k2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x) * U + threadIdx.x; base < nnz;
       base += stride) {
    uint64_t kk[U];
    double vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + (int64_t)u * blockDim.x;
      const int64_t ee = e < nnz ? e : base;
      kk[u] = __ldcs(reinterpret_cast<const unsigned long long*>(keys) + ee);
      vv[u] = e < nnz ? __ldcs(vals + ee) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (base + (int64_t)u * blockDim.x >= nnz) continue;
      const uint64_t j = kk[u] & ((uint64_t(1) << 40) - 1);
      const uint32_t row = (uint32_t)(kk[u] >> 40);
      const uint32_t t = rrf_entry_q(r, j, j + count_le_tab_s(dsm, nd_s, r.d, cnt, shift, j));
      uint64_t hi, lo;
      to_fixed(pk_neg(t) ? -vv[u] : vv[u], S, hi, lo);
      unsigned long long* cell = acc + 4 * ((uint64_t)row * k2 + pk_bucket(t));
      if (two) {
        atomicAdd(cell, (unsigned long long)(lo & 0xffffffffffffULL));
        atomicAdd(cell + 1, (unsigned long long)((hi << 16) | (lo >> 48)));
      } else {
        atomicAdd(cell, (unsigned long long)(lo & 0xffffffffULL));
        atomicAdd(cell + 1, (unsigned long long)(lo >> 32));
        atomicAdd(cell + 2, (unsigned long long)(long long)(int32_t)(uint32_t)hi);
      }
    }
  }
}

// st1 = double(acc) * 2^-S, correctly rounded
__global__ void k_fixed_to_double(const unsigned long long* __restrict__ acc, int64_t n, int S,
                                  const unsigned int* __restrict__ rowmax,
                                  double* __restrict__ out) {
  const bool two = *rowmax < kFxTwoLimbMax;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t lo, hi;
    if (two) {  // value = L1 2^48 + L0 (L0 unsigned, L1 signed)
      const uint64_t L0 = acc[4 * i], L1 = acc[4 * i + 1];
      const uint64_t low = L1 << 48;
      lo = low + L0;
      hi = (uint64_t)((int64_t)L1 >> 16) + (lo < low ? 1ULL : 0ULL);
    } else {  // value = L2 2^64 + L1 2^32 + L0 (L0, L1 unsigned sums, L2 signed)
      const uint64_t L0 = acc[4 * i], L1 = acc[4 * i + 1], L2 = acc[4 * i + 2];
      lo = L0 + (L1 << 32);
      hi = (L1 >> 32) + (lo < L0 ? 1ULL : 0ULL) + L2;
    }
    const bool neg = (hi >> 63) != 0;
    if (neg) {
      lo = ~lo + 1;
      hi = ~hi + (lo == 0 ? 1 : 0);
    }
    double d;
    if (hi == 0 && lo == 0) {
      d = 0.0;
    } else {
      // leading bit position, take 53 bits, round to nearest even on the rest
      const int lz = hi ? __clzll((long long)hi) : 64 + __clzll((long long)lo);
      const int top = 127 - lz;  // index of the leading one
      uint64_t mant;
      bool half = false, sticky = false;
      if (top < 53) {
        mant = lo;  // exact
      } else {
        const int drop = top - 52;  // bits below the 53-bit mantissa
        // mant = (hi:lo) >> drop
        mant = drop >= 64 ? (hi >> (drop - 64)) : ((lo >> drop) | (drop ? (hi << (64 - drop)) : 0));
        // the dropped bits
        uint64_t rl, rh;  // (hi:lo) & ((1 << drop) - 1)
        if (drop >= 64) {
          rl = lo;
          rh = drop == 64 ? 0 : (hi & ((1ULL << (drop - 64)) - 1));
        } else {
          rl = lo & ((1ULL << drop) - 1);
          rh = 0;
        }
        // half = bit drop-1, sticky = any lower bit
        const int hb = drop - 1;
        half = hb >= 64 ? ((rh >> (hb - 64)) & 1) : ((rl >> hb) & 1);
        if (hb >= 64) sticky = (rl != 0) || ((rh & ((1ULL << (hb - 64)) - 1)) != 0);
        else sticky = (rl & ((1ULL << hb) - 1)) != 0;
        if (half && (sticky || (mant & 1))) ++mant;  // may carry to 2^53: still exact in double
        d = ldexp((double)mant, drop);
        d = ldexp(d, -S);
        out[i] = neg ? -d : d;
        continue;
      }
      d = (double)mant;
    }
    d = ldexp(d, -S);
    out[i] = neg ? -d : d;
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

extern "C" int skx_value_range(const double* vals, int64_t nnz, int* out3, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  k_value_range_init<<<1, 1, 0, st>>>(out3);
  if (nnz > 0) {
    const unsigned g = (unsigned)imin((nnz + 255) / 256, (int64_t)num_sms() * 8);
    k_value_range<<<g, 256, 0, st>>>(vals, nnz, out3);
  }
  return check_launch("k_value_range", nnz > 0 ? 2 : 1);
}

extern "C" int skx_rrf_stage1_fx(int ndim, const int64_t* shape_h, int mode, int64_t nnz,
                                 const int32_t* coords, const double* vals, int emax, uint64_t k0,
                                 uint64_t k1, uint64_t p0, uint32_t has_pending, uint32_t pending,
                                 uint64_t sign_q0, const uint64_t* rej, int64_t nrej, int64_t k2,
                                 double* stage1, void* ws, size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(ndim >= 2 && ndim <= 5, "skx_rrf_stage1_fx: order 2..5");
  SKX_REQUIRE(mode >= 0 && mode < ndim, "skx_rrf_stage1_fx: mode out of range");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_rrf_stage1_fx: ws_bytes is NULL");
  SKX_REQUIRE(nnz < (int64_t(1) << 32), "skx_rrf_stage1_fx: more than 2^32 nonzeros");
  SKX_REQUIRE(nrej < (int64_t(1) << 32), "skx_rrf_stage1_fx: rejection list too long");
  const int64_t sn = shape_h[mode];
  const int64_t cells = sn * k2;
  // (grouping the nonzeros by row block first, so the atomics hit an
  // L2-resident slice of the accumulators, measured no faster: the
  // reductions are bound by the L2 atomic units, not by HBM)
  // coarse row histogram: blocks of 2^CB rows, at most 32768 bins (128 KB of
  // shared memory): 8-row blocks up to s_n = 262144 (config 5: ~40000
  // nonzeros per block, under the 2^16 two-limb bound)
  int CB = 0;
  while (((sn + (int64_t(1) << CB) - 1) >> CB) > 32768) ++CB;
  const int nbins = (int)((sn + (int64_t(1) << CB) - 1) >> CB);
  Arena ar(ws, *ws_bytes);
  unsigned long long* acc = ar.take<unsigned long long>((size_t)cells * 4);
  unsigned int* hist = ar.take<unsigned int>((size_t)nbins + 1);
  unsigned int* rowmax = ar.take<unsigned int>(1);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_rrf_stage1_fx: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int S = 94 - (emax + 1);
  cudaMemsetAsync(acc, 0, (size_t)cells * 32, st);
  cudaMemsetAsync(hist, 0, ((size_t)nbins + 1) * sizeof(unsigned int), st);
  int launches = nnz > 0 ? 2 : 1;
  {
    const size_t hs = (size_t)nbins * sizeof(unsigned int);
    cudaFuncSetAttribute(k_row_hist_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hs);
    if (nnz > 0)
      k_row_hist_coarse<<<(unsigned)imin((nnz + 255) / 256, (int64_t)num_sms() * 2), 256, hs, st>>>(
          coords + (int64_t)mode * nnz, nnz, CB, nbins, hist);
    k_max_u32<<<1, 1024, 0, st>>>(hist, nbins, rowmax);
  }
  if (nnz > 0) {
    RrfRng r = make_rng(k0, k1, p0, has_pending, pending, sign_q0, rej, nrej, k2);
    CooSoA cs{};
    for (int k = 0; k < ndim; ++k) {
      cs.c[k] = coords + (int64_t)k * nnz;
      cs.ext[k] = shape_h[k];
    }
    constexpr int U = 4;
    auto kern = ndim == 2 ? k_rrf_coo_fx<1, U>
              : ndim == 3 ? k_rrf_coo_fx<2, U>
              : ndim == 4 ? k_rrf_coo_fx<3, U>
                          : k_rrf_coo_fx<4, U>;
    // One 256-thread CTA per SM, grid-stride: the pass is bound by the L2
    // atomic rate (~2 reductions per nonzero), not by SM resources -- with
    // every resident slot taken (8 CTAs per SM) it ran no faster (60.3 vs 60.8
    // ms per mode at config 5) but starved the rejection scan it overlaps
    // (84 -> 75 ms per scan, 480 -> 457 ms per call).  SKX_FX_BLOCKS: A/B.
    int64_t nblk = num_sms();
    if (const char* b = getenv("SKX_FX_BLOCKS")) nblk = imax(1, atoll(b));
    const int64_t blocks = imax(1, imin((nnz + 256 * U - 1) / (256 * U), nblk));
    kern<<<(unsigned)blocks, 256, 0, st>>>(r, cs, mode, nnz, vals, S, rowmax, acc);
    ++launches;
  }
  const unsigned g = (unsigned)imin((cells + 255) / 256, (int64_t)num_sms() * 16);
  k_fixed_to_double<<<g, 256, 0, st>>>(acc, cells, S, rowmax, stage1);
  return check_launch("skx_rrf_stage1_fx", launches + 1);
}

// Chunk-wise form of skx_rrf_stage1_fx for a COO tensor that arrives in
// pieces (host upload pipelined with the sketch): the caller owns the
// accumulator (s_mode x k2 cells of 32 bytes, zeroed), adds chunk after chunk
// (coords = first nonzero of the chunk in each of the ndim SoA rows, rows ld
// apart) and finally converts.  Same sums as the one-shot call.  max_per_cell:
// the caller's bound on the nonzeros of any 2^CB-row block of the mode (from
// the host staging), or -1 when unknown -- two-limb reductions when it is
// below 2^16, else three.
__global__ void k_u32_set(unsigned int* p, unsigned int v) { *p = v; }

extern "C" int skx_rrf_stage1_fx_acc(int ndim, const int64_t* shape_h, int mode, int64_t n,
                                     const int32_t* coords, int64_t ld, const double* vals,
                                     int emax, uint64_t k0, uint64_t k1, uint64_t p0,
                                     uint32_t has_pending, uint32_t pending, uint64_t sign_q0,
                                     const uint64_t* rej, int64_t nrej, int64_t k2,
                                     unsigned long long* acc, unsigned int* limb_flag,
                                     int64_t max_per_cell, void* stream) {
  SKX_REQUIRE(ndim >= 2 && ndim <= 5, "skx_rrf_stage1_fx_acc: order 2..5");
  SKX_REQUIRE(mode >= 0 && mode < ndim, "skx_rrf_stage1_fx_acc: mode out of range");
  SKX_REQUIRE(nrej < (int64_t(1) << 32), "skx_rrf_stage1_fx_acc: rejection list too long");
  cudaStream_t st = (cudaStream_t)stream;
  k_u32_set<<<1, 1, 0, st>>>(limb_flag, (max_per_cell >= 0 && max_per_cell < 0xffffffffLL)
                                            ? (unsigned int)max_per_cell : 0xffffffffu);
  if (n <= 0) return check_launch("skx_rrf_stage1_fx_acc", 1);
  RrfRng r = make_rng(k0, k1, p0, has_pending, pending, sign_q0, rej, nrej, k2);
  CooSoA cs{};
  for (int k = 0; k < ndim; ++k) {
    cs.c[k] = coords + (int64_t)k * ld;
    cs.ext[k] = shape_h[k];
  }
  constexpr int U = 4;
  auto kern = ndim == 2 ? k_rrf_coo_fx<1, U>
            : ndim == 3 ? k_rrf_coo_fx<2, U>
            : ndim == 4 ? k_rrf_coo_fx<3, U>
                        : k_rrf_coo_fx<4, U>;
  // one CTA per SM (atomic-rate bound; see skx_rrf_stage1_fx)
  int64_t nblk = num_sms();
  if (const char* b = getenv("SKX_FX_BLOCKS")) nblk = imax(1, atoll(b));
  const int64_t blocks = imax(1, imin((n + 256 * U - 1) / (256 * U), nblk));
  kern<<<(unsigned)blocks, 256, 0, st>>>(r, cs, mode, n, vals, 94 - (emax + 1), limb_flag, acc);
  return check_launch("skx_rrf_stage1_fx_acc", 2);
}

extern "C" int skx_rrf_stage1_fx_convert(const unsigned long long* acc, int64_t cells, int emax,
                                         const unsigned int* limb_flag, double* stage1,
                                         void* stream) {
  if (cells <= 0) return SKX_OK;
  const unsigned g = (unsigned)imin((cells + 255) / 256, (int64_t)num_sms() * 16);
  k_fixed_to_double<<<g, 256, 0, (cudaStream_t)stream>>>(acc, cells, 94 - (emax + 1), limb_flag,
                                                         stage1);
  return check_launch("k_fixed_to_double");
}

// Partition of an order-3..5 COO by output row block for up to two modes
// (the RRF modes of a leverage run): records {key = i_n << 40 | j, value},
// j the flat other-mode index (others ascending, first slowest), grouped by
// row block i_n >> shift (order inside a block is not fixed -- stage 1's
// integer sums do not depend on it).
extern "C" int skx_rrf_partition(int ndim, const int64_t* shape_h, int64_t nnz,
                                 const int32_t* coords, const double* vals, int nmode,
                                 const int* modes_h, uint64_t* key0, double* val0, uint64_t* key1,
                                 double* val1, void* ws, size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(ndim >= 2 && ndim <= 5, "skx_rrf_partition: order 2..5");
  SKX_REQUIRE(nmode >= 1 && nmode <= 2, "skx_rrf_partition: one or two modes");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_rrf_partition: ws_bytes is NULL");
  PartPlan pp{};
  pp.nmode = nmode;
  uint64_t P[2] = {1, 1};
  for (int md = 0; md < nmode; ++md) {
    const int mode = modes_h[md];
    SKX_REQUIRE(mode >= 0 && mode < ndim, "skx_rrf_partition: mode out of range");
    pp.mode[md] = mode;
    int sh = 0;
    while (((shape_h[mode] + (int64_t(1) << sh) - 1) >> sh) > kPartMaxBk) ++sh;
    pp.shift[md] = sh;
    pp.nbk[md] = (int)((shape_h[mode] + (int64_t(1) << sh) - 1) >> sh);
    SKX_REQUIRE(shape_h[mode] < (int64_t(1) << 24), "skx_rrf_partition: extent too large");
    for (int k = 0; k < ndim; ++k)
      if (k != mode) P[md] *= (uint64_t)shape_h[k];
    SKX_REQUIRE(P[md] < (uint64_t(1) << 40), "skx_rrf_partition: other-mode index beyond 2^40");
  }
  const int64_t ntile = (nnz + kPartTile - 1) / kPartTile;
  const size_t ncnt = (size_t)2 * kPartMaxBk * (size_t)imax(ntile, 1);
  Arena ar(ws, *ws_bytes);
  unsigned long long* cnt = ar.take<unsigned long long>(ncnt);
  unsigned long long* off = ar.take<unsigned long long>(ncnt);
  size_t cb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cb, cnt, off, (int)(kPartMaxBk * imax(ntile, 1)));
  void* tmp = ar.take<char>(cb);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_rrf_partition: workspace too small");
  if (nnz == 0) return SKX_OK;
  cudaStream_t st = (cudaStream_t)stream;
  CooSoA cs{};
  for (int k = 0; k < ndim; ++k) {
    cs.c[k] = coords + (int64_t)k * nnz;
    cs.ext[k] = shape_h[k];
  }
  const unsigned g = (unsigned)imin(ntile, (int64_t)num_sms() * 8);
  k_part_count<<<g, 256, 0, st>>>(cs, nnz, pp, ntile, cnt);
  for (int md = 0; md < nmode; ++md) {
    const size_t o = (size_t)md * kPartMaxBk * ntile;
    size_t cb2 = cb;
    cub::DeviceScan::ExclusiveSum(tmp, cb2, cnt + o, off + o, (int)(pp.nbk[md] * ntile), st);
  }
  auto kern = ndim == 2 ? k_part_scatter<1>
            : ndim == 3 ? k_part_scatter<2>
            : ndim == 4 ? k_part_scatter<3>
                        : k_part_scatter<4>;
  kern<<<g, 256, 0, st>>>(cs, nnz, vals, pp, ntile, off, key0, val0, key1, val1);
  return check_launch("skx_rrf_partition", 2 + 2 * nmode);
}

// RRF stage 1 of one mode from its partitioned records (skx_rrf_partition):
// same exact fixed-point sums as skx_rrf_stage1_fx, accumulators hit in L2.
// rows: the mode's coordinate row of the COO (for the limb-count bound).
extern "C" int skx_rrf_stage1_rec(int64_t sn, uint64_t P, int64_t nnz, const int32_t* rows,
                                  const uint64_t* keys, const double* vals, int emax, uint64_t k0,
                                  uint64_t k1, uint64_t p0, uint32_t has_pending, uint32_t pending,
                                  uint64_t sign_q0, const uint64_t* rej, int64_t nrej, int64_t k2,
                                  double* stage1, void* ws, size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(ws_bytes != nullptr, "skx_rrf_stage1_rec: ws_bytes is NULL");
  SKX_REQUIRE(nrej < (int64_t(1) << 32), "skx_rrf_stage1_rec: rejection list too long");
  const int64_t cells = sn * k2;
  int CB = 0;
  while (((sn + (int64_t(1) << CB) - 1) >> CB) > 32768) ++CB;
  const int nbins = (int)((sn + (int64_t(1) << CB) - 1) >> CB);
  Arena ar(ws, *ws_bytes);
  unsigned long long* acc = ar.take<unsigned long long>((size_t)cells * 4);
  unsigned int* hist = ar.take<unsigned int>((size_t)nbins + 1);
  unsigned int* rowmax = ar.take<unsigned int>(1);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_rrf_stage1_rec: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int S = 94 - (emax + 1);
  cudaMemsetAsync(acc, 0, (size_t)cells * 32, st);
  cudaMemsetAsync(hist, 0, ((size_t)nbins + 1) * sizeof(unsigned int), st);
  int launches = 1;
  {
    const size_t hs = (size_t)nbins * sizeof(unsigned int);
    cudaFuncSetAttribute(k_row_hist_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hs);
    if (nnz > 0) {
      k_row_hist_coarse<<<(unsigned)imin((nnz + 255) / 256, (int64_t)num_sms() * 2), 256, hs, st>>>(
          rows, nnz, CB, nbins, hist);
      ++launches;
    }
    k_max_u32<<<1, 1024, 0, st>>>(hist, nbins, rowmax);
  }
  if (nnz > 0) {
    RrfRng r = make_rng(k0, k1, p0, has_pending, pending, sign_q0, rej, nrej, k2);
    constexpr int U = 4;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rrf_rec_fx<U>, 256, 0);
    if (per_sm < 1) per_sm = 1;
    const int64_t blocks =
        imax(1, imin((nnz + 256 * U - 1) / (256 * U), (int64_t)num_sms() * per_sm));
    k_rrf_rec_fx<U><<<(unsigned)blocks, 256, 0, st>>>(r, P, nnz, keys, vals, S, rowmax, acc);
    ++launches;
  }
  const unsigned g = (unsigned)imin((cells + 255) / 256, (int64_t)num_sms() * 16);
  k_fixed_to_double<<<g, 256, 0, st>>>(acc, cells, S, rowmax, stage1);
  return check_launch("skx_rrf_stage1_rec", launches + 1);
}
