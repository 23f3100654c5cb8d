// Device layouts of a COO tensor (the B200 counterpart of the reference's
// cached unfoldings, src/tensors.py:151-194 / mode_sort :89-95).
//
// Fibre-major layout of mode n: nonzeros ordered by (i_n, other modes
// ascending) -- a stable sort by i_n of the lexsorted input -- stored as
// AoS records {int32 other coords..., double value} so a sketch kernel reads
// one 16-byte record per nonzero (order 3), plus int64 column offsets colptr.
// Built by one packing pass and a cub onesweep radix sort over only the
// ceil(log2 s_n) key bits (skipped for mode 0, already in order).
#include <cub/cub.cuh>

#include <string.h>

#include <vector>

#include "skx_common.cuh"

namespace skx {

struct __align__(16) Rec16 {
  int32_t c[2];
  double v;
};
struct __align__(8) Rec24 {
  int32_t c[4];
  double v;
};

// Optional TensorSketch packing (order 3): the composite bucket h and sign of
// the record's other-mode pair are stored in the spare high bits of the second
// coordinate word -- c1 | h << bb | neg << 31 -- so the RHS sketch of this mode
// needs no table lookups.  Consumers recover c1 with the mask (1 << bb) - 1.
struct TsPack {
  const uint32_t* ta;  // packed table of the first other mode (NULL: no packing)
  const uint32_t* tb;  // of the second other mode
  uint32_t m;
  int bb;
};

// Slot j of a record holds mode j + (j >= mode): compile-time slot indices keep
// the record in registers (a runtime-indexed array would live in local memory).
template <class Rec>
__global__ void k_pack(int ndim, int mode, int64_t nnz, const int32_t* __restrict__ coords,
                       const double* __restrict__ vals, uint32_t* __restrict__ keys,
                       Rec* __restrict__ rec, TsPack tp) {
  constexpr int NS = (int)(sizeof(Rec::c) / sizeof(int32_t));
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  Rec r;
#pragma unroll
  for (int j = 0; j < NS; ++j) {
    const int src = j + (j >= mode ? 1 : 0);
    r.c[j] = (j < ndim - 1) ? __ldcs(coords + (int64_t)src * nnz + e) : 0;
  }
  if (NS == 2 && tp.ta != nullptr) {
    const uint32_t a = __ldg(tp.ta + r.c[0]), b = __ldg(tp.tb + r.c[1]);
    uint32_t h = pk_bucket(a) + pk_bucket(b);
    if (h >= tp.m) h -= tp.m;
    r.c[1] = (int32_t)((uint32_t)r.c[1] | (h << tp.bb) | ((a ^ b) & 0x80000000u));
  }
  r.v = __ldcs(vals + e);
  rec[e] = r;
  if (keys) keys[e] = (uint32_t)__ldcs(coords + (int64_t)mode * nnz + e);
}

// Records [lo, hi) of a packing pass whose coordinate rows have stride ld
// (chunk-wise mode-0 layout of a COO that arrives in pieces)
template <class Rec>
__global__ void k_pack_range(int ndim, int mode, int64_t ld, int64_t lo, int64_t hi,
                             const int32_t* __restrict__ coords, const double* __restrict__ vals,
                             Rec* __restrict__ rec) {
  constexpr int NS = (int)(sizeof(Rec::c) / sizeof(int32_t));
  const int64_t e = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= hi) return;
  Rec r;
#pragma unroll
  for (int j = 0; j < NS; ++j) {
    const int src = j + (j >= mode ? 1 : 0);
    r.c[j] = (j < ndim - 1) ? __ldcs(coords + (int64_t)src * ld + e) : 0;
  }
  r.v = __ldcs(vals + e);
  rec[e] = r;
}

// colptr[c] = first position whose key >= c (keys sorted), c in [0, s]
__global__ void k_bounds_u32(const uint32_t* __restrict__ keys, int64_t n, int64_t s,
                             int64_t* __restrict__ colptr) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c > s) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)keys[mid] < c) lo = mid + 1; else hi = mid;
  }
  colptr[c] = lo;
}

__global__ void k_bounds_i32(const int32_t* __restrict__ keys, int64_t n, int64_t s,
                             int64_t* __restrict__ colptr) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c > s) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)keys[mid] < c) lo = mid + 1; else hi = mid;
  }
  colptr[c] = lo;
}

// Modes >= 1: records are packed in input order with their i_n keys and
// radix-sorted as (key, record) pairs -- a stable sort by i_n.  (Sorting
// (key, position) pairs and gathering the records afterwards moves fewer bytes
// per pass, but the random 16-byte gather measured slower at 1e8-1e9 nnz.)
template <class Rec>
static int build(int ndim, const int64_t* shape_h, int mode, int64_t nnz, const int32_t* coords,
                 const double* vals, void* rec_out, int64_t* colptr, void* ws, size_t* ws_bytes,
                 cudaStream_t s, TsPack tp = TsPack{nullptr, nullptr, 0, 0}) {
  const int64_t sn = shape_h[mode];
  Arena ar(ws, *ws_bytes);
  uint32_t* k_in = nullptr;
  uint32_t* k_out = nullptr;
  Rec* r_in = nullptr;
  void* tmp = nullptr;
  size_t cb = 0;
  if (mode != 0) {
    k_in = ar.take<uint32_t>(nnz);
    k_out = ar.take<uint32_t>(nnz);
    r_in = ar.take<Rec>(nnz);
    cub::DeviceRadixSort::SortPairs(nullptr, cb, k_in, k_out, r_in, (Rec*)rec_out, (int64_t)nnz, 0,
                                    32, s);
    tmp = ar.take<char>(cb);
  }
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_coo_fibre: workspace too small");
  SKX_REQUIRE(nnz < (int64_t(1) << 32), "skx_coo_fibre: more than 2^32 nonzeros per shard");
  const unsigned g = (unsigned)((nnz + 255) / 256);
  const unsigned gb = (unsigned)((sn + 1 + 255) / 256);
  if (mode == 0) {
    if (nnz) k_pack<Rec><<<g, 256, 0, s>>>(ndim, 0, nnz, coords, vals, nullptr, (Rec*)rec_out, tp);
    k_bounds_i32<<<gb, 256, 0, s>>>(coords, nnz, sn, colptr);
    return check_launch("skx_coo_fibre(mode 0)", 2);
  }
  int bits = 1;
  while ((int64_t(1) << bits) < sn) ++bits;
  if (nnz) k_pack<Rec><<<g, 256, 0, s>>>(ndim, mode, nnz, coords, vals, k_in, r_in, tp);
  cub::DeviceRadixSort::SortPairs(tmp, cb, k_in, k_out, r_in, (Rec*)rec_out, (int64_t)nnz, 0, bits,
                                  s);
  k_bounds_u32<<<gb, 256, 0, s>>>(k_out, nnz, sn, colptr);
  return check_launch("skx_coo_fibre", 3);
}

}  // namespace skx

using namespace skx;

extern "C" int skx_coo_rec_words(int ndim) { return ndim - 1 <= 2 ? 2 : (ndim - 1 <= 4 ? 3 : -1); }

extern "C" int skx_coo_fibre(int ndim, const int64_t* shape_h, int mode, int64_t nnz,
                             const int32_t* coords, const double* vals, void* rec_out,
                             int64_t* colptr, void* ws, size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(ndim >= 2 && ndim <= 5, "skx_coo_fibre: sparse order 2..5 supported");
  SKX_REQUIRE(mode >= 0 && mode < ndim, "skx_coo_fibre: mode out of range");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_coo_fibre: ws_bytes is NULL");
  for (int k = 0; k < ndim; ++k)
    SKX_REQUIRE(shape_h[k] >= 1 && shape_h[k] < (int64_t(1) << 31), "skx_coo_fibre: extent range");
  cudaStream_t s = (cudaStream_t)stream;
  if (ndim - 1 <= 2)
    return build<Rec16>(ndim, shape_h, mode, nnz, coords, vals, rec_out, colptr, ws, ws_bytes, s);
  return build<Rec24>(ndim, shape_h, mode, nnz, coords, vals, rec_out, colptr, ws, ws_bytes, s);
}

// Chunk of the mode-0 fibre layout of a lexsorted COO (records in input
// order; colptr = the mode-0 slice pointers): the records of nonzeros
// [lo, hi) from coordinate rows of stride ld.  Built as the chunks of a host
// upload land, so the layout is complete with the last chunk.
extern "C" int skx_coo_pack0_range(int ndim, int64_t ld, int64_t lo, int64_t hi,
                                   const int32_t* coords, const double* vals, void* rec_out,
                                   void* stream) {
  SKX_REQUIRE(ndim >= 2 && ndim <= 5, "skx_coo_pack0_range: sparse order 2..5 supported");
  SKX_REQUIRE(lo >= 0 && lo <= hi && hi <= ld, "skx_coo_pack0_range: bad range");
  if (hi == lo) return SKX_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned g = (unsigned)((hi - lo + 255) / 256);
  if (ndim - 1 <= 2)
    k_pack_range<Rec16><<<g, 256, 0, s>>>(ndim, 0, ld, lo, hi, coords, vals, (Rec16*)rec_out);
  else
    k_pack_range<Rec24><<<g, 256, 0, s>>>(ndim, 0, ld, lo, hi, coords, vals, (Rec24*)rec_out);
  return check_launch("skx_coo_pack0_range");
}

static int bits_for(int64_t n) {  // bits to hold 0..n-1
  int b = 0;
  while ((int64_t(1) << b) < n) ++b;
  return b;
}

extern "C" int skx_coo_fibre_ts(const int64_t* shape_h, int mode, int64_t nnz,
                                const int32_t* coords, const double* vals, const uint32_t* tab,
                                const int64_t* tab_off_h, int64_t m, void* rec_out,
                                int64_t* colptr, uint32_t* c1_mask, void* ws, size_t* ws_bytes,
                                void* stream) {
  SKX_REQUIRE(mode >= 0 && mode < 3, "skx_coo_fibre_ts: mode out of range (order 3)");
  SKX_REQUIRE(ws_bytes != nullptr && c1_mask != nullptr, "skx_coo_fibre_ts: NULL output");
  for (int k = 0; k < 3; ++k)
    SKX_REQUIRE(shape_h[k] >= 1 && shape_h[k] < (int64_t(1) << 31), "skx_coo_fibre_ts: extent range");
  const int b_other = mode == 2 ? 1 : 2;  // second other mode
  const int bb = bits_for(shape_h[b_other]);
  SKX_REQUIRE(m >= 1 && bb + bits_for(m) <= 31,
              "skx_coo_fibre_ts: %d coordinate bits + bucket bits of m=%lld exceed 31", bb,
              (long long)m);
  *c1_mask = bb >= 32 ? 0xffffffffu : ((1u << bb) - 1u);
  TsPack tp{tab + tab_off_h[0], tab + tab_off_h[1], (uint32_t)m, bb};
  return build<Rec16>(3, shape_h, mode, nnz, coords, vals, rec_out, colptr, ws, ws_bytes,
                      (cudaStream_t)stream, tp);
}

// ---------------------------------------------------------------------------
// Compact host staging of a lexsorted order-3 COO (SparseTensor.from_sorted):
// the mode-0 coordinate as slice pointers ptr0 (s_0 + 1 int64), and per
// nonzero ONE uint32: (d << b2) | i2, where d = i1 - (previous i1 in the same
// slice) (the first of a slice: i1 itself) -- lexsorted, so d >= 0 -- with
// the escape d = 2^(32-b2) - 1 for the rare value that does not fit (the full
// i1 is then in the sorted exception list).  4 bytes of coordinates per
// nonzero cross PCIe instead of 12; this kernel restores the int32 SoA device
// layout (3 rows of ld) for the slices [s_lo, s_hi): warp per slice, a
// segmented scan of the deltas (an escape restarts the running sum).
namespace skx {
__global__ void __launch_bounds__(256) k_coo_unpack3(const int64_t* __restrict__ ptr0, int64_t s_lo,
                                                     int64_t s_hi, const uint32_t* __restrict__ packed,
                                                     int b2, const int64_t* __restrict__ exc_idx,
                                                     const int32_t* __restrict__ exc_val,
                                                     int64_t n_exc, int32_t* __restrict__ coords,
                                                     int64_t ld) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t tw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t m2 = (1u << b2) - 1u, esc = (1u << (32 - b2)) - 1u;
  for (int64_t s = s_lo + gw; s < s_hi; s += tw) {
    const int64_t e0 = ptr0[s], e1 = ptr0[s + 1];
    int32_t carry = 0;
    for (int64_t base = e0; base < e1; base += 32) {
      const int64_t e = base + lane;
      int32_t v = 0, i2 = 0;
      bool abs_ = false;
      if (e < e1) {
        const uint32_t w = __ldcs(packed + e);
        i2 = (int32_t)(w & m2);
        const uint32_t d = w >> b2;
        if (d == esc) {  // full i1 from the exception list
          int64_t lo = 0, hi = n_exc;
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (exc_idx[mid] < e) lo = mid + 1; else hi = mid;
          }
          v = exc_val[lo];
          abs_ = true;
        } else {
          v = (int32_t)d;
          abs_ = (e == e0);  // the first of a slice is stored absolute (d = i1)
        }
      }
      // inclusive segmented scan: an absolute entry restarts the sum
      int32_t sum = v;
      bool seg = abs_;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t ps = __shfl_up_sync(0xffffffffu, sum, o);
        const bool pf = __shfl_up_sync(0xffffffffu, seg, o);
        if (lane >= o && !seg) {
          sum += ps;
          seg = pf;
        }
      }
      const int32_t i1 = seg ? sum : sum + carry;
      if (e < e1) {
        __stcs(coords + e, (int32_t)s);
        __stcs(coords + ld + e, i1);
        __stcs(coords + 2 * ld + e, i2);
      }
      carry = __shfl_sync(0xffffffffu, i1, 31);
      // (lanes past e1 hold garbage; the loop ends there)
    }
  }
}

}  // namespace skx

extern "C" int skx_coo_unpack3(const int64_t* ptr0, int64_t s_lo, int64_t s_hi,
                               const uint32_t* packed, int b2, const int64_t* exc_idx,
                               const int32_t* exc_val, int64_t n_exc, int32_t* coords, int64_t ld,
                               void* stream) {
  using namespace skx;
  SKX_REQUIRE(b2 >= 1 && b2 <= 24, "skx_coo_unpack3: 1 <= b2 <= 24");
  SKX_REQUIRE(s_lo >= 0 && s_hi >= s_lo, "skx_coo_unpack3: bad slice range");
  if (s_hi == s_lo) return SKX_OK;
  const int64_t blocks = imin((s_hi - s_lo + 7) / 8, (int64_t)num_sms() * 16);
  k_coo_unpack3<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(ptr0, s_lo, s_hi, packed, b2,
                                                                     exc_idx, exc_val, n_exc, coords, ld);
  return check_launch("k_coo_unpack3");
}


// Host side of the compact order-3 staging (one pass over the caller's
// int64 (nnz, 3) coordinates, at SparseTensor construction), validating them
// on the way (src/tensors.py:35-60 semantics): *status = 0 ok, 1 a
// coordinate out of range, 2 not strictly lexsorted (unsorted or duplicate).
// Outputs: slice pointers ptr0[s0 + 1], packed[e] = (d << b2) | i2 with d the
// i1 increment inside the slice (absolute at a slice start); escapes (d >=
// 2^(32-b2) - 1) listed in exc_idx / exc_val (capacity cap; *n_exc receives
// the count even when it exceeds cap -- the caller retries with more room).
extern "C" int skx_stage_compact3(const int64_t* coords, int64_t nnz, int64_t s0, int64_t s1,
                                  int64_t s2, int b2, int64_t* ptr0, uint32_t* packed,
                                  int64_t* exc_idx, int32_t* exc_val, int64_t cap, int64_t* n_exc,
                                  int* status) {
  SKX_REQUIRE(b2 >= 1 && b2 <= 24 && s2 <= (int64_t(1) << b2), "skx_stage_compact3: bad b2");
  const uint64_t esc = (1ull << (32 - b2)) - 1;
  int64_t prev0 = -1, prev1 = 0, prev2 = -1, nx = 0;
  *status = 0;
  for (int64_t e = 0; e < nnz; ++e) {
    const int64_t i0 = coords[3 * e], i1 = coords[3 * e + 1], i2 = coords[3 * e + 2];
    if (i0 < 0 || i0 >= s0 || i1 < 0 || i1 >= s1 || i2 < 0 || i2 >= s2) {
      *status = 1;
      return SKX_OK;
    }
    uint64_t d;
    if (i0 != prev0) {
      if (i0 < prev0) {
        *status = 2;
        return SKX_OK;
      }
      for (int64_t s = prev0 + 1; s <= i0; ++s) ptr0[s] = e;
      d = (uint64_t)i1;
      prev0 = i0;
    } else {
      if (i1 < prev1 || (i1 == prev1 && i2 <= prev2)) {
        *status = 2;
        return SKX_OK;
      }
      d = (uint64_t)(i1 - prev1);
    }
    prev1 = i1;
    prev2 = i2;
    if (d >= esc) {
      if (nx < cap) {
        exc_idx[nx] = e;
        exc_val[nx] = (int32_t)i1;
      }
      ++nx;
      d = esc;
    }
    packed[e] = (uint32_t)((d << b2) | (uint64_t)i2);
  }
  for (int64_t s = prev0 + 1; s <= s0; ++s) ptr0[s] = nnz;
  *n_exc = nx;
  return SKX_OK;
}

extern "C" int skx_stage_stats3(const int64_t* coords, const double* vals, int64_t nnz, int64_t s1,
                                int64_t s2, int* vrange3, int64_t* rowmax2) {
  int emax = -100000, emin = 100000, bad = 0;
  for (int64_t e = 0; e < nnz; ++e) {
    uint64_t b;
    memcpy(&b, vals + e, 8);
    const int ex = (int)((b >> 52) & 0x7ff);
    if (ex == 0x7ff) bad = 1;
    else if (ex == 0) { if ((b << 12) != 0) bad = 1; }
    else {
      emax = ex - 1023 > emax ? ex - 1023 : emax;
      emin = ex - 1023 < emin ? ex - 1023 : emin;
    }
  }
  vrange3[0] = emax;
  vrange3[1] = emin;
  vrange3[2] = bad;
  const int64_t ext[2] = {s1, s2};
  for (int md = 0; md < 2; ++md) {
    int CB = 0;
    while (((ext[md] + (int64_t(1) << CB) - 1) >> CB) > 32768) ++CB;
    const int64_t nbins = (ext[md] + (int64_t(1) << CB) - 1) >> CB;
    std::vector<int64_t> h((size_t)nbins, 0);
    for (int64_t e = 0; e < nnz; ++e) ++h[(size_t)(coords[3 * e + 1 + md] >> CB)];
    int64_t mx = 0;
    for (int64_t b = 0; b < nbins; ++b) mx = h[(size_t)b] > mx ? h[(size_t)b] : mx;
    rowmax2[md] = mx;
  }
  return 0;
}
