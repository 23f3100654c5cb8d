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
