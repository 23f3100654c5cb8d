// K1/K2: TensorSketch (src/sketching.py:25-43, 67-175) and the shared
// "sketch a tensor unfolding" machinery also used by the range finder (K4).
//
// Layout of every sketch output: Y^T, s_n x m row-major (row i_n holds the
// reference's column i_n of the m x s_n sketch), so one i_n owns one
// contiguous m-vector.
//
// Determinism: no floating-point atomics anywhere.  Each output vector is
// owned by one warp (sparse, gather) or built from per-warp shared-memory
// accumulators reduced in a fixed order (dense rows), so results are bitwise
// reproducible run to run (pkg/tests/test_tucker.py:200-209 demands that).
#include <cub/cub.cuh>

#include "skx_common.cuh"

namespace skx {

// =========================================================== table building
struct Coeffs {
  int nmodes;
  int64_t ext[16];
  int64_t off[16];
  int64_t c[16][9];
};

__device__ __forceinline__ uint64_t horner(const int64_t* c, int nc, uint64_t x) {
  const uint64_t P = 2147483647ULL;
  uint64_t acc = (uint64_t)c[0];
  for (int i = 1; i < nc; ++i) acc = (acc * x + (uint64_t)c[i]) % P;
  return acc;
}

__global__ void k_ts_tables(Coeffs cf, int64_t m, uint32_t* tab) {
  const int k = blockIdx.y;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= cf.ext[k]) return;
  uint64_t h = horner(cf.c[k], 4, (uint64_t)i) % (uint64_t)m;
  uint64_t g = horner(cf.c[k] + 4, 5, (uint64_t)i) % 2ULL;  // sign = 1 - 2g
  tab[cf.off[k] + i] = (uint32_t)h | (g ? 0x80000000u : 0u);
}

// ======================================================= sparse RHS sketch
// Fibre-major records (skx_coo_fibre): the nonzeros of column i_n are
// contiguous and ordered by the other-mode index j.  Each warp owns an
// nnz-balanced contiguous range of columns (so its records, output rows and
// TLB entries are walked in address order) and a private accumulator of m
// doubles in shared memory.  Contributions enter in ascending-j order, so each
// Y cell is the same sequential sum numpy's add.at forms; a finished column is
// streamed out and the accumulator re-zeroed (empty columns write zeros).
//
// Per chunk of 32*U nonzeros: the records (16 or 24 bytes) were loaded one
// chunk earlier (two register buffers that swap by name: the loop body is
// written twice) and prefetched into L2 PF chunks before that; table lookups
// give bucket/sign; when the chunk lies inside one column, the match_any of
// all U slices issue back to back before the ordered read-modify-writes.
struct OtherTabs {
  int n;
  const uint32_t* t[15];
};

// shared-memory words (doubles) per warp of the sparse RHS kernel
__host__ __device__ __forceinline__ int64_t rhs_warp_words(int64_t m) {
  return (m + 32 + (m + 7) / 8 + 1) & ~int64_t(1);  // even: 16-byte aligned per warp
}

template <int U, int NO>
struct RhsRecs {
  int32_t c[U][4];
  double v[U];
};

template <int U, int NO>
__device__ __forceinline__ void rhs_load(const double* __restrict__ rec, int64_t base, int64_t e_end,
                                         int lane, RhsRecs<U, NO>& r) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t e = base + u * 32 + lane;
    if (e < e_end) {
      load_rec<NO>(rec, e, r.c[u], r.v[u]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) r.c[u][k] = 0;
      r.v[u] = 0.0;
    }
  }
}

// PK: the layout carries each record's bucket/sign (skx_coo_fibre_ts, order 3):
// bucket = (c1 >> bb) & (2^31 - 1) >> bb, sign bit 31; no table lookups.
// Otherwise the last other coordinate is c1 & c1_mask.
template <int U, int NO, int PF, bool PK>
__global__ void __launch_bounds__(256) k_ts_rhs_coo(OtherTabs ot, int64_t s_n,
                                                    const int64_t* __restrict__ colptr,
                                                    const double* __restrict__ rec, int64_t m,
                                                    uint32_t c1_mask, int bb,
                                                    double* __restrict__ yt) {
  extern __shared__ double smem[];
  constexpr int RW = NO <= 2 ? 2 : 3;  // record words
  constexpr int CH = 32 * U;
  constexpr int LINES = CH * RW * 8 / 128;  // 128-byte lines per chunk, one per lane
  static_assert(LINES <= 32, "chunk too large for one prefetch instruction");
  const int64_t nnz = colptr[s_n];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  // per warp: acc (m doubles), stage (32 doubles), duplicate tags (m bytes)
  double* acc = smem + (size_t)wid * rhs_warp_words(m);
  double* stage = acc + m;
  uint8_t* tags = reinterpret_cast<uint8_t*>(stage + 32);
  const uint32_t mm = (uint32_t)m;
  const int64_t W = (int64_t)gridDim.x * nw, gw = blockIdx.x * (int64_t)nw + wid;
  auto col_at = [&](int64_t w) -> int64_t {  // first column starting at/after w's share
    if (w >= W) return s_n;
    const int64_t target = (nnz * w) / W;
    int64_t lo = 0, hi = s_n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (colptr[mid] < target) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  const int64_t c0 = gw == 0 ? 0 : col_at(gw), c1 = col_at(gw + 1);
  if (c0 >= c1) return;
  for (int64_t h = lane; h < m; h += 32) acc[h] = 0.0;
  __syncwarp();
  const int64_t ebeg = colptr[c0], eend = colptr[c1];
  int64_t col = c0, cbeg = ebeg, cend = colptr[c0 + 1];
  auto flush = [&]() {  // write the finished column, re-zero, advance
    double* dst = yt + col * m;
    if ((m & 1) == 0) {  // 16-byte aligned rows
      const double2 z = make_double2(0.0, 0.0);
      for (int64_t h = lane; h < (m >> 1); h += 32) {
        __stcs(reinterpret_cast<double2*>(dst) + h, reinterpret_cast<const double2*>(acc)[h]);
        reinterpret_cast<double2*>(acc)[h] = z;
      }
    } else {
      for (int64_t h = lane; h < m; h += 32) {
        __stcs(dst + h, acc[h]);
        acc[h] = 0.0;
      }
    }
    __syncwarp();
    ++col;
    cbeg = cend;
    cend = col < s_n ? colptr[col + 1] : INT64_MAX;
  };
  auto prefetch = [&](int64_t from) {
    const char* p = reinterpret_cast<const char*>(rec + from * RW) + lane * 128;
    if (lane < LINES && from + lane * (128 / (RW * 8)) < eend)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  };
  auto process = [&](int64_t base, const RhsRecs<U, NO>& r) {
    uint32_t hb[U];
    double xs[U];
    if (PK) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t w = (uint32_t)r.c[u][NO - 1];
        hb[u] = (w & 0x7fffffffu) >> bb;
        xs[u] = __longlong_as_double(__double_as_longlong(r.v[u]) ^ ((unsigned long long)(w >> 31) << 63));
      }
    } else {
      uint32_t t[U][NO];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < NO; ++k) {
          const uint32_t c = (uint32_t)r.c[u][k] & (k == NO - 1 ? c1_mask : 0xffffffffu);
          t[u][k] = __ldg(ot.t[k] + c);
        }
#pragma unroll
      for (int u = 0; u < U; ++u) {  // bucket sums reduced mod m by conditional subtraction
        uint32_t h = 0, neg = 0;
#pragma unroll
        for (int k = 0; k < NO; ++k) {
          h += pk_bucket(t[u][k]);
          if (h >= mm) h -= mm;
          neg ^= pk_neg(t[u][k]);
        }
        hb[u] = h;
        xs[u] = neg ? -r.v[u] : r.v[u];
      }
    }
    const int64_t nvalid = imin((int64_t)CH, eend - base);
    if (base >= cbeg && base + nvalid <= cend) {  // chunk inside the current column
#pragma unroll
      for (int u = 0; u < U; ++u)
        warp_ordered_add(acc, u * 32 + lane < nvalid ? hb[u] : kNoBucket, xs[u], stage, tags);
      return;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t sub = base + u * 32;
      if (sub >= eend) break;
      const int hi = (int)imin(eend - sub, (int64_t)32);
      while (true) {
        // lanes of this slice inside the current column: [lo, min(cend - sub, hi))
        const int lo = (int)imax(cbeg - sub, (int64_t)0);
        const int64_t ce = cend - sub;
        const int top = ce < hi ? (int)ce : hi;
        warp_ordered_add(acc, lane >= lo && lane < top ? hb[u] : kNoBucket, xs[u], stage, tags);
        if (ce >= hi) break;
        flush();
      }
    }
  };
#pragma unroll 1
  for (int p = 1; p <= PF; ++p) prefetch(ebeg + p * CH);
  RhsRecs<U, NO> ra, rb;
  rhs_load<U, NO>(rec, ebeg, eend, lane, ra);
#pragma unroll 1
  for (int64_t base = ebeg; base < eend; base += 2 * CH) {
    prefetch(base + (PF + 1) * CH);
    rhs_load<U, NO>(rec, base + CH, eend, lane, rb);
    process(base, ra);
    if (base + CH >= eend) break;
    prefetch(base + (PF + 2) * CH);
    rhs_load<U, NO>(rec, base + 2 * CH, eend, lane, ra);
    process(base + CH, rb);
  }
  while (col < c1) flush();  // trailing (possibly empty) columns of the range
}

// ======================================================== dense RHS sketch
// View the C-order tensor as [A, s_n, B] around the target mode.  Element
// (a, i_n, b) belongs to other-index j = a*B + b.  Its bucket/sign come from
// either two partial packed tables (TensorSketch: tabA over a, tabB over b,
// buckets add mod m) or one full table over j (range finder).
struct DenseView {
  int64_t A, s_n, B;
};

template <bool FULL>
__device__ __forceinline__ uint32_t dense_bucket(const uint32_t* tA, const uint32_t* tB,
                                                 int64_t a, int64_t b, int64_t B, int64_t m,
                                                 uint32_t& neg) {
  if (FULL) {
    uint32_t t = __ldg(tA + a * B + b);
    neg = pk_neg(t);
    return pk_bucket(t);
  }
  uint32_t ta = __ldg(tA + a), tb = __ldg(tB + b);
  neg = pk_neg(ta) ^ pk_neg(tb);
  uint32_t h = pk_bucket(ta) + pk_bucket(tb);
  return h >= (uint32_t)m ? h - (uint32_t)m : h;
}

// Row form: the flat (i_n, j) index space (j = a B + b over the other modes,
// i_n-major) is split into equal contiguous ranges, one per warp of a
// persistent grid.  A warp walks its range in chunks of 32 U values with a
// private shared-memory accumulator (ordered adds, as in the sparse kernel),
// the next chunk already in registers and the one PF chunks ahead prefetched
// into L2; when its range crosses into the next i_n it streams the
// accumulator out to part[(warp + i_n) m ..] (injective: ranges are ordered)
// and k_sum_flat adds each i_n's pieces in warp order.
template <bool FULL, int U, int PF>
__global__ void __launch_bounds__(256) k_dense_flat(const double* __restrict__ t, DenseView v,
                                                    const uint32_t* __restrict__ tA,
                                                    const uint32_t* __restrict__ tB, int64_t m,
                                                    int64_t per, double* __restrict__ part) {
  extern __shared__ double smem[];
  constexpr int64_t CH = 32 * U;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int64_t ww = rhs_warp_words(m);  // acc (m), stage (32), duplicate tags (m bytes)
  double* acc = smem + (size_t)wid * ww;
  double* stage = acc + m;
  // tag-based duplicate detection pays off once collisions among 32 lanes are
  // rare; small sketches (RRF, k2 ~ 1e2) take the match_any path throughout
  uint8_t* tags = m >= 1024 ? reinterpret_cast<uint8_t*>(stage + 32) : nullptr;
  const int64_t B = v.B, P = v.A * v.B, total = v.s_n * P;
  const int64_t rs = v.s_n * B;                                 // stride of a
  const uint32_t qc = (uint32_t)(CH / B), rc = (uint32_t)(CH % B);  // a, b advance per chunk
  const int64_t dstep = (int64_t)qc * rs + rc, wrap = rs - B;   // pointer advance, wrap fix
  const uint32_t Bu = (uint32_t)B;
  const int64_t gw = blockIdx.x * (int64_t)nw + wid;
  int64_t f = imin(gw * per, total);
  const int64_t fend = imin(f + per, total);
  if (f >= fend) return;
  for (int64_t h = lane; h < m; h += 32) acc[h] = 0.0;
  __syncwarp();
  int64_t in = f / P;
  while (f < fend) {
    const int64_t jend = imin((in + 1) * P, fend) - in * P;
    int64_t j = f - in * P;
    const double* base = t + in * B;
    // per slice u: element pointer, b (and a for the split tables; the full
    // table is indexed by j itself), advanced incrementally by one chunk
    const double* p[U];
    uint32_t a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t jj = j + u * 32 + lane;
      const int64_t aa = jj / B;
      a[u] = (uint32_t)aa;
      b[u] = (uint32_t)(jj - aa * B);
      p[u] = base + aa * rs + b[u];
    }
    const uint32_t* tp = tA + j + lane;  // FULL table, slice u at tp + 32 u
    // L2 prefetch cursor: 16 lanes x 128 bytes = one chunk, PF chunks ahead
    int64_t pj = j + PF * CH + (lane & 15) * 16;
    const double* pp;
    uint32_t pb;
    {
      const int64_t pa = pj / B;
      pb = (uint32_t)(pj - pa * B);
      pp = base + pa * rs + pb;
    }
    auto step = [&](const double*& q, uint32_t& bb, uint32_t& aa) {
      q += dstep;
      bb += rc;
      aa += qc;
      if (bb >= Bu) {
        bb -= Bu;
        q += wrap;
        ++aa;
      }
    };
    // raw loads only: value and table words are consumed one chunk later
    auto load = [&](int64_t j0, double (&x)[U], uint32_t (&ka)[U], uint32_t (&kb)[U]) {
      const bool whole = j0 + CH <= jend;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (whole || j0 + u * 32 + lane < jend) {
          if (FULL) {
            ka[u] = __ldg(tp + u * 32);
          } else {
            ka[u] = __ldg(tA + a[u]);
            kb[u] = __ldg(tB + b[u]);
          }
          x[u] = __ldcs(p[u]);
        } else {
          ka[u] = kNoBucket;
          kb[u] = 0;
          x[u] = 0.0;
        }
        step(p[u], b[u], a[u]);
      }
      tp += CH;
    };
    auto process = [&](const double (&x)[U], const uint32_t (&ka)[U], const uint32_t (&kb)[U]) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        uint32_t bk = kNoBucket, neg = 0;
        if (ka[u] != kNoBucket) {
          if (FULL) {
            bk = pk_bucket(ka[u]);
            neg = pk_neg(ka[u]);
          } else {
            const uint32_t h = pk_bucket(ka[u]) + pk_bucket(kb[u]);
            bk = h >= (uint32_t)m ? h - (uint32_t)m : h;
            neg = pk_neg(ka[u]) ^ pk_neg(kb[u]);
          }
        }
        // sign flip on the high word (one LOP3 instead of two selects)
        const double sx = __longlong_as_double(__double_as_longlong(x[u]) ^
                                               ((unsigned long long)neg << 63));
        warp_ordered_add(acc, bk, sx, stage, tags);
      }
    };
    auto ahead = [&](int64_t j0, double (&x)[U], uint32_t (&ka)[U], uint32_t (&kb)[U]) {
      load(j0, x, ka, kb);
      if (lane < 16 && pj < jend) asm volatile("prefetch.global.L2 [%0];" ::"l"(pp));
      uint32_t dummy = 0;
      step(pp, pb, dummy);
      pj += CH;
    };
    double xc[U], xn[U];
    uint32_t ac[U], bc[U], an[U], bn[U];
    load(j, xc, ac, bc);
    while (true) {
      const bool more = j + CH < jend;
      if (more) ahead(j + CH, xn, an, bn);
      process(xc, ac, bc);
      j += CH;
      if (!more) break;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        xc[u] = xn[u];
        ac[u] = an[u];
        bc[u] = bn[u];
      }
    }
    double* dst = part + (gw + in) * m;
    for (int64_t h = lane; h < m; h += 32) {
      dst[h] = acc[h];
      acc[h] = 0.0;
    }
    __syncwarp();
    f = (in + 1) * P;
    ++in;
  }
}

// yt[i_n, h] = sum over the warps w whose range meets i_n (in order) of
// part[(w + i_n) m + h]
__global__ void k_sum_flat(const double* __restrict__ part, int64_t s_n, int64_t P, int64_t per,
                           int64_t m, double* __restrict__ yt) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= s_n * m) return;
  const int64_t in = idx / m, h = idx - in * m;
  const int64_t w0 = in * P / per, w1 = ((in + 1) * P - 1) / per;
  double s = 0.0;
  for (int64_t w = w0; w <= w1; ++w) s += part[(w + in) * m + h];
  yt[idx] = s;
}

// ---- gather form for B == 1 (target mode is the fastest-varying one): rows
// of s_n contiguous values share one bucket; the columns are sorted by bucket
// (ascending index inside a bucket) and each bucket's rows are summed.
template <bool FULL>
__global__ void k_bucket_keys(const uint32_t* __restrict__ tA, int64_t A, uint32_t* keys,
                              uint32_t* idx, uint32_t* neg) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= A) return;
  uint32_t t = __ldg(tA + a);
  keys[a] = pk_bucket(t);
  idx[a] = (uint32_t)a;
  neg[a] = pk_neg(t);
}

__global__ void k_run_bounds(const uint32_t* __restrict__ keys, int64_t n, int64_t m,
                             int64_t* __restrict__ start) {
  // start[c] = first position with key >= c, for c in [0, m]; keys sorted
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c > m) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if ((int64_t)keys[mid] < c) lo = mid + 1; else hi = mid;
  }
  start[c] = lo;
}

// Task = (bucket c, segment k, column block); segment k covers rows
// [k seg, (k+1) seg) of c's run, the last segment the rest; the partial sums
// are then added segment by segment (fixed order, deterministic) by
// k_sum_segs.  Keeps the GPU busy when the bucket count m is small (RRF:
// k2 ~ 1e2 buckets) or the runs are long.
template <int CPL>
__global__ void __launch_bounds__(256) k_gather_rows_seg(const double* __restrict__ t, int64_t s_n,
                                                         const int64_t* __restrict__ start,
                                                         const uint32_t* __restrict__ list,
                                                         const uint32_t* __restrict__ neg_of,
                                                         int64_t m, int64_t seg, int64_t nseg,
                                                         double* __restrict__ part) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ncb = (s_n + 32 * CPL - 1) / (32 * CPL);
  const int64_t task = blockIdx.x * (int64_t)(blockDim.x >> 5) + wid;
  if (task >= m * nseg * ncb) return;
  const int64_t cb = task % ncb, ck = task / ncb;
  const int64_t c = ck / nseg, k = ck - c * nseg;
  const int64_t col0 = cb * 32 * CPL;
  double acc[CPL];
#pragma unroll
  for (int u = 0; u < CPL; ++u) acc[u] = 0.0;
  const int64_t rs = start[c], re = start[c + 1];
  const int64_t r0 = imin(rs + k * seg, re), r1 = k == nseg - 1 ? re : imin(r0 + seg, re);
  // RB rows in flight per iteration (loads first, then the adds in row order)
  constexpr int RB = 4;
  int64_t r = r0;
  for (; r + RB <= r1; r += RB) {
    double x[RB][CPL];
    bool ng[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      const uint32_t a = list[r + q];
      ng[q] = neg_of[a] != 0;
      const double* row = t + (int64_t)a * s_n;
#pragma unroll
      for (int u = 0; u < CPL; ++u) {
        const int64_t col = col0 + u * 32 + lane;
        x[q][u] = col < s_n ? __ldcs(row + col) : 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < RB; ++q)
#pragma unroll
      for (int u = 0; u < CPL; ++u) acc[u] += ng[q] ? -x[q][u] : x[q][u];
  }
  for (; r < r1; ++r) {
    const uint32_t a = list[r];
    const bool ng = neg_of[a] != 0;
    const double* row = t + (int64_t)a * s_n;
#pragma unroll
    for (int u = 0; u < CPL; ++u) {
      const int64_t col = col0 + u * 32 + lane;
      if (col < s_n) {
        const double x = __ldcs(row + col);
        acc[u] += ng ? -x : x;
      }
    }
  }
  double* dst = part + ck * s_n;
#pragma unroll
  for (int u = 0; u < CPL; ++u) {
    const int64_t col = col0 + u * 32 + lane;
    if (col < s_n) dst[col] = acc[u];
  }
}

// yt[col, c] = sum_k part[(c, k), col], k ascending
__global__ void k_sum_segs(const double* __restrict__ part, int64_t m, int64_t nseg, int64_t s_n,
                           double* __restrict__ yt) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= m * s_n) return;
  const int64_t col = idx / m, c = idx - col * m;
  double s = 0.0;
  for (int64_t k = 0; k < nseg; ++k) s += part[(c * nseg + k) * s_n + col];
  yt[col * m + c] = s;
}

}  // namespace skx

using namespace skx;

extern "C" int skx_ts_tables(int nmodes, const int64_t* extents_h, const int64_t* coeffs_h,
                             int64_t m, uint32_t* tab, void* stream) {
  SKX_REQUIRE(nmodes >= 1 && nmodes <= 16, "skx_ts_tables: 1..16 modes supported");
  SKX_REQUIRE(m >= 1 && m < (int64_t(1) << 31), "skx_ts_tables: m out of range");
  Coeffs cf{};
  cf.nmodes = nmodes;
  int64_t off = 0, mx = 0;
  for (int k = 0; k < nmodes; ++k) {
    cf.ext[k] = extents_h[k];
    cf.off[k] = off;
    off += extents_h[k];
    mx = extents_h[k] > mx ? extents_h[k] : mx;
    for (int i = 0; i < 9; ++i) cf.c[k][i] = coeffs_h[k * 9 + i];
  }
  if (mx == 0) return SKX_OK;
  dim3 grid((unsigned)((mx + 255) / 256), nmodes);
  k_ts_tables<<<grid, 256, 0, (cudaStream_t)stream>>>(cf, m, tab);
  return check_launch("k_ts_tables");
}

extern "C" int skx_ts_rhs_coo(int n_other, int64_t s_n, const int64_t* colptr, const void* rec,
                              const uint32_t* tab, const int64_t* tab_off_h, int64_t m,
                              uint32_t c1_mask, int packed_bb, double* yt, void* stream) {
  SKX_REQUIRE(n_other >= 1 && n_other <= 4, "skx_ts_rhs_coo: 1..4 other modes (sparse order <= 5)");
  SKX_REQUIRE(packed_bb < 0 || n_other == 2, "skx_ts_rhs_coo: packed layouts are order 3");
  const int nw = warps_per_cta_for(rhs_warp_words(m) * 8);
  SKX_REQUIRE(nw >= 1, "skx_ts_rhs_coo: sketch size %lld exceeds shared-memory capacity",
              (long long)m);
  if (s_n == 0) return SKX_OK;
  OtherTabs ot{};
  ot.n = n_other;
  if (packed_bb < 0)
    for (int k = 0; k < n_other; ++k) ot.t[k] = tab + tab_off_h[k];
  const size_t smem = (size_t)nw * rhs_warp_words(m) * 8;
  // L2 prefetch distance 4 chunks (measured at config 4, packed layout:
  // PF = 1 / 2-4 / 6 / 8 -> 0.67 / 0.605 / 0.614 / 0.638 ms per mode)
  auto kern = packed_bb >= 0 ? k_ts_rhs_coo<4, 2, 4, true>
            : n_other == 1   ? k_ts_rhs_coo<4, 1, 4, false>
            : n_other == 2   ? k_ts_rhs_coo<4, 2, 4, false>
            : n_other == 3   ? k_ts_rhs_coo<4, 3, 4, false>
                             : k_ts_rhs_coo<4, 4, 4, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = imin((int64_t)num_sms() * per_sm, (s_n + nw - 1) / nw);
  kern<<<(unsigned)blocks, nw * 32, smem, (cudaStream_t)stream>>>(
      ot, s_n, colptr, (const double*)rec, m, c1_mask, packed_bb < 0 ? 0 : packed_bb, yt);
  return check_launch("k_ts_rhs_coo");
}

// Shared by TS (two partial tables) and the range finder (one full table).
static int dense_sketch(bool full, const double* t, int ndim, const int64_t* shape_h, int mode,
                        const uint32_t* tA, const uint32_t* tB, int64_t m, double* yt, void* ws,
                        size_t* ws_bytes, cudaStream_t s) {
  SKX_REQUIRE(ws_bytes != nullptr, "dense sketch: ws_bytes is NULL");
  SKX_REQUIRE(mode >= 0 && mode < ndim, "dense sketch: mode out of range");
  DenseView v{1, shape_h[mode], 1};
  for (int k = 0; k < mode; ++k) v.A *= shape_h[k];
  for (int k = mode + 1; k < ndim; ++k) v.B *= shape_h[k];
  const int64_t P = v.A * v.B;
  Arena ar(ws, *ws_bytes);
  if (v.B == 1) {
    // gather form over buckets of a (= j)
    uint32_t* k_in = ar.take<uint32_t>(P);
    uint32_t* k_out = ar.take<uint32_t>(P);
    uint32_t* v_in = ar.take<uint32_t>(P);
    uint32_t* v_out = ar.take<uint32_t>(P);
    uint32_t* neg = ar.take<uint32_t>(P);
    int64_t* start = ar.take<int64_t>(m + 1);
    // segments of kSeg rows (about 2 x the mean run length / kSeg per bucket)
    constexpr int64_t kSeg = 256;
    const int64_t nseg = imax(1, 2 * ((P / imax(m, 1) + kSeg - 1) / kSeg));
    double* part = ar.take<double>((size_t)m * nseg * v.s_n);
    size_t cub_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, k_in, k_out, v_in, v_out, (int)P, 0, 32, s);
    void* cub_tmp = ar.take<char>(cub_bytes);
    if (ws == nullptr) {
      *ws_bytes = ar.used + 256;
      return SKX_OK;
    }
    SKX_REQUIRE(ar.ok(), "dense sketch: workspace too small");
    SKX_REQUIRE(P < (int64_t(1) << 31), "dense sketch: too many columns for the gather form");
    if (full) {
      k_bucket_keys<true><<<(unsigned)((P + 255) / 256), 256, 0, s>>>(tA, P, k_in, v_in, neg);
    } else {
      k_bucket_keys<false><<<(unsigned)((P + 255) / 256), 256, 0, s>>>(tA, P, k_in, v_in, neg);
    }
    int bits = 1;
    while ((int64_t(1) << bits) < m) ++bits;
    cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, k_in, k_out, v_in, v_out, (int)P, 0, bits,
                                    s);
    k_run_bounds<<<(unsigned)((m + 1 + 255) / 256), 256, 0, s>>>(k_out, P, m, start);
    const int64_t s_n = v.s_n;
    if (s_n <= 32 * 4) {
      const int64_t tasks = m * nseg * ((s_n + 127) / 128);
      k_gather_rows_seg<4><<<(unsigned)((tasks + 7) / 8), 256, 0, s>>>(t, s_n, start, v_out, neg, m,
                                                                       kSeg, nseg, part);
    } else {
      const int64_t tasks = m * nseg * ((s_n + 255) / 256);
      k_gather_rows_seg<8><<<(unsigned)((tasks + 7) / 8), 256, 0, s>>>(t, s_n, start, v_out, neg, m,
                                                                       kSeg, nseg, part);
    }
    k_sum_segs<<<(unsigned)((m * s_n + 255) / 256), 256, 0, s>>>(part, m, nseg, s_n, yt);
    return check_launch("dense sketch (gather form)", 5);
  }
  const int nw = warps_per_cta_for(rhs_warp_words(m) * 8);
  SKX_REQUIRE(nw >= 1, "dense sketch: sketch size %lld exceeds shared-memory capacity",
              (long long)m);
  SKX_REQUIRE(v.A < (int64_t(1) << 31) && v.B < (int64_t(1) << 31),
              "dense sketch: other-mode extents too large for the row form");
  const size_t smem = (size_t)nw * rhs_warp_words(m) * 8;
  auto kern = full ? k_dense_flat<true, 8, 6> : k_dense_flat<false, 8, 6>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem);
  if (per_sm < 1) per_sm = 1;
  // one range per resident warp, but at least 16K values per range
  const int64_t total = v.s_n * P;
  int64_t blocks = (int64_t)num_sms() * per_sm;
  blocks = imax(1, imin(blocks, (total + 16384 * nw - 1) / (16384 * nw)));
  const int64_t W = blocks * nw;
  const int64_t per = (total + W - 1) / W;
  double* part = ar.take<double>((size_t)(W + v.s_n) * m);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "dense sketch: workspace too small");
  kern<<<(unsigned)blocks, nw * 32, smem, s>>>(t, v, tA, tB, m, per, part);
  k_sum_flat<<<(unsigned)((v.s_n * m + 255) / 256), 256, 0, s>>>(part, v.s_n, P, per, m, yt);
  return check_launch("dense sketch (row form)", 2);
}

namespace skx {
// Mode-last copy of a dense tensor viewed as [A, S, B]: out[a, b, s] = in[a, s, b]
// (batched transposes of S x B panels through 32 x 32 shared-memory tiles,
// coalesced on both sides).  Feeds the gather form of the dense sketches.
__global__ void __launch_bounds__(256) k_mode_last(const double* __restrict__ in, int64_t S,
                                                   int64_t B, double* __restrict__ out) {
  __shared__ double tile[32][33];
  const int64_t a = blockIdx.z;
  const int64_t s0 = blockIdx.y * 32, b0 = blockIdx.x * 32;
  const double* src = in + a * S * B;
  double* dst = out + a * S * B;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int64_t s = s0 + ty + k, b = b0 + tx;
    if (s < S && b < B) tile[ty + k][tx] = __ldcs(src + s * B + b);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int64_t b = b0 + ty + k, s = s0 + tx;
    if (s < S && b < B) dst[b * S + s] = tile[tx][ty + k];
  }
}

}  // namespace skx

extern "C" int skx_mode_last(const double* t, int ndim, const int64_t* shape_h, int mode,
                             double* out, void* stream) {
  using namespace skx;
  SKX_REQUIRE(ndim >= 1 && mode >= 0 && mode < ndim, "skx_mode_last: bad mode");
  int64_t A = 1, B = 1;
  for (int k = 0; k < mode; ++k) A *= shape_h[k];
  for (int k = mode + 1; k < ndim; ++k) B *= shape_h[k];
  const int64_t S = shape_h[mode];
  if (A * S * B == 0) return SKX_OK;
  SKX_REQUIRE(A < 65536, "skx_mode_last: leading extent product too large for the grid");
  dim3 grid((unsigned)((B + 31) / 32), (unsigned)((S + 31) / 32), (unsigned)A);
  k_mode_last<<<grid, 256, 0, (cudaStream_t)stream>>>(t, S, B, out);
  return check_launch("k_mode_last");
}

// Partial TS tables for the [A, s_n, B] split of a dense tensor: combine the
// per-mode tables of modes before / after the target mode.
namespace skx {
__global__ void k_combine_tabs(OtherTabs ot, int nmodes_part, const int64_t* __restrict__ dummy,
                               int64_t n, int64_t m, uint32_t* out, int first, int64_t ext0,
                               int64_t ext1, int64_t ext2, int64_t ext3, int64_t ext4,
                               int64_t ext5, int64_t ext6, int64_t ext7) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= n) return;
  const int64_t ext[8] = {ext0, ext1, ext2, ext3, ext4, ext5, ext6, ext7};
  uint64_t hs = 0;
  uint32_t neg = 0;
  int64_t rem = x;
  for (int k = nmodes_part - 1; k >= 0; --k) {
    const int64_t i = rem % ext[k];
    rem /= ext[k];
    const uint32_t t = __ldg(ot.t[first + k] + i);
    hs += pk_bucket(t);
    neg ^= pk_neg(t);
  }
  out[x] = (uint32_t)(hs % (uint64_t)m) | (neg ? 0x80000000u : 0u);
}
}  // namespace skx

extern "C" int skx_ts_rhs_dense(const double* t, int ndim, const int64_t* shape_h, int mode,
                                const uint32_t* tab, const int64_t* tab_off_h, int64_t m,
                                double* yt, void* ws, size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(ndim >= 2 && ndim <= 9, "skx_ts_rhs_dense: 2..9 modes supported");
  SKX_REQUIRE(mode >= 0 && mode < ndim, "skx_ts_rhs_dense: mode out of range");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_ts_rhs_dense: ws_bytes is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  int64_t A = 1, B = 1;
  for (int k = 0; k < mode; ++k) A *= shape_h[k];
  for (int k = mode + 1; k < ndim; ++k) B *= shape_h[k];
  // partial tables live at the front of the workspace
  Arena ar(ws, *ws_bytes);
  uint32_t* tA = ar.take<uint32_t>(A);
  uint32_t* tB = ar.take<uint32_t>(B);
  size_t inner = 0;
  int rc = dense_sketch(false, t, ndim, shape_h, mode, nullptr, nullptr, m, yt, nullptr, &inner, s);
  if (rc) return rc;
  char* inner_ws = ar.take<char>(inner);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_ts_rhs_dense: workspace too small");
  OtherTabs ot{};
  ot.n = ndim - 1;
  for (int k = 0; k < ndim - 1; ++k) ot.t[k] = tab + tab_off_h[k];
  int64_t ex[8] = {1, 1, 1, 1, 1, 1, 1, 1};
  // modes before the target: others 0..mode-1
  for (int k = 0; k < mode; ++k) ex[k] = shape_h[k];
  if (mode == 0) {
    // A == 1: bucket 0 / sign + for the empty prefix
    cudaMemsetAsync(tA, 0, sizeof(uint32_t), s);
  } else {
    k_combine_tabs<<<(unsigned)((A + 255) / 256), 256, 0, s>>>(
        ot, mode, nullptr, A, m, tA, 0, ex[0], ex[1], ex[2], ex[3], ex[4], ex[5], ex[6], ex[7]);
  }
  int64_t ey[8] = {1, 1, 1, 1, 1, 1, 1, 1};
  for (int k = mode + 1; k < ndim; ++k) ey[k - mode - 1] = shape_h[k];
  if (mode == ndim - 1) {
    cudaMemsetAsync(tB, 0, sizeof(uint32_t), s);
  } else {
    k_combine_tabs<<<(unsigned)((B + 255) / 256), 256, 0, s>>>(ot, ndim - 1 - mode, nullptr, B, m,
                                                               tB, mode, ey[0], ey[1], ey[2], ey[3],
                                                               ey[4], ey[5], ey[6], ey[7]);
  }
  SKX_TRY(check_launch("k_combine_tabs", 2));
  return dense_sketch(false, t, ndim, shape_h, mode, tA, tB, m, yt, inner_ws, &inner, s);
}

namespace skx {
struct CombPack {
  int n;
  int64_t ext[15];
  const uint32_t* t[15];
};
__global__ void k_ts_combine(CombPack cp, int64_t P, int64_t m, uint32_t* __restrict__ out) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; x < P; x += stride) {
    uint64_t hs = 0;
    uint32_t neg = 0;
    int64_t rem = x;
    for (int k = cp.n - 1; k >= 0; --k) {
      const int64_t i = rem % cp.ext[k];
      rem /= cp.ext[k];
      const uint32_t t = __ldg(cp.t[k] + i);
      hs += pk_bucket(t);
      neg ^= pk_neg(t);
    }
    out[x] = (uint32_t)(hs % (uint64_t)m) | (neg ? 0x80000000u : 0u);
  }
}
}  // namespace skx

extern "C" int skx_ts_combine(int n, const int64_t* ext_h, const uint32_t* tab,
                              const int64_t* tab_off_h, int64_t m, int64_t P, uint32_t* out,
                              void* stream) {
  SKX_REQUIRE(n >= 1 && n <= 15, "skx_ts_combine: 1..15 modes");
  CombPack cp{};
  cp.n = n;
  for (int k = 0; k < n; ++k) {
    cp.ext[k] = ext_h[k];
    cp.t[k] = tab + tab_off_h[k];
  }
  if (P == 0) return SKX_OK;
  const int blocks = (int)imin((P + 255) / 256, (int64_t)num_sms() * 16);
  k_ts_combine<<<blocks, 256, 0, (cudaStream_t)stream>>>(cp, P, m, out);
  return check_launch("k_ts_combine");
}

extern "C" int skx_rrf_stage1_dense(const double* t, int ndim, const int64_t* shape_h, int mode,
                                    const uint32_t* tab, int64_t k2, double* stage1, void* ws,
                                    size_t* ws_bytes, void* stream) {
  return dense_sketch(true, t, ndim, shape_h, mode, tab, nullptr, k2, stage1, ws, ws_bytes,
                      (cudaStream_t)stream);
}
