// K3: leverage-score row sampling of a Kronecker chain and the matching fibre
// gather (src/sketching.py:193-217, 262-287; src/linalg.py:73-84).
#include <cub/cub.cuh>

#include <stdlib.h>

#include "skx_common.cuh"

namespace skx {

// p = max(s,0)/sum; cdf = cumsum(p); cdf /= cdf[-1] over kLevChunks fixed
// chunks (deterministic; rounding differs from numpy's sequential cumsum only
// in the last bits).  Each chunk is one thread's sequential pass; the chunks
// are spread over kLevChunks/32 one-warp CTAs so the ~2 s IEEE divisions run on
// many SMs, and the two cross-chunk sums are a single thread's fixed-order
// loop (k_lev_total, k_lev_offsets).
constexpr int kLevChunks = 1024;

__device__ __forceinline__ void lev_chunk(int64_t s, int t, int64_t& lo, int64_t& hi) {
  const int64_t per = (s + kLevChunks - 1) / kLevChunks;
  lo = imin(t * per, s);
  hi = imin(lo + per, s);
}

__global__ void k_lev_sums(const double* __restrict__ sc, int64_t s, double* __restrict__ part) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  int64_t lo, hi;
  lev_chunk(s, t, lo, hi);
  double acc = 0.0;
  for (int64_t i = lo; i < hi; ++i) acc += fmax(sc[i], 0.0);
  part[t] = acc;
}

__global__ void k_lev_total(double* __restrict__ part, double* __restrict__ tot) {
  if (threadIdx.x != 0) return;
  double t = 0.0;
  for (int i = 0; i < kLevChunks; ++i) t += part[i];
  tot[0] = t;
}

__global__ void k_lev_scan(const double* __restrict__ sc, int64_t s, const double* __restrict__ tot_p,
                           double* __restrict__ p, double* __restrict__ cdf,
                           double* __restrict__ part) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  int64_t lo, hi;
  lev_chunk(s, t, lo, hi);
  const double tot = tot_p[0];
  double run = 0.0;
  for (int64_t i = lo; i < hi; ++i) {
    const double pi = fmax(sc[i], 0.0) / tot;
    p[i] = pi;
    run += pi;
    cdf[i] = run;
  }
  part[t] = run;
}

// exclusive prefix of the chunk totals; tot[1] = cdf[s-1] after the offsets
__global__ void k_lev_offsets(int64_t s, double* __restrict__ part, double* __restrict__ tot) {
  if (threadIdx.x != 0) return;
  const int64_t per = (s + kLevChunks - 1) / kLevChunks;
  const int c_last = (int)((s - 1) / per);
  double t = 0.0, last = 0.0;
  for (int i = 0; i < kLevChunks; ++i) {
    const double v = part[i];
    part[i] = t;
    if (i == c_last) last = v + t;  // the last element's run plus its offset
    t += v;
  }
  tot[1] = last;
}

__global__ void k_lev_final(int64_t s, const double* __restrict__ part,
                            const double* __restrict__ tot, double* __restrict__ cdf) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  int64_t lo, hi;
  lev_chunk(s, t, lo, hi);
  const double offs = part[t], L = tot[1];
  for (int64_t i = lo; i < hi; ++i) cdf[i] = (cdf[i] + offs) / L;
}

// The same five steps in ONE CTA (kLevFusedThreads threads, each owning the
// chunks t, t + kLevFusedThreads, ...): identical arithmetic and order, so
// identical bits; one launch and one SM instead of five launches over 32 SMs
// (the leverage path runs beside the fitness pass, where every extra launch
// waits for a free SM slot).
constexpr int kLevFusedThreads = 512;
constexpr int kLevPer = kLevChunks / kLevFusedThreads;

// Loads of a thread's chunk in batches of kLevB (independent loads in flight:
// a sequential loop with stores between its loads issued one L2 round trip
// per element, ~1 ms per 2e5 scores); the arithmetic and its order are those
// of the element-by-element loop, so the bits are unchanged.
constexpr int kLevB = 8;

__global__ void __launch_bounds__(kLevFusedThreads) k_lev_prepare1(const double* __restrict__ sc,
                                                                  int64_t s, double* __restrict__ p,
                                                                  double* __restrict__ cdf) {
  __shared__ double part[kLevChunks];
  __shared__ double tot[2];
  const int t0 = threadIdx.x;
#pragma unroll
  for (int u = 0; u < kLevPer; ++u) {
    int64_t lo, hi;
    lev_chunk(s, t0 + u * kLevFusedThreads, lo, hi);
    double acc = 0.0;
    for (int64_t i = lo; i < hi; i += kLevB) {
      double x[kLevB];
#pragma unroll
      for (int b = 0; b < kLevB; ++b) x[b] = i + b < hi ? __ldg(sc + i + b) : 0.0;
#pragma unroll
      for (int b = 0; b < kLevB; ++b)
        if (i + b < hi) acc += fmax(x[b], 0.0);
    }
    part[t0 + u * kLevFusedThreads] = acc;
  }
  __syncthreads();
  if (t0 == 0) {
    double t = 0.0;
    for (int i = 0; i < kLevChunks; ++i) t += part[i];
    tot[0] = t;
  }
  __syncthreads();
  const double total = tot[0];
#pragma unroll
  for (int u = 0; u < kLevPer; ++u) {
    int64_t lo, hi;
    lev_chunk(s, t0 + u * kLevFusedThreads, lo, hi);
    double run = 0.0;
    for (int64_t i = lo; i < hi; i += kLevB) {
      double x[kLevB];
#pragma unroll
      for (int b = 0; b < kLevB; ++b) x[b] = i + b < hi ? __ldg(sc + i + b) : 0.0;
#pragma unroll
      for (int b = 0; b < kLevB; ++b) {
        if (i + b >= hi) break;
        const double pi = fmax(x[b], 0.0) / total;
        p[i + b] = pi;
        run += pi;
        cdf[i + b] = run;
      }
    }
    part[t0 + u * kLevFusedThreads] = run;
  }
  __syncthreads();
  if (t0 == 0) {
    const int64_t per = (s + kLevChunks - 1) / kLevChunks;
    const int c_last = (int)((s - 1) / per);
    double t = 0.0, last = 0.0;
    for (int i = 0; i < kLevChunks; ++i) {
      const double v = part[i];
      part[i] = t;
      if (i == c_last) last = v + t;
      t += v;
    }
    tot[1] = last;
  }
  __syncthreads();
  const double L = tot[1];
#pragma unroll
  for (int u = 0; u < kLevPer; ++u) {
    int64_t lo, hi;
    lev_chunk(s, t0 + u * kLevFusedThreads, lo, hi);
    const double offs = part[t0 + u * kLevFusedThreads];
    for (int64_t i = lo; i < hi; i += kLevB) {
      double x[kLevB];
#pragma unroll
      for (int b = 0; b < kLevB; ++b) x[b] = i + b < hi ? cdf[i + b] : 0.0;
#pragma unroll
      for (int b = 0; b < kLevB; ++b)
        if (i + b < hi) cdf[i + b] = (x[b] + offs) / L;
    }
  }
}

struct PtrPack {
  const double* p[15];
  const double* c[15];
  int64_t ext[15];
};

__global__ void k_lev_sample(int n_other, PtrPack pk, int64_t m, uint64_t k0, uint64_t k1,
                             uint64_t p0, int64_t* __restrict__ idx, double* __restrict__ w) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  double pp = 1.0;
  for (int k = 0; k < n_other; ++k) {
    const double u = u64_to_unit(philox_raw(k0, k1, p0 + (uint64_t)(k * m + j)));
    // searchsorted(cdf, u, side='right'): first i with cdf[i] > u
    const double* c = pk.c[k];
    int64_t lo = 0, hi = pk.ext[k];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (c[mid] <= u) lo = mid + 1; else hi = mid;
    }
    if (lo >= pk.ext[k]) lo = pk.ext[k] - 1;  // unreachable: cdf[-1] == 1 > u
    idx[j * n_other + k] = lo;
    pp *= pk.p[k][lo];
  }
  w[j] = 1.0 / sqrt((double)m * pp);
}

struct FacPack {
  const double* a[15];
  int64_t R[15];
};

// z column-major (ld = m): z[col*m + j], col = (p_1, ..., p_k) first slowest.
__global__ void k_kron_rows(int n_other, FacPack fp, int64_t r, const int64_t* __restrict__ idx,
                            const double* __restrict__ w, int64_t m, double* __restrict__ z) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m * r) return;
  const int64_t j = e % m, col = e / m;
  // decode col into per-mode column indices (last mode fastest)
  int64_t rem = col;
  int64_t pc[15];
  for (int k = n_other - 1; k >= 0; --k) {
    pc[k] = rem % fp.R[k];
    rem /= fp.R[k];
  }
  double prod = fp.a[0][idx[j * n_other] * fp.R[0] + pc[0]];
  for (int k = 1; k < n_other; ++k) prod *= fp.a[k][idx[j * n_other + k] * fp.R[k] + pc[k]];
  z[e] = w[j] * prod;
}

// Y[j, i_n] = w_j * T[multi(flat_j) with i_n inserted], row-major m x s_n.
struct ShapePack {
  int ndim, mode;
  int64_t shape[16];
  int64_t stride[16];
};

__global__ void k_gather_dense(const double* __restrict__ t, ShapePack sp, int n_other,
                               const int64_t* __restrict__ idx, const double* __restrict__ w,
                               int64_t m, double* __restrict__ y) {
  const int64_t s_n = sp.shape[sp.mode];
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m * s_n) return;
  const int64_t j = e / s_n, in = e - j * s_n;
  int64_t off = in * sp.stride[sp.mode];
  int kk = 0;
  for (int k = 0; k < sp.ndim; ++k) {
    if (k == sp.mode) continue;
    off += idx[j * n_other + kk] * sp.stride[k];
    ++kk;
  }
  y[e] = w[j] * t[off];
}

// ---- sparse gather: keys = flat_other * s_n + i_n, sorted ascending.
__device__ __forceinline__ int64_t lower_bound_i64(const int64_t* a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_gather_coo_count(int n_other, PtrPack pk, int64_t s_n, int64_t nnz,
                                   const int64_t* __restrict__ keys, const int64_t* __restrict__ idx,
                                   int64_t m, int64_t* __restrict__ lo_out, int64_t* __restrict__ cnt) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  int64_t flat = 0;
  for (int k = 0; k < n_other; ++k) flat = flat * pk.ext[k] + idx[j * n_other + k];
  const int64_t a = lower_bound_i64(keys, nnz, flat * s_n);
  const int64_t b = lower_bound_i64(keys, nnz, (flat + 1) * s_n);
  lo_out[j] = a;
  cnt[j] = b - a;
}

__global__ void k_gather_coo_write(const int64_t* __restrict__ keys, const double* __restrict__ vals,
                                   int64_t s_n, const int64_t* __restrict__ lo_in,
                                   const int64_t* __restrict__ cnt, const int64_t* __restrict__ off,
                                   const double* __restrict__ w, int64_t m, int64_t cap,
                                   int64_t* __restrict__ hit_col, double* __restrict__ hit_val) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int64_t a = lo_in[j], c = cnt[j], o = off[j];
  for (int64_t t = 0; t < c; ++t) {
    if (o + t >= cap) break;
    hit_col[o + t] = keys[a + t] % s_n;
    hit_val[o + t] = w[j] * vals[a + t];
  }
}

// ---- sparse gather without a sorted key array: one pass over the lexsorted
// COO keeps the nonzeros whose other-mode index is among the sampled ones
// (~m nnz / P_n of them: ~160 at config 5).  A 64 Kbit shared-memory bitmap of
// the sampled flats rejects almost every nonzero with one shared load; the
// rare bitmap hits are confirmed by binary search in the sorted flats.  The
// bitmap is a two-probe Bloom filter over 2^18 bits (32 KB): at m = 6400 about
// 0.2% of the nonzeros reach the (L2-latency-bound) binary search.
struct CoordPack {
  const int32_t* c[8];
  int64_t ext[8];
};

constexpr int kBloomBits = 18;

__device__ __forceinline__ uint2 flat_hash2(uint64_t f) {
  const uint64_t a = f * 0x9E3779B97F4A7C15ull, b = (f ^ (f >> 29)) * 0xBF58476D1CE4E5B9ull;
  return make_uint2((uint32_t)(a >> (64 - kBloomBits)), (uint32_t)(b >> (64 - kBloomBits)));
}

__global__ void __launch_bounds__(256) k_filter_fibers(int ndim, int mode, CoordPack cp,
                                                       int64_t nnz, const double* __restrict__ vals,
                                                       const int64_t* __restrict__ sflat, int64_t m,
                                                       int64_t* __restrict__ out_key,
                                                       double* __restrict__ out_val, int64_t cap,
                                                       unsigned long long* __restrict__ count) {
  __shared__ uint32_t bits[1 << (kBloomBits - 5)];
  for (int i = threadIdx.x; i < (1 << (kBloomBits - 5)); i += blockDim.x) bits[i] = 0u;
  __syncthreads();
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
    const uint2 h = flat_hash2((uint64_t)sflat[j]);
    atomicOr(&bits[h.x >> 5], 1u << (h.x & 31));
    atomicOr(&bits[h.y >> 5], 1u << (h.y & 31));
  }
  __syncthreads();
  const int64_t s_n = cp.ext[mode];
  constexpr int U = 4;  // elements per thread per pass, loads issued first
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e0 < nnz; e0 += U * stride) {
    int64_t flat[U];
#pragma unroll
    for (int u = 0; u < U; ++u) flat[u] = 0;
    for (int k = 0; k < ndim; ++k) {
      if (k == mode) continue;
      int32_t c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = e0 + u * stride;
        c[u] = e < nnz ? __ldcs(cp.c[k] + e) : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) flat[u] = flat[u] * cp.ext[k] + c[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * stride;
      const uint2 h = flat_hash2((uint64_t)flat[u]);
      if (e >= nnz || !((bits[h.x >> 5] >> (h.x & 31)) & (bits[h.y >> 5] >> (h.y & 31)) & 1u))
        continue;
      int64_t lo = 0, hi = m;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (sflat[mid] < flat[u]) lo = mid + 1; else hi = mid;
      }
      if (lo < m && sflat[lo] == flat[u]) {
        const unsigned long long slot = atomicAdd(count, 1ull);
        if ((int64_t)slot < cap) {
          out_key[slot] = flat[u] * s_n + cp.c[mode][e];
          out_val[slot] = vals[e];
        }
      }
    }
  }
}

// Order-3 form of k_filter_fibers: each thread takes four consecutive
// nonzeros with one 16-byte load per other-mode coordinate row (the generic
// kernel spends most of its issue slots on per-element 4-byte loads and 64-bit
// index arithmetic: ALU 66%, 0.29 of HBM), a 2^19-bit Bloom filter in 64 KB of
// shared memory (2 probes: ~0.06% false positives at m = 6400 instead of
// ~0.23%, so fewer L2-latency binary searches), and a persistent grid (the
// filter is built once per CTA, not once per 1024 nonzeros).  Same output set
// (the slot order of the hits is not fixed; the caller sorts the keys).
constexpr int kBloomBits3 = 19;

__device__ __forceinline__ uint2 flat_hash2_b(uint64_t f, int bb) {
  const uint64_t a = f * 0x9E3779B97F4A7C15ull, b = (f ^ (f >> 29)) * 0xBF58476D1CE4E5B9ull;
  return make_uint2((uint32_t)(a >> (64 - bb)), (uint32_t)(b >> (64 - bb)));
}

template <int U>
__global__ void __launch_bounds__(256) k_filter_fibers3v(
    const int32_t* __restrict__ ca, const int32_t* __restrict__ cb, int64_t ext_b,
    const int32_t* __restrict__ cmode, int64_t s_n, int64_t nnz, const double* __restrict__ vals,
    const int64_t* __restrict__ sflat, int64_t m, int64_t* __restrict__ out_key,
    double* __restrict__ out_val, int64_t cap, unsigned long long* __restrict__ count) {
  extern __shared__ uint32_t bits3[];
  constexpr int NW = 1 << (kBloomBits3 - 5);
  for (int i = threadIdx.x; i < NW; i += blockDim.x) bits3[i] = 0u;
  __syncthreads();
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
    const uint2 h = flat_hash2_b((uint64_t)sflat[j], kBloomBits3);
    atomicOr(&bits3[h.x >> 5], 1u << (h.x & 31));
    atomicOr(&bits3[h.y >> 5], 1u << (h.y & 31));
  }
  __syncthreads();
  auto probe = [&](int64_t e, int64_t flat) {
    const uint2 h = flat_hash2_b((uint64_t)flat, kBloomBits3);
    if (!((bits3[h.x >> 5] >> (h.x & 31)) & (bits3[h.y >> 5] >> (h.y & 31)) & 1u)) return;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (sflat[mid] < flat) lo = mid + 1; else hi = mid;
    }
    if (lo < m && sflat[lo] == flat) {
      const unsigned long long slot = atomicAdd(count, 1ull);
      if ((int64_t)slot < cap) {
        out_key[slot] = flat * s_n + cmode[e];
        out_val[slot] = vals[e];
      }
    }
  };
  const int64_t n4 = nnz >> 2;
  const int4* a4 = reinterpret_cast<const int4*>(ca);
  const int4* b4 = reinterpret_cast<const int4*>(cb);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // register double buffer: the next U groups' loads are in flight while the
  // current ones are probed
  int4 av[U], bv[U];
  auto load = [&](int64_t g0, int4* a, int4* b) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t g = g0 + u * stride;
      a[u] = g < n4 ? __ldcs(a4 + g) : make_int4(0, 0, 0, 0);
      b[u] = g < n4 ? __ldcs(b4 + g) : make_int4(0, 0, 0, 0);
    }
  };
  int64_t g0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  load(g0, av, bv);
  for (; g0 < n4; g0 += U * stride) {
    int4 an[U], bn[U];
    load(g0 + U * stride, an, bn);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t g = g0 + u * stride;
      if (g >= n4) continue;
      probe(4 * g + 0, (int64_t)av[u].x * ext_b + bv[u].x);
      probe(4 * g + 1, (int64_t)av[u].y * ext_b + bv[u].y);
      probe(4 * g + 2, (int64_t)av[u].z * ext_b + bv[u].z);
      probe(4 * g + 3, (int64_t)av[u].w * ext_b + bv[u].w);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      av[u] = an[u];
      bv[u] = bn[u];
    }
  }
  if (blockIdx.x == 0)
    for (int64_t e = 4 * n4 + threadIdx.x; e < nnz; e += blockDim.x)
      probe(e, (int64_t)ca[e] * ext_b + cb[e]);
}

// ---- sampled fibres of an order-3 tensor from its mode-0 fibre layout ----
// Modes 1 and 2 of a leverage sub-problem sample fibres (i0, i_b): every
// hit lies in slice i0 of the mode-0 layout (records {i1, i2 | sketch bits,
// v} sorted by (i1, i2)).  Mode 2 (fibre (i0, i1)): the hits are the
// records of slice i0 with c1 == i1, a contiguous run found by binary
// search.  Mode 1 (fibre (i0, i2)): a warp scans the slice (~nnz/s0 records)
// for c2 == i2.  Hits come out per sample in ascending column order, as the
// key-sorted gather gives them.  Replaces the full pass over the coordinates
// (12 B/nnz per sub-problem) for these modes.
template <bool WRITE>
__global__ void __launch_bounds__(256) k_slice_hits(int mode, const int64_t* __restrict__ colptr0,
                                                    const int4* __restrict__ rec0, uint32_t c1_mask,
                                                    const int64_t* __restrict__ idx,
                                                    const double* __restrict__ w, int64_t m,
                                                    int64_t* __restrict__ cnt,
                                                    const int64_t* __restrict__ off,
                                                    int64_t* __restrict__ hit_col,
                                                    double* __restrict__ hit_val, int64_t cap) {
  const int lane = threadIdx.x & 31;
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (j >= m) return;
  const int64_t i0 = idx[2 * j];
  const int32_t tgt = (int32_t)idx[2 * j + 1];
  int64_t a = colptr0[i0], b = colptr0[i0 + 1];
  const double wj = WRITE ? w[j] : 0.0;
  int64_t o = WRITE ? off[j] : 0;
  if (mode == 2) {
    // run of records with c1 == tgt (c1 = record.x, sorted ascending)
    int64_t lo = a, hi = b;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(&rec0[mid].x) < tgt) lo = mid + 1; else hi = mid;
    }
    int64_t lo2 = lo;
    hi = b;
    while (lo2 < hi) {
      const int64_t mid = (lo2 + hi) >> 1;
      if (__ldg(&rec0[mid].x) <= tgt) lo2 = mid + 1; else hi = mid;
    }
    if (!WRITE) {
      if (lane == 0) cnt[j] = lo2 - lo;
      return;
    }
    for (int64_t e = lo + lane; e < lo2 && o + (e - lo) < cap; e += 32) {
      const int4 r = __ldg(&rec0[e]);
      hit_col[o + (e - lo)] = (int64_t)((uint32_t)r.y & c1_mask);
      hit_val[o + (e - lo)] = wj * __hiloint2double(r.w, r.z);
    }
    return;
  }
  // mode 1: scan the slice for c2 == tgt
  int64_t found = 0;
  for (int64_t base = a; base < b; base += 32) {
    const int64_t e = base + lane;
    int4 r = make_int4(0, -1, 0, 0);
    bool hit = false;
    if (e < b) {
      r = __ldg(&rec0[e]);
      hit = (int32_t)((uint32_t)r.y & c1_mask) == tgt;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, hit);
    if (WRITE && hit) {
      const int64_t at = o + found + __popc(bal & ((1u << lane) - 1u));
      if (at < cap) {  // (a fixed-capacity caller checks the total on the device)
        hit_col[at] = (int64_t)r.x;
        hit_val[at] = wj * __hiloint2double(r.w, r.z);
      }
    }
    found += __popc(bal);
  }
  if (!WRITE && lane == 0) cnt[j] = found;
}

}  // namespace skx

using namespace skx;

extern "C" int skx_filter_fibers_coo(int ndim, const int64_t* shape_h, int mode, int64_t nnz,
                                     const int32_t* const* coords_h, const double* vals,
                                     const int64_t* sflat, int64_t m, int64_t* out_key,
                                     double* out_val, int64_t cap, uint64_t* count,
                                     void* stream) {
  SKX_REQUIRE(ndim >= 2 && ndim <= 8 && mode >= 0 && mode < ndim,
              "skx_filter_fibers_coo: order 2..8 and a valid mode");
  SKX_REQUIRE(m >= 1, "skx_filter_fibers_coo: empty sample");
  cudaStream_t s = (cudaStream_t)stream;
  CoordPack cp{};
  for (int k = 0; k < ndim; ++k) {
    cp.c[k] = coords_h[k];
    cp.ext[k] = shape_h[k];
  }
  cudaMemsetAsync(count, 0, sizeof(uint64_t), s);
  if (nnz == 0) return check_launch("skx_filter_fibers_coo");
  if (ndim == 3) {
    int o[2], k2 = 0;
    for (int k = 0; k < 3; ++k)
      if (k != mode) o[k2++] = k;
    const bool al = ((uintptr_t)cp.c[o[0]] % 16 == 0) && ((uintptr_t)cp.c[o[1]] % 16 == 0);
    if (al) {
      const size_t smem = (size_t)(1 << (kBloomBits3 - 5)) * 4;
      const int64_t blocks = imax(1, imin((nnz + 2047) / 2048, (int64_t)num_sms() * 2));
      // U groups of four nonzeros (2 x 16-byte loads each) per thread, double
      // buffered (config 5, beside K7: U = 2: filter 2.9 ms per pass, call
      // 447 ms; U = 4: 2.57 ms but 449 ms -- its registers crowd K7; without
      // the double buffer U = 2 / 4 / 8 took 3.93 / 3.11 / 5.63 ms)
#ifndef SKX_FILTER_U
#define SKX_FILTER_U 2
#endif
      cudaFuncSetAttribute(k_filter_fibers3v<SKX_FILTER_U>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_filter_fibers3v<SKX_FILTER_U><<<(unsigned)blocks, 256, smem, s>>>(
          cp.c[o[0]], cp.c[o[1]], shape_h[o[1]], cp.c[mode], shape_h[mode], nnz, vals, sflat, m,
          out_key, out_val, cap, (unsigned long long*)count);
      return check_launch("k_filter_fibers3v");
    }
  }
  const int64_t blocks = imin((nnz + 1023) / 1024, (int64_t)num_sms() * 16);
  k_filter_fibers<<<(unsigned)blocks, 256, 0, s>>>(ndim, mode, cp, nnz, vals, sflat, m, out_key,
                                                   out_val, cap, (unsigned long long*)count);
  return check_launch("k_filter_fibers");
}

extern "C" int skx_lev_prepare(const double* scores, int64_t s, double* p, double* cdf, void* ws,
                               size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(s >= 1, "skx_lev_prepare: empty score vector");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_lev_prepare: ws_bytes is NULL");
  Arena ar(ws, *ws_bytes);
  double* part = ar.take<double>(kLevChunks);
  double* tot = ar.take<double>(2);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_lev_prepare: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  if (getenv("SKX_LEV_5K") == nullptr) {  // (the five-launch form stays for A/B runs)
    k_lev_prepare1<<<1, kLevFusedThreads, 0, st>>>(scores, s, p, cdf);
    return check_launch("k_lev_prepare1");
  }
  const unsigned g = kLevChunks / 32;
  k_lev_sums<<<g, 32, 0, st>>>(scores, s, part);
  k_lev_total<<<1, 32, 0, st>>>(part, tot);
  k_lev_scan<<<g, 32, 0, st>>>(scores, s, tot, p, cdf, part);
  k_lev_offsets<<<1, 32, 0, st>>>(s, part, tot);
  k_lev_final<<<g, 32, 0, st>>>(s, part, tot, cdf);
  return check_launch("lev_prepare", 5);
}

extern "C" int skx_lev_sample(int n_other, const int64_t* ext_h, const double* const* p_h,
                              const double* const* cdf_h, int64_t m, uint64_t k0, uint64_t k1,
                              uint64_t p0, int64_t* idx, double* w, void* stream) {
  SKX_REQUIRE(n_other >= 1 && n_other <= 15, "skx_lev_sample: 1..15 modes");
  SKX_REQUIRE(m >= 1, "skx_lev_sample: sample count must be positive");
  PtrPack pk{};
  for (int k = 0; k < n_other; ++k) {
    pk.p[k] = p_h[k];
    pk.c[k] = cdf_h[k];
    pk.ext[k] = ext_h[k];
  }
  k_lev_sample<<<(unsigned)((m + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n_other, pk, m, k0, k1,
                                                                              p0, idx, w);
  return check_launch("k_lev_sample");
}

extern "C" int skx_kron_rows(int n_other, const int64_t* ranks_h, const double* const* factors_h,
                             const int64_t* idx, const double* w, int64_t m, double* z,
                             void* stream) {
  SKX_REQUIRE(n_other >= 1 && n_other <= 15, "skx_kron_rows: 1..15 modes");
  FacPack fp{};
  int64_t r = 1;
  for (int k = 0; k < n_other; ++k) {
    fp.a[k] = factors_h[k];
    fp.R[k] = ranks_h[k];
    r *= ranks_h[k];
  }
  const int64_t n = m * r;
  if (n == 0) return SKX_OK;
  k_kron_rows<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n_other, fp, r, idx, w,
                                                                              m, z);
  return check_launch("k_kron_rows");
}

extern "C" int skx_gather_fibers_dense(const double* t, int ndim, const int64_t* shape_h, int mode,
                                       const int64_t* idx, const double* w, int64_t m, double* y,
                                       void* stream) {
  SKX_REQUIRE(ndim >= 2 && ndim <= 16 && mode >= 0 && mode < ndim, "skx_gather_fibers_dense: bad mode");
  ShapePack sp{};
  sp.ndim = ndim;
  sp.mode = mode;
  int64_t st = 1;
  for (int k = ndim - 1; k >= 0; --k) {
    sp.shape[k] = shape_h[k];
    sp.stride[k] = st;
    st *= shape_h[k];
  }
  const int64_t n = m * shape_h[mode];
  if (n == 0) return SKX_OK;
  k_gather_dense<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(t, sp, ndim - 1, idx,
                                                                                 w, m, y);
  return check_launch("k_gather_dense");
}

extern "C" int skx_gather_fibers_coo(int n_other, const int64_t* ext_h, int64_t s_n, int64_t nnz,
                                     const int64_t* keys, const double* vals, const int64_t* idx,
                                     const double* w, int64_t m, int64_t* hit_off, int64_t* hit_col,
                                     double* hit_val, int64_t cap, void* ws, size_t* ws_bytes,
                                     void* stream) {
  SKX_REQUIRE(n_other >= 1 && n_other <= 15, "skx_gather_fibers_coo: 1..15 modes");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_gather_fibers_coo: ws_bytes is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  Arena ar(ws, *ws_bytes);
  int64_t* lo = ar.take<int64_t>(m);
  int64_t* cnt = ar.take<int64_t>(m + 1);
  size_t cb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cb, cnt, hit_off, (int)(m + 1), s);
  void* tmp = ar.take<char>(cb);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_gather_fibers_coo: workspace too small");
  PtrPack pk{};
  for (int k = 0; k < n_other; ++k) pk.ext[k] = ext_h[k];
  const unsigned g = (unsigned)((m + 255) / 256);
  cudaMemsetAsync(cnt + m, 0, sizeof(int64_t), s);
  k_gather_coo_count<<<g, 256, 0, s>>>(n_other, pk, s_n, nnz, keys, idx, m, lo, cnt);
  cub::DeviceScan::ExclusiveSum(tmp, cb, cnt, hit_off, (int)(m + 1), s);
  k_gather_coo_write<<<g, 256, 0, s>>>(keys, vals, s_n, lo, cnt, hit_off, w, m, cap, hit_col,
                                       hit_val);
  return check_launch("gather_fibers_coo", 3);
}

extern "C" int skx_slice_hits(int mode, int64_t s0, const int64_t* colptr0, const void* rec0,
                              uint32_t c1_mask, const int64_t* idx, const double* w, int64_t m,
                              int64_t* hit_off, int64_t* hit_col, double* hit_val, int64_t cap,
                              void* ws, size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(mode == 1 || mode == 2, "skx_slice_hits: mode 1 or 2 of an order-3 tensor");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_slice_hits: ws_bytes is NULL");
  (void)s0;
  Arena ar(ws, *ws_bytes);
  int64_t* cnt = ar.take<int64_t>(m + 1);
  size_t cb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cb, cnt, hit_off, (int)(m + 1));
  void* tmp = ar.take<char>(cb);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_slice_hits: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned g = (unsigned)((m * 32 + 255) / 256);
  const int4* r = (const int4*)rec0;
  if (hit_col == nullptr) {  // count pass: hit_off[m] = total
    cudaMemsetAsync(cnt + m, 0, sizeof(int64_t), st);
    k_slice_hits<false><<<g, 256, 0, st>>>(mode, colptr0, r, c1_mask, idx, w, m, cnt, nullptr,
                                           nullptr, nullptr, 0);
    cub::DeviceScan::ExclusiveSum(tmp, cb, cnt, hit_off, (int)(m + 1), st);
    return check_launch("k_slice_hits(count)", 2);
  }
  SKX_REQUIRE(cap >= 0, "skx_slice_hits: negative capacity");
  k_slice_hits<true><<<g, 256, 0, st>>>(mode, colptr0, r, c1_mask, idx, w, m, nullptr, hit_off,
                                        hit_col, hit_val, cap);
  return check_launch("k_slice_hits(write)");
}
