// Shared device/host helpers for libskx (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <string>

#include "../../include/skx.h"

namespace skx {

__host__ __device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }
__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// ---------------------------------------------------------------- host side
void set_error(const char* fmt, ...);
extern std::atomic<long long> g_launches;

inline int check_launch(const char* what, int nlaunch = 1) {
  g_launches.fetch_add(nlaunch, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return SKX_ECUDA;
  }
  return SKX_OK;
}

#define SKX_TRY(x)            \
  do {                        \
    int _rc = (x);            \
    if (_rc != SKX_OK) return _rc; \
  } while (0)

#define SKX_REQUIRE(cond, ...)     \
  do {                             \
    if (!(cond)) {                 \
      ::skx::set_error(__VA_ARGS__); \
      return SKX_EINVAL;           \
    }                              \
  } while (0)

inline int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

inline int max_smem_optin() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (n <= 0) n = 227 * 1024;
  }
  return n;
}

inline int max_smem_sm() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    if (n <= 0) n = 228 * 1024;
  }
  return n;
}

// Warps per CTA (<= 8) maximising resident warps per SM when every warp needs
// `per_warp` bytes of shared memory (1 KB per CTA is reserved by the driver).
inline int warps_per_cta_for(int64_t per_warp) {
  int best = 0, best_nw = 0;
  for (int nw = 1; nw <= 8; ++nw) {
    const int64_t cta = nw * per_warp;
    if (cta > max_smem_optin()) break;
    const int ctas = (int)(max_smem_sm() / (cta + 1024));
    if (ctas * nw > best) best = ctas * nw, best_nw = nw;
  }
  return best_nw;
}

// Bump-allocator over a caller-provided workspace (no hidden allocations).
struct Arena {
  char* base;
  size_t cap, used = 0;
  Arena(void* p, size_t c) : base((char*)p), cap(c) {}
  template <class T>
  T* take(size_t n) {
    size_t off = (used + 255) & ~size_t(255);
    used = off + n * sizeof(T);
    return (base && used <= cap) ? (T*)(base + off) : nullptr;
  }
  bool ok() const { return base == nullptr || used <= cap; }
};

// ---------------------------------------------------------------- device side
// Philox4x64-10 exactly as numpy's Philox bit generator (Random123 constants).
// Raw u64 number p of a stream with key (k0, k1) is word (p & 3) of the block
// computed at counter (p/4 + 1, 0, 0, 0)  (numpy pre-increments the counter).
struct U64x4 {
  uint64_t v[4];
};

__device__ __forceinline__ U64x4 philox_block(uint64_t k0, uint64_t k1, uint64_t c0) {
  uint64_t x0 = c0, x1 = 0, x2 = 0, x3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    const uint64_t m0 = 0xD2E7470EE14C6C93ULL, m1 = 0xCA5A826395121157ULL;
    uint64_t hi0 = __umul64hi(m0, x0), lo0 = m0 * x0;
    uint64_t hi1 = __umul64hi(m1, x2), lo1 = m1 * x2;
    uint64_t n0 = hi1 ^ x1 ^ k0;
    uint64_t n2 = hi0 ^ x3 ^ k1;
    x0 = n0;
    x1 = lo1;
    x2 = n2;
    x3 = lo0;
  }
  U64x4 o;
  o.v[0] = x0;
  o.v[1] = x1;
  o.v[2] = x2;
  o.v[3] = x3;
  return o;
}

__device__ __forceinline__ uint64_t philox_raw(uint64_t k0, uint64_t k1, uint64_t p) {
  U64x4 b = philox_block(k0, k1, (p >> 2) + 1);
  uint64_t w = p & 3;
  return w == 0 ? b.v[0] : w == 1 ? b.v[1] : w == 2 ? b.v[2] : b.v[3];
}

__device__ __forceinline__ double u64_to_unit(uint64_t r) {
  return (double)(r >> 11) * (1.0 / 9007199254740992.0);
}

// 32-bit draw number q of a "u32 run" that starts at raw index p0, optionally
// preceded by a buffered high half (numpy's has_uint32 / uinteger).
struct U32Stream {
  uint64_t k0, k1, p0;
  uint32_t has_pending, pending;
  __device__ __forceinline__ uint32_t at(uint64_t q) const {
    if (has_pending) {
      if (q == 0) return pending;
      q -= 1;
    }
    uint64_t r = philox_raw(k0, k1, p0 + (q >> 1));
    return (q & 1) ? (uint32_t)(r >> 32) : (uint32_t)r;
  }
};

// Fibre-major COO record (skx_layout.cu): NO other-mode int32 coordinates then
// the f64 value; stride RW 8-byte words (2 for NO <= 2: one 16-byte load).
template <int NO>
__device__ __forceinline__ void load_rec(const double* __restrict__ rec, int64_t e, int32_t* c,
                                         double& v) {
  if (NO <= 2) {
    const int4 q = __ldcs(reinterpret_cast<const int4*>(rec) + e);
    c[0] = q.x;
    if (NO > 1) c[1] = q.y;
    v = __hiloint2double(q.w, q.z);
  } else {
    const int2* p = reinterpret_cast<const int2*>(rec + e * 3);
    const int2 a = __ldcs(p), b = __ldcs(p + 1);
    c[0] = a.x;
    c[1] = a.y;
    c[2] = b.x;
    if (NO > 3) c[3] = b.y;
    v = __ldcs(rec + e * 3 + 2);
  }
}

// Packed sketch table entry: low 31 bits bucket, bit 31 set for sign -1.
__device__ __forceinline__ uint32_t pk_bucket(uint32_t e) { return e & 0x7fffffffu; }
__device__ __forceinline__ uint32_t pk_neg(uint32_t e) { return e >> 31; }

// Ordered, deterministic warp accumulation into a warp-private shared-memory
// vector: lanes holding the same bucket are summed in lane order by the lowest
// lane of the group, which then performs the only write to that bucket.
// Every lane must call this (full-warp convergent); inactive lanes pass
// kNoBucket.
//
// Duplicate detection: match_any costs ~375 cycles of latency and ~62 SM
// cycles of issue per call on B200 when the 32 values are distinct (measured;
// ~2 cycles when they are equal), so with `tags` (one byte per bucket,
// warp-private, contents irrelevant between calls) every lane first stores
// its lane id at tags[bucket] and reads it back: if no lane sees a foreign id
// the buckets are distinct and each lane adds directly; only slices with a
// real duplicate pay for match_any.
constexpr uint32_t kNoBucket = 0xffffffffu;

__device__ __forceinline__ void warp_ordered_add_slow(double* acc, uint32_t bucket, double val,
                                                      double* stage) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned peers = __match_any_sync(0xffffffffu, bucket);
  stage[lane] = val;
  __syncwarp();
  if (lane == (unsigned)(__ffs(peers) - 1) && bucket != kNoBucket) {
    double s = acc[bucket];
    unsigned mask = peers;
    while (mask) {
      const int l = __ffs(mask) - 1;
      s += stage[l];
      mask &= mask - 1;
    }
    acc[bucket] = s;
  }
}

__device__ __forceinline__ void warp_ordered_add(double* acc, uint32_t bucket, double val,
                                                 double* stage, uint8_t* tags = nullptr) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const bool has = bucket != kNoBucket;
  bool distinct;
  if (tags != nullptr) {
    if (has) tags[bucket] = (uint8_t)lane;
    __syncwarp();
    // lanes whose tag store was overwritten share their bucket with another lane
    const unsigned lose = __ballot_sync(full, has && tags[bucket] != (uint8_t)lane);
    if (lose == 0u) {
      if (has) acc[bucket] += val;
    } else {
      // rare collision path: resolve one group per losing lane (shfl + ballot,
      // ~10x cheaper than match_any on 32 distinct values); each group's
      // lowest lane adds its members in lane order, everyone else directly
      stage[lane] = val;
      __syncwarp();
      unsigned pend = lose, grouped = 0u;
      while (pend) {
        const uint32_t bl = __shfl_sync(full, bucket, __ffs(pend) - 1);
        const unsigned peers = __ballot_sync(full, bucket == bl);
        grouped |= peers;
        pend &= ~peers;
        if (lane == (unsigned)(__ffs(peers) - 1)) {
          double s = acc[bl];
          unsigned mask = peers;
          while (mask) {
            s += stage[__ffs(mask) - 1];
            mask &= mask - 1;
          }
          acc[bl] = s;
        }
      }
      if (has && !((grouped >> lane) & 1u)) acc[bucket] += val;
    }
    __syncwarp();
    return;
  } else {
    const unsigned peers = __match_any_sync(full, bucket);
    distinct = __all_sync(full, peers == (1u << lane) || !has);
  }
  if (distinct) {
    if (has) acc[bucket] += val;
  } else {
    warp_ordered_add_slow(acc, bucket, val, stage);
  }
  __syncwarp();
}

}  // namespace skx
