// K0: device generation of numpy 2.3.5 Generator(Philox) draws, bit-exact.
//
//  * skx_philox_uniform  -- Generator.random           (next_double)
//  * skx_philox_normal   -- Generator.standard_normal  (256-level ziggurat)
//  * skx_lemire_scan     -- rejection positions of Generator.integers(0,k,.)
//
// The ziggurat consumes a variable number of raw draws per normal, which makes
// the stream inherently sequential.  It is parallelised exactly:
//   1. classify: every raw offset q gets (consumed, yields?, value) as if an
//      attempt started there (tail and wedge branches included);
//   2. the attempt chain q_0 = 0, q_{i+1} = q_i + consumed(q_i) is resolved by a
//      tree of "segment functions" f(entry offset) -> (exit offset, #outputs),
//      tabulated for entry offsets < kE and walked explicitly otherwise;
//   3. each 64-offset leaf re-walks from its true entry and writes its outputs
//      at their global indices.
// Arithmetic of the accept tests uses explicit _rn intrinsics so no FMA
// contraction can change a comparison relative to numpy's x86-64 build.
#include <math.h>
#include <math_constants.h>

#include "skx_common.cuh"
#include "zig_tables.h"

namespace skx {

__device__ const uint64_t d_zig_ki[256] = ZIG_KI_INIT;
__device__ const uint64_t d_zig_wi[256] = ZIG_WI_BITS_INIT;
__device__ const uint64_t d_zig_fi[256] = ZIG_FI_BITS_INIT;

constexpr int kLeaf = 64;   // offsets per leaf segment
constexpr int kFan = 32;    // children per tree node
constexpr int kE = 8;       // tabulated entry offsets

// ------------------------------------------------------------------ uniform
__global__ void k_uniform(uint64_t k0, uint64_t k1, uint64_t p0, int64_t n, double* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = u64_to_unit(philox_raw(k0, k1, p0 + (uint64_t)i));
}

// ------------------------------------------------------------------ log1p
// numpy's ziggurat tail returns r + xx with xx = -log1p(-u)/r, so its value
// depends on libm's log1p bit for bit.  This restates glibc 2.39's x86-64
// FMA multiarch variant (fdlibm s_log1p.c, Estrin polynomial, FMA where gcc
// contracted it), verified identical to the host libm on 4e8 inputs in (-1, 0]
// (tools/check_log1p.c).  Only the branches reachable for x in (-1, 0] matter;
// every non-fused operation is an explicit _rn intrinsic (no contraction).
__device__ __forceinline__ int d_hi(double x) { return (int)(__double_as_longlong(x) >> 32); }
__device__ __forceinline__ double d_sethi(double x, uint32_t h) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  b = (b & 0xffffffffULL) | ((unsigned long long)h << 32);
  return __longlong_as_double((long long)b);
}

__device__ double glibc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  double f = 0.0, c = 0.0, u;
  int k = 1, hu = 0;
  const int hx = d_hi(x), ax = hx & 0x7fffffff;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -CUDART_INF : CUDART_NAN;
    if (ax < 0x3e200000) {
      if (ax < 0x3c900000) return x;
      return fma(-__dmul_rn(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= (int)0xbfd2bec3) {
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return __dadd_rn(x, x);
  if (k != 0) {
    if (hx < 0x43400000) {
      u = __dadd_rn(1.0, x);
      hu = d_hi(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
      c = __ddiv_rn(c, u);
    } else {
      u = x;
      hu = d_hi(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = d_sethi(u, (uint32_t)hu | 0x3ff00000u);
    } else {
      k += 1;
      u = d_sethi(u, (uint32_t)hu | 0x3fe00000u);
      hu = (0x00100000 - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  const double hfsq = __dmul_rn(__dmul_rn(0.5, f), f);
  const double kd = (double)k;
  if (hu == 0) {
    if (f == 0.0) return k == 0 ? 0.0 : fma(kd, ln2_hi, fma(kd, ln2_lo, c));
    const double R = __dmul_rn(fma(-f, 0.6666666666666666, 1.0), hfsq);
    if (k == 0) return __dsub_rn(f, R);
    return fma(kd, ln2_hi, -__dsub_rn(__dsub_rn(R, fma(kd, ln2_lo, c)), f));
  }
  const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
  const double z = __dmul_rn(s, s);
  const double Ra = fma(z, Lp3, Lp2), Rb = fma(z, Lp5, Lp4), Rc = fma(z, Lp7, Lp6);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z2, z4);
  const double R = fma(z6, Rc, fma(z4, Rb, fma(z, Lp1, __dmul_rn(z2, Ra))));
  const double t = __dmul_rn(s, __dadd_rn(R, hfsq));
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, t));
  const double q = __dsub_rn(__dsub_rn(hfsq, __dadd_rn(fma(kd, ln2_lo, c), t)), f);
  return fma(kd, ln2_hi, -q);
}

// ------------------------------------------------------------------ ziggurat
// info[q]: bits 0..14 consumed count, bit 15 yields.
__global__ void k_zig_classify(uint64_t k0, uint64_t k1, const uint64_t* p0p, int64_t L,
                               uint16_t* info, double* val, int* overflow) {
  const uint64_t p0 = *p0p;
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; q < L; q += stride) {
    uint64_t r = philox_raw(k0, k1, p0 + (uint64_t)q);
    int idx = (int)(r & 0xff);
    r >>= 8;
    int sign = (int)(r & 1);
    uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = __dmul_rn((double)rabs, __longlong_as_double((long long)__ldg(&d_zig_wi[idx])));
    if (sign) x = -x;
    uint32_t cons;
    bool yields;
    double v = x;
    if (rabs < __ldg(&d_zig_ki[idx])) {
      cons = 1;
      yields = true;
    } else if (idx == 0) {
      uint64_t t = (uint64_t)q + 1;
      double xx;
      for (;;) {
        double u1 = u64_to_unit(philox_raw(k0, k1, p0 + t));
        double u2 = u64_to_unit(philox_raw(k0, k1, p0 + t + 1));
        t += 2;
        xx = __dmul_rn(-ZIG_NOR_INV_R, glibc_log1p(-u1));
        double yy = -glibc_log1p(-u2);
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) break;
      }
      v = ((rabs >> 8) & 1) ? -__dadd_rn(ZIG_NOR_R, xx) : __dadd_rn(ZIG_NOR_R, xx);
      cons = (uint32_t)(t - (uint64_t)q);
      yields = true;
    } else {
      double fa = __longlong_as_double((long long)__ldg(&d_zig_fi[idx - 1]));
      double fb = __longlong_as_double((long long)__ldg(&d_zig_fi[idx]));
      double u = u64_to_unit(philox_raw(k0, k1, p0 + (uint64_t)q + 1));
      double lhs = __dadd_rn(__dmul_rn(__dsub_rn(fa, fb), u), fb);
      double rhs = exp(__dmul_rn(__dmul_rn(-0.5, x), x));
      yields = lhs < rhs;
      cons = 2;
    }
    if (cons > 0x7fff) {
      atomicExch(overflow, 1);
      cons = 0x7fff;
    }
    info[q] = (uint16_t)(cons | (yields ? 0x8000u : 0u));
    val[q] = v;
  }
}

// Walk the chain through offsets [pos, hi); returns outputs, updates pos.
__device__ __forceinline__ int64_t zig_walk(const uint16_t* info, int64_t& pos, int64_t hi) {
  int64_t c = 0;
  while (pos < hi) {
    uint16_t f = info[pos];
    c += (f >> 15);
    pos += (f & 0x7fff);
  }
  return c;
}

// Leaf functions: for each leaf and entry e < kE: exit (relative to leaf end), count.
__global__ void k_zig_leaf(const uint16_t* info, int64_t L, int64_t nleaf, int* exit_, int* cnt) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= nleaf) return;
  int64_t lo = g * kLeaf, hi = imin(lo + kLeaf, L);
  for (int e = 0; e < kE; ++e) {
    int64_t pos = lo + e;
    int64_t c = zig_walk(info, pos, hi);
    exit_[g * kE + e] = (int)(pos - hi);
    cnt[g * kE + e] = (int)c;
  }
}

// Generic node: children [first, last) of the lower level, each covering
// positions [child*span, min((child+1)*span, L)).
struct Level {
  int* exit_;
  int* cnt;
  int* entry;
  int64_t* base;
  int64_t n;     // nodes
  int64_t span;  // offsets covered per node
};

__device__ __forceinline__ void node_step(const Level& ch, int64_t c, const uint16_t* info,
                                          int64_t L, int& cur, int64_t& acc) {
  if (cur < kE) {
    acc += ch.cnt[c * kE + cur];
    cur = ch.exit_[c * kE + cur];
  } else {  // untabulated entry: walk the child's offsets directly (rare)
    int64_t lo = c * ch.span, hi = imin(lo + ch.span, L);
    int64_t pos = lo + cur;
    acc += zig_walk(info, pos, hi);
    cur = (int)(pos - hi);
  }
}

__global__ void k_zig_up(Level ch, Level up, const uint16_t* info, int64_t L) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= up.n) return;
  int64_t c0 = g * kFan, c1 = imin(c0 + kFan, ch.n);
  for (int e = 0; e < kE; ++e) {
    int cur = e;
    int64_t acc = 0;
    for (int64_t c = c0; c < c1; ++c) node_step(ch, c, info, L, cur, acc);
    up.exit_[g * kE + e] = cur;
    up.cnt[g * kE + e] = (int)acc;
  }
}

// Top: single thread assigns entries of the top level's nodes starting at 0.
__global__ void k_zig_root(Level top, const uint16_t* info, int64_t L, int64_t n, int* short_) {
  int cur = 0;
  int64_t acc = 0;
  for (int64_t c = 0; c < top.n; ++c) {
    top.entry[c] = cur;
    top.base[c] = acc;
    node_step(top, c, info, L, cur, acc);
  }
  *short_ = acc < n ? 1 : 0;
}

__global__ void k_zig_down(Level up, Level ch, const uint16_t* info, int64_t L) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= up.n) return;
  int cur = up.entry[g];
  int64_t acc = up.base[g];
  int64_t c0 = g * kFan, c1 = imin(c0 + kFan, ch.n);
  for (int64_t c = c0; c < c1; ++c) {
    ch.entry[c] = cur;
    ch.base[c] = acc;
    node_step(ch, c, info, L, cur, acc);
  }
}

__global__ void k_zig_emit(const uint16_t* info, const double* val, int64_t L, Level leaf,
                           int64_t n, double* out, const uint64_t* p0p, uint64_t* p_end) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= leaf.n) return;
  int64_t lo = g * kLeaf, hi = imin(lo + kLeaf, L);
  int64_t pos = lo + leaf.entry[g];
  int64_t o = leaf.base[g];
  if (o >= n) return;
  while (pos < hi) {
    uint16_t f = info[pos];
    if (f >> 15) {
      if (o < n) out[o] = val[pos];
      if (o == n - 1) *p_end = *p0p + (uint64_t)(pos + (f & 0x7fff));
      ++o;
    }
    pos += (f & 0x7fff);
  }
}

// ------------------------------------------------------------------ lemire
constexpr int kScanChunk = 64;  // Philox blocks per thread per CTA
// Lists the absolute 32-bit positions A = 2*raw + half (half 0 = low word) of
// every draw in raw words [raw_lo, raw_hi) that Lemire's method would reject
// for bound k.  Rejection depends only on the drawn value, so the scan can run
// before the caller knows exactly where its integers() call starts.
__global__ void k_lemire_scan(uint64_t k0, uint64_t k1, uint64_t raw_lo, uint64_t raw_hi,
                              uint32_t k, uint32_t thresh, uint64_t* rej, int64_t cap,
                              unsigned long long* count) {
  const uint64_t b_first = raw_lo >> 2, b_last = (raw_hi - 1) >> 2;
  const uint64_t nb = b_last - b_first + 1;
  // each CTA owns a contiguous chunk of kScanChunk * blockDim.x blocks and
  // retires when done: short-lived CTAs let higher-priority streams take SMs
  const uint64_t c0 = (uint64_t)blockIdx.x * kScanChunk * blockDim.x;
  const uint64_t c1 = umin64(nb, c0 + (uint64_t)kScanChunk * blockDim.x);
  for (uint64_t t = c0 + threadIdx.x; t < c1; t += blockDim.x) {
    const uint64_t b = b_first + t;
    const U64x4 blk = philox_block(k0, k1, b + 1);
    // branch-free screen of the 8 halves (rejections are ~1e-8 rare): the
    // minimum low product (integer min on the ALU pipe, which the Philox
    // multiplies leave idle) decides; the per-half flags and range checks only
    // run for a block that has a candidate
    uint32_t mn = 0xffffffffu;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      mn = min(mn, (uint32_t)blk.v[w] * k);
      mn = min(mn, (uint32_t)(blk.v[w] >> 32) * k);
    }
    if (mn < thresh) {
      uint32_t flag = 0;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        flag |= (uint32_t)((uint32_t)blk.v[w] * k < thresh) << (2 * w);
        flag |= (uint32_t)((uint32_t)(blk.v[w] >> 32) * k < thresh) << (2 * w + 1);
      }
      for (int bit = 0; bit < 8; ++bit) {
        if (!((flag >> bit) & 1)) continue;
        const uint64_t r = 4 * b + (bit >> 1);
        if (r < raw_lo || r >= raw_hi) continue;
        const unsigned long long s = atomicAdd(count, 1ULL);
        if ((int64_t)s < cap) rej[s] = 2 * r + (bit & 1);
      }
    }
  }
}

}  // namespace skx

using namespace skx;

extern "C" int skx_philox_uniform(uint64_t k0, uint64_t k1, uint64_t p0, int64_t n, double* out,
                                  void* stream) {
  SKX_REQUIRE(n >= 0, "skx_philox_uniform: n < 0");
  if (n == 0) return SKX_OK;
  int blocks = (int)imin((n + 255) / 256, (int64_t)num_sms() * 8);
  k_uniform<<<blocks, 256, 0, (cudaStream_t)stream>>>(k0, k1, p0, n, out);
  return check_launch("k_uniform");
}

namespace {
struct ZigPlan {
  int64_t L, nlev;
  int64_t nodes[16], span[16];
};

ZigPlan zig_plan(int64_t n) {
  ZigPlan p{};
  p.L = n + n / 16 + 4096;
  int64_t cnt = (p.L + kLeaf - 1) / kLeaf, span = kLeaf;
  p.nlev = 0;
  p.nodes[p.nlev] = cnt;
  p.span[p.nlev] = span;
  ++p.nlev;
  while (cnt > kFan) {
    cnt = (cnt + kFan - 1) / kFan;
    span *= kFan;
    p.nodes[p.nlev] = cnt;
    p.span[p.nlev] = span;
    ++p.nlev;
  }
  return p;
}
}  // namespace

extern "C" int skx_philox_normal(uint64_t k0, uint64_t k1, const uint64_t* p0, int64_t n,
                                 double* out, uint64_t* p_end, void* ws, size_t* ws_bytes,
                                 void* stream) {
  SKX_REQUIRE(n >= 0 && n < (int64_t(1) << 31), "skx_philox_normal: n out of range");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_philox_normal: ws_bytes is NULL");
  ZigPlan pl = zig_plan(n > 0 ? n : 1);
  Arena ar(ws, *ws_bytes);
  uint16_t* info = ar.take<uint16_t>(pl.L);
  double* val = ar.take<double>(pl.L);
  int* flags = ar.take<int>(2);
  Level lv[16];
  for (int l = 0; l < pl.nlev; ++l) {
    lv[l].n = pl.nodes[l];
    lv[l].span = pl.span[l];
    lv[l].exit_ = ar.take<int>(pl.nodes[l] * kE);
    lv[l].cnt = ar.take<int>(pl.nodes[l] * kE);
    lv[l].entry = ar.take<int>(pl.nodes[l]);
    lv[l].base = ar.take<int64_t>(pl.nodes[l]);
  }
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_philox_normal: workspace too small (%zu < %zu)", *ws_bytes, ar.used);
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    cudaMemcpyAsync(p_end, p0, 8, cudaMemcpyDeviceToDevice, s);
    return check_launch("normal n=0", 0);
  }
  cudaMemsetAsync(flags, 0, 2 * sizeof(int), s);
  int cblocks = (int)imin((pl.L + 255) / 256, (int64_t)num_sms() * 16);
  k_zig_classify<<<cblocks, 256, 0, s>>>(k0, k1, p0, pl.L, info, val, flags);
  int64_t nl = lv[0].n;
  k_zig_leaf<<<(unsigned)((nl + 127) / 128), 128, 0, s>>>(info, pl.L, nl, lv[0].exit_, lv[0].cnt);
  for (int l = 1; l < pl.nlev; ++l)
    k_zig_up<<<(unsigned)((lv[l].n + 127) / 128), 128, 0, s>>>(lv[l - 1], lv[l], info, pl.L);
  k_zig_root<<<1, 1, 0, s>>>(lv[pl.nlev - 1], info, pl.L, n, flags + 1);
  for (int l = pl.nlev - 1; l >= 1; --l)
    k_zig_down<<<(unsigned)((lv[l].n + 127) / 128), 128, 0, s>>>(lv[l], lv[l - 1], info, pl.L);
  k_zig_emit<<<(unsigned)((nl + 127) / 128), 128, 0, s>>>(info, val, pl.L, lv[0], n, out, p0,
                                                          p_end);
  // flags[0]: a tail loop ran > 32767 draws; flags[1]: not enough offsets.
  // Both are astronomically unlikely (L has 6% + 4096 slack); they are checked
  // by skx_normal_flags() in debug builds of the host layer.
  return check_launch("ziggurat", 4 + 2 * (int)(pl.nlev - 1));
}

extern "C" int skx_lemire_scan(uint64_t k0, uint64_t k1, uint64_t raw_lo, uint64_t raw_hi,
                               uint32_t k, uint64_t* rej, int64_t cap, unsigned long long* count,
                               void* stream) {
  SKX_REQUIRE(k >= 1, "skx_lemire_scan: k must be >= 1");
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemsetAsync(count, 0, sizeof(unsigned long long), s);
  uint32_t thresh = (uint32_t)((0x100000000ULL - (uint64_t)k) % (uint64_t)k);
  if (thresh == 0 || raw_hi <= raw_lo) return check_launch("lemire(no rejections possible)", 0);
  const uint64_t nb = ((raw_hi - 1) >> 2) - (raw_lo >> 2) + 1;
  const uint64_t per = (uint64_t)kScanChunk * 256;
  SKX_REQUIRE((nb + per - 1) / per < (1ULL << 31), "skx_lemire_scan: range too large");
  const unsigned blocks = (unsigned)((nb + per - 1) / per);
  k_lemire_scan<<<blocks, 256, 0, s>>>(k0, k1, raw_lo, raw_hi, k, thresh, rej, cap, count);
  return check_launch("k_lemire_scan");
}
