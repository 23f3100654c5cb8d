/*
 * oracle/rngref.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the numpy 2.3.5 random-stream contract that the
 * reference `sketchals` package (/root/reference/pkg/src/sketchals) draws all
 * its randomness from.  The algorithms live in a third-party dependency that is
 * NOT vendored under /root/reference:
 *
 *   numpy 2.3.5  numpy/random/src/philox/philox.h      Philox4x64-10, counter
 *                                                       pre-incremented per block
 *                numpy/random/src/distributions/distributions.c
 *                  buffered_bounded_lemire_uint32       Lemire bounded uint32
 *                  next_double                           (u64 >> 11) * 2^-53
 *                  random_standard_normal               256-level ziggurat
 *
 * Reference call sites that depend on this contract:
 *   src/rng.py:16-26            make_rng / split_rng -> Generator(Philox(SeedSequence))
 *   src/sketching.py:36,42      rng.integers(0, 2^31-1, size=deg+1)  (TS hash/sign coeffs)
 *   src/sketching.py:56         rng.integers(0, m, n); rng.integers(0, 2, n)  (RRF tables)
 *   src/sketching.py:211        rng.choice(s, m, p)   -> random(m) + searchsorted
 *   src/sketching.py:323        rng.standard_normal((k2, k1))
 *   src/linalg.py:107           rng.standard_normal((s_n, width))
 *
 * Stream addressing used everywhere in this repo: raw u64 number p (0-based,
 * counted from a generator whose counter words are all zero) is word p%4 of
 * the Philox block computed with counter (p/4 + 1, 0, 0, 0).
 *
 * Pinned by tests/test_oracle_rng.py against numpy's own Generator output.
 * Built by oracle/Makefile into oracle/_build/librngref.so.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "zig_tables.h"

typedef unsigned __int128 u128;

static void philox_block(uint64_t k0, uint64_t k1, uint64_t c0, uint64_t c1,
                         uint64_t c2, uint64_t c3, uint64_t out[4]) {
  uint64_t x0 = c0, x1 = c1, x2 = c2, x3 = c3;
  for (int round = 0; round < 10; ++round) {
    if (round) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    u128 p0 = (u128)0xD2E7470EE14C6C93ULL * x0;
    u128 p1 = (u128)0xCA5A826395121157ULL * x2;
    uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    uint64_t n0 = hi1 ^ x1 ^ k0;
    uint64_t n2 = hi0 ^ x3 ^ k1;
    x0 = n0;
    x1 = lo1;
    x2 = n2;
    x3 = lo0;
  }
  out[0] = x0;
  out[1] = x1;
  out[2] = x2;
  out[3] = x3;
}

uint64_t rr_raw(uint64_t k0, uint64_t k1, uint64_t p) {
  uint64_t b[4];
  philox_block(k0, k1, (p >> 2) + 1, 0, 0, 0, b);
  return b[p & 3];
}

void rr_raw_fill(uint64_t k0, uint64_t k1, uint64_t p0, int64_t n, uint64_t *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = rr_raw(k0, k1, p0 + (uint64_t)i);
}

/* numpy next_double */
void rr_uniform_fill(uint64_t k0, uint64_t k1, uint64_t p0, int64_t n, double *out) {
  for (int64_t i = 0; i < n; ++i)
    out[i] = (double)(rr_raw(k0, k1, p0 + (uint64_t)i) >> 11) * (1.0 / 9007199254740992.0);
}

/* 32-bit cursor over the raw stream, mirroring Philox's has_uint32 buffer. */
typedef struct {
  uint64_t k0, k1, p;    /* next raw u64 index                    */
  int has;               /* a buffered high half is pending         */
  uint32_t pending;
} cur32;

static uint32_t next32(cur32 *c) {
  if (c->has) {
    c->has = 0;
    return c->pending;
  }
  uint64_t r = rr_raw(c->k0, c->k1, c->p++);
  c->has = 1;
  c->pending = (uint32_t)(r >> 32);
  return (uint32_t)r;
}

/*
 * Generator.integers(0, k, n) for 1 <= k < 2^32 (int64 output).
 * state_io[0] = next raw index, [1] = has_uint32, [2] = uinteger; updated.
 */
void rr_bounded_fill(uint64_t k0, uint64_t k1, uint64_t *state_io, uint64_t k,
                     int64_t n, int64_t *out) {
  cur32 c = {k0, k1, state_io[0], (int)state_io[1], (uint32_t)state_io[2]};
  const uint32_t kk = (uint32_t)k;
  const uint32_t thresh = (uint32_t)((0x100000000ULL - k) % k);
  for (int64_t i = 0; i < n; ++i) {
    if (k == 1) { out[i] = 0; continue; }
    uint64_t mm = (uint64_t)next32(&c) * kk;
    while ((uint32_t)mm < thresh) mm = (uint64_t)next32(&c) * kk;
    out[i] = (int64_t)(mm >> 32);
  }
  state_io[0] = c.p;
  state_io[1] = (uint64_t)c.has;
  state_io[2] = c.pending;
}

static double bits2d(uint64_t b) {
  double d;
  memcpy(&d, &b, 8);
  return d;
}

static double next_dbl(uint64_t k0, uint64_t k1, uint64_t *p) {
  return (double)(rr_raw(k0, k1, (*p)++) >> 11) * (1.0 / 9007199254740992.0);
}

/* Generator.standard_normal(n); *p_io = next raw index, updated. */
void rr_normal_fill(uint64_t k0, uint64_t k1, uint64_t *p_io, int64_t n, double *out) {
  uint64_t p = *p_io;
  for (int64_t i = 0; i < n; ++i) {
    for (;;) {
      uint64_t r = rr_raw(k0, k1, p++);
      int idx = (int)(r & 0xff);
      r >>= 8;
      int sign = (int)(r & 1);
      uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
      volatile double x = (double)rabs * bits2d(ZIG_WI_BITS[idx]);
      if (sign) x = -x;
      if (rabs < ZIG_KI[idx]) { out[i] = x; break; }
      if (idx == 0) {
        double xx, yy;
        for (;;) {
          xx = -ZIG_NOR_INV_R * log1p(-next_dbl(k0, k1, &p));
          yy = -log1p(-next_dbl(k0, k1, &p));
          if (yy + yy > xx * xx) break;
        }
        out[i] = ((rabs >> 8) & 1) ? -(ZIG_NOR_R + xx) : ZIG_NOR_R + xx;
        break;
      }
      double fa = bits2d(ZIG_FI_BITS[idx - 1]), fb = bits2d(ZIG_FI_BITS[idx]);
      volatile double lhs = (fa - fb) * next_dbl(k0, k1, &p);
      lhs = lhs + fb;
      if (lhs < exp(-0.5 * x * x)) { out[i] = x; break; }
    }
  }
  *p_io = p;
}

/* TensorSketch polynomial hash over GF(2^31-1), Horner in uint64
 * (reference src/sketching.py:25-31). out[i] = poly(i) (before mod m / mod 2). */
void rr_poly_hash(const int64_t *coeffs, int ncoef, int64_t n, uint64_t *out) {
  const uint64_t P = 2147483647ULL;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t acc = (uint64_t)coeffs[0];
    for (int c = 1; c < ncoef; ++c) acc = (acc * (uint64_t)i + (uint64_t)coeffs[c]) % P;
    out[i] = acc;
  }
}
