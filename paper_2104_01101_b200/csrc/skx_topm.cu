// Deterministic leverage sampling: the m largest products of one score per
// mode (src/sketching.py:224-259, `_top_m_products`), in the reference's
// best-first pop order.
//
// Per mode the scores are radix-sorted descending with ties by ascending
// index (np.lexsort((arange, -s))).  The pop order of the reference's heap is
// then reproduced exactly by the same best-first search on the device: the
// frontier is a binary min-heap keyed by (-product, original multi-index)
// (keys are unique, so the order does not depend on the heap implementation),
// neighbours of a popped position tuple (one coordinate + 1) are pushed once
// (open-addressing hash set of linearised positions).  Candidate enumeration
// plus a global sort is NOT equivalent when products tie (zero scores, equal
// rows): a tuple only enters the frontier once a predecessor is popped, so
// within a tie group the order is a priority-topological order, not a sort.
//
// The search is inherently sequential (m pops, m*k pushes); it runs in one
// thread with the heap in global memory (L1/L2 resident: m*k*24 bytes).
#include <cub/cub.cuh>

#include "skx_common.cuh"

namespace skx {

constexpr int kTopmMaxModes = 15;

struct TopmPack {
  const double* s[kTopmMaxModes];   // scores sorted descending
  const int64_t* o[kTopmMaxModes];  // original index of each sorted entry
  int64_t len[kTopmMaxModes];
  int64_t stride[kTopmMaxModes];    // C-order strides over len (first slowest)
};

__global__ void k_iota64(int64_t* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = i;
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

// a before b in the reference's heap: larger product first, then smaller
// original multi-index (lexicographic == numeric on the C-order linear index)
__device__ __forceinline__ bool topm_less(double pa, int64_t oa, double pb, int64_t ob) {
  return (-pa < -pb) || (!(-pb < -pa) && oa < ob);
}

__global__ void k_topm_heap(int k, TopmPack pk, int64_t m, int64_t cap, double* hp, int64_t* ho,
                            int64_t* hl, int64_t* set, int64_t set_mask, int64_t* idx) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t n = 0;
  auto push = [&](double p, int64_t o, int64_t l) {
    int64_t i = n++;
    while (i > 0) {
      int64_t par = (i - 1) >> 1;
      if (!topm_less(p, o, hp[par], ho[par])) break;
      hp[i] = hp[par];
      ho[i] = ho[par];
      hl[i] = hl[par];
      i = par;
    }
    hp[i] = p;
    ho[i] = o;
    hl[i] = l;
  };
  auto insert = [&](int64_t key) -> bool {  // true if newly inserted
    uint64_t h = mix64((uint64_t)key) & (uint64_t)set_mask;
    while (true) {
      int64_t cur = set[h];
      if (cur == key) return false;
      if (cur < 0) {
        set[h] = key;
        return true;
      }
      h = (h + 1) & (uint64_t)set_mask;
    }
  };
  // product left to right (float(np.prod([...])) of k doubles)
  auto prod_of = [&](const int64_t* pos) {
    double p = pk.s[0][pos[0]];
    for (int j = 1; j < k; ++j) p *= pk.s[j][pos[j]];
    return p;
  };
  int64_t pos[kTopmMaxModes];
  for (int j = 0; j < k; ++j) pos[j] = 0;
  {
    int64_t o = 0;
    for (int j = 0; j < k; ++j) o += pk.o[j][0] * pk.stride[j];
    insert(0);
    push(prod_of(pos), o, 0);
  }
  for (int64_t out = 0; out < m; ++out) {
    // pop the root
    const int64_t lin = hl[0];
    const int64_t orig = ho[0];
    --n;
    if (n > 0) {
      const double lp = hp[n];
      const int64_t lo = ho[n], ll = hl[n];
      int64_t i = 0;
      while (true) {
        int64_t c = 2 * i + 1;
        if (c >= n) break;
        if (c + 1 < n && topm_less(hp[c + 1], ho[c + 1], hp[c], ho[c])) ++c;
        if (!topm_less(hp[c], ho[c], lp, lo)) break;
        hp[i] = hp[c];
        ho[i] = ho[c];
        hl[i] = hl[c];
        i = c;
      }
      hp[i] = lp;
      ho[i] = lo;
      hl[i] = ll;
    }
    // emit the original multi-index, decode the position tuple
    int64_t rem = orig, rl = lin;
    for (int j = k - 1; j >= 0; --j) {
      idx[out * k + j] = rem % pk.len[j];
      rem /= pk.len[j];
      pos[j] = rl % pk.len[j];
      rl /= pk.len[j];
    }
    if (out + 1 == m) break;
    for (int j = 0; j < k; ++j) {
      if (pos[j] + 1 >= pk.len[j]) continue;
      const int64_t nl = lin + pk.stride[j];
      if (!insert(nl)) continue;
      pos[j] += 1;
      int64_t o = 0;
      for (int q = 0; q < k; ++q) o += pk.o[q][pos[q]] * pk.stride[q];
      const double p = prod_of(pos);
      pos[j] -= 1;
      if (n < cap) push(p, o, nl);
    }
  }
}

}  // namespace skx

using namespace skx;

extern "C" int skx_top_m_products(int k, const int64_t* len_h, const double* const* scores_h,
                                  int64_t m, int64_t* idx, void* ws, size_t* ws_bytes,
                                  void* stream) {
  SKX_REQUIRE(k >= 1 && k <= kTopmMaxModes, "skx_top_m_products: 1..15 modes");
  SKX_REQUIRE(m >= 1, "skx_top_m_products: sample count must be positive");
  SKX_REQUIRE(ws_bytes != nullptr, "skx_top_m_products: ws_bytes is NULL");
  double total = 1.0;
  int64_t maxlen = 0;
  for (int j = 0; j < k; ++j) {
    SKX_REQUIRE(len_h[j] >= 1, "skx_top_m_products: empty score list");
    total *= (double)len_h[j];
    maxlen = imax(maxlen, len_h[j]);
  }
  SKX_REQUIRE((double)m <= total, "skx_top_m_products: cannot select %lld rows from %.0f",
              (long long)m, total);
  SKX_REQUIRE(total < 9.0e18, "skx_top_m_products: index space too large");
  const int64_t cap = m * k + 1;
  int64_t set_size = 1;
  while (set_size < 2 * cap + 16) set_size <<= 1;
  size_t sort_bytes = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, (const double*)nullptr,
                                            (double*)nullptr, (const int64_t*)nullptr,
                                            (int64_t*)nullptr, maxlen);
  Arena ar(ws, *ws_bytes);
  double* srt[kTopmMaxModes];
  int64_t* ord[kTopmMaxModes];
  for (int j = 0; j < k; ++j) {
    srt[j] = ar.take<double>(len_h[j]);
    ord[j] = ar.take<int64_t>(len_h[j]);
  }
  int64_t* iota = ar.take<int64_t>(maxlen);
  void* tmp = ar.take<char>(sort_bytes);
  double* hp = ar.take<double>(cap);
  int64_t* ho = ar.take<int64_t>(cap);
  int64_t* hl = ar.take<int64_t>(cap);
  int64_t* set = ar.take<int64_t>(set_size);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_top_m_products: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  int launches = 0;
  k_iota64<<<(unsigned)imin((maxlen + 255) / 256, 1024), 256, 0, st>>>(iota, maxlen);
  ++launches;
  TopmPack pk{};
  int64_t stride = 1;
  for (int j = k - 1; j >= 0; --j) {
    pk.stride[j] = stride;
    stride *= len_h[j];
  }
  for (int j = 0; j < k; ++j) {
    size_t tb = sort_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(tmp, tb, scores_h[j], srt[j], iota,
                                                              ord[j], len_h[j], 0, 64, st);
    if (e != cudaSuccess) {
      set_error("skx_top_m_products: sort: %s", cudaGetErrorString(e));
      return SKX_ECUDA;
    }
    launches += 3;
    pk.s[j] = srt[j];
    pk.o[j] = ord[j];
    pk.len[j] = len_h[j];
  }
  cudaMemsetAsync(set, 0xFF, (size_t)set_size * sizeof(int64_t), st);
  k_topm_heap<<<1, 32, 0, st>>>(k, pk, m, cap, hp, ho, hl, set, set_size - 1, idx);
  ++launches;
  return check_launch("k_topm_heap", launches);
}
