// Composite C-ABI entries of SURVEY 8(b)'s minimum export list that a C,
// ctypes, cgo or JNI caller binds without the Python layer: the fitness of a
// Tucker or CP model against a tensor (src/tensors.py:339-368) as one call
// each, and a thin NCCL binding for the multi-GPU reductions.
// They compose the kernels the Python layer drives (skx_tucker_cross_coo,
// skx_cp_cross_fibre3 / _coo, skx_ttm_lead, skx_sumsq) plus small
// deterministic finishing kernels, with the same workspace convention
// (ws = NULL: size query) and no host synchronisation.
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>
#include <stdlib.h>
#include <string.h>

#include "skx_common.cuh"

namespace skx {

// 1 - sqrt(max(||T||^2 - 2 cross + ||model||^2, 0)) / ||T||  (src/tensors.py:362-368)
__global__ void k_fit_finish(const double* norm2, const double* cross, const double* modsq,
                             double* fit) {
  const double n2 = *norm2;
  double r2 = n2 - 2.0 * (*cross) + *modsq;
  if (r2 < 0.0) r2 = 0.0;
  *fit = 1.0 - sqrt(r2) / sqrt(n2);
}

// <a, b> over n doubles in one CTA, fixed order (deterministic): the dense
// Tucker cross term <ttmc(T, {A}), C> (at most 32^ndim entries)
__global__ void __launch_bounds__(256) k_dot_small(const double* __restrict__ a,
                                                   const double* __restrict__ b, int64_t n,
                                                   double* __restrict__ out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(a[i], b[i], s);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if ((int)threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

constexpr int kGramChunks = 296;  // fixed row chunks: deterministic partial sums

// part[c][p * R + q] = sum over rows of chunk c (in order) of a_ip a_iq, R <= 32
__global__ void __launch_bounds__(256) k_gram_part(const double* __restrict__ a, int64_t s, int R,
                                                   double* __restrict__ part) {
  const int64_t per = (s + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = imin(s, lo + per);
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int p = e / R, q = e - p * R;
    double acc = 0.0;
    for (int64_t i = lo; i < hi; ++i) acc = fma(a[i * R + p], a[i * R + q], acc);
    part[(int64_t)blockIdx.x * R * R + e] = acc;
  }
}

// ||CP model||^2 = sum_pq (w_p w_q) prod_n (A_n^T A_n)_pq from the factors'
// Gram partials (summed in chunk order), then the fitness
__global__ void __launch_bounds__(1024) k_cp_fit_finish(const double* __restrict__ part, int ndim,
                                                        int chunks, int R,
                                                        const double* __restrict__ w,
                                                        const double* norm2, const double* cross,
                                                        double* fit) {
  __shared__ double red[1024];
  double v = 0.0;
  const int e = threadIdx.x;
  if (e < R * R) {
    const int p = e / R, q = e - p * R;
    double had = w[p] * w[q];
    for (int n = 0; n < ndim; ++n) {
      double g = 0.0;
      for (int c = 0; c < chunks; ++c) g += part[((int64_t)n * chunks + c) * R * R + e];
      had *= g;
    }
    v = had;
  }
  red[e] = v;
  __syncthreads();
  for (int h = 512; h > 0; h >>= 1) {
    if (e < h) red[e] += red[e + h];
    __syncthreads();
  }
  if (e == 0) {
    const double n2 = *norm2;
    double r2 = n2 - 2.0 * (*cross) + red[0];
    if (r2 < 0.0) r2 = 0.0;
    *fit = 1.0 - sqrt(r2) / sqrt(n2);
  }
}

}  // namespace skx

using namespace skx;

extern "C" int skx_fitness_tucker_coo(int ndim, const int64_t* shape_h, const int64_t* ranks_h,
                                      int64_t nnz, const int32_t* coords, const double* vals,
                                      const double* const* factors_h, const double* core,
                                      const int64_t* colptr0, const void* rec0, uint32_t c1_mask,
                                      const double* norm2, double* fit, void* ws,
                                      size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(ws_bytes != nullptr, "skx_fitness_tucker_coo: ws_bytes is NULL");
  SKX_REQUIRE(ndim >= 1 && ndim <= 8, "skx_fitness_tucker_coo: order 1..8");
  int64_t ncore = 1;
  for (int k = 0; k < ndim; ++k) ncore *= ranks_h[k];
  size_t cross_ws = 0, sq_ws = 0;
  SKX_TRY(skx_tucker_cross_coo(ndim, shape_h, ranks_h, nnz, coords, vals, factors_h, core, colptr0,
                               rec0, c1_mask, nullptr, nullptr, &cross_ws, stream));
  SKX_TRY(skx_sumsq(core, ncore, nullptr, nullptr, &sq_ws, stream));
  size_t sq_ws2 = 0;
  SKX_TRY(skx_sumsq(vals, nnz, nullptr, nullptr, &sq_ws2, stream));
  sq_ws = sq_ws > sq_ws2 ? sq_ws : sq_ws2;
  Arena ar(ws, *ws_bytes);
  double* sc = ar.take<double>(4);  // cross, ||C||^2, ||T||^2
  char* wc = ar.take<char>(cross_ws);
  char* ws2 = ar.take<char>(sq_ws);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_fitness_tucker_coo: workspace too small");
  SKX_REQUIRE(nnz > 0 || norm2 != nullptr, "skx_fitness_tucker_coo: zero-norm tensor");
  size_t b = cross_ws;
  SKX_TRY(skx_tucker_cross_coo(ndim, shape_h, ranks_h, nnz, coords, vals, factors_h, core, colptr0,
                               rec0, c1_mask, sc + 0, wc, &b, stream));
  b = sq_ws;
  SKX_TRY(skx_sumsq(core, ncore, sc + 1, ws2, &b, stream));
  if (norm2 == nullptr) {
    b = sq_ws;
    SKX_TRY(skx_sumsq(vals, nnz, sc + 2, ws2, &b, stream));
    norm2 = sc + 2;
  }
  k_fit_finish<<<1, 1, 0, (cudaStream_t)stream>>>(norm2, sc + 0, sc + 1, fit);
  return check_launch("skx_fitness_tucker_coo");
}

extern "C" int skx_fitness_tucker_dense(int ndim, const int64_t* shape_h, const double* t,
                                        const int64_t* ranks_h, const double* const* factors_h,
                                        const double* core, const double* norm2, double* fit,
                                        void* ws, size_t* ws_bytes, void* stream) {
  SKX_REQUIRE(ws_bytes != nullptr, "skx_fitness_tucker_dense: ws_bytes is NULL");
  SKX_REQUIRE(ndim >= 1 && ndim <= 8, "skx_fitness_tucker_dense: order 1..8");
  int64_t numel = 1, ncore = 1, big = 0;
  int64_t shp[8];
  for (int k = 0; k < ndim; ++k) {
    SKX_REQUIRE(ranks_h[k] >= 1 && ranks_h[k] <= 32 && ranks_h[k] <= shape_h[k],
                "skx_fitness_tucker_dense: ranks 1..min(32, s_k)");
    numel *= shape_h[k];
    ncore *= ranks_h[k];
    shp[k] = shape_h[k];
  }
  // mode products in ascending mode order (the first streams the tensor
  // once): the largest intermediate is after the first product
  {
    int64_t cur = numel;
    for (int k = 0; k < ndim; ++k) {
      cur = cur / shp[k] * ranks_h[k];
      big = cur > big ? cur : big;
    }
  }
  size_t sq_ws = 0;
  SKX_TRY(skx_sumsq(t, numel, nullptr, nullptr, &sq_ws, stream));
  Arena ar(ws, *ws_bytes);
  double* sc = ar.take<double>(4);
  double* buf0 = ar.take<double>((size_t)big);
  double* buf1 = ar.take<double>((size_t)big);
  char* ws2 = ar.take<char>(sq_ws);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_fitness_tucker_dense: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const double* cur = t;
  double* bufs[2] = {buf0, buf1};
  for (int k = 0; k < ndim; ++k) {
    int64_t B = 1, P = 1;
    for (int j = 0; j < k; ++j) B *= shp[j];
    for (int j = k + 1; j < ndim; ++j) P *= shp[j];
    double* out = bufs[k & 1];
    SKX_TRY(skx_ttm_lead(cur, B, shp[k], P, factors_h[k], (int)ranks_h[k], out, stream));
    shp[k] = ranks_h[k];
    cur = out;
  }
  k_dot_small<<<1, 256, 0, st>>>(cur, core, ncore, sc + 0);
  size_t b = sq_ws;
  SKX_TRY(skx_sumsq(core, ncore, sc + 1, ws2, &b, stream));
  if (norm2 == nullptr) {
    b = sq_ws;
    SKX_TRY(skx_sumsq(t, numel, sc + 2, ws2, &b, stream));
    norm2 = sc + 2;
  }
  k_fit_finish<<<1, 1, 0, st>>>(norm2, sc + 0, sc + 1, fit);
  return check_launch("skx_fitness_tucker_dense", 2);
}

extern "C" int skx_fitness_cp_coo(int ndim, const int64_t* shape_h, int R, int64_t nnz,
                                  const int32_t* coords, const double* vals,
                                  const double* const* factors_h, const double* weights,
                                  const int64_t* colptr0, const void* rec0, uint32_t c1_mask,
                                  const double* norm2, double* fit, void* ws, size_t* ws_bytes,
                                  void* stream) {
  SKX_REQUIRE(ws_bytes != nullptr, "skx_fitness_cp_coo: ws_bytes is NULL");
  SKX_REQUIRE(ndim >= 1 && ndim <= 8, "skx_fitness_cp_coo: order 1..8");
  SKX_REQUIRE(R >= 1 && R <= 32, "skx_fitness_cp_coo: rank 1..32");
  const bool fibre = ndim == 3 && colptr0 != nullptr && rec0 != nullptr;
  size_t cross_ws = 0, sq_ws = 0;
  if (fibre)
    SKX_TRY(skx_cp_cross_fibre3(shape_h[0], colptr0, rec0, c1_mask, R, factors_h, weights, nullptr,
                                nullptr, &cross_ws, stream));
  else
    SKX_TRY(skx_cp_cross_coo(ndim, shape_h, R, nnz, coords, vals, factors_h, weights, nullptr,
                             nullptr, &cross_ws, stream));
  SKX_TRY(skx_sumsq(vals, nnz, nullptr, nullptr, &sq_ws, stream));
  Arena ar(ws, *ws_bytes);
  double* sc = ar.take<double>(4);
  double* part = ar.take<double>((size_t)ndim * kGramChunks * R * R);
  char* wc = ar.take<char>(cross_ws);
  char* ws2 = ar.take<char>(sq_ws);
  if (ws == nullptr) {
    *ws_bytes = ar.used + 256;
    return SKX_OK;
  }
  SKX_REQUIRE(ar.ok(), "skx_fitness_cp_coo: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  size_t b = cross_ws;
  if (fibre)
    SKX_TRY(skx_cp_cross_fibre3(shape_h[0], colptr0, rec0, c1_mask, R, factors_h, weights, sc + 0,
                                wc, &b, stream));
  else
    SKX_TRY(skx_cp_cross_coo(ndim, shape_h, R, nnz, coords, vals, factors_h, weights, sc + 0, wc,
                             &b, stream));
  if (norm2 == nullptr) {
    b = sq_ws;
    SKX_TRY(skx_sumsq(vals, nnz, sc + 2, ws2, &b, stream));
    norm2 = sc + 2;
  }
  for (int k = 0; k < ndim; ++k)
    k_gram_part<<<kGramChunks, 256, 0, st>>>(factors_h[k], shape_h[k], R,
                                            part + (int64_t)k * kGramChunks * R * R);
  k_cp_fit_finish<<<1, 1024, 0, st>>>(part, ndim, kGramChunks, R, weights, norm2, sc + 0, fit);
  return check_launch("skx_fitness_cp_coo", ndim + 1);
}

// ---------------------------------------------------------------- NCCL
// libnccl is opened at run time (the one already in the process when a
// framework loaded it, else the system's libnccl.so.2): libskx keeps no link
// dependency on it and callers that never reduce never load it.
namespace {
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                 ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*get_error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h != nullptr) {
      api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
      api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
      api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
      api.all_reduce = (decltype(api.all_reduce))dlsym(h, "ncclAllReduce");
      api.reduce_scatter = (decltype(api.reduce_scatter))dlsym(h, "ncclReduceScatter");
      api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
      api.get_error_string = (decltype(api.get_error_string))dlsym(h, "ncclGetErrorString");
      api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce &&
               api.reduce_scatter && api.all_gather && api.get_error_string;
    }
  }
  return api;
}

int nccl_rc(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return SKX_OK;
  set_error("%s: %s", what, nccl().get_error_string ? nccl().get_error_string(r) : "NCCL error");
  return SKX_ECUDA;
}
}  // namespace

#define SKX_NCCL_READY(what) \
  SKX_REQUIRE(nccl().ok, "%s: libnccl.so.2 not found or incomplete", what)

extern "C" int skx_nccl_unique_id(void* id_out) {
  SKX_REQUIRE(id_out != nullptr, "skx_nccl_unique_id: id_out is NULL");
  SKX_NCCL_READY("skx_nccl_unique_id");
  ncclUniqueId id;
  SKX_TRY(nccl_rc(nccl().get_unique_id(&id), "ncclGetUniqueId"));
  memcpy(id_out, &id, sizeof(id));
  return SKX_OK;
}

extern "C" int skx_nccl_init(const void* unique_id, int rank, int nranks, void** comm_out) {
  SKX_REQUIRE(unique_id != nullptr && comm_out != nullptr, "skx_nccl_init: NULL argument");
  SKX_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "skx_nccl_init: rank %d of %d", rank,
              nranks);
  SKX_NCCL_READY("skx_nccl_init");
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  ncclComm_t c = nullptr;
  SKX_TRY(nccl_rc(nccl().comm_init_rank(&c, nranks, id, rank), "ncclCommInitRank"));
  *comm_out = (void*)c;
  return SKX_OK;
}

extern "C" int skx_nccl_destroy(void* comm) {
  SKX_REQUIRE(comm != nullptr, "skx_nccl_destroy: NULL communicator");
  SKX_NCCL_READY("skx_nccl_destroy");
  return nccl_rc(nccl().comm_destroy((ncclComm_t)comm), "ncclCommDestroy");
}

extern "C" int skx_allreduce_sum(void* comm, const double* send, double* recv, int64_t count,
                                 void* stream) {
  SKX_REQUIRE(comm != nullptr && count >= 0, "skx_allreduce_sum: bad arguments");
  SKX_NCCL_READY("skx_allreduce_sum");
  return nccl_rc(nccl().all_reduce(send, recv, (size_t)count, ncclFloat64, ncclSum,
                                   (ncclComm_t)comm, (cudaStream_t)stream),
                 "ncclAllReduce");
}

extern "C" int skx_reduce_scatter_sum(void* comm, const double* send, double* recv,
                                      int64_t recv_count, void* stream) {
  SKX_REQUIRE(comm != nullptr && recv_count >= 0, "skx_reduce_scatter_sum: bad arguments");
  SKX_NCCL_READY("skx_reduce_scatter_sum");
  return nccl_rc(nccl().reduce_scatter(send, recv, (size_t)recv_count, ncclFloat64, ncclSum,
                                       (ncclComm_t)comm, (cudaStream_t)stream),
                 "ncclReduceScatter");
}

extern "C" int skx_allgather(void* comm, const double* send, double* recv, int64_t send_count,
                             void* stream) {
  SKX_REQUIRE(comm != nullptr && send_count >= 0, "skx_allgather: bad arguments");
  SKX_NCCL_READY("skx_allgather");
  return nccl_rc(nccl().all_gather(send, recv, (size_t)send_count, ncclFloat64, (ncclComm_t)comm,
                                   (cudaStream_t)stream),
                 "ncclAllGather");
}
