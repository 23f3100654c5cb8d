// Microbenchmark: random gathers of 160-byte factor rows (2e5 x 20 f64,
// L2-resident) through the TMA unit's tile::gather4 mode (4 rows per
// instruction, sm_100a), NBUF-deep per-warp pipelines, rows consumed from
// shared memory.  Compare with tools/micro/gather.cu (LSU gathers).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4 gather4.cu -lcuda && ./gather4
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int R = 20;
constexpr int ROWB = R * 8;
constexpr int BATCH = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int WARPS, int NBUF, bool CONSUME>
__global__ void __launch_bounds__(WARPS * 32) k_g4(const __grid_constant__ CUtensorMap tm,
                                                 const int* __restrict__ idx, int64_t n, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[WARPS][NBUF];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* buf = sm + (size_t)wid * NBUF * BATCH * ROWB;
  if (lane == 0)
    for (int b = 0; b < NBUF; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[wid][b])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  const int64_t gw = blockIdx.x * (int64_t)WARPS + wid;
  const int64_t tw = (int64_t)gridDim.x * WARPS;
  const int64_t nb = n / BATCH;
  double acc = 0.0;
  uint32_t phase = 0;  // bit b = parity of slot b
  auto issue = [&](int64_t b, int slot) {
    const uint32_t mb = smem_u32(&bar[wid][slot]);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(BATCH * ROWB));
    __syncwarp();
    if (lane < BATCH / 4) {
      const int4 r = reinterpret_cast<const int4*>(idx + b * BATCH)[lane];
      const uint32_t dst = smem_u32(buf + (size_t)slot * BATCH * ROWB + lane * 4 * ROWB);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
          ::"r"(dst), "l"(&tm), "r"(mb), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w)
          : "memory");
    }
  };
  int64_t b = gw;
  for (int s = 0; s < NBUF - 1; ++s)
    if (b + s * tw < nb) issue(b + s * tw, s);
  int slot = 0;
  for (; b < nb; b += tw) {
    const int64_t nx = b + (NBUF - 1) * tw;
    if (nx < nb) issue(nx, (slot + NBUF - 1) % NBUF);
    const uint32_t mb = smem_u32(&bar[wid][slot]);
    uint32_t done = 0;
    const uint32_t ph = (phase >> slot) & 1;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(mb), "r"(ph));
    phase ^= 1u << slot;
    if (CONSUME) {
      const double2* rows = reinterpret_cast<const double2*>(buf + (size_t)slot * BATCH * ROWB);
#pragma unroll
      for (int e = 0; e < BATCH * R / 2 / 32; ++e) {
        const double2 v = rows[e * 32 + lane];
        acc += v.x + v.y;
      }
    }
    __syncwarp();
    slot = (slot + 1) % NBUF;
  }
  if (acc == 12345.678) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int WARPS, int NBUF, bool CONSUME>
void bench(const CUtensorMap& tm, const int* idx, int64_t n, double* out, int sms) {
  auto kern = k_g4<WARPS, NBUF, CONSUME>;
  const size_t smem = (size_t)WARPS * NBUF * BATCH * ROWB;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    kern<<<sms * per_sm, WARPS * 32, smem>>>(tm, idx, n, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep == 2)
      printf("gather4 warps %d nbuf %d consume %d (%d CTA/SM): %.3f ms  %.2f Grows/s  %.2f TB/s\n", WARPS,
             NBUF, (int)CONSUME, per_sm, ms, n / ms / 1e6, n * (double)ROWB / ms / 1e9);
  }
}

int main() {
  const int64_t rows = 200000, n = 1 << 26;
  double* A;
  int* idx;
  double* out;
  CK(cudaMalloc(&A, rows * ROWB));
  CK(cudaMalloc(&idx, n * 4));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(A, 0, rows * ROWB));
  int* h = (int*)malloc(n * 4);
  uint64_t x = 88172645463325252ULL;
  for (int64_t i = 0; i < n; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    h[i] = (int)(x % rows);
  }
  CK(cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t dims[2] = {R, (cuuint64_t)rows};
  cuuint64_t strides[1] = {ROWB};
  cuuint32_t box[2] = {R, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult rc = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc %d\n", (int)rc);
  if (rc != CUDA_SUCCESS) return 1;
  // correctness: gather rows of a table with A[r][k] = r * 100 + k
  {
    double* hA = (double*)malloc(rows * ROWB);
    for (int64_t r = 0; r < rows; ++r)
      for (int k = 0; k < R; ++k) hA[r * R + k] = r * 100.0 + k;
    CK(cudaMemcpy(A, hA, rows * ROWB, cudaMemcpyHostToDevice));
    free(hA);
  }
  bench<4, 4, true>(tm, idx, n, out, sms);
  bench<4, 4, false>(tm, idx, n, out, sms);
  bench<8, 4, true>(tm, idx, n, out, sms);
  bench<8, 4, false>(tm, idx, n, out, sms);
  bench<8, 6, true>(tm, idx, n, out, sms);
  bench<4, 8, true>(tm, idx, n, out, sms);
  bench<8, 8, false>(tm, idx, n, out, sms);
  return 0;
}
