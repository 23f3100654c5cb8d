// Microbenchmark: random gathers of 160-byte rows (a 2e5 x 20 f64 factor,
// L2-resident) -- the access pattern of the fitness kernel K7 -- through
//   (a) cp.async.bulk (TMA unit, one bulk copy per row) into shared memory,
//   (b) LDG.128 with 10 lanes per row (3 rows per warp instruction),
//   (c) LDG.64 with 4 lanes per row as DMMA A-fragments (K7's current way).
// Reports rows/s and GB/s of useful row bytes.  Development tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather gather.cu && ./gather
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int R = 20;
constexpr int ROWB = R * 8;
constexpr int WARPS = 8;
constexpr int BATCH = 32;  // rows per warp batch

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(WARPS * 32) k_tma(const double* __restrict__ A, const int* __restrict__ idx,
                                                  int64_t n, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* buf = sm + (size_t)wid * 2 * BATCH * ROWB;
  __shared__ __align__(8) uint64_t bar[WARPS][2];
  if (lane == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[wid][b])));
  }
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  const int64_t gw = blockIdx.x * (int64_t)WARPS + wid;
  const int64_t tw = (int64_t)gridDim.x * WARPS;
  const int64_t nb = n / BATCH;
  double acc = 0.0;
  uint32_t phase[2] = {0, 0};
  auto issue = [&](int64_t b, int slot) {
    const uint32_t mb = smem_u32(&bar[wid][slot]);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(BATCH * ROWB));
    __syncwarp();
    const int r = idx[b * BATCH + lane];
    const double* src = A + (int64_t)r * R;
    const uint32_t dst = smem_u32(buf + (size_t)slot * BATCH * ROWB + lane * ROWB);
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(ROWB), "r"(mb) : "memory");
  };
  int64_t b = gw;
  if (b < nb) issue(b, 0);
  int slot = 0;
  for (; b < nb; b += tw) {
    if (b + tw < nb) issue(b + tw, slot ^ 1);
    const uint32_t mb = smem_u32(&bar[wid][slot]);
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(mb), "r"(phase[slot]));
    phase[slot] ^= 1;
    const double* rows = reinterpret_cast<const double*>(buf + (size_t)slot * BATCH * ROWB);
    for (int e = lane; e < BATCH * R; e += 32) acc += rows[e];
    __syncwarp();
    slot ^= 1;
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void __launch_bounds__(256) k_ldg10(const double* __restrict__ A, const int* __restrict__ idx,
                                               int64_t n, double* out) {
  // 10 lanes per row, 3 rows per instruction (lanes 30, 31 idle)
  const int lane = threadIdx.x & 31, grp = lane / 10, ch = lane % 10;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t tw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int64_t base = gw * 12; base + 12 <= n; base += tw * 12) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t e = base + u * 3 + (grp < 3 ? grp : 2);
      const double2* row = reinterpret_cast<const double2*>(A + (int64_t)idx[e] * R);
      v[u] = grp < 3 ? __ldg(row + ch) : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y;
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void __launch_bounds__(256) k_ldg4(const double* __restrict__ A, const int* __restrict__ idx,
                                              int64_t n, double* out) {
  // K7 today: 8 rows per instruction, lane (q, c) loads k = 4 ks + c (5 LDG.64)
  const int lane = threadIdx.x & 31, q = lane >> 2, c = lane & 3;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t tw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int64_t base = gw * 16; base + 16 <= n; base += tw * 16) {
    double a[2][5];
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const double* row = A + (int64_t)idx[base + g * 8 + q] * R;
#pragma unroll
      for (int ks = 0; ks < 5; ++ks) a[g][ks] = __ldg(row + ks * 4 + c);
    }
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
      for (int ks = 0; ks < 5; ++ks) acc += a[g][ks];
  }
  if (acc == 12345.678) out[0] = acc;
}


__global__ void __launch_bounds__(256) k_ldgf16(const double* __restrict__ A, const int* __restrict__ idx,
                                                int64_t n, double* out) {
  // register fragments for the K7 dot, 16-byte loads: lane (q, c) of a group of
  // 8 rows loads cols {2c, 2c+1} and {8+2c, 9+2c} of row q plus cols 16..19
  // (the same 32 bytes for the 4 lanes of a quad)
  const int lane = threadIdx.x & 31, q = lane >> 2, c = lane & 3;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t tw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int64_t base = gw * 16; base + 16 <= n; base += tw * 16) {
    double2 v[2][4];
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const double2* row = reinterpret_cast<const double2*>(A + (int64_t)idx[base + g * 8 + q] * R);
      v[g][0] = __ldg(row + c);
      v[g][1] = __ldg(row + 4 + c);
      v[g][2] = __ldg(row + 8);
      v[g][3] = __ldg(row + 9);
    }
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += v[g][u].x + v[g][u].y;
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void __launch_bounds__(256) k_ldgf16b(const double* __restrict__ A, const int* __restrict__ idx,
                                                 int64_t n, double* out) {
  // as k_ldgf16 but cols 16..19 one per lane (LDG.64): 2 LDG.128 + 1 LDG.64
  const int lane = threadIdx.x & 31, q = lane >> 2, c = lane & 3;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t tw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int64_t base = gw * 16; base + 16 <= n; base += tw * 16) {
    double2 v[2][2];
    double t[2];
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const double* rp = A + (int64_t)idx[base + g * 8 + q] * R;
      const double2* row = reinterpret_cast<const double2*>(rp);
      v[g][0] = __ldg(row + c);
      v[g][1] = __ldg(row + 4 + c);
      t[g] = __ldg(rp + 16 + c);
    }
#pragma unroll
    for (int g = 0; g < 2; ++g) acc += v[g][0].x + v[g][0].y + v[g][1].x + v[g][1].y + t[g];
  }
  if (acc == 12345.678) out[0] = acc;
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
  const size_t smem = (size_t)WARPS * 2 * BATCH * ROWB;
  CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int which = 0; which < 5; ++which) {
    for (int ctas_per_sm = 1; ctas_per_sm <= 4; ctas_per_sm *= 2) {
      const int grid = sms * ctas_per_sm * (which == 0 ? 1 : 4);
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (which == 0) k_tma<<<grid, WARPS * 32, smem>>>(A, idx, n, out);
        else if (which == 1) k_ldg10<<<grid, 256>>>(A, idx, n, out);
        else if (which == 2) k_ldg4<<<grid, 256>>>(A, idx, n, out);
        else if (which == 3) k_ldgf16<<<grid, 256>>>(A, idx, n, out);
        else k_ldgf16b<<<grid, 256>>>(A, idx, n, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2)
          printf("%-8s grid %6d: %.3f ms  %.2f Grows/s  %.2f TB/s rows\n",
                 which == 0 ? "tma" : which == 1 ? "ldg10" : which == 2 ? "ldg4(K7)" : which == 3 ? "ldgf16" : "ldgf16b", grid, ms, n / ms / 1e6,
                 n * (double)ROWB / ms / 1e9);
      }
    }
  }
  return 0;
}
