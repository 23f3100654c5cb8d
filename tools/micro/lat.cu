// Latency microbenchmarks (dependent chains, one warp): DFMA, DDIV, DSQRT,
// shfl, LDS.64.  Development tool.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, int n) {
  __shared__ double sm[64];
  sm[threadIdx.x] = a + threadIdx.x;
  __syncwarp();
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-9);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0000001 / x;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x);
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  long long t4 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < n; ++i) { x += sm[idx]; idx = ((int)x) & 31; }
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) x = x * 1.0000001;
  long long t6 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMallocManaged(&c, 64);
  for (int rep = 0; rep < 2; ++rep) { k<<<1, 32>>>(o, c, 1.5, 1000); cudaDeviceSynchronize(); }
  const char* nm[] = {"DFMA", "DDIV", "DSQRT", "SHFL", "LDS+cvt+add", "DMUL"};
  for (int i = 0; i < 6; ++i) printf("%s: %.1f cycles\n", nm[i], c[i] / 1000.0);
}
