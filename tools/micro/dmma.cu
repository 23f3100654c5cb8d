// FP64 tensor-core issue microbenchmark: register-only chains of
// mma.sync f64 at the shapes PTX offers (m8n8k4; m16n8k4/k8/k16 on sm_90+),
// to find the shape that reaches the FP64 peak on sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma dmma.cu && ./dmma
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k884(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double d[CH][2];
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = 0;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.0) out[0] = s;
}

template <int CH>
__global__ void k1684(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + blockIdx.x * 1e-6;
  double d[CH][4];
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = 0;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3]) : "d"(a0), "d"(a1), "d"(b));
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 12345.0) out[0] = s;
}

template <int CH>
__global__ void k1688(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 1.0 + blockIdx.x * 1e-6, b1 = b0 + 1;
  double d[CH][4];
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = 0;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 12345.0) out[0] = s;
}

template <int CH>
__global__ void k16816(double* out, int iters) {
  double a[8], b[4];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int k = 0; k < 4; ++k) b[k] = 1.0 + blockIdx.x * 1e-6 + k;
  double d[CH][4];
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = 0;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 12345.0) out[0] = s;
}

__global__ void kdfma(double* out, int iters) {
  double x[8];
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3 + c;
  const double m = 1.0000001, a = 1e-9;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], m, a);
  double s = 0;
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 12345.0) out[0] = s;
}

template <int CH, int NF>
__global__ void kmix(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double d[CH][2], x[NF];
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = 0;
  for (int c = 0; c < NF; ++c) x[c] = threadIdx.x * 1e-3 + c;
  const double m = 1.0000001, ad = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int c = 0; c < NF; ++c) x[c] = fma(x[c], m, ad);
  }
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  for (int c = 0; c < NF; ++c) s += x[c];
  if (s == 12345.0) out[0] = s;
}

template <typename K>
void run(const char* name, K kern, int threads, double flop_per_iter_per_warp, int iters) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  for (int per_sm : {1, 2, 4, 8}) {
    const int blocks = sms * per_sm;
    kern<<<blocks, threads>>>(out, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = flop_per_iter_per_warp * iters * (threads / 32) * (double)blocks;
    printf("%-22s blocks/SM %d threads %d: %.2f TFLOP/s\n", name, per_sm, threads, fl / ms / 1e9);
  }
  cudaFree(out);
}

int main() {
  const int it = 4096;
  run("m8n8k4 x4", k884<4>, 256, 4 * 2.0 * 8 * 8 * 4, it);
  run("m8n8k4 x8", k884<8>, 256, 8 * 2.0 * 8 * 8 * 4, it);
  run("m16n8k4 x4", k1684<4>, 256, 4 * 2.0 * 16 * 8 * 4, it);
  run("m16n8k8 x4", k1688<4>, 256, 4 * 2.0 * 16 * 8 * 8, it);
  run("m16n8k16 x4", k16816<4>, 256, 4 * 2.0 * 16 * 8 * 16, it / 2);
  run("dfma x8", kdfma, 256, 8 * 2.0 * 32, it);
  run("mix 4 dmma + 8 dfma", kmix<4, 8>, 256, 4 * 2.0 * 256 + 8 * 2.0 * 32, it);
  run("mix 4 dmma + 16 dfma", kmix<4, 16>, 256, 4 * 2.0 * 256 + 16 * 2.0 * 32, it);
  run("mix 4 dmma + 32 dfma", kmix<4, 32>, 256, 4 * 2.0 * 256 + 32 * 2.0 * 32, it);
  return 0;
}
