// fp64 peak microbenchmark: DFMA (CUDA cores) vs DMMA (mma.sync f64 tensor
// cores) on one B200.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma884_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  double c[4][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.0) out[0] = s;
}

#ifdef WITH_M16
__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + i * 1e-3;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 0.5 + i * 1e-3;
  double c[2][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]),
                     "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 2; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 12345.0) out[0] = s;
}
#endif

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    dim3 g(sms * 8), b(256);
    cudaEventRecord(e0);
    dfma_kernel<<<g, b>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)g.x * b.x;
    printf("DFMA        %.2f TFLOP/s\n", flops / ms / 1e9);
    cudaEventRecord(e0);
    dmma884_kernel<<<g, b>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 256 * 4 * iters * (double)g.x * (b.x / 32);
    printf("DMMA m8n8k4 %.2f TFLOP/s\n", flops / ms / 1e9);
#ifdef WITH_M16
    cudaEventRecord(e0);
    dmma16816_kernel<<<g, b>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * 8 * 16 * 2 * iters * (double)g.x * (b.x / 32);
    printf("DMMA m16n8k16 %.2f TFLOP/s\n", flops / ms / 1e9);
#endif
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
