// Microbenchmark: FP64 DFMA and DMMA (mma.sync m8n8k4 f64) throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; i++) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += x[i];
  if (s == 12345.678) out[0] = s;
}
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
int main2();
int main() {
  main2();
  double* o;
  cudaMalloc(&o, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; rep++) {
    int iters = 20000, blocks = sms * 8, threads = 256;
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(o, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)blocks * threads;
    printf("DFMA: %.2f TFLOP/s (%.2f ms)\n", flops / ms / 1e9, ms);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 256 * 8 * iters * (double)blocks * (threads / 32);
    printf("DMMA m8n8k4: %.2f TFLOP/s (%.2f ms) %s\n", flops / ms / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
// mixed: each warp issues both DMMA and DFMA streams
__global__ void mixed_kernel(double* out, int iters, double a2, double b2) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
  double x[8];
#pragma unroll
  for (int i = 0; i < 4; i++) c[i][0] = c[i][1] = 0.0;
#pragma unroll
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
      x[2 * i] = fma(x[2 * i], a2, b2);
      x[2 * i + 1] = fma(x[2 * i + 1], a2, b2);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.678) out[0] = s;
}
int main2() {
  double* o;
  cudaMalloc(&o, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; rep++) {
    int iters = 20000, blocks = sms * 8, threads = 256;
    cudaEventRecord(e0);
    mixed_kernel<<<blocks, threads>>>(o, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl_mma = 2.0 * 256 * 4 * iters * (double)blocks * (threads / 32);
    double fl_fma = 2.0 * 8 * iters * (double)blocks * threads;
    printf("mixed: %.2f TFLOP/s total (mma %.2f + fma %.2f) (%.2f ms)\n", (fl_mma + fl_fma) / ms / 1e9,
           fl_mma / ms / 1e9, fl_fma / ms / 1e9, ms);
  }
  return 0;
}
