// Dependent-chain latency of the fp64 special functions and __syncthreads on this B200 (DESIGN section 6,
// k_prepare row): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/t_fp64lat tools/t_fp64lat.cu
#include <cstdio>
__global__ void k(double* out, double x0, int which, long long* cyc) {
  double x = x0;
  long long t0 = clock64();
  for (int i = 0; i < 256; i++) {
    switch (which) {
      case 0: x = sqrt(x) + 1.5; break;
      case 1: x = 1.0 / x + 1.5; break;
      case 2: x = rsqrt(x) + 1.5; break;
      case 3: x = log(x) + 2.5; break;
      case 4: x = fma(x, 0.999, 0.5); break;
      case 5: x = x / (x + 0.25); x += 1.5; break;
      case 6: x = exp(-x) + 1.5; break;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void kbar(long long* cyc, int n) {
  __shared__ double s[1024];
  long long t0 = clock64();
  for (int i = 0; i < n; i++) { s[threadIdx.x] += 1.0; __syncthreads(); }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8192); cudaMalloc(&c, 8);
  const char* nm[] = {"sqrt", "rcp", "rsqrt", "log", "fma", "div", "exp"};
  for (int w = 0; w < 7; w++) {
    long long h;
    k<<<1, 32>>>(o, 2.0, w, c); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, 2.0, w, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-6s %.1f cycles per dependent op\n", nm[w], h / 256.0);
  }
  for (int th : {128, 512, 1024}) {
    long long h;
    kbar<<<1, th>>>(c, 1000); cudaDeviceSynchronize();
    kbar<<<1, th>>>(c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("syncthreads (%d threads): %.1f cycles\n", th, h / 1000.0);
  }
  return 0;
}
