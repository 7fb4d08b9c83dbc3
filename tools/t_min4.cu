#include <cstdio>
#include <cuda_runtime.h>
static constexpr int LD = 41;
// variant: flat arrays, no early return inside the loop
__device__ __noinline__ bool chol_flat(const double* A, double* L, int p, int* s_fail) {
  const int t = threadIdx.x;
  if (t == 0) *s_fail = 0;
  for (int e = t; e < 40 * LD; e += blockDim.x) L[e] = 0.0;
  __syncthreads();
  bool ok = true;
  for (int j = 0; j < p; j++) {
    if (t == 0) {
      double s = A[j * LD + j];
      for (int k = 0; k < j; k++) s -= L[j * LD + k] * L[j * LD + k];
      if (!(s > 0.0)) *s_fail = 1;
      L[j * LD + j] = s > 0.0 ? sqrt(s) : 1.0;
    }
    __syncthreads();
    if (*s_fail) { ok = false; break; }
    for (int i = j + 1 + t; i < p; i += blockDim.x) {
      double s = A[i * LD + j];
      for (int k = 0; k < j; k++) s -= L[i * LD + k] * L[j * LD + k];
      L[i * LD + j] = s / L[j * LD + j];
    }
    __syncthreads();
  }
  return ok;
}
__global__ void kmin(const double* sg, int p, double* outL) {
  __shared__ double A[40 * LD], L[40 * LD];
  __shared__ int s_fail;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) A[(e / p) * LD + e % p] = sg[e];
  __syncthreads();
  bool ok = chol_flat(A, L, p, &s_fail);
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) outL[e] = L[(e / p) * LD + e % p];
  if (threadIdx.x == 0) outL[25] = ok;
}
int main() {
  double h[26], *d, *o;
  for (int e = 0; e < 25; e++) h[e] = (e % 6 == 0) ? 4.0 : (e % 5 < e / 5 || e / 5 < e % 5 ? 1.0 : 0.0);
  cudaMalloc(&d, 200); cudaMalloc(&o, 208);
  cudaMemcpy(d, h, 200, cudaMemcpyHostToDevice);
  kmin<<<1, 256>>>(d, 5, o);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(h, o, 208, cudaMemcpyDeviceToHost);
  for (int i = 0; i < 5; i++) printf("  %.6f %.6f %.6f %.6f %.6f\n", h[i*5], h[i*5+1], h[i*5+2], h[i*5+3], h[i*5+4]);
  printf("ok %g\n", h[25]);
}
