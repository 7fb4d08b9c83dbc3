#include <cstdio>
#include <cuda_runtime.h>
static constexpr int LD = 41;
__device__ __forceinline__ bool chol(const double (*A)[LD], double (*L)[LD], int p, int* s_fail) {
  const int t = threadIdx.x;
  if (t == 0) *s_fail = 0;
  for (int e = t; e < 40 * LD; e += blockDim.x) (&L[0][0])[e] = 0.0;
  __syncthreads();
  for (int j = 0; j < p; j++) {
    if (t == 0) {
      double s = A[j][j];
      for (int k = 0; k < j; k++) s -= L[j][k] * L[j][k];
      if (!(s > 0.0)) *s_fail = 1;
      L[j][j] = s > 0.0 ? sqrt(s) : 1.0;
    }
    __syncthreads();
    if (*s_fail) return false;
    for (int i = j + 1 + t; i < p; i += blockDim.x) {
      double s = A[i][j];
      for (int k = 0; k < j; k++) s -= L[i][k] * L[j][k];
      L[i][j] = s / L[j][j];
    }
    __syncthreads();
  }
  return true;
}
template <int V>
__global__ void kmin(const double* sg, int p, double* outL) {
  if (V == 0) {
    __shared__ double A[40][LD], L[40][LD];
    __shared__ int s_fail;
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) A[e / p][e % p] = sg[e];
    __syncthreads();
    bool ok = chol(A, L, p, &s_fail);
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) outL[e] = L[e / p][e % p];
    if (threadIdx.x == 0) outL[25] = ok;
  } else if (V == 1) {
    __shared__ __align__(16) double A[40][LD];
    __shared__ __align__(16) double L[40][LD];
    __shared__ __align__(16) int s_fail;
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) A[e / p][e % p] = sg[e];
    __syncthreads();
    bool ok = chol(A, L, p, &s_fail);
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) outL[e] = L[e / p][e % p];
    if (threadIdx.x == 0) outL[25] = ok;
  } else if (V == 2) {
    __shared__ double A[40][LD];
    __shared__ double L[40][LD];
    __shared__ int s_fail;
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) A[e / p][e % p] = sg[e];
    __syncthreads();
    bool ok = chol(A, L, p, &s_fail);
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) outL[e] = L[e / p][e % p];
    if (threadIdx.x == 0) outL[25] = ok;
  } else {
    __shared__ double A[40][LD], L[40][LD];
    __shared__ int s_fail;
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) A[e / p][e % p] = sg[e];
    __syncthreads();
    bool ok = chol(A, L, p, &s_fail);
    __syncthreads();
    if (threadIdx.x == 0) for (int e = 0; e < 25; e++) outL[e] = L[e / p][e % p];
    if (threadIdx.x == 0) outL[25] = ok;
  }
}
template <int V> void run(const char* name, double* d, double* o) {
  kmin<V><<<1, 256>>>(d, 5, o);
  double h[26];
  printf("%s: %s\n", name, cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(h, o, 208, cudaMemcpyDeviceToHost);
  for (int i = 0; i < 5; i++) printf("  %g %g %g %g %g\n", h[i*5], h[i*5+1], h[i*5+2], h[i*5+3], h[i*5+4]);
}
int main() {
  double h[25], *d, *o;
  for (int e = 0; e < 25; e++) h[e] = (e % 6 == 0) ? 4.0 : 0.0;
  cudaMalloc(&d, 200); cudaMalloc(&o, 208);
  cudaMemcpy(d, h, 200, cudaMemcpyHostToDevice);
  run<0>("orig", d, o); 
}
