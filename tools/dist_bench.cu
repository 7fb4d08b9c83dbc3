// Micro-benchmark of distance-pass kernel variants (H6) on synthetic data: p, m = 1M rows, 8 blocks x
// 2 starts.  Not part of the library; used to choose the k_dist_mma2 configuration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/dist_bench tools/dist_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// NS starts share the A fragments; CINIT: centring folded into the accumulators; else (z - mu) per element
template <int P, int MB, int NS, int MINB, bool CINIT>
__global__ void __launch_bounds__(256, MINB) kvar(const double* __restrict__ Zall, long long m, long long blk_stride,
                                                  const double* __restrict__ ops /* [inst][P + P(P+1)/2] */,
                                                  double* __restrict__ d2_all) {
  constexpr int KB = (P + 3) / 4, NB = (P + 7) / 8, CS = P + P * (P + 1) / 2;
  __shared__ double bsm[NS][KB * NB * 32];
  __shared__ double musm[NS][KB * 4];
  __shared__ double csm[NS][NB * 8];
  const int blk = blockIdx.y;  // block; starts NS*blk + u  (NS = 1: instance = blockIdx.y)
  const double* Z = Zall + (long long)(NS == 2 ? blk : blk / 2) * blk_stride;
  double* d2[NS];
  for (int u = 0; u < NS; u++) {
    const int id = NS * blk + u;
    const double* cs = ops + (long long)id * CS;
    d2[u] = d2_all + (long long)id * m;
    for (int e = threadIdx.x; e < KB * NB * 32; e += blockDim.x) {
      const int ln = e & 31, b = e >> 5, kb = b / NB, nb = b - kb * NB;
      const int k = 4 * kb + (ln & 3), j = 8 * nb + (ln >> 2);
      bsm[u][e] = (j < P && k <= j) ? cs[P + j * (j + 1) / 2 + k] : 0.0;
    }
    for (int e = threadIdx.x; e < KB * 4; e += blockDim.x) musm[u][e] = e < P ? cs[e] : 0.0;
    for (int j = threadIdx.x; j < NB * 8; j += blockDim.x) {
      double c = 0.0;
      if (j < P)
        for (int k = 0; k <= j; k++) c = fma(cs[P + j * (j + 1) / 2 + k], cs[k], c);
      csm[u][j] = -c;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const long long ntiles = (m + 8 * MB - 1) / (8 * MB);
  const long long warp0 = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  for (long long tile = warp0; tile < ntiles; tile += (long long)gridDim.x * 8) {
    const long long r0 = tile * 8 * MB;
    double acc[NS][MB][NB][2];
#pragma unroll
    for (int u = 0; u < NS; u++)
#pragma unroll
      for (int nb = 0; nb < NB; nb++)
#pragma unroll
        for (int mb = 0; mb < MB; mb++) {
          acc[u][mb][nb][0] = CINIT ? csm[u][8 * nb + 2 * t] : 0.0;
          acc[u][mb][nb][1] = CINIT ? csm[u][8 * nb + 2 * t + 1] : 0.0;
        }
#pragma unroll
    for (int kb = 0; kb < KB; kb++) {
      const int k = 4 * kb + t;
      double a[MB];
#pragma unroll
      for (int mb = 0; mb < MB; mb++) {
        const long long row = r0 + mb * 8 + g;
        a[mb] = (k < P && row < m) ? __ldg(Z + (long long)k * m + row) : 0.0;
      }
#pragma unroll
      for (int nb = 0; nb < NB; nb++) {
        if (8 * nb + 7 < 4 * kb) continue;
#pragma unroll
        for (int u = 0; u < NS; u++) {
          const double bv = bsm[u][(kb * NB + nb) * 32 + lane];
#pragma unroll
          for (int mb = 0; mb < MB; mb++) {
            const double av = CINIT ? a[mb] : (a[mb] != 0.0 || true ? a[mb] - (k < P ? musm[u][4 * kb + t] : 0.0) : 0.0);
            dmma(acc[u][mb][nb][0], acc[u][mb][nb][1], av, bv);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < NS; u++)
#pragma unroll
      for (int mb = 0; mb < MB; mb++) {
        double s = 0.0;
#pragma unroll
        for (int nb = 0; nb < NB; nb++) s = fma(acc[u][mb][nb][0], acc[u][mb][nb][0], fma(acc[u][mb][nb][1], acc[u][mb][nb][1], s));
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        const long long row = r0 + mb * 8 + g;
        if (t == 0 && row < m) d2[u][row] = s;
      }
  }
}

// staged variant: persistent grid (one CTA per SM), flattened (instance, tile) space, tiles of
// 8 * MB * 8 rows streamed through shared memory by cp.async NST deep, operator (B fragments) in
// registers, reloaded when the CTA's range crosses into the next instance
__device__ __forceinline__ void cpa8(double* d, const double* s) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(d)), "l"(s));
}
template <int P, int MB, int NST>
__global__ void __launch_bounds__(256, 1) kstaged(const double* __restrict__ Zall, long long m, long long blk_stride,
                                                  const double* __restrict__ ops, double* __restrict__ d2_all,
                                                  int ninst) {
  constexpr int KB = (P + 3) / 4, NB = (P + 7) / 8, CS = P + P * (P + 1) / 2;
  constexpr int TR = 8 * 8 * MB;   // rows per tile
  constexpr int LD = TR + 4;
  extern __shared__ double sm[];   // [NST][P][LD]
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, warp = threadIdx.x >> 5, tid = threadIdx.x;
  const long long tpi = (m + TR - 1) / TR, total = tpi * ninst;
  const long long t0 = total * blockIdx.x / gridDim.x, t1 = total * (blockIdx.x + 1) / gridDim.x;
  const int ntile = (int)(t1 - t0);
  auto issue = [&](int i) {
    if (i < ntile) {
      const long long tt = t0 + i;
      const int id = (int)(tt / tpi);
      const double* Z = Zall + (long long)(id / 2) * blk_stride;
      const long long row0 = (tt - (long long)id * tpi) * TR;
      const int rows = (int)min((long long)TR, m - row0);
      double* T = sm + (size_t)(i % NST) * P * LD;
      for (int e = tid; e < P * TR; e += 256) {
        const int k = e / TR, r = e - k * TR;
        if (r < rows) cpa8(T + k * LD + r, Z + (long long)k * m + row0 + r);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double bf[KB][NB], mu[KB];
  int cur = -1;
  for (int f = 0; f < NST - 1; f++) issue(f);
  for (int i = 0; i < ntile; i++) {
    issue(i + NST - 1);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NST - 1));
    __syncthreads();
    const long long tt = t0 + i;
    const int id = (int)(tt / tpi);
    if (id != cur) {
      const double* cs = ops + (long long)id * CS;
#pragma unroll
      for (int kb = 0; kb < KB; kb++) {
        const int k = 4 * kb + t;
        mu[kb] = k < P ? cs[k] : 0.0;
#pragma unroll
        for (int nb = 0; nb < NB; nb++) {
          const int j = 8 * nb + g;
          bf[kb][nb] = (j < P && k <= j) ? cs[P + j * (j + 1) / 2 + k] : 0.0;
        }
      }
      cur = id;
    }
    const long long row0 = (tt - (long long)id * tpi) * TR;
    const double* T = sm + (size_t)(i % NST) * P * LD;
    double acc[MB][NB][2];
#pragma unroll
    for (int mb = 0; mb < MB; mb++)
#pragma unroll
      for (int nb = 0; nb < NB; nb++) acc[mb][nb][0] = acc[mb][nb][1] = 0.0;
#pragma unroll
    for (int kb = 0; kb < KB; kb++) {
      const int k = 4 * kb + t;
      double a[MB];
#pragma unroll
      for (int mb = 0; mb < MB; mb++) a[mb] = k < P ? T[k * LD + (warp * MB + mb) * 8 + g] - mu[kb] : 0.0;
#pragma unroll
      for (int nb = 0; nb < NB; nb++) {
        if (8 * nb + 7 < 4 * kb) continue;
#pragma unroll
        for (int mb = 0; mb < MB; mb++) dmma(acc[mb][nb][0], acc[mb][nb][1], a[mb], bf[kb][nb]);
      }
    }
    double* d2 = d2_all + (long long)id * m;
#pragma unroll
    for (int mb = 0; mb < MB; mb++) {
      double s = 0.0;
#pragma unroll
      for (int nb = 0; nb < NB; nb++) s = fma(acc[mb][nb][0], acc[mb][nb][0], fma(acc[mb][nb][1], acc[mb][nb][1], s));
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      const long long row = row0 + (warp * MB + mb) * 8 + g;
      if (t == 0 && row < m) d2[row] = s;
    }
    __syncthreads();
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
}

template <int P, int MB, int NST>
float run_staged(const double* Z, long long m, long long bs, const double* ops, double* d2, int nblk, double bytes,
                 double flops) {
  constexpr int TR = 8 * 8 * MB, LD = TR + 4;
  const int smem = NST * P * LD * 8;
  cudaFuncSetAttribute(kstaged<P, MB, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; w++) kstaged<P, MB, NST><<<148, 256, smem>>>(Z, m, bs, ops, d2, 2 * nblk);
  cudaEventRecord(e0);
  const int R = 10;
  for (int r = 0; r < R; r++) kstaged<P, MB, NST><<<148, 256, smem>>>(Z, m, bs, ops, d2, 2 * nblk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= R;
  printf("%-34s P=%2d MB=%d NST=%d smem=%d: %.3f ms  eff %.0f GB/s  %.1f TF/s  %s\n", "staged persistent", P, MB, NST,
         smem, ms, bytes / ms / 1e6, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  return ms;
}

template <int P, int MB, int NS, int MINB, bool CINIT>
float run(const char* name, const double* Z, long long m, long long bs, const double* ops, double* d2, int nblk,
          double bytes, double flops) {
  const int items = NS == 2 ? nblk : 2 * nblk;
  const long long tiles = (m + 8 * MB - 1) / (8 * MB);
  long long gx = (tiles + 7) / 8;
  const long long cap = std::max<long long>(1, 148LL * MINB * 2 / items);
  if (gx > cap) gx = cap;
  dim3 grid((unsigned)gx, items);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; w++) kvar<P, MB, NS, MINB, CINIT><<<grid, 256>>>(Z, m, bs, ops, d2);
  cudaEventRecord(e0);
  const int R = 10;
  for (int r = 0; r < R; r++) kvar<P, MB, NS, MINB, CINIT><<<grid, 256>>>(Z, m, bs, ops, d2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= R;
  printf("%-34s P=%2d MB=%d NS=%d MINB=%d CINIT=%d grid=%lldx%d: %.3f ms  eff %.0f GB/s  %.1f TF/s  %s\n", name, P, MB,
         NS, MINB, (int)CINIT, gx, items, ms, bytes / ms / 1e6, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  return ms;
}

template <int P>
void suite(long long m, int nblk) {
  const long long bs = (long long)P * m;
  const int CS = P + P * (P + 1) / 2;
  double *Z, *ops, *d2;
  cudaMalloc(&Z, sizeof(double) * bs * nblk);
  cudaMalloc(&ops, sizeof(double) * CS * 2 * nblk);
  cudaMalloc(&d2, sizeof(double) * m * 2 * nblk);
  std::vector<double> h(bs * nblk);
  for (size_t i = 0; i < h.size(); i++) h[i] = ((i * 2654435761ull) % 1000003) / 500001.5 - 1.0;
  cudaMemcpy(Z, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  std::vector<double> o(CS * 2 * nblk);
  for (size_t i = 0; i < o.size(); i++) o[i] = ((i * 40503ull) % 1009) / 1009.0 - 0.3;
  cudaMemcpy(ops, o.data(), o.size() * 8, cudaMemcpyHostToDevice);
  const double inst = 2.0 * nblk;
  const double eff_bytes = inst * m * (8.0 * P + 8.0);
  const double flops = inst * m * ((double)P * (P + 1) + 2.0 * P);
  printf("--- P=%d m=%lld blocks=%d (effective bytes: 8(p+1) per row per start)\n", P, m, nblk);
  run<P, 3, 1, 2, false>("baseline (mu subtract, 1 start)", Z, m, bs, ops, d2, nblk, eff_bytes, flops);
  run<P, 3, 1, 2, true>("c-init, 1 start", Z, m, bs, ops, d2, nblk, eff_bytes, flops);
  run<P, 4, 1, 1, true>("c-init, 1 start, MB4 minb1", Z, m, bs, ops, d2, nblk, eff_bytes, flops);
  run<P, 2, 2, 2, true>("c-init, 2 starts MB2 minb2", Z, m, bs, ops, d2, nblk, eff_bytes, flops);
  run<P, 2, 2, 1, true>("c-init, 2 starts MB2 minb1", Z, m, bs, ops, d2, nblk, eff_bytes, flops);
  run<P, 3, 2, 1, true>("c-init, 2 starts MB3 minb1", Z, m, bs, ops, d2, nblk, eff_bytes, flops);
  run<P, 1, 2, 2, true>("c-init, 2 starts MB1 minb2", Z, m, bs, ops, d2, nblk, eff_bytes, flops);
  run_staged<P, 2, 3>(Z, m, bs, ops, d2, nblk, eff_bytes, flops);
  run_staged<P, 2, 4>(Z, m, bs, ops, d2, nblk, eff_bytes, flops);
  run_staged<P, 3, 3>(Z, m, bs, ops, d2, nblk, eff_bytes, flops);
  run_staged<P, 1, 4>(Z, m, bs, ops, d2, nblk, eff_bytes, flops);
  cudaFree(Z);
  cudaFree(ops);
  cudaFree(d2);
}

int main() {
  suite<40>(1000000, 8);
  suite<20>(1000000, 1);
  suite<10>(100000, 1);
  return 0;
}
