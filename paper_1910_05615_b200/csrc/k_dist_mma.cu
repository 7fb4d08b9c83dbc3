// H6 on the FP64 tensor pipe: the C-step distance pass as a small dense
// contraction Y = (Z - mu) M^T with DMMA (mma.sync m8n8k4 f64), then
// d_i^2 = ||Y_i||^2 (§3.4).
//
// Measured on this B200 (tools/fp64_peak.cu): DMMA 37.0 TF/s vs DFMA 33.6 TF/s,
// and the two share one FP64 pipe.  At p = 40 the pass needs 5.4 flop per byte
// of X, at the FP64 ridge, so instruction issue decides: one DMMA does 256 FMA
// where a DFMA does 32, and the operator M = L^-1 (lower triangular) lives in
// registers as B fragments for the whole kernel.  Blocks of M^T that are
// entirely above the diagonal are skipped (20 of 50 8x4 blocks at p = 40; 30 are executed).
//
// Fragment layout of m8n8k4 f64 (g = lane >> 2, t = lane & 3):
//   A (8 x 4, rows x k):  A[g][t]          -> (Z - mu)[row0 + g][4 kb + t]
//   B (4 x 8, k x n):     B[t][g]          -> M[8 nb + g][4 kb + t]
//   C (8 x 8):            C[g][2t], C[g][2t+1]
#include "rtd_internal.h"

namespace rtd {

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// MINB CTAs per SM (register budget); CINIT folds the centring into the accumulators (d = M z - M mu,
// the same arithmetic object) instead of subtracting mu from every A element.  tools/dist_bench.cu
// compared the variants on a B200 (profiles/r01_dist_bench.txt): at p = 40 the pass is DMMA-bound
// (0.70 of the measured DMMA peak) and neither CINIT, 4 m-blocks at 1 CTA/SM, nor one pass shared by
// the two starts of a block (loads once, two operators) is faster; in the pipeline (config 3) the
// p = 20 winner of the isolated test was not, so every p uses MB 4 (p <= 24) / 3, 2 CTAs/SM, subtract.
// Each start has its own pass; the L2 serves the second start's reads of a block when both run.
template <int P, int MB, int MINB, bool CINIT>
__global__ void __launch_bounds__(256, MINB) k_dist_mma(const double* __restrict__ Zall, long long m,
                                                        long long blk_stride, const int* __restrict__ inst, int nstart,
                                                        const double* __restrict__ cstage, int cstride,
                                                        double* __restrict__ d2_all) {
  constexpr int KB = (P + 3) / 4;
  constexpr int NB = (P + 7) / 8;
  // operator fragments in shared memory: lane-major, conflict-free; each is reused by MB m-blocks
  __shared__ double bsm[KB * NB * 32];
  __shared__ double musm[KB * 4];
  __shared__ double csm[NB * 8];
  const int slot = blockIdx.y;
  const int id = inst[slot];
  const double* __restrict__ Z = Zall + (long long)(id / nstart) * blk_stride;
  double* __restrict__ d2 = d2_all + (long long)id * m;
  const double* __restrict__ cs = cstage + (long long)slot * cstride;
  for (int e = threadIdx.x; e < KB * NB * 32; e += blockDim.x) {
    const int ln = e & 31, blk = e >> 5, kb = blk / NB, nb = blk - kb * NB;
    const int k = 4 * kb + (ln & 3), j = 8 * nb + (ln >> 2);
    bsm[e] = (j < P && k <= j) ? cs[P + j * (j + 1) / 2 + k] : 0.0;
  }
  for (int e = threadIdx.x; e < KB * 4; e += blockDim.x) musm[e] = e < P ? cs[e] : 0.0;
  if (CINIT) {
    for (int j = threadIdx.x; j < NB * 8; j += blockDim.x) {  // c_j = (M mu)_j, fixed order
      double c = 0.0;
      if (j < P)
        for (int k = 0; k <= j; k++) c = fma(cs[P + j * (j + 1) / 2 + k], cs[k], c);
      csm[j] = -c;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const long long rows_per_tile = 8 * MB;
  const long long ntiles = (m + rows_per_tile - 1) / rows_per_tile;
  const long long warp0 = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long tile = warp0; tile < ntiles; tile += nwarps) {
    const long long r0 = tile * rows_per_tile;
    double acc[MB][NB][2];
#pragma unroll
    for (int mb = 0; mb < MB; mb++)
#pragma unroll
      for (int nb = 0; nb < NB; nb++) {
        acc[mb][nb][0] = CINIT ? csm[8 * nb + 2 * t] : 0.0;
        acc[mb][nb][1] = CINIT ? csm[8 * nb + 2 * t + 1] : 0.0;
      }
#pragma unroll
    for (int kb = 0; kb < KB; kb++) {
      const int k = 4 * kb + t;
      const double muk = musm[4 * kb + t];
      double a[MB];
#pragma unroll
      for (int mb = 0; mb < MB; mb++) {
        const long long row = r0 + mb * 8 + g;
        a[mb] = (k < P && row < m) ? (CINIT ? __ldg(Z + (long long)k * m + row)
                                            : __dsub_rn(__ldg(Z + (long long)k * m + row), muk)) : 0.0;
      }
#pragma unroll
      for (int nb = 0; nb < NB; nb++) {
        if (8 * nb + 7 < 4 * kb) continue;  // block entirely above the diagonal of M
        const double bv = bsm[(kb * NB + nb) * 32 + lane];
#pragma unroll
        for (int mb = 0; mb < MB; mb++) dmma_8x8x4(acc[mb][nb][0], acc[mb][nb][1], a[mb], bv);
      }
    }
#pragma unroll
    for (int mb = 0; mb < MB; mb++) {
      double s = 0.0;
#pragma unroll
      for (int nb = 0; nb < NB; nb++) {
        s = fma(acc[mb][nb][0], acc[mb][nb][0], s);
        s = fma(acc[mb][nb][1], acc[mb][nb][1], s);
      }
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      const long long row = r0 + mb * 8 + g;
      if (t == 0 && row < m) d2[row] = s;
    }
  }
}

// Variant I of the paper's Table 1 ("D" switched off): the distance by the
// explicit inverse, d_i^2 = u_i^T Sigma^-1 u_i with u_i = z_i - mu, as y = Sigma^-1 u on DMMA (the full
// p x p operator: no block is skipped) followed by the dot product u . y (u re-read, L1-resident).
// The operator of slot s is [mu (P) | Sigma^-1 row-major (P*P)] at cstage + s * cstride.
template <int P, int MB>
__global__ void __launch_bounds__(256, 2) k_dist_inv(const double* __restrict__ Zall, long long m, long long blk_stride,
                                                     const int* __restrict__ inst, int nstart,
                                                     const double* __restrict__ cstage, int cstride,
                                                     double* __restrict__ d2_all) {
  constexpr int KB = (P + 3) / 4;
  constexpr int NB = (P + 7) / 8;
  __shared__ double bsm[KB * NB * 32];
  __shared__ double musm[NB * 8];
  const int slot = blockIdx.y;
  const int id = inst[slot];
  const double* __restrict__ Z = Zall + (long long)(id / nstart) * blk_stride;
  double* __restrict__ d2 = d2_all + (long long)id * m;
  const double* __restrict__ cs = cstage + (long long)slot * cstride;
  for (int e = threadIdx.x; e < KB * NB * 32; e += blockDim.x) {
    const int ln = e & 31, blk = e >> 5, kb = blk / NB, nb = blk - kb * NB;
    const int k = 4 * kb + (ln & 3), j = 8 * nb + (ln >> 2);
    bsm[e] = (j < P && k < P) ? cs[P + j * P + k] : 0.0;  // B[k][j] = Sigma^-1[j][k] (symmetric)
  }
  for (int e = threadIdx.x; e < NB * 8; e += blockDim.x) musm[e] = e < P ? cs[e] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const long long rows_per_tile = 8 * MB;
  const long long ntiles = (m + rows_per_tile - 1) / rows_per_tile;
  const long long warp0 = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long tile = warp0; tile < ntiles; tile += nwarps) {
    const long long r0 = tile * rows_per_tile;
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
      for (int mb = 0; mb < MB; mb++) {
        const long long row = r0 + mb * 8 + g;
        a[mb] = (k < P && row < m) ? __dsub_rn(__ldg(Z + (long long)k * m + row), musm[k]) : 0.0;
      }
#pragma unroll
      for (int nb = 0; nb < NB; nb++) {
        const double bv = bsm[(kb * NB + nb) * 32 + lane];
#pragma unroll
        for (int mb = 0; mb < MB; mb++) dmma_8x8x4(acc[mb][nb][0], acc[mb][nb][1], a[mb], bv);
      }
    }
#pragma unroll
    for (int mb = 0; mb < MB; mb++) {
      const long long row = r0 + mb * 8 + g;
      double s = 0.0;
      if (row < m) {
#pragma unroll
        for (int nb = 0; nb < NB; nb++) {
          const int j = 8 * nb + 2 * t;
          if (j < P) s = fma(__dsub_rn(__ldg(Z + (long long)j * m + row), musm[j]), acc[mb][nb][0], s);
          if (j + 1 < P) s = fma(__dsub_rn(__ldg(Z + (long long)(j + 1) * m + row), musm[j + 1]), acc[mb][nb][1], s);
        }
      }
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      // a full quadratic form can round (or, under a drifted SMW inverse, fall) below zero; the select's
      // keys take the IEEE bits of d^2 >= 0, so clamp (this also maps -0.0 to +0.0)
      if (t == 0 && row < m) d2[row] = fmax(s, 0.0);
    }
  }
}

template <int P>
static void dist_inv_launch(const double* Zall, long long m, long long blk_stride, const int* inst, int nstart,
                            int ninst, const double* cstage, int cstride, double* d2_all, cudaStream_t st) {
  constexpr int MB = P <= 24 ? 4 : 2;
  const long long tiles = (m + 8 * MB - 1) / (8 * MB);
  const long long need = (tiles + 7) / 8;
  const long long cap = std::max<long long>(1, 148LL * 2 * 2 / std::max(1, ninst));
  k_dist_inv<P, MB><<<dim3((unsigned)std::min(need, cap), ninst), 256, 0, st>>>(Zall, m, blk_stride, inst, nstart,
                                                                                 cstage, cstride, d2_all);
}

template <int P>
static void dist_mma_launch(const double* Zall, long long m, long long blk_stride, const int* inst, int nstart,
                            int ninst, const double* cstage, int cstride, double* d2_all, cudaStream_t st) {
  constexpr int MB = P <= 24 ? 4 : 3, MINB = 2;
  constexpr bool SMALL = false;
  const long long tiles = (m + 8 * MB - 1) / (8 * MB);
  const long long need = (tiles + 7) / 8;  // 8 warps per CTA
  const long long cap = std::max<long long>(1, 148LL * MINB * 2 / std::max(1, ninst));
  k_dist_mma<P, MB, MINB, SMALL><<<dim3((unsigned)std::min(need, cap), ninst), 256, 0, st>>>(
      Zall, m, blk_stride, inst, nstart, cstage, cstride, d2_all);
}

// H12 flagging pass on DMMA for row-major X: d_i^2 = ||M (x_i - mu)||^2, flags_i = d_i^2 > c2.  Each warp
// streams its own tiles of 8 MB consecutive rows (contiguous in row-major X) into shared memory by
// cp.async, two tiles per warp in flight (the next one copies while the current one is contracted), row
// stride P + 1 so the A-fragment reads (8 rows x 4 columns per lane group) are conflict-free.  The
// operator [mu | M packed lower] is read from the staged buffer cs.
template <int P, int MB>
__global__ void __launch_bounds__(256, 4) k_flag_mma(const double* __restrict__ X, long long n, int log_transform,
                                                     const double* __restrict__ cs, double c2,
                                                     uint8_t* __restrict__ flags, double* __restrict__ rd2) {
  constexpr int KB = (P + 3) / 4, NB = (P + 7) / 8, S = P + 1, TR = 8 * MB, TE = TR * P;
  __shared__ double bsm[KB * NB * 32];
  __shared__ double musm[KB * 4];
  extern __shared__ double xt[];  // [warp][2][TR * S]
  for (int e = threadIdx.x; e < KB * NB * 32; e += blockDim.x) {
    const int ln = e & 31, blk = e >> 5, kb = blk / NB, nb = blk - kb * NB;
    const int k = 4 * kb + (ln & 3), j = 8 * nb + (ln >> 2);
    bsm[e] = (j < P && k <= j) ? cs[P + j * (j + 1) / 2 + k] : 0.0;
  }
  for (int e = threadIdx.x; e < KB * 4; e += blockDim.x) musm[e] = e < P ? cs[e] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, w = threadIdx.x >> 5;
  double* wbuf = xt + (size_t)w * 2 * TR * S;
  const long long ntiles = (n + TR - 1) / TR;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  auto issue = [&](long long tile, int buf) {
    if (tile < ntiles) {
      const long long r0 = tile * TR;
      const int cnt = (int)min((long long)TR, n - r0) * P;
      double* dst = wbuf + buf * TR * S;
      const double* src = X + r0 * P;
      for (int e = lane; e < cnt; e += 32) {
        const int r = e / P, k = e - r * P;
        cp_async8(dst + r * S + k, src + e);
      }
    }
    cp_async_commit();
  };
  long long tile = (long long)blockIdx.x * (blockDim.x >> 5) + w;
  issue(tile, 0);
  for (int it = 0; tile < ntiles; tile += nw, it++) {
    issue(tile + nw, (it + 1) & 1);
    cp_async_wait<1>();
    __syncwarp();
    const double* T = wbuf + (it & 1) * TR * S;
    const long long r0 = tile * TR;
    const int rows = (int)min((long long)TR, n - r0);
    double acc[MB][NB][2];
#pragma unroll
    for (int mb = 0; mb < MB; mb++)
#pragma unroll
      for (int nb = 0; nb < NB; nb++) acc[mb][nb][0] = acc[mb][nb][1] = 0.0;
#pragma unroll
    for (int kb = 0; kb < KB; kb++) {
      const int k = 4 * kb + t;
      const double muk = musm[4 * kb + t];
      double a[MB];
#pragma unroll
      for (int mb = 0; mb < MB; mb++) {
        const int r = mb * 8 + g;
        double v = 0.0;
        if (k < P && r < rows) {
          v = T[r * S + k];
          if (log_transform) v = log(v);
          v = __dsub_rn(v, muk);
        }
        a[mb] = v;
      }
#pragma unroll
      for (int nb = 0; nb < NB; nb++) {
        if (8 * nb + 7 < 4 * kb) continue;  // block entirely above the diagonal of M
        const double bv = bsm[(kb * NB + nb) * 32 + lane];
#pragma unroll
        for (int mb = 0; mb < MB; mb++) dmma_8x8x4(acc[mb][nb][0], acc[mb][nb][1], a[mb], bv);
      }
    }
#pragma unroll
    for (int mb = 0; mb < MB; mb++) {
      double s = 0.0;
#pragma unroll
      for (int nb = 0; nb < NB; nb++) {
        s = fma(acc[mb][nb][0], acc[mb][nb][0], s);
        s = fma(acc[mb][nb][1], acc[mb][nb][1], s);
      }
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      const int r = mb * 8 + g;
      if (t == 0 && r < rows) {
        if (flags) flags[r0 + r] = s > c2 ? 1 : 0;
        if (rd2) rd2[r0 + r] = s;
      }
    }
    __syncwarp();  // the buffer just read is refilled by the next issue
  }
  cp_async_wait<0>();
}

template <int P>
static void flag_mma_launch(const double* X, long long n, int log_transform, const double* cs, double c2,
                            uint8_t* flags, double* rd2, cudaStream_t st) {
  constexpr int MB = 1, S = P + 1, TR = 8 * MB;
  const int smem = 8 * 2 * TR * S * (int)sizeof(double);
  static const bool attr = [&] {
    set_max_dyn_smem(reinterpret_cast<const void*>(k_flag_mma<P, MB>), smem);
    return true;
  }();
  (void)attr;
  const long long tiles = (n + TR - 1) / TR;
  const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>((tiles + 7) / 8, 592));
  k_flag_mma<P, MB><<<grid, 256, smem, st>>>(X, n, log_transform, cs, c2, flags, rd2);
}

#define RTD_DISPATCH_P8(p, F, ...)                                                                          \
  switch (p) {                                                                                           \
    case 8: F<8>(__VA_ARGS__); break; case 9: F<9>(__VA_ARGS__); break; case 10: F<10>(__VA_ARGS__); break; \
    case 11: F<11>(__VA_ARGS__); break; case 12: F<12>(__VA_ARGS__); break; case 13: F<13>(__VA_ARGS__); break; \
    case 14: F<14>(__VA_ARGS__); break; case 15: F<15>(__VA_ARGS__); break; case 16: F<16>(__VA_ARGS__); break; \
    case 17: F<17>(__VA_ARGS__); break; case 18: F<18>(__VA_ARGS__); break; case 19: F<19>(__VA_ARGS__); break; \
    case 20: F<20>(__VA_ARGS__); break; case 21: F<21>(__VA_ARGS__); break; case 22: F<22>(__VA_ARGS__); break; \
    case 23: F<23>(__VA_ARGS__); break; case 24: F<24>(__VA_ARGS__); break; case 25: F<25>(__VA_ARGS__); break; \
    case 26: F<26>(__VA_ARGS__); break; case 27: F<27>(__VA_ARGS__); break; case 28: F<28>(__VA_ARGS__); break; \
    case 29: F<29>(__VA_ARGS__); break; case 30: F<30>(__VA_ARGS__); break; case 31: F<31>(__VA_ARGS__); break; \
    case 32: F<32>(__VA_ARGS__); break; case 33: F<33>(__VA_ARGS__); break; case 34: F<34>(__VA_ARGS__); break; \
    case 35: F<35>(__VA_ARGS__); break; case 36: F<36>(__VA_ARGS__); break; case 37: F<37>(__VA_ARGS__); break; \
    case 38: F<38>(__VA_ARGS__); break; case 39: F<39>(__VA_ARGS__); break; case 40: F<40>(__VA_ARGS__); break; \
    default: throw std::string("dist_mma: p out of range");                                               \
  }

bool dist_mma_supported(int p) { return p >= 8 && p <= RTD_MAXP; }

void launch_dist_inv(int p, const double* Zall, long long m, long long blk_stride, const int* inst, int nstart,
                     int ninst, const double* cstage, int cstride, double* d2_all, cudaStream_t st) {
  RTD_DISPATCH_P8(p, dist_inv_launch, Zall, m, blk_stride, inst, nstart, ninst, cstage, cstride, d2_all, st);
  RTD_LAUNCHED();
}

void launch_flag_mma(int p, const double* X, long long n, int log_transform, const double* cs, double c2,
                     uint8_t* flags, double* rd2, cudaStream_t st) {
  RTD_DISPATCH_P8(p, flag_mma_launch, X, n, log_transform, cs, c2, flags, rd2, st);
  RTD_LAUNCHED();
}

void launch_dist_mma(int p, const double* Zall, long long m, long long blk_stride, const int* inst, int nstart,
                     int ninst, const double* cstage, int cstride, double* d2_all, cudaStream_t st) {
  RTD_DISPATCH_P8(p, dist_mma_launch, Zall, m, blk_stride, inst, nstart, ninst, cstage, cstride, d2_all, st);
  RTD_LAUNCHED();
}

}  // namespace rtd
