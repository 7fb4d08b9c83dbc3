// Streaming kernels: layout transforms, the C-step distance pass (H6, ★),
// refinement GEMMs, norms and the row-major flag pass (H12).
//
// Distance (§3.4): d_i^2 = ||L^-1 (z_i - mu)||^2
// with M = L^-1 packed lower-triangular in the constant bank (one slot per
// instance), compile-time P so the triangular mat-vec is fully unrolled:
// P(P+1)/2 + P DFMA per row, X read once, coalesced (Z is column-major).
#include <cmath>
#include <mutex>

#include "rtd_internal.h"

namespace rtd {

__constant__ double c_mat[RTD_CONST_DOUBLES];

namespace {
struct DevConst {
  std::mutex mu;
  cudaEvent_t done = nullptr;  // completion of the last lease's consumers (any stream)
};
DevConst g_const[128];
}  // namespace

ConstLease::ConstLease(const double* dev_src, size_t count, cudaStream_t st) : st_(st) {
  RTD_CU(cudaGetDevice(&dev_));
  DevConst& g = g_const[dev_ & 127];
  g.mu.lock();
  try {
    if (!g.done) RTD_CU(cudaEventCreateWithFlags(&g.done, cudaEventDisableTiming));
    else RTD_CU(cudaStreamWaitEvent(st, g.done, 0));
    RTD_CU(cudaMemcpyToSymbolAsync(c_mat, dev_src, count * sizeof(double), 0, cudaMemcpyDeviceToDevice, st));
  } catch (...) {
    g.mu.unlock();
    throw;
  }
}

ConstLease::~ConstLease() {
  DevConst& g = g_const[dev_ & 127];
  cudaEventRecord(g.done, st_);
  g.mu.unlock();
}

#define RTD_DISPATCH_P(p, F, ...)                                                                        \
  switch (p) {                                                                                         \
    case 1: F<1>(__VA_ARGS__); break; case 2: F<2>(__VA_ARGS__); break; case 3: F<3>(__VA_ARGS__); break;  \
    case 4: F<4>(__VA_ARGS__); break; case 5: F<5>(__VA_ARGS__); break; case 6: F<6>(__VA_ARGS__); break;  \
    case 7: F<7>(__VA_ARGS__); break; case 8: F<8>(__VA_ARGS__); break; case 9: F<9>(__VA_ARGS__); break;  \
    case 10: F<10>(__VA_ARGS__); break; case 11: F<11>(__VA_ARGS__); break; case 12: F<12>(__VA_ARGS__); break; \
    case 13: F<13>(__VA_ARGS__); break; case 14: F<14>(__VA_ARGS__); break; case 15: F<15>(__VA_ARGS__); break; \
    case 16: F<16>(__VA_ARGS__); break; case 17: F<17>(__VA_ARGS__); break; case 18: F<18>(__VA_ARGS__); break; \
    case 19: F<19>(__VA_ARGS__); break; case 20: F<20>(__VA_ARGS__); break; case 21: F<21>(__VA_ARGS__); break; \
    case 22: F<22>(__VA_ARGS__); break; case 23: F<23>(__VA_ARGS__); break; case 24: F<24>(__VA_ARGS__); break; \
    case 25: F<25>(__VA_ARGS__); break; case 26: F<26>(__VA_ARGS__); break; case 27: F<27>(__VA_ARGS__); break; \
    case 28: F<28>(__VA_ARGS__); break; case 29: F<29>(__VA_ARGS__); break; case 30: F<30>(__VA_ARGS__); break; \
    case 31: F<31>(__VA_ARGS__); break; case 32: F<32>(__VA_ARGS__); break; case 33: F<33>(__VA_ARGS__); break; \
    case 34: F<34>(__VA_ARGS__); break; case 35: F<35>(__VA_ARGS__); break; case 36: F<36>(__VA_ARGS__); break; \
    case 37: F<37>(__VA_ARGS__); break; case 38: F<38>(__VA_ARGS__); break; case 39: F<39>(__VA_ARGS__); break; \
    case 40: F<40>(__VA_ARGS__); break;                                                                \
    default: throw std::string("p out of range");                                                     \
  }

// ------------------------------------------------------------------ transpose + validate
static constexpr int TT_ROWS = 64;

// Row-major X (optionally ln) -> column-major Xc through a shared-memory tile of TT_ROWS rows, with the
// finiteness check (first bad row into *bad); p a compile-time constant (no runtime divisions), each CTA
// walking several tiles; the tile's loads are issued back to back (unrolled, TT_ROWS * P / 256 each).
template <int P>
__global__ void __launch_bounds__(256) k_transpose_t(const double* __restrict__ X, long long n, int log_transform,
                                                     double* __restrict__ Xc, unsigned long long* __restrict__ bad) {
  constexpr int S = P + 1, CNT = TT_ROWS * P, PER = (CNT + 255) / 256;
  __shared__ double tile[TT_ROWS * S];
  unsigned long long mybad = ~0ull;
  const long long ntiles = (n + TT_ROWS - 1) / TT_ROWS;
  for (long long tb = blockIdx.x; tb < ntiles; tb += gridDim.x) {
    const long long r0 = tb * TT_ROWS;
    const int rows = (int)min((long long)TT_ROWS, n - r0);
    const int cnt = rows * P;
    double v[PER];
#pragma unroll
    for (int u = 0; u < PER; u++) {
      const int e = threadIdx.x + u * 256;
      v[u] = e < cnt ? __ldg(X + r0 * P + e) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < PER; u++) {
      const int e = threadIdx.x + u * 256;
      if (e < cnt) {
        const int r = e / P, k = e - r * P;
        double x = v[u];
        bool ok = isfinite(x);
        if (log_transform) {
          ok = ok && x > 0.0;
          x = log(x);
        }
        if (!ok) mybad = min(mybad, (unsigned long long)(r0 + r));
        tile[r * S + k] = x;
      }
    }
    __syncthreads();
    if (rows == TT_ROWS) {
#pragma unroll
      for (int u = 0; u < PER; u++) {
        const int e = threadIdx.x + u * 256;
        if (e < CNT) {
          const int k = e / TT_ROWS, r = e - k * TT_ROWS;
          Xc[(long long)k * n + r0 + r] = tile[r * S + k];
        }
      }
    } else {
      for (int e = threadIdx.x; e < cnt; e += 256) {
        const int k = e / rows, r = e - k * rows;
        Xc[(long long)k * n + r0 + r] = tile[r * S + k];
      }
    }
    __syncthreads();
  }
  if (mybad != ~0ull) atomicMin(bad, mybad);
}

template <int P>
static void transpose_t_launch(const double* X, long long n, int log_transform, double* Xc, unsigned long long* bad,
                               cudaStream_t st) {
  const long long ntiles = (n + TT_ROWS - 1) / TT_ROWS;
  k_transpose_t<P><<<(unsigned)std::min<long long>(ntiles, 148 * 12), 256, 0, st>>>(X, n, log_transform, Xc, bad);
}

void launch_transpose(const double* X, long long n, int p, int log_transform, double* Xc, unsigned long long* bad,
                      cudaStream_t st) {
  RTD_DISPATCH_P(p, transpose_t_launch, X, n, log_transform, Xc, bad, st);
  RTD_LAUNCHED();
}

// ------------------------------------------------------------------ Feistel partition (reading R13)
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ unsigned long long feistel_dec(unsigned long long y, unsigned long long seed, int half) {
  const unsigned long long mask = (1ull << half) - 1ull;
  unsigned long long L = y >> half, R = y & mask;
  for (int r = 5; r >= 0; r--) {
    // forward: (L, R) -> (R, L ^ F_r(R)); inverse: R_prev = L, L_prev = R ^ F_r(L)
    unsigned long long F = splitmix64(seed ^ ((unsigned long long)r * 0x9E3779B97F4A7C15ull) ^ L) & mask;
    unsigned long long Lp = R ^ F;
    R = L;
    L = Lp;
  }
  return (L << half) | R;
}

__device__ __forceinline__ long long feistel_inv(long long t, long long n, unsigned long long seed, int half) {
  unsigned long long x = feistel_dec((unsigned long long)t, seed, half);
  while (x >= (unsigned long long)n) x = feistel_dec(x, seed, half);
  return (long long)x;
}

static int feistel_half(long long n) {
  int bits = 0;
  while ((1ll << bits) < n) bits++;  // ceil(log2 n) == bit_length(n-1)
  if (bits < 2) bits = 2;
  bits += bits & 1;
  return bits / 2;
}

__global__ void k_build_Z_identity(const double* __restrict__ Xc, long long n, int p, long long m, int q,
                                   const UniOut* __restrict__ uni, double* __restrict__ Z) {
  // contiguous blocks: Z[b][k][s] = (Xc[k][b*m+s] - loc_k)/scale_k, block by block (no per-element
  // 64-bit division of the flat index), 4 loads in flight per thread
  const int k = blockIdx.y;
  const double loc = uni[k].loc, sc = uni[k].scale;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int b = 0; b < q; b++) {
    const double* __restrict__ src = Xc + (long long)k * n + (long long)b * m;
    double* __restrict__ dst = Z + ((long long)b * p + k) * m;
    for (long long s0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; s0 < m; s0 += 4 * stride) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; u++) v[u] = s0 + u * stride < m ? __ldg(src + s0 + u * stride) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (s0 + u * stride < m) dst[s0 + u * stride] = __ddiv_rn(__dsub_rn(v[u], loc), sc);
    }
  }
}

// The same map with the rows' norms ||z_i|| of S~2 in the same pass: a thread owns
// BZR rows of one block and walks the columns, so the sum of squares runs in registers, sequential
// over k without FMA (the arithmetic of k_norms) -- the initial-estimator pass then needs no norms
// of its own and both of its moment matrices come from one read of Z (MOM_WRAPXI).
static constexpr int BZR = 4;
__global__ void __launch_bounds__(256) k_build_Z_norms(const double* __restrict__ Xc, long long n, int p, long long m,
                                                       const UniOut* __restrict__ uni, double* __restrict__ Z,
                                                       double* __restrict__ r) {
  const int b = blockIdx.y;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long s0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; s0 < m; s0 += BZR * stride) {
    double sq[BZR];
#pragma unroll
    for (int u = 0; u < BZR; u++) sq[u] = 0.0;
    for (int k = 0; k < p; k++) {
      const double loc = __ldg(&uni[k].loc), sc = __ldg(&uni[k].scale);
      const double* __restrict__ src = Xc + (long long)k * n + (long long)b * m;
      double* __restrict__ dst = Z + ((long long)b * p + k) * m;
      double v[BZR];
#pragma unroll
      for (int u = 0; u < BZR; u++) v[u] = s0 + u * stride < m ? __ldg(src + s0 + u * stride) : 0.0;
#pragma unroll
      for (int u = 0; u < BZR; u++) {
        const double z = __ddiv_rn(__dsub_rn(v[u], loc), sc);
        sq[u] = __dadd_rn(sq[u], __dmul_rn(z, z));
        if (s0 + u * stride < m) dst[s0 + u * stride] = z;
      }
    }
#pragma unroll
    for (int u = 0; u < BZR; u++)
      if (s0 + u * stride < m) r[(long long)b * m + s0 + u * stride] = __dsqrt_rn(sq[u]);
  }
}

__global__ void k_build_Z_perm(const double* __restrict__ X, long long n, int p, long long m, int q,
                               unsigned long long seed, int half, int log_transform, const UniOut* __restrict__ uni,
                               double* __restrict__ Z, long long* __restrict__ rowmap, double* __restrict__ r) {
  const long long total = (long long)q * m;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    long long b = t / m, s = t - b * m;
    long long row = feistel_inv(t, n, seed, half);
    if (rowmap) rowmap[t] = row;
    const double* xr = X + row * p;
    double sq = 0.0;
    for (int k = 0; k < p; k++) {
      double v = xr[k];
      if (log_transform) v = log(v);
      const double z = __ddiv_rn(__dsub_rn(v, uni[k].loc), uni[k].scale);
      Z[(b * p + k) * m + s] = z;
      sq = __dadd_rn(sq, __dmul_rn(z, z));
    }
    if (r) r[t] = __dsqrt_rn(sq);
  }
}

void launch_build_Z(const double* Xc, const double* X, long long n, int p, int q, long long m, int perm,
                    unsigned long long seed, int log_transform, const UniOut* uni, double* Z, long long* rowmap,
                    double* r_out, cudaStream_t st) {
  if (!perm && r_out) {
    const unsigned gx = (unsigned)std::max<long long>(1, std::min<long long>((m + 256 * BZR - 1) / (256 * BZR),
                                                                            (148LL * 8 + q - 1) / q));
    k_build_Z_norms<<<dim3(gx, q), 256, 0, st>>>(Xc, n, p, m, uni, Z, r_out);
  } else if (!perm) {
    const unsigned gx = (unsigned)std::max<long long>(1, std::min<long long>((m + 1023) / 1024, 148 * 8));
    k_build_Z_identity<<<dim3(gx, p), 256, 0, st>>>(Xc, n, p, m, q, uni, Z);
  } else {
    long long total = (long long)q * m;
    unsigned gx = (unsigned)std::min<long long>((total + 255) / 256, 148 * 32);
    k_build_Z_perm<<<gx, 256, 0, st>>>(X, n, p, m, q, seed, feistel_half(n), log_transform, uni, Z, rowmap, r_out);
  }
  RTD_LAUNCHED();
}

// ------------------------------------------------------------------ distance pass (H6)
template <int P>
__global__ void __launch_bounds__(256) k_dist(const double* __restrict__ Zall, long long m, long long blk_stride,
                                              const int* __restrict__ inst, int nstart, int cstride,
                                              double* __restrict__ d2_all) {
  const int id = inst[blockIdx.y];
  const double* __restrict__ Z = Zall + (long long)(id / nstart) * blk_stride;
  double* __restrict__ d2 = d2_all + (long long)id * m;
  const double* cm = c_mat + blockIdx.y * cstride;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    double z[P];
#pragma unroll
    for (int k = 0; k < P; k++) z[k] = __dsub_rn(Z[k * m + i], cm[k]);
    double acc = 0.0;
    int off = P;
#pragma unroll
    for (int j = 0; j < P; j++) {
      double y = 0.0;
#pragma unroll
      for (int k = 0; k <= j; k++) y = fma(cm[off + k], z[k], y);
      off += j + 1;
      acc = fma(y, y, acc);
    }
    d2[i] = acc;
  }
}

template <int P>
static void dist_launch(const double* Zall, long long m, long long blk_stride, const int* inst, int nstart, int ninst,
                        int cstride, double* d2_all, cudaStream_t st) {
  long long need = (m + 255) / 256;
  unsigned gx = (unsigned)std::min<long long>(need, std::max<long long>(1, 148LL * 8 / std::max(1, ninst)));
  k_dist<P><<<dim3(gx, ninst), 256, 0, st>>>(Zall, m, blk_stride, inst, nstart, cstride, d2_all);
}

void launch_dist(int p, const double* Zall, long long m, long long blk_stride, const int* inst, int nstart, int ninst,
                 int cstride, double* d2_all, cudaStream_t st) {
  RTD_DISPATCH_P(p, dist_launch, Zall, m, blk_stride, inst, nstart, ninst, cstride, d2_all, st);
  RTD_LAUNCHED();
}

// ------------------------------------------------------------------ refinement GEMM: out = Z W
template <int P>
__global__ void __launch_bounds__(256) k_matmul(const double* __restrict__ Z, long long m, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    double z[P];
#pragma unroll
    for (int k = 0; k < P; k++) z[k] = Z[k * m + i];
#pragma unroll
    for (int j = 0; j < P; j++) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < P; k++) acc = fma(z[k], c_mat[k * P + j], acc);
      out[j * m + i] = acc;
    }
  }
}

template <int P>
static void matmul_launch(const double* Z, long long m, double* out, cudaStream_t st) {
  long long need = (m + 255) / 256;
  unsigned gx = (unsigned)std::min<long long>(need, 148LL * 8);
  k_matmul<P><<<gx, 256, 0, st>>>(Z, m, out);
}

void launch_matmul(int p, const double* Z, long long m, double* out, cudaStream_t st) {
  RTD_DISPATCH_P(p, matmul_launch, Z, m, out, st);
  RTD_LAUNCHED();
}

// ------------------------------------------------------------------ norms ||z_i|| (sequential over k, no FMA)
__global__ void k_norms(const double* __restrict__ Z, long long m, int p, long long blk_stride, double* __restrict__ r) {
  const int b = blockIdx.y;
  const double* Zb = Z + b * blk_stride;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < p; k++) {
      double v = Zb[(long long)k * m + i];
      acc = __dadd_rn(acc, __dmul_rn(v, v));
    }
    r[(long long)b * m + i] = __dsqrt_rn(acc);
  }
}

void launch_norms(const double* Z, long long m, int p, int nblk, long long blk_stride, double* r, cudaStream_t st) {
  unsigned gx = (unsigned)std::min<long long>((m + 255) / 256, 148LL * 8);
  k_norms<<<dim3(gx, nblk), 256, 0, st>>>(Z, m, p, blk_stride, r);
  RTD_LAUNCHED();
}

// ------------------------------------------------------------------ flag pass over row-major X (H12)
static constexpr int FL_ROWS = 128;

template <int P>
__global__ void __launch_bounds__(FL_ROWS) k_flag(const double* __restrict__ X, long long n, int log_transform,
                                                  double c2, uint8_t* __restrict__ flags, double* __restrict__ rd2) {
  constexpr int S = P | 1;  // odd row stride: conflict-free 8-byte row reads
  __shared__ double tile[FL_ROWS * S];
  for (long long r0 = (long long)blockIdx.x * FL_ROWS; r0 < n; r0 += (long long)gridDim.x * FL_ROWS) {
    const int rows = (int)min((long long)FL_ROWS, n - r0);
    const int cnt = rows * P;
    const double* src = X + r0 * P;
    __syncthreads();
    for (int e = threadIdx.x; e < cnt; e += FL_ROWS) {
      int r = e / P, k = e - r * P;
      double v = src[e];
      if (log_transform) v = log(v);
      tile[r * S + k] = v;
    }
    __syncthreads();
    if (threadIdx.x < rows) {
      double z[P];
#pragma unroll
      for (int k = 0; k < P; k++) z[k] = __dsub_rn(tile[threadIdx.x * S + k], c_mat[k]);
      double acc = 0.0;
      int off = P;
#pragma unroll
      for (int j = 0; j < P; j++) {
        double y = 0.0;
#pragma unroll
        for (int k = 0; k <= j; k++) y = fma(c_mat[off + k], z[k], y);
        off += j + 1;
        acc = fma(y, y, acc);
      }
      const long long i = r0 + threadIdx.x;
      if (flags) flags[i] = acc > c2 ? 1 : 0;
      if (rd2) rd2[i] = acc;
    }
  }
}

template <int P>
static void flag_launch(const double* X, long long n, int log_transform, double c2, uint8_t* flags, double* rd2,
                        cudaStream_t st) {
  long long need = (n + FL_ROWS - 1) / FL_ROWS;
  unsigned gx = (unsigned)std::min<long long>(need, 148LL * 16);
  k_flag<P><<<gx, FL_ROWS, 0, st>>>(X, n, log_transform, c2, flags, rd2);
}

void launch_flag(int p, const double* X, long long n, int log_transform, double c2, uint8_t* flags, double* rd2,
                 cudaStream_t st) {
  RTD_DISPATCH_P(p, flag_launch, X, n, log_transform, c2, flags, rd2, st);
  RTD_LAUNCHED();
}

}  // namespace rtd
