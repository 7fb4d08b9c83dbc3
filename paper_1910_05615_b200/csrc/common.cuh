// Device helpers shared by the RT-DetMCD kernels (sm_100a).
// Double-double (dd) arithmetic is used only where the univariate MCD window
// objective needs more than fp64 (reading R2): prefix sums of y and
// y^2 over sorted columns, evaluated with error ~2^-104 relative.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define RTD_MAXP 40
#define RTD_CONST_DOUBLES 8192

namespace rtd {

struct dd {
  double hi, lo;
};

__host__ __device__ __forceinline__ dd dd_make(double a) { return {a, 0.0}; }

__device__ __forceinline__ dd two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  double bb = __dsub_rn(s, a);
  double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, e};
}

__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  double e = __dsub_rn(b, __dsub_rn(s, a));
  return {s, e};
}

__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  double lo = __dadd_rn(s.lo, t.hi);
  s = quick_two_sum(s.hi, lo);
  lo = __dadd_rn(s.lo, t.lo);
  return quick_two_sum(s.hi, lo);
}

__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }

__device__ __forceinline__ dd two_prod(double a, double b) {
  double p = __dmul_rn(a, b);
  double e = __fma_rn(a, b, -p);
  return {p, e};
}

__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  double t = __fma_rn(a.hi, b.lo, __fma_rn(a.lo, b.hi, p.lo));
  return quick_two_sum(p.hi, t);
}

__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  double t = __fma_rn(a.lo, b, p.lo);
  return quick_two_sum(p.hi, t);
}

__device__ __forceinline__ dd dd_div_d(dd a, double b) {
  double q1 = __ddiv_rn(a.hi, b);
  dd r = dd_sub(a, two_prod(q1, b));
  double q2 = __ddiv_rn(r.hi, b);
  r = dd_sub(r, two_prod(q2, b));
  double q3 = __ddiv_rn(r.hi, b);
  dd q = quick_two_sum(q1, q2);
  return dd_add(q, dd_make(q3));
}

// round-to-nearest double of a normalised dd
__device__ __forceinline__ double dd_to_d(dd a) { return __dadd_rn(a.hi, a.lo); }

__device__ __forceinline__ bool dd_lt(dd a, dd b) { return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo); }

// pair of running sums (sum y, sum y^2) in dd
struct dd2 {
  dd s1, s2;
};

__device__ __forceinline__ dd2 dd2_zero() { return {{0.0, 0.0}, {0.0, 0.0}}; }
__device__ __forceinline__ dd2 dd2_add(dd2 a, dd2 b) { return {dd_add(a.s1, b.s1), dd_add(a.s2, b.s2)}; }
__device__ __forceinline__ dd2 dd2_sub(dd2 a, dd2 b) { return {dd_sub(a.s1, b.s1), dd_sub(a.s2, b.s2)}; }
__device__ __forceinline__ dd2 dd2_of(double y) { return {dd_make(y), two_prod(y, y)}; }
// (y, d^2) with d = y - c rounded: the reweighting sums (sum y for the mean, sum (y - c)^2 for the
// variance about the raw location c, free of the cancellation of sum y^2 - (sum y)^2 / k)
__device__ __forceinline__ dd2 dd2_of_dev(double y, double d) { return {dd_make(y), two_prod(d, d)}; }

// reweighted variance numerator sum (y - loc)^2 from K = (sum y, sum (y - c)^2) over k kept values,
// loc = round(sum y) / k:  sum (d - D)^2 = K.s2 - 2 D sum(y - c) + k D^2,  D = loc - c (exact, dd)
__device__ __forceinline__ dd kept_sq_about_loc(const dd2& K, double c, double loc, double k) {
  const dd B = dd_sub(K.s1, two_prod(c, k));
  const dd D = two_sum(loc, -c);
  return dd_add(K.s2, dd_sub(dd_mul(dd_mul_d(D, k), D), dd_mul_d(dd_mul(D, B), 2.0)));
}

__device__ __forceinline__ dd2 shfl_dd2(dd2 v, int src) {
  dd2 r;
  r.s1.hi = __shfl_sync(0xffffffffu, v.s1.hi, src);
  r.s1.lo = __shfl_sync(0xffffffffu, v.s1.lo, src);
  r.s2.hi = __shfl_sync(0xffffffffu, v.s2.hi, src);
  r.s2.lo = __shfl_sync(0xffffffffu, v.s2.lo, src);
  return r;
}
__device__ __forceinline__ dd2 shfl_up_dd2(dd2 v, int d) {
  dd2 r;
  r.s1.hi = __shfl_up_sync(0xffffffffu, v.s1.hi, d);
  r.s1.lo = __shfl_up_sync(0xffffffffu, v.s1.lo, d);
  r.s2.hi = __shfl_up_sync(0xffffffffu, v.s2.hi, d);
  r.s2.lo = __shfl_up_sync(0xffffffffu, v.s2.lo, d);
  return r;
}
__device__ __forceinline__ dd2 shfl_down_dd2(dd2 v, int d) {
  dd2 r;
  r.s1.hi = __shfl_down_sync(0xffffffffu, v.s1.hi, d);
  r.s1.lo = __shfl_down_sync(0xffffffffu, v.s1.lo, d);
  r.s2.hi = __shfl_down_sync(0xffffffffu, v.s2.hi, d);
  r.s2.lo = __shfl_down_sync(0xffffffffu, v.s2.lo, d);
  return r;
}

// Block-wide exclusive scan of dd2 values (blockDim.x multiple of 32, <= 1024).
// Returns exclusive prefix for this thread; *total receives the block total.
// Fixed association order (deterministic run to run).
__device__ __forceinline__ dd2 block_exscan_dd2(dd2 v, dd2* total, dd2* smem /* >= 33 */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  dd2 inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    dd2 t = shfl_up_dd2(inc, d);
    if (lane >= d) inc = dd2_add(t, inc);
  }
  dd2 exw = shfl_up_dd2(inc, 1);
  if (lane == 0) exw = dd2_zero();
  if (lane == 31) smem[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    dd2 w = lane < nw ? smem[lane] : dd2_zero();
    dd2 wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      dd2 t = shfl_up_dd2(wi, d);
      if (lane >= d) wi = dd2_add(t, wi);
    }
    dd2 wex = shfl_up_dd2(wi, 1);
    if (lane == 0) wex = dd2_zero();
    if (lane < nw) smem[lane] = wex;
    if (lane == nw - 1) smem[32] = wi;
  }
  __syncthreads();
  dd2 ex = dd2_add(smem[wid], exw);
  *total = smem[32];
  __syncthreads();
  return ex;
}

// Block-wide fixed-order sum of dd2 (result valid in all threads).
__device__ __forceinline__ dd2 block_sum_dd2(dd2 v, dd2* smem /* >= 33 */) {
  dd2 tot;
  block_exscan_dd2(v, &tot, smem);
  return tot;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
  return v;
}

// cp.async (LDGSTS) staging of 8-byte elements (any double alignment)
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Order-preserving 64-bit key of a double (NaN-free input) and back.
__device__ __forceinline__ unsigned long long ord_key64(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val64(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

// In-register bitonic sort of N = V * blockDim.x keys (N a power of two), element e = threadIdx.x * V + k in
// x[k]: strides below V inside a thread, below 32 V by warp shuffles, the rest through xs[N] (two barriers
// per such stage).  For 4096 keys and 1024 threads: 15 shared-memory stages instead of the 78 barriers of
// a shared-memory network (k_q_sample 43 -> ~6 us).
template <int V, int S>
__device__ __forceinline__ void bitonic_inreg_s(unsigned long long (&x)[V], int size) {
#pragma unroll
  for (int k = 0; k < V; k++) {
    if ((k & S) == 0) {  // compile-time: only the V/2 pairs of this stride
      const int e = threadIdx.x * V + k;
      const bool up = (e & size) == 0;
      const unsigned long long a = x[k], b = x[k + S];
      const unsigned long long lo = a < b ? a : b, hi = a < b ? b : a;
      x[k] = up ? lo : hi;
      x[k + S] = up ? hi : lo;
    }
  }
}
template <int V>
__device__ __forceinline__ void bitonic_inreg_stage(unsigned long long (&x)[V], int stride, int size) {
  if constexpr (V > 1) if (stride == 1) { bitonic_inreg_s<V, 1>(x, size); return; }
  if constexpr (V > 2) if (stride == 2) { bitonic_inreg_s<V, (V > 2 ? 2 : 1)>(x, size); return; }
  if constexpr (V > 4) if (stride == 4) { bitonic_inreg_s<V, (V > 4 ? 4 : 1)>(x, size); return; }
  if constexpr (V > 8) if (stride == 8) { bitonic_inreg_s<V, (V > 8 ? 8 : 1)>(x, size); return; }
  if constexpr (V > 16) if (stride == 16) { bitonic_inreg_s<V, (V > 16 ? 16 : 1)>(x, size); return; }
}
template <int V>
__device__ void block_bitonic_keys(unsigned long long (&x)[V], unsigned long long* xs) {
  const int lane = threadIdx.x & 31;
  const int N = V * (int)blockDim.x;
  for (int size = 2; size <= N; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride < V) {
        bitonic_inreg_stage<V>(x, stride, size);
      } else if (stride < V * 32) {
        const int lm = stride / V;
        const bool lower = (lane & lm) == 0;
#pragma unroll
        for (int k = 0; k < V; k++) {
          const int e = threadIdx.x * V + k;
          const unsigned long long o = __shfl_xor_sync(0xffffffffu, x[k], lm);
          const bool keep_min = ((e & size) == 0) == lower;
          x[k] = keep_min ? (x[k] < o ? x[k] : o) : (x[k] < o ? o : x[k]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < V; k++) xs[threadIdx.x * V + k] = x[k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < V; k++) {
          const int e = threadIdx.x * V + k;
          const unsigned long long o = xs[e ^ stride];
          const bool keep_min = ((e & size) == 0) == ((e & stride) == 0);
          x[k] = keep_min ? (x[k] < o ? x[k] : o) : (x[k] < o ? o : x[k]);
        }
        __syncthreads();
      }
    }
  }
}

// Two order statistics (ranks ra, rb, 0-based) of N = V * blockDim.x ordered 64-bit keys x, without sorting:
// radix levels of 12 bits (sign + exponent first), a 4096-bin histogram per rank and level among the keys
// that share the rank's prefix so far, until the rank's bin holds a single key (then that key is the order
// statistic, exactly) or 60 bits are fixed (then the prefix, low bits cleared for ra / set for rb).  Normal
// columns stop after two or three levels; a column 1e9 + N(0,1) needs four.  Used for routing maps (bucket
// ranges) only.  hist: shared, 2 x 4096 unsigned; blockDim.x == 1024.
__device__ __forceinline__ void rank_bin_4096(const unsigned* h, long long rank, int* s_bin, long long* s_bef,
                                              long long* wsum) {
  // thread t owns bins 4t .. 4t+3; block exclusive scan of the per-thread sums
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  long long c[4], loc = 0;
#pragma unroll
  for (int e = 0; e < 4; e++) {
    c[e] = h[4 * t + e];
    loc += c[e];
  }
  long long inc = loc;
  for (int d = 1; d < 32; d <<= 1) {
    const long long v = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += v;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (t < 32) {
    long long v = wsum[t], x = v;
    for (int d = 1; d < 32; d <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    wsum[t] = x - v;
  }
  __syncthreads();
  long long before = wsum[w] + inc - loc;
#pragma unroll
  for (int e = 0; e < 4; e++) {
    if (c[e] > 0 && before <= rank && rank < before + c[e]) {
      *s_bin = 4 * t + e;
      *s_bef = before;
    }
    before += c[e];
  }
  __syncthreads();
}
template <int V>
__device__ void block_quantile_keys2(const unsigned long long (&x)[V], long long ra, long long rb, unsigned* hist,
                                     unsigned long long* out) {
  __shared__ long long wsum[32];
  __shared__ int s_bin[2];
  __shared__ long long s_bef[2];
  __shared__ unsigned long long s_key[2];
  const int t = threadIdx.x;
  unsigned long long pre[2] = {0ull, 0ull};
  long long rk[2] = {ra, rb};
  bool done[2] = {false, false};
  for (int lev = 0; lev < 5 && !(done[0] && done[1]); lev++) {
    const int sh = 52 - 12 * lev;  // this level's digit: bits [sh, sh + 12)
    for (int i = t; i < 2 * 4096; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < V; k++) {
      const unsigned dig = (unsigned)(x[k] >> sh) & 4095u;
#pragma unroll
      for (int j = 0; j < 2; j++)
        if (!done[j] && (lev == 0 || (x[k] >> (sh + 12)) == pre[j])) atomicAdd(&hist[4096 * j + dig], 1u);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 2; j++) {
      if (done[j]) continue;  // (uniform)
      rank_bin_4096(hist + 4096 * j, rk[j], &s_bin[j], &s_bef[j], wsum);
      const unsigned cnt = hist[4096 * j + s_bin[j]];
      pre[j] = (pre[j] << 12) | (unsigned)s_bin[j];
      rk[j] -= s_bef[j];
      if (cnt == 1u) {  // the rank's key is the only one with this prefix
#pragma unroll
        for (int k = 0; k < V; k++)
          if ((x[k] >> sh) == pre[j]) s_key[j] = x[k];
        done[j] = true;
      } else if (lev == 4) {
        s_key[j] = j == 0 ? (pre[j] << 4) : ((pre[j] << 4) | 15ull);
        done[j] = true;
      }
      __syncthreads();
    }
  }
  if (t == 0) {
    out[0] = s_key[0];
    out[1] = s_key[1];
  }
  __syncthreads();
}

}  // namespace rtd
