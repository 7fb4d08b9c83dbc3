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

}  // namespace rtd
