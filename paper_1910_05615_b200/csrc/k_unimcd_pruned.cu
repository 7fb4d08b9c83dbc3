// K1 without a full sort: the exact univariate MCD window by bucketing and
// bounding (the estimator is PAPER.md:430-453, §3.1).
//
// The raw MCD of a column is the h-window of consecutive order statistics
// with the smallest sum of squares; only the order statistics at the two ends
// of near-optimal windows need to be known exactly.  Per column:
//   1. a strided sample fixes a monotone bucket map over its [0.5%, 99.5%]
//      range (4096 buckets incl. an underflow and an overflow bucket);
//   2. one pass builds per-CTA shared-memory histograms (count, sum) that are
//      folded into global memory;
//   3. one CTA bounds h*SQ(s) for every start s from the bucket data: r
//      elements of a partially covered bucket lie in its value range, and the
//      sum of squares of a bucket with count r and sum S lies in
//      [S^2/r, S(L+U) - rLU]; it keeps the starts whose lower bound is <= the
//      smallest upper bound;
//   4. one pass gathers the elements of the buckets that hold candidate
//      window ends and sums (double-double, fixed order) everything below them;
//   5. the gathered sets are sorted (segmented radix sort), prefix-summed in
//      double-double, and h*SQ(s) is evaluated exactly for every candidate s:
//      argmin, ties -> lowest s (reading R2);
//   6. one pass sums the kept points of the reweighting step (reading R4).
// A column whose candidate sets do not fit (massive ties, extreme shapes)
// makes the caller fall back to the full radix-sort path (same result).
#include <cstdio>
#include <cstdlib>

#include <cub/device/device_segmented_radix_sort.cuh>

#include "rtd_internal.h"

namespace rtd {

static constexpr int NBK = 4096;         // buckets per column (incl. underflow 0 and overflow NBK-1)
static constexpr int SAMPLE = 4096;      // strided sample for the bucket map
static constexpr int CAP = 65536;        // max gathered elements per side per column
static constexpr int PCTA = 32;          // CTAs per column in the streaming passes (fixed -> deterministic)
static constexpr int PT = 256;

struct PrunedCol {
  double lo, hi, w, inv_w;   // bucket map
  double cmin, cmax;         // column min / max
  long long smin, smax;      // candidate window starts
  int bs_lo, bs_hi, be_lo, be_hi;  // gathered bucket ranges (start side / end side)
  long long cs_lo, ce_lo;    // C[bs_lo], C[be_lo]
  int status;                // 0 ok, 1 fall back
  int pad;
};

__device__ __forceinline__ int bucket_of(double y, const PrunedCol& c) {
  if (y < c.lo) return 0;
  if (y >= c.hi) return NBK - 1;
  double t = __dmul_rn(__dsub_rn(y, c.lo), c.inv_w);
  int b = 1 + (int)t;
  return b > NBK - 2 ? NBK - 2 : b;
}

// value range of bucket b (fuzzed by 1e-6 bucket widths against rounding in bucket_of)
__device__ __forceinline__ double bucket_lo(int b, const PrunedCol& c) {
  return b == 0 ? c.cmin : (b == NBK - 1 ? c.hi : c.lo + ((double)(b - 1) - 1e-6) * c.w);
}
__device__ __forceinline__ double bucket_hi(int b, const PrunedCol& c) {
  return b == 0 ? c.lo : (b == NBK - 1 ? c.cmax : c.lo + ((double)b + 1e-6) * c.w);
}

__device__ __forceinline__ unsigned long long ord_key(double x) {
  unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
  unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// Running (sum y, sum y^2) of one thread in double-double, adding one double at a time with
// error-free transformations (two-sum, two-product) and no per-element renormalisation: the
// rounding errors are collected in the low words (17 fp64 ops per element instead of 23).  A thread adds at most a
// few thousand terms, so the low words stay exact to ~2^-100 relative; thread partials are folded
// with the full dd2_add.
struct ddacc {
  double h1, l1, h2, l2;
};
__device__ __forceinline__ ddacc ddacc_zero() { return {0.0, 0.0, 0.0, 0.0}; }
__device__ __forceinline__ void ddacc_add(ddacc& a, double v) {
  const double s = __dadd_rn(a.h1, v);
  const double bb = __dsub_rn(s, a.h1);
  const double e = __dadd_rn(__dsub_rn(a.h1, __dsub_rn(s, bb)), __dsub_rn(v, bb));
  a.h1 = s;
  a.l1 = __dadd_rn(a.l1, e);
  const double pr = __dmul_rn(v, v);
  const double pe = __fma_rn(v, v, -pr);
  const double s2 = __dadd_rn(a.h2, pr);
  const double b2 = __dsub_rn(s2, a.h2);
  const double e2 = __dadd_rn(__dsub_rn(a.h2, __dsub_rn(s2, b2)), __dsub_rn(pr, b2));
  a.h2 = s2;
  a.l2 = __dadd_rn(a.l2, __dadd_rn(e2, pe));
}
// the reweighting form: sum y and sum d^2 (d = y - c already rounded)
__device__ __forceinline__ void ddacc_add_dev(ddacc& a, double v, double dv) {
  const double s = __dadd_rn(a.h1, v);
  const double bb = __dsub_rn(s, a.h1);
  const double e = __dadd_rn(__dsub_rn(a.h1, __dsub_rn(s, bb)), __dsub_rn(v, bb));
  a.h1 = s;
  a.l1 = __dadd_rn(a.l1, e);
  const double pr = __dmul_rn(dv, dv);
  const double pe = __fma_rn(dv, dv, -pr);
  const double s2 = __dadd_rn(a.h2, pr);
  const double b2 = __dsub_rn(s2, a.h2);
  const double e2 = __dadd_rn(__dsub_rn(a.h2, __dsub_rn(s2, b2)), __dsub_rn(pr, b2));
  a.h2 = s2;
  a.l2 = __dadd_rn(a.l2, __dadd_rn(e2, pe));
}
__device__ __forceinline__ dd2 ddacc_dd2(const ddacc& a) {
  return {quick_two_sum(a.h1, a.l1), quick_two_sum(a.h2, a.l2)};
}

static constexpr int ILP = 8;  // elements loaded per thread before they are consumed (latency hiding)

__device__ void smem_bitonic(double* a, int npow2) {
  for (int k = 2; k <= npow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
        int ixj = i ^ j;
        if (ixj > i) {
          bool up = (i & k) == 0;
          double x = a[i], y = a[ixj];
          if ((x > y) == up) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

// 1. bucket map from a strided sample
__global__ void __launch_bounds__(1024) k_pr_sample(const double* __restrict__ cols, long long len,
                                                    PrunedCol* __restrict__ pc, unsigned long long* __restrict__ mm) {
  __shared__ double s[SAMPLE];
  const int col = blockIdx.x;
  const double* y = cols + (long long)col * len;
  for (int i = threadIdx.x; i < SAMPLE; i += blockDim.x) s[i] = y[(long long)i * len / SAMPLE];
  __syncthreads();
  smem_bitonic(s, SAMPLE);
  if (threadIdx.x == 0) {
    PrunedCol c;
    memset(&c, 0, sizeof(c));
    double ql = s[SAMPLE / 200], qh = s[SAMPLE - 1 - SAMPLE / 200];
    double span = qh - ql;
    c.lo = ql - 0.05 * span;
    c.hi = qh + 0.05 * span;
    c.w = (c.hi - c.lo) / (double)(NBK - 2);
    c.inv_w = 1.0 / c.w;
    c.status = (span > 0.0 && isfinite(span) && c.w > 0.0) ? 0 : 1;
    pc[col] = c;
    mm[2 * col] = ~0ull;
    mm[2 * col + 1] = 0ull;
  }
}

// 2. histogram per bucket: the count and, for interior buckets, the sum of the 16-bit fixed-point
//    offsets q = floor(2^16 (y - L_b) / w) of its elements (native 32-bit shared atomics; a CTA takes at
//    most 65536 elements so a bucket's sum fits 32 bits).  An element with offset q lies in
//    [L_b + w (q - 1) 2^-16, L_b + w (q + 2) 2^-16] (the margin covers the rounding of the offset), so
//    the bucket sum is known to an interval (k_pr_scan).  The under- and overflow buckets' sums are
//    accumulated in registers (fp64) and added once per warp.
__global__ void __launch_bounds__(PT) k_pr_hist(const double* __restrict__ cols, long long len,
                                                const PrunedCol* __restrict__ pc, int* __restrict__ cnt,
                                                unsigned long long* __restrict__ tq, double* __restrict__ esum,
                                                unsigned long long* __restrict__ mm) {
  __shared__ unsigned int hc[NBK];
  __shared__ unsigned int hq[NBK];
  const int col = blockIdx.y;
  const PrunedCol c = pc[col];
  if (c.status) return;
  for (int b = threadIdx.x; b < NBK; b += PT) {
    hc[b] = 0u;
    hq[b] = 0u;
  }
  __syncthreads();
  const double* y = cols + (long long)col * len;
  unsigned long long kmin = ~0ull, kmax = 0ull;
  double e0 = 0.0, e1 = 0.0, a0 = 0.0, a1 = 0.0;  // end-bucket sums and sums of magnitudes
  const long long per = (len + gridDim.x - 1) / gridDim.x;
  const long long i0 = blockIdx.x * per, i1 = min(len, i0 + per);
  for (long long base = i0 + threadIdx.x; base < i1; base += (long long)PT * ILP) {
    double v[ILP];
#pragma unroll
    for (int k = 0; k < ILP; k++) {
      const long long i = base + (long long)k * PT;
      v[k] = i < i1 ? __ldg(y + i) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < ILP; k++) {
      if (base + (long long)k * PT < i1) {
        const int b = bucket_of(v[k], c);
        atomicAdd(&hc[b], 1u);
        if (b == 0) {
          e0 += v[k];
          a0 += fabs(v[k]);
        } else if (b == NBK - 1) {
          e1 += v[k];
          a1 += fabs(v[k]);
        } else {
          const double tt = __dsub_rn(__dmul_rn(__dsub_rn(v[k], c.lo), c.inv_w), (double)(b - 1));
          const int q = (int)fmin(fmax(__dmul_rn(tt, 65536.0), 0.0), 65535.0);
          atomicAdd(&hq[b], (unsigned int)q);
        }
        const unsigned long long kk = ord_key(v[k]);
        kmin = min(kmin, kk);
        kmax = max(kmax, kk);
      }
    }
  }
  for (int d = 16; d > 0; d >>= 1) {
    kmin = min(kmin, __shfl_down_sync(0xffffffffu, kmin, d));
    kmax = max(kmax, __shfl_down_sync(0xffffffffu, kmax, d));
    e0 += __shfl_down_sync(0xffffffffu, e0, d);
    e1 += __shfl_down_sync(0xffffffffu, e1, d);
    a0 += __shfl_down_sync(0xffffffffu, a0, d);
    a1 += __shfl_down_sync(0xffffffffu, a1, d);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mm[2 * col], kmin);
    atomicMax(&mm[2 * col + 1], kmax);
    if (a0 != 0.0) {
      atomicAdd(&esum[4 * col], e0);
      atomicAdd(&esum[4 * col + 2], a0);
    }
    if (a1 != 0.0) {
      atomicAdd(&esum[4 * col + 1], e1);
      atomicAdd(&esum[4 * col + 3], a1);
    }
  }
  __syncthreads();
  int* cn = cnt + (long long)col * NBK;
  unsigned long long* tqc = tq + (long long)col * NBK;
  for (int b = threadIdx.x; b < NBK; b += PT)
    if (hc[b]) {
      atomicAdd(&cn[b], (int)hc[b]);
      if (hq[b]) atomicAdd(&tqc[b], (unsigned long long)hq[b]);
    }
}

// 3a. prefix arrays over buckets (one CTA per column): rank offsets C, the interval [Slo, Shi] of
//     every bucket's sum (fixed-point offsets, k_pr_hist; the end buckets' fp64 sums widened by 1e-12
//     relative) and its prefix sums A1lo / A1hi, bounds on the sums of squares Q2lo / Q2hi; margins E1,
//     E2 for the rounding of these fp64 evaluations
struct BucketScan {
  double E1, E2;
};

__device__ __forceinline__ void bucket_sum_interval(int b, int r, unsigned long long T, const double* es,
                                                    const PrunedCol& c, double& Slo, double& Shi) {
  if (r == 0) {
    Slo = Shi = 0.0;
  } else if (b == 0 || b == NBK - 1) {
    // an fp64 sum of r terms in any order is within (r + 2) u sum|y| of the exact sum (u = 2^-53;
    // the sum of magnitudes itself carries a relative error below (r + 2) u, hence the factor 2)
    const double S = es[b == 0 ? 0 : 1], Sa = es[b == 0 ? 2 : 3];
    const double err = 2.0 * ((double)r + 2.0) * 0x1p-53 * Sa + 1e-300;
    Slo = S - err;
    Shi = S + err;
  } else {
    const double rd = (double)r, Lb = c.lo + (double)(b - 1) * c.w, u = c.w * (1.0 / 65536.0);
    Slo = fmax(rd * bucket_lo(b, c), rd * Lb + u * ((double)T - rd));
    Shi = fmin(rd * bucket_hi(b, c), rd * Lb + u * ((double)T + 2.0 * rd));
  }
}

__global__ void __launch_bounds__(1024) k_pr_scan(PrunedCol* __restrict__ pc, const int* __restrict__ cnt,
                                                  const unsigned long long* __restrict__ tq,
                                                  const double* __restrict__ esum,
                                                  const unsigned long long* __restrict__ mm, long long* __restrict__ Cg,
                                                  double* __restrict__ A1g, double* __restrict__ Q2log,
                                                  double* __restrict__ Q2hig, double* __restrict__ sbg,
                                                  BucketScan* __restrict__ bsc) {
  __shared__ double red_d[32];
  __shared__ long long wc[32];
  __shared__ double w1[32], wh[32], wlo[32], whi[32];
  const int col = blockIdx.x;
  PrunedCol c = pc[col];
  if (c.status) return;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int* cn = cnt + (long long)col * NBK;
  const unsigned long long* tqc = tq + (long long)col * NBK;
  const double* es = esum + 4 * col;
  double* sblo = sbg + (long long)col * 2 * NBK;
  double* sbhi = sblo + NBK;
  c.cmin = ord_val(mm[2 * col]);
  c.cmax = ord_val(mm[2 * col + 1]);
  long long* C = Cg + (long long)col * (NBK + 1);
  double* A1lo = A1g + (long long)col * 2 * (NBK + 1);
  double* A1hi = A1lo + (NBK + 1);
  double* Q2lo = Q2log + (long long)col * (NBK + 1);
  double* Q2hi = Q2hig + (long long)col * (NBK + 1);
  constexpr int per = NBK / 1024;
  double slo[per], shi[per], qlo[per], qhi[per];
  long long lc = 0;
  double l1 = 0.0, lh = 0.0, llo = 0.0, lhi = 0.0, abs1 = 0.0;
#pragma unroll
  for (int e = 0; e < per; e++) {
    const int b = t * per + e;
    const int r = cn[b];
    bucket_sum_interval(b, r, tqc[b], es, c, slo[e], shi[e]);
    sblo[b] = slo[e];
    sbhi[b] = shi[e];
    const double L = bucket_lo(b, c), U = bucket_hi(b, c), rd = (double)r;
    qlo[e] = 0.0;
    qhi[e] = 0.0;
    if (r > 0) {
      const double mn2 = (slo[e] <= 0.0 && shi[e] >= 0.0) ? 0.0 : fmin(slo[e] * slo[e], shi[e] * shi[e]);
      const double mx2 = fmax(slo[e] * slo[e], shi[e] * shi[e]);
      qlo[e] = mn2 / rd;
      qhi[e] = fmax(fmax(slo[e] * (L + U), shi[e] * (L + U)) - rd * L * U, mx2 / rd);
    }
    lc += r;
    l1 += slo[e];
    lh += shi[e];
    llo += qlo[e];
    lhi += qhi[e];
    abs1 += fmax(fabs(slo[e]), fabs(shi[e]));
  }
  long long ic = lc;
  double i1 = l1, ih = lh, ilo = llo, ihi = lhi;
  for (int d = 1; d < 32; d <<= 1) {
    long long vc = __shfl_up_sync(0xffffffffu, ic, d);
    double v1 = __shfl_up_sync(0xffffffffu, i1, d);
    double vh = __shfl_up_sync(0xffffffffu, ih, d);
    double vlo = __shfl_up_sync(0xffffffffu, ilo, d);
    double vhi = __shfl_up_sync(0xffffffffu, ihi, d);
    if (lane >= d) {
      ic += vc;
      i1 += v1;
      ih += vh;
      ilo += vlo;
      ihi += vhi;
    }
  }
  if (lane == 31) {
    wc[w] = ic;
    w1[w] = i1;
    wh[w] = ih;
    wlo[w] = ilo;
    whi[w] = ihi;
  }
  __syncthreads();
  if (w == 0) {
    long long vc = wc[lane];
    double v1 = w1[lane], vh = wh[lane], vlo = wlo[lane], vhi = whi[lane];
    long long xc = vc;
    double x1 = v1, xh = vh, xlo = vlo, xhi = vhi;
    for (int d = 1; d < 32; d <<= 1) {
      long long yc = __shfl_up_sync(0xffffffffu, xc, d);
      double y1 = __shfl_up_sync(0xffffffffu, x1, d);
      double yh = __shfl_up_sync(0xffffffffu, xh, d);
      double ylo = __shfl_up_sync(0xffffffffu, xlo, d);
      double yhi = __shfl_up_sync(0xffffffffu, xhi, d);
      if (lane >= d) {
        xc += yc;
        x1 += y1;
        xh += yh;
        xlo += ylo;
        xhi += yhi;
      }
    }
    wc[lane] = xc - vc;
    w1[lane] = x1 - v1;
    wh[lane] = xh - vh;
    wlo[lane] = xlo - vlo;
    whi[lane] = xhi - vhi;
  }
  __syncthreads();
  long long ec = wc[w] + ic - lc;
  double e1 = w1[w] + i1 - l1, eh = wh[w] + ih - lh, elo = wlo[w] + ilo - llo, ehi = whi[w] + ihi - lhi;
#pragma unroll
  for (int e = 0; e < per; e++) {
    const int b = t * per + e;
    C[b] = ec;
    A1lo[b] = e1;
    A1hi[b] = eh;
    Q2lo[b] = elo;
    Q2hi[b] = ehi;
    ec += cn[b];
    e1 += slo[e];
    eh += shi[e];
    elo += qlo[e];
    ehi += qhi[e];
  }
  if (t == 1023) {
    C[NBK] = ec;
    A1lo[NBK] = e1;
    A1hi[NBK] = eh;
    Q2lo[NBK] = elo;
    Q2hi[NBK] = ehi;
  }
  for (int d = 16; d > 0; d >>= 1) abs1 += __shfl_down_sync(0xffffffffu, abs1, d);
  if (lane == 0) red_d[w] = abs1;
  __syncthreads();
  if (t == 1023) {
    double tot_abs1 = 0.0;
    for (int k = 0; k < 32; k++) tot_abs1 += red_d[k];
    bsc[col] = {1e-10 * (tot_abs1 + 1e-300), 1e-10 * (fabs(ehi) + 1e-300)};
    pc[col] = c;  // with column min / max
  }
}

// bounds on h*SQ(s) for one start s (start bucket b, end bucket be)
struct VBound {
  double lo, hi;
};

__device__ __forceinline__ VBound window_bounds(long long s, long long h, int b, int be, const PrunedCol& c,
                                                const long long* C, const double* A1, const double* Q2lo,
                                                const double* Q2hi, const int* cn, const double* sb,
                                                BucketScan m) {
  const double hd = (double)h;
  const double L1 = bucket_lo(b, c), U1 = bucket_hi(b, c), L2 = bucket_lo(be, c), U2 = bucket_hi(be, c);
  const double mx1 = fmax(L1 * L1, U1 * U1), mn1 = (L1 <= 0 && U1 >= 0) ? 0.0 : fmin(L1 * L1, U1 * U1);
  const double mx2 = fmax(L2 * L2, U2 * U2), mn2 = (L2 <= 0 && U2 >= 0) ? 0.0 : fmin(L2 * L2, U2 * U2);
  double lo1, hi1, lo2, hi2;
  if (be == b) {
    lo1 = hd * L1;
    hi1 = hd * U1;
    lo2 = hd * mn1;
    hi2 = hd * mx1;
  } else {
    const double n1 = (double)cn[b], n2 = (double)cn[be];
    // bucket sums are intervals: sb[0..NBK) lower ends, sb[NBK..2NBK) upper ends; A1 likewise
    const double Sblo = sb[b], Sbhi = sb[NBK + b], Selo = sb[be], Sehi = sb[NBK + be];
    const double r1 = (double)(C[b + 1] - s), r2 = (double)(s + h - C[be]);
    // top r1 elements of bucket b: mean >= bucket mean; the other n1 - r1 are >= L1
    const double t1lo = fmax(r1 * L1, r1 * Sblo * __drcp_rn(n1)), t1hi = fmin(r1 * U1, Sbhi - (n1 - r1) * L1);
    // bottom r2 elements of bucket be: mean <= bucket mean; the other n2 - r2 are <= U2
    const double t2lo = fmax(r2 * L2, Selo - (n2 - r2) * U2), t2hi = fmin(r2 * U2, r2 * Sehi * __drcp_rn(n2));
    const double F1lo = A1[be] - A1[b + 1], F1hi = A1[NBK + 1 + be] - A1[NBK + 1 + b + 1];
    lo1 = F1lo + fmin(t1lo, t1hi) + fmin(t2lo, t2hi) - m.E1;
    hi1 = F1hi + fmax(t1lo, t1hi) + fmax(t2lo, t2hi) + m.E1;
    lo2 = (Q2lo[be] - Q2lo[b + 1]) + r1 * mn1 + r2 * mn2 - m.E2;
    hi2 = (Q2hi[be] - Q2hi[b + 1]) + r1 * mx1 + r2 * mx2 + m.E2;
  }
  const double sq_hi_1 = fmax(lo1 * lo1, hi1 * hi1);
  const double sq_lo_1 = (lo1 <= 0 && hi1 >= 0) ? 0.0 : fmin(lo1 * lo1, hi1 * hi1);
  const double slack = 1e-9 * (hd * fabs(hi2) + sq_hi_1) + 1e-300;
  return {hd * lo2 - sq_hi_1 - slack, hd * hi2 - sq_lo_1 + slack};
}

__device__ __forceinline__ int rank_bucket(const long long* C, long long r) {  // largest b with C[b] <= r
  int lo = 0, hi = NBK - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (C[mid] <= r) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// partial-bucket sums of one window start s (start bucket b, end bucket be), see window_bounds
struct PartBounds {
  double t1lo, t1hi, t2lo, t2hi;
};
__device__ __forceinline__ PartBounds part_bounds(long long s, long long h, int b, int be, const PrunedCol& c,
                                                  const long long* C, const int* cn, const double* sb) {
  const double L1 = bucket_lo(b, c), U1 = bucket_hi(b, c), L2 = bucket_lo(be, c), U2 = bucket_hi(be, c);
  const double n1 = (double)cn[b], n2 = (double)cn[be];
  const double Sblo = sb[b], Sbhi = sb[NBK + b], Selo = sb[be], Sehi = sb[NBK + be];
  const double r1 = (double)(C[b + 1] - s), r2 = (double)(s + h - C[be]);
  const double a = fmax(r1 * L1, r1 * Sblo * __drcp_rn(n1)), bb = fmin(r1 * U1, Sbhi - (n1 - r1) * L1);
  const double d = fmax(r2 * L2, Selo - (n2 - r2) * U2), e = fmin(r2 * U2, r2 * Sehi * __drcp_rn(n2));
  return {fmin(a, bb), fmax(a, bb), fmin(d, e), fmax(d, e)};
}

// Lower bound of h*SQ(s) valid for every s in [sa, sb] (same b, be, b != be): the partial
// sums are monotone in s (t1 decreases, t2 increases), so the extremes come from the endpoints.
__device__ __forceinline__ double chunk_lower(long long sa, long long sb, long long h, int b, int be,
                                              const PrunedCol& c, const long long* C, const double* A1,
                                              const double* Q2lo, const int* cn, const double* sbk, BucketScan m) {
  const double hd = (double)h;
  const PartBounds pa = part_bounds(sa, h, b, be, c, C, cn, sbk), pb = part_bounds(sb, h, b, be, c, C, cn, sbk);
  const double F1lo = A1[be] - A1[b + 1], F1hi = A1[NBK + 1 + be] - A1[NBK + 1 + b + 1];
  const double lo1 = F1lo + fmin(pa.t1lo, pb.t1lo) + fmin(pa.t2lo, pb.t2lo) - m.E1;
  const double hi1 = F1hi + fmax(pa.t1hi, pb.t1hi) + fmax(pa.t2hi, pb.t2hi) + m.E1;
  const double L1 = bucket_lo(b, c), U1 = bucket_hi(b, c), L2 = bucket_lo(be, c), U2 = bucket_hi(be, c);
  const double mn1 = (L1 <= 0 && U1 >= 0) ? 0.0 : fmin(L1 * L1, U1 * U1);
  const double mn2 = (L2 <= 0 && U2 >= 0) ? 0.0 : fmin(L2 * L2, U2 * U2);
  double lo2 = INFINITY;
  for (int k = 0; k < 2; k++) {
    const long long s = k ? sb : sa;
    lo2 = fmin(lo2, (Q2lo[be] - Q2lo[b + 1]) + (double)(C[b + 1] - s) * mn1 + (double)(s + h - C[be]) * mn2);
  }
  lo2 -= m.E2;
  const double sq_hi_1 = fmax(lo1 * lo1, hi1 * hi1);
  const double slack = 1e-9 * (hd * fabs(lo2) + sq_hi_1) + 1e-300;
  return hd * lo2 - sq_hi_1 - slack;
}

static constexpr int CHUNK = 32;  // starts per chunk in the coarse lower-bound pass

// 3b. mode 0: upper bounds on a stride-CHUNK subset of starts (any subset gives a valid bound on the
//             minimum) -> per-CTA minimum;
//     mode 1: chunk lower bounds over all starts -> per-CTA range of candidate chunks;
//     mode 2: per-start lower bounds inside the candidate chunk range -> per-CTA candidate range.
__global__ void __launch_bounds__(PT) k_pr_bound(long long len, long long h, const PrunedCol* __restrict__ pc,
                                                 const int* __restrict__ cnt, const double* __restrict__ sbg,
                                                 const long long* __restrict__ Cg, const double* __restrict__ A1g,
                                                 const double* __restrict__ Q2log, const double* __restrict__ Q2hig,
                                                 const BucketScan* __restrict__ bsc, int mode,
                                                 const double* __restrict__ best_ub, const long long* __restrict__ crange,
                                                 double* __restrict__ ub_part, long long* __restrict__ range_part) {
  __shared__ double rd[PT / 32];
  __shared__ long long ra[PT / 32], rb[PT / 32];
  const int col = blockIdx.y;
  const PrunedCol c = pc[col];
  if (c.status) return;
  const long long* C = Cg + (long long)col * (NBK + 1);
  const double* A1 = A1g + (long long)col * 2 * (NBK + 1);  // [lo | hi] prefix sums of bucket sums
  const double* Q2lo = Q2log + (long long)col * (NBK + 1);
  const double* Q2hi = Q2hig + (long long)col * (NBK + 1);
  const int* cn = cnt + (long long)col * NBK;
  const double* sbk = sbg + (long long)col * 2 * NBK;       // [lo | hi] bucket sums
  const BucketScan m = bsc[col];
  const long long nwin = len - h + 1;
  const long long gtid = (long long)blockIdx.x * PT + threadIdx.x;
  const long long nthreads = (long long)gridDim.x * PT;
  const double bub = mode ? best_ub[col] : 0.0;
  double ub = INFINITY;
  long long cmin = 0x7fffffffffffffffLL, cmax = -1;
  // modes 0 and 1: every thread takes a contiguous range of sampled starts / chunks, finds the
  // start and end buckets once by binary search and then only walks them forward
  const long long nchunks = (nwin + CHUNK - 1) / CHUNK;
  const long long cper = (nchunks + nthreads - 1) / nthreads;
  const long long ch0 = gtid * cper, ch1 = min(nchunks, ch0 + cper);
  if (mode == 0) {
    if (ch0 < ch1) {
      int b = rank_bucket(C, ch0 * CHUNK), be = rank_bucket(C, ch0 * CHUNK + h - 1);
      for (long long ch = ch0; ch < ch1; ch++) {
        const long long s = ch * CHUNK;
        while (C[b + 1] <= s) b++;
        while (C[be + 1] <= s + h - 1) be++;
        ub = fmin(ub, window_bounds(s, h, b, be, c, C, A1, Q2lo, Q2hi, cn, sbk, m).hi);
      }
    }
  } else if (mode == 1) {
    // the thread's contiguous range of starts, cut only where the start bucket or the end bucket
    // changes: one lower bound per maximal (b, be) segment (about 2 NBK segments per column)
    if (ch0 < ch1) {
      const long long s1e = min(nwin, ch1 * CHUNK);
      long long sa = ch0 * CHUNK;
      int b = rank_bucket(C, sa), be = rank_bucket(C, sa + h - 1);
      while (sa < s1e) {
        while (C[b + 1] <= sa) b++;
        while (C[be + 1] <= sa + h - 1) be++;
        const long long sb = min(min(s1e, C[b + 1]), C[be + 1] - h + 1) - 1;  // same (b, be) on [sa, sb]
        const double lo = (b == be) ? -INFINITY : chunk_lower(sa, sb, h, b, be, c, C, A1, Q2lo, cn, sbk, m);
        if (lo <= bub) {
          cmin = min(cmin, sa);
          cmax = max(cmax, sb);
        }
        sa = sb + 1;
      }
    }
  } else {
    const long long lo_s = crange[2 * col], hi_s = crange[2 * col + 1];
    if (lo_s <= hi_s) {
      const long long cnt_s = hi_s - lo_s + 1;
      const long long per = (cnt_s + nthreads - 1) / nthreads;
      const long long s0 = lo_s + gtid * per, s1e = min(hi_s + 1, s0 + per);
      if (s0 < s1e) {
        int b = rank_bucket(C, s0), be = rank_bucket(C, s0 + h - 1);
        for (long long s = s0; s < s1e; s++) {
          while (C[b + 1] <= s) b++;
          while (C[be + 1] <= s + h - 1) be++;
          if (window_bounds(s, h, b, be, c, C, A1, Q2lo, Q2hi, cn, sbk, m).lo <= bub) {
            cmin = min(cmin, s);
            cmax = max(cmax, s);
          }
        }
      }
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (mode == 0) {
    for (int d = 16; d > 0; d >>= 1) ub = fmin(ub, __shfl_down_sync(0xffffffffu, ub, d));
    if (lane == 0) rd[w] = ub;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = 1; k < PT / 32; k++) ub = fmin(ub, rd[k]);
      ub_part[(long long)col * gridDim.x + blockIdx.x] = ub;
    }
  } else {
    for (int d = 16; d > 0; d >>= 1) {
      cmin = min(cmin, __shfl_down_sync(0xffffffffu, cmin, d));
      cmax = max(cmax, __shfl_down_sync(0xffffffffu, cmax, d));
    }
    if (lane == 0) {
      ra[w] = cmin;
      rb[w] = cmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = 1; k < PT / 32; k++) {
        cmin = min(cmin, ra[k]);
        cmax = max(cmax, rb[k]);
      }
      range_part[((long long)col * gridDim.x + blockIdx.x) * 2] = cmin;
      range_part[((long long)col * gridDim.x + blockIdx.x) * 2 + 1] = cmax;
    }
  }
}

__global__ void k_pr_ubmin(const PrunedCol* __restrict__ pc, const double* __restrict__ ub_part, int nb,
                           double* __restrict__ best_ub) {
  const int col = blockIdx.x;
  if (pc[col].status || threadIdx.x != 0) return;
  double ub = INFINITY;
  for (int k = 0; k < nb; k++) ub = fmin(ub, ub_part[(long long)col * nb + k]);
  best_ub[col] = ub;
}

__global__ void k_pr_range(const PrunedCol* __restrict__ pc, const long long* __restrict__ range_part, int nb,
                           long long* __restrict__ crange) {
  const int col = blockIdx.x;
  if (pc[col].status || threadIdx.x != 0) return;
  long long smin = 0x7fffffffffffffffLL, smax = -1;
  for (int k = 0; k < nb; k++) {
    smin = min(smin, range_part[((long long)col * nb + k) * 2]);
    smax = max(smax, range_part[((long long)col * nb + k) * 2 + 1]);
  }
  crange[2 * col] = smin;
  crange[2 * col + 1] = smax;
}

// 3c. candidate range -> gathered bucket ranges
__global__ void k_pr_cand(long long len, long long h, PrunedCol* __restrict__ pc, const long long* __restrict__ Cg,
                          const long long* __restrict__ crange) {
  const int col = blockIdx.x;
  PrunedCol c = pc[col];
  if (c.status || threadIdx.x != 0) return;
  const long long* C = Cg + (long long)col * (NBK + 1);
  const long long smin = crange[2 * col], smax = crange[2 * col + 1];
  c.smin = smin;
  c.smax = smax;
  if (smax < smin) {
    c.status = 1;
  } else {
    c.bs_lo = rank_bucket(C, smin);
    c.bs_hi = rank_bucket(C, smax);
    c.be_lo = rank_bucket(C, smin + h);
    c.be_hi = rank_bucket(C, min(smax + h, len - 1));
    c.cs_lo = C[c.bs_lo];
    c.ce_lo = C[c.be_lo];
    const long long ns = C[c.bs_hi + 1] - C[c.bs_lo], ne = C[c.be_hi + 1] - C[c.be_lo];
    if (ns > CAP || ne > CAP) c.status = 1;
  }
  pc[col] = c;
}

// 4. gather candidate-end elements and sum, in double-double, the elements strictly between the
//    two gathered bucket ranges' lower ends: K = sum over buckets [bs_lo, be_lo).  The window sum of
//    start s is then K + (first s + h - ce_lo sorted E elements) - (first s - cs_lo sorted S elements):
//    every window sum shares the same K, so elements below bs_lo never need to be summed.
__global__ void __launch_bounds__(PT) k_pr_gather(const double* __restrict__ cols, long long len,
                                                  const PrunedCol* __restrict__ pc, double* __restrict__ g,
                                                  int* __restrict__ gcount, dd2* __restrict__ below) {
  __shared__ dd2 sm[33];
  const int col = blockIdx.y;
  const PrunedCol c = pc[col];
  if (c.status) return;
  const double* y = cols + (long long)col * len;
  double* S = g + (long long)(2 * col) * CAP;
  double* E = g + (long long)(2 * col + 1) * CAP;
  ddacc acc = ddacc_zero();
  const long long per = (len + PCTA - 1) / PCTA;
  const long long i0 = blockIdx.x * per, i1 = min(len, i0 + per);
  for (long long base = i0 + threadIdx.x; base < i1; base += (long long)PT * ILP) {
    double v[ILP];
#pragma unroll
    for (int k = 0; k < ILP; k++) {
      const long long i = base + (long long)k * PT;
      v[k] = i < i1 ? __ldg(y + i) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < ILP; k++) {
      if (base + (long long)k * PT >= i1) continue;
      const int b = bucket_of(v[k], c);
      if (b >= c.bs_lo && b < c.be_lo) ddacc_add(acc, v[k]);
      if (b >= c.bs_lo && b <= c.bs_hi) {
        const int pos = atomicAdd(&gcount[2 * col], 1);
        if (pos < CAP) S[pos] = v[k];
      }
      if (b >= c.be_lo && b <= c.be_hi) {
        const int pos = atomicAdd(&gcount[2 * col + 1], 1);
        if (pos < CAP) E[pos] = v[k];
      }
    }
  }
  dd2 te = block_sum_dd2(ddacc_dd2(acc), sm);
  if (threadIdx.x == 0) {
    below[((long long)col * PCTA + blockIdx.x) * 2] = dd2_zero();
    below[((long long)col * PCTA + blockIdx.x) * 2 + 1] = te;
  }
}

__global__ void k_pr_segs(const int* __restrict__ gcount, int nseg, int* __restrict__ sbeg, int* __restrict__ send) {
  for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
    sbeg[i] = i * CAP;
    send[i] = i * CAP + min(gcount[i], CAP);
  }
}

// 5a. double-double prefix sums of each sorted gathered segment (one CTA per segment)
__device__ void prefix_body(const double* v, int cn, int col, int side, const dd2* __restrict__ below,
                            dd2* __restrict__ P) {
  __shared__ dd2 sm[33];
  __shared__ dd2 base;
  const int t = threadIdx.x;
  if (t == 0) {
    dd2 B = dd2_zero();
    for (int k = 0; k < PCTA; k++) B = dd2_add(B, below[((long long)col * PCTA + k) * 2 + side]);
    base = B;
  }
  __syncthreads();
  const int per = (cn + blockDim.x - 1) / blockDim.x;
  const int i0 = t * per, i1 = min(cn, i0 + per);
  dd2 loc = dd2_zero();
  for (int i = i0; i < i1; i++) loc = dd2_add(loc, dd2_of(v[i]));
  dd2 tot;
  dd2 ex = block_exscan_dd2(loc, &tot, sm);
  ex = dd2_add(base, ex);
  for (int i = i0; i < i1; i++) {
    P[i] = ex;
    ex = dd2_add(ex, dd2_of(v[i]));
  }
  if (t == 0) P[cn] = dd2_add(base, tot);
}

__global__ void __launch_bounds__(1024) k_pr_prefix(const PrunedCol* __restrict__ pc, const double* __restrict__ gsorted,
                                                    const int* __restrict__ gcount, const dd2* __restrict__ below,
                                                    dd2* __restrict__ pref) {
  const int seg = blockIdx.x, col = seg >> 1, side = seg & 1;
  if (pc[col].status) return;
  const int cn = min(gcount[seg], CAP);
  prefix_body(gsorted + (long long)seg * CAP, cn, col, side, below, pref + (long long)seg * (CAP + 1));
}

// 5a'. the common case, every gathered segment holding at most SMAX elements: sort the segment in
//      shared memory (bitonic) and take its prefix sums in the same CTA (replaces the segmented radix
//      sort's passes and the separate prefix launch)
static constexpr int SMAX = 16384;
__global__ void __launch_bounds__(1024) k_pr_sortprefix(const PrunedCol* __restrict__ pc, const double* __restrict__ g,
                                                        const int* __restrict__ gcount, const dd2* __restrict__ below,
                                                        dd2* __restrict__ pref) {
  extern __shared__ double sv[];
  const int seg = blockIdx.x, col = seg >> 1, side = seg & 1;
  if (pc[col].status) return;
  const int cn = min(gcount[seg], CAP);
  int np2 = 1;
  while (np2 < cn) np2 <<= 1;
  const double* src = g + (long long)seg * CAP;
  for (int i = threadIdx.x; i < np2; i += blockDim.x) sv[i] = i < cn ? src[i] : INFINITY;
  __syncthreads();
  smem_bitonic(sv, np2);
  prefix_body(sv, cn, col, side, below, pref + (long long)seg * (CAP + 1));
}

__device__ __forceinline__ bool win_better2(double ahi, double alo, long long as, double bhi, double blo, long long bs) {
  if (ahi != bhi) return ahi < bhi;
  if (alo != blo) return alo < blo;
  return as < bs;
}

struct WinBest {
  double vhi, vlo;
  long long s;
};

// 5b. exact objective of every candidate start; per-CTA best, grid (chunks, ncols)
__global__ void __launch_bounds__(PT) k_pr_eval(long long h, const PrunedCol* __restrict__ pc,
                                                const dd2* __restrict__ pref, WinBest* __restrict__ part, int nch) {
  __shared__ WinBest wb[PT / 32];
  const int col = blockIdx.y;
  const PrunedCol c = pc[col];
  if (c.status) return;
  const dd2* Ps = pref + (long long)(2 * col) * (CAP + 1);
  const dd2* Pe = pref + (long long)(2 * col + 1) * (CAP + 1);
  const double hd = (double)h;
  double bhi = INFINITY, blo = 0.0;
  long long bs = 0x7fffffffffffffffLL;
  for (long long s = c.smin + blockIdx.x * (long long)PT + threadIdx.x; s <= c.smax; s += (long long)gridDim.x * PT) {
    const dd2 Pl = Ps[s - c.cs_lo], Pr = Pe[s + h - c.ce_lo];
    dd S1 = dd_sub(Pr.s1, Pl.s1);
    dd S2 = dd_sub(Pr.s2, Pl.s2);
    dd v = dd_sub(dd_mul_d(S2, hd), dd_mul(S1, S1));
    if (win_better2(v.hi, v.lo, s, bhi, blo, bs)) {
      bhi = v.hi;
      blo = v.lo;
      bs = s;
    }
  }
  for (int d = 16; d > 0; d >>= 1) {
    double ohi = __shfl_down_sync(0xffffffffu, bhi, d);
    double olo = __shfl_down_sync(0xffffffffu, blo, d);
    long long os = __shfl_down_sync(0xffffffffu, bs, d);
    if (win_better2(ohi, olo, os, bhi, blo, bs)) {
      bhi = ohi;
      blo = olo;
      bs = os;
    }
  }
  if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = {bhi, blo, bs};
  __syncthreads();
  if (threadIdx.x == 0) {
    WinBest b = wb[0];
    for (int k = 1; k < PT / 32; k++)
      if (win_better2(wb[k].vhi, wb[k].vlo, wb[k].s, b.vhi, b.vlo, b.s)) b = wb[k];
    part[(long long)col * nch + blockIdx.x] = b;
  }
}

// 5c. argmin over chunks; raw location / variance
__global__ void k_pr_raw(long long h, const PrunedCol* __restrict__ pc, const dd2* __restrict__ pref,
                         const WinBest* __restrict__ part, int nch, UniConst uc, UniOut* __restrict__ out) {
  const int col = blockIdx.x;
  const PrunedCol c = pc[col];
  if (c.status || threadIdx.x != 0) return;
  WinBest b = part[(long long)col * nch];
  for (int k = 1; k < nch; k++) {
    const WinBest o = part[(long long)col * nch + k];
    if (win_better2(o.vhi, o.vlo, o.s, b.vhi, b.vlo, b.s)) b = o;
  }
  const dd2* Ps = pref + (long long)(2 * col) * (CAP + 1);
  const dd2* Pe = pref + (long long)(2 * col + 1) * (CAP + 1);
  const long long s = b.s;
  const dd2 Pl = Ps[s - c.cs_lo], Pr = Pe[s + h - c.ce_lo];
  const dd S1 = dd_sub(Pr.s1, Pl.s1);
  const double hd = (double)h;
  UniOut o;
  memset(&o, 0, sizeof(o));
  o.start = s;
  o.raw_loc = dd_to_d(dd_div_d(S1, hd));
  const dd v = {b.vhi, b.vlo};
  o.raw_var = h > 1 ? dd_to_d(dd_div_d(dd_div_d(v, hd), (double)(h - 1))) : 0.0;
  o.var0 = uc.c_raw * o.raw_var;
  o.status = o.var0 > 0.0 ? 0 : 1;
  out[col] = o;
}

// 6. reweighting sums over kept points (fixed-order per-CTA partials)
__global__ void __launch_bounds__(PT) k_pr_keep(const double* __restrict__ cols, long long len, UniConst uc,
                                                const UniOut* __restrict__ out, dd2* __restrict__ part,
                                                long long* __restrict__ kcnt) {
  __shared__ dd2 sm[33];
  __shared__ long long kc[PT / 32];
  const int col = blockIdx.y;
  const UniOut o = out[col];
  const double* y = cols + (long long)col * len;
  const double loc0 = o.raw_loc, thresh = uc.q1 * o.var0;
  const long long per = (len + PCTA - 1) / PCTA;
  const long long i0 = blockIdx.x * per, i1 = min(len, i0 + per);
  ddacc acc = ddacc_zero();
  long long k = 0;
  for (long long base = i0 + threadIdx.x; base < i1; base += (long long)PT * ILP) {
    double v[ILP];
#pragma unroll
    for (int u = 0; u < ILP; u++) {
      const long long i = base + (long long)u * PT;
      v[u] = i < i1 ? __ldg(y + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < ILP; u++) {
      if (base + (long long)u * PT >= i1) continue;
      const double d = __dsub_rn(v[u], loc0);
      if (__dmul_rn(d, d) <= thresh) {
        ddacc_add_dev(acc, v[u], d);
        k++;
      }
    }
  }
  dd2 tot = block_sum_dd2(ddacc_dd2(acc), sm);
  for (int d = 16; d > 0; d >>= 1) k += __shfl_down_sync(0xffffffffu, k, d);
  if ((threadIdx.x & 31) == 0) kc[threadIdx.x >> 5] = k;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long kt = 0;
    for (int q = 0; q < PT / 32; q++) kt += kc[q];
    part[(long long)col * PCTA + blockIdx.x] = tot;
    kcnt[(long long)col * PCTA + blockIdx.x] = kt;
  }
}

__global__ void k_pr_final(UniConst uc, const dd2* __restrict__ part, const long long* __restrict__ kcnt,
                           UniOut* __restrict__ out) {
  const int col = blockIdx.x;
  if (threadIdx.x != 0) return;
  UniOut o = out[col];
  dd2 K = dd2_zero();
  long long k = 0;
  for (int q = 0; q < PCTA; q++) {
    K = dd2_add(K, part[(long long)col * PCTA + q]);
    k += kcnt[(long long)col * PCTA + q];
  }
  o.kept = k;
  if (o.status || k < 2) {
    o.status = 1;
  } else {
    const double Sd = dd_to_d(K.s1);
    const double loc = Sd / (double)k;
    const dd q = kept_sq_about_loc(K, o.raw_loc, loc, (double)k);
    const double var = uc.c_rew * (dd_to_d(q) / (double)(k - 1));
    o.loc = loc;
    o.scale = sqrt(var);
    if (!(var > 0.0)) o.status = 1;
  }
  out[col] = o;
}

struct PrScratch {
  PrunedCol* pc;
  int* cnt;
  unsigned long long* tq;  // fixed-point offset sums per bucket
  double* esum;            // under- / overflow bucket sums and sums of magnitudes [col][4]
  double* sbb;             // [col][lo | hi] bucket sum intervals
  unsigned long long* mm;
  double *g, *gsorted;
  int* gcount;
  int *sbeg, *send;
  dd2* below;
  dd2* pref;
  WinBest* part;
  dd2* kpart;
  long long* kcnt;
  void* cub_tmp;
  size_t cub_bytes;
  int nch;
  long long* C;
  double *A1, *Q2lo, *Q2hi, *ub_part, *best_ub;
  BucketScan* bsc;
  long long* range_part;
  long long* crange;
  int nbound;
};

static size_t seg_sort_bytes(int nseg) {
  size_t b = 0;
  cub::DeviceSegmentedRadixSort::SortKeys(nullptr, b, (const double*)nullptr, (double*)nullptr, nseg * CAP, nseg,
                                          (const int*)nullptr, (const int*)nullptr);
  return b;
}

static void carve_pr(Arena& A, PrScratch& s, int ncols) {
  s.pc = A.take<PrunedCol>(ncols);
  s.cnt = A.take<int>((size_t)ncols * NBK);
  s.tq = A.take<unsigned long long>((size_t)ncols * NBK);
  s.esum = A.take<double>((size_t)ncols * 4);
  s.sbb = A.take<double>((size_t)ncols * 2 * NBK);
  s.mm = A.take<unsigned long long>(2 * (size_t)ncols);
  s.g = A.take<double>((size_t)2 * ncols * CAP);
  s.gsorted = A.take<double>((size_t)2 * ncols * CAP);
  s.gcount = A.take<int>(2 * (size_t)ncols);
  s.sbeg = A.take<int>(2 * (size_t)ncols);
  s.send = A.take<int>(2 * (size_t)ncols);
  s.below = A.take<dd2>((size_t)ncols * PCTA * 2);
  s.pref = A.take<dd2>((size_t)2 * ncols * (CAP + 1));
  s.nch = 16;
  s.part = A.take<WinBest>((size_t)ncols * s.nch);
  s.kpart = A.take<dd2>((size_t)ncols * PCTA);
  s.kcnt = A.take<long long>((size_t)ncols * PCTA);
  s.cub_bytes = seg_sort_bytes(2 * ncols);
  s.cub_tmp = A.take<char>(s.cub_bytes);
  s.C = A.take<long long>((size_t)ncols * (NBK + 1));
  s.A1 = A.take<double>((size_t)ncols * 2 * (NBK + 1));
  s.Q2lo = A.take<double>((size_t)ncols * (NBK + 1));
  s.Q2hi = A.take<double>((size_t)ncols * (NBK + 1));
  s.bsc = A.take<BucketScan>(ncols);
  s.nbound = std::max(1, 148 * 8 / ncols);
  s.ub_part = A.take<double>((size_t)ncols * s.nbound);
  s.best_ub = A.take<double>(ncols);
  s.range_part = A.take<long long>((size_t)ncols * s.nbound * 2);
  s.crange = A.take<long long>((size_t)ncols * 2);
}

// Returns true when every column was resolved by the pruned path (out_dev filled);
// false means the caller must run the full-sort path for this batch.
bool unimcd_pruned(Arena& A, cudaStream_t st, const double* cols, long long len, int ncols, UniConst uc,
                   UniOut* out_dev) {
  PrScratch s;
  carve_pr(A, s, ncols);
  if (A.base == nullptr) return true;  // dry run
  const long long h = len / 2 + 1;
  RTD_CU(cudaMemsetAsync(s.cnt, 0, (size_t)ncols * NBK * sizeof(int), st));
  RTD_CU(cudaMemsetAsync(s.tq, 0, (size_t)ncols * NBK * sizeof(unsigned long long), st));
  RTD_CU(cudaMemsetAsync(s.esum, 0, (size_t)ncols * 4 * sizeof(double), st));
  RTD_CU(cudaMemsetAsync(s.gcount, 0, 2 * (size_t)ncols * sizeof(int), st));
  k_pr_sample<<<ncols, 1024, 0, st>>>(cols, len, s.pc, s.mm);
  RTD_LAUNCHED();
  // ~64K elements per CTA: many CTAs per column so the 4-CTA/SM waves quantise finely (a CTA flushes its
  // 4096-bin histogram with global atomics, about 1/8 of its element count)
  const unsigned gx = (unsigned)std::max<long long>(1, (len + 65535) / 65536);  // <= 65536 elements per CTA
  k_pr_hist<<<dim3(gx, ncols), PT, 0, st>>>(cols, len, s.pc, s.cnt, s.tq, s.esum, s.mm);
  RTD_LAUNCHED();
  k_pr_scan<<<ncols, 1024, 0, st>>>(s.pc, s.cnt, s.tq, s.esum, s.mm, s.C, s.A1, s.Q2lo, s.Q2hi, s.sbb, s.bsc);
  RTD_LAUNCHED();
  for (int mode = 0; mode < 3; mode++) {
    k_pr_bound<<<dim3(s.nbound, ncols), PT, 0, st>>>(len, h, s.pc, s.cnt, s.sbb, s.C, s.A1, s.Q2lo, s.Q2hi, s.bsc,
                                                      mode, s.best_ub, s.crange, s.ub_part, s.range_part);
    RTD_LAUNCHED();
    if (mode == 0) k_pr_ubmin<<<ncols, 32, 0, st>>>(s.pc, s.ub_part, s.nbound, s.best_ub);
    else k_pr_range<<<ncols, 32, 0, st>>>(s.pc, s.range_part, s.nbound, s.crange);
    RTD_LAUNCHED();
  }
  k_pr_cand<<<ncols, 32, 0, st>>>(len, h, s.pc, s.C, s.crange);
  RTD_LAUNCHED();
  k_pr_gather<<<dim3(PCTA, ncols), PT, 0, st>>>(cols, len, s.pc, s.g, s.gcount, s.below);
  RTD_LAUNCHED();
  std::vector<PrunedCol> hc(ncols);
  std::vector<int> gc(2 * ncols);
  fetch(st, {{hc.data(), s.pc, ncols * sizeof(PrunedCol)}, {gc.data(), s.gcount, 2 * ncols * sizeof(int)}});
  static const bool dbg = getenv("RTD_DEBUG_PRUNED") != nullptr;
  if (dbg) {
    for (int j = 0; j < ncols; j++)
      fprintf(stderr, "pruned len=%lld col=%d status=%d s=[%lld,%lld] bs=[%d,%d] be=[%d,%d] span=%g\n", len, j,
              hc[j].status, hc[j].smin, hc[j].smax, hc[j].bs_lo, hc[j].bs_hi, hc[j].be_lo, hc[j].be_hi,
              hc[j].hi - hc[j].lo);
  }
  for (int j = 0; j < ncols; j++)
    if (hc[j].status) return false;
  int gmax = 0;
  for (int v : gc) gmax = std::max(gmax, v);
  if (gmax <= SMAX) {
    static const int smem = [] {
      cudaFuncSetAttribute(k_pr_sortprefix, cudaFuncAttributeMaxDynamicSharedMemorySize, SMAX * (int)sizeof(double));
      return SMAX * (int)sizeof(double);
    }();
    int np2 = 1;
    while (np2 < gmax) np2 <<= 1;
    k_pr_sortprefix<<<2 * ncols, 1024, std::min(smem, np2 * (int)sizeof(double)), st>>>(s.pc, s.g, s.gcount, s.below,
                                                                                         s.pref);
    RTD_LAUNCHED();
  } else {
    k_pr_segs<<<1, 256, 0, st>>>(s.gcount, 2 * ncols, s.sbeg, s.send);
    RTD_LAUNCHED();
    size_t bytes = s.cub_bytes;
    count_sort();
    RTD_CU(cub::DeviceSegmentedRadixSort::SortKeys(s.cub_tmp, bytes, s.g, s.gsorted, 2 * ncols * CAP, 2 * ncols,
                                                   s.sbeg, s.send, 0, 64, st));
    k_pr_prefix<<<2 * ncols, 1024, 0, st>>>(s.pc, s.gsorted, s.gcount, s.below, s.pref);
    RTD_LAUNCHED();
  }
  k_pr_eval<<<dim3(s.nch, ncols), PT, 0, st>>>(h, s.pc, s.pref, s.part, s.nch);
  RTD_LAUNCHED();
  k_pr_raw<<<ncols, 32, 0, st>>>(h, s.pc, s.pref, s.part, s.nch, uc, out_dev);
  RTD_LAUNCHED();
  k_pr_keep<<<dim3(PCTA, ncols), PT, 0, st>>>(cols, len, uc, out_dev, s.kpart, s.kcnt);
  RTD_LAUNCHED();
  k_pr_final<<<ncols, 32, 0, st>>>(uc, s.kpart, s.kcnt, out_dev);
  RTD_LAUNCHED();
  return true;
}

}  // namespace rtd
