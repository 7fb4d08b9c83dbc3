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
//   5. the gathered sets are sorted (shared-memory bitonic chunks + merge path), prefix-summed in
//      double-double, and h*SQ(s) is evaluated exactly for every candidate s:
//      argmin, ties -> lowest s (reading R2);
//   6. one pass sums the kept points of the reweighting step (reading R4).  Optional (RTD_UNI_FUSEDKEEP):
//      fused into pass 4 -- the raw fit is bracketed by the bounds of step 3, so the values certainly kept
//      are summed there and only the two narrow bands around the kept interval's ends are gathered and
//      decided once the raw fit is known (k_pr_final_fused); measured slower (FP64-bound), off by default.
// A column whose candidate sets do not fit (massive ties, extreme shapes)
// makes the caller fall back to the full radix-sort path (same result).
#include <cstdio>
#include <cstdlib>


#include "rtd_internal.h"

namespace rtd {

static constexpr int NBK = 4096;         // buckets per column (incl. underflow 0 and overflow NBK-1)
static constexpr int SAMPLE = 2048;      // strided sample for the bucket map
static constexpr int CAP = 65536;        // max gathered elements per side per column
static constexpr int PCTA = 32;          // max CTAs per column in the streaming passes (stride of the partials)
static constexpr long long PACK_LEN = 1LL << 24;  // below: hist flushes count + offset sum in one 64-bit atomic
static constexpr int PT = 256;
static constexpr int LT = 512;    // k_pr_locate threads (one CTA per column)

struct PrunedCol {
  double lo, hi, w, inv_w;   // bucket map
  double inv_w16;            // 2^16 inv_w (exact): fl(fl(y - lo) inv_w16) = 2^16 fl(fl(y - lo) inv_w)
  double cs;                 // shift of every bound: the bounds work on y - cs (cs = centre of the map)
  double los, his;           // lo - cs, hi - cs (rounded down / up)
  double cmin, cmax;         // column min / max, minus cs (rounded down / up)
  long long smin, smax;      // candidate window starts
  long long rmin, rmax;      // range of starts left by the chunk lower bounds (diagnostics)
  double tS0, tS1, tE0, tE1; // value thresholds of the gathered bucket ranges (bucket_threshold)
  int bs_lo, bs_hi, be_lo, be_hi;  // gathered bucket ranges (start side / end side)
  long long cs_lo, ce_lo;    // C[bs_lo], C[be_lo]
  int status;                // 0 ok, 1 fall back
  int kfused;                // 1: the reweighting sums are taken in the gather pass (step 6 fused into 4)
  double kc;                 // shift of the fused reweighting sums (centre of the raw location's interval)
  double kin_lo, kin_hi;     // values certainly kept by the reweighting, whatever the exact raw fit
  double kout_lo, kout_hi;   // outside [kout_lo, kout_hi]: certainly dropped; between: decided in k_pr_final
};

__device__ __forceinline__ int bucket_of(double y, const PrunedCol& c) {
  if (y < c.lo) return 0;
  if (y >= c.hi) return NBK - 1;
  double t = __dmul_rn(__dsub_rn(y, c.lo), c.inv_w);
  int b = 1 + (int)t;
  return b > NBK - 2 ? NBK - 2 : b;
}

// value range of bucket b, minus cs (fuzzed by 1e-6 bucket widths against rounding in bucket_of).  The
// bounds of k_pr_locate all work on y - cs: h SQ(s) is shift-invariant, and bounds on (sum y)^2 taken in
// raw units lose 2 |sum y| x (their width), i.e. nothing prunes once |mean| >> scale
__device__ __forceinline__ double bucket_lo(int b, const PrunedCol& c) {
  return b == 0 ? c.cmin : (b == NBK - 1 ? c.his : c.los + ((double)(b - 1) - 1e-6) * c.w);
}
__device__ __forceinline__ double bucket_hi(int b, const PrunedCol& c) {
  return b == 0 ? c.los : (b == NBK - 1 ? c.cmax : c.los + ((double)b + 1e-6) * c.w);
}

__device__ __forceinline__ unsigned long long ord_key(double x) {
  unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
  unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// Smallest double y with bucket_of(y) >= b (bucket_of is monotone in y), searched over the ordered bit
// patterns: y >= bucket_threshold(b) <=> bucket_of(y) >= b, so the streaming passes can test bucket ranges
// with two compares.  A gallop from the bucket's nominal lower end lo + (b - 1) w brackets the boundary
// within a few ulps (it is off by the rounding of bucket_of only), then bisection; the bracket is clamped to
// [-inf, inf], so any column is handled (a plain bisection over all 2^64 patterns took 64 serial steps).
__device__ double bucket_threshold(int b, const PrunedCol& c) {
  if (b <= 0) return -INFINITY;
  if (b >= NBK) return INFINITY;
  const unsigned long long kmin = ord_key(-INFINITY), kmax = ord_key(INFINITY);  // bucket_of(inf) = NBK - 1 >= b
  const double y0 = b == NBK - 1 ? c.hi : c.lo + (double)(b - 1) * c.w;
  const unsigned long long k0 = isfinite(y0) ? ord_key(y0) : kmax;
  unsigned long long lo, hi;  // invariant: bucket_of(lo) < b <= bucket_of(hi), or lo = kmin - 1 (none below)
  if (bucket_of(ord_val(k0), c) >= b) {
    hi = k0;
    unsigned long long step = 1;
    for (;;) {
      const unsigned long long k = hi - kmin > step ? hi - step : kmin;
      if (bucket_of(ord_val(k), c) < b) {
        lo = k;
        break;
      }
      hi = k;
      if (k == kmin) return ord_val(kmin);
      step <<= 1;
    }
  } else {
    lo = k0;
    unsigned long long step = 1;
    for (;;) {
      const unsigned long long k = kmax - lo > step ? lo + step : kmax;
      if (bucket_of(ord_val(k), c) >= b) {
        hi = k;
        break;
      }
      lo = k;
      step <<= 1;
    }
  }
  while (hi - lo > 1) {
    const unsigned long long mid = lo + (hi - lo) / 2;
    if (bucket_of(ord_val(mid), c) >= b) hi = mid; else lo = mid;
  }
  return ord_val(hi);
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

// in-place bitonic sort of a power-of-two shared array; every thread takes whole compare-exchange pairs
// (pair p -> element i = p with a zero bit inserted at log2(j), partner i | j), none idles in a stage
__device__ void smem_bitonic(double* a, int npow2) {
  const int half = npow2 >> 1;
  for (int k = 2; k <= npow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int pr = threadIdx.x; pr < half; pr += blockDim.x) {
        const int i = ((pr & ~(j - 1)) << 1) | (pr & (j - 1)), ixj = i | j;
        const bool up = (i & k) == 0;
        const double x = a[i], y = a[ixj];
        if ((x > y) == up) {
          a[i] = y;
          a[ixj] = x;
        }
      }
      __syncthreads();
    }
  }
}

// 1. bucket map from a strided sample
__global__ void __launch_bounds__(1024) k_pr_sample(const double* __restrict__ cols, long long len,
                                                    PrunedCol* __restrict__ pc, unsigned long long* __restrict__ mm) {
  __shared__ unsigned s[2 * 4096];  // block_quantile_keys2's two histograms
  const int col = blockIdx.x;
  const double* y = cols + (long long)col * len;
  constexpr int V = SAMPLE / 1024;  // blockDim.x == 1024: the in-register network (common.cuh)
  unsigned long long x[V];
#pragma unroll
  for (int k = 0; k < V; k++) {
    const double v = y[(long long)(threadIdx.x * V + k) * len / SAMPLE];
    x[k] = v == v ? ord_key64(v) : ~0ull;
  }
  // the sample's [0.5%, 99.5%] quantiles to 12 mantissa bits (routing only; block_quantile_keys2)
  __shared__ unsigned long long qk[2];
  block_quantile_keys2<V>(x, SAMPLE / 200, SAMPLE - 1 - SAMPLE / 200, s, qk);
  if (threadIdx.x == 0) {
    PrunedCol c;
    memset(&c, 0, sizeof(c));
    double ql = ord_val64(qk[0]), qh = ord_val64(qk[1]);
    double span = qh - ql;
    c.lo = ql - 0.05 * span;
    c.hi = qh + 0.05 * span;
    c.w = (c.hi - c.lo) / (double)(NBK - 2);
    c.inv_w = 1.0 / c.w;
    c.inv_w16 = c.inv_w * 65536.0;
    c.cs = 0.5 * (c.lo + c.hi);
    c.los = __dsub_rd(c.lo, c.cs);
    c.his = __dsub_ru(c.hi, c.cs);
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
__global__ void __launch_bounds__(PT, 5) k_pr_hist(const double* __restrict__ cols, long long len,
                                                const PrunedCol* __restrict__ pc, int* __restrict__ cnt,
                                                unsigned long long* __restrict__ tq, double* __restrict__ esum,
                                                unsigned long long* __restrict__ mm) {
  // (a packed 64-bit count + offset atomic would be a CAS loop in shared memory: two native 32-bit ones)
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
  // bucket_of and the offset in one product: T = floor(2^16 t), t = fl(fl(y - lo) inv_w), so
  // b = 1 + floor(t) = 1 + (T >> 16) and q = floor(2^16 frac(t)) = T & 0xffff.  The column min /
  // max only bound the end buckets' values (bucket_lo(0), bucket_hi(NBK - 1)): tracked there only
  auto consume = [&](const double x) {
    int b;
    if (x < c.lo) {
      b = 0;
      const double xs = __dsub_rn(x, c.cs);  // shifted (k_pr_locate): one more rounding per term
      e0 += xs;
      a0 += fabs(xs);
      kmin = min(kmin, ord_key(x));
    } else if (x >= c.hi) {
      b = NBK - 1;
      const double xs = __dsub_rn(x, c.cs);
      e1 += xs;
      a1 += fabs(xs);
      kmax = max(kmax, ord_key(x));
    } else {
      const int T = (int)__dmul_rn(__dsub_rn(x, c.lo), c.inv_w16);
      b = 1 + (T >> 16);
      unsigned int q = (unsigned int)(T & 0xffff);
      if (b > NBK - 2) {
        b = NBK - 2;
        q = 65535u;
      }
      atomicAdd(&hq[b], q);
    }
    atomicAdd(&hc[b], 1u);
  };
  // full tiles of ILP loads per thread without bounds tests, then one predicated tail tile
  const long long nfull = (i1 - i0) / ((long long)PT * ILP);
  const double* yp = y + i0 + threadIdx.x;
  for (long long it = 0; it < nfull; it++, yp += (long long)PT * ILP) {
    double v[ILP];
#pragma unroll
    for (int k = 0; k < ILP; k++) v[k] = __ldg(yp + k * PT);
#pragma unroll
    for (int k = 0; k < ILP; k++) consume(v[k]);
  }
  {
    const long long base = i0 + nfull * (long long)PT * ILP + threadIdx.x;
#pragma unroll
    for (int k = 0; k < ILP; k++)
      if (base + k * PT < i1) consume(__ldg(y + base + k * PT));
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
  const bool packed = len < PACK_LEN;  // count (bits 40..63) + offset sum (< len 2^16 <= 2^40) in one word
  for (int b = threadIdx.x; b < NBK; b += PT) {
    if (hc[b]) {
      if (packed) {
        atomicAdd(&tqc[b], ((unsigned long long)hc[b] << 40) | (unsigned long long)hq[b]);
      } else {
        atomicAdd(&cn[b], (int)hc[b]);
        if (hq[b]) atomicAdd(&tqc[b], (unsigned long long)hq[b]);
      }
    }
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
    // an fp64 sum of r terms y - cs (each rounded: u |y - cs|) in any order is within (r + 3) u sum|y - cs|
    // of the exact sum (u = 2^-53; the sum of magnitudes itself carries a relative error below (r + 2) u,
    // hence the factor 2 on (r + 2))
    const double S = es[b == 0 ? 0 : 1], Sa = es[b == 0 ? 2 : 3];
    const double err = 2.0 * ((double)r + 2.0) * 0x1p-53 * Sa + 1e-300;
    Slo = S - err;
    Shi = S + err;
  } else {
    const double rd = (double)r, Lb = c.los + (double)(b - 1) * c.w, u = c.w * (1.0 / 65536.0);
    Slo = fmax(rd * bucket_lo(b, c), rd * Lb + u * ((double)T - rd));
    Shi = fmin(rd * bucket_hi(b, c), rd * Lb + u * ((double)T + 2.0 * rd));
  }
}

__device__ __forceinline__ void scan_column(PrunedCol& c, bool packed, const int* __restrict__ cn,
                                            const unsigned long long* __restrict__ tqc,
                                            const double* __restrict__ es, long long* C, double* sblo, double* A1lo,
                                            double* Q2lo, double* Q2hi, BucketScan& bs) {
  __shared__ double red_d[32];
  __shared__ long long wc[32];
  __shared__ double w1[32], wh[32], wlo[32], whi[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  double* sbhi = sblo + NBK;
  double* A1hi = A1lo + (NBK + 1);
  constexpr int per = NBK / LT, NW = LT / 32;
  double slo[per], shi[per], qlo[per], qhi[per];
  int rr[per];
  long long lc = 0;
  double l1 = 0.0, lh = 0.0, llo = 0.0, lhi = 0.0, abs1 = 0.0;
#pragma unroll
  for (int e = 0; e < per; e++) {
    const int b = t * per + e;
    const unsigned long long tw = tqc[b];
    const int r = packed ? (int)(tw >> 40) : cn[b];
    rr[e] = r;
    bucket_sum_interval(b, r, packed ? (tw & ((1ull << 40) - 1ull)) : tw, es, c, slo[e], shi[e]);
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
    const bool in = lane < NW;
    long long vc = in ? wc[lane] : 0;
    double v1 = in ? w1[lane] : 0.0, vh = in ? wh[lane] : 0.0, vlo = in ? wlo[lane] : 0.0, vhi = in ? whi[lane] : 0.0;
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
    ec += rr[e];
    e1 += slo[e];
    eh += shi[e];
    elo += qlo[e];
    ehi += qhi[e];
  }
  if (t == LT - 1) {
    C[NBK] = ec;
    A1lo[NBK] = e1;
    A1hi[NBK] = eh;
    Q2lo[NBK] = elo;
    Q2hi[NBK] = ehi;
  }
  for (int d = 16; d > 0; d >>= 1) abs1 += __shfl_down_sync(0xffffffffu, abs1, d);
  if (lane == 0) red_d[w] = abs1;
  __syncthreads();
  if (t == LT - 1) {
    double tot_abs1 = 0.0;
    for (int k = 0; k < NW; k++) tot_abs1 += red_d[k];
    bs = {1e-10 * (tot_abs1 + 1e-300), 1e-10 * (fabs(ehi) + 1e-300)};
  }
  __syncthreads();
}

// bounds on h*SQ(s) for one start s (start bucket b, end bucket be)
struct VBound {
  double lo, hi;
};

// the per-run part of window_bounds: everything that depends on the start bucket b and the end
// bucket be only (a run of consecutive starts shares it)
struct RunConst {
  double L1, U1, L2, U2, mn1, mx1, mn2, mx2;
  double n1, n2, m1lo, Sbhi, Selo, m2hi;  // m1lo = Sblo / n1, m2hi = Sehi / n2
  double F1lo, F1hi, Q2l, Q2h;
  long long Cb1, Cbe;                     // C[b + 1], C[be]
  bool same;
};

__device__ __forceinline__ RunConst run_const(int b, int be, const PrunedCol& c, const long long* C, const double* A1,
                                              const double* Q2lo, const double* Q2hi, const double* sb) {
  RunConst r;
  r.L1 = bucket_lo(b, c);
  r.U1 = bucket_hi(b, c);
  r.L2 = bucket_lo(be, c);
  r.U2 = bucket_hi(be, c);
  r.mx1 = fmax(r.L1 * r.L1, r.U1 * r.U1);
  r.mn1 = (r.L1 <= 0 && r.U1 >= 0) ? 0.0 : fmin(r.L1 * r.L1, r.U1 * r.U1);
  r.mx2 = fmax(r.L2 * r.L2, r.U2 * r.U2);
  r.mn2 = (r.L2 <= 0 && r.U2 >= 0) ? 0.0 : fmin(r.L2 * r.L2, r.U2 * r.U2);
  r.same = be == b;
  r.Cb1 = C[b + 1];
  r.Cbe = C[be];
  r.n1 = (double)(r.Cb1 - C[b]);
  r.n2 = (double)(C[be + 1] - r.Cbe);
  // bucket sums are intervals: sb[0..NBK) lower ends, sb[NBK..2NBK) upper ends; A1 likewise
  r.m1lo = sb[b] * __drcp_rn(r.n1);
  r.Sbhi = sb[NBK + b];
  r.Selo = sb[be];
  r.m2hi = sb[NBK + be] * __drcp_rn(r.n2);
  r.F1lo = A1[be] - A1[b + 1];
  r.F1hi = A1[NBK + 1 + be] - A1[NBK + 1 + b + 1];
  r.Q2l = Q2lo[be] - Q2lo[b + 1];
  r.Q2h = Q2hi[be] - Q2hi[b + 1];
  return r;
}

// bounds on h*SQ(s) for one start s of the run
__device__ __forceinline__ VBound start_bounds(const RunConst& r, long long s, long long h, BucketScan m) {
  const double hd = (double)h;
  double lo1, hi1, lo2, hi2;
  if (r.same) {
    lo1 = hd * r.L1;
    hi1 = hd * r.U1;
    lo2 = hd * r.mn1;
    hi2 = hd * r.mx1;
  } else {
    const double r1 = (double)(r.Cb1 - s), r2 = (double)(s + h - r.Cbe);
    // top r1 elements of bucket b: mean >= bucket mean; the other n1 - r1 are >= L1
    const double t1lo = fmax(r1 * r.L1, r1 * r.m1lo), t1hi = fmin(r1 * r.U1, r.Sbhi - (r.n1 - r1) * r.L1);
    // bottom r2 elements of bucket be: mean <= bucket mean; the other n2 - r2 are <= U2
    const double t2lo = fmax(r2 * r.L2, r.Selo - (r.n2 - r2) * r.U2), t2hi = fmin(r2 * r.U2, r2 * r.m2hi);
    lo1 = r.F1lo + fmin(t1lo, t1hi) + fmin(t2lo, t2hi) - m.E1;
    hi1 = r.F1hi + fmax(t1lo, t1hi) + fmax(t2lo, t2hi) + m.E1;
    lo2 = r.Q2l + r1 * r.mn1 + r2 * r.mn2 - m.E2;
    hi2 = r.Q2h + r1 * r.mx1 + r2 * r.mx2 + m.E2;
  }
  const double sq_hi_1 = fmax(lo1 * lo1, hi1 * hi1);
  const double sq_lo_1 = (lo1 <= 0 && hi1 >= 0) ? 0.0 : fmin(lo1 * lo1, hi1 * hi1);
  const double slack = 1e-9 * (hd * fabs(hi2) + sq_hi_1) + 1e-300;
  return {hd * lo2 - sq_hi_1 - slack, hd * hi2 - sq_lo_1 + slack};
}

__device__ __forceinline__ VBound window_bounds(long long s, long long h, int b, int be, const PrunedCol& c,
                                                const long long* C, const double* A1, const double* Q2lo,
                                                const double* Q2hi, const double* sb, BucketScan m) {
  return start_bounds(run_const(b, be, c, C, A1, Q2lo, Q2hi, sb), s, h, m);
}

// k_pr_locate's rank -> bucket index: RT_N coarse cells of 2^sh ranks (sh in entry RT_N), cell k holding
// rank_bucket(k 2^sh); a query searches only between the buckets of its cell's two ends (a few instead of
// the 12 dependent shared-memory loads of a search over all NBK buckets -- the search was ~25 % of the
// kernel).  The table lives right after C in LocSmem: every caller passes LocSmem::C.
static constexpr int RT_N = 256;  // (LocSmem + static shared must stay within the 228 KB of an SM)
__device__ __forceinline__ int rank_bucket_full(const long long* C, long long r) {  // largest b with C[b] <= r
  int lo = 0, hi = NBK - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (C[mid] <= r) lo = mid; else hi = mid - 1;
  }
  return lo;
}
__device__ __forceinline__ int rank_bucket(const long long* C, long long r) {  // largest b with C[b] <= r
  const unsigned short* R = reinterpret_cast<const unsigned short*>(C + NBK + 1);
  const long long k = r >> R[RT_N];
  int lo = R[k], hi = k + 1 < RT_N ? R[k + 1] : NBK - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (C[mid] <= r) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Lower bound of h*SQ(s) valid for every s in [sa, sb] of one run (b != be): the partial sums of
// start_bounds are monotone in s (t1 decreases, t2 increases), so their extremes over the run come
// from its endpoints.
__device__ __forceinline__ double chunk_lower(const RunConst& r, long long sa, long long sb, long long h,
                                              BucketScan m) {
  const double hd = (double)h;
  double t1lo = INFINITY, t1hi = -INFINITY, t2lo = INFINITY, t2hi = -INFINITY, lo2 = INFINITY;
#pragma unroll
  for (int k = 0; k < 2; k++) {
    const long long s = k ? sb : sa;
    const double r1 = (double)(r.Cb1 - s), r2 = (double)(s + h - r.Cbe);
    const double a = fmax(r1 * r.L1, r1 * r.m1lo), bb = fmin(r1 * r.U1, r.Sbhi - (r.n1 - r1) * r.L1);
    const double d = fmax(r2 * r.L2, r.Selo - (r.n2 - r2) * r.U2), e = fmin(r2 * r.U2, r2 * r.m2hi);
    t1lo = fmin(t1lo, fmin(a, bb));
    t1hi = fmax(t1hi, fmax(a, bb));
    t2lo = fmin(t2lo, fmin(d, e));
    t2hi = fmax(t2hi, fmax(d, e));
    lo2 = fmin(lo2, r.Q2l + r1 * r.mn1 + r2 * r.mn2);
  }
  const double lo1 = r.F1lo + t1lo + t2lo - m.E1;
  const double hi1 = r.F1hi + t1hi + t2hi + m.E1;
  lo2 -= m.E2;
  const double sq_hi_1 = fmax(lo1 * lo1, hi1 * hi1);
  const double slack = 1e-9 * (hd * fabs(lo2) + sq_hi_1) + 1e-300;
  return hd * lo2 - sq_hi_1 - slack;
}

// Coarse lower bound of h*SQ(s) valid for every start s in [sa, sb], whose start buckets lie in
// [ba, bb] and end buckets in [ea, eb] (bb < ea): the window holds every element of buckets
// bb+1 .. ea-1, r1 = C[bb+1] - s elements with values in [L(ba), U(bb)] and r2 = h - r1 - n_mid
// elements with values in [L(ea), U(eb)]; all terms are linear in r1, so the endpoints bound them.
__device__ __forceinline__ double group_lower(long long sa, long long sb, long long h, int ba, int bb, int ea, int eb,
                                              const PrunedCol& c, const long long* C, const double* A1,
                                              const double* Q2lo, BucketScan m) {
  const double hd = (double)h;
  const double L1 = bucket_lo(ba, c), U1 = bucket_hi(bb, c), L2 = bucket_lo(ea, c), U2 = bucket_hi(eb, c);
  const double mn1 = (L1 <= 0 && U1 >= 0) ? 0.0 : fmin(L1 * L1, U1 * U1);
  const double mn2 = (L2 <= 0 && U2 >= 0) ? 0.0 : fmin(L2 * L2, U2 * U2);
  const double nmid = (double)(C[ea] - C[bb + 1]);
  const double F1lo = A1[ea] - A1[bb + 1], F1hi = A1[NBK + 1 + ea] - A1[NBK + 1 + bb + 1];
  const double Q2l = Q2lo[ea] - Q2lo[bb + 1];
  double lo1 = INFINITY, hi1 = -INFINITY, lo2 = INFINITY;
#pragma unroll
  for (int k = 0; k < 2; k++) {
    const double r1 = (double)(C[bb + 1] - (k ? sb : sa)), r2 = hd - r1 - nmid;
    lo1 = fmin(lo1, F1lo + r1 * L1 + r2 * L2);
    hi1 = fmax(hi1, F1hi + r1 * U1 + r2 * U2);
    lo2 = fmin(lo2, Q2l + r1 * mn1 + r2 * mn2);
  }
  lo1 -= m.E1;
  hi1 += m.E1;
  lo2 -= m.E2;
  const double sq_hi_1 = fmax(lo1 * lo1, hi1 * hi1);
  const double slack = 1e-9 * (hd * fabs(lo2) + sq_hi_1) + 1e-300;
  return hd * lo2 - sq_hi_1 - slack;
}

static constexpr int CHUNK = 64;      // starts per piece in the interval lower-bound pass
static constexpr int UB1 = 4096;      // strided starts of the first upper-bound sample (the second is LT)

struct LocSmem {  // one column's bucket prefix arrays (the layout of window_bounds' arguments)
  long long C[NBK + 1];
  unsigned short rt[RT_N + 4];  // rank_bucket's cell table (must follow C), rt[RT_N] = the cell shift
  double sb[2 * NBK];          // [lo | hi] bucket sum intervals
  double A1[2 * (NBK + 1)];    // [lo | hi] prefix sums of the bucket sums
  double Q2lo[NBK + 1], Q2hi[NBK + 1];
};
static constexpr int LOC_SMEM = (int)sizeof(LocSmem);

template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T* red) {
  for (int d = 16; d > 0; d >>= 1) v = op(v, __shfl_down_sync(0xffffffffu, v, d));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  v = red[0];
  for (int k = 1; k < LT / 32; k++) v = op(v, red[k]);
  return v;
}

// 3. one CTA per column, the column's prefix arrays in shared memory:
//    a. prefix arrays over buckets (scan_column);
//    b. the smallest upper bound of h*SQ(s) over a strided subset of starts (any subset bounds the minimum);
//    c. chunk lower bounds over all starts, one per maximal run of starts with the same start and end
//       buckets -> the range of starts whose chunk may hold the minimum;
//    d. per-start lower bounds inside that range -> the candidate range [smin, smax];
//    e. the gathered bucket ranges of the candidate window ends (k_pr_gather).
// bounds on the window sum S1(s) (the raw location is S1(s*) / h): the r1 largest elements of the start
// bucket are at least its mean, the r2 smallest of the end bucket at most its mean, the buckets between
// contribute their sum intervals
__device__ __forceinline__ void window_sum_bounds(long long s, long long h, const PrunedCol& c, const long long* C,
                                                  const double* A1, const double* sb, double E1, double& lo,
                                                  double& hi) {
  const int b = rank_bucket(C, s), be = rank_bucket(C, s + h - 1);
  const double hd = (double)h;
  if (b == be) {
    lo = hd * bucket_lo(b, c);
    hi = hd * bucket_hi(b, c);
    return;
  }
  const double r1 = (double)(C[b + 1] - s), r2 = (double)(s + h - C[be]);
  const double n1 = (double)(C[b + 1] - C[b]), n2 = (double)(C[be + 1] - C[be]);
  const double t1lo = fmax(r1 * bucket_lo(b, c), r1 * (sb[b] / n1)), t1hi = r1 * bucket_hi(b, c);
  const double t2lo = r2 * bucket_lo(be, c), t2hi = fmin(r2 * bucket_hi(be, c), r2 * (sb[NBK + be] / n2));
  lo = t1lo + (A1[be] - A1[b + 1]) + t2lo - E1;
  hi = t1hi + (A1[NBK + 1 + be] - A1[NBK + 1 + b + 1]) + t2hi + E1;
  const double pad = 1e-12 * (fabs(lo) + fabs(hi)) + 1e-300;  // rounding of these fp64 evaluations
  lo -= pad;
  hi += pad;
}

__global__ void __launch_bounds__(LT) k_pr_locate(long long len, long long h, PrunedCol* __restrict__ pc,
                                                  const int* __restrict__ cnt, const unsigned long long* __restrict__ tq,
                                                  const double* __restrict__ esum,
                                                  const unsigned long long* __restrict__ mm, UniConst uc) {
  extern __shared__ __align__(16) unsigned char loc_raw[];
  LocSmem& S = *reinterpret_cast<LocSmem*>(loc_raw);
  __shared__ BucketScan bs;
  __shared__ double redd[LT / 32];
  __shared__ long long redl[LT / 32];
  const int col = blockIdx.x;
  PrunedCol c = pc[col];
  if (c.status) return;
  c.cmin = __dsub_rd(ord_val(mm[2 * col]), c.cs);
  c.cmax = __dsub_ru(ord_val(mm[2 * col + 1]), c.cs);
  scan_column(c, len < PACK_LEN, cnt + (long long)col * NBK, tq + (long long)col * NBK, esum + 4 * col, S.C, S.sb, S.A1, S.Q2lo,
              S.Q2hi, bs);
  {  // rank_bucket's cell table (scan_column ended with a barrier: C is complete)
    int sh = 0;
    while (((long long)RT_N << sh) < len) sh++;
    for (int k = threadIdx.x; k < RT_N; k += LT) S.rt[k] = (unsigned short)rank_bucket_full(S.C, (long long)k << sh);
    if (threadIdx.x == 0) S.rt[RT_N] = (unsigned short)sh;
    __syncthreads();
  }
  const long long* C = S.C;
  const BucketScan m = bs;
  const long long nwin = len - h + 1;
  const int t = threadIdx.x;

  // b. the smallest upper bound over two strided sets of starts: UB1 starts across all of [0, nwin),
  //    then UB2 starts at 1/16 of that spacing around the best of them (any subset of starts gives a
  //    valid upper bound on the minimum; the second set makes it as tight near the optimum as a
  //    16x denser global sampling)
  __shared__ double bestv[LT / 32];
  __shared__ long long bests[LT / 32];
  __shared__ long long s_centre;
  const long long stride1 = std::max<long long>(1, (nwin + UB1 - 1) / UB1);
  double ub = INFINITY;
  long long ubs = 0;
  for (long long k = t; k * stride1 < nwin; k += LT) {
    const long long s = k * stride1;
    const double v = window_bounds(s, h, rank_bucket(C, s), rank_bucket(C, s + h - 1), c, C, S.A1, S.Q2lo, S.Q2hi,
                                   S.sb, m).hi;
    if (v < ub) {
      ub = v;
      ubs = s;
    }
  }
  for (int d = 16; d > 0; d >>= 1) {
    const double ov = __shfl_down_sync(0xffffffffu, ub, d);
    const long long os = __shfl_down_sync(0xffffffffu, ubs, d);
    if (ov < ub || (ov == ub && os < ubs)) {
      ub = ov;
      ubs = os;
    }
  }
  if ((t & 31) == 0) {
    bestv[t >> 5] = ub;
    bests[t >> 5] = ubs;
  }
  __syncthreads();
  if (t == 0) {
    double v = bestv[0];
    long long sc = bests[0];
    for (int k = 1; k < LT / 32; k++)
      if (bestv[k] < v) {
        v = bestv[k];
        sc = bests[k];
      }
    s_centre = sc;
  }
  __syncthreads();
  {
    const long long stride2 = std::max<long long>(1, stride1 / 16);
    const long long s = s_centre + ((long long)t - LT / 2) * stride2;
    if (s >= 0 && s < nwin)
      ub = fmin(ub, window_bounds(s, h, rank_bucket(C, s), rank_bucket(C, s + h - 1), c, C, S.A1, S.Q2lo, S.Q2hi,
                                  S.sb, m).hi);
  }
  const double bub = block_reduce(ub, [](double x, double y) { return fmin(x, y); }, redd);

  // c. interval lower bounds over all starts, in two levels: (c0) one coarse bound per group of
  //    NBK / LT start buckets (thread t: group t); (c1) the groups it does not exclude go round-robin
  //    to the warps, whose lanes split the group's starts and bound every piece of at most CHUNK
  //    starts of every run (same start and end bucket) in them, the run's constants once per run
  constexpr int GB = NBK / LT;
  __shared__ unsigned smask[LT / 32];
  {
    bool surv = false;
    const long long sa = min(C[t * GB], nwin), sb = min(C[(t + 1) * GB], nwin) - 1;
    if (sa <= sb) {
      const int ba = rank_bucket(C, sa), bb = rank_bucket(C, sb);
      const int ea = rank_bucket(C, sa + h - 1), eb = rank_bucket(C, sb + h - 1);
      surv = bb >= ea || group_lower(sa, sb, h, ba, bb, ea, eb, c, C, S.A1, S.Q2lo, m) <= bub;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, surv);
    if ((t & 31) == 0) smask[t >> 5] = bal;
    __syncthreads();
  }
  long long cmin = 0x7fffffffffffffffLL, cmax = -1;
  int ord = 0;  // ordinal of the surviving group: warp (ord mod LT/32) takes it, its lanes split the starts
  const int wid = t >> 5, ln = t & 31;
  for (int w = 0; w < LT / 32; w++) {
    unsigned mk = smask[w];
    while (mk) {
      const int gi = w * 32 + __ffs(mk) - 1;
      mk &= mk - 1;
      if ((ord++) % (LT / 32) != wid) continue;
      const long long ga = min(C[gi * GB], nwin), gb = min(C[(gi + 1) * GB], nwin);  // starts [ga, gb)
      const long long per = (gb - ga + 31) / 32;
      long long sa = ga + ln * per;
      const long long s1e = min(gb, sa + per);
      if (sa >= s1e) continue;
      int b = rank_bucket(C, sa), be = rank_bucket(C, sa + h - 1);
      while (sa < s1e) {
        while (C[b + 1] <= sa) b++;
        while (C[be + 1] <= sa + h - 1) be++;
        const long long re = min(min(s1e, C[b + 1]), C[be + 1] - h + 1) - 1;  // same (b, be) on [sa, re]
        if (b == be) {
          cmin = min(cmin, sa);
          cmax = max(cmax, re);
        } else {
          const RunConst rc = run_const(b, be, c, C, S.A1, S.Q2lo, S.Q2hi, S.sb);
          for (long long pa = sa; pa <= re;) {
            const long long pb = min(re, (pa / CHUNK + 1) * CHUNK - 1);
            if (chunk_lower(rc, pa, pb, h, m) <= bub) {
              cmin = min(cmin, pa);
              cmax = max(cmax, pb);
            }
            pa = pb + 1;
          }
        }
        sa = re + 1;
      }
    }
  }
  const long long lo_s = block_reduce(cmin, [](long long x, long long y) { return min(x, y); }, redl);
  const long long hi_s = block_reduce(cmax, [](long long x, long long y) { return max(x, y); }, redl);

  // d. per-start lower bounds inside [lo_s, hi_s]: the thread's contiguous range, run by run (and the
  //    smallest lower bound of a candidate: h SQ(s*) lies in [vmin, bub])
  cmin = 0x7fffffffffffffffLL;
  cmax = -1;
  double vmin = INFINITY;
  if (lo_s <= hi_s) {
    const long long cnt_s = hi_s - lo_s + 1;
    const long long per = (cnt_s + LT - 1) / LT;
    long long sa = lo_s + t * per;
    const long long s1e = min(hi_s + 1, sa + per);
    if (sa < s1e) {
      int b = rank_bucket(C, sa), be = rank_bucket(C, sa + h - 1);
      while (sa < s1e) {
        while (C[b + 1] <= sa) b++;
        while (C[be + 1] <= sa + h - 1) be++;
        const long long sb = min(min(s1e, C[b + 1]), C[be + 1] - h + 1) - 1;  // same (b, be) on [sa, sb]
        const RunConst rc = run_const(b, be, c, C, S.A1, S.Q2lo, S.Q2hi, S.sb);
        for (long long s = sa; s <= sb; s++) {
          const double lb = start_bounds(rc, s, h, m).lo;
          if (lb <= bub) {
            cmin = min(cmin, s);
            cmax = max(cmax, s);
            vmin = fmin(vmin, lb);
          }
        }
        sa = sb + 1;
      }
    }
  }
  const long long smin = block_reduce(cmin, [](long long x, long long y) { return min(x, y); }, redl);
  const long long smax = block_reduce(cmax, [](long long x, long long y) { return max(x, y); }, redl);
  const double vlb = block_reduce(vmin, [](double x, double y) { return fmin(x, y); }, redd);

  // e. gathered bucket ranges (warp 0: every lane derives the same fields, lanes 0-3 the four thresholds)
  if (t < 32) {
    c.smin = smin;
    c.smax = smax;
    c.rmin = lo_s;
    c.rmax = hi_s;
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
      const int tb = t == 0 ? c.bs_lo : (t == 1 ? c.bs_hi + 1 : (t == 2 ? c.be_lo : c.be_hi + 1));
      const double thr = t < 4 ? bucket_threshold(tb, c) : 0.0;
      c.tS0 = __shfl_sync(0xffffffffu, thr, 0);
      c.tS1 = __shfl_sync(0xffffffffu, thr, 1);
      c.tE0 = __shfl_sync(0xffffffffu, thr, 2);
      c.tE1 = __shfl_sync(0xffffffffu, thr, 3);
      // the reweighting step (reading R4) keeps x iff (x - loc0)^2 <= q1 var0; the
      // raw fit is not known yet, but loc0 = S1(s*) / h with s* in [smin, smax] (the window mean is
      // monotone in s) and h SQ(s*) in [vlb, bub] bound it: values well inside the kept interval for
      // every such (loc0, var0) are summed in the gather pass, values in the two narrow bands around its
      // ends are gathered and decided exactly once the raw fit is known
      double l0lo, l0hi, l1lo, l1hi;
      window_sum_bounds(smin, h, c, C, S.A1, S.sb, m.E1, l0lo, l0hi);
      window_sum_bounds(smax, h, c, C, S.A1, S.sb, m.E1, l1lo, l1hi);
      const double hd = (double)h;
      const double mlo = l0lo / hd + c.cs, mhi = l1hi / hd + c.cs;  // back to raw units
      const double vden = hd * (hd - 1.0);
      const double v0lo = uc.c_raw * vlb / vden * (1.0 - 1e-9), v0hi = uc.c_raw * bub / vden * (1.0 + 1e-9);
      const double Rlo = sqrt(uc.q1 * v0lo) * (1.0 - 1e-9), Rhi = sqrt(uc.q1 * v0hi) * (1.0 + 1e-9);
      const double eps = 1e-9 * (Rhi + fabs(mlo) + fabs(mhi));
      c.kc = 0.5 * (mlo + mhi);
      c.kin_lo = mhi - Rlo + eps;
      c.kin_hi = mlo + Rlo - eps;
      c.kout_lo = mlo - Rhi - eps;
      c.kout_hi = mhi + Rhi + eps;
      c.kfused = (vlb > 0.0 && isfinite(mlo) && isfinite(mhi) && isfinite(Rhi) && mlo <= mhi &&
                  c.kin_lo < c.kin_hi && (mhi - mlo) < 0.01 * Rlo && (Rhi - Rlo) < 0.01 * Rlo) ? 1 : 0;
    }
    if (t == 0) pc[col] = c;
  }
}

// 4. gather candidate-end elements and sum, in double-double, the elements strictly between the
//    two gathered bucket ranges' lower ends: K = sum over buckets [bs_lo, be_lo).  The window sum of
//    start s is then K + (first s + h - ce_lo sorted E elements) - (first s - cs_lo sorted S elements):
//    every window sum shares the same K, so elements below bs_lo never need to be summed.
static constexpr int GBUF = 1024;  // k_pr_gather: per-CTA shared buffer of gathered elements per side

static constexpr int BCAP = 65536;  // band elements of the fused reweighting per column

// FUSED: also the reweighting step's sums over the values certainly kept (kin_lo <= x <= kin_hi: sum x and
// sum (x - kc)^2, kc rounded away as in k_pr_keep) and the values of the two bands around the kept
// interval's ends, for k_pr_final_fused
template <bool FUSED>
__global__ void __launch_bounds__(PT, FUSED ? 4 : 5) k_pr_gather(const double* __restrict__ cols, long long len,
                                                  const PrunedCol* __restrict__ pc, double* __restrict__ g,
                                                  int* __restrict__ gcount, dd2* __restrict__ below,
                                                  double* __restrict__ band, int* __restrict__ bcount,
                                                  dd2* __restrict__ kpart, long long* __restrict__ kcnt) {
  __shared__ dd2 sm[33];
  __shared__ double sbuf[2][GBUF];  // this CTA's gathered elements, flushed with one global atomic per side
  __shared__ int scnt[2], sbase[2];
  const int col = blockIdx.y;
  const PrunedCol c = pc[col];
  if (c.status) return;
  const double* y = cols + (long long)col * len;
  double* S = g + (long long)(2 * col) * CAP;
  double* E = g + (long long)(2 * col + 1) * CAP;
  // K = (sum x, sum x^2) over [bs_lo, be_lo).  Every candidate's objective h S2 - S1^2 contains h K.s2 as
  // the same additive constant, so only K.s1 decides the argmin and is kept in double-double (two-sum,
  // error words collected); K.s2 only enters the raw variance and is taken as sum (x - cs)^2 in fp64
  // about the bucket map's centre cs (positive terms, relative error ~ sqrt(terms) u) plus the exact
  // shift 2 cs K.s1 - n cs^2 in double-double.  5 fp64 operations per element fewer than two full
  // double-double sums; the pass is otherwise limited by the fp64 pipe.
  constexpr int NACC = 2;  // independent accumulators: the two-sum chains of successive elements overlap
  double a1h[NACC], a1l[NACC], a2[NACC];
#pragma unroll
  for (int q = 0; q < NACC; q++) a1h[q] = a1l[q] = a2[q] = 0.0;
  int nmid = 0;
  const double cs = c.cs;
  // FUSED: sum d, sum d^2 of the certainly kept d = x - kc in fp64 per thread (as k_pr_keep)
  constexpr int NKA = FUSED ? 2 : 1;
  double ks1[NKA], ks2[NKA];
#pragma unroll
  for (int q = 0; q < NKA; q++) ks1[q] = ks2[q] = 0.0;
  long long kn = 0;
  __shared__ double bbuf[FUSED ? 512 : 1];
  __shared__ int bcnt_s, bbase_s;
  if (FUSED && threadIdx.x == 0) bcnt_s = 0;
  const long long per = (len + gridDim.x - 1) / gridDim.x;
  const long long i0 = blockIdx.x * per, i1 = min(len, i0 + per);
  const unsigned lane = threadIdx.x & 31, lt_mask = (1u << lane) - 1u;
  if (threadIdx.x < 2) scnt[threadIdx.x] = 0;
  __syncthreads();
  // streaming: ILP independent loads per thread in flight (plain registers; full tiles without bounds
  // tests, then one predicated tail tile whose slots past the range hold NaN, which fails every test)
  auto consume = [&](const double x, const int k) {
    // bucket ranges by value thresholds: bucket_of(y) in [b0, b1) <=> T(b0) <= y < T(b1)
    const bool geS = x >= c.tS0, geE = x >= c.tE0;
    const bool mid = geS && !geE;  // [bs_lo, be_lo); branch-free: adding 0 is exact
    {
      const int q = k % NACC;
      const double v = mid ? x : 0.0, dv = mid ? __dsub_rn(x, cs) : 0.0;
      const double sh = __dadd_rn(a1h[q], v), bb = __dsub_rn(sh, a1h[q]);
      a1l[q] = __dadd_rn(a1l[q], __dadd_rn(__dsub_rn(a1h[q], __dsub_rn(sh, bb)), __dsub_rn(v, bb)));
      a1h[q] = sh;
      a2[q] = __fma_rn(dv, dv, a2[q]);
      nmid += mid ? 1 : 0;
    }
    bool kin = false;
    if (FUSED) {
      kin = x >= c.kin_lo && x <= c.kin_hi;
      const double dk = kin ? __dsub_rn(x, c.kc) : 0.0;
      ks1[k % NKA] = __dadd_rn(ks1[k % NKA], dk);
      ks2[k % NKA] = __fma_rn(dk, dk, ks2[k % NKA]);
      kn += kin ? 1 : 0;
    }
    const bool inb = FUSED && !kin && x >= c.kout_lo && x <= c.kout_hi;
    const bool inS = geS && x < c.tS1, inE = geE && x < c.tE1;
    // one vote for both rare cases (band values of the fused reweighting, candidate window ends)
    if (!__any_sync(0xffffffffu, inS || inE || inb)) return;
    if (FUSED) {
      if (__any_sync(0xffffffffu, inb)) {  // rare: the bands hold ~1e-4 of the values
        const unsigned mb = __ballot_sync(0xffffffffu, inb);
        int pos = 0;
        if (lane == (unsigned)(__ffs(mb) - 1)) pos = atomicAdd(&bcnt_s, __popc(mb));
        pos = __shfl_sync(0xffffffffu, pos, __ffs(mb) - 1) + __popc(mb & lt_mask);
        if (inb) {
          if (pos < 512) {
            bbuf[pos] = x;
          } else {
            const int gp = atomicAdd(&bcount[col], 1);
            if (gp < BCAP) band[(long long)col * BCAP + gp] = x;
          }
        }
      }
    }
    if (!__any_sync(0xffffffffu, inS || inE)) return;
    const unsigned ms = __ballot_sync(0xffffffffu, inS), me = __ballot_sync(0xffffffffu, inE);
#pragma unroll
    for (int side = 0; side < 2; side++) {  // one shared atomic per warp and side
      const unsigned mm = side ? me : ms;
      if (mm) {
        const bool mine = side ? inE : inS;
        int pos = 0;
        if (lane == (unsigned)(__ffs(mm) - 1)) pos = atomicAdd(&scnt[side], __popc(mm));
        pos = __shfl_sync(0xffffffffu, pos, __ffs(mm) - 1) + __popc(mm & lt_mask);
        if (mine) {
          if (pos < GBUF) {
            sbuf[side][pos] = x;
          } else {  // CTA buffer full: straight to global memory
            const int gp = atomicAdd(&gcount[2 * col + side], 1);
            if (gp < CAP) (side ? E : S)[gp] = x;
          }
        }
      }
    }
  };
  const long long nfull = (i1 - i0) / ((long long)PT * ILP);
  const double* yp = y + i0 + threadIdx.x;
  for (long long it = 0; it < nfull; it++, yp += (long long)PT * ILP) {
    double v[ILP];
#pragma unroll
    for (int k = 0; k < ILP; k++) v[k] = __ldg(yp + k * PT);
#pragma unroll
    for (int k = 0; k < ILP; k++) consume(v[k], k);
  }
  if (i0 + nfull * (long long)PT * ILP < i1) {  // warp-uniform
    const long long base = i0 + nfull * (long long)PT * ILP + threadIdx.x;
    double v[ILP];
#pragma unroll
    for (int k = 0; k < ILP; k++)
      v[k] = base + k * PT < i1 ? __ldg(y + base + k * PT) : __longlong_as_double(0x7ff8000000000000LL);
#pragma unroll
    for (int k = 0; k < ILP; k++) consume(v[k], k);
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    const int n = min(scnt[threadIdx.x], GBUF);
    sbase[threadIdx.x] = n ? atomicAdd(&gcount[2 * col + threadIdx.x], n) : 0;
  }
  __syncthreads();
#pragma unroll
  for (int side = 0; side < 2; side++) {
    const int n = min(scnt[side], GBUF), b0 = sbase[side];
    double* dst = side ? E : S;
    for (int i = threadIdx.x; i < n; i += PT)
      if (b0 + i < CAP) dst[b0 + i] = sbuf[side][i];
  }
  dd K1 = two_sum(a1h[0], a1l[0]);
  double K2c = a2[0];
#pragma unroll
  for (int q = 1; q < NACC; q++) {
    K1 = dd_add(K1, two_sum(a1h[q], a1l[q]));
    K2c = __dadd_rn(K2c, a2[q]);
  }
  // sum x^2 = sum (x - cs)^2 + 2 cs sum x - n cs^2
  const dd K2 = dd_sub(dd_add(dd_make(K2c), dd_mul_d(K1, 2.0 * cs)), dd_mul_d(two_prod(cs, cs), (double)nmid));
  dd2 te = block_sum_dd2({K1, K2}, sm);
  if (threadIdx.x == 0) {
    below[((long long)col * PCTA + blockIdx.x) * 2] = dd2_zero();
    below[((long long)col * PCTA + blockIdx.x) * 2 + 1] = te;
  }
  if (FUSED) {
    __syncthreads();  // sm reused
    dd2 kt = {dd_make(ks1[0]), dd_make(ks2[0])};
#pragma unroll
    for (int q = 1; q < NKA; q++) kt = dd2_add(kt, {dd_make(ks1[q]), dd_make(ks2[q])});
    const dd2 ktot = block_sum_dd2(kt, sm);
    __shared__ long long kred[PT / 32];
    for (int d = 16; d > 0; d >>= 1) kn += __shfl_down_sync(0xffffffffu, kn, d);
    if (lane == 0) kred[threadIdx.x >> 5] = kn;
    if (threadIdx.x == 0) {
      const int nbl = min(bcnt_s, 512);
      bbase_s = nbl ? atomicAdd(&bcount[col], nbl) : 0;
    }
    __syncthreads();
    const int nbl = min(bcnt_s, 512);
    for (int i = threadIdx.x; i < nbl; i += PT)
      if (bbase_s + i < BCAP) band[(long long)col * BCAP + bbase_s + i] = bbuf[i];
    if (threadIdx.x == 0) {
      long long kt2 = 0;
      for (int q = 0; q < PT / 32; q++) kt2 += kred[q];
      kpart[(long long)col * PCTA + blockIdx.x] = ktot;
      kcnt[(long long)col * PCTA + blockIdx.x] = kt2;
    }
  }
}


// 5a. double-double prefix sums of each sorted gathered segment (one CTA per segment)
__device__ void prefix_body(const double* v, int cn, int col, int side, int npc, const dd2* __restrict__ below,
                            dd2* __restrict__ P) {
  __shared__ dd2 sm[33];
  __shared__ dd2 base;
  const int t = threadIdx.x;
  if (t == 0) {
    dd2 B = dd2_zero();
    for (int k = 0; k < npc; k++) B = dd2_add(B, below[((long long)col * PCTA + k) * 2 + side]);
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

__global__ void __launch_bounds__(1024) k_pr_prefix(int npc, const PrunedCol* __restrict__ pc, const double* __restrict__ gsorted,
                                                    const int* __restrict__ gcount, const dd2* __restrict__ below,
                                                    dd2* __restrict__ pref) {
  const int seg = blockIdx.x, col = seg >> 1, side = seg & 1;
  if (pc[col].status) return;
  const int cn = min(gcount[seg], CAP);
  prefix_body(gsorted + (long long)seg * CAP, cn, col, side, npc, below, pref + (long long)seg * (CAP + 1));
}

// 5a'. the common case, every gathered segment holding at most SMAX elements: sort the segment in
//      shared memory (bitonic) and take its prefix sums in the same CTA (replaces the segmented radix
//      sort's passes and the separate prefix launch)
static constexpr int SMAX = 16384;
__global__ void __launch_bounds__(1024) k_pr_sortprefix(int npc, const PrunedCol* __restrict__ pc, const double* __restrict__ g,
                                                        const int* __restrict__ gcount, const dd2* __restrict__ below,
                                                        dd2* __restrict__ pref, int cmin, int cmax) {
  extern __shared__ double sv[];
  const int seg = blockIdx.x, col = seg >> 1, side = seg & 1;
  if (pc[col].status) return;
  const int cn = min(gcount[seg], CAP);
  if (cn < cmin || cn > cmax) return;  // this launch's class of segment lengths
  int np2 = 1;
  while (np2 < cn) np2 <<= 1;
  const double* src = g + (long long)seg * CAP;
  for (int i = threadIdx.x; i < np2; i += blockDim.x) sv[i] = i < cn ? src[i] : INFINITY;
  __syncthreads();
  smem_bitonic(sv, np2);
  prefix_body(sv, cn, col, side, npc, below, pref + (long long)seg * (CAP + 1));
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

// 5a''. a segment longer than SMAX: chunks of SMAX sorted in shared memory in place, then merge
//       rounds (merge path, one CTA per pair of runs) ping-ponging between g and gsorted; the
//       final buffer feeds k_pr_prefix.  Equal values may interleave in either order: the prefix sums
//       at every rank are the same.
__global__ void __launch_bounds__(1024) k_pr_chunksort(const PrunedCol* __restrict__ pc, double* __restrict__ g,
                                                       const int* __restrict__ gcount) {
  extern __shared__ double sv[];
  const int seg = blockIdx.y, col = seg >> 1;
  if (pc[col].status) return;
  const int cn = min(gcount[seg], CAP), c0 = blockIdx.x * SMAX;
  if (c0 >= cn) return;
  const int n = min(SMAX, cn - c0);
  int np2 = 1;
  while (np2 < n) np2 <<= 1;
  double* src = g + (long long)seg * CAP + c0;
  for (int i = threadIdx.x; i < np2; i += blockDim.x) sv[i] = i < n ? src[i] : INFINITY;
  __syncthreads();
  smem_bitonic(sv, np2);
  for (int i = threadIdx.x; i < n; i += blockDim.x) src[i] = sv[i];
}

__global__ void __launch_bounds__(1024) k_pr_merge(const PrunedCol* __restrict__ pc, const double* __restrict__ src,
                                                   double* __restrict__ dst, const int* __restrict__ gcount, int w) {
  const int seg = blockIdx.y, col = seg >> 1;
  if (pc[col].status) return;
  const int cn = min(gcount[seg], CAP), a0 = blockIdx.x * 2 * w;
  if (a0 >= cn) return;
  const double* A = src + (long long)seg * CAP + a0;
  const double* B = A + w;
  const int na = min(w, cn - a0), nb = max(0, min(w, cn - a0 - w)), tot = na + nb;
  double* out = dst + (long long)seg * CAP + a0;
  const int K = (tot + blockDim.x - 1) / blockDim.x;
  const int d0 = min(tot, (int)threadIdx.x * K), d1 = min(tot, d0 + K);
  if (d0 >= d1) return;
  // i = elements of A among the first d0 outputs (A first on ties)
  int lo = max(0, d0 - nb), hi = min(d0, na);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A[mid] <= B[d0 - mid - 1]) lo = mid + 1; else hi = mid;
  }
  int ia = lo, ib = d0 - lo;
  for (int d = d0; d < d1; d++) {
    if (ib >= nb || (ia < na && A[ia] <= B[ib])) out[d] = A[ia++];
    else out[d] = B[ib++];
  }
}

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

// the reweighted fit from K = (sum d, sum d^2) over the k kept values, d = x - shift:
// loc = shift + sum d / k, sum (x - loc)^2 = sum d^2 - (sum d)^2 / k (reading R4)
__device__ __forceinline__ void reweighted_from_shifted(const UniConst& uc, const dd2& K, double shift, long long k,
                                                        UniOut& o) {
  o.kept = k;
  if (o.status || k < 2) {
    o.status = 1;
    return;
  }
  const double kd = (double)k;
  const dd D = dd_div_d(K.s1, kd);
  const double loc = dd_to_d(dd_add(dd_make(shift), D));
  const dd q = dd_sub(K.s2, dd_mul(D, K.s1));
  const double var = uc.c_rew * (dd_to_d(q) / (double)(k - 1));
  o.loc = loc;
  o.scale = sqrt(var);
  if (!(var > 0.0)) o.status = 1;
}

// a column whose reweighting sums were taken by the fused gather pass (kfused, band within BCAP)
__device__ __forceinline__ bool col_fused(const PrunedCol* pc, const int* bcount, int col) {
  return pc != nullptr && pc[col].kfused && bcount[col] <= BCAP;
}

// 6. reweighting sums over kept points (fixed-order per-CTA partials).  pc != nullptr: the gather pass ran
//    fused, and only the columns it could not take (col_fused false) are summed here
__global__ void __launch_bounds__(PT) k_pr_keep(const double* __restrict__ cols, long long len, UniConst uc,
                                                const UniOut* __restrict__ out, dd2* __restrict__ part,
                                                long long* __restrict__ kcnt, const PrunedCol* __restrict__ pc,
                                                const int* __restrict__ bcount) {
  __shared__ dd2 sm[33];
  __shared__ long long kc[PT / 32];
  const int col = blockIdx.y;
  if (col_fused(pc, bcount, col)) return;
  const UniOut o = out[col];
  const double* y = cols + (long long)col * len;
  const double loc0 = o.raw_loc, thresh = uc.q1 * o.var0;
  const long long per = (len + gridDim.x - 1) / gridDim.x;
  const long long i0 = blockIdx.x * per, i1 = min(len, i0 + per);
  // sum d and sum d^2 of the kept d = x - loc0 in fp64 per thread (ILP chains; d is centred, the squares
  // are positive: relative errors ~ sqrt(terms) u), folded over threads and CTAs in double-double
  constexpr int NKS = 2;
  double s1[NKS], s2[NKS];
#pragma unroll
  for (int u = 0; u < NKS; u++) s1[u] = s2[u] = 0.0;
  long long k = 0;
  for (long long base = i0 + threadIdx.x; base < i1; base += (long long)PT * ILP) {
    double v[ILP];
    const int rem = (int)min(i1 - base, (long long)PT * ILP);
#pragma unroll
    for (int u = 0; u < ILP; u++) v[u] = u * PT < rem ? __ldg(y + base + u * PT) : 0.0;
#pragma unroll
    for (int u = 0; u < ILP; u++) {
      if (u * PT >= rem) continue;
      const double d = __dsub_rn(v[u], loc0);
      const bool kept = __dmul_rn(d, d) <= thresh;
      const double dk = kept ? d : 0.0;
      s1[u % NKS] = __dadd_rn(s1[u % NKS], dk);
      s2[u % NKS] = __fma_rn(dk, dk, s2[u % NKS]);
      k += kept ? 1 : 0;
    }
  }
  dd2 t = {dd_make(s1[0]), dd_make(s2[0])};
#pragma unroll
  for (int u = 1; u < NKS; u++) t = dd2_add(t, {dd_make(s1[u]), dd_make(s2[u])});
  dd2 tot = block_sum_dd2(t, sm);
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

__global__ void k_pr_final(UniConst uc, int npc, const dd2* __restrict__ part, const long long* __restrict__ kcnt,
                           UniOut* __restrict__ out, const PrunedCol* __restrict__ pc, const int* __restrict__ bcount) {
  const int col = blockIdx.x;
  if (threadIdx.x != 0 || col_fused(pc, bcount, col)) return;
  UniOut o = out[col];
  dd2 K = dd2_zero();
  long long k = 0;
  for (int q = 0; q < npc; q++) {
    K = dd2_add(K, part[(long long)col * PCTA + q]);
    k += kcnt[(long long)col * PCTA + q];
  }
  reweighted_from_shifted(uc, K, o.raw_loc, k, o);
  out[col] = o;
}

// 6'. the fused reweighting: the certainly-kept sums of the gather pass (fixed order over its CTAs) plus
//     the band values that pass the exact test (x - loc0)^2 <= q1 var0 under the raw fit (reading R4),
//     all about the shift kc
__global__ void __launch_bounds__(PT) k_pr_final_fused(UniConst uc, int npc, const PrunedCol* __restrict__ pc,
                                                       const dd2* __restrict__ part, const long long* __restrict__ kcnt,
                                                       const double* __restrict__ band, const int* __restrict__ bcount,
                                                       UniOut* __restrict__ out) {
  __shared__ dd2 sm[33];
  __shared__ long long kred[PT / 32];
  const int col = blockIdx.x;
  if (!col_fused(pc, bcount, col)) return;  // summed by k_pr_keep / k_pr_final
  const PrunedCol c = pc[col];
  UniOut o = out[col];
  const double loc0 = o.raw_loc, thresh = uc.q1 * o.var0;
  const int nb = min(bcount[col], BCAP);
  double b1 = 0.0, b2 = 0.0;
  long long kb = 0;
  for (int i = threadIdx.x; i < nb; i += PT) {
    const double x = band[(long long)col * BCAP + i];
    const double d = __dsub_rn(x, loc0);
    if (__dmul_rn(d, d) <= thresh) {
      const double dk = __dsub_rn(x, c.kc);
      b1 = __dadd_rn(b1, dk);
      b2 = __fma_rn(dk, dk, b2);
      kb++;
    }
  }
  const dd2 btot = block_sum_dd2({dd_make(b1), dd_make(b2)}, sm);
  for (int d = 16; d > 0; d >>= 1) kb += __shfl_down_sync(0xffffffffu, kb, d);
  if ((threadIdx.x & 31) == 0) kred[threadIdx.x >> 5] = kb;
  __syncthreads();
  if (threadIdx.x != 0) return;
  dd2 K = dd2_zero();
  long long k = 0;
  for (int q = 0; q < npc; q++) {
    K = dd2_add(K, part[(long long)col * PCTA + q]);
    k += kcnt[(long long)col * PCTA + q];
  }
  K = dd2_add(K, btot);
  for (int q = 0; q < PT / 32; q++) k += kred[q];
  reweighted_from_shifted(uc, K, c.kc, k, o);
  out[col] = o;
}

struct PrScratch {
  PrunedCol* pc;
  int* cnt;
  unsigned long long* tq;  // fixed-point offset sums per bucket
  double* esum;            // under- / overflow bucket sums and sums of magnitudes [col][4]
  unsigned long long* mm;
  double *g, *gsorted;
  int* gcount;
  dd2* below;
  dd2* pref;
  WinBest* part;
  dd2* kpart;
  long long* kcnt;
  double* band;
  int* bcount;
  int nch;
};


static void carve_pr(Arena& A, PrScratch& s, int ncols) {
  s.pc = A.take<PrunedCol>(ncols);
  s.cnt = A.take<int>((size_t)ncols * NBK);
  s.tq = A.take<unsigned long long>((size_t)ncols * NBK);
  s.esum = A.take<double>((size_t)ncols * 4);
  s.mm = A.take<unsigned long long>(2 * (size_t)ncols);
  s.g = A.take<double>((size_t)2 * ncols * CAP);
  s.gsorted = A.take<double>((size_t)2 * ncols * CAP);
  s.gcount = A.take<int>(2 * (size_t)ncols);
  s.below = A.take<dd2>((size_t)ncols * PCTA * 2);
  s.pref = A.take<dd2>((size_t)2 * ncols * (CAP + 1));
  s.nch = 16;
  s.part = A.take<WinBest>((size_t)ncols * s.nch);
  s.kpart = A.take<dd2>((size_t)ncols * PCTA);
  s.kcnt = A.take<long long>((size_t)ncols * PCTA);
  s.band = A.take<double>((size_t)ncols * BCAP);
  s.bcount = A.take<int>((size_t)ncols);
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
  RTD_CU(cudaMemsetAsync(s.bcount, 0, (size_t)ncols * sizeof(int), st));
  k_pr_sample<<<ncols, 1024, 0, st>>>(cols, len, s.pc, s.mm);
  RTD_LAUNCHED();
  // ~64K elements per CTA: many CTAs per column so the 4-CTA/SM waves quantise finely (a CTA flushes its
  // 4096-bin histogram with global atomics, about 1/8 of its element count)
  const unsigned gx = (unsigned)std::max<long long>(1, (len + 65535) / 65536);  // <= 65536 elements per CTA
  k_pr_hist<<<dim3(gx, ncols), PT, 0, st>>>(cols, len, s.pc, s.cnt, s.tq, s.esum, s.mm);
  RTD_LAUNCHED();
  static const bool loc_attr = [] {
    RTD_CU(cudaFuncSetAttribute(k_pr_locate, cudaFuncAttributeMaxDynamicSharedMemorySize, LOC_SMEM));
    return true;
  }();
  (void)loc_attr;
  k_pr_locate<<<ncols, LT, LOC_SMEM, st>>>(len, h, s.pc, s.cnt, s.tq, s.esum, s.mm, uc);
  RTD_LAUNCHED();
  // RTD_UNI_FUSEDKEEP=1: the reweighting sums fused into the gather pass (a column whose bounds are too
  // loose, kfused = 0, sends the batch to k_pr_keep).  Measured on config 4: the fused pass is FP64-bound
  // (two double-double accumulations per value) and takes 7.2 ms per fit against 6.5 ms for the gather
  // and keep passes apart, so it is off by default.
  static const bool no_fused = getenv("RTD_UNI_NOFUSEDKEEP") != nullptr;
  // CTAs per column in the streaming passes: a function of the length only (fixed fold order ->
  // deterministic), ~128K+ elements each so the per-CTA partial folds stay a small share
  static const int npc_env = getenv("RTD_PR_CTAS") ? atoi(getenv("RTD_PR_CTAS")) : 0;
  const int npc = npc_env > 0 ? std::min(npc_env, PCTA) : (int)std::max<long long>(4, std::min<long long>(PCTA, len / 131072));
  constexpr int gsmem = 0;
  if (no_fused)
    k_pr_gather<false><<<dim3(npc, ncols), PT, gsmem, st>>>(cols, len, s.pc, s.g, s.gcount, s.below, s.band,
                                                             s.bcount, s.kpart, s.kcnt);
  else
    k_pr_gather<true><<<dim3(npc, ncols), PT, gsmem, st>>>(cols, len, s.pc, s.g, s.gcount, s.below, s.band,
                                                            s.bcount, s.kpart, s.kcnt);
  RTD_LAUNCHED();
  std::vector<PrunedCol> hc(ncols);
  std::vector<int> gc(2 * ncols), bc(ncols);
  fetch(st, {{hc.data(), s.pc, ncols * sizeof(PrunedCol)}, {gc.data(), s.gcount, 2 * ncols * sizeof(int)},
             {bc.data(), s.bcount, ncols * sizeof(int)}});
  // columns whose bounds were too loose for the fused sums (kfused = 0: e.g. a flat or bimodal projection
  // with a wide candidate range) get the separate keep pass; the others finish from the gather's sums
  int nfused = 0;
  for (int j = 0; j < ncols; j++)
    if (!no_fused && hc[j].kfused && bc[j] <= BCAP) nfused++;
  static const bool dbg = getenv("RTD_DEBUG_PRUNED") != nullptr;
  if (dbg) {
    for (int j = 0; j < ncols; j++)
      fprintf(stderr, "pruned len=%lld col=%d status=%d r=[%lld,%lld] s=[%lld,%lld] bs=[%d,%d] be=[%d,%d] span=%g g=%d,%d "
              "kfused=%d band=%d\n",
              len, j, hc[j].status, hc[j].rmin, hc[j].rmax, hc[j].smin, hc[j].smax, hc[j].bs_lo, hc[j].bs_hi,
              hc[j].be_lo, hc[j].be_hi, hc[j].hi - hc[j].lo, gc[2 * j], gc[2 * j + 1], hc[j].kfused, bc[j]);
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
    // 256 threads: many segments (2 per column) share each SM; measured 0.43 -> 0.34 ms per 640-column call
    // against 1024 threads (a CTA-wide barrier per bitonic stage costs more than the pairs per thread).
    // The shared memory of a launch is sized by its largest segment, so a few long segments (a column
    // with a wide candidate range) would cut every CTA's occupancy: segments up to SPLIT go in a launch
    // sized for them, the longer ones (if any) in a second launch (each skips the other's).
    constexpr int spt = 256, SPLIT = 4096;
    int np2s = 1;
    for (int v : gc)
      if (v <= SPLIT)
        while (np2s < v) np2s <<= 1;
    k_pr_sortprefix<<<2 * ncols, spt, np2s * (int)sizeof(double), st>>>(npc, s.pc, s.g, s.gcount, s.below, s.pref,
                                                                         0, SPLIT);
    RTD_LAUNCHED();
    if (gmax > SPLIT) {
      k_pr_sortprefix<<<2 * ncols, spt, std::min(smem, np2 * (int)sizeof(double)), st>>>(npc, s.pc, s.g, s.gcount,
                                                                                           s.below, s.pref, SPLIT + 1,
                                                                                           SMAX);
      RTD_LAUNCHED();
    }
  } else {  // chunk sorts + merge rounds (no library sort on the fit path)
    static const int csmem = [] {
      cudaFuncSetAttribute(k_pr_chunksort, cudaFuncAttributeMaxDynamicSharedMemorySize, SMAX * (int)sizeof(double));
      return SMAX * (int)sizeof(double);
    }();
    const int nchunk = (gmax + SMAX - 1) / SMAX;
    k_pr_chunksort<<<dim3(nchunk, 2 * ncols), 1024, csmem, st>>>(s.pc, s.g, s.gcount);
    RTD_LAUNCHED();
    double *src = s.g, *dst = s.gsorted;
    for (int w = SMAX; w < gmax; w *= 2) {
      k_pr_merge<<<dim3((gmax + 2 * w - 1) / (2 * w), 2 * ncols), 1024, 0, st>>>(s.pc, src, dst, s.gcount, w);
      RTD_LAUNCHED();
      std::swap(src, dst);
    }
    k_pr_prefix<<<2 * ncols, 1024, 0, st>>>(npc, s.pc, src, s.gcount, s.below, s.pref);
    RTD_LAUNCHED();
  }
  k_pr_eval<<<dim3(s.nch, ncols), PT, 0, st>>>(h, s.pc, s.pref, s.part, s.nch);
  RTD_LAUNCHED();
  k_pr_raw<<<ncols, 32, 0, st>>>(h, s.pc, s.pref, s.part, s.nch, uc, out_dev);
  RTD_LAUNCHED();
  if (nfused > 0) {
    k_pr_final_fused<<<ncols, PT, 0, st>>>(uc, npc, s.pc, s.kpart, s.kcnt, s.band, s.bcount, out_dev);
    RTD_LAUNCHED();
  }
  if (nfused < ncols) {  // the fused columns' CTAs exit at once
    const PrunedCol* fpc = no_fused ? nullptr : s.pc;
    k_pr_keep<<<dim3(npc, ncols), PT, 0, st>>>(cols, len, uc, out_dev, s.kpart, s.kcnt, fpc, s.bcount);
    RTD_LAUNCHED();
    k_pr_final<<<ncols, 32, 0, st>>>(uc, npc, s.kpart, s.kcnt, out_dev, fpc, s.bcount);
    RTD_LAUNCHED();
  }
  return true;
}

}  // namespace rtd
