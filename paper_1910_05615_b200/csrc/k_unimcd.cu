// K1: batched univariate reweighted MCD (§3.1).
//
// For every column: sort (CUB radix sort of fp64 keys), then evaluate the
// window objective h*SQ(s) = h*S2(s) - S1(s)^2 for every start s from
// double-double prefix sums, take the argmin (ties -> lowest s, reading R2),
// and finish the raw and reweighted estimates (readings R3, R4):
//   loc0 = S1(s*)/h, var0 = c(h/n,1) SQ(s*)/(h-1),
//   kept = {(y-loc0)^2 <= chi2_{1,.975} var0} (a contiguous range of the sorted column),
//   loc = round(sum kept)/k, scale^2 = c(.975,1) sum_kept (y-loc)^2/(k-1).
// Prefix sums are never materialised: each window CTA rebuilds the two
// prefix streams it needs (P(s) and P(s+h)) from per-chunk totals.
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>

#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "rtd_internal.h"

namespace rtd {

bool unimcd_pruned(Arena& A, cudaStream_t st, const double* cols, long long len, int ncols, UniConst uc,
                   UniOut* out_dev);

static constexpr int UCH = 1024;   // elements per chunk
static constexpr int UTH = 256;    // threads per CTA (4 elements each)
static constexpr int UPT = UCH / UTH;

__global__ void __launch_bounds__(UTH) k_uni_chunksum(const double* __restrict__ sorted, long long len, int nchunks,
                                                      dd2* __restrict__ csum) {
  __shared__ dd2 sm[33];
  const int col = blockIdx.y;
  const long long s0 = (long long)blockIdx.x * UCH;
  const double* y = sorted + (long long)col * len;
  dd2 acc = dd2_zero();
#pragma unroll
  for (int e = 0; e < UPT; e++) {
    long long i = s0 + threadIdx.x * UPT + e;
    if (i < len) acc = dd2_add(acc, dd2_of(y[i]));
  }
  dd2 tot = block_sum_dd2(acc, sm);
  if (threadIdx.x == 0) csum[(long long)col * nchunks + blockIdx.x] = tot;
}

// Prefix sums of chunk totals ANCHORED at the chunk boundary nearest the middle of the sorted column:
// coff[col][c] = P(c UCH) - P(A UCH), i.e. the sum of chunks [A, c) for c >= A and minus the sum of
// chunks [c, A) for c < A.  Every window sum is a difference of two such values, and no partial sum
// reaches past the window ends into the tails (a sorted column with entries of magnitude 1e12 at both
// ends would otherwise lose the window sums to cancellation in the prefix differences).
__global__ void __launch_bounds__(1024) k_uni_chunkscan(const dd2* __restrict__ csum, int nchunks,
                                                        dd2* __restrict__ coff) {
  __shared__ dd2 sm[33];
  const int col = blockIdx.y;
  const dd2* cs = csum + (long long)col * nchunks;
  dd2* co = coff + (long long)col * (nchunks + 1);
  const int A = nchunks / 2;
  {  // forward: chunks [A, nchunks)
    const int nf = nchunks - A;
    const int per = (nf + blockDim.x - 1) / blockDim.x;
    const int c0 = A + threadIdx.x * per, c1 = min(nchunks, c0 + per);
    dd2 loc = dd2_zero();
    for (int c = c0; c < c1; c++) loc = dd2_add(loc, cs[c]);
    dd2 tot;
    dd2 ex = block_exscan_dd2(loc, &tot, sm);
    for (int c = c0; c < c1; c++) {
      co[c] = ex;
      ex = dd2_add(ex, cs[c]);
    }
    if (threadIdx.x == 0) co[nchunks] = tot;
  }
  {  // backward: chunks A-1, A-2, ..., 0
    const int per = (A + blockDim.x - 1) / blockDim.x;
    const int i0 = threadIdx.x * per, i1 = min(A, i0 + per);
    dd2 loc = dd2_zero();
    for (int i = i0; i < i1; i++) loc = dd2_add(loc, cs[A - 1 - i]);
    dd2 tot;
    dd2 ex = block_exscan_dd2(loc, &tot, sm);
    for (int i = i0; i < i1; i++) {
      ex = dd2_add(ex, cs[A - 1 - i]);
      co[A - 1 - i] = {dd_neg(ex.s1), dd_neg(ex.s2)};
    }
  }
}

// P(t) - P(anchor) of (y_i, y_i^2), block-cooperative; all threads get the value.
__device__ dd2 block_prefix_at(const double* __restrict__ y, const dd2* __restrict__ co, long long t, dd2* sm) {
  const long long c = t / UCH;
  const long long s0 = c * UCH;
  dd2 acc = dd2_zero();
#pragma unroll
  for (int e = 0; e < UPT; e++) {
    long long i = s0 + threadIdx.x * UPT + e;
    if (i < t) acc = dd2_add(acc, dd2_of(y[i]));
  }
  dd2 tot = block_sum_dd2(acc, sm);
  return dd2_add(co[c], tot);
}

struct WinPartial {
  double vhi, vlo;
  long long s;
};

__device__ __forceinline__ bool win_better(double ahi, double alo, long long as, double bhi, double blo, long long bs) {
  if (ahi != bhi) return ahi < bhi;
  if (alo != blo) return alo < blo;
  return as < bs;
}

// window objective for starts s in [blockIdx.x*UCH, +UCH) ∩ [0, nwin)
__global__ void __launch_bounds__(UTH) k_uni_window(const double* __restrict__ sorted, long long len, long long h,
                                                    int nchunks, const dd2* __restrict__ coff, int nwchunks,
                                                    WinPartial* __restrict__ part) {
  __shared__ dd2 sm[33];
  __shared__ WinPartial wsm[UTH / 32];
  const int col = blockIdx.y;
  const double* y = sorted + (long long)col * len;
  const dd2* co = coff + (long long)col * (nchunks + 1);
  const long long nwin = len - h + 1;
  const long long s0 = (long long)blockIdx.x * UCH;
  // left stream P(s), s = s0 + 4t + e ; s0 is a chunk boundary
  double yl[UPT], yr[UPT];
#pragma unroll
  for (int e = 0; e < UPT; e++) {
    long long i = s0 + threadIdx.x * UPT + e;
    yl[e] = i < len ? y[i] : 0.0;
  }
  dd2 tl = dd2_zero();
#pragma unroll
  for (int e = 0; e < UPT; e++) tl = dd2_add(tl, dd2_of(yl[e]));
  dd2 totl;
  dd2 exl = block_exscan_dd2(tl, &totl, sm);
  exl = dd2_add(co[blockIdx.x], exl);
  // right stream P(s + h)
  const long long a = s0 + h;
  dd2 Pa = block_prefix_at(y, co, a, sm);
#pragma unroll
  for (int e = 0; e < UPT; e++) {
    long long i = a + threadIdx.x * UPT + e;
    yr[e] = i < len ? y[i] : 0.0;
  }
  dd2 tr = dd2_zero();
#pragma unroll
  for (int e = 0; e < UPT; e++) tr = dd2_add(tr, dd2_of(yr[e]));
  dd2 totr;
  dd2 exr = block_exscan_dd2(tr, &totr, sm);
  exr = dd2_add(Pa, exr);
  double bhi = __longlong_as_double(0x7ff0000000000000LL), blo = 0.0;
  long long bs = 0x7fffffffffffffffLL;
  const double hd = (double)h;
#pragma unroll
  for (int e = 0; e < UPT; e++) {
    long long s = s0 + threadIdx.x * UPT + e;
    if (s < nwin) {
      dd S1 = dd_sub(exr.s1, exl.s1);
      dd S2 = dd_sub(exr.s2, exl.s2);
      dd v = dd_sub(dd_mul_d(S2, hd), dd_mul(S1, S1));
      if (win_better(v.hi, v.lo, s, bhi, blo, bs)) {
        bhi = v.hi;
        blo = v.lo;
        bs = s;
      }
    }
    exl = dd2_add(exl, dd2_of(yl[e]));
    exr = dd2_add(exr, dd2_of(yr[e]));
  }
  // block argmin
  for (int d = 16; d > 0; d >>= 1) {
    double ohi = __shfl_down_sync(0xffffffffu, bhi, d);
    double olo = __shfl_down_sync(0xffffffffu, blo, d);
    long long os = __shfl_down_sync(0xffffffffu, bs, d);
    if (win_better(ohi, olo, os, bhi, blo, bs)) {
      bhi = ohi;
      blo = olo;
      bs = os;
    }
  }
  if ((threadIdx.x & 31) == 0) wsm[threadIdx.x >> 5] = {bhi, blo, bs};
  __syncthreads();
  if (threadIdx.x == 0) {
    WinPartial b = wsm[0];
    for (int w = 1; w < UTH / 32; w++)
      if (win_better(wsm[w].vhi, wsm[w].vlo, wsm[w].s, b.vhi, b.vlo, b.s)) b = wsm[w];
    part[(long long)col * nwchunks + blockIdx.x] = b;
  }
}

// first index in [lo, hi) with pred true (pred monotone false -> true; hi if none), by one warp:
// 32 probes per round, ballot, narrow to one of 32 sub-ranges
template <class Pred>
__device__ __forceinline__ long long warp_partition_point(long long lo, long long hi, Pred pred) {
  const int lane = threadIdx.x & 31;
  while (hi - lo > 32) {
    const long long step = (hi - lo + 31) / 32;
    const long long pos = min(hi - 1, lo + (lane + 1) * step - 1);
    const unsigned b = __ballot_sync(0xffffffffu, pred(pos));
    if (b == 0u) return hi;  // the last probe is hi - 1: nothing in range is true
    const int f = __ffs(b) - 1;  // first probe that holds: the point is in (pos_{f-1}, pos_f]
    const long long nlo = f == 0 ? lo : lo + f * step;
    hi = min(hi, lo + (f + 1) * step);
    lo = nlo;
  }
  const long long pos = lo + lane;
  const unsigned b = __ballot_sync(0xffffffffu, pos < hi && pred(pos));
  return b ? lo + (__ffs(b) - 1) : hi;
}

__device__ __forceinline__ bool uni_keep(double y, double loc0, double thresh) {
  double d = __dsub_rn(y, loc0);
  return __dmul_rn(d, d) <= thresh;
}

// (d, d^2) of the SHIFTED value d = y - c, d exact as a double-double (two-sum): the window objective
// h S2 - S1^2 is shift-invariant, and with c = the column's median its terms are of the size of the spread,
// not of the offset -- a column 1e8 + 1e-6 N(0,1) keeps its argmin (unshifted, S2 ~ h 1e16 and S1^2 cancel
// to ~30 digits, past what double-double holds)
__device__ __forceinline__ dd2 dd2_sh(double y, double c) {
  const dd d = two_sum(y, -c);
  dd p = two_prod(d.hi, d.hi);
  p = quick_two_sum(p.hi, __fma_rn(2.0 * d.hi, d.lo, p.lo));
  return {d, p};
}

__global__ void __launch_bounds__(UTH) k_uni_final(const double* __restrict__ sorted, long long len, long long h,
                                                   int nchunks, const dd2* __restrict__ coff, int nwchunks,
                                                   const WinPartial* __restrict__ part, UniConst uc,
                                                   UniOut* __restrict__ out) {
  __shared__ dd2 sm[33];
  __shared__ WinPartial wsm[UTH / 32];
  __shared__ long long s_lohi[2];
  const int col = blockIdx.x;
  const double* y = sorted + (long long)col * len;
  const dd2* co = coff + (long long)col * (nchunks + 1);
  const WinPartial* pp = part + (long long)col * nwchunks;
  double bhi = __longlong_as_double(0x7ff0000000000000LL), blo = 0.0;
  long long bs = 0x7fffffffffffffffLL;
  for (int c = threadIdx.x; c < nwchunks; c += blockDim.x) {
    WinPartial w = pp[c];
    if (win_better(w.vhi, w.vlo, w.s, bhi, blo, bs)) {
      bhi = w.vhi;
      blo = w.vlo;
      bs = w.s;
    }
  }
  for (int d = 16; d > 0; d >>= 1) {
    double ohi = __shfl_down_sync(0xffffffffu, bhi, d);
    double olo = __shfl_down_sync(0xffffffffu, blo, d);
    long long os = __shfl_down_sync(0xffffffffu, bs, d);
    if (win_better(ohi, olo, os, bhi, blo, bs)) {
      bhi = ohi;
      blo = olo;
      bs = os;
    }
  }
  if ((threadIdx.x & 31) == 0) wsm[threadIdx.x >> 5] = {bhi, blo, bs};
  __syncthreads();
  WinPartial best = wsm[0];
  for (int w = 1; w < UTH / 32; w++)
    if (win_better(wsm[w].vhi, wsm[w].vlo, wsm[w].s, best.vhi, best.vlo, best.s)) best = wsm[w];
  __syncthreads();
  const long long s = best.s;
  dd2 P0 = block_prefix_at(y, co, s, sm);
  dd2 P1 = block_prefix_at(y, co, s + h, sm);
  dd S1 = dd_sub(P1.s1, P0.s1);
  const double hd = (double)h;
  const double loc0 = dd_to_d(dd_div_d(S1, hd));
  dd v = {best.vhi, best.vlo};
  const double var_raw = h > 1 ? dd_to_d(dd_div_d(dd_div_d(v, hd), (double)(h - 1))) : 0.0;
  const double var0 = uc.c_raw * var_raw;
  const double thresh = uc.q1 * var0;
  if (threadIdx.x < 32) {  // three 32-ary searches by warp 0 (a serial binary search is 3 x 15 dependent loads)
    // i0 = first index with y >= loc0
    const long long i0 = warp_partition_point(0, len, [&](long long i) { return y[i] >= loc0; });
    // first kept index in [0, i0] (keep is false then true on [0, i0))
    const long long klo = warp_partition_point(0, i0, [&](long long i) { return uni_keep(y[i], loc0, thresh); });
    // first non-kept index in [i0, len) (keep is true then false)
    const long long khi = warp_partition_point(i0, len, [&](long long i) { return !uni_keep(y[i], loc0, thresh); });
    if (threadIdx.x == 0) {
      s_lohi[0] = klo;
      s_lohi[1] = khi;
    }
  }
  __syncthreads();
  const long long klo = s_lohi[0], khi = s_lohi[1];
  const long long k = khi - klo;
  // sums over the kept range accumulated directly (no prefix differences)
  dd2 kacc = dd2_zero();
  for (long long i = klo + threadIdx.x; i < khi; i += blockDim.x)
    kacc = dd2_add(kacc, dd2_of_dev(y[i], __dsub_rn(y[i], loc0)));
  const dd2 Kd = block_sum_dd2(kacc, sm);
  if (threadIdx.x == 0) {
    UniOut o;
    o.raw_loc = loc0;
    o.raw_var = var_raw;
    o.var0 = var0;
    o.start = s;
    o.kept = k;
    o.pad = 0;
    o.status = 0;
    o.loc = 0.0;
    o.scale = 0.0;
    if (!(var0 > 0.0) || k < 2) {
      o.status = 1;
    } else {
      const dd2 K = Kd;
      const double Sd = dd_to_d(K.s1);
      const double loc = Sd / (double)k;
      // sum (y - loc)^2 from sum y and sum (y - loc0)^2 (no cancellation of sum y^2)
      const dd q = kept_sq_about_loc(K, loc0, loc, (double)k);
      const double var = uc.c_rew * (dd_to_d(q) / (double)(k - 1));
      o.loc = loc;
      o.scale = sqrt(var);
      if (!(var > 0.0)) o.status = 1;
    }
    out[col] = o;
  }
}

// ---------------------------------------------------------------- short columns in one kernel
// len <= USMALL: one CTA of 1024 threads per column does the whole estimator in shared memory --
// a bitonic sort (flip form: the virtual +inf padding up to the next power of two is never touched),
// per-thread chunk totals and their block scan in double-double, the window objective of every start
// (ties -> lowest s), the raw estimate and the reweighting -- so a short column costs one launch
// instead of two radix sorts and four passes (the stream of BASELINE config 5, 20,000 rows).
static constexpr int USMALL = 16384;  // shared-memory capacity bound
static constexpr int USMALL_USE = 4096;  // measured: faster than the radix-sort path up to here (config 1:
                                         // 3 calls 1.06 -> 0.21 ms), slower at 20,000 rows (config 5)
static constexpr int UST = 1024;
static constexpr int USORTED = 24576;  // presorted columns up to here fit k_uni_small's shared memory

__device__ __forceinline__ void u_cmpswap(double* v, int i, int j) {
  const double a = v[i], b = v[j];
  if (a > b) {
    v[i] = b;
    v[j] = a;
  }
}

// P(t) = sum_{i<t} (y_i, y_i^2) from the chunk prefixes cpre (chunk c = [c per, (c+1) per))
__device__ __forceinline__ dd2 u_prefix(const double* v, const dd2* cpre, int per, int t, double cm) {
  const int c = t / per;
  dd2 acc = cpre[c];
  for (int i = c * per; i < t; i++) acc = dd2_add(acc, dd2_sh(v[i], cm));
  return acc;
}

// PRESORTED: the columns arrive sorted (k_uni_cluster_sort) and only the scans, the window objective and
// the reweighting run here -- up to USORTED rows (the column and the chunk prefixes in shared memory)
template <bool PRESORTED>
__global__ void __launch_bounds__(UST) k_uni_small(const double* __restrict__ cols, int len, int h, UniConst uc,
                                                   UniOut* __restrict__ out) {
  extern __shared__ double usm[];
  double* v = usm;                                   // [len]
  dd2* cpre = reinterpret_cast<dd2*>(usm + ((len + 3) & ~3));  // [UST + 1]
  __shared__ dd2 sm[33];
  __shared__ WinPartial wsm[UST / 32];
  const int col = blockIdx.x, t = threadIdx.x;
  const double* y = cols + (long long)col * len;
  for (int i = t; i < len; i += UST) v[i] = y[i];
  int N = 1;
  while (N < len && !PRESORTED) N <<= 1;
  __syncthreads();
  for (int lk = 1; (1 << lk) <= N && !PRESORTED; lk++) {
    const int k = 1 << lk;
    for (int q = t; q < N / 2; q += UST) {  // flip step: i in the lower half of its k-block
      const int i = ((q >> (lk - 1)) << lk) | (q & (k / 2 - 1)), j = i ^ (k - 1);
      if (j < len) u_cmpswap(v, i, j);
    }
    __syncthreads();
    for (int ld = lk - 2; ld >= 0; ld--) {
      const int d = 1 << ld;
      for (int q = t; q < N / 2; q += UST) {
        const int i = ((q >> ld) << (ld + 1)) | (q & (d - 1)), j = i + d;
        if (j < len) u_cmpswap(v, i, j);
      }
      __syncthreads();
    }
  }
  // chunk totals and their exclusive scan (values shifted by the median cm, see dd2_sh)
  const int per = (len + UST - 1) / UST;
  const int c0 = t * per, c1 = min(len, c0 + per);
  const double cm = v[len / 2];
  dd2 loc = dd2_zero();
  for (int i = c0; i < c1; i++) loc = dd2_add(loc, dd2_sh(v[i], cm));
  // prefixes anchored at chunk UST/2 (see k_uni_chunkscan): cpre[c] = P(c per) - P(UST/2 per)
  constexpr int AN = UST / 2;
  dd2 tot;
  const dd2 fex = block_exscan_dd2(t >= AN ? loc : dd2_zero(), &tot, sm);  // chunks [AN, t)
  cpre[t] = loc;  // chunk totals, read back reversed below
  __syncthreads();
  const dd2 rin = t < AN ? cpre[AN - 1 - t] : dd2_zero();
  dd2 btot;
  const dd2 bex = block_exscan_dd2(rin, &btot, sm);  // chunks AN-1, ..., AN-t
  __syncthreads();
  if (t >= AN) cpre[t] = fex;
  else {
    const dd2 b = dd2_add(bex, rin);  // chunks [AN-1-t, AN)
    cpre[AN - 1 - t] = {dd_neg(b.s1), dd_neg(b.s2)};
  }
  if (t == 0) cpre[UST] = tot;
  __syncthreads();
  const dd2 ex = cpre[t];
  // window objective h S2 - S1^2 for starts s in [c0, c1) with s < nwin
  const int nwin = len - h + 1;
  double bhi = __longlong_as_double(0x7ff0000000000000LL), blo = 0.0;
  long long bs = 0x7fffffffffffffffLL;
  const double hd = (double)h;
  if (c0 < nwin) {
    dd2 Pl = ex;
    dd2 Pr = u_prefix(v, cpre, per, c0 + h, cm);
    const int e1 = min(c1, nwin);
    for (int s = c0; s < e1; s++) {
      const dd S1 = dd_sub(Pr.s1, Pl.s1);
      const dd S2 = dd_sub(Pr.s2, Pl.s2);
      const dd w = dd_sub(dd_mul_d(S2, hd), dd_mul(S1, S1));
      if (win_better(w.hi, w.lo, s, bhi, blo, bs)) {
        bhi = w.hi;
        blo = w.lo;
        bs = s;
      }
      Pl = dd2_add(Pl, dd2_sh(v[s], cm));
      if (s + h < len) Pr = dd2_add(Pr, dd2_sh(v[s + h], cm));
    }
  }
  for (int d = 16; d > 0; d >>= 1) {
    const double ohi = __shfl_down_sync(0xffffffffu, bhi, d);
    const double olo = __shfl_down_sync(0xffffffffu, blo, d);
    const long long os = __shfl_down_sync(0xffffffffu, bs, d);
    if (win_better(ohi, olo, os, bhi, blo, bs)) {
      bhi = ohi;
      blo = olo;
      bs = os;
    }
  }
  if ((t & 31) == 0) wsm[t >> 5] = {bhi, blo, bs};
  __syncthreads();
  __shared__ int s_k[2];
  __shared__ double s_f[4];
  if (t == 0) {
  WinPartial best = wsm[0];
  for (int w = 1; w < UST / 32; w++)
    if (win_better(wsm[w].vhi, wsm[w].vlo, wsm[w].s, best.vhi, best.vlo, best.s)) best = wsm[w];
  const int s = (int)best.s;
  const dd S1 = dd_sub(u_prefix(v, cpre, per, s + h, cm).s1, u_prefix(v, cpre, per, s, cm).s1);
  const double loc0 = dd_to_d(dd_add(dd_div_d(S1, hd), dd_make(cm)));
  const dd wv = {best.vhi, best.vlo};
  const double var_raw = h > 1 ? dd_to_d(dd_div_d(dd_div_d(wv, hd), (double)(h - 1))) : 0.0;
  const double var0 = uc.c_raw * var_raw;
  const double thresh = uc.q1 * var0;
  int lo = 0, hi = len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (v[mid] < loc0) lo = mid + 1; else hi = mid;
  }
  const int i0 = lo;
  lo = 0;
  hi = i0;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (uni_keep(v[mid], loc0, thresh)) hi = mid; else lo = mid + 1;
  }
  const int klo = lo;
  lo = i0;
  hi = len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (uni_keep(v[mid], loc0, thresh)) lo = mid + 1; else hi = mid;
  }
  const int khi = lo;
  s_k[0] = klo;
  s_k[1] = khi;
  s_f[0] = loc0;
  s_f[1] = var_raw;
  s_f[2] = var0;
  s_f[3] = (double)s;
  }
  __syncthreads();
  // sums over the kept range accumulated directly (no prefix differences)
  const int klo = s_k[0], khi = s_k[1];
  dd2 kacc = dd2_zero();
  const double c0v = s_f[0];
  for (int i = klo + t; i < khi; i += UST) kacc = dd2_add(kacc, dd2_of_dev(v[i], __dsub_rn(v[i], c0v)));
  const dd2 Kd = block_sum_dd2(kacc, sm);
  if (t != 0) return;
  const double loc0 = s_f[0], var_raw = s_f[1], var0 = s_f[2];
  const int s = (int)s_f[3];
  UniOut o;
  o.raw_loc = loc0;
  o.raw_var = var_raw;
  o.var0 = var0;
  o.start = s;
  o.kept = khi - klo;
  o.pad = 0;
  o.status = 0;
  o.loc = 0.0;
  o.scale = 0.0;
  const long long k = khi - klo;
  if (!(var0 > 0.0) || k < 2) {
    o.status = 1;
  } else {
    const dd2 K = Kd;
    const double Sd = dd_to_d(K.s1);
    const double lc = Sd / (double)k;
    const dd q = kept_sq_about_loc(K, loc0, lc, (double)k);
    const double var = uc.c_rew * (dd_to_d(q) / (double)(k - 1));
    o.loc = lc;
    o.scale = sqrt(var);
    if (!(var > 0.0)) o.status = 1;
  }
  out[col] = o;
}

// ------------------------------------------------------------------ cluster sort of short columns
// Columns of up to UCS_CL * UCS_CAP = 32768 rows (config 5: 20,000) are sorted by one 8-CTA thread-block
// cluster each, instead of by two device-wide CUB radix sorts:
//   1. every CTA sorts a contiguous eighth of the column, padded to 4096 with keys above all others, by a
//      bitonic network held in registers (4 values per thread): strides < 4 inside a thread, < 128 by warp
//      shuffles,
//      larger ones through shared memory;
//   2. three merge rounds pair the sorted runs (8 -> 4 -> 2 -> 1 per cluster): each CTA finds where its
//      stretch of the merged run starts and ends in the two input runs (merge path, a 32-ary search by
//      one warp over the runs where they live -- the shared memory of the other CTAs, DSMEM), copies the
//      two sub-ranges into its own shared memory and merges them there, every thread a stretch of its own
//      (merge path again, stable: ties take the left run first).
// The sorted column is written back for the window kernels below.
static constexpr int UCS_CL = 8;      // CTAs per cluster (one column)
static constexpr int UCS_CAP = 4096;  // values per CTA
static constexpr int UCS_T = 1024;
static constexpr int UCS_V = UCS_CAP / UCS_T;  // values per thread in the local sort (4)

__device__ __forceinline__ unsigned long long ucs_key(double x) {  // order-preserving key of x
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double ucs_val(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

// smallest i in [lo, hi] with A(i) > B(o - i - 1) (hi if none) -- the merge-path split of output o, stable;
// evaluated by the 32 lanes of one warp (32-ary search), A / B read through `elem`
template <class F>
__device__ __forceinline__ int ucs_split(int o, int lo, int hi, int gA, int gB, F elem, int lane) {
  while (lo < hi) {
    const int step = (hi - lo + 31) / 32;
    const int i = lo + lane * step;
    const bool pr = i < hi ? (elem(gA + i) > elem(gB + o - i - 1)) : true;
    const unsigned bal = __ballot_sync(0xffffffffu, pr);
    if (bal == 0u) {  // the split lies beyond the last probe
      lo = lo + 31 * step + 1;
      continue;
    }
    const int f = __ffs(bal) - 1;  // first lane whose probe is at or past the split
    const int nhi = min(hi, lo + f * step);
    const int nlo = f == 0 ? lo : lo + (f - 1) * step + 1;
    lo = nlo;
    hi = nhi;
  }
  return lo;
}

// a bitonic stage whose pairs lie inside a thread (stride S < UCS_V, compile time: x stays in registers)
template <int S>
__device__ __forceinline__ void ucs_reg_stage(unsigned long long (&x)[UCS_V], int t, int size) {
#pragma unroll
  for (int k = 0; k < UCS_V; k++) {
    if ((k & S) == 0) {
      const int e = t * UCS_V + k;
      const bool up = (e & size) == 0;
      const unsigned long long a = x[k], b = x[k + S];
      const unsigned long long lo = a < b ? a : b, hi = a < b ? b : a;
      x[k] = up ? lo : hi;
      x[k + S] = up ? hi : lo;
    }
  }
}

__global__ void __cluster_dims__(UCS_CL, 1, 1) __launch_bounds__(UCS_T, 1)
    k_uni_cluster_sort(const double* __restrict__ cols, long long len, double* __restrict__ sorted) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ unsigned long long ucs_dyn[];  // [2][UCS_CAP] runs (read remotely), [2][UCS_CAP] local copies
  // values as order-preserving 64-bit keys (integer compares in the network and the merges)
  __shared__ int s_split[2];
  const int r = (int)cluster.block_rank();
  const int col = blockIdx.x / UCS_CL;
  const int t = threadIdx.x, lane = t & 31;
  const int n = (int)len;
  const int nloc = (n + UCS_CL - 1) / UCS_CL;
  const int r0 = min(n, r * nloc), cnt = min(n, r0 + nloc) - r0;
  const double* y = cols + (long long)col * len;
  unsigned long long* xs = ucs_dyn + UCS_CAP;  // exchange buffer of the local sort
  // ---- 1. local bitonic sort in registers: element e = t * UCS_V + k
  unsigned long long x[UCS_V];
#pragma unroll
  for (int k = 0; k < UCS_V; k++) {
    const int e = t * UCS_V + k;
    x[k] = e < cnt ? ucs_key(y[r0 + e]) : ~0ull;  // padding above every key
  }
  for (int size = 2; size <= UCS_CAP; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride < UCS_V) {
        if (stride == 4) ucs_reg_stage<4>(x, t, size);
        else if (stride == 2) ucs_reg_stage<2>(x, t, size);
        else ucs_reg_stage<1>(x, t, size);
      } else if (stride < UCS_V * 32) {
        const int lm = stride / UCS_V;
        const bool lower = (lane & lm) == 0;
#pragma unroll
        for (int k = 0; k < UCS_V; k++) {
          const int e = t * UCS_V + k;
          const unsigned long long o = __shfl_xor_sync(0xffffffffu, x[k], lm);
          const bool keep_min = ((e & size) == 0) == lower;
          x[k] = keep_min ? (x[k] < o ? x[k] : o) : (x[k] < o ? o : x[k]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < UCS_V; k++) xs[t * UCS_V + k] = x[k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < UCS_V; k++) {
          const int e = t * UCS_V + k;
          const unsigned long long o = xs[e ^ stride];
          const bool keep_min = ((e & size) == 0) == ((e & stride) == 0);
          x[k] = keep_min ? (x[k] < o ? x[k] : o) : (x[k] < o ? o : x[k]);
        }
        __syncthreads();
      }
    }
  }
  unsigned long long* v = ucs_dyn;
#pragma unroll
  for (int k = 0; k < UCS_V; k++) {
    const int e = t * UCS_V + k;
    if (e < cnt) v[e] = x[k];
  }
  cluster.sync();
  // ---- 2. merge rounds over the cluster
  int cur = 0;
  unsigned long long* la = ucs_dyn + 2 * UCS_CAP;
  unsigned long long* lb = ucs_dyn + 3 * UCS_CAP;
  for (int span = 1; span < UCS_CL; span <<= 1) {
    const unsigned long long* src = ucs_dyn + cur * UCS_CAP;
    unsigned long long* dst = ucs_dyn + (cur ^ 1) * UCS_CAP;
    const int grp = r / (2 * span);
    const int gs = min(n, grp * 2 * span * nloc), gm = min(n, gs + span * nloc), ge = min(n, gm + span * nloc);
    const int na = gm - gs, nb = ge - gm;
    auto elem = [&](int g) -> unsigned long long {  // global position g of the current runs, in CTA g / nloc
      const int q = g / nloc;
      return cluster.map_shared_rank(src, q)[g - q * nloc];
    };
    const int olo = r0 - gs, ohi = olo + cnt;  // this CTA's outputs, relative to the group
    if (t < 64) {
      const int o = t < 32 ? olo : ohi;
      const int sp = ucs_split(o, max(0, o - nb), min(o, na), gs, gm, elem, lane);
      if (lane == 0) s_split[t >> 5] = sp;
    }
    __syncthreads();
    const int ia = s_split[0], ib = s_split[1];
    const int ja = olo - ia, jb = ohi - ib;  // B sub-range [ja, jb)
    const int nla = ib - ia, nlb = jb - ja;
    for (int e = t; e < nla; e += UCS_T) la[e] = elem(gs + ia + e);
    for (int e = t; e < nlb; e += UCS_T) lb[e] = elem(gm + ja + e);
    __syncthreads();
    const int ept = (cnt + UCS_T - 1) / UCS_T;
    const int o0 = min(cnt, t * ept), o1 = min(cnt, o0 + ept);
    if (o0 < o1) {
      int lo = max(0, o0 - nlb), hi = min(o0, nla);
      while (lo < hi) {
        const int i = (lo + hi) >> 1;
        if (la[i] <= lb[o0 - i - 1]) lo = i + 1;
        else hi = i;
      }
      int i = lo, j = o0 - lo;
      for (int o = o0; o < o1; o++) {
        const bool takeA = j >= nlb || (i < nla && la[i] <= lb[j]);
        dst[o] = takeA ? la[i++] : lb[j++];
      }
    }
    cur ^= 1;
    cluster.sync();  // the round's outputs are complete everywhere (and nobody still reads src)
  }
  const unsigned long long* fin = ucs_dyn + cur * UCS_CAP;
  double* out = sorted + (long long)col * len;
  for (int i = t; i < cnt; i += UCS_T) out[r0 + i] = ucs_val(fin[i]);
  cluster.sync();  // no CTA leaves while another may still read its buffers
}

// ------------------------------------------------------------------ the whole estimator of a short column
// on one cluster: k_uni_cluster_sort's sort (512 threads x 8 keys per CTA, 96 KB of shared memory, so two
// CTAs -- and twice the clusters -- fit per SM; 16 columns no longer take two waves) followed, in the same
// kernel, by k_uni_small's scans, window objective and reweighting on the sorted column spread over the 8
// CTAs (readings R2-R4):
//   - chunk c = (CTA q, thread t) holds local positions [t per, (t+1) per) of the CTA's sorted run; chunk
//     totals (sum y, sum y^2) in double-double, scanned per CTA forwards and backwards, and the CTA totals
//     exchanged through DSMEM: prefixes ANCHORED at the first position of CTA 4 (~ the median, as
//     k_uni_small's anchor: no window sum ever reaches into the tails);
//   - every thread evaluates h S2 - S1^2 for the starts of its chunk, P(s + h) read from the CTA that holds
//     position s + h (its chunk prefix + at most `per` values, DSMEM); argmin per CTA, then over the cluster
//     in rank order (ties -> lowest s);
//   - the raw fit from the best window (every CTA, the same arithmetic), the kept values summed per CTA and
//     folded in rank order by CTA 0, which writes the column's UniOut.
// One launch per call instead of two, and the tail work runs on 8 SMs instead of one.
static constexpr int UCM_T = 512;
static constexpr int UCM_V = UCS_CAP / UCM_T;  // 8 keys per thread in the local sort

template <int S>
__device__ __forceinline__ void ucm_reg_stage(unsigned long long (&x)[UCM_V], int t, int size) {
#pragma unroll
  for (int k = 0; k < UCM_V; k++) {
    if ((k & S) == 0) {
      const int e = t * UCM_V + k;
      const bool up = (e & size) == 0;
      const unsigned long long a = x[k], b = x[k + S];
      const unsigned long long lo = a < b ? a : b, hi = a < b ? b : a;
      x[k] = up ? lo : hi;
      x[k + S] = up ? hi : lo;
    }
  }
}

__global__ void __cluster_dims__(UCS_CL, 1, 1) __launch_bounds__(UCM_T, 2)
    k_uni_cluster_mcd(const double* __restrict__ cols, long long len, long long hl, UniConst uc,
                      UniOut* __restrict__ out) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ unsigned long long ucm_dyn[];  // [3][UCS_CAP]: runs 0 / 1, the merge inputs (la | lb)
  __shared__ int s_split[2];
  __shared__ dd2 sm[33];
  __shared__ dd2 s_tot;           // this CTA's total, read by the cluster
  __shared__ WinPartial s_best;   // this CTA's best window, read by the cluster
  __shared__ dd2 s_kept;          // this CTA's kept sums, read by CTA 0
  __shared__ long long s_kcnt;
  __shared__ double s_fin[4];     // loc0, var_raw, var0, s*
  const int r = (int)cluster.block_rank();
  const int col = blockIdx.x / UCS_CL;
  const int t = threadIdx.x, lane = t & 31;
  const int n = (int)len, h = (int)hl;
  const int nloc = (n + UCS_CL - 1) / UCS_CL;
  const int r0 = min(n, r * nloc), cnt = min(n, r0 + nloc) - r0;
  const double* y = cols + (long long)col * len;
  unsigned long long* xs = ucm_dyn + UCS_CAP;
  // ---- 1. local bitonic sort in registers (element e = t * UCM_V + k)
  unsigned long long x[UCM_V];
#pragma unroll
  for (int k = 0; k < UCM_V; k++) {
    const int e = t * UCM_V + k;
    x[k] = e < cnt ? ucs_key(y[r0 + e]) : ~0ull;
  }
  for (int size = 2; size <= UCS_CAP; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride < UCM_V) {
        if (stride == 4) ucm_reg_stage<4>(x, t, size);
        else if (stride == 2) ucm_reg_stage<2>(x, t, size);
        else ucm_reg_stage<1>(x, t, size);
      } else if (stride < UCM_V * 32) {
        const int lm = stride / UCM_V;
        const bool lower = (lane & lm) == 0;
#pragma unroll
        for (int k = 0; k < UCM_V; k++) {
          const int e = t * UCM_V + k;
          const unsigned long long o = __shfl_xor_sync(0xffffffffu, x[k], lm);
          const bool keep_min = ((e & size) == 0) == lower;
          x[k] = keep_min ? (x[k] < o ? x[k] : o) : (x[k] < o ? o : x[k]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < UCM_V; k++) xs[t * UCM_V + k] = x[k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < UCM_V; k++) {
          const int e = t * UCM_V + k;
          const unsigned long long o = xs[e ^ stride];
          const bool keep_min = ((e & size) == 0) == ((e & stride) == 0);
          x[k] = keep_min ? (x[k] < o ? x[k] : o) : (x[k] < o ? o : x[k]);
        }
        __syncthreads();
      }
    }
  }
#pragma unroll
  for (int k = 0; k < UCM_V; k++) {
    const int e = t * UCM_V + k;
    if (e < cnt) ucm_dyn[e] = x[k];
  }
  cluster.sync();
  // ---- 2. merge rounds over the cluster (as k_uni_cluster_sort; la | lb share one buffer: nla + nlb = cnt)
  int cur = 0;
  unsigned long long* la = ucm_dyn + 2 * UCS_CAP;
  for (int span = 1; span < UCS_CL; span <<= 1) {
    const unsigned long long* src = ucm_dyn + cur * UCS_CAP;
    unsigned long long* dst = ucm_dyn + (cur ^ 1) * UCS_CAP;
    const int grp = r / (2 * span);
    const int gs = min(n, grp * 2 * span * nloc), gm = min(n, gs + span * nloc), ge = min(n, gm + span * nloc);
    const int na = gm - gs, nb = ge - gm;
    auto elem = [&](int g) -> unsigned long long {
      const int q = g / nloc;
      return cluster.map_shared_rank(src, q)[g - q * nloc];
    };
    const int olo = r0 - gs, ohi = olo + cnt;
    if (t < 64) {
      const int o = t < 32 ? olo : ohi;
      const int sp = ucs_split(o, max(0, o - nb), min(o, na), gs, gm, elem, lane);
      if (lane == 0) s_split[t >> 5] = sp;
    }
    __syncthreads();
    const int ia = s_split[0], ib = s_split[1];
    const int ja = olo - ia, jb = ohi - ib;
    const int nla = ib - ia, nlb = jb - ja;
    unsigned long long* lb = la + nla;
    for (int e = t; e < nla; e += UCM_T) la[e] = elem(gs + ia + e);
    for (int e = t; e < nlb; e += UCM_T) lb[e] = elem(gm + ja + e);
    __syncthreads();
    const int ept = (cnt + UCM_T - 1) / UCM_T;
    const int o0 = min(cnt, t * ept), o1 = min(cnt, o0 + ept);
    if (o0 < o1) {
      int lo = max(0, o0 - nlb), hi = min(o0, nla);
      while (lo < hi) {
        const int i = (lo + hi) >> 1;
        if (la[i] <= lb[o0 - i - 1]) lo = i + 1;
        else hi = i;
      }
      int i = lo, j = o0 - lo;
      for (int o = o0; o < o1; o++) {
        const bool takeA = j >= nlb || (i < nla && la[i] <= lb[j]);
        dst[o] = takeA ? la[i++] : lb[j++];
      }
    }
    cur ^= 1;
    cluster.sync();
  }
  // ---- 3. the sorted values (into the last round's source buffer: the keys stay readable), chunk totals
  //         of the values shifted by the column's median (dd2_sh) and anchored chunk prefixes
  const unsigned long long* kfin = ucm_dyn + cur * UCS_CAP;
  double* v = reinterpret_cast<double*>(ucm_dyn + (cur ^ 1) * UCS_CAP);
  dd2* cpre = reinterpret_cast<dd2*>(ucm_dyn + 2 * UCS_CAP);  // [UCM_T] (the merge buffer is free now)
  __shared__ double s_cm;
  for (int i = t; i < cnt; i += UCM_T) v[i] = ucs_val(kfin[i]);
  if (t == 0) {
    const int qm = (n / 2) / nloc;
    s_cm = ucs_val(*cluster.map_shared_rank(kfin + (n / 2 - qm * nloc), qm));
  }
  __syncthreads();
  const double cm = s_cm;
  const int per = (nloc + UCM_T - 1) / UCM_T;  // the same chunk geometry in every CTA
  const int c0 = min(cnt, t * per), c1 = min(cnt, c0 + per);
  dd2 loc = dd2_zero();
  for (int i = c0; i < c1; i++) loc = dd2_add(loc, dd2_sh(v[i], cm));
  constexpr int AQ = UCS_CL / 2;  // anchor: the first position of CTA AQ
  dd2 ctot;
  const dd2 fex = block_exscan_dd2(loc, &ctot, sm);  // chunks [0, t) of this CTA
  cpre[t] = loc;
  __syncthreads();
  const dd2 rin = cpre[UCM_T - 1 - t];
  dd2 btot;
  const dd2 bex = block_exscan_dd2(rin, &btot, sm);  // chunks above UCM_T - 1 - t
  __syncthreads();
  // local parts: forward prefix for CTAs >= AQ, minus the suffix (from the chunk start on) below AQ
  if (r >= AQ) cpre[t] = fex;
  else cpre[UCM_T - 1 - t] = dd2_add(bex, rin);  // (negated with the cross-CTA part below)
  if (t == 0) s_tot = ctot;
  cluster.sync();  // every CTA's total is published
  dd2 off = dd2_zero(), Pn = dd2_zero();  // cross-CTA part of this CTA's prefixes; anchored P(n)
  if (r >= AQ) {
    for (int q = AQ; q < r; q++) off = dd2_add(off, *cluster.map_shared_rank(&s_tot, q));
  } else {
    for (int q = r + 1; q < AQ; q++) off = dd2_add(off, *cluster.map_shared_rank(&s_tot, q));
  }
  for (int q = AQ; q < UCS_CL; q++) Pn = dd2_add(Pn, *cluster.map_shared_rank(&s_tot, q));
  {
    const dd2 lp = cpre[t];
    if (r >= AQ) {
      cpre[t] = dd2_add(off, lp);
    } else {
      const dd2 b = dd2_add(off, lp);
      cpre[t] = {dd_neg(b.s1), dd_neg(b.s2)};
    }
  }
  cluster.sync();  // every CTA's anchored chunk prefixes are final
  // anchored P(G) for a global position G in [0, n] (remote chunk prefix + the chunk's values before G)
  auto prefix_at = [&](int G) -> dd2 {
    if (G >= n) return Pn;
    const int q = G / nloc, l = G - q * nloc, tc = l / per;
    const dd2* cq = reinterpret_cast<const dd2*>(cluster.map_shared_rank(ucm_dyn + 2 * UCS_CAP, q));
    dd2 acc = cq[tc];
    const double* vq = cluster.map_shared_rank(v, q);
    for (int i = tc * per; i < l; i++) acc = dd2_add(acc, dd2_sh(vq[i], cm));
    return acc;
  };
  // ---- 4. window objective of the starts in this thread's chunk
  const int nwin = n - h + 1;
  const double hd = (double)h;
  double bhi = __longlong_as_double(0x7ff0000000000000LL), blo = 0.0;
  long long bs = 0x7fffffffffffffffLL;
  {
    const int ga = r0 + c0, gb = min(r0 + c1, nwin);
    if (ga < gb) {
      dd2 Pl = cpre[t];
      dd2 Pr = prefix_at(ga + h);
      int G = ga + h, q = G / nloc, l = G - q * nloc;
      const double* vq = cluster.map_shared_rank(v, q < UCS_CL ? q : UCS_CL - 1);
      for (int sg = ga; sg < gb; sg++) {
        const dd S1 = dd_sub(Pr.s1, Pl.s1);
        const dd S2 = dd_sub(Pr.s2, Pl.s2);
        const dd w = dd_sub(dd_mul_d(S2, hd), dd_mul(S1, S1));
        if (win_better(w.hi, w.lo, sg, bhi, blo, bs)) {
          bhi = w.hi;
          blo = w.lo;
          bs = sg;
        }
        Pl = dd2_add(Pl, dd2_sh(v[sg - r0], cm));
        if (G < n) {
          Pr = dd2_add(Pr, dd2_sh(vq[l], cm));
          G++;
          if (++l == nloc && G < n) {
            q++;
            l = 0;
            vq = cluster.map_shared_rank(v, q);
          }
        }
      }
    }
  }
  for (int d = 16; d > 0; d >>= 1) {
    const double ohi = __shfl_down_sync(0xffffffffu, bhi, d);
    const double olo = __shfl_down_sync(0xffffffffu, blo, d);
    const long long os = __shfl_down_sync(0xffffffffu, bs, d);
    if (win_better(ohi, olo, os, bhi, blo, bs)) {
      bhi = ohi;
      blo = olo;
      bs = os;
    }
  }
  __shared__ WinPartial wsm[UCM_T / 32];
  if (lane == 0) wsm[t >> 5] = {bhi, blo, bs};
  __syncthreads();
  if (t == 0) {
    WinPartial best = wsm[0];
    for (int w = 1; w < UCM_T / 32; w++)
      if (win_better(wsm[w].vhi, wsm[w].vlo, wsm[w].s, best.vhi, best.vlo, best.s)) best = wsm[w];
    s_best = best;
  }
  cluster.sync();  // every CTA's best window is published
  // ---- 5. the raw fit (every CTA, identical) and the kept sums
  if (t == 0) {
    WinPartial best = *cluster.map_shared_rank(&s_best, 0);
    for (int q = 1; q < UCS_CL; q++) {
      const WinPartial w = *cluster.map_shared_rank(&s_best, q);
      if (win_better(w.vhi, w.vlo, w.s, best.vhi, best.vlo, best.s)) best = w;
    }
    const int sb = (int)best.s;
    const dd S1 = dd_sub(prefix_at(sb + h).s1, prefix_at(sb).s1);
    const double loc0 = dd_to_d(dd_add(dd_div_d(S1, hd), dd_make(cm)));
    const dd wv = {best.vhi, best.vlo};
    const double var_raw = h > 1 ? dd_to_d(dd_div_d(dd_div_d(wv, hd), (double)(h - 1))) : 0.0;
    s_fin[0] = loc0;
    s_fin[1] = var_raw;
    s_fin[2] = uc.c_raw * var_raw;
    s_fin[3] = (double)sb;
  }
  __syncthreads();
  const double loc0 = s_fin[0], var0 = s_fin[2], thresh = uc.q1 * var0;
  dd2 kacc = dd2_zero();
  long long kc = 0;
  for (int i = c0; i < c1; i++)
    if (uni_keep(v[i], loc0, thresh)) {
      kacc = dd2_add(kacc, dd2_of_dev(v[i], __dsub_rn(v[i], loc0)));
      kc++;
    }
  const dd2 Kc = block_sum_dd2(kacc, sm);
  for (int d = 16; d > 0; d >>= 1) kc += __shfl_down_sync(0xffffffffu, kc, d);
  __shared__ long long kred[UCM_T / 32];
  if (lane == 0) kred[t >> 5] = kc;
  __syncthreads();
  if (t == 0) {
    long long k = 0;
    for (int w = 0; w < UCM_T / 32; w++) k += kred[w];
    s_kept = Kc;
    s_kcnt = k;
  }
  cluster.sync();  // every CTA's kept sums are published
  if (r == 0 && t == 0) {
    dd2 K = dd2_zero();
    long long k = 0;
    for (int q = 0; q < UCS_CL; q++) {
      K = dd2_add(K, *cluster.map_shared_rank(&s_kept, q));
      k += *cluster.map_shared_rank(&s_kcnt, q);
    }
    UniOut o;
    o.raw_loc = loc0;
    o.raw_var = s_fin[1];
    o.var0 = var0;
    o.start = (long long)s_fin[3];
    o.kept = k;
    o.pad = 0;
    o.status = 0;
    o.loc = 0.0;
    o.scale = 0.0;
    if (!(var0 > 0.0) || k < 2) {
      o.status = 1;
    } else {
      const double lc = dd_to_d(K.s1) / (double)k;
      const dd qv = kept_sq_about_loc(K, loc0, lc, (double)k);
      const double var = uc.c_rew * (dd_to_d(qv) / (double)(k - 1));
      o.loc = lc;
      o.scale = sqrt(var);
      if (!(var > 0.0)) o.status = 1;
    }
    out[col] = o;
  }
  cluster.sync();  // no CTA leaves while another may still read its shared memory
}

struct UniScratch {
  double* sorted;
  double* tmpk;
  uint8_t *ids, *tmpid, *idout;
  dd2* csum;
  dd2* coff;
  WinPartial* part;
  void* cub_tmp;
  size_t cub_bytes;
};

__global__ void k_fill_colid(uint8_t* __restrict__ ids, long long len, long long total) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x)
    ids[i] = (uint8_t)(i / len);
}

static int id_bits(int ncols) {
  int b = 1;
  while ((1 << b) < ncols) b++;
  return b;
}

// All ncols columns are sorted with two device-wide radix sorts instead of
// ncols small ones: (value -> column id) by the fp64 key, then a stable sort
// by column id, which leaves every column sorted and contiguous.
static constexpr int USORT = 256;  // columns per pass of the sort path (8-bit segment ids)

static size_t cub_sort_bytes_raw(long long len, int ncols);
// memoised: CUB's temporary-storage query runs occupancy queries on the host (~40 us per call, three calls
// per fit, with the GPU idle behind them on a latency-bound fit)
static size_t cub_sort_bytes(long long len, int ncols) {
  static std::mutex mu;
  static std::map<std::pair<long long, int>, size_t> memo;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = memo.find({len, ncols});
    if (it != memo.end()) return it->second;
  }
  const size_t v = cub_sort_bytes_raw(len, ncols);
  std::lock_guard<std::mutex> lk(mu);
  memo[{len, ncols}] = v;
  return v;
}
static size_t cub_sort_bytes_raw(long long len, int ncols) {
  const long long N = len * ncols;
  size_t b1 = 0, b2 = 0;
  if (ncols == 1) {
    cub::DeviceRadixSort::SortKeys(nullptr, b1, (const double*)nullptr, (double*)nullptr, (int)N);
    return b1;
  }
  cub::DeviceRadixSort::SortPairs(nullptr, b1, (const double*)nullptr, (double*)nullptr, (const uint8_t*)nullptr,
                                  (uint8_t*)nullptr, (int)N);
  cub::DeviceRadixSort::SortPairs(nullptr, b2, (const uint8_t*)nullptr, (uint8_t*)nullptr, (const double*)nullptr,
                                  (double*)nullptr, (int)N, 0, id_bits(ncols));
  return std::max(b1, b2);
}

void unimcd_batch(Arena& A, cudaStream_t st, const double* cols, long long len, int ncols, UniConst uc,
                  UniOut* out_dev) {
  static const bool no_small = getenv("RTD_UNI_NOSMALL") != nullptr;
  if (len <= USMALL_USE && len >= 2 && !no_small) {
    if (A.base == nullptr) return;  // no scratch
    const int smem = (int)((((len + 3) & ~3LL) * sizeof(double)) + (UST + 1) * sizeof(dd2));
    static const bool attr = [] {
      cudaFuncSetAttribute(k_uni_small<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(USMALL * sizeof(double) + (UST + 1) * sizeof(dd2)));
      return true;
    }();
    (void)attr;
    k_uni_small<false><<<ncols, UST, smem, st>>>(cols, (int)len, (int)(len / 2 + 1), uc, out_dev);
    RTD_LAUNCHED();
    return;
  }
  const long long h = len / 2 + 1;
  const int nchunks = (int)((len + UCH - 1) / UCH);
  const long long nwin = len - h + 1;
  const int nwchunks = (int)((nwin + UCH - 1) / UCH);
  // the sort path takes at most USORT columns per pass (8-bit column ids in the segmented sort)
  const int sc = std::min(ncols, USORT);
  const long long N = len * sc;
  UniScratch s;
  s.sorted = A.take<double>((size_t)N);
  s.tmpk = sc > 1 ? A.take<double>((size_t)N) : nullptr;
  s.ids = sc > 1 ? A.take<uint8_t>((size_t)N) : nullptr;
  s.tmpid = sc > 1 ? A.take<uint8_t>((size_t)N) : nullptr;
  s.idout = sc > 1 ? A.take<uint8_t>((size_t)N) : nullptr;
  s.csum = A.take<dd2>((size_t)sc * nchunks);
  s.coff = A.take<dd2>((size_t)sc * (nchunks + 1));
  s.part = A.take<WinPartial>((size_t)sc * nwchunks);
  s.cub_bytes = cub_sort_bytes(len, sc);
  s.cub_tmp = A.take<char>(s.cub_bytes);
  // Large columns: exact window by bucketing + bounds (k_unimcd_pruned.cu), every column in one pass;
  // the sort path below is the fallback and the small-n path.
  static const bool force_sort = getenv("RTD_UNI_FULLSORT") != nullptr;
  static const long long pruned_min = getenv("RTD_UNI_PRUNED_MIN") ? atoll(getenv("RTD_UNI_PRUNED_MIN")) : (1LL << 16);
  if (len >= pruned_min && !force_sort) {  // below: the two radix sorts measured faster (config 5)
    const bool done = unimcd_pruned(A, st, cols, len, ncols, uc, out_dev);
    if (A.base == nullptr) return;  // dry run (both paths measured)
    if (done) return;
  }
  if (A.base == nullptr) return;  // dry run
  static const bool no_csort = getenv("RTD_UNI_NOCLUSTERSORT") != nullptr;
  const bool csort = !no_csort && len <= (long long)UCS_CL * UCS_CAP;
  for (int c0 = 0; c0 < ncols; c0 += USORT) {
    const int nc = std::min(USORT, ncols - c0);
    const double* cc = cols + (long long)c0 * len;
    const long long Nc = len * nc;
    size_t bytes = s.cub_bytes;
    static const bool split = getenv("RTD_UNI_CLUSTER_SPLIT") != nullptr;  // r02 path: sort, then k_uni_small
    if (csort && !split && len <= (long long)UCS_CL * UCS_CAP && len / 2 + 1 <= (long long)UCS_CL * UCS_CAP) {
      // sort + scans + window + reweighting in one cluster launch per batch of columns
      const int dyn = 3 * UCS_CAP * (int)sizeof(unsigned long long);
      set_max_dyn_smem(reinterpret_cast<const void*>(k_uni_cluster_mcd), dyn);
      k_uni_cluster_mcd<<<nc * UCS_CL, UCM_T, dyn, st>>>(cc, len, h, uc, out_dev + c0);
      RTD_LAUNCHED();
      continue;
    }
    if (csort) {  // one 8-CTA cluster per column, no library sort
      const int dyn = 4 * UCS_CAP * (int)sizeof(unsigned long long);
      set_max_dyn_smem(reinterpret_cast<const void*>(k_uni_cluster_sort), dyn);
      k_uni_cluster_sort<<<nc * UCS_CL, UCS_T, dyn, st>>>(cc, len, s.sorted);
      RTD_LAUNCHED();
      if (len <= USORTED) {  // the scans, windows and reweighting of each sorted column in one CTA
        const int smem = (int)((((len + 3) & ~3LL) * sizeof(double)) + (UST + 1) * sizeof(dd2));
        set_max_dyn_smem(reinterpret_cast<const void*>(k_uni_small<true>), smem);
        k_uni_small<true><<<nc, UST, smem, st>>>(s.sorted, (int)len, (int)h, uc, out_dev + c0);
        RTD_LAUNCHED();
        continue;
      }
    } else if (nc == 1) {
      count_sort();
      RTD_CU(cub::DeviceRadixSort::SortKeys(s.cub_tmp, bytes, cc, s.sorted, (int)Nc, 0, 64, st));
    } else {
      k_fill_colid<<<(unsigned)std::min<long long>((Nc + 255) / 256, 148 * 16), 256, 0, st>>>(s.ids, len, Nc);
      RTD_LAUNCHED();
      count_sort();
      RTD_CU(cub::DeviceRadixSort::SortPairs(s.cub_tmp, bytes, cc, s.tmpk, s.ids, s.tmpid, (int)Nc, 0, 64, st));
      bytes = s.cub_bytes;
      count_sort();
      RTD_CU(cub::DeviceRadixSort::SortPairs(s.cub_tmp, bytes, s.tmpid, s.idout, s.tmpk, s.sorted, (int)Nc, 0,
                                             id_bits(nc), st));
    }
    k_uni_chunksum<<<dim3(nchunks, nc), UTH, 0, st>>>(s.sorted, len, nchunks, s.csum);
    RTD_LAUNCHED();
    k_uni_chunkscan<<<dim3(1, nc), 1024, 0, st>>>(s.csum, nchunks, s.coff);
    RTD_LAUNCHED();
    k_uni_window<<<dim3(nwchunks, nc), UTH, 0, st>>>(s.sorted, len, h, nchunks, s.coff, nwchunks, s.part);
    RTD_LAUNCHED();
    k_uni_final<<<nc, UTH, 0, st>>>(s.sorted, len, h, nchunks, s.coff, nwchunks, s.part, uc, out_dev + c0);
    RTD_LAUNCHED();
  }
}

}  // namespace rtd
