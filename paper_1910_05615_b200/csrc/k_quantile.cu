// Exact order statistics of the norms ||z_i|| of each block without sorting them, for the
// S~2 cut-offs A = median, B = A + 1.5 IQR (type-7 quantiles, reading R6).
//
// Per block: a strided sample fixes a monotone bucket map over its [0.5%, 99.5%] range
// (4096 buckets, under- and overflow buckets at the ends); one pass counts the bucket
// occupancies; a scan finds the bucket and the in-bucket offset of each target rank
// (j and j + 1 of each of the three quantiles); one pass gathers the elements of those
// buckets; each target is then read off its bucket's elements sorted in shared memory.
// The values returned are the exact order statistics (the bucket map only routes).
// A block whose target bucket holds more than QCAP elements (massive ties) is flagged
// and the caller sorts that block instead (same result).
#include <cstdlib>

#include "rtd_internal.h"

namespace rtd {

static constexpr int QNB = 4096;
static constexpr int QSAMPLE = 4096;
static constexpr int QCAP = 16384;  // elements of a target bucket sorted in shared memory (128 KB)
static constexpr int QT = 256;
static constexpr int QTARGETS = 6;

struct QMap {
  double lo, hi, inv_w;
  int status;  // 0 ok, 1 fall back to sorting
  int nbk;     // distinct target buckets
  int bk[QTARGETS];
  long long off[QTARGETS];  // in-bucket offset of each target rank
  int slot[QTARGETS];       // which gathered bucket holds each target
};

__device__ __forceinline__ int qbucket(double y, const QMap& c) {
  if (y < c.lo) return 0;
  if (y >= c.hi) return QNB - 1;
  int b = 1 + (int)__dmul_rn(__dsub_rn(y, c.lo), c.inv_w);
  return b > QNB - 2 ? QNB - 2 : (b < 1 ? 1 : b);
}

__device__ void q_bitonic(double* a, int npow2) {
  for (int k = 2; k <= npow2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const double x = a[i], y = a[ixj];
          if ((x > y) == up) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
}

__global__ void __launch_bounds__(1024) k_q_sample(const double* __restrict__ r_all, long long m, QMap* __restrict__ maps,
                                                   unsigned int* __restrict__ cnt_all, int* __restrict__ gcount) {
  __shared__ double s[QSAMPLE];
  const int b = blockIdx.x;
  const double* r = r_all + (long long)b * m;
  constexpr int V = QSAMPLE / 1024;  // blockDim.x == 1024
  unsigned long long x[V];
#pragma unroll
  for (int k = 0; k < V; k++) {
    const double y = r[(long long)(threadIdx.x * V + k) * m / QSAMPLE];
    x[k] = y == y ? ord_key64(y) : ~0ull;  // (a NaN norm sorts last; the input check rejects it anyway)
  }
  for (int i = threadIdx.x; i < QNB; i += blockDim.x) cnt_all[(long long)b * QNB + i] = 0u;
  if (threadIdx.x < QTARGETS) gcount[b * QTARGETS + threadIdx.x] = 0;
  // the sample's [0.5%, 99.5%] quantiles to 12 mantissa bits (the map only routes: any monotone map is exact)
  __shared__ unsigned long long qk[2];
  block_quantile_keys2<V>(x, QSAMPLE / 200, QSAMPLE - 1 - QSAMPLE / 200, reinterpret_cast<unsigned*>(s), qk);
  if (threadIdx.x == 0) {
    QMap c;
    memset(&c, 0, sizeof(c));
    const double ql = ord_val64(qk[0]), qh = ord_val64(qk[1]);
    const double span = qh - ql;
    c.lo = ql - 0.05 * span;
    c.hi = qh + 0.05 * span;
    const double w = (c.hi - c.lo) / (double)(QNB - 2);
    c.inv_w = w > 0.0 ? 1.0 / w : 0.0;
    c.status = (span > 0.0 && isfinite(span) && w > 0.0) ? 0 : 1;
    maps[b] = c;
  }
}

__global__ void __launch_bounds__(QT) k_q_hist(const double* __restrict__ r_all, long long m, const QMap* __restrict__ maps,
                                               unsigned int* __restrict__ cnt_all) {
  __shared__ unsigned int h[QNB];
  const int b = blockIdx.y;
  const QMap c = maps[b];
  if (c.status) return;
  for (int i = threadIdx.x; i < QNB; i += QT) h[i] = 0u;
  __syncthreads();
  const double* r = r_all + (long long)b * m;
  for (long long i = blockIdx.x * (long long)QT + threadIdx.x; i < m; i += (long long)gridDim.x * QT)
    atomicAdd(&h[qbucket(r[i], c)], 1u);
  __syncthreads();
  unsigned int* g = cnt_all + (long long)b * QNB;
  for (int i = threadIdx.x; i < QNB; i += QT)
    if (h[i]) atomicAdd(&g[i], h[i]);
}

// target ranks (0-based) j, j+1 of the type-7 positions (m - 1) * {0.25, 0.5, 0.75}
__device__ __forceinline__ long long q_target(long long m, int k) {
  const double prob = k < 2 ? 0.25 : (k < 4 ? 0.5 : 0.75);
  const long long j = (long long)floor((double)(m - 1) * prob);
  return min(m - 1, j + (k & 1));
}

__global__ void __launch_bounds__(1024) k_q_find(long long m, QMap* __restrict__ maps,
                                                 const unsigned int* __restrict__ cnt_all) {
  __shared__ long long wsum[32];
  __shared__ long long C[QNB + 1];
  const int b = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  QMap c = maps[b];
  if (c.status) return;
  const unsigned int* cn = cnt_all + (long long)b * QNB;
  constexpr int PER = QNB / 1024;
  long long loc = 0, v[PER];
#pragma unroll
  for (int e = 0; e < PER; e++) {
    v[e] = cn[t * PER + e];
    loc += v[e];
  }
  long long inc = loc;
  for (int d = 1; d < 32; d <<= 1) {
    long long x = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += x;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    long long x = wsum[lane], xi = x;
    for (int d = 1; d < 32; d <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, xi, d);
      if (lane >= d) xi += y;
    }
    wsum[lane] = xi - x;
  }
  __syncthreads();
  long long before = wsum[w] + inc - loc;
#pragma unroll
  for (int e = 0; e < PER; e++) {
    C[t * PER + e] = before;
    before += v[e];
  }
  if (t == 1023) C[QNB] = before;
  __syncthreads();
  if (t == 0) {
    c.nbk = 0;
    for (int k = 0; k < QTARGETS; k++) {
      const long long rk = q_target(m, k);
      int lo = 0, hi = QNB - 1;  // largest bucket with C[b] <= rk
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (C[mid] <= rk) lo = mid; else hi = mid - 1;
      }
      int sl = -1;
      for (int u = 0; u < c.nbk; u++)
        if (c.bk[u] == lo) sl = u;
      if (sl < 0) {
        sl = c.nbk++;
        c.bk[sl] = lo;
      }
      c.slot[k] = sl;
      c.off[k] = rk - C[lo];
      if (C[lo + 1] - C[lo] > QCAP) c.status = 1;
    }
    maps[b] = c;
  }
}

__global__ void __launch_bounds__(QT) k_q_gather(const double* __restrict__ r_all, long long m, const QMap* __restrict__ maps,
                                                 double* __restrict__ gbuf, int* __restrict__ gcount) {
  const int b = blockIdx.y;
  const QMap c = maps[b];
  if (c.status) return;
  const double* r = r_all + (long long)b * m;
  for (long long i = blockIdx.x * (long long)QT + threadIdx.x; i < m; i += (long long)gridDim.x * QT) {
    const double y = r[i];
    const int bk = qbucket(y, c);
    for (int u = 0; u < c.nbk; u++)
      if (bk == c.bk[u]) {
        const int pos = atomicAdd(&gcount[b * QTARGETS + u], 1);
        if (pos < QCAP) gbuf[((long long)b * QTARGETS + u) * QCAP + pos] = y;
      }
  }
}

// one CTA per (target, block): sort the target's bucket in shared memory, read the element at the offset
__global__ void __launch_bounds__(1024) k_q_pick(const QMap* __restrict__ maps, const double* __restrict__ gbuf,
                                                 const int* __restrict__ gcount, double* __restrict__ qv) {
  extern __shared__ double a[];  // QCAP doubles
  const int k = blockIdx.x, b = blockIdx.y;
  const QMap c = maps[b];
  if (c.status) return;
  const int u = c.slot[k];
  const int n = min(gcount[b * QTARGETS + u], QCAP);
  int np2 = 1;
  while (np2 < n) np2 <<= 1;
  const double* src = gbuf + ((long long)b * QTARGETS + u) * QCAP;
  for (int i = threadIdx.x; i < np2; i += blockDim.x) a[i] = i < n ? src[i] : INFINITY;
  __syncthreads();
  q_bitonic(a, np2);
  if (threadIdx.x == 0) qv[b * QTARGETS + k] = a[c.off[k]];
}

// fallback for a flagged block: read the targets off the sorted block
__global__ void k_q_from_sorted(const double* __restrict__ sorted, long long m, int b, double* __restrict__ qv) {
  if (threadIdx.x < QTARGETS) qv[b * QTARGETS + threadIdx.x] = sorted[q_target(m, threadIdx.x)];
}

// Fallback for a flagged block (a target bucket over QCAP elements: massive ties, or a degenerate sample span),
// on the device: the six order statistics by an exact radix select over all m norms (ordered 64-bit keys,
// digits of 12 bits from the top, a 4096-bin shared histogram per level among the keys that share the
// target's prefix, the last level 4 bits) -- one CTA per block, exits at once for an unflagged one.  No host
// round trip decides whether it is needed (the bucketed path used to read the flags back).
__global__ void __launch_bounds__(1024) k_q_exact(const double* __restrict__ r_all, long long m,
                                                  const QMap* __restrict__ maps, double* __restrict__ qv) {
  __shared__ unsigned int h[4096];
  __shared__ long long wsum[32];
  __shared__ int s_bin;
  __shared__ long long s_bef;
  const int b = blockIdx.x;
  if (!maps[b].status) return;
  const double* r = r_all + (long long)b * m;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  for (int k = 0; k < QTARGETS; k++) {
    long long rank = q_target(m, k);  // 0-based
    unsigned long long pre = 0ull;
    int plen = 0;
    while (plen < 64) {
      const int dig = plen + 12 <= 64 ? 12 : 64 - plen, sh = 64 - plen - dig;
      for (int i = t; i < 4096; i += blockDim.x) h[i] = 0u;
      __syncthreads();
      for (long long i = t; i < m; i += blockDim.x) {
        const unsigned long long key = ord_key64(r[i]);
        if (plen == 0 || (key >> (64 - plen)) == pre) atomicAdd(&h[(unsigned)(key >> sh) & ((1u << dig) - 1u)], 1u);
      }
      __syncthreads();
      // thread t owns bins 4t .. 4t+3 (1024 threads)
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
        const long long v = wsum[t];
        long long x = v;
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
          s_bin = 4 * t + e;
          s_bef = before;
        }
        before += c[e];
      }
      __syncthreads();
      pre = (pre << dig) | (unsigned long long)s_bin;
      rank -= s_bef;
      plen += dig;
      __syncthreads();
    }
    if (t == 0) qv[b * QTARGETS + k] = ord_val64(pre);
  }
}

// A = median, B = A + 1.5 IQR from the six order statistics (type-7 interpolation)
__global__ void k_q_cutoffs(const double* __restrict__ qv, long long m, int nb, double* __restrict__ AB,
                            int* __restrict__ ok) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  auto q7 = [&](int k, double prob) {
    const double hpos = (double)(m - 1) * prob;
    const double g = hpos - floor(hpos);
    const double y0 = qv[b * QTARGETS + 2 * k], y1 = qv[b * QTARGETS + 2 * k + 1];
    if ((long long)floor(hpos) + 1 >= m) return y0;
    return y0 + g * (y1 - y0);
  };
  const double A = q7(1, 0.5);
  const double iqr = q7(2, 0.75) - q7(0, 0.25);
  AB[2 * b] = A;
  AB[2 * b + 1] = A + 1.5 * iqr;
  ok[b] = iqr > 0.0 ? 1 : 0;
}

// median rule of the raw scatter: out[b] = (median of block b's d^2 / chi2_{p,0.5}) * Sigma_H of the chosen
// start; the median is the type-7 interpolation at 0.5 (numpy's median) of the targets j, j+1
__global__ void k_scale_median(const double* __restrict__ sig_all, const int* __restrict__ chosen_inst,
                               const double* __restrict__ qv, long long m, int p, double chi2half,
                               double* __restrict__ out_all) {
  const int b = blockIdx.x;
  const int ci = chosen_inst[b];
  if (ci < 0) return;
  const double hpos = (double)(m - 1) * 0.5;
  const double g = hpos - floor(hpos);
  const double y0 = qv[b * QTARGETS + 2], y1 = qv[b * QTARGETS + 3];
  const double med = ((long long)floor(hpos) + 1 >= m) ? y0 : y0 + g * (y1 - y0);
  const double f = med / chi2half;
  const double* S = sig_all + (long long)ci * RTD_MAXP * RTD_MAXP;
  double* O = out_all + (long long)b * RTD_MAXP * RTD_MAXP;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) O[e] = f * S[e];
}

void launch_scale_median(const double* sig_all, const int* chosen_inst, const double* qv, int q, long long m, int p,
                         double chi2half, double* out_all, cudaStream_t st) {
  k_scale_median<<<q, 256, 0, st>>>(sig_all, chosen_inst, qv, m, p, chi2half, out_all);
  RTD_LAUNCHED();
}

size_t quantile_scratch_bytes(int nb) {
  return (size_t)nb * (sizeof(QMap) + QNB * sizeof(unsigned int) + QTARGETS * (sizeof(int) + QCAP * sizeof(double) +
                                                                               sizeof(double))) + 4096;
}

// qv[nb][6] for the norms r_all[nb][m]; returns the blocks that must be sorted instead (host list)
void launch_quantiles(const double* r_all, long long m, int nb, char* scratch, double* qv, cudaStream_t st,
                      std::vector<int>& fallback) {
  Arena A;
  A.base = scratch;
  A.cap = quantile_scratch_bytes(nb);
  QMap* maps = A.take<QMap>(nb);
  unsigned int* cnt = A.take<unsigned int>((size_t)nb * QNB);
  int* gcount = A.take<int>((size_t)nb * QTARGETS);
  double* gbuf = A.take<double>((size_t)nb * QTARGETS * QCAP);
  k_q_sample<<<nb, 1024, 0, st>>>(r_all, m, maps, cnt, gcount);
  RTD_LAUNCHED();
  const unsigned gx = (unsigned)std::max<long long>(1, std::min<long long>((m + QT - 1) / QT, 148LL * 4 / nb + 1));
  k_q_hist<<<dim3(gx, nb), QT, 0, st>>>(r_all, m, maps, cnt);
  RTD_LAUNCHED();
  k_q_find<<<nb, 1024, 0, st>>>(m, maps, cnt);
  RTD_LAUNCHED();
  k_q_gather<<<dim3(gx, nb), QT, 0, st>>>(r_all, m, maps, gbuf, gcount);
  RTD_LAUNCHED();
  static const bool attr = [] {
    RTD_CU(cudaFuncSetAttribute(k_q_pick, cudaFuncAttributeMaxDynamicSharedMemorySize, QCAP * (int)sizeof(double)));
    return true;
  }();
  (void)attr;
  k_q_pick<<<dim3(QTARGETS, nb), 1024, QCAP * sizeof(double), st>>>(maps, gbuf, gcount, qv);
  RTD_LAUNCHED();
  fallback.clear();
  static const bool host_fb = getenv("RTD_Q_HOSTFALLBACK") != nullptr;  // r02: flags read back, CUB sort
  if (!host_fb) {
    k_q_exact<<<nb, 1024, 0, st>>>(r_all, m, maps, qv);
    RTD_LAUNCHED();
    return;
  }
  std::vector<QMap> h(nb);
  RTD_CU(cudaMemcpyAsync(h.data(), maps, nb * sizeof(QMap), cudaMemcpyDeviceToHost, st));
  RTD_CU(cudaStreamSynchronize(st));
  for (int b = 0; b < nb; b++)
    if (h[b].status) fallback.push_back(b);
}

void launch_q_from_sorted(const double* sorted, long long m, int b, double* qv, cudaStream_t st) {
  k_q_from_sorted<<<1, 32, 0, st>>>(sorted, m, b, qv);
  RTD_LAUNCHED();
}

void launch_q_cutoffs(const double* qv, long long m, int nb, double* AB, int* ok, cudaStream_t st) {
  k_q_cutoffs<<<(nb + 127) / 128, 128, 0, st>>>(qv, m, nb, AB, ok);
  RTD_LAUNCHED();
}

}  // namespace rtd
