// K7: exact selection of the h-subset (C-step items 2-3).
//
// H_new = the h rows with the smallest (d_i^2, i) — ties at the h-th distance
// broken by row position (reading R11).  Instead of sorting, an exact radix
// select walks the 95-bit composite key C_i = (bits(d_i^2) << 32) | i, which
// is unique per row and ordered like (d^2, i) because d^2 >= 0 so its IEEE
// bits are order-preserving.  Each level resolves 12 bits with a shared-memory
// histogram; selection stops as soon as the bin holding the h-th key is fully
// inside the subset.  Membership is then one comparison per row, and the
// number of rows whose membership changed (|delta|) is
// counted for the convergence test.
#include "rtd_internal.h"

namespace rtd {

static constexpr int SEL_BITS = 12;
static constexpr int SEL_BINS = 1 << SEL_BITS;
static constexpr int SEL_LEVELS = 8;  // 96 bits >= 95
static constexpr int SEL_T = 256;

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 composite(double d2, long long i) {
  unsigned long long key = (unsigned long long)__double_as_longlong(d2);
  return ((u128)key << 32) | (u128)(unsigned int)i;
}

__global__ void k_sel_init(const int* __restrict__ inst, SelState* __restrict__ st_all, long long h) {
  const int id = inst[blockIdx.x];
  if (threadIdx.x == 0) {
    SelState s;
    s.prefix_hi = 0;
    s.prefix_lo = 0;
    s.rank = h;
    s.level = 0;
    s.done = 0;
    s.count_in = 0;
    st_all[id] = s;
  }
}

__global__ void __launch_bounds__(SEL_T) k_sel_hist(const double* __restrict__ d2_all, long long m,
                                                    const int* __restrict__ inst, const SelState* __restrict__ st_all,
                                                    unsigned int* __restrict__ hist_all, int level) {
  __shared__ unsigned int sh[SEL_BINS];
  const int id = inst[blockIdx.y];
  const SelState s = st_all[id];
  if (s.done || s.level != level) return;
  for (int b = threadIdx.x; b < SEL_BINS; b += SEL_T) sh[b] = 0;
  __syncthreads();
  const double* d2 = d2_all + (long long)id * m;
  const u128 prefix = ((u128)s.prefix_hi << 64) | (u128)s.prefix_lo;
  const int shift_pref = 96 - SEL_BITS * level;        // bits above this level
  const int shift_dig = 96 - SEL_BITS * (level + 1);
  for (long long i = blockIdx.x * (long long)SEL_T + threadIdx.x; i < m; i += (long long)gridDim.x * SEL_T) {
    u128 C = composite(d2[i], i);
    if (level == 0 || (C >> shift_pref) == prefix) {
      unsigned int dig = (unsigned int)(C >> shift_dig) & (SEL_BINS - 1);
      atomicAdd(&sh[dig], 1u);
    }
  }
  __syncthreads();
  unsigned int* hg = hist_all + (long long)id * SEL_BINS;
  for (int b = threadIdx.x; b < SEL_BINS; b += SEL_T)
    if (sh[b]) atomicAdd(&hg[b], sh[b]);
}

__global__ void __launch_bounds__(1024) k_sel_scan(const int* __restrict__ inst, SelState* __restrict__ st_all,
                                                   unsigned int* __restrict__ hist_all, int level) {
  __shared__ long long wsum[32];
  __shared__ int found_bin;
  __shared__ long long found_before, found_cnt;
  const int id = inst[blockIdx.x];
  SelState s = st_all[id];
  if (s.done || s.level != level) return;
  unsigned int* hg = hist_all + (long long)id * SEL_BINS;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  // 4 bins per thread, contiguous
  long long c[4], loc = 0;
#pragma unroll
  for (int e = 0; e < 4; e++) {
    c[e] = hg[t * 4 + e];
    loc += c[e];
  }
  long long inc = loc;
  for (int d = 1; d < 32; d <<= 1) {
    long long v = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += v;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    long long v = wsum[lane], vi = v;
    for (int d = 1; d < 32; d <<= 1) {
      long long u = __shfl_up_sync(0xffffffffu, vi, d);
      if (lane >= d) vi += u;
    }
    wsum[lane] = vi - v;
  }
  __syncthreads();
  long long before = wsum[w] + inc - loc;
#pragma unroll
  for (int e = 0; e < 4; e++) {
    if (c[e] > 0 && before < s.rank && s.rank <= before + c[e]) {
      found_bin = t * 4 + e;
      found_before = before;
      found_cnt = c[e];
    }
    before += c[e];
  }
  __syncthreads();
  // clear this instance's histogram for the next level
#pragma unroll
  for (int e = 0; e < 4; e++) hg[t * 4 + e] = 0;
  if (t == 0) {
    u128 prefix = ((u128)s.prefix_hi << 64) | (u128)s.prefix_lo;
    prefix = (prefix << SEL_BITS) | (u128)found_bin;
    s.prefix_hi = (unsigned long long)(prefix >> 64);
    s.prefix_lo = (unsigned long long)prefix;
    s.count_in += found_before;
    s.rank -= found_before;
    s.level = level + 1;
    if (found_cnt == s.rank || s.level == SEL_LEVELS) s.done = 1;
    st_all[id] = s;
  }
}

__global__ void __launch_bounds__(SEL_T) k_sel_member(const double* __restrict__ d2_all, long long m,
                                                      const int* __restrict__ inst,
                                                      const SelState* __restrict__ st_all,
                                                      uint8_t* __restrict__ mem_new_all,
                                                      const uint8_t* __restrict__ mem_old_all,
                                                      int* __restrict__ changed) {
  __shared__ int wc[SEL_T / 32];
  const int id = inst[blockIdx.y];
  const SelState s = st_all[id];
  const u128 prefix = ((u128)s.prefix_hi << 64) | (u128)s.prefix_lo;
  const int sh = 96 - SEL_BITS * s.level;
  const double* d2 = d2_all + (long long)id * m;
  uint8_t* mn = mem_new_all + (long long)id * m;
  const uint8_t* mo = mem_old_all + (long long)id * m;
  int cnt = 0;
  for (long long i = blockIdx.x * (long long)SEL_T + threadIdx.x; i < m; i += (long long)gridDim.x * SEL_T) {
    u128 C = composite(d2[i], i);
    uint8_t in = (C >> sh) <= prefix ? 1 : 0;
    mn[i] = in;
    cnt += (in != mo[i]);
  }
  for (int d = 16; d > 0; d >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, d);
  if ((threadIdx.x & 31) == 0) wc[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int k = 0; k < SEL_T / 32; k++) tot += wc[k];
    if (tot) atomicAdd(&changed[id], tot);
  }
}

void launch_select(const double* d2_all, long long m, long long h, const int* inst, int ninst, SelState* st_all,
                   unsigned int* hist_all, uint8_t* mem_new_all, const uint8_t* mem_old_all, int* changed,
                   cudaStream_t st) {
  k_sel_init<<<ninst, 32, 0, st>>>(inst, st_all, h);
  RTD_LAUNCHED();
  unsigned gx = (unsigned)std::min<long long>((m + SEL_T - 1) / SEL_T, std::max(1, 148 * 4 / std::max(1, ninst)));
  for (int L = 0; L < SEL_LEVELS; L++) {
    k_sel_hist<<<dim3(gx, ninst), SEL_T, 0, st>>>(d2_all, m, inst, st_all, hist_all, L);
    RTD_LAUNCHED();
    k_sel_scan<<<ninst, 1024, 0, st>>>(inst, st_all, hist_all, L);
    RTD_LAUNCHED();
  }
  unsigned gm = (unsigned)std::min<long long>((m + SEL_T - 1) / SEL_T, std::max(1, 148 * 8 / std::max(1, ninst)));
  k_sel_member<<<dim3(gm, ninst), SEL_T, 0, st>>>(d2_all, m, inst, st_all, mem_new_all, mem_old_all, changed);
  RTD_LAUNCHED();
}

}  // namespace rtd
