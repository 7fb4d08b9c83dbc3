// K7: exact selection of the h-subset (C-step items 2-3).
//
// H_new = the h rows with the smallest (d_i^2, i) — ties at the h-th distance
// broken by row position (reading R11).  Instead of sorting, an exact radix
// select walks the 96-bit composite key C_i = (bits(d_i^2) << 32) | i, which
// is unique per row and ordered like (d^2, i) because d^2 >= 0 so its IEEE
// bits are order-preserving.  Each level resolves a digit of the key with a
// shared-memory histogram; selection stops as soon as the bin holding the h-th
// key is fully inside the subset.  Membership is then one comparison per row,
// and the rows whose membership changed (delta) are listed.
//
// First level: from the second C-step on, the h-th distance moves little, so
// the first digit is the top 24 bits of the key (sign, exponent, 12 mantissa
// bits) measured from the previous step's h-th key minus 2048: 4094 bins of
// relative width 2^-12 around it, everything below / above counted in the two
// end bins (warp-aggregated, no atomic contention).  If the h-th key falls in
// an end bin the level is discarded and the plain 12-bit levels run.  Each
// level is one launch: the last CTA of an instance to finish its histogram
// (threadfence + counter) scans it and advances the state.
//
// Candidate mode: once the bin holding the h-th key is at most 24 bits wide and holds at most SEL_CAND rows
// (after the centred level, or the second plain one), no further level runs: the membership pass decides
// every row outside the bin, reserves a changed-list slot (in row order) for every row inside it and lists
// them; k_sel_fixup then ranks the listed keys among themselves (counting), decides their membership, fills
// the slots of those that changed (a slot left 0 is skipped by the consumers) and records the h-th key --
// one pass over d^2 fewer per step (two when a third level was needed).
#include "rtd_internal.h"

namespace rtd {

static constexpr int SEL_BITS = 12;
static constexpr int SEL_BINS = 1 << SEL_BITS;
static constexpr int SEL_MAXLEV = 10;  // 1 centred level that may fail + 8 plain levels (96 bits) + slack
static constexpr int SEL_FAST = 3;     // levels launched before the host checks completion
static constexpr int SEL_T = 256;
static constexpr int SILP = 4;         // rows per thread in flight in the membership pass
static constexpr int SILP_L = 16;      // ... in the histogram levels (4 left the centred level latency-bound, ~2 TB/s)

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 composite(double d2, long long i) {
  unsigned long long key = (unsigned long long)__double_as_longlong(d2);
  return ((u128)key << 32) | (u128)(unsigned int)i;
}

__global__ void k_sel_init(const int* __restrict__ inst, SelState* __restrict__ st_all, unsigned int* __restrict__ cnt_all,
                           long long h, int* __restrict__ cand_cnt) {
  const int id = inst[blockIdx.x];
  if (threadIdx.x == 0) {
    const SelState old = st_all[id];
    SelState s;
    s.prefix_hi = 0;
    s.prefix_lo = 0;
    s.rank = h;
    s.plen = 0;
    s.done = 0;
    s.count_in = 0;
    s.centred = 0;
    s.base = 0;
    s.candok = 0;
    s.bincnt = 0;
    if (old.valid && old.plen >= 24) {
      const u128 pre = ((u128)old.prefix_hi << 64) | (u128)old.prefix_lo;
      const unsigned long long top24 = (unsigned long long)(pre >> (old.plen - 24));
      s.centred = 1;
      s.base = top24 > 2048 ? top24 - 2048 : 0;
    }
    s.valid = 0;
    st_all[id] = s;
    cnt_all[id] = 0;
    cand_cnt[id] = 0;
  }
}

// one level: histogram of the current digit (CTAs of blockIdx.y's instance), then the last CTA scans it
__global__ void __launch_bounds__(SEL_T) k_sel_level(const double* __restrict__ d2_all, long long m,
                                                     const int* __restrict__ inst, SelState* __restrict__ st_all,
                                                     unsigned int* __restrict__ hist_all,
                                                     unsigned int* __restrict__ cnt_all, int cand_mode) {
  __shared__ unsigned int sh[SEL_BINS];
  __shared__ long long wsum[SEL_T / 32];
  __shared__ int found_bin;
  __shared__ long long found_before, found_cnt;
  __shared__ bool last;
  const int id = inst[blockIdx.y];
  SelState s = st_all[id];
  if (s.done || s.candok) return;
  for (int b = threadIdx.x; b < SEL_BINS; b += SEL_T) sh[b] = 0;
  __syncthreads();
  const double* d2 = d2_all + (long long)id * m;
  const u128 prefix = ((u128)s.prefix_hi << 64) | (u128)s.prefix_lo;
  const bool centred = s.centred && s.plen == 0;
  const int lane = threadIdx.x & 31;
  unsigned int below = 0, above = 0;
  // SILP loads in flight per thread (a one-load-per-iteration loop left the pass at ~1.6 TB/s)
  const long long stride = (long long)gridDim.x * SEL_T;
  for (long long i0 = blockIdx.x * (long long)SEL_T + threadIdx.x; i0 < m; i0 += stride * SILP_L) {
    double v[SILP_L];
#pragma unroll
    for (int u = 0; u < SILP_L; u++) {
      const long long i = i0 + u * stride;
      v[u] = i < m ? __ldg(d2 + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < SILP_L; u++) {
      const long long i = i0 + u * stride;
      if (i >= m) break;
      if (centred) {
        const unsigned long long top24 = (unsigned long long)__double_as_longlong(v[u]) >> 40;
        if (top24 < s.base) below++;
        else if (top24 >= s.base + (SEL_BINS - 2)) above++;
        else atomicAdd(&sh[top24 - s.base + 1], 1u);
      } else {
        const u128 C = composite(v[u], i);
        if (s.plen == 0 || (C >> (96 - s.plen)) == prefix)
          atomicAdd(&sh[(unsigned int)(C >> (96 - s.plen - SEL_BITS)) & (SEL_BINS - 1)], 1u);
      }
    }
  }
  if (centred) {
    for (int d = 16; d > 0; d >>= 1) {
      below += __shfl_down_sync(0xffffffffu, below, d);
      above += __shfl_down_sync(0xffffffffu, above, d);
    }
    if (lane == 0) {
      if (below) atomicAdd(&sh[0], below);
      if (above) atomicAdd(&sh[SEL_BINS - 1], above);
    }
  }
  __syncthreads();
  unsigned int* hg = hist_all + (long long)id * SEL_BINS;
  for (int b = threadIdx.x; b < SEL_BINS; b += SEL_T)
    if (sh[b]) atomicAdd(&hg[b], sh[b]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&cnt_all[id], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  // ---- scan (last CTA of the instance): 16 contiguous bins per thread
  __threadfence();
  constexpr int PER = SEL_BINS / SEL_T;
  const int t = threadIdx.x, w = t >> 5;
  long long c[PER], loc = 0;
#pragma unroll
  for (int e = 0; e < PER; e++) {
    c[e] = atomicAdd(&hg[t * PER + e], 0u);  // coherent read of the global histogram
    loc += c[e];
  }
  long long inc = loc;
  for (int d = 1; d < 32; d <<= 1) {
    long long v = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += v;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (t == 0) {
    long long acc = 0;
    for (int k = 0; k < SEL_T / 32; k++) {
      long long v = wsum[k];
      wsum[k] = acc;
      acc += v;
    }
  }
  __syncthreads();
  long long before = wsum[w] + inc - loc;
#pragma unroll
  for (int e = 0; e < PER; e++) {
    if (c[e] > 0 && before < s.rank && s.rank <= before + c[e]) {
      found_bin = t * PER + e;
      found_before = before;
      found_cnt = c[e];
    }
    before += c[e];
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < PER; e++) hg[t * PER + e] = 0;  // clean for the next level
  if (t == 0) {
    cnt_all[id] = 0;
    if (centred && (found_bin == 0 || found_bin == SEL_BINS - 1)) {
      s.centred = 0;  // the h-th key left the window: plain levels from the top
    } else {
      u128 pre = prefix;
      if (centred) {
        pre = (u128)(s.base + (unsigned long long)found_bin - 1ull);
        s.plen = 24;
        s.centred = 0;
      } else {
        pre = (pre << SEL_BITS) | (u128)found_bin;
        s.plen += SEL_BITS;
      }
      s.prefix_hi = (unsigned long long)(pre >> 64);
      s.prefix_lo = (unsigned long long)pre;
      s.count_in += found_before;
      s.rank -= found_before;
      s.bincnt = found_cnt;
      if (found_cnt == s.rank || s.plen >= 96) {
        s.done = 1;
        s.valid = 1;
      } else if (cand_mode && s.plen >= 24 && found_cnt <= SEL_CAND) {
        s.candok = 1;
      }
    }
    st_all[id] = s;
  }
}

// Membership of every row, the count of rows whose membership changed, and the
// ordered list of those rows (row + 1 entering, -(row + 1) leaving):
// CTA x owns rows [x seg_len, (x+1) seg_len) and writes its changed rows, in row
// order, to list[x seg_len ...] with the count in seg_cnt[x].  The update-based
// moments then gather only those rows, in a fixed order (deterministic sums).
__global__ void __launch_bounds__(SEL_T) k_sel_member(const double* __restrict__ d2_all, long long m,
                                                      const int* __restrict__ inst,
                                                      const SelState* __restrict__ st_all,
                                                      uint8_t* __restrict__ mem_new_all,
                                                      const uint8_t* __restrict__ mem_old_all,
                                                      int* __restrict__ changed, int* __restrict__ list_all,
                                                      int* __restrict__ seg_cnt_all, long long seg_len,
                                                      SelCand* __restrict__ cand_all, int* __restrict__ cand_cnt) {
  __shared__ int wc2[SILP][SEL_T / 32];
  __shared__ int woff2[SILP + 1][SEL_T / 32];
  __shared__ int s_ncd;
  const int id = inst[blockIdx.y];
  const SelState s = st_all[id];
  if (!s.done && !s.candok) {  // more levels needed: the host relaunches the selection (launch_select_finish)
    if (blockIdx.x == 0 && threadIdx.x == 0) changed[id] = -1;
    return;
  }
  const bool cmode = !s.done;  // candidate mode: the rows of the prefix's bin are listed, decided by k_sel_fixup
  if (threadIdx.x == 0) s_ncd = 0;
  __syncthreads();
  const u128 prefix = ((u128)s.prefix_hi << 64) | (u128)s.prefix_lo;
  const int sh = 96 - s.plen;
  const bool fast = s.plen >= 1 && s.plen <= 64;
  const int sh64 = 64 - s.plen;
  const unsigned long long p64 = s.prefix_lo;
  const double* d2 = d2_all + (long long)id * m;
  uint8_t* mn = mem_new_all + (long long)id * m;
  const uint8_t* mo = mem_old_all + (long long)id * m;
  const long long r_begin = (long long)blockIdx.x * seg_len, r_end = min(m, r_begin + seg_len);
  int* list = list_all + (long long)id * m + r_begin;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int base = 0;  // entries written by this CTA so far (uniform)
  // SILP sub-chunks of SEL_T rows per iteration: their loads in flight together, one offset scan for all
  // (sub-chunk-major = row order), two barriers per SILP * SEL_T rows
  for (long long c0 = r_begin; c0 < r_end; c0 += (long long)SEL_T * SILP) {
    double dv[SILP];
    uint8_t ov[SILP];
#pragma unroll
    for (int u = 0; u < SILP; u++) {
      const long long i = c0 + u * SEL_T + threadIdx.x;
      dv[u] = i < r_end ? __ldg(d2 + i) : 0.0;
      ov[u] = i < r_end ? mo[i] : 0;
    }
    bool ch[SILP], in[SILP], cd[SILP];
    unsigned bal[SILP];
    int real = 0;  // candidate rows (reserved slots) among this thread's
#pragma unroll
    for (int u = 0; u < SILP; u++) {
      const long long i = c0 + u * SEL_T + threadIdx.x;
      ch[u] = in[u] = cd[u] = false;
      if (i < r_end) {
        if (fast) {  // the prefix lies inside the d^2 bits: 64-bit compares
          const unsigned long long top = (unsigned long long)__double_as_longlong(dv[u]) >> sh64;
          in[u] = cmode ? top < p64 : top <= p64;
          cd[u] = cmode && top == p64;
        } else {
          const u128 top = composite(dv[u], i) >> sh;
          in[u] = cmode ? top < prefix : top <= prefix;
          cd[u] = cmode && top == prefix;
        }
        if (!cd[u]) mn[i] = in[u] ? 1 : 0;
        ch[u] = cd[u] || ((in[u] ? 1 : 0) != ov[u]);
      }
      bal[u] = __ballot_sync(0xffffffffu, ch[u]);
      real += cd[u] ? 1 : 0;
      if (lane == 0) wc2[u][w] = __popc(bal[u]);
    }
    if (real) atomicAdd(&s_ncd, real);  // (candidate rows of this CTA: rare)
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int u = 0; u < SILP; u++)
        for (int k = 0; k < SEL_T / 32; k++) {
          woff2[u][k] = acc;
          acc += wc2[u][k];
        }
      woff2[SILP][0] = acc;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < SILP; u++)
      if (ch[u]) {
        const long long i = c0 + u * SEL_T + threadIdx.x;
        const int pos = base + woff2[u][w] + __popc(bal[u] & ((1u << lane) - 1u));
        if (cd[u]) {  // a reserved slot, filled by k_sel_fixup if the row changed
          list[pos] = 0;
          const int k = atomicAdd(&cand_cnt[id], 1);
          if (k < SEL_CAND)
            cand_all[(long long)id * SEL_CAND + k] = {(unsigned long long)__double_as_longlong(dv[u]), (int)i,
                                                      (int)(r_begin + pos)};
        } else {
          list[pos] = in[u] ? (int)(i + 1) : -(int)(i + 1);
        }
      }
    base += woff2[SILP][0];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    seg_cnt_all[(long long)id * gridDim.x + blockIdx.x] = base;
    // entries written minus the reserved candidate slots (changed[id] was zeroed by the host before the select)
    if (base - s_ncd) atomicAdd(&changed[id], base - s_ncd);
  }
}

// Candidate mode: rank the bin's rows among themselves by their composite keys (bits(d^2), row) -- unique --,
// in iff fewer than `rank` of them are smaller; the h-th key is recorded as the state's full 96-bit prefix
// (done, valid: it centres the next step's first level).
__global__ void __launch_bounds__(256) k_sel_fixup(long long m, const int* __restrict__ inst,
                                                    SelState* __restrict__ st_all, uint8_t* __restrict__ mem_new_all,
                                                    const uint8_t* __restrict__ mem_old_all, int* __restrict__ changed,
                                                    int* __restrict__ list_all, const SelCand* __restrict__ cand_all,
                                                    const int* __restrict__ cand_cnt) {
  extern __shared__ unsigned long long fx[];  // [SEL_CAND] d^2 bits, then [SEL_CAND] rows
  unsigned int* fr = reinterpret_cast<unsigned int*>(fx + SEL_CAND);
  __shared__ int s_chg;
  const int id = inst[blockIdx.y];  // blockIdx.x: a slice of the candidates (every CTA ranks against all)
  const SelState s = st_all[id];
  if (!s.candok || s.done) return;
  const int n = min(cand_cnt[id], SEL_CAND);
  const SelCand* cd = cand_all + (long long)id * SEL_CAND;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    fx[j] = cd[j].kb;
    fr[j] = (unsigned)cd[j].row;
  }
  if (threadIdx.x == 0) s_chg = 0;
  __syncthreads();
  uint8_t* mn = mem_new_all + (long long)id * m;
  const uint8_t* mo = mem_old_all + (long long)id * m;
  int chg = 0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const unsigned long long kj = fx[j];
    const unsigned rj = fr[j];
    long long less = 0;
    for (int k = 0; k < n; k++) less += (fx[k] < kj || (fx[k] == kj && fr[k] < rj)) ? 1 : 0;
    const bool in = less < s.rank;
    mn[rj] = in ? 1 : 0;
    if ((in ? 1 : 0) != mo[rj]) {
      list_all[(long long)id * m + cd[j].listpos] = in ? (int)(rj + 1) : -(int)(rj + 1);
      chg++;
    }
    if (less == s.rank - 1) {  // the h-th key
      SelState o = s;
      const u128 C = ((u128)kj << 32) | (u128)rj;
      o.prefix_hi = (unsigned long long)(C >> 64);
      o.prefix_lo = (unsigned long long)C;
      o.plen = 96;
      o.rank = 1;
      o.done = 1;
      o.valid = 1;
      o.candok = 0;
      st_all[id] = o;
    }
  }
  for (int d = 16; d > 0; d >>= 1) chg += __shfl_down_sync(0xffffffffu, chg, d);
  if ((threadIdx.x & 31) == 0 && chg) atomicAdd(&s_chg, chg);
  __syncthreads();
  if (threadIdx.x == 0 && s_chg) atomicAdd(&changed[id], s_chg);
}

static unsigned sel_grid(long long m, int ninst) {
  static const int per_sm = getenv("RTD_SEL_CTAS_PER_SM") ? atoi(getenv("RTD_SEL_CTAS_PER_SM")) : 4;
  return (unsigned)std::min<long long>((m + SEL_T - 1) / SEL_T, std::max(1, 148 * per_sm / std::max(1, ninst)));
}

bool sel_cand_mode() {
  static const bool off = getenv("RTD_SEL_NOCAND") != nullptr;  // r02 path: radix levels to the end
  return !off;
}

static void launch_fixup(long long m, const int* inst, int ninst, SelState* st_all, uint8_t* mem_new_all,
                         const uint8_t* mem_old_all, int* changed, int* list_all, const SelCand* cand_all,
                         const int* cand_cnt, cudaStream_t st) {
  if (!sel_cand_mode()) return;
  constexpr int smem = SEL_CAND * (int)(sizeof(unsigned long long) + sizeof(unsigned int));
  static const bool attr = [] {
    RTD_CU(cudaFuncSetAttribute(k_sel_fixup, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    return true;
  }();
  (void)attr;
  k_sel_fixup<<<dim3(8, ninst), 256, smem, st>>>(m, inst, st_all, mem_new_all, mem_old_all, changed, list_all, cand_all,
                                         cand_cnt);
  RTD_LAUNCHED();
}

void launch_select(const double* d2_all, long long m, long long h, const int* inst, int ninst, SelState* st_all,
                   unsigned int* hist_all, unsigned int* cnt_all, uint8_t* mem_new_all, const uint8_t* mem_old_all,
                   int* changed, int* list_all, int* seg_cnt_all, int nseg, long long seg_len, SelCand* cand_all,
                   int* cand_cnt, cudaStream_t st, int nfast) {
  k_sel_init<<<ninst, 32, 0, st>>>(inst, st_all, cnt_all, h, cand_cnt);
  RTD_LAUNCHED();
  const unsigned gx = sel_grid(m, ninst);
  const int cm = sel_cand_mode() ? 1 : 0;
  for (int L = 0; L < nfast; L++) {  // (a level exits at once once the instance is done or in candidate mode)
    k_sel_level<<<dim3(gx, ninst), SEL_T, 0, st>>>(d2_all, m, inst, st_all, hist_all, cnt_all, cm);
    RTD_LAUNCHED();
  }
  k_sel_member<<<dim3(nseg, ninst), SEL_T, 0, st>>>(d2_all, m, inst, st_all, mem_new_all, mem_old_all, changed,
                                                     list_all, seg_cnt_all, seg_len, cand_all, cand_cnt);
  RTD_LAUNCHED();
  launch_fixup(m, inst, ninst, st_all, mem_new_all, mem_old_all, changed, list_all, cand_all, cand_cnt, st);
}

// the rare case: some instance needed more than SEL_FAST levels (changed[id] == -1 after launch_select)
void launch_select_finish(const double* d2_all, long long m, const int* inst, int ninst, SelState* st_all,
                          unsigned int* hist_all, unsigned int* cnt_all, uint8_t* mem_new_all,
                          const uint8_t* mem_old_all, int* changed, int* list_all, int* seg_cnt_all, int nseg,
                          long long seg_len, SelCand* cand_all, int* cand_cnt, cudaStream_t st) {
  const unsigned gx = sel_grid(m, ninst);
  const int cm = sel_cand_mode() ? 1 : 0;
  for (int L = 0; L < SEL_MAXLEV - 1; L++) {  // (as many as the state may still need; done levels exit at once)
    k_sel_level<<<dim3(gx, ninst), SEL_T, 0, st>>>(d2_all, m, inst, st_all, hist_all, cnt_all, cm);
    RTD_LAUNCHED();
  }
  k_sel_member<<<dim3(nseg, ninst), SEL_T, 0, st>>>(d2_all, m, inst, st_all, mem_new_all, mem_old_all, changed,
                                                     list_all, seg_cnt_all, seg_len, cand_all, cand_cnt);
  RTD_LAUNCHED();
  launch_fixup(m, inst, ninst, st_all, mem_new_all, mem_old_all, changed, list_all, cand_all, cand_cnt, st);
}

}  // namespace rtd
