// K4 / K11: single-CTA dense linear algebra for p <= 40, one CTA per instance.
//   k_prepare   Cholesky Sigma = L L^T, log det = 2 sum log L_jj
//               (PAPER.md:637-641), exact inverse -> ||Sigma||_1 ||Sigma^-1||_1 >= kappa_max
//               test, and the distance operator [mu | L^-1] staged
//               for the constant bank.
//   k_jacobi    cyclic Jacobi eigen-decomposition with round-robin parallel
//               pairs, eigenvalues descending and the
//               kappa_max check of refinement step 2.
//   k_refine    Sigma_k = V D~ V^T, Sigma_k^{+-1/2}.
//   k_sums_to_cov  mean / covariance from shifted sums (eqs. cstep4a/b).
//   k_aggregate entrywise median, KL ranking, ceil(q/2) kept, pooling.
#include <algorithm>

#include <cooperative_groups.h>

#include "rtd_internal.h"
#include "rtd_linalg.h"
#include <cstdio>
#include <cstdlib>

namespace rtd {

static constexpr int LT = 256;
static constexpr int LD = RTD_MAXP + 1;

// The helpers take flat shared arrays (row stride LD) and contain no early
// return inside loops: nvcc 12.9 for sm_100a emitted a use-before-def register
// (stores landing one element off) for a 2-D-array-parameter version with an
// in-loop return (tools/t_min3.cu reproduces it; tools/t_min4.cu is this form).

// Cholesky of the p x p matrix in A into L; returns false if not PD.  Right-looking: per column j
// one pivot (every thread reads the same updated diagonal, so the decision is uniform), the column
// scaled by 1 / L_jj and a rank-1 update of the trailing triangle in parallel -- two barriers per
// column and no dependent chain longer than one FMA (the left-looking form had a length-j dot product
// on one thread per column: ~64 us per launch at p = 40, dominated by barrier waits).
__device__ __noinline__ bool block_cholesky(const double* A, double* L, int p, int* s_fail) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = blockDim.x >> 5;
  if (t == 0) *s_fail = 0;
  // rows to warps, columns to lanes: no integer division in the index maps
  for (int i = wid; i < RTD_MAXP; i += nw)
    for (int k = lane; k < LD; k += 32) L[i * LD + k] = (i < p && k <= i) ? A[i * LD + k] : 0.0;
  __syncthreads();
  bool ok = true;
  for (int j = 0; j < p; j++) {
    const double d = L[j * LD + j];
    if (!(d > 0.0) || !isfinite(d)) {
      ok = false;
      break;
    }
    const double r = sqrt(d);
    __syncthreads();  // every thread has read the pivot before it is overwritten
    if (t == 0) L[j * LD + j] = r;
    for (int i = j + 1 + t; i < p; i += blockDim.x) L[i * LD + j] /= r;
    __syncthreads();
    for (int i = j + 1 + wid; i < p; i += nw) {
      const double lij = L[i * LD + j];
      for (int k = j + 1 + lane; k <= i; k += 32) L[i * LD + k] = fma(-lij, L[k * LD + j], L[i * LD + k]);
    }
    __syncthreads();
  }
  if (!ok && t == 0) *s_fail = 1;
  __syncthreads();
  return ok;
}

// Li = L^-1 (lower triangular): row-wise forward substitution L X = I, right-looking -- row k of X
// is final once divided by L_kk, then its contribution is removed from the rows below in parallel.
__device__ __noinline__ void block_tri_inverse(const double* L, double* Li, int p) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = blockDim.x >> 5;
  for (int i = wid; i < RTD_MAXP; i += nw)
    for (int k = lane; k < LD; k += 32) Li[i * LD + k] = (i == k && i < p) ? 1.0 : 0.0;
  __syncthreads();
  for (int k = 0; k < p; k++) {
    for (int c = t; c <= k; c += blockDim.x) Li[k * LD + c] /= L[k * LD + k];
    __syncthreads();
    for (int i = k + 1 + wid; i < p; i += nw) {
      const double lik = L[i * LD + k];
      for (int c = lane; c <= k; c += 32) Li[i * LD + c] = fma(-lik, Li[k * LD + c], Li[i * LD + c]);
    }
    __syncthreads();
  }
}

// Cholesky Sigma = L L^T and Li = L^-1 in ONE right-looking loop (same quantities as block_cholesky +
// block_tri_inverse): at step j the pivot r = sqrt(L_jj) is read by every thread (a uniform decision), column j
// of L and row j of Li (final after the earlier steps) are scaled by 1 / r, then the trailing triangle of L
// and the rows below j of Li are updated in one phase -- two barriers per step instead of five, the
// reciprocal computed once per thread instead of a division per element.  r is kept in rd[] until the loop
// ends (the pivot entry is read unsynchronised at the top of the step).
__device__ __noinline__ bool block_chol_inv(const double* A, double* L, double* Li, double* rd, int p, int* s_fail) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = blockDim.x >> 5;
  if (t == 0) *s_fail = 0;
  for (int i = wid; i < RTD_MAXP; i += nw)
    for (int k = lane; k < LD; k += 32) {
      L[i * LD + k] = (i < p && k <= i) ? A[i * LD + k] : 0.0;
      Li[i * LD + k] = (i == k && i < p) ? 1.0 : 0.0;
    }
  __syncthreads();
  bool ok = true;
  // two columns per step (a 2 x 2 pivot block, every thread computing it redundantly from the same shared
  // values): half the barriers of the one-column loop; a last single column when p is odd
  int j = 0;
  for (; j + 1 < p; j += 2) {
    const double d0 = L[j * LD + j];
    if (!(d0 > 0.0) || !isfinite(d0)) {
      ok = false;
      break;
    }
    const double r0i = rsqrt(d0), r0 = d0 * r0i;
    const double l10 = L[(j + 1) * LD + j] * r0i;
    const double d1 = fma(-l10, l10, L[(j + 1) * LD + j + 1]);
    if (!(d1 > 0.0) || !isfinite(d1)) {
      ok = false;
      break;
    }
    const double r1i = rsqrt(d1), r1 = d1 * r1i;
    if (t == 0) {
      rd[j] = r0;
      rd[j + 1] = r1;
    }
    for (int e = t; e < p; e += blockDim.x) {
      if (e >= j + 2) {  // columns j, j+1 of L below the pivot block
        const double li0 = L[e * LD + j] * r0i;
        L[e * LD + j] = li0;
        L[e * LD + j + 1] = fma(-li0, l10, L[e * LD + j + 1]) * r1i;
      } else {           // rows j, j+1 of Li (columns 0..j+1; Li[j][j+1] = 0)
        const double a0 = Li[j * LD + e] * r0i;
        Li[j * LD + e] = a0;
        Li[(j + 1) * LD + e] = fma(-l10, a0, Li[(j + 1) * LD + e]) * r1i;
      }
    }
    __syncthreads();
    if (t == 0) L[(j + 1) * LD + j] = l10;
    for (int i = j + 2 + wid; i < p; i += nw) {  // rank-2 updates of the rows below the block
      const double a0 = L[i * LD + j], a1 = L[i * LD + j + 1];
      for (int k = lane; k <= j + 1; k += 32)
        Li[i * LD + k] = fma(-a1, Li[(j + 1) * LD + k], fma(-a0, Li[j * LD + k], Li[i * LD + k]));
      for (int k = j + 2 + lane; k <= i; k += 32)
        L[i * LD + k] = fma(-a1, L[k * LD + j + 1], fma(-a0, L[k * LD + j], L[i * LD + k]));
    }
    __syncthreads();
  }
  if (ok && j < p) {  // the last column (p odd): its pivot and row j of Li
    const double d = L[j * LD + j];
    if (!(d > 0.0) || !isfinite(d)) {
      ok = false;
    } else {
      const double ri = rsqrt(d);
      if (t == 0) rd[j] = d * ri;
      for (int e = t; e <= j; e += blockDim.x) Li[j * LD + e] *= ri;
    }
    __syncthreads();
  }
  if (ok)
    for (int j = t; j < p; j += blockDim.x) L[j * LD + j] = rd[j];
  if (!ok && t == 0) *s_fail = 1;
  __syncthreads();
  return ok;
}

__device__ __noinline__ double block_max_colsum_abs(const double* A, int p, double* red) {
  const int t = threadIdx.x;
  if (t < p) {
    double s = 0.0;
    for (int i = 0; i < p; i++) s += fabs(A[i * LD + t]);
    red[t] = s;
  }
  __syncthreads();
  // every warp takes the max of the p column sums by a butterfly (max is exact: any order gives the same value)
  const int lane = t & 31;
  double mx = lane < p ? red[lane] : 0.0;
  if (lane + 32 < p) mx = fmax(mx, red[lane + 32]);
  for (int d = 16; d > 0; d >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
  __syncthreads();
  return mx;
}

// Sigma^-1 = Li^T Li into B
__device__ __noinline__ void block_inv_from_li(const double* Li, double* B, int p) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = wid; i < p; i += nw)
    for (int j = lane; j < p; j += 32) {
      const int k0 = i > j ? i : j;
      double s = 0.0;
      for (int k = k0; k < p; k++) s += Li[k * LD + i] * Li[k * LD + j];
      B[i * LD + j] = s;
    }
  __syncthreads();
}

__global__ void __launch_bounds__(512) k_prepare(const int* __restrict__ inst, const double* __restrict__ mu_all,
                                                const double* __restrict__ sigma_all, int p, double kappa_max,
                                                double* __restrict__ cstage, int cstride, double* __restrict__ logdet_out,
                                                double* __restrict__ cond_out, int* __restrict__ status_out,
                                                double* __restrict__ traj, int traj_stride, int step,
                                                int full_inverse, const int* __restrict__ skip) {
  __shared__ double A[RTD_MAXP * LD], L[RTD_MAXP * LD], Li[RTD_MAXP * LD];
  __shared__ double red[RTD_MAXP];
  __shared__ int s_fail;
  const int slot = blockIdx.x;
  const int id = inst[slot];
  const int t = threadIdx.x;
  if (status_out && status_out[id] != 0) return;  // instance no longer active
  if (skip && skip[id]) return;                    // operator already updated (SMW variant)
  const double* sg = sigma_all + (long long)id * RTD_MAXP * RTD_MAXP;
  for (int e = t; e < p * p; e += blockDim.x) A[(e / p) * LD + e % p] = sg[e];
  __syncthreads();
  const bool ok = block_chol_inv(A, L, Li, red, p, &s_fail);
  if (!ok) {
    if (t == 0 && status_out) status_out[id] = ST_NOT_PD;
    return;
  }
  const double n1 = block_max_colsum_abs(A, p, red);
  block_inv_from_li(Li, A, p);  // A <- Sigma^-1
  const double n1i = block_max_colsum_abs(A, p, red);
  const double kappa = n1 * n1i;
  if (t < p) red[t] = log(L[t * LD + t]);  // the logs in parallel, summed in row order by thread 0
  __syncthreads();
  if (t == 0) {
    double ld = 0.0;
    for (int j = 0; j < p; j++) ld += red[j];
    ld *= 2.0;
    if (logdet_out) logdet_out[id] = ld;
    if (cond_out) cond_out[id] = kappa;
    if (traj) traj[(long long)id * traj_stride + step] = ld;
    if (status_out && !(kappa < kappa_max)) status_out[id] = ST_COND;
  }
  if (cstage) {
    double* cs = cstage + (long long)slot * cstride;
    const double* mu = mu_all + (long long)id * RTD_MAXP;
    for (int k = t; k < p; k += blockDim.x) cs[k] = mu[k];
    if (full_inverse) {  // [mu | Sigma^-1 row-major]: variant I of Table 1 (distances by the inverse)
      for (int e = t; e < p * p; e += blockDim.x) cs[p + e] = A[(e / p) * LD + e % p];
    } else {             // [mu | L^-1 packed lower]: §3.4 (distances by the Cholesky factor); row j per warp
      const int lane = t & 31, nw = blockDim.x >> 5;
      for (int j = t >> 5; j < p; j += nw)
        for (int k = lane; k <= j; k += 32) cs[p + j * (j + 1) / 2 + k] = Li[j * LD + k];
    }
  }
}

// ------------------------------------------------------------------ the whole C-step loop of a short block
// For short blocks (p <= 16, see csteps_small_supported) the per-step work is tiny and the loop of run_csteps (about ten
// launches and a host synchronisation per step) is latency-bound, so one CTA of 1024 threads runs the
// loop of one instance to the end: Cholesky, 1-norm condition and log det
// (the block_* helpers above), the distances d_i^2 = ||L^-1 (z_i - mu)||^2 into shared memory, the
// exact selection of the h smallest (d^2, row) composite keys by a 12-bit radix select (warp-aggregated
// shared atomics), the membership as bits and its change count (stop when H_new == H_old), and the
// mean / covariance of H_new by DMMA about the current centre (dense every step: the moments are the
// exact ones of the final subset, reading R12).  Same statuses, step counts and trajectory as run_csteps.
static constexpr int CS_SMALL_M = 20480;
static constexpr int CS_T = 512;
static constexpr int CS_W = CS_T / 32;

__device__ __forceinline__ void cs_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int NB>
__global__ void __launch_bounds__(CS_T, 1) k_csteps_small(const double* __restrict__ Zall, int m, int p,
                                                          long long blk_stride, int nstart, const int* __restrict__ inst,
                                                          int h, double kappa_max, int max_steps,
                                                          double* __restrict__ mu_all, double* __restrict__ sigma_all,
                                                          int* __restrict__ status_all, int* __restrict__ steps_all,
                                                          double* __restrict__ logdet_all, double* __restrict__ traj,
                                                          int traj_stride, uint8_t* __restrict__ mem_all) {
  constexpr int NBLK = NB * (NB + 1) / 2;
  constexpr int NRED = NBLK * 64 + 8 * NB + 1;  // per-warp partial: 8x8 blocks, S1, count
  extern __shared__ double dsm[];               // A, L, Li (block_* layout) then d^2 [m] / moment partials
  double* A = dsm;
  double* L = dsm + RTD_MAXP * LD;
  double* Li = dsm + 2 * RTD_MAXP * LD;
  double* dyn = dsm + 3 * RTD_MAXP * LD;
  __shared__ double red[RTD_MAXP];
  __shared__ double mu_s[16], sg_s[16 * 16];
  __shared__ unsigned int hist[4096];
  __shared__ unsigned int cur[CS_SMALL_M / 32], prv[CS_SMALL_M / 32];
  __shared__ long long wsum[CS_W];
  __shared__ int s_fail, s_stat, s_found, s_done, s_changed;
  __shared__ long long s_before, s_cnt;
  __shared__ unsigned long long s_pre_hi, s_pre_lo;
  __shared__ double s_logdet;
  const int id = inst[blockIdx.x];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, g = lane >> 2, tq = lane & 3;
  const double* __restrict__ Z = Zall + (long long)(id / nstart) * blk_stride;
  const int nwords = (m + 31) / 32;
  for (int e = t; e < p; e += CS_T) mu_s[e] = mu_all[(long long)id * RTD_MAXP + e];
  for (int e = t; e < p * p; e += CS_T) sg_s[e] = sigma_all[(long long)id * RTD_MAXP * RTD_MAXP + e];
  for (int w = t; w < nwords; w += CS_T) prv[w] = 0u;
  if (t == 0) s_stat = ST_ACTIVE;
  __syncthreads();
  int step = 1;
  for (; step <= max_steps; step++) {
    // ---- factor: Cholesky, condition monitor, log det (k_prepare)
    for (int e = t; e < p * p; e += CS_T) A[(e / p) * LD + e % p] = sg_s[e];
    __syncthreads();
    if (!block_chol_inv(A, L, Li, red, p, &s_fail)) {
      if (t == 0) s_stat = ST_NOT_PD;
      break;
    }
    const double n1 = block_max_colsum_abs(A, p, red);
    block_inv_from_li(Li, A, p);
    const double kappa = n1 * block_max_colsum_abs(A, p, red);
    if (t < p) red[t] = log(L[t * LD + t]);  // the logs in parallel (a dependent fp64 log is ~280 cycles)
    __syncthreads();
    if (t == 0) {
      double ld = 0.0;
      for (int j = 0; j < p; j++) ld += red[j];
      ld *= 2.0;
      s_logdet = ld;
      if (traj) traj[(long long)id * traj_stride + step] = ld;
      if (!(kappa < kappa_max)) s_stat = ST_COND;
    }
    __syncthreads();
    if (s_stat != ST_ACTIVE) break;
    // ---- distances (CS_R rows per thread in flight: the rows of Z come from L2 / HBM)
    constexpr int CS_R = 4;
    for (int i0 = t; i0 < m; i0 += CS_T * CS_R) {
      double u[CS_R][8 * NB];
#pragma unroll
      for (int r = 0; r < CS_R; r++) {
        const int i = i0 + r * CS_T;
#pragma unroll
        for (int k = 0; k < 8 * NB; k++) u[r][k] = (k < p && i < m) ? __ldg(Z + (long long)k * m + i) : 0.0;
      }
#pragma unroll
      for (int r = 0; r < CS_R; r++) {
        const int i = i0 + r * CS_T;
        if (i >= m) continue;
        double d = 0.0;
#pragma unroll
        for (int j = 0; j < 8 * NB; j++) {
          if (j < p) {
            double y = 0.0;
#pragma unroll
            for (int k = 0; k <= j; k++) y = fma(Li[j * LD + k], __dsub_rn(u[r][k], mu_s[k]), y);
            d = fma(y, y, d);
          }
        }
        dyn[i] = d;
      }
    }
    __syncthreads();
    // ---- exact selection of the h smallest composite keys (bits(d^2) << 32 | row)
    if (t == 0) {
      s_pre_hi = 0ull;
      s_pre_lo = 0ull;
      s_done = 0;
      s_before = h;  // rank still needed
    }
    int plen = 0;
    __syncthreads();
    while (true) {
      for (int b = t; b < 4096; b += CS_T) hist[b] = 0u;
      __syncthreads();
      const unsigned __int128 pre = ((unsigned __int128)s_pre_hi << 64) | s_pre_lo;
      for (int i0 = 0; i0 < m; i0 += CS_T) {
        const int i = i0 + t;
        bool take = false;
        unsigned dig = 0;
        if (i < m) {
          const unsigned __int128 C = ((unsigned __int128)(unsigned long long)__double_as_longlong(dyn[i]) << 32) | (unsigned)i;
          take = plen == 0 || (C >> (96 - plen)) == pre;
          dig = (unsigned)(C >> (96 - plen - 12)) & 4095u;
        }
        const unsigned act = __ballot_sync(0xffffffffu, take);
        if (take) {
          const unsigned same = __match_any_sync(act, dig);
          if ((__ffs(same) - 1) == lane) atomicAdd(&hist[dig], (unsigned)__popc(same));
        }
      }
      __syncthreads();
      // scan of 4096 bins: BPT per thread
      constexpr int BPT = 4096 / CS_T;
      long long c[BPT], loc = 0;
#pragma unroll
      for (int e = 0; e < BPT; e++) {
        c[e] = hist[t * BPT + e];
        loc += c[e];
      }
      long long inc = loc;
      for (int d = 1; d < 32; d <<= 1) {
        const long long v = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += v;
      }
      if (lane == 31) wsum[warp] = inc;
      __syncthreads();
      if (t == 0) {
        long long acc = 0;
        for (int w = 0; w < CS_W; w++) {
          const long long v = wsum[w];
          wsum[w] = acc;
          acc += v;
        }
      }
      __syncthreads();
      const long long rank = s_before;
      long long before = wsum[warp] + inc - loc;
#pragma unroll
      for (int e = 0; e < BPT; e++) {
        if (c[e] > 0 && before < rank && rank <= before + c[e]) {
          s_found = t * BPT + e;
          s_cnt = c[e];
          s_pre_lo = (unsigned long long)before;  // temporarily: keys before the bin
        }
        before += c[e];
      }
      __syncthreads();
      if (t == 0) {
        const long long bef = (long long)s_pre_lo;
        const unsigned __int128 np = (pre << 12) | (unsigned __int128)s_found;
        s_pre_hi = (unsigned long long)(np >> 64);
        s_pre_lo = (unsigned long long)np;
        s_before = rank - bef;
        s_done = (s_cnt == s_before || plen + 12 >= 96) ? 1 : 0;
      }
      plen += 12;
      __syncthreads();
      if (s_done) break;
    }
    // ---- membership bits and the changed-row count
    {
      const unsigned __int128 pre = ((unsigned __int128)s_pre_hi << 64) | s_pre_lo;
      if (t == 0) s_changed = 0;
      __syncthreads();
      int chg = 0;
      for (int i0 = 0; i0 < m; i0 += CS_T) {
        const int i = i0 + t;
        bool in = false;
        if (i < m) {
          const unsigned __int128 C = ((unsigned __int128)(unsigned long long)__double_as_longlong(dyn[i]) << 32) | (unsigned)i;
          in = (C >> (96 - plen)) <= pre;
        }
        const unsigned wb = __ballot_sync(0xffffffffu, in);
        if (lane == 0 && i0 / 32 + warp < nwords) {
          const int w = i0 / 32 + warp;
          cur[w] = wb;
          chg += __popc(wb ^ prv[w]);
        }
      }
      if (lane == 0 && chg) atomicAdd(&s_changed, chg);
      __syncthreads();
    }
    if (step > 1 && s_changed == 0) {
      if (t == 0) s_stat = ST_CONVERGED;
      __syncthreads();
      break;
    }
    // ---- moments of H_new about the current centre (DMMA per warp on 4-row groups)
    {
      double acc[NBLK][2], s1[NB], cntw = 0.0;
#pragma unroll
      for (int k = 0; k < NBLK; k++) acc[k][0] = acc[k][1] = 0.0;
#pragma unroll
      for (int b = 0; b < NB; b++) s1[b] = 0.0;
      constexpr int CS_G = 8;  // 4-row groups per warp iteration, loads issued first
      for (int rb = warp * 4 * CS_G; rb < m; rb += CS_W * 4 * CS_G) {
        double w[CS_G], u[CS_G][NB];
#pragma unroll
        for (int q = 0; q < CS_G; q++) {
          const int row = rb + 4 * q + tq;
          w[q] = (row < m && ((cur[row >> 5] >> (row & 31)) & 1u)) ? 1.0 : 0.0;
#pragma unroll
          for (int b = 0; b < NB; b++) {
            const int col = 8 * b + g;
            u[q][b] = (w[q] != 0.0 && col < p) ? __ldg(Z + (long long)col * m + row) : 0.0;
          }
        }
#pragma unroll
        for (int q = 0; q < CS_G; q++) {
          if (!__any_sync(0xffffffffu, w[q] != 0.0)) continue;
          double uu[NB], wu[NB];
#pragma unroll
          for (int b = 0; b < NB; b++) {
            const int col = 8 * b + g;
            uu[b] = (w[q] != 0.0 && col < p) ? __dsub_rn(u[q][b], mu_s[col]) : 0.0;
            wu[b] = w[q] * uu[b];
            s1[b] += wu[b];
          }
          if (g == 0) cntw += w[q];
          int k = 0;
#pragma unroll
          for (int jb = 0; jb < NB; jb++)
#pragma unroll
            for (int kb = 0; kb <= jb; kb++) {
              cs_dmma(acc[k][0], acc[k][1], wu[jb], uu[kb]);
              k++;
            }
        }
      }
#pragma unroll
      for (int b = 0; b < NB; b++) {
        s1[b] += __shfl_xor_sync(0xffffffffu, s1[b], 1);
        s1[b] += __shfl_xor_sync(0xffffffffu, s1[b], 2);
      }
      double* rw = dyn + (size_t)warp * NRED;
#pragma unroll
      for (int k = 0; k < NBLK; k++) {
        rw[k * 64 + g * 8 + 2 * tq] = acc[k][0];
        rw[k * 64 + g * 8 + 2 * tq + 1] = acc[k][1];
      }
      if (tq == 0) {
#pragma unroll
        for (int b = 0; b < NB; b++) rw[NBLK * 64 + 8 * b + g] = s1[b];
      }
      (void)cntw;
      __syncthreads();
      // fixed-order sum over the warps -> (mu, Sigma) of H_new
      const double hd = (double)h;
      if (t < p * p) {
        const int j = t / p, k = t - j * p;
        const int a = j > k ? j : k, bq = j > k ? k : j;  // lower-triangle entry (a >= bq)
        const int ja = a >> 3, kbq = bq >> 3;
        const int blk = ja * (ja + 1) / 2 + kbq;
        const int e = blk * 64 + (a & 7) * 8 + (bq & 7);
        double s2 = 0.0, sa = 0.0, sb = 0.0;
        for (int w = 0; w < CS_W; w++) {
          const double* rr = dyn + (size_t)w * NRED;
          s2 += rr[e];
          sa += rr[NBLK * 64 + a];
          sb += rr[NBLK * 64 + bq];
        }
        red[0] = 0.0;  // (keeps the shared array referenced; the values below are per thread)
        sg_s[t] = (s2 - sa * sb / hd) / (hd - 1.0);
        if (j == k) A[j] = sa;  // S1_j, parked until every thread read mu_s
      }
      __syncthreads();
      if (t < p) mu_s[t] = mu_s[t] + A[t] / hd;
      for (int w = t; w < nwords; w += CS_T) prv[w] = cur[w];
      __syncthreads();
    }
  }
  if (step > max_steps) {
    step = max_steps;
    if (t == 0) s_stat = ST_MAXSTEPS;
  }
  __syncthreads();
  const int stat = s_stat;
  if (stat == ST_MAXSTEPS) {  // log det of the final (mu, Sigma)
    for (int e = t; e < p * p; e += CS_T) A[(e / p) * LD + e % p] = sg_s[e];
    __syncthreads();
    if (block_cholesky(A, L, p, &s_fail) && t == 0) {
      double ld = 0.0;
      for (int j = 0; j < p; j++) ld += log(L[j * LD + j]);
      s_logdet = 2.0 * ld;
    }
    __syncthreads();
  }
  for (int e = t; e < p; e += CS_T) mu_all[(long long)id * RTD_MAXP + e] = mu_s[e];
  for (int e = t; e < p * p; e += CS_T) sigma_all[(long long)id * RTD_MAXP * RTD_MAXP + e] = sg_s[e];
  for (int i = t; i < m; i += CS_T) mem_all[(long long)id * m + i] = (uint8_t)((cur[i >> 5] >> (i & 31)) & 1u);
  if (t == 0) {
    status_all[id] = stat;
    steps_all[id] = step;
    logdet_all[id] = s_logdet;
  }
}

// ------------------------------------------------------------------ the C-step loop of a mid-size block
// on a thread-block CLUSTER (config 5: 20,000 rows, p = 8): the loop of k_csteps_small with the rows of the
// block split over the CL CTAs of a cluster (one instance per cluster), so every per-step pass runs on CL
// SMs, and the three couplings go through distributed shared memory (DSMEM) instead of kernel launches
// and host round trips:
//   - the radix select: each CTA histograms its rows' composite keys, every CTA reads the CL histograms
//     of the cluster (map_shared_rank) and takes the same decision;
//   - the changed-row count: CL partial counts summed in rank order;
//   - the moments of H_new: each CTA's fixed-order warp-reduced partial sums, folded in rank order by every
//     CTA (identical (mu, Sigma) on all of them, deterministic).
// The Cholesky / condition / log det of the (tiny) p x p scatter is recomputed by every CTA.
static constexpr int CSC_CL = 8;                       // CTAs per cluster (one instance)
__device__ unsigned long long g_csc_prof[64 * 8];      // RTD_DEBUG_CSC: phase timestamps of cluster 0, rank 0
__device__ __forceinline__ void csc_mark(int step, int ph, bool on) {
  if (on && step < 64) {
    unsigned long long tt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
    g_csc_prof[step * 8 + ph] = tt;
  }
}
static constexpr int CSC_ROWS = 2560;                  // rows per CTA at most (m <= 20480)
static constexpr int CSC_CAND = 64;                    // rows of the h-th key's bin resolved by counting

template <int NB>
__global__ void __cluster_dims__(CSC_CL, 1, 1) __launch_bounds__(CS_T, 1)
    k_csteps_cluster(const double* __restrict__ Zall, int m, int p, long long blk_stride, int nstart,
                     const int* __restrict__ inst, int h, double kappa_max, int max_steps,
                     double* __restrict__ mu_all, double* __restrict__ sigma_all, int* __restrict__ status_all,
                     int* __restrict__ steps_all, double* __restrict__ logdet_all, double* __restrict__ traj,
                     int traj_stride, uint8_t* __restrict__ mem_all) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int NBLK = NB * (NB + 1) / 2;
  constexpr int NRED = NBLK * 64 + 8 * NB + 1;
  extern __shared__ double dsm[];  // A, L, Li (block_* layout), then d^2 of this CTA's rows / warp partials
  double* A = dsm;
  double* L = dsm + RTD_MAXP * LD;
  double* Li = dsm + 2 * RTD_MAXP * LD;
  double* dyn = dsm + 3 * RTD_MAXP * LD;
  __shared__ double red[RTD_MAXP];
  __shared__ double mu_s[16], sg_s[16 * 16];
  __shared__ double part[NRED];                      // this CTA's moment partial (read by the cluster)
  __shared__ __align__(16) unsigned int hist[4096];  // this CTA's histogram (read by the cluster)
  __shared__ __align__(16) unsigned int tot[4096];   // the cluster's histogram
  __shared__ unsigned int cur[CSC_ROWS / 32], prv[CSC_ROWS / 32];
  __shared__ long long wsum[CS_W];
  __shared__ int s_fail, s_stat, s_found, s_done, s_chg_local, s_ncand, s_have_prev;
  __shared__ long long s_before, s_cnt;
  __shared__ unsigned long long s_pre_hi, s_pre_lo, s_cbase;
  __shared__ unsigned __int128 cand[CSC_CAND];  // this CTA's rows of the h-th key's bin (read by the cluster)
  __shared__ double s_logdet;
  const int cr = (int)cluster.block_rank();
  const int id = inst[blockIdx.x / CSC_CL];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, g = lane >> 2, tq = lane & 3;
  const double* __restrict__ Z = Zall + (long long)(id / nstart) * blk_stride;
  const int mloc = (m + CSC_CL - 1) / CSC_CL;
  const int r0 = min(m, cr * mloc), r1 = min(m, r0 + mloc), nl = r1 - r0;
  const int nwords = (nl + 31) / 32;
  for (int e = t; e < p; e += CS_T) mu_s[e] = mu_all[(long long)id * RTD_MAXP + e];
  for (int e = t; e < p * p; e += CS_T) sg_s[e] = sigma_all[(long long)id * RTD_MAXP * RTD_MAXP + e];
  for (int w = t; w < CSC_ROWS / 32; w += CS_T) prv[w] = cur[w] = 0u;
  if (t == 0) {
    s_stat = ST_ACTIVE;
    s_have_prev = 0;
    s_cbase = 0ull;
  }
  __syncthreads();
  int step = 1;
  const bool prof = blockIdx.x == 0 && t == 0;
  for (; step <= max_steps; step++) {
    csc_mark(step, 0, prof);
    // ---- factor (every CTA, identical)
    for (int e = t; e < p * p; e += CS_T) A[(e / p) * LD + e % p] = sg_s[e];
    __syncthreads();
    if (!block_chol_inv(A, L, Li, red, p, &s_fail)) {
      if (t == 0) s_stat = ST_NOT_PD;
      break;
    }
    const double n1 = block_max_colsum_abs(A, p, red);
    block_inv_from_li(Li, A, p);
    const double kappa = n1 * block_max_colsum_abs(A, p, red);
    if (t < p) red[t] = log(L[t * LD + t]);  // the logs in parallel (a dependent fp64 log is ~280 cycles)
    __syncthreads();
    if (t == 0) {
      double ld = 0.0;
      for (int j = 0; j < p; j++) ld += red[j];
      ld *= 2.0;
      s_logdet = ld;
      if (traj && cr == 0) traj[(long long)id * traj_stride + step] = ld;
      if (!(kappa < kappa_max)) s_stat = ST_COND;
    }
    __syncthreads();
    if (s_stat != ST_ACTIVE) break;
    csc_mark(step, 1, prof);
    // ---- distances of this CTA's rows
    constexpr int CS_R = 4;
    for (int i0 = r0 + t; i0 < r1; i0 += CS_T * CS_R) {
      double u[CS_R][8 * NB];
#pragma unroll
      for (int r = 0; r < CS_R; r++) {
        const int i = i0 + r * CS_T;
#pragma unroll
        for (int k = 0; k < 8 * NB; k++) u[r][k] = (k < p && i < r1) ? __ldg(Z + (long long)k * m + i) : 0.0;
      }
#pragma unroll
      for (int r = 0; r < CS_R; r++) {
        const int i = i0 + r * CS_T;
        if (i >= r1) continue;
        double d = 0.0;
#pragma unroll
        for (int j = 0; j < 8 * NB; j++) {
          if (j < p) {
            double y = 0.0;
#pragma unroll
            for (int k = 0; k <= j; k++) y = fma(Li[j * LD + k], __dsub_rn(u[r][k], mu_s[k]), y);
            d = fma(y, y, d);
          }
        }
        dyn[i - r0] = d;
      }
    }
    // ---- exact selection of the h smallest composite keys (bits(d^2) << 32 | row) over the cluster.
    //      From the second step on, the first level is CENTRED on the previous step's h-th key (as
    //      k_sel_level): its top 24 bits minus 2048 give 4094 bins of relative width 2^-12, everything below /
    //      above in the two end bins (a miss falls back to the plain 12-bit levels).  Once the bin holding the
    //      h-th key has at most CSC_CAND rows, the rows of that bin are collected (every CTA's few, through
    //      DSMEM) and the h-th key is found among them by counting -- instead of further histogram levels
    //      (each one a 4096-bin clear, two cluster barriers and 128 KB of DSMEM reads per CTA).
    if (t == 0) {
      s_pre_hi = 0ull;
      s_pre_lo = 0ull;
      s_done = 0;
      s_before = h;
    }
    int plen = 0;
    bool centred = s_have_prev != 0;
    const unsigned long long cbase = s_cbase;
    __syncthreads();
    csc_mark(step, 2, prof);
    while (true) {
      for (int b = t; b < 4096; b += CS_T) hist[b] = 0u;
      __syncthreads();
      const unsigned __int128 pre = ((unsigned __int128)s_pre_hi << 64) | s_pre_lo;
      unsigned below = 0, above = 0;
      for (int i0 = 0; i0 < nl; i0 += CS_T) {
        const int il = i0 + t;
        bool take = false;
        unsigned dig = 0;
        if (il < nl) {
          const unsigned long long kb = (unsigned long long)__double_as_longlong(dyn[il]);
          if (centred) {
            const unsigned long long top24 = kb >> 40;
            if (top24 < cbase) below++;
            else if (top24 >= cbase + 4094) above++;
            else {
              take = true;
              dig = (unsigned)(top24 - cbase + 1);
            }
          } else {
            const unsigned __int128 C = ((unsigned __int128)kb << 32) | (unsigned)(r0 + il);
            take = plen == 0 || (C >> (96 - plen)) == pre;
            dig = (unsigned)(C >> (96 - plen - 12)) & 4095u;
          }
        }
        const unsigned act = __ballot_sync(0xffffffffu, take);
        if (take) {
          const unsigned same = __match_any_sync(act, dig);
          if ((__ffs(same) - 1) == lane) atomicAdd(&hist[dig], (unsigned)__popc(same));
        }
      }
      if (centred) {
        for (int d = 16; d > 0; d >>= 1) {
          below += __shfl_down_sync(0xffffffffu, below, d);
          above += __shfl_down_sync(0xffffffffu, above, d);
        }
        if (lane == 0) {
          if (below) atomicAdd(&hist[0], below);
          if (above) atomicAdd(&hist[4095], above);
        }
      }
      if (plen == 0) csc_mark(step, 6, prof);
      cluster.sync();  // every CTA's histogram is complete
      if (plen == 0) csc_mark(step, 7, prof);
      constexpr int BPT = 4096 / CS_T;
      // the cluster's histogram: coalesced 16-byte DSMEM reads of the CL histograms (rank order) into tot
      for (int v = t; v < 4096 / 4; v += CS_T) {
        uint4 sum = make_uint4(0u, 0u, 0u, 0u);
        for (int q = 0; q < CSC_CL; q++) {
          const uint4 r = reinterpret_cast<const uint4*>(cluster.map_shared_rank(hist, q))[v];
          sum.x += r.x;
          sum.y += r.y;
          sum.z += r.z;
          sum.w += r.w;
        }
        reinterpret_cast<uint4*>(tot)[v] = sum;
      }
      __syncthreads();
      long long c[BPT], loc = 0;
#pragma unroll
      for (int e = 0; e < BPT; e++) {
        c[e] = tot[t * BPT + e];
        loc += c[e];
      }
      long long inc = loc;
      for (int d = 1; d < 32; d <<= 1) {
        const long long v = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += v;
      }
      if (lane == 31) wsum[warp] = inc;
      cluster.sync();  // all remote reads of the histograms done (they are reset next round)
      if (t == 0) {
        long long acc = 0;
        for (int w = 0; w < CS_W; w++) {
          const long long v = wsum[w];
          wsum[w] = acc;
          acc += v;
        }
      }
      __syncthreads();
      const long long rank = s_before;
      long long before = wsum[warp] + inc - loc;
#pragma unroll
      for (int e = 0; e < BPT; e++) {
        if (c[e] > 0 && before < rank && rank <= before + c[e]) {
          s_found = t * BPT + e;
          s_cnt = c[e];
          s_pre_lo = (unsigned long long)before;
        }
        before += c[e];
      }
      __syncthreads();
      if (centred) {
        const bool miss = s_found == 0 || s_found == 4095;
        __syncthreads();  // every thread has read s_found before thread 0 rewrites the state
        if (t == 0) {
          if (miss) {  // the h-th key left the window: plain levels from the top
            s_pre_hi = 0ull;
            s_pre_lo = 0ull;
          } else {
            const long long bef = (long long)s_pre_lo;
            s_pre_hi = 0ull;
            s_pre_lo = cbase + (unsigned long long)s_found - 1ull;
            s_before = rank - bef;
            s_done = s_cnt == s_before ? 1 : 0;
          }
        }
        if (!miss) plen = 24;
        centred = false;
      } else {
        if (t == 0) {
          const long long bef = (long long)s_pre_lo;
          const unsigned __int128 np = (pre << 12) | (unsigned __int128)s_found;
          s_pre_hi = (unsigned long long)(np >> 64);
          s_pre_lo = (unsigned long long)np;
          s_before = rank - bef;
          s_done = (s_cnt == s_before || plen + 12 >= 96) ? 1 : 0;
        }
        plen += 12;
      }
      __syncthreads();
      if (s_done) break;
      if (plen >= 24 && s_cnt <= CSC_CAND) {
        // candidate resolution: the bin's rows (at most CSC_CAND over the cluster) collected per CTA
        const unsigned __int128 bp = ((unsigned __int128)s_pre_hi << 64) | s_pre_lo;
        if (t == 0) s_ncand = 0;
        __syncthreads();
        for (int il = t; il < nl; il += CS_T) {
          const unsigned __int128 C =
              ((unsigned __int128)(unsigned long long)__double_as_longlong(dyn[il]) << 32) | (unsigned)(r0 + il);
          if ((C >> (96 - plen)) == bp) cand[atomicAdd(&s_ncand, 1)] = C;  // < CSC_CAND: a subset of the bin
        }
        cluster.sync();  // every CTA's candidates are listed
        const long long need = s_before;  // rank of the h-th key inside the bin (1-based)
        const int ntot = (int)s_cnt;
        if (t < ntot) {
          int q = 0, j = t;  // candidate t of the concatenation in rank order
          while (j >= *cluster.map_shared_rank(&s_ncand, q)) {
            j -= *cluster.map_shared_rank(&s_ncand, q);
            q++;
          }
          const unsigned __int128 mine = cluster.map_shared_rank(cand, q)[j];
          int less = 0;
          for (int qq = 0; qq < CSC_CL; qq++) {
            const int nq = *cluster.map_shared_rank(&s_ncand, qq);
            const unsigned __int128* cq = cluster.map_shared_rank(cand, qq);
            for (int k = 0; k < nq; k++) less += cq[k] < mine ? 1 : 0;
          }
          if (less == need - 1) {  // the h-th key (keys are unique: the row index is part of them)
            s_pre_hi = (unsigned long long)(mine >> 64);
            s_pre_lo = (unsigned long long)mine;
          }
        }
        plen = 96;
        // (the lists are rewritten only in the next step's select, after the member phase's cluster barrier)
        __syncthreads();
        break;
      }
    }
    if (t == 0) {  // centre the next step's first level on this step's h-th key
      const unsigned __int128 fp = ((unsigned __int128)s_pre_hi << 64) | s_pre_lo;
      const unsigned long long top24 = plen >= 24 ? (unsigned long long)(fp >> (plen - 24)) : 0ull;
      s_have_prev = plen >= 24 ? 1 : 0;
      s_cbase = top24 > 2048 ? top24 - 2048 : 0ull;
    }
    csc_mark(step, 3, prof);
    // ---- membership bits of this CTA's rows and the cluster's changed-row count
    {
      const unsigned __int128 pre = ((unsigned __int128)s_pre_hi << 64) | s_pre_lo;
      if (t == 0) s_chg_local = 0;
      __syncthreads();
      int chg = 0;
      for (int i0 = 0; i0 < nl; i0 += CS_T) {
        const int il = i0 + t;
        bool in = false;
        if (il < nl) {
          const unsigned __int128 C =
              ((unsigned __int128)(unsigned long long)__double_as_longlong(dyn[il]) << 32) | (unsigned)(r0 + il);
          in = (C >> (96 - plen)) <= pre;
        }
        const unsigned wb = __ballot_sync(0xffffffffu, in);
        if (lane == 0 && i0 / 32 + warp < nwords) {
          const int w = i0 / 32 + warp;
          cur[w] = wb;
          chg += __popc(wb ^ prv[w]);
        }
      }
      if (lane == 0 && chg) atomicAdd(&s_chg_local, chg);
      cluster.sync();
      long long changed = 0;
      for (int q = 0; q < CSC_CL; q++) changed += *cluster.map_shared_rank(&s_chg_local, q);
      if (step > 1 && changed == 0) {
        if (t == 0) s_stat = ST_CONVERGED;
        cluster.sync();  // no CTA resets s_chg_local before every CTA read it
        break;
      }
    }
    csc_mark(step, 4, prof);
    // ---- moments of H_new about the current centre: this CTA's rows on DMMA, folded in rank order
    {
      double acc[NBLK][2], s1[NB];
#pragma unroll
      for (int k = 0; k < NBLK; k++) acc[k][0] = acc[k][1] = 0.0;
#pragma unroll
      for (int b = 0; b < NB; b++) s1[b] = 0.0;
      constexpr int CS_G = 8;
      for (int rb = warp * 4 * CS_G; rb < nl; rb += CS_W * 4 * CS_G) {
        double w[CS_G], u[CS_G][NB];
#pragma unroll
        for (int q = 0; q < CS_G; q++) {
          const int rl = rb + 4 * q + tq;
          w[q] = (rl < nl && ((cur[rl >> 5] >> (rl & 31)) & 1u)) ? 1.0 : 0.0;
#pragma unroll
          for (int b = 0; b < NB; b++) {
            const int col = 8 * b + g;
            u[q][b] = (w[q] != 0.0 && col < p) ? __ldg(Z + (long long)col * m + r0 + rl) : 0.0;
          }
        }
#pragma unroll
        for (int q = 0; q < CS_G; q++) {
          if (!__any_sync(0xffffffffu, w[q] != 0.0)) continue;
          double uu[NB], wu[NB];
#pragma unroll
          for (int b = 0; b < NB; b++) {
            const int col = 8 * b + g;
            uu[b] = (w[q] != 0.0 && col < p) ? __dsub_rn(u[q][b], mu_s[col]) : 0.0;
            wu[b] = w[q] * uu[b];
            s1[b] += wu[b];
          }
          int k = 0;
#pragma unroll
          for (int jb = 0; jb < NB; jb++)
#pragma unroll
            for (int kb = 0; kb <= jb; kb++) {
              cs_dmma(acc[k][0], acc[k][1], wu[jb], uu[kb]);
              k++;
            }
        }
      }
#pragma unroll
      for (int b = 0; b < NB; b++) {
        s1[b] += __shfl_xor_sync(0xffffffffu, s1[b], 1);
        s1[b] += __shfl_xor_sync(0xffffffffu, s1[b], 2);
      }
      double* rw = dyn + (size_t)warp * NRED;  // d^2 no longer needed this step
      __syncthreads();
#pragma unroll
      for (int k = 0; k < NBLK; k++) {
        rw[k * 64 + g * 8 + 2 * tq] = acc[k][0];
        rw[k * 64 + g * 8 + 2 * tq + 1] = acc[k][1];
      }
      if (tq == 0) {
#pragma unroll
        for (int b = 0; b < NB; b++) rw[NBLK * 64 + 8 * b + g] = s1[b];
      }
      __syncthreads();
      for (int e = t; e < NRED - 1; e += CS_T) {  // this CTA's partial: fixed-order sum over its warps
        double v = 0.0;
        for (int w = 0; w < CS_W; w++) v += dyn[(size_t)w * NRED + e];
        part[e] = v;
      }
      cluster.sync();  // every CTA's partial is complete
      const double hd = (double)h;
      double sg_new = 0.0, s1j = 0.0;
      if (t < p * p) {
        const int j = t / p, k = t - j * p;
        const int a = j > k ? j : k, bq = j > k ? k : j;
        const int ja = a >> 3, kbq = bq >> 3;
        const int blk = ja * (ja + 1) / 2 + kbq;
        const int e = blk * 64 + (a & 7) * 8 + (bq & 7);
        double s2 = 0.0, sa = 0.0, sb = 0.0;
        for (int q = 0; q < CSC_CL; q++) {  // rank order
          const double* rr = cluster.map_shared_rank(part, q);
          s2 += rr[e];
          sa += rr[NBLK * 64 + a];
          sb += rr[NBLK * 64 + bq];
        }
        sg_new = (s2 - sa * sb / hd) / (hd - 1.0);
        s1j = sa;
      }
      cluster.sync();  // all remote reads of the partials done
      if (t < p * p) {
        const int j = t / p, k = t - j * p;
        sg_s[t] = sg_new;
        if (j == k) A[j] = s1j;
      }
      __syncthreads();
      if (t < p) mu_s[t] = mu_s[t] + A[t] / hd;
      for (int w = t; w < nwords; w += CS_T) prv[w] = cur[w];
      __syncthreads();
      csc_mark(step, 5, prof);
    }
  }
  if (step > max_steps) {
    step = max_steps;
    if (t == 0) s_stat = ST_MAXSTEPS;
  }
  __syncthreads();
  const int stat = s_stat;
  if (stat == ST_MAXSTEPS) {
    for (int e = t; e < p * p; e += CS_T) A[(e / p) * LD + e % p] = sg_s[e];
    __syncthreads();
    if (block_cholesky(A, L, p, &s_fail) && t == 0) {
      double ld = 0.0;
      for (int j = 0; j < p; j++) ld += log(L[j * LD + j]);
      s_logdet = 2.0 * ld;
    }
    __syncthreads();
  }
  for (int il = t; il < nl; il += CS_T)
    mem_all[(long long)id * m + r0 + il] = (uint8_t)((cur[il >> 5] >> (il & 31)) & 1u);
  if (cr == 0) {
    for (int e = t; e < p; e += CS_T) mu_all[(long long)id * RTD_MAXP + e] = mu_s[e];
    for (int e = t; e < p * p; e += CS_T) sigma_all[(long long)id * RTD_MAXP * RTD_MAXP + e] = sg_s[e];
    if (t == 0) {
      status_all[id] = stat;
      steps_all[id] = step;
      logdet_all[id] = s_logdet;
    }
  }
  cluster.sync();  // no CTA leaves while another may still read its shared memory
}

bool csteps_cluster_supported(long long m, int p) {
  static const bool off = getenv("RTD_NO_CLUSTER_CSTEPS") != nullptr;
  return !off && m > 4096 && m <= (long long)CSC_CL * CSC_ROWS && p >= 1 && p <= 16;
}

void launch_csteps_cluster(const double* Zall, long long m, int p, long long blk_stride, int nstart, const int* inst,
                           int ninst, long long h, double kappa_max, int max_steps, double* mu_all, double* sigma_all,
                           int* status_all, int* steps_all, double* logdet_all, double* traj, int traj_stride,
                           uint8_t* mem_all, cudaStream_t st) {
  const int nb = (p + 7) / 8;
  const int nred = (nb * (nb + 1) / 2) * 64 + 8 * nb + 1;
  const size_t dyn = (3 * (size_t)RTD_MAXP * LD + std::max<size_t>((size_t)CSC_ROWS, (size_t)CS_W * nred)) *
                     sizeof(double);
  if (nb == 1) {
    set_max_dyn_smem(reinterpret_cast<const void*>(k_csteps_cluster<1>), (int)dyn);
    k_csteps_cluster<1><<<ninst * CSC_CL, CS_T, dyn, st>>>(Zall, (int)m, p, blk_stride, nstart, inst, (int)h,
                                                           kappa_max, max_steps, mu_all, sigma_all, status_all,
                                                           steps_all, logdet_all, traj, traj_stride, mem_all);
  } else {
    set_max_dyn_smem(reinterpret_cast<const void*>(k_csteps_cluster<2>), (int)dyn);
    k_csteps_cluster<2><<<ninst * CSC_CL, CS_T, dyn, st>>>(Zall, (int)m, p, blk_stride, nstart, inst, (int)h,
                                                           kappa_max, max_steps, mu_all, sigma_all, status_all,
                                                           steps_all, logdet_all, traj, traj_stride, mem_all);
  }
  RTD_LAUNCHED();
  static const bool dbg = getenv("RTD_DEBUG_CSC") != nullptr;
  if (dbg) {
    static int calls = 0;
    unsigned long long pr[64 * 8];
    RTD_CU(cudaStreamSynchronize(st));
    RTD_CU(cudaMemcpyFromSymbol(pr, g_csc_prof, sizeof(pr)));
    if (calls++ < 3) {
      for (int s = 1; s < 12 && pr[s * 8 + 5] > pr[s * 8]; s++)
        fprintf(stderr, "[csc] step %d: factor %.1f dist %.1f select %.1f (hist1 %.1f sync1 %.1f) member %.1f moments %.1f us\n", s,
                (pr[s * 8 + 1] - pr[s * 8]) * 1e-3, (pr[s * 8 + 2] - pr[s * 8 + 1]) * 1e-3,
                (pr[s * 8 + 6] - pr[s * 8 + 2]) * 1e-3, (pr[s * 8 + 7] - pr[s * 8 + 6]) * 1e-3,
                (pr[s * 8 + 3] - pr[s * 8 + 2]) * 1e-3, (pr[s * 8 + 4] - pr[s * 8 + 3]) * 1e-3,
                (pr[s * 8 + 5] - pr[s * 8 + 4]) * 1e-3);
    }
  }
}

// used up to 4096 rows: measured faster than the multi-launch loop there (config 1, 1000 x 5: fit + flag
// 1.69 -> 0.98 ms) but slower at 20,000 rows (config 5: one SM per instance is too little for the
// per-step passes), where run_csteps' grid-wide kernels win despite their launches
bool csteps_small_supported(long long m, int p) { return m <= 4096 && m >= 2 && p >= 1 && p <= 16; }

void launch_csteps_small(const double* Zall, long long m, int p, long long blk_stride, int nstart, const int* inst,
                         int ninst, long long h, double kappa_max, int max_steps, double* mu_all, double* sigma_all,
                         int* status_all, int* steps_all, double* logdet_all, double* traj, int traj_stride,
                         uint8_t* mem_all, cudaStream_t st) {
  const int nb = (p + 7) / 8;
  const int nred = (nb * (nb + 1) / 2) * 64 + 8 * nb + 1;
  const size_t dyn = (3 * (size_t)RTD_MAXP * LD + std::max<size_t>((size_t)m, (size_t)CS_W * nred)) * sizeof(double);
  const int dmax = (int)((3 * (size_t)RTD_MAXP * LD + CS_SMALL_M) * sizeof(double));
  if (nb == 1) {
    static const bool a1 = [dmax] {
      cudaFuncSetAttribute(k_csteps_small<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, dmax);
      return true;
    }();
    (void)a1;
    k_csteps_small<1><<<ninst, CS_T, dyn, st>>>(Zall, (int)m, p, blk_stride, nstart, inst, (int)h, kappa_max,
                                                max_steps, mu_all, sigma_all, status_all, steps_all, logdet_all, traj,
                                                traj_stride, mem_all);
  } else {
    static const bool a2 = [dmax] {
      cudaFuncSetAttribute(k_csteps_small<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, dmax);
      return true;
    }();
    (void)a2;
    k_csteps_small<2><<<ninst, CS_T, dyn, st>>>(Zall, (int)m, p, blk_stride, nstart, inst, (int)h, kappa_max,
                                                max_steps, mu_all, sigma_all, status_all, steps_all, logdet_all, traj,
                                                traj_stride, mem_all);
  }
  RTD_LAUNCHED();
}

void launch_prepare(const int* inst, int ninst, const double* mu_all, const double* sigma_all, int p, double kappa_max,
                    double* cstage, int cstride, double* logdet_out, double* cond_out, int* status_out, double* traj,
                    int traj_stride, int step, cudaStream_t st, int full_inverse, const int* skip) {
  k_prepare<<<ninst, 512, 0, st>>>(inst, mu_all, sigma_all, p, kappa_max, cstage, cstride, logdet_out, cond_out,
                                  status_out, traj, traj_stride, step, full_inverse, skip);
  RTD_LAUNCHED();
}

// ------------------------------------------------------------------ single-swap inverse update (SMW variant)
// when a C-step interchanges exactly two cases (sum |delta_i| = 2), the inverse of the
// sscp matrix is updated directly by Sherman-Morrison-Woodbury and the determinant by
// det(Lambda + delta u v^T) = Delta det(Lambda), Delta = 1 + delta v^T Lambda^-1 u, the cases taken in
// row order with u = z - mu (mean before the case), v = z - mu' (after), as in the update loop
// (PAPER.md:685-709).  Sigma = Lambda / (h - 1) has the same h before and after a swap, so
// Sigma^-1_new = (h - 1) Lambda^-1_new and log det Sigma changes by sum log Delta.
// sinv_all[id]: Sigma^-1 (row-major p x p) of the operator used by this step's distances; mu_all: the
// mean of the old subset (before this step's moment update).  On success smw_valid[id] = 1 (the next
// step skips k_prepare for the instance); a non-positive Delta leaves it 0 (full recompute).
__global__ void __launch_bounds__(64) k_smw_update(const int* __restrict__ inst, const double* __restrict__ Zall,
                                                   long long m, long long blk_stride, int nstart,
                                                   const double* __restrict__ mu_all,
                                                   const int* __restrict__ list_all, const int* __restrict__ seg_cnt_all,
                                                   int nseg, long long seg_len, int p, long long h,
                                                   double* __restrict__ sinv_all, double* __restrict__ logdet,
                                                   int* __restrict__ smw_valid) {
  __shared__ double A[RTD_MAXP * LD];
  __shared__ double mu[RTD_MAXP], z[RTD_MAXP], u[RTD_MAXP], v[RTD_MAXP], Au[RTD_MAXP], vA[RTD_MAXP];
  __shared__ int rows[2];  // list entries: +(row + 1) entering, -(row + 1) leaving (k_sel_member)
  __shared__ double s_delta;
  __shared__ int s_ok;
  const int id = inst[blockIdx.x], t = threadIdx.x;
  double* S = sinv_all + (long long)id * RTD_MAXP * RTD_MAXP;
  const double* Z = Zall + (long long)(id / nstart) * blk_stride;
  if (t == 0) {  // the two changed rows, in row order (segments are ordered, each segment's list too)
    int k = 0;
    for (int sgi = 0; sgi < nseg && k < 2; sgi++) {
      const int c = seg_cnt_all[(long long)id * nseg + sgi];
      for (int j = 0; j < c && k < 2; j++) {
        const int e = list_all[(long long)id * m + (long long)sgi * seg_len + j];
        if (e != 0) rows[k++] = e;  // (0: a reserved slot of an unchanged candidate row)
      }
    }
    s_ok = k == 2;
  }
  const double hm1 = (double)(h - 1);
  for (int e = t; e < p * p; e += blockDim.x) A[(e / p) * LD + e % p] = S[e] / hm1;  // Lambda^-1
  for (int k = t; k < p; k += blockDim.x) mu[k] = mu_all[(long long)id * RTD_MAXP + k];
  __syncthreads();
  if (!s_ok) return;
  double n = (double)h, dld = 0.0;
  for (int c = 0; c < 2; c++) {
    const long long r = (long long)abs(rows[c]) - 1;
    const double delta = rows[c] > 0 ? 1.0 : -1.0;  // entering / leaving
    const double n1 = n + delta;
    for (int k = t; k < p; k += blockDim.x) {
      z[k] = Z[(long long)k * m + r];
      const double mk = mu[k] + delta * (z[k] - mu[k]) / n1;
      u[k] = z[k] - mu[k];
      v[k] = z[k] - mk;
    }
    __syncthreads();
    for (int k = t; k < p; k += blockDim.x) {
      double a = 0.0, b = 0.0;
      for (int j = 0; j < p; j++) {
        a = fma(A[k * LD + j], u[j], a);  // (Lambda^-1 u)_k
        b = fma(v[j], A[j * LD + k], b);  // (v^T Lambda^-1)_k
      }
      Au[k] = a;
      vA[k] = b;
    }
    __syncthreads();
    if (t == 0) {
      double d = 0.0;
      for (int k = 0; k < p; k++) d = fma(v[k], Au[k], d);
      s_delta = 1.0 + delta * d;
    }
    __syncthreads();
    const double D = s_delta;
    if (!(D > 0.0) || !isfinite(D)) return;  // not PD after the update: k_prepare recomputes
    const double f = delta / D;
    for (int e = t; e < p * p; e += blockDim.x) {
      const int i = e / p, j = e - i * p;
      A[i * LD + j] -= f * Au[i] * vA[j];
    }
    dld += log(D);
    for (int k = t; k < p; k += blockDim.x) mu[k] += delta * (z[k] - mu[k]) / n1;
    n = n1;
    __syncthreads();
  }
  for (int e = t; e < p * p; e += blockDim.x) S[e] = A[(e / p) * LD + e % p] * hm1;
  if (t == 0) {
    logdet[id] += dld;
    smw_valid[id] = 1;
  }
}

void launch_smw_update(const int* inst, int ninst, const double* Zall, long long m, long long blk_stride, int nstart,
                       const double* mu_all, const int* list_all, const int* seg_cnt_all,
                       int nseg, long long seg_len, int p, long long h, double* sinv_all, double* logdet,
                       int* smw_valid, cudaStream_t st) {
  k_smw_update<<<ninst, 64, 0, st>>>(inst, Zall, m, blk_stride, nstart, mu_all, list_all, seg_cnt_all,
                                     nseg, seg_len, p, h, sinv_all, logdet, smw_valid);
  RTD_LAUNCHED();
}

// Per slot of this step's instance list (SMW variant), after k_prepare: an instance whose inverse was
// updated by k_smw_update gets the operator [mu | Sigma^-1 (symmetrised)] staged from it and the 1-norm
// condition check of k_prepare (||Sigma||_1 ||Sigma^-1||_1 < kappa_max); any other
// instance's exact inverse (staged by k_prepare) is kept as the base of the next update.
__global__ void __launch_bounds__(64) k_smw_stage(const int* __restrict__ inst, const double* __restrict__ mu_all,
                                                  const double* __restrict__ sigma_all, int p, double kappa_max,
                                                  double* __restrict__ cstage, int cstride,
                                                  double* __restrict__ sinv_all, int* __restrict__ smw_valid,
                                                  double* __restrict__ cond_out, int* __restrict__ status) {
  __shared__ double red[2][RTD_MAXP];
  const int slot = blockIdx.x, id = inst[slot], t = threadIdx.x;
  if (status[id] != 0) return;
  double* cs = cstage + (long long)slot * cstride;
  double* S = sinv_all + (long long)id * RTD_MAXP * RTD_MAXP;
  if (!smw_valid[id]) {
    for (int e = t; e < p * p; e += blockDim.x) S[e] = cs[p + e];
    return;
  }
  const double* mu = mu_all + (long long)id * RTD_MAXP;
  const double* sg = sigma_all + (long long)id * RTD_MAXP * RTD_MAXP;
  for (int k = t; k < p; k += blockDim.x) cs[k] = mu[k];
  for (int e = t; e < p * p; e += blockDim.x) {
    const int i = e / p, j = e - i * p;
    cs[p + e] = 0.5 * (S[e] + S[j * p + i]);
  }
  for (int j = t; j < p; j += blockDim.x) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < p; i++) {
      a += fabs(sg[i * p + j]);
      b += fabs(S[i * p + j]);
    }
    red[0][j] = a;
    red[1][j] = b;
  }
  __syncthreads();
  if (t == 0) {
    double n1 = 0.0, n1i = 0.0;
    for (int j = 0; j < p; j++) {
      n1 = fmax(n1, red[0][j]);
      n1i = fmax(n1i, red[1][j]);
    }
    const double kappa = n1 * n1i;
    cond_out[id] = kappa;
    if (!(kappa < kappa_max)) status[id] = ST_COND;
    smw_valid[id] = 0;
  }
}

void launch_smw_stage(const int* inst, int ninst, const double* mu_all, const double* sigma_all, int p,
                      double kappa_max, double* cstage, int cstride, double* sinv_all, int* smw_valid,
                      double* cond_out, int* status, cudaStream_t st) {
  k_smw_stage<<<ninst, 64, 0, st>>>(inst, mu_all, sigma_all, p, kappa_max, cstage, cstride, sinv_all, smw_valid,
                                    cond_out, status);
  RTD_LAUNCHED();
}

// ------------------------------------------------------------------ sums -> (mu, Sigma)
// sums: [S1 (p)] [S2 packed lower (p(p+1)/2)] [count] about shift c.
// mode 0: mu = c + S1/n, Sigma = (S2 - S1 S1^T / n) / (n - 1) * factor   (n = count or given)
__global__ void k_sums_to_cov(const int* __restrict__ inst, const double* __restrict__ sums_all, int np,
                              const double* __restrict__ shift_all, int p, double n_given, double factor,
                              double* __restrict__ mu_all, double* __restrict__ sigma_all) {
  const int id = inst ? inst[blockIdx.x] : blockIdx.x;
  const double* S = sums_all + (long long)id * np;
  const double n = n_given > 0 ? n_given : S[np - 1];
  const double* c = shift_all ? shift_all + (long long)id * RTD_MAXP : nullptr;
  double* mu = mu_all + (long long)id * RTD_MAXP;
  double* sg = sigma_all + (long long)id * RTD_MAXP * RTD_MAXP;
  for (int k = threadIdx.x; k < p; k += blockDim.x) mu[k] = (c ? c[k] : 0.0) + S[k] / n;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    int j = e / p, k = e - j * p;
    int a = j > k ? j : k, b = j > k ? k : j;
    double s2 = S[p + a * (a + 1) / 2 + b];
    sg[e] = factor * ((s2 - S[j] * S[k] / n) / (n - 1.0));
  }
}

void launch_sums_to_cov(const int* inst, int ninst, const double* sums_all, int np, const double* shift_all, int p,
                        double n_given, double factor, double* mu_all, double* sigma_all, cudaStream_t st) {
  k_sums_to_cov<<<ninst, 256, 0, st>>>(inst, sums_all, np, shift_all, p, n_given, factor, mu_all, sigma_all);
  RTD_LAUNCHED();
}

// S~2 = S2 / n (uncentred second moment)
__global__ void k_sums_to_second(const double* __restrict__ sums_all, int np, int p, double n,
                                 double* __restrict__ out_all) {
  const int b = blockIdx.x;
  const double* S = sums_all + (long long)b * np;
  double* o = out_all + (long long)b * RTD_MAXP * RTD_MAXP;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    int j = e / p, k = e - j * p;
    int a = j > k ? j : k, bb = j > k ? k : j;
    o[e] = S[p + a * (a + 1) / 2 + bb] / n;
  }
}

void launch_sums_to_second(const double* sums_all, int nb, int np, int p, double n, double* out_all, cudaStream_t st) {
  k_sums_to_second<<<nb, 256, 0, st>>>(sums_all, np, p, n, out_all);
  RTD_LAUNCHED();
}

__global__ void k_copy_vec(const int* __restrict__ inst, const double* __restrict__ src, double* __restrict__ dst,
                           int p) {
  const int id = inst[blockIdx.x];
  for (int k = threadIdx.x; k < p; k += blockDim.x) dst[(long long)id * RTD_MAXP + k] = src[(long long)id * RTD_MAXP + k];
}

void launch_copy_vec(const int* inst, int ninst, const double* src, double* dst, int p, cudaStream_t st) {
  k_copy_vec<<<ninst, 64, 0, st>>>(inst, src, dst, p);
  RTD_LAUNCHED();
}

// ------------------------------------------------------------------ Jacobi eigen-decomposition
__global__ void __launch_bounds__(LT) k_jacobi(const double* __restrict__ A_all, int p, double kappa_max,
                                               double* __restrict__ V_all, double* __restrict__ lam_all,
                                               int* __restrict__ ok_all) {
  __shared__ double A[RTD_MAXP][LD], V[RTD_MAXP][LD];
  __shared__ double cs[RTD_MAXP / 2 + 1], sn[RTD_MAXP / 2 + 1];
  __shared__ int pa[RTD_MAXP / 2 + 1], qa[RTD_MAXP / 2 + 1];
  __shared__ int order[RTD_MAXP + 2];
  __shared__ double red[LT];
  __shared__ int s_stop, s_rot;
  const int b = blockIdx.x, t = threadIdx.x;
  const double* Ain = A_all + (long long)b * RTD_MAXP * RTD_MAXP;
  for (int e = t; e < p * p; e += blockDim.x) {
    int i = e / p, j = e - i * p;
    A[i][j] = 0.5 * (Ain[i * p + j] + Ain[j * p + i]);
    V[i][j] = (i == j) ? 1.0 : 0.0;
  }
  const int n2 = p + (p & 1);
  if (t < n2) order[t] = t;
  __syncthreads();
  for (int sweep = 0; sweep < 60; sweep++) {
    // convergence: off-diagonal mass relative to the total
    double off = 0.0, tot = 0.0;
    for (int e = t; e < p * p; e += blockDim.x) {
      int i = e / p, j = e - i * p;
      double v = A[i][j] * A[i][j];
      tot += v;
      if (i != j) off += v;
    }
    for (int d = 16; d > 0; d >>= 1) {
      off += __shfl_down_sync(0xffffffffu, off, d);
      tot += __shfl_down_sync(0xffffffffu, tot, d);
    }
    if ((t & 31) == 0) {
      red[t >> 5] = off;
      red[32 + (t >> 5)] = tot;
    }
    __syncthreads();
    if (t == 0) {
      double so = 0.0, st = 0.0;
      for (int k = 0; k < (int)(blockDim.x >> 5); k++) {
        so += red[k];
        st += red[32 + k];
      }
      s_stop = (so <= 1e-32 * st) || so == 0.0;
    }
    if (t == 0) s_rot = 0;
    __syncthreads();
    if (s_stop) break;
    for (int round = 0; round < n2 - 1; round++) {
      if (t < n2 / 2) {
        // round-robin positions: 0 fixed, 1..n2-1 rotated right by one per round (period n2 - 1, so every
        // sweep starts from the identity); computed, not stored, so no thread shifts a shared array
        auto ord = [&](int k) { return k == 0 ? 0 : 1 + ((k - 1 - round) % (n2 - 1) + (n2 - 1)) % (n2 - 1); };
        int P = ord(t), Q = ord(n2 - 1 - t);
        if (P > Q) { int tmp = P; P = Q; Q = tmp; }
        double c = 1.0, s = 0.0;
        if (Q < p && A[P][Q] != 0.0 && 1e18 * fabs(A[P][Q]) <= fmin(fabs(A[P][P]), fabs(A[Q][Q]))) {
          // below the rounding of both diagonal entries (the classical threshold test): dropped, so a
          // sweep can end without rotations and the loop terminates
          A[P][Q] = 0.0;
          A[Q][P] = 0.0;
        } else if (Q < p && A[P][Q] != 0.0) {
          s_rot = 1;
          // t = sign(tau) / (|tau| + sqrt(1 + tau^2)), tau = h / a_pq, h = (a_qq - a_pp) / 2, written
          // without the first division: t = sign(tau) |a_pq| / (|h| + sqrt(h^2 + a_pq^2)); c = rsqrt(1 + t^2)
          // (a shorter chain of the slow fp64 operations on the critical path of every round)
          const double apq = A[P][Q];
          const double hh = 0.5 * (A[Q][Q] - A[P][P]);
          const bool pos = hh == 0.0 || ((hh > 0.0) == (apq > 0.0));
          const double tt = (pos ? fabs(apq) : -fabs(apq)) / (fabs(hh) + sqrt(fma(hh, hh, apq * apq)));
          c = rsqrt(fma(tt, tt, 1.0));
          s = tt * c;
        }
        pa[t] = P;
        qa[t] = Q;
        cs[t] = c;
        sn[t] = s;
      }
      __syncthreads();
      // rows: A <- P^T A (pair k per warp, column j per lane: no integer division per element)
      const int npr = n2 / 2, nwp = blockDim.x >> 5, wid = t >> 5, ln = t & 31;
      for (int k = wid; k < npr; k += nwp) {
        const int P = pa[k], Q = qa[k];
        if (Q >= p || sn[k] == 0.0) continue;
        const double c = cs[k], s = sn[k];
        for (int j = ln; j < p; j += 32) {
          const double ap = A[P][j], aq = A[Q][j];
          A[P][j] = c * ap - s * aq;
          A[Q][j] = s * ap + c * aq;
        }
      }
      __syncthreads();
      // columns: A <- A P, V <- V P (pair k per warp, row i per lane)
      for (int k = wid; k < npr; k += nwp) {
        const int P = pa[k], Q = qa[k];
        if (Q >= p || sn[k] == 0.0) continue;
        const double c = cs[k], s = sn[k];
        for (int i = ln; i < p; i += 32) {
          const double ap = A[i][P], aq = A[i][Q];
          A[i][P] = c * ap - s * aq;
          A[i][Q] = s * ap + c * aq;
          const double vp = V[i][P], vq = V[i][Q];
          V[i][P] = c * vp - s * vq;
          V[i][Q] = s * vp + c * vq;
        }
      }
      __syncthreads();
      if (t < n2 / 2) {
        int P = pa[t], Q = qa[t];
        if (Q < p && sn[t] != 0.0) {
          A[P][Q] = 0.0;
          A[Q][P] = 0.0;
        }
      }
      __syncthreads();
    }
    if (!s_rot) break;  // a sweep without a rotation: converged
  }
  // sort eigenvalues descending (stable), normalise signs
  if (t == 0) {
    int idx[RTD_MAXP];
    for (int k = 0; k < p; k++) idx[k] = k;
    for (int i = 1; i < p; i++) {  // insertion sort, stable
      int v = idx[i];
      int j = i - 1;
      while (j >= 0 && A[idx[j]][idx[j]] < A[v][v]) {
        idx[j + 1] = idx[j];
        j--;
      }
      idx[j + 1] = v;
    }
    for (int k = 0; k < p; k++) order[k] = idx[k];
    double lmax = A[idx[0]][idx[0]], lmin = A[idx[p - 1]][idx[p - 1]];
    ok_all[b] = (lmin > 0.0 && lmax / lmin <= kappa_max) ? 1 : 0;
  }
  __syncthreads();
  double* Vo = V_all + (long long)b * RTD_MAXP * RTD_MAXP;
  double* lo = lam_all + (long long)b * RTD_MAXP;
  if (t < p) {
    const int src = order[t];
    lo[t] = A[src][src];
    int km = 0;
    double vm = fabs(V[0][src]);
    for (int i = 1; i < p; i++)
      if (fabs(V[i][src]) > vm) { vm = fabs(V[i][src]); km = i; }
    const double sg = V[km][src] < 0 ? -1.0 : 1.0;
    for (int i = 0; i < p; i++) Vo[i * p + t] = sg * V[i][src];
  }
}

// One-sided (Hestenes) Jacobi for the symmetric positive semi-definite inputs (S~1, S~2, Sigma_k: Gram
// matrices): the columns of A are rotated in place, A <- A J, V <- V J, until every pair is orthogonal to
// |a_P . a_Q| <= tol ||a_P|| ||a_Q||; then A V = V diag(lambda) and lambda_j = v_j . a_j (the
// eigenvectors of the initial estimates).  One warp per pair of the round-robin schedule computes the pair's
// three dot products (butterfly shuffles: every lane holds the same sums), the rotation in registers and
// the two column updates, so a round is one barrier and one chain of slow fp64 operations (the two-sided
// form needed four barriers and a shared-memory hand-off of (c, s) per round: 0.83 ms for the 16 40 x 40
// matrices of config 4, 57 us for config 5's two 8 x 8).
__device__ int g_jacobi_sweeps[64];  // RTD_DEBUG_JACOBI: sweeps of the first 64 matrices of the last launch
static constexpr int JCS = 64;  // column stride of the column-major copies (rows lane and lane + 32)
__global__ void __launch_bounds__(32 * (RTD_MAXP / 2)) k_jacobi_os(const double* __restrict__ A_all, int p,
                                                                   double kappa_max, double* __restrict__ V_all,
                                                                   double* __restrict__ lam_all,
                                                                   int* __restrict__ ok_all) {
  __shared__ double Ac[RTD_MAXP][JCS], Vc[RTD_MAXP][JCS];
  __shared__ double lam_s[RTD_MAXP], nrm[RTD_MAXP];
  __shared__ int order[RTD_MAXP];
  __shared__ int s_rot[3];
  __shared__ unsigned char pq[RTD_MAXP - 1][RTD_MAXP / 2][2];  // round-robin schedule: (P, Q) of pair w in a round
  const int b = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5, nw = blockDim.x >> 5;
  const double* Ain = A_all + (long long)b * RTD_MAXP * RTD_MAXP;
  for (int j = w; j < RTD_MAXP; j += nw)
    for (int i = lane; i < JCS; i += 32) {
      const bool in = i < p && j < p;
      Ac[j][i] = in ? 0.5 * (Ain[i * p + j] + Ain[j * p + i]) : 0.0;
      Vc[j][i] = (in && i == j) ? 1.0 : 0.0;
    }
  if (t < 3) s_rot[t] = 0;
  const int n2 = p + (p & 1);
  // positions: 0 fixed, 1..n2-1 rotated right by one per round (period n2 - 1: every sweep starts from the
  // identity); tabulated once (the integer modulo per round and lane was on the critical path)
  for (int e = t; e < (n2 - 1) * (n2 / 2); e += blockDim.x) {
    const int round = e / (n2 / 2), k = e - round * (n2 / 2);
    auto ord = [&](int x) { return x == 0 ? 0 : 1 + ((x - 1 - round) % (n2 - 1) + (n2 - 1)) % (n2 - 1); };
    int P = ord(k), Q = ord(n2 - 1 - k);
    if (P > Q) { const int tmp = P; P = Q; Q = tmp; }
    pq[round][k][0] = (unsigned char)P;
    pq[round][k][1] = (unsigned char)Q;
  }
  // rotate while |a_P . a_Q| > tol ||a_P|| ||a_Q||: the rounding of a rotation leaves a few eps of relative
  // non-orthogonality, so tol must sit above it or the sweeps never end (LAPACK's dgesvj: sqrt(m) eps)
  constexpr double tol = 1e-14;
  int lanes = 1;  // lanes holding rows (rows lane and lane + 32)
  while (lanes < 32 && lanes < p) lanes <<= 1;
  __syncthreads();
  for (int sweep = 0; sweep < 60; sweep++) {
    const int fs = sweep % 3;
    if (t == 0) s_rot[(sweep + 1) % 3] = 0;  // the next sweep's flag (triple-buffered: no reader races)
    // squared column norms, recomputed at every sweep and carried through the rotations of the sweep
    // (a_P' = c a_P - s a_Q: alpha' = c^2 alpha - 2 c s gamma + s^2 beta, beta' = s^2 alpha + 2 c s gamma +
    // c^2 beta), so a round reduces one dot product instead of three
    for (int j = w; j < p; j += nw) {
      double v = fma(Ac[j][lane], Ac[j][lane], Ac[j][lane + 32] * Ac[j][lane + 32]);
      for (int d = 1; d < lanes; d <<= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
      if (lane == 0) nrm[j] = v;
    }
    __syncthreads();
    for (int round = 0; round < n2 - 1; round++) {
      if (w < n2 / 2) {
        const int P = pq[round][w][0], Q = pq[round][w][1];
        if (Q < p) {
          double aP0 = Ac[P][lane], aP1 = Ac[P][lane + 32], aQ0 = Ac[Q][lane], aQ1 = Ac[Q][lane + 32];
          const double al = nrm[P], be = nrm[Q];
          double ga = fma(aP0, aQ0, aP1 * aQ1);
          // butterfly over the lanes that hold rows (the others hold zeros): every such lane gets the sum
          for (int d = 1; d < lanes; d <<= 1) ga += __shfl_xor_sync(0xffffffffu, ga, d);
          if (ga != 0.0 && ga * ga > tol * tol * al * be) {
            // the rotation zeroing a_P . a_Q (zeta = (be - al) / (2 ga), t = tan theta = sign(zeta) / (|zeta| +
            // sqrt(1 + zeta^2))) from two rsqrt and no division: with h = (be - al) / 2, r = sqrt(h^2 + ga^2),
            // cos^2 theta = (1 + |h| / r) / 2 (>= 1/2: no cancellation), sin theta = sign(h ga) |ga| / (2 r cos theta)
            const double hh = 0.5 * (be - al);
            const bool pos = hh == 0.0 || ((hh > 0.0) == (ga > 0.0));
            const double ir = rsqrt(fma(hh, hh, ga * ga));
            const double c2 = 0.5 * fma(fabs(hh), ir, 1.0), rc = rsqrt(c2);
            const double c = c2 * rc, s = (pos ? fabs(ga) : -fabs(ga)) * ir * 0.5 * rc;
            Ac[P][lane] = c * aP0 - s * aQ0;
            Ac[Q][lane] = s * aP0 + c * aQ0;
            Ac[P][lane + 32] = c * aP1 - s * aQ1;
            Ac[Q][lane + 32] = s * aP1 + c * aQ1;
            const double vP0 = Vc[P][lane], vP1 = Vc[P][lane + 32], vQ0 = Vc[Q][lane], vQ1 = Vc[Q][lane + 32];
            Vc[P][lane] = c * vP0 - s * vQ0;
            Vc[Q][lane] = s * vP0 + c * vQ0;
            Vc[P][lane + 32] = c * vP1 - s * vQ1;
            Vc[Q][lane + 32] = s * vP1 + c * vQ1;
            if (lane == 0) {
              s_rot[fs] = 1;
              const double cc = c * c, ss = s * s, cs2 = 2.0 * c * s * ga;
              nrm[P] = fma(cc, al, fma(ss, be, -cs2));
              nrm[Q] = fma(ss, al, fma(cc, be, cs2));
            }
          }
        }
      }
      __syncthreads();
    }
    if (!s_rot[fs]) {  // a sweep without a rotation: converged
      if (t == 0 && b < 64) g_jacobi_sweeps[b] = sweep + 1;
      break;
    }
  }
  // lambda_j = v_j . (A v_j), the rotated column a_j = A v_j (one warp per column)
  for (int j = w; j < p; j += nw) {
    double v = fma(Vc[j][lane], Ac[j][lane], Vc[j][lane + 32] * Ac[j][lane + 32]);
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (lane == 0) lam_s[j] = v;
  }
  __syncthreads();
  // sort eigenvalues descending (stable), normalise signs (largest |component| positive)
  if (t == 0) {
    int idx[RTD_MAXP];
    for (int k = 0; k < p; k++) idx[k] = k;
    for (int i = 1; i < p; i++) {
      const int v = idx[i];
      int j = i - 1;
      while (j >= 0 && lam_s[idx[j]] < lam_s[v]) {
        idx[j + 1] = idx[j];
        j--;
      }
      idx[j + 1] = v;
    }
    for (int k = 0; k < p; k++) order[k] = idx[k];
    const double lmax = lam_s[idx[0]], lmin = lam_s[idx[p - 1]];
    ok_all[b] = (lmin > 0.0 && lmax / lmin <= kappa_max) ? 1 : 0;
  }
  __syncthreads();
  double* Vo = V_all + (long long)b * RTD_MAXP * RTD_MAXP;
  double* lo = lam_all + (long long)b * RTD_MAXP;
  for (int k = w; k < p; k += nw) {  // output column k = eigenvector order[k]
    const int src = order[k];
    const double x0 = Vc[src][lane], x1 = lane + 32 < p ? Vc[src][lane + 32] : 0.0;
    // row index of the largest |component| (lowest row on ties, as the serial scan)
    double vm = fabs(x0);
    int km = lane < p ? lane : RTD_MAXP;
    if (lane + 32 < p && fabs(x1) > vm) {
      vm = fabs(x1);
      km = lane + 32;
    }
    if (lane >= p) vm = -1.0;
    for (int d = 16; d > 0; d >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, vm, d);
      const int ok = __shfl_xor_sync(0xffffffffu, km, d);
      if (ov > vm || (ov == vm && ok < km)) {
        vm = ov;
        km = ok;
      }
    }
    const double sg = Vc[src][km] < 0 ? -1.0 : 1.0;
    if (lane < p) Vo[lane * p + k] = sg * x0;
    if (lane + 32 < p) Vo[(lane + 32) * p + k] = sg * x1;
    if (lane == 0) lo[k] = lam_s[src];
  }
}

void launch_jacobi(const double* A_all, int nb, int p, double kappa_max, double* V_all, double* lam_all, int* ok_all,
                   cudaStream_t st) {
  static const bool two_sided = getenv("RTD_JACOBI_TWOSIDED") != nullptr;
  if (two_sided) {
    k_jacobi<<<nb, LT, 0, st>>>(A_all, p, kappa_max, V_all, lam_all, ok_all);
  } else {
    const int npr = std::max(1, (p + (p & 1)) / 2);
    k_jacobi_os<<<nb, 32 * npr, 0, st>>>(A_all, p, kappa_max, V_all, lam_all, ok_all);
  }
  RTD_LAUNCHED();
  static const bool dbg = getenv("RTD_DEBUG_JACOBI") != nullptr;
  if (dbg && !two_sided) {
    int sw[64];
    RTD_CU(cudaStreamSynchronize(st));
    RTD_CU(cudaMemcpyFromSymbol(sw, g_jacobi_sweeps, sizeof(sw)));
    fprintf(stderr, "[jacobi] p=%d nb=%d sweeps:", p, nb);
    for (int i = 0; i < std::min(nb, 64); i++) fprintf(stderr, " %d", sw[i]);
    fprintf(stderr, "\n");
  }
}

// ------------------------------------------------------------------ refinement matrices
// which: 0 -> Sigma = V diag(d) V^T ; 1 -> V diag(d^-1/2) V^T ; 2 -> V diag(d^1/2) V^T
__global__ void k_vdv(const double* __restrict__ V_all, const double* __restrict__ d_all, int p, int which,
                      double* __restrict__ out_all) {
  const int b = blockIdx.x;
  const double* V = V_all + (long long)b * RTD_MAXP * RTD_MAXP;
  const double* d = d_all + (long long)b * RTD_MAXP;
  double* o = out_all + (long long)b * RTD_MAXP * RTD_MAXP;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    int i = e / p, j = e - i * p;
    double s = 0.0;
    for (int k = 0; k < p; k++) {
      double dk = which == 0 ? d[k] : (which == 1 ? 1.0 / sqrt(d[k]) : sqrt(d[k]));
      s += V[i * p + k] * dk * V[j * p + k];
    }
    o[e] = s;
  }
}

void launch_vdv(const double* V_all, const double* d_all, int nb, int p, int which, double* out_all, cudaStream_t st) {
  k_vdv<<<nb, 256, 0, st>>>(V_all, d_all, p, which, out_all);
  RTD_LAUNCHED();
}

// y = A x for nb instances (A p x p row-major, stride MAXP^2; x, y stride MAXP)
__global__ void k_matvec(const double* __restrict__ A_all, const double* __restrict__ x_all, int p,
                         double* __restrict__ y_all) {
  const int b = blockIdx.x;
  const double* A = A_all + (long long)b * RTD_MAXP * RTD_MAXP;
  const double* x = x_all + (long long)b * RTD_MAXP;
  for (int i = threadIdx.x; i < p; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < p; k++) s += A[i * p + k] * x[k];
    y_all[(long long)b * RTD_MAXP + i] = s;
  }
}

void launch_matvec(const double* A_all, const double* x_all, int nb, int p, double* y_all, cudaStream_t st) {
  k_matvec<<<nb, 64, 0, st>>>(A_all, x_all, p, y_all);
  RTD_LAUNCHED();
}

// ------------------------------------------------------------------ type-7 quantile cutoffs of sorted norms
__global__ void k_lr_cutoffs(const double* __restrict__ rs_all, long long m, double* __restrict__ AB, int* __restrict__ ok) {
  const int b = blockIdx.x;
  if (threadIdx.x != 0) return;
  const double* y = rs_all + (long long)b * m;
  auto q7 = [&](double prob) {
    double hpos = (double)(m - 1) * prob;
    long long j = (long long)floor(hpos);
    double g = hpos - (double)j;
    if (j + 1 >= m) return y[m - 1];
    return y[j] + g * (y[j + 1] - y[j]);
  };
  double A = q7(0.5);
  double iqr = q7(0.75) - q7(0.25);
  AB[2 * b] = A;
  AB[2 * b + 1] = A + 1.5 * iqr;
  ok[b] = iqr > 0.0 ? 1 : 0;
}

void launch_lr_cutoffs(const double* rs_all, int nb, long long m, double* AB, int* ok, cudaStream_t st) {
  k_lr_cutoffs<<<nb, 32, 0, st>>>(rs_all, m, AB, ok);
  RTD_LAUNCHED();
}

// ------------------------------------------------------------------ aggregation of q block fits (K11)
// in: mu[b][MAXP], sig[b][MAXP^2] for nv valid blocks (ids ascending), m rows per block.
// out: mu_raw, sigma_raw; kept[b] flags; keys[b]
// (a) entrywise median over the nv valid fits (even count -> mean of the two middle values, R14):
//     one thread per entry, order statistics by counting (no per-thread arrays, any nv)
__global__ void __launch_bounds__(LT) k_agg_median(const double* __restrict__ mu_base, const double* __restrict__ sig_base,
                                                   const int* __restrict__ ids, int nv, int p,
                                                   double* __restrict__ med /* [p + p*p] */) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= p + p * p) return;
  auto val = [&](int l) {
    return e < p ? mu_base[(long long)ids[l] * RTD_MAXP + e] : sig_base[(long long)ids[l] * RTD_MAXP * RTD_MAXP + e - p];
  };
  // k-th smallest (0-based) with ties: the value x_l with #{x < x_l} <= k < #{x <= x_l}
  auto kth = [&](int k) {
    double r = 0.0;
    for (int l = 0; l < nv; l++) {
      const double x = val(l);
      int lt = 0, le = 0;
      for (int u = 0; u < nv; u++) {
        const double y = val(u);
        lt += y < x;
        le += y <= x;
      }
      if (lt <= k && k < le) r = x;
    }
    return r;
  };
  med[e] = (nv & 1) ? kth(nv / 2) : 0.5 * (kth(nv / 2 - 1) + kth(nv / 2));
}

// (b) KL' key of every fit, one CTA per fit: tr(S_med S_l^-1) + log det S_l + (mu_med - mu_l)^T S_l^-1 (...)
//     (reading R15; INFINITY when S_l is not positive definite)
__global__ void __launch_bounds__(LT) k_agg_keys(const double* __restrict__ mu_base, const double* __restrict__ sig_base,
                                                 const int* __restrict__ ids, int p, const double* __restrict__ med,
                                                 double* __restrict__ keys) {
  __shared__ double A[RTD_MAXP * LD], L[RTD_MAXP * LD], Li[RTD_MAXP * LD];
  __shared__ double dm[RTD_MAXP], red[LT / 32];
  __shared__ int s_fail;
  const int l = blockIdx.x, t = threadIdx.x;
  const double* S = sig_base + (long long)ids[l] * RTD_MAXP * RTD_MAXP;
  const double* mu = mu_base + (long long)ids[l] * RTD_MAXP;
  for (int e = t; e < p * p; e += blockDim.x) A[(e / p) * LD + e % p] = S[e];
  for (int k = t; k < p; k += blockDim.x) dm[k] = med[k] - mu[k];
  __syncthreads();
  if (!block_cholesky(A, L, p, &s_fail)) {
    if (t == 0) keys[l] = INFINITY;
    return;
  }
  block_tri_inverse(L, Li, p);
  block_inv_from_li(Li, A, p);  // A = S_l^-1
  const double* smed = med + p;
  double part = 0.0;
  for (int e = t; e < p * p; e += blockDim.x) {
    const int i = e / p, k = e - i * p;
    part += smed[i * p + k] * A[k * LD + i] + dm[i] * A[i * LD + k] * dm[k];
  }
  if (t < p) part += 2.0 * log(L[t * LD + t]);
  for (int d = 16; d > 0; d >>= 1) part += __shfl_down_sync(0xffffffffu, part, d);
  if ((t & 31) == 0) red[t >> 5] = part;
  __syncthreads();
  if (t == 0) {
    double k = 0.0;
    for (int w = 0; w < LT / 32; w++) k += red[w];
    keys[l] = k;
  }
}

// (c) keep ceil(nv/2) smallest keys (ties -> lower block position), single-pass pooling (eqs. covpool)
//     in block order with weight m (reading R15)
__global__ void __launch_bounds__(LT) k_agg_pool(const double* __restrict__ mu_base, const double* __restrict__ sig_base,
                                                 const int* __restrict__ ids, int nv, int p, double m,
                                                 const double* __restrict__ keys, double* __restrict__ mu_out,
                                                 double* __restrict__ sig_out, int* __restrict__ kept,
                                                 double* __restrict__ scratch) {
  __shared__ int s_order[1024];
  __shared__ double mup[RTD_MAXP], dmu[RTD_MAXP];
  __shared__ double np_s;
  const int t = threadIdx.x;
  if (t == 0) {
    for (int l = 0; l < nv; l++) s_order[l] = l;
    for (int i = 1; i < nv; i++) {
      int v = s_order[i], j = i - 1;
      while (j >= 0 && (keys[s_order[j]] > keys[v])) { s_order[j + 1] = s_order[j]; j--; }
      s_order[j + 1] = v;
    }
    const int keep = (nv + 1) / 2;
    for (int l = 0; l < nv; l++) kept[l] = 0;
    for (int i = 0; i < keep; i++) kept[s_order[i]] = 1;
  }
  __syncthreads();
  double* Lam = scratch;
  int first = 1;
  for (int l = 0; l < nv; l++) {
    if (!kept[l]) continue;
    const double* S = sig_base + (long long)ids[l] * RTD_MAXP * RTD_MAXP;
    const double* mu = mu_base + (long long)ids[l] * RTD_MAXP;
    if (first) {
      for (int e = t; e < p * p; e += blockDim.x) Lam[e] = (m - 1.0) * S[e];
      for (int k = t; k < p; k += blockDim.x) mup[k] = mu[k];
      if (t == 0) np_s = m;
      first = 0;
      __syncthreads();
      continue;
    }
    for (int k = t; k < p; k += blockDim.x) dmu[k] = mu[k] - mup[k];
    __syncthreads();
    const double npool = np_s;
    const double w = npool * m / (npool + m);
    for (int e = t; e < p * p; e += blockDim.x) {
      int i = e / p, j = e - i * p;
      Lam[e] = Lam[e] + (m - 1.0) * S[e] + dmu[i] * dmu[j] * w;
    }
    for (int k = t; k < p; k += blockDim.x) mup[k] = (npool * mup[k] + m * mu[k]) / (npool + m);
    __syncthreads();
    if (t == 0) np_s = npool + m;
    __syncthreads();
  }
  for (int k = t; k < p; k += blockDim.x) mu_out[k] = mup[k];
  for (int e = t; e < p * p; e += blockDim.x) sig_out[e] = Lam[e] / (np_s - 1.0);
}

void launch_aggregate(const double* mu_base, const double* sig_base, const int* ids, int nv, int p, double m,
                      double* mu_out, double* sig_out, int* kept, double* keys, double* scratch, cudaStream_t st) {
  if (nv > 1024) throw std::string("aggregate: at most 1024 blocks");
  double* med = scratch + RTD_MAXP * RTD_MAXP;  // [p + p*p] after the pooling scratch
  k_agg_median<<<(p + p * p + LT - 1) / LT, LT, 0, st>>>(mu_base, sig_base, ids, nv, p, med);
  RTD_LAUNCHED();
  k_agg_keys<<<nv, LT, 0, st>>>(mu_base, sig_base, ids, p, med, keys);
  RTD_LAUNCHED();
  k_agg_pool<<<1, LT, 0, st>>>(mu_base, sig_base, ids, nv, p, m, keys, mu_out, sig_out, kept, scratch);
  RTD_LAUNCHED();
}

// ------------------------------------------------------------------ pool reweight partial sums over blocks
// sums[b][np] about the common shift c; out mu, Sigma = factor * (S2 - S1 S1^T/k)/(k-1)
__global__ void k_pool_sums(const double* __restrict__ sums_all, int nb, int np, double* __restrict__ out) {
  for (int e = threadIdx.x; e < np; e += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nb; b++) s += sums_all[(long long)b * np + e];
    out[e] = s;
  }
}

void launch_pool_sums(const double* sums_all, int nb, int np, double* out, cudaStream_t st) {
  k_pool_sums<<<1, 256, 0, st>>>(sums_all, nb, np, out);
  RTD_LAUNCHED();
}

// mu_X = loc + scale mu_Z ; Sigma_X = diag(scale) Sigma_Z diag(scale)
__global__ void k_destandardize(const UniOut* __restrict__ uni, const double* __restrict__ mu_z,
                                const double* __restrict__ sig_z, int p, double* __restrict__ mu_x,
                                double* __restrict__ sig_x) {
  for (int k = threadIdx.x; k < p; k += blockDim.x) mu_x[k] = uni[k].loc + uni[k].scale * mu_z[k];
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    int i = e / p, j = e - i * p;
    sig_x[e] = sig_z[e] * (uni[i].scale * uni[j].scale);
  }
}

void launch_destandardize(const UniOut* uni, const double* mu_z, const double* sig_z, int p, double* mu_x,
                          double* sig_x, cudaStream_t st) {
  k_destandardize<<<1, 256, 0, st>>>(uni, mu_z, sig_z, p, mu_x, sig_x);
  RTD_LAUNCHED();
}

}  // namespace rtd
