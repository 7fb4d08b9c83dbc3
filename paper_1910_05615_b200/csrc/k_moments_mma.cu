// Moments and the refinement GEMMs on the FP64 tensor pipe (DMMA m8n8k4).
//
// k_moments_mma: S2 = sum_r w_r u_r u_r^T (lower 8x8 blocks), S1 = sum_r w_r u_r,
//   count = sum_r w_r over the rows of a block, for every MomMode of
//   k_moments.cu (wrapping S~1, LR-GSSCM S~2, C-step dense / delta moments,
//   reweighting).  Each warp takes 4 rows per step: lane (g, t) loads
//   u[r0 + t][8b + g] for every 8-column group b and feeds it as the A operand
//   (scaled by w) of block row b and as the B operand of block column b, so
//   one load serves (NB+1)/2 DMMAs.  Groups of 4 rows whose weights are all
//   zero (most rows of the update-based C-step) are skipped
//   without reading Z; the update-based C-step (MOM_DELTA) reads only the
//   ordered changed-row list written by the select (k_sel_member), a gather of
//   the entering / leaving rows.  Partials are reduced in a fixed order
//   (deterministic).
// k_matmul_mma: out = Z W (W full p x p, e.g. the eigenvectors V or
//   Sigma^-1/2 of the refinement), column-major out.
#include <algorithm>
#include <cstdlib>

#include "rtd_internal.h"

namespace rtd {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double wrap_g2(double z) {
  const double b = 1.5, c = 4.0, q1 = 1.541, q2 = 0.862;
  double az = fabs(z);
  if (az <= b) return z;
  if (az <= c) {
    double t = __dmul_rn(q1, tanh(__dmul_rn(q2, __dsub_rn(c, az))));
    return z > 0 ? t : (z < 0 ? -t : 0.0);
  }
  return 0.0;
}

static constexpr int MW = 8;  // warps per CTA
static constexpr int RG = 4;  // 4-row groups per warp iteration (loads in flight)

// per-warp results -> shared memory -> fixed-order sum over the warps -> this CTA's partial row
template <int NB>
__device__ __forceinline__ void mom_epilogue(double (&acc)[NB * (NB + 1) / 2][2], double (&s1)[NB], double cnt,
                                             double* red, const MomArgs& a, int slot, int p, int NP) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, warp = threadIdx.x >> 5;
  // reduce: S1 over the 4 t-lanes, count over the t-lanes of g == 0
#pragma unroll
  for (int b = 0; b < NB; b++) {
    s1[b] += __shfl_xor_sync(0xffffffffu, s1[b], 1);
    s1[b] += __shfl_xor_sync(0xffffffffu, s1[b], 2);
  }
  cnt += __shfl_xor_sync(0xffffffffu, cnt, 1);
  cnt += __shfl_xor_sync(0xffffffffu, cnt, 2);
  double* rw = red + warp * NP;
  for (int e = lane; e < NP; e += 32) rw[e] = 0.0;
  __syncwarp();
  if (t == 0) {
#pragma unroll
    for (int b = 0; b < NB; b++)
      if (8 * b + g < p) rw[8 * b + g] = s1[b];
  }
  if (lane == 0) rw[NP - 1] = cnt;
  {
    int k = 0;
#pragma unroll
    for (int jb = 0; jb < NB; jb++)
#pragma unroll
      for (int kb = 0; kb <= jb; kb++) {
        const int j = 8 * jb + g;
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int kk = 8 * kb + 2 * t + e;
          if (j < p && kk < p && kk <= j) rw[p + j * (j + 1) / 2 + kk] = acc[k][e];
        }
        k++;
      }
  }
  __syncthreads();
  double* out = a.partial + ((long long)slot * a.ctas + blockIdx.x) * NP;
  for (int e = threadIdx.x; e < NP; e += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < MW; q++) s += red[q * NP + e];
    out[e] = s;
  }
}

// ---------------------------------------------------------------- staged dense moments
// Same sums as k_moments_mma for the dense modes (WRAP, XI, MEMBER, REWEIGHT), with the rows of Z
// streamed through shared memory by cp.async in SR-row tiles, NST stages deep: the loads of the next
// tiles are in flight while the DMMAs of the current one run (ncu put the register-fed kernel at
// 16 long-scoreboard stalls per issue and 35 % DMMA activity).  The per-row weight source (membership
// byte, norm, d^2) is loaded into a register one issue ahead and stored, as the weight, at the next
// issue.  Warp w takes 4-row groups 2w, 2w+1 of each 64-row tile.
static constexpr int SR = 64;        // rows per tile
static constexpr int SLD = SR + 4;   // padded column stride in shared memory (doubles)
static constexpr int NST = 3;        // pipeline stages


template <int NB, int MODE>
__global__ void __launch_bounds__(MW * 32, 2) k_moments_st(MomArgs a) {
  constexpr int NBLK = NB * (NB + 1) / 2;
  extern __shared__ double smem[];  // [NST][p][SLD] tiles, [NST][SR] weights; reused by the epilogue
  const int slot = blockIdx.y;
  const int id = a.inst[slot];
  const int blk = id / a.nstart;
  const int p = a.p;
  const long long m = a.m;
  const double* __restrict__ Z = a.Z + (long long)blk * a.blk_stride;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, warp = threadIdx.x >> 5;
  const int tid = threadIdx.x;
  const int NP = p + p * (p + 1) / 2 + 1;
  double* tiles = smem;
  double* wts = smem + (size_t)NST * p * SLD;
  __shared__ int s_wn;                                   // MOM_WRAP: tanh-branch entries of the tile
  int* wl = reinterpret_cast<int*>(wts + NST * SR);      // MOM_WRAP: their positions (p * SR ints)
  if (MODE == MOM_WRAP && threadIdx.x == 0) s_wn = 0;
  double sh[NB];
#pragma unroll
  for (int b = 0; b < NB; b++)
    sh[b] = (MODE >= MOM_MEMBER && 8 * b + g < p) ? a.shift[(long long)id * RTD_MAXP + 8 * b + g] : 0.0;
  double A = 0.0, B = 0.0;
  if (MODE == MOM_XI) {
    A = a.AB[2 * blk];
    B = a.AB[2 * blk + 1];
  }
  double acc[NBLK][2];
#pragma unroll
  for (int k = 0; k < NBLK; k++) acc[k][0] = acc[k][1] = 0.0;
  double s1[NB];
#pragma unroll
  for (int b = 0; b < NB; b++) s1[b] = 0.0;
  double cnt = 0.0;
  long long per = (m + a.ctas - 1) / a.ctas;
  per = (per + 3) / 4 * 4;
  const long long r_begin = (long long)blockIdx.x * per, r_end = min(m, r_begin + per);
  const int ntile = r_end > r_begin ? (int)((r_end - r_begin + SR - 1) / SR) : 0;
  // weight of row r (0 beyond the range)
  auto wsrc = [&](long long r) -> double {
    if (r >= r_end) return 0.0;
    if (MODE == MOM_WRAP) return 1.0;
    if (MODE == MOM_MEMBER) return (double)a.mem_new[(long long)id * m + r];
    if (MODE == MOM_XI) {
      const double rr = a.r[(long long)blk * m + r];
      const double xi = rr <= A ? 1.0 : (rr <= B ? __ddiv_rn(__dsub_rn(B, rr), __dsub_rn(B, A)) : 0.0);
      return __dmul_rn(xi, xi);
    }
    return a.d2[(long long)id * m + r] <= a.c2 ? 1.0 : 0.0;
  };
  double wpend = 0.0;
  int wpend_stage = -1;
  auto issue = [&](int tile) {
    if (wpend_stage >= 0 && tid < SR) wts[wpend_stage * SR + tid] = wpend;  // weight loaded one issue ago
    wpend_stage = -1;
    if (tile < ntile) {
      const int stg = tile % NST;
      const long long row0 = r_begin + (long long)tile * SR;
      const int rows = (int)min((long long)SR, r_end - row0);
      double* T = tiles + (size_t)stg * p * SLD;
      for (int e = tid; e < p * SR; e += MW * 32) {
        const int k = e / SR, r = e - k * SR;
        if (r < rows) cp_async8(T + k * SLD + r, Z + (long long)k * m + row0 + r);
      }
      if (tid < SR) {
        wpend = wsrc(row0 + tid);
        wpend_stage = stg;
      }
    }
    cp_async_commit();
  };
  issue(0);
  issue(1);
  for (int tile = 0; tile < ntile; tile++) {
    issue(tile + 2);  // stores tile+1's weights, fetches tile+2 into the stage tile-1 used
    cp_async_wait<2>();
    __syncthreads();
    const int stg = tile % NST;
    const double* T = tiles + (size_t)stg * p * SLD;
    const double* W = wts + stg * SR;
    if (MODE == MOM_WRAP && a.r_out) {
      // the norms ||z_i|| of the tile's rows for S~2 from the raw tile, before psi:
      // 4 threads per row, fixed-order combination
      const int row = tid >> 2, part = tid & 3;
      const int rows_n = (int)min((long long)SR, r_end - (r_begin + (long long)tile * SR));
      double sq = 0.0;
      for (int k = part; k < p; k += 4) {
        const double v = T[k * SLD + row];
        sq = __dadd_rn(sq, __dmul_rn(v, v));
      }
      sq = __dadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, 1));
      sq = __dadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, 2));
      if (part == 0 && row < rows_n) a.r_out[(long long)blk * m + r_begin + (long long)tile * SR + row] = __dsqrt_rn(sq);
      __syncthreads();  // the raw tile is read before psi overwrites it
    }
    if (MODE == MOM_WRAP) {
      // psi of the tile in place: identity and zero branches directly, the tanh
      // branch (b < |z| <= c, a minority of the entries) compacted into a list and evaluated once per
      // listed entry instead of by every warp whose lanes hold any such entry
      double* Tw = tiles + (size_t)stg * p * SLD;
      const int rows_t = (int)min((long long)SR, r_end - (r_begin + (long long)tile * SR));
      for (int e0 = 0; e0 < p * SR; e0 += MW * 32) {
        const int e = e0 + tid, k = e / SR, r = e - k * SR;
        const bool in = e < p * SR && r < rows_t;
        const double z = in ? Tw[k * SLD + r] : 0.0, az = fabs(z);
        const bool need = in && az > 1.5 && az <= 4.0;
        if (in && az > 4.0) Tw[k * SLD + r] = 0.0;
        const unsigned bal = __ballot_sync(0xffffffffu, need);
        if (bal) {
          int pos = 0;
          if (lane == (unsigned)(__ffs(bal) - 1)) pos = atomicAdd(&s_wn, __popc(bal));
          pos = __shfl_sync(0xffffffffu, pos, __ffs(bal) - 1) + __popc(bal & ((1u << lane) - 1u));
          if (need) wl[pos] = k * SLD + r;
        }
      }
      __syncthreads();
      const int nw = s_wn;
      for (int i = tid; i < nw; i += MW * 32) Tw[wl[i]] = wrap_g2(Tw[wl[i]]);
      __syncthreads();
      if (tid == 0) s_wn = 0;  // every thread has read the count; the next use follows two barriers
    }
#pragma unroll
    for (int q = 0; q < 2; q++) {
      const int r = (2 * warp + q) * 4 + t;  // row of this lane in the tile
      const double w = W[r];
      if (!__any_sync(0xffffffffu, w != 0.0)) continue;
      double u[NB];
#pragma unroll
      for (int b = 0; b < NB; b++) {
        const int col = 8 * b + g;
        double v = (w != 0.0 && col < p) ? T[col * SLD + r] : 0.0;  // MOM_WRAP: psi already applied
        if (MODE >= MOM_MEMBER) v = (w != 0.0 && col < p) ? __dsub_rn(v, sh[b]) : 0.0;
        u[b] = v;
      }
      double wu[NB];
#pragma unroll
      for (int b = 0; b < NB; b++) {
        wu[b] = w * u[b];
        s1[b] += wu[b];
      }
      if (g == 0) cnt += w;
      int k = 0;
#pragma unroll
      for (int jb = 0; jb < NB; jb++)
#pragma unroll
        for (int kb = 0; kb <= jb; kb++) {
          dmma(acc[k][0], acc[k][1], wu[jb], u[kb]);
          k++;
        }
    }
    __syncthreads();  // the stage of this tile is refilled two issues later
  }
  cp_async_wait<0>();
  __syncthreads();
  mom_epilogue<NB>(acc, s1, cnt, smem, a, slot, p, NP);
}

template <int NB, int MODE>
__global__ void __launch_bounds__(MW * 32, 2) k_moments_mma(MomArgs a) {
  constexpr int NBLK = NB * (NB + 1) / 2;
  extern __shared__ double red[];  // [MW][NP]
  const int slot = blockIdx.y;
  const int id = a.inst[slot];
  const int blk = id / a.nstart;
  const int p = a.p;
  const long long m = a.m;
  const double* __restrict__ Z = a.Z + (long long)blk * a.blk_stride;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, warp = threadIdx.x >> 5;
  const int NP = p + p * (p + 1) / 2 + 1;
  const double* shift = (MODE >= MOM_MEMBER) ? a.shift + (long long)id * RTD_MAXP : nullptr;
  double sh[NB];
#pragma unroll
  for (int b = 0; b < NB; b++) sh[b] = (shift && 8 * b + g < p) ? shift[8 * b + g] : 0.0;
  double A = 0.0, B = 0.0;
  if (MODE == MOM_XI) {
    A = a.AB[2 * blk];
    B = a.AB[2 * blk + 1];
  }
  double acc[NBLK][2];
#pragma unroll
  for (int k = 0; k < NBLK; k++) acc[k][0] = acc[k][1] = 0.0;
  double s1[NB];
#pragma unroll
  for (int b = 0; b < NB; b++) s1[b] = 0.0;
  double cnt = 0.0;
  // rows of this CTA: contiguous range, 4-row groups interleaved over warps; the update-based
  // C-step (MOM_DELTA) walks instead the ordered list of changed rows of segment blockIdx.x
  long long per = (m + a.ctas - 1) / a.ctas;
  per = (per + 3) / 4 * 4;
  long long r_begin = (long long)blockIdx.x * per, r_end = min(m, r_begin + per);
  const int* lst = nullptr;
  if (MODE == MOM_DELTA) {
    lst = a.list + (long long)id * m + (long long)blockIdx.x * a.seg_len;
    r_begin = 0;
    r_end = a.seg_cnt[(long long)id * a.ctas + blockIdx.x];
  }
  // RG groups of 4 rows per warp iteration: all of their loads are issued before the first DMMA
  for (long long rb = r_begin + 4LL * RG * warp; rb < r_end; rb += 4LL * RG * MW) {
    long long row[RG];
    double w[RG];
    bool anyw = false;
#pragma unroll
    for (int q = 0; q < RG; q++) {
      row[q] = rb + 4 * q + t;
      w[q] = 0.0;
      if (MODE == MOM_DELTA) {
        if (row[q] < r_end) {
          const int e = lst[row[q]];  // 0: a reserved slot of an unchanged candidate row (k_sel_fixup)
          w[q] = e > 0 ? 1.0 : (e < 0 ? -1.0 : 0.0);
          row[q] = e != 0 ? (e > 0 ? e : -e) - 1 : 0;
        }
      } else if (row[q] < r_end) {
        if (MODE == MOM_WRAP) {
          w[q] = 1.0;
        } else if (MODE == MOM_XI) {
          const double r = a.r[(long long)blk * m + row[q]];
          const double xi = r <= A ? 1.0 : (r <= B ? __ddiv_rn(__dsub_rn(B, r), __dsub_rn(B, A)) : 0.0);
          w[q] = __dmul_rn(xi, xi);
        } else if (MODE == MOM_MEMBER) {
          w[q] = (double)a.mem_new[(long long)id * m + row[q]];
        } else {
          w[q] = a.d2[(long long)id * m + row[q]] <= a.c2 ? 1.0 : 0.0;
        }
      }
      anyw |= w[q] != 0.0;
    }
    if (!__any_sync(0xffffffffu, anyw)) continue;
    double u[RG][NB];
#pragma unroll
    for (int q = 0; q < RG; q++)
#pragma unroll
      for (int b = 0; b < NB; b++) {
        const int col = 8 * b + g;
        u[q][b] = (w[q] != 0.0 && col < p) ? Z[(long long)col * m + row[q]] : 0.0;
      }
#pragma unroll
    for (int q = 0; q < RG; q++) {
#pragma unroll
      for (int b = 0; b < NB; b++) {
        if (MODE == MOM_WRAP) u[q][b] = wrap_g2(u[q][b]);
        else if (MODE >= MOM_MEMBER) u[q][b] = (w[q] != 0.0 && 8 * b + g < p) ? __dsub_rn(u[q][b], sh[b]) : 0.0;
      }
      double wu[NB];
#pragma unroll
      for (int b = 0; b < NB; b++) {
        wu[b] = w[q] * u[q][b];
        s1[b] += wu[b];
      }
      if (g == 0) cnt += w[q];
      int k = 0;
#pragma unroll
      for (int jb = 0; jb < NB; jb++)
#pragma unroll
        for (int kb = 0; kb <= jb; kb++) {
          dmma(acc[k][0], acc[k][1], wu[jb], u[q][kb]);  // A[j][r] = w_r u_r[8jb+j], B[r][k] = u_r[8kb+k]
          k++;
        }
    }
  }
  mom_epilogue<NB>(acc, s1, cnt, red, a, slot, p, NP);
}

template <int NB>
static void moments_mma_nb(int mode, const MomArgs& a, int ninst, cudaStream_t st) {
  const int NP = mom_np(a.p);
  dim3 grid(a.ctas, ninst);
  // staged only where it measured faster on the B200 (config 4, p = 40: dense moments 4.9 -> 3.8 ms per
  // fit); at p <= 24 or short blocks (configs 1-3, 5) the register-fed kernel is faster
  static const bool unstaged = getenv("RTD_MOM_UNSTAGED") != nullptr;
  if (mode != MOM_DELTA && NB >= 4 && a.m >= 65536 && !unstaged) {
    const size_t smem = std::max((size_t)MW * NP * sizeof(double),
                                 ((size_t)NST * a.p * SLD + (size_t)NST * SR) * sizeof(double) +
                                 (size_t)a.p * SR * sizeof(int));
#define RTD_ST_CASE(M)                                                                                   \
  case M:                                                                                                \
    set_max_dyn_smem(reinterpret_cast<const void*>(k_moments_st<NB, M>), (int)smem); \
    k_moments_st<NB, M><<<grid, MW * 32, smem, st>>>(a);                                                 \
    break;
    switch (mode) {
      RTD_ST_CASE(MOM_WRAP)
      RTD_ST_CASE(MOM_XI)
      RTD_ST_CASE(MOM_MEMBER)
      RTD_ST_CASE(MOM_REWEIGHT)
    }
#undef RTD_ST_CASE
    return;
  }
  const size_t smem = (size_t)MW * NP * sizeof(double);
#define RTD_MM_CASE(M)                                                                                   \
  case M:                                                                                                \
    set_max_dyn_smem(reinterpret_cast<const void*>(k_moments_mma<NB, M>), (int)smem);                   \
    k_moments_mma<NB, M><<<grid, MW * 32, smem, st>>>(a);                                                \
    break;
  switch (mode) {
    RTD_MM_CASE(MOM_WRAP)
    RTD_MM_CASE(MOM_XI)
    RTD_MM_CASE(MOM_MEMBER)
    RTD_MM_CASE(MOM_DELTA)
    RTD_MM_CASE(MOM_REWEIGHT)
  }
#undef RTD_MM_CASE
}

bool moments_staged(int mode, const MomArgs& a) {
  static const bool unstaged = getenv("RTD_MOM_UNSTAGED") != nullptr;
  return mode != MOM_DELTA && (a.p + 7) / 8 >= 4 && a.m >= 65536 && !unstaged;
}

void launch_moments_mma(int mode, const MomArgs& a, int ninst, cudaStream_t st) {
  switch ((a.p + 7) / 8) {
    case 1: moments_mma_nb<1>(mode, a, ninst, st); break;
    case 2: moments_mma_nb<2>(mode, a, ninst, st); break;
    case 3: moments_mma_nb<3>(mode, a, ninst, st); break;
    case 4: moments_mma_nb<4>(mode, a, ninst, st); break;
    case 5: moments_mma_nb<5>(mode, a, ninst, st); break;
    default: throw std::string("moments_mma: p out of range");
  }
  RTD_LAUNCHED();
}

// ------------------------------------------------------------------ out = Z W on DMMA
// Batched over work items (blockIdx.y = i): slot = slot_of[i] (or i), Z = Zall + blk_of_slot[slot] *
// blk_stride (or Zall), W = W_all + slot * RTD_MAXP^2, out = out_all + i * p * m.
// BSM: B fragments of W in shared memory (lane-major, conflict-free) instead of registers, so that
// two CTAs fit on an SM at p = 40 (the register-held form runs one CTA of 8 warps at 180 registers)
template <int NB, int MB, bool BSM>
__global__ void __launch_bounds__(256, BSM ? 2 : 1) k_matmul_mma(const double* __restrict__ Zall, long long m, int p,
                                                    long long blk_stride, const int* __restrict__ slot_of,
                                                    const int* __restrict__ blk_of_slot,
                                                    const double* __restrict__ W_all, double* __restrict__ out_all) {
  constexpr int KB = 2 * NB;  // k-blocks of 4 (k padded to 8 NB)
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int slot = slot_of ? slot_of[blockIdx.y] : (int)blockIdx.y;
  const double* __restrict__ Z = Zall + (blk_of_slot ? (long long)blk_of_slot[slot] * blk_stride : 0LL);
  const double* __restrict__ W = W_all + (long long)slot * RTD_MAXP * RTD_MAXP;
  double* __restrict__ out = out_all + (long long)blockIdx.y * p * m;
  __shared__ double bsm[BSM ? KB * NB * 32 : 1];
  double bf[BSM ? 1 : KB][BSM ? 1 : NB];
  if (BSM) {
    for (int e = threadIdx.x; e < KB * NB * 32; e += blockDim.x) {
      const int ln = e & 31, b = e >> 5, kb = b / NB, nb = b - kb * NB;
      const int k = 4 * kb + (ln & 3), j = 8 * nb + (ln >> 2);
      bsm[e] = (k < p && j < p) ? W[k * p + j] : 0.0;
    }
    __syncthreads();
  } else {
#pragma unroll
    for (int kb = 0; kb < KB; kb++)
#pragma unroll
      for (int nb = 0; nb < NB; nb++) {
        const int k = 4 * kb + t, j = 8 * nb + g;
        if (!BSM) bf[kb][nb] = (k < p && j < p) ? W[k * p + j] : 0.0;
      }
  }
  const long long rows_per_tile = 8 * MB;
  const long long ntiles = (m + rows_per_tile - 1) / rows_per_tile;
  const long long warp0 = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long tile = warp0; tile < ntiles; tile += nwarps) {
    const long long r0 = tile * rows_per_tile;
    double acc[MB][NB][2];
#pragma unroll
    for (int mb = 0; mb < MB; mb++)
#pragma unroll
      for (int nb = 0; nb < NB; nb++) acc[mb][nb][0] = acc[mb][nb][1] = 0.0;
#pragma unroll
    for (int kb = 0; kb < KB; kb++) {
      const int k = 4 * kb + t;
      double av[MB];
#pragma unroll
      for (int mb = 0; mb < MB; mb++) {
        const long long row = r0 + mb * 8 + g;
        av[mb] = (k < p && row < m) ? Z[(long long)k * m + row] : 0.0;
      }
#pragma unroll
      for (int nb = 0; nb < NB; nb++) {
        const double bv = BSM ? bsm[(kb * NB + nb) * 32 + lane] : bf[BSM ? 0 : kb][BSM ? 0 : nb];
#pragma unroll
        for (int mb = 0; mb < MB; mb++) dmma(acc[mb][nb][0], acc[mb][nb][1], av[mb], bv);
      }
    }
#pragma unroll
    for (int mb = 0; mb < MB; mb++) {
      const long long row = r0 + mb * 8 + g;
      if (row >= m) continue;
#pragma unroll
      for (int nb = 0; nb < NB; nb++) {
        const int j = 8 * nb + 2 * t;
        if (j < p) out[(long long)j * m + row] = acc[mb][nb][0];
        if (j + 1 < p) out[(long long)(j + 1) * m + row] = acc[mb][nb][1];
      }
    }
  }
}

// Two work items of the same block in one CTA (the refinement's two starts share Z): each A fragment
// of Z feeds the DMMAs of both W, so Z is read once per pair.  pairs[2y], pairs[2y+1]: the items of CTA
// row y (the second -1 for a lone item).  B fragments of both W in shared memory (lane-major).
template <int NB, int MB, int MINB>
__global__ void __launch_bounds__(256, MINB) k_matmul_pair(const double* __restrict__ Zall, long long m, int p,
                                                        long long blk_stride, const int* __restrict__ slot_of,
                                                        const int* __restrict__ blk_of_slot,
                                                        const int* __restrict__ pairs,
                                                        const double* __restrict__ W_all,
                                                        double* __restrict__ out_all) {
  constexpr int KB = 2 * NB;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int i0 = pairs[2 * blockIdx.y], i1 = pairs[2 * blockIdx.y + 1];
  const bool two = i1 >= 0;
  const int s0 = slot_of[i0], s1 = two ? slot_of[i1] : s0;
  const double* __restrict__ Z = Zall + (long long)blk_of_slot[s0] * blk_stride;
  double* __restrict__ out0 = out_all + (long long)i0 * p * m;
  double* __restrict__ out1 = out_all + (long long)(two ? i1 : i0) * p * m;
  __shared__ double bsm[2][KB * NB * 32];
  for (int e = threadIdx.x; e < KB * NB * 32; e += blockDim.x) {
    const int ln = e & 31, b = e >> 5, kb = b / NB, nb = b - kb * NB;
    const int k = 4 * kb + (ln & 3), j = 8 * nb + (ln >> 2);
    const bool in = k < p && j < p;
    bsm[0][e] = in ? W_all[(long long)s0 * RTD_MAXP * RTD_MAXP + k * p + j] : 0.0;
    bsm[1][e] = in ? W_all[(long long)s1 * RTD_MAXP * RTD_MAXP + k * p + j] : 0.0;
  }
  __syncthreads();
  const long long rows_per_tile = 8 * MB;
  const long long ntiles = (m + rows_per_tile - 1) / rows_per_tile;
  const long long warp0 = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long tile = warp0; tile < ntiles; tile += nwarps) {
    const long long r0 = tile * rows_per_tile;
    double acc[2][MB][NB][2];
#pragma unroll
    for (int w = 0; w < 2; w++)
#pragma unroll
      for (int mb = 0; mb < MB; mb++)
#pragma unroll
        for (int nb = 0; nb < NB; nb++) acc[w][mb][nb][0] = acc[w][mb][nb][1] = 0.0;
#pragma unroll
    for (int kb = 0; kb < KB; kb++) {
      const int k = 4 * kb + t;
      double av[MB];
#pragma unroll
      for (int mb = 0; mb < MB; mb++) {
        const long long row = r0 + mb * 8 + g;
        av[mb] = (k < p && row < m) ? Z[(long long)k * m + row] : 0.0;
      }
#pragma unroll
      for (int nb = 0; nb < NB; nb++) {
        const double b0 = bsm[0][(kb * NB + nb) * 32 + lane];
#pragma unroll
        for (int mb = 0; mb < MB; mb++) dmma(acc[0][mb][nb][0], acc[0][mb][nb][1], av[mb], b0);
        if (two) {
          const double b1 = bsm[1][(kb * NB + nb) * 32 + lane];
#pragma unroll
          for (int mb = 0; mb < MB; mb++) dmma(acc[1][mb][nb][0], acc[1][mb][nb][1], av[mb], b1);
        }
      }
    }
#pragma unroll
    for (int w = 0; w < 2; w++) {
      if (w == 1 && !two) break;
      double* __restrict__ out = w ? out1 : out0;
#pragma unroll
      for (int mb = 0; mb < MB; mb++) {
        const long long row = r0 + mb * 8 + g;
        if (row >= m) continue;
#pragma unroll
        for (int nb = 0; nb < NB; nb++) {
          const int j = 8 * nb + 2 * t;
          if (j < p) out[(long long)j * m + row] = acc[w][mb][nb][0];
          if (j + 1 < p) out[(long long)(j + 1) * m + row] = acc[w][mb][nb][1];
        }
      }
    }
  }
}

template <int NB>
static void matmul_pair_nb(const double* Z, long long m, int p, long long blk_stride, const int* slot_of,
                           const int* blk_of_slot, const int* pairs, int npairs, const double* W, double* out,
                           cudaStream_t st) {
  // variant 0: 2 m-blocks per warp at 1 CTA/SM (no spills); 1: 1 m-block at 2 CTAs/SM
  static const int variant = getenv("RTD_MATMUL_PAIR_VARIANT") ? atoi(getenv("RTD_MATMUL_PAIR_VARIANT")) : 0;
  if (variant == 1) {
    constexpr int MB = 1;
    const long long tiles = (m + 8 * MB - 1) / (8 * MB);
    const unsigned grid = (unsigned)std::min<long long>((tiles + 7) / 8, std::max(1, 148 * 4 / std::max(1, npairs)));
    k_matmul_pair<NB, MB, 2><<<dim3(grid, npairs), 256, 0, st>>>(Z, m, p, blk_stride, slot_of, blk_of_slot, pairs, W,
                                                                 out);
    return;
  }
  constexpr int MB = 2;
  const long long tiles = (m + 8 * MB - 1) / (8 * MB);
  const unsigned grid = (unsigned)std::min<long long>((tiles + 7) / 8, std::max(1, 148 * 8 / std::max(1, npairs)));
  k_matmul_pair<NB, MB, 1><<<dim3(grid, npairs), 256, 0, st>>>(Z, m, p, blk_stride, slot_of, blk_of_slot, pairs, W,
                                                               out);
}

void launch_matmul_mma_pairs(int p, const double* Zall, long long m, long long blk_stride, const int* slot_of,
                             const int* blk_of_slot, const int* pairs, int npairs, const double* W_all,
                             double* out_all, cudaStream_t st) {
  switch ((p + 7) / 8) {
    case 4: matmul_pair_nb<4>(Zall, m, p, blk_stride, slot_of, blk_of_slot, pairs, npairs, W_all, out_all, st); break;
    case 5: matmul_pair_nb<5>(Zall, m, p, blk_stride, slot_of, blk_of_slot, pairs, npairs, W_all, out_all, st); break;
    default: throw std::string("matmul_pair: p out of range");
  }
  RTD_LAUNCHED();
}

template <int NB>
static void matmul_mma_nb(const double* Z, long long m, int p, long long blk_stride, const int* slot_of,
                          const int* blk_of_slot, int nitems, const double* W, double* out, cudaStream_t st) {
  // p > 24: B in shared memory, 2 CTAs/SM, 3 m-blocks per warp (measured on config 4: the two refinement
  // GEMMs 6.46 -> 5.13 ms per fit; RTD_MATMUL_VARIANT=0 selects the register-held form)
  static const int variant = getenv("RTD_MATMUL_VARIANT") ? atoi(getenv("RTD_MATMUL_VARIANT")) : 1;
  if (NB >= 4 && variant == 1) {
    constexpr int MB = 3;
    const long long tiles = (m + 8 * MB - 1) / (8 * MB);
    const unsigned grid = (unsigned)std::min<long long>((tiles + 7) / 8, std::max(1, 148 * 4 / std::max(1, nitems)));
    k_matmul_mma<NB, MB, true><<<dim3(grid, nitems), 256, 0, st>>>(Z, m, p, blk_stride, slot_of, blk_of_slot, W, out);
    return;
  }
  constexpr int MB = NB <= 3 ? 4 : 2;
  const long long tiles = (m + 8 * MB - 1) / (8 * MB);
  const unsigned grid = (unsigned)std::min<long long>((tiles + 7) / 8, std::max(1, 148 * 4 / std::max(1, nitems)));
  k_matmul_mma<NB, MB, false><<<dim3(grid, nitems), 256, 0, st>>>(Z, m, p, blk_stride, slot_of, blk_of_slot, W, out);
}

void launch_matmul_mma_batch(int p, const double* Zall, long long m, long long blk_stride, const int* slot_of,
                             const int* blk_of_slot, int nitems, const double* W_all, double* out_all,
                             cudaStream_t st) {
  switch ((p + 7) / 8) {
    case 1: matmul_mma_nb<1>(Zall, m, p, blk_stride, slot_of, blk_of_slot, nitems, W_all, out_all, st); break;
    case 2: matmul_mma_nb<2>(Zall, m, p, blk_stride, slot_of, blk_of_slot, nitems, W_all, out_all, st); break;
    case 3: matmul_mma_nb<3>(Zall, m, p, blk_stride, slot_of, blk_of_slot, nitems, W_all, out_all, st); break;
    case 4: matmul_mma_nb<4>(Zall, m, p, blk_stride, slot_of, blk_of_slot, nitems, W_all, out_all, st); break;
    case 5: matmul_mma_nb<5>(Zall, m, p, blk_stride, slot_of, blk_of_slot, nitems, W_all, out_all, st); break;
    default: throw std::string("matmul_mma: p out of range");
  }
  RTD_LAUNCHED();
}

}  // namespace rtd
