// H6, the C-step distance pass (§3.4), TMA-fed: d_i^2 = ||M (z_i - mu)||^2 with
// M = L^-1 (lower triangular, Sigma = L L^T) on the FP64 tensor pipe (DMMA m8n8k4), for one or TWO
// starts of the same block per CTA (the two initial estimators' C-steps of a block read the same rows:
// the tile is loaded once and contracted with both operators).
//
// Data movement (B200-native): a producer warp streams tiles of TR rows x P columns of the block's
// column-major Z into a ring of NS shared-memory stages with cp.async.bulk.tensor (TMA, 3-D tensor
// map over [blocks][columns][rows]); completion is signalled on a per-stage mbarrier (complete_tx),
// the 8 consumer warps release a stage through a second mbarrier.  No per-thread address arithmetic,
// no register staging, loads of the next NS-1 tiles always in flight.  TR = 8 G rows with G odd, so a
// column of the tile is 8 mod 16 doubles long and the A-fragment reads (8 consecutive rows x 4 columns
// per warp) fill exactly two shared-memory wavefronts.
//
// Default variant (V = 2, RTD_DIST_TMA_VARIANT): G = 23 row groups per tile (TR = 184), consumer warp w
// takes groups w, w + 8, w + 16; the two starts of a pair are contracted TOGETHER from the same raw A
// fragments (one shared-memory read feeds both operators' DMMAs) and the centring enters the
// accumulators, y = M z - M mu (the same arithmetic object as M (z - mu); no per-element subtraction):
// 2 x 3 x NB independent accumulator chains per warp.  Measured on config 4 (p = 40, 13 passes per
// fit): 9.5 ms per fit against 10.4 ms for V = 0 (one start at a time, centred A) and 10.3 ms for the
// register-fed k_dist_mma.  Blocks of M^T entirely above the diagonal are skipped (20 of 50 8x4 blocks
// at p = 40: 30 executed).  Epilogue: d^2 = sum of squares of the accumulators (two shuffles).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "rtd_internal.h"
#include "tma.cuh"

namespace rtd {

using namespace tma;

namespace {

__device__ __forceinline__ void dmma_t(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// V = 0: tiles of G = 31 row groups (TR = 248 rows) for 8 consumer warps taking groups w, w+8, w+16, w+24
//        (MB = 4), one CTA per SM;  V = 1: G = 15 (TR = 120), MB = 2, two CTAs per SM.
template <int P, int V>
struct DistTmaCfg {
  static constexpr int NCW = 8;                              // consumer warps (+ 1 producer warp)
  static constexpr int G = V == 1 ? 15 : (V == 2 ? (P <= 24 ? 15 : 23) : 31);  // 8-row groups per tile (odd: TR = 8 mod 16)
  static constexpr bool JOINT = V == 2;                      // both starts of a pair in one register pass
  static constexpr int MB = (G + NCW - 1) / NCW;             // groups per consumer warp
  static constexpr int MINB = (V == 1 || (V == 2 && P <= 24)) ? 2 : 1;  // CTAs per SM
  // V = 2: G = 23 (TR = 184), MB = 3, one CTA per SM, and the two starts of a pair contracted together from the same raw A fragments: the
  //        centring enters the accumulators (y = M z - M mu, the same arithmetic object)
  static constexpr int TR = 8 * G;
  static constexpr int KB = (P + 3) / 4, NB = (P + 7) / 8;
  static constexpr int TILE = TR * P;                        // doubles per stage (the TMA box)
  static constexpr int STG = (TILE + 15) / 16 * 16;          // stage stride: 128-byte aligned TMA destinations
  static constexpr int OPD = KB * NB * 32 + KB * 4 + NB * 8; // operator fragments + mu + (-M mu) per start
  static constexpr int BUDGET = 220 * 1024 / MINB - 2 * OPD * 8 - 256;
  static constexpr int NS = std::max(2, std::min(8, BUDGET / (STG * 8)));
  static constexpr size_t SMEM = (size_t)NS * STG * 8 + 2 * (size_t)OPD * 8 + 2 * NS * 8 + 128;
};

}  // namespace

// grid (ctas_per_item, nitems); item y = slots pairs[2y], pairs[2y+1] (-1: a lone start)
template <int P, int V>
__global__ void __launch_bounds__((DistTmaCfg<P, V>::NCW + 1) * 32, DistTmaCfg<P, V>::MINB)
    k_dist_tma(const __grid_constant__ CUtensorMap zmap, long long m, const int* __restrict__ pairs,
               const int* __restrict__ inst, int nstart, const double* __restrict__ cstage, int cstride,
               double* __restrict__ d2_all, int tiles_per_cta) {
  using C = DistTmaCfg<P, V>;
  constexpr int MB = C::MB, NCW = C::NCW, G = C::G, TR = C::TR, KB = C::KB, NB = C::NB, NS = C::NS,
                TILE = C::TILE, STG = C::STG;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* tiles = reinterpret_cast<double*>(smraw);
  double* ops = tiles + (size_t)NS * STG;  // [2][OPD]: B fragments then mu
  uint64_t* full = reinterpret_cast<uint64_t*>(ops + 2 * C::OPD);
  uint64_t* empty = full + NS;

  const int s0 = pairs[2 * blockIdx.y], s1 = pairs[2 * blockIdx.y + 1];
  const bool two = s1 >= 0;
  const int id0 = inst[s0], id1 = two ? inst[s1] : id0;
  const int blk = id0 / nstart;
  const long long ntiles = (m + TR - 1) / TR;
  const long long t_begin = (long long)blockIdx.x * tiles_per_cta;
  const long long t_end = std::min<long long>(ntiles, t_begin + tiles_per_cta);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // operators of the start(s): B[k][j] = M[j][k] lane-major per 8x4 block, mu padded to 4 KB
  for (int w = 0; w < (two ? 2 : 1); w++) {
    const double* cs = cstage + (long long)(w ? s1 : s0) * cstride;
    double* bsm = ops + w * C::OPD;
    for (int e = threadIdx.x; e < KB * NB * 32; e += blockDim.x) {
      const int ln = e & 31, b = e >> 5, kb = b / NB, nb = b - kb * NB;
      const int k = 4 * kb + (ln & 3), j = 8 * nb + (ln >> 2);
      bsm[e] = (j < P && k <= j) ? cs[P + j * (j + 1) / 2 + k] : 0.0;
    }
    for (int e = threadIdx.x; e < KB * 4; e += blockDim.x) bsm[KB * NB * 32 + e] = e < P ? cs[e] : 0.0;
    if (C::JOINT)
      for (int j = threadIdx.x; j < NB * 8; j += blockDim.x) {  // c_j = -(M mu)_j, fixed order
        double c = 0.0;
        if (j < P)
          for (int k = 0; k <= j; k++) c = fma(cs[P + j * (j + 1) / 2 + k], cs[k], c);
        bsm[KB * NB * 32 + KB * 4 + j] = -c;
      }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (t_begin >= t_end) return;

  if (warp == NCW) {  // producer: one lane issues the TMA loads of this CTA's tiles into the ring
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&zmap)) : "memory");
      for (long long it = 0; it < t_end - t_begin; it++) {
        const int s = (int)(it % NS);
        mbar_wait(&empty[s], (uint32_t)(((it / NS) & 1) ^ 1));
        mbar_expect_tx(&full[s], (uint32_t)(TILE * 8));
        tma_load_3d(tiles + (size_t)s * STG, &zmap, &full[s], (int)((t_begin + it) * TR), 0, blk);
      }
    }
    return;
  }

  // consumers: warp w contracts row groups w, w + 8, ... of every tile
  const int g = lane >> 2, t = lane & 3;
  double* d2a = d2_all + (long long)id0 * m;
  double* d2b = d2_all + (long long)id1 * m;
  for (long long it = 0; it < t_end - t_begin; it++) {
    const int s = (int)(it % NS);
    mbar_wait(&full[s], (uint32_t)((it / NS) & 1));
    const double* T = tiles + (size_t)s * STG;
    const long long tr0 = (t_begin + it) * TR;
    if (C::JOINT && two) {
      const double* b0 = ops;
      const double* b1 = ops + C::OPD;
      double acc[2][MB][NB][2];
#pragma unroll
      for (int nb = 0; nb < NB; nb++) {
        const double c00 = b0[KB * NB * 32 + KB * 4 + 8 * nb + 2 * t], c01 = b0[KB * NB * 32 + KB * 4 + 8 * nb + 2 * t + 1];
        const double c10 = b1[KB * NB * 32 + KB * 4 + 8 * nb + 2 * t], c11 = b1[KB * NB * 32 + KB * 4 + 8 * nb + 2 * t + 1];
#pragma unroll
        for (int mb = 0; mb < MB; mb++) {
          acc[0][mb][nb][0] = c00;
          acc[0][mb][nb][1] = c01;
          acc[1][mb][nb][0] = c10;
          acc[1][mb][nb][1] = c11;
        }
      }
#pragma unroll
      for (int kb = 0; kb < KB; kb++) {
        const int k = 4 * kb + t;
        double a[MB];
#pragma unroll
        for (int mb = 0; mb < MB; mb++) {
          const int grp = warp + NCW * mb;
          a[mb] = (k < P && grp < G) ? T[k * TR + grp * 8 + g] : 0.0;
        }
#pragma unroll
        for (int nb = 0; nb < NB; nb++) {
          if (8 * nb + 7 < 4 * kb) continue;
          const double bv0 = b0[(kb * NB + nb) * 32 + lane], bv1 = b1[(kb * NB + nb) * 32 + lane];
#pragma unroll
          for (int mb = 0; mb < MB; mb++)
            if (MB * NCW == G || warp + NCW * mb < G) {
              dmma_t(acc[0][mb][nb][0], acc[0][mb][nb][1], a[mb], bv0);
              dmma_t(acc[1][mb][nb][0], acc[1][mb][nb][1], a[mb], bv1);
            }
        }
      }
#pragma unroll
      for (int w = 0; w < 2; w++) {
        double* d2 = w ? d2b : d2a;
#pragma unroll
        for (int mb = 0; mb < MB; mb++) {
          double v = 0.0;
#pragma unroll
          for (int nb = 0; nb < NB; nb++) {
            v = fma(acc[w][mb][nb][0], acc[w][mb][nb][0], v);
            v = fma(acc[w][mb][nb][1], acc[w][mb][nb][1], v);
          }
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          const int grp = warp + NCW * mb;
          const long long row = tr0 + grp * 8 + g;
          if (t == 0 && grp < G && row < m) d2[row] = v;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      continue;
    }
    for (int w = 0; w < (two ? 2 : 1); w++) {
      const double* bsm = ops + w * C::OPD;
      const double* musm = bsm + KB * NB * 32;
      double acc[MB][NB][2];
#pragma unroll
      for (int mb = 0; mb < MB; mb++)
#pragma unroll
        for (int nb = 0; nb < NB; nb++) acc[mb][nb][0] = acc[mb][nb][1] = 0.0;
#pragma unroll
      for (int kb = 0; kb < KB; kb++) {
        const int k = 4 * kb + t;
        const double muk = musm[k];
        double a[MB];
#pragma unroll
        for (int mb = 0; mb < MB; mb++) {
          const int grp = warp + NCW * mb;
          a[mb] = (k < P && grp < G) ? __dsub_rn(T[k * TR + grp * 8 + g], muk) : 0.0;
        }
#pragma unroll
        for (int nb = 0; nb < NB; nb++) {
          if (8 * nb + 7 < 4 * kb) continue;  // block entirely above the diagonal of M
          const double bv = bsm[(kb * NB + nb) * 32 + lane];
#pragma unroll
          for (int mb = 0; mb < MB; mb++)
            if (MB * NCW == G || warp + NCW * mb < G) dmma_t(acc[mb][nb][0], acc[mb][nb][1], a[mb], bv);
        }
      }
      double* d2 = w ? d2b : d2a;
#pragma unroll
      for (int mb = 0; mb < MB; mb++) {
        double v = 0.0;
#pragma unroll
        for (int nb = 0; nb < NB; nb++) {
          v = fma(acc[mb][nb][0], acc[mb][nb][0], v);
          v = fma(acc[mb][nb][1], acc[mb][nb][1], v);
        }
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        const int grp = warp + NCW * mb;
        const long long row = tr0 + grp * 8 + g;
        if (t == 0 && grp < G && row < m) d2[row] = v;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// ------------------------------------------------------------------ refinement GEMMs, TMA-fed
// out = Z W for the two starts of a block at once (the scores T = Z V and the
// sphered data Z~ = Z Sigma^-1/2 of the refinement): tiles of G = 23 row groups of 8 (TR = 184 rows) in a
// 3-stage ring loaded by TMA, every one of the 8 warps contracting its groups (w, w + 8, w + 16) -- lane 0
// of warp 0 also issues the loads, so the CTA has 8 warps and 255 registers per thread (a separate
// producer warp would make one SM sub-partition hold 3 warps: 168 registers, spills) -- each raw A
// fragment of Z feeding the DMMAs of both W (full p x p operators, B fragments in shared memory), the
// accumulators stored straight to the column-major outputs.  grid (ctas_per_item, nitems); item y =
// work items pairs[2y], pairs[2y+1] (-1: a lone item).
template <int P>
struct MatTmaCfg {
  static constexpr int NW = 8, G = 23, MB = 3, TR = 8 * G;
  static constexpr int KB = (P + 3) / 4, NB = (P + 7) / 8;
  static constexpr int TILE = TR * P, STG = (TILE + 15) / 16 * 16;
  static constexpr int OPW = KB * NB * 32;
  static constexpr int NS = std::max(3, std::min(8, (200 * 1024 - 2 * OPW * 8) / (STG * 8)));
  static constexpr size_t SMEM = (size_t)NS * STG * 8 + 2 * (size_t)OPW * 8 + 2 * NS * 8 + 128;
};

template <int P>
__global__ void __launch_bounds__(MatTmaCfg<P>::NW * 32, 1)
    k_matmul_tma(const __grid_constant__ CUtensorMap zmap, long long m, const int* __restrict__ pairs,
                 const int* __restrict__ slot_of, const int* __restrict__ blk_of_slot, const double* __restrict__ W_all,
                 double* __restrict__ out_all, int tiles_per_cta) {
  using C = MatTmaCfg<P>;
  constexpr int MB = C::MB, NW = C::NW, G = C::G, TR = C::TR, KB = C::KB, NB = C::NB, NS = C::NS,
                TILE = C::TILE, STG = C::STG, OPW = C::OPW;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* tiles = reinterpret_cast<double*>(smraw);
  double* ops = tiles + (size_t)NS * STG;  // [2][OPW]
  uint64_t* full = reinterpret_cast<uint64_t*>(ops + 2 * OPW);
  uint64_t* empty = full + NS;
  const int i0 = pairs[2 * blockIdx.y], i1 = pairs[2 * blockIdx.y + 1];
  const bool two = i1 >= 0;
  const int s0 = slot_of[i0], s1 = two ? slot_of[i1] : s0;
  const int blk = blk_of_slot[s0];
  const long long ntiles = (m + TR - 1) / TR;
  const long long t_begin = (long long)blockIdx.x * tiles_per_cta;
  const long long t_end = min(ntiles, t_begin + tiles_per_cta);
  const int nt = (int)max(0LL, t_end - t_begin);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int w = 0; w < 2; w++) {  // B[k][j] = W[k][j] lane-major per 8x4 block (a lone item: W twice)
    const double* W = W_all + (long long)(w ? s1 : s0) * RTD_MAXP * RTD_MAXP;
    for (int e = threadIdx.x; e < OPW; e += blockDim.x) {
      const int ln = e & 31, b = e >> 5, kb = b / NB, nb = b - kb * NB;
      const int k = 4 * kb + (ln & 3), j = 8 * nb + (ln >> 2);
      ops[w * OPW + e] = (k < P && j < P) ? W[k * P + j] : 0.0;
    }
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < NS; q++) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int j) {  // tile j into stage j % NS once every warp released its previous use
    if (j >= nt) return;
    const int q = j % NS;
    mbar_wait(&empty[q], (uint32_t)(((j / NS) & 1) ^ 1));
    mbar_expect_tx(&full[q], (uint32_t)(TILE * 8));
    tma_load_3d(tiles + (size_t)q * STG, &zmap, &full[q], (int)((t_begin + j) * TR), 0, blk);
  };
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&zmap)) : "memory");
    for (int j = 0; j < NS - 1; j++) issue(j);
  }
  const int g = lane >> 2, t = lane & 3;
  double* __restrict__ out0 = out_all + (long long)i0 * P * m;
  double* __restrict__ out1 = out_all + (long long)(two ? i1 : i0) * P * m;
  for (int it = 0; it < nt; it++) {
    const int q = it % NS;
    if (threadIdx.x == 0 && it >= 1) issue(it + NS - 2);  // the stage of tile it - 2
    mbar_wait(&full[q], (uint32_t)((it / NS) & 1));
    const double* T = tiles + (size_t)q * STG;
    const long long tr0 = (t_begin + it) * TR;
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
      double a[MB];
#pragma unroll
      for (int mb = 0; mb < MB; mb++) {
        const int grp = warp + NW * mb;
        a[mb] = (k < P && grp < G) ? T[k * TR + grp * 8 + g] : 0.0;
      }
#pragma unroll
      for (int nb = 0; nb < NB; nb++) {
        const double bv0 = ops[(kb * NB + nb) * 32 + lane], bv1 = ops[OPW + (kb * NB + nb) * 32 + lane];
#pragma unroll
        for (int mb = 0; mb < MB; mb++)
          if (MB * NW == G || warp + NW * mb < G) {
            dmma_t(acc[0][mb][nb][0], acc[0][mb][nb][1], a[mb], bv0);
            dmma_t(acc[1][mb][nb][0], acc[1][mb][nb][1], a[mb], bv1);  // a lone item: a discarded copy
          }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[q]);  // the tile is no longer read
#pragma unroll
    for (int w = 0; w < 2; w++) {
      double* __restrict__ out = w ? out1 : out0;
#pragma unroll
      for (int mb = 0; mb < MB; mb++) {
        const int grp = warp + NW * mb;
        const long long row = tr0 + grp * 8 + g;
        if (grp >= G || row >= m || (w == 1 && !two)) continue;
#pragma unroll
        for (int nb = 0; nb < NB; nb++) {
          const int j = 8 * nb + 2 * t;
          if (j < P) out[(long long)j * m + row] = acc[w][mb][nb][0];
          if (j + 1 < P) out[(long long)(j + 1) * m + row] = acc[w][mb][nb][1];
        }
      }
    }
  }
}

namespace {

template <int P>
void matmul_tma_launch(const double* Zall, long long m, int nblk, const int* slot_of, const int* blk_of_slot,
                       const int* pairs, int npairs, const double* W_all, double* out_all, cudaStream_t st) {
  using C = MatTmaCfg<P>;
  CUtensorMap map;
  if (!encode_blocks(&map, Zall, m, P, nblk, C::TR)) throw std::string("cuTensorMapEncodeTiled failed for the GEMM");
  const long long ntiles = (m + C::TR - 1) / C::TR;
  const long long per_item = std::max<long long>(1, 148LL / npairs);
  const int tpc = (int)std::max<long long>(1, (ntiles + per_item - 1) / per_item);
  const unsigned gx = (unsigned)((ntiles + tpc - 1) / tpc);
  set_max_dyn_smem(reinterpret_cast<const void*>(k_matmul_tma<P>), (int)C::SMEM);
  k_matmul_tma<P><<<dim3(gx, npairs), C::NW * 32, C::SMEM, st>>>(map, m, pairs, slot_of, blk_of_slot, W_all, out_all,
                                                                  tpc);
}

}  // namespace

void launch_matmul_tma(int p, const double* Zall, long long m, int nblk, const int* slot_of, const int* blk_of_slot,
                       const int* pairs, int npairs, const double* W_all, double* out_all, cudaStream_t st) {
  switch (p) {
#define RTD_MT_CASE(P) \
  case P: matmul_tma_launch<P>(Zall, m, nblk, slot_of, blk_of_slot, pairs, npairs, W_all, out_all, st); break;
    RTD_MT_CASE(8) RTD_MT_CASE(9) RTD_MT_CASE(10) RTD_MT_CASE(11) RTD_MT_CASE(12) RTD_MT_CASE(13)
    RTD_MT_CASE(14) RTD_MT_CASE(15) RTD_MT_CASE(16) RTD_MT_CASE(17) RTD_MT_CASE(18) RTD_MT_CASE(19)
    RTD_MT_CASE(20) RTD_MT_CASE(21) RTD_MT_CASE(22) RTD_MT_CASE(23) RTD_MT_CASE(24) RTD_MT_CASE(25)
    RTD_MT_CASE(26) RTD_MT_CASE(27) RTD_MT_CASE(28) RTD_MT_CASE(29) RTD_MT_CASE(30) RTD_MT_CASE(31)
    RTD_MT_CASE(32) RTD_MT_CASE(33) RTD_MT_CASE(34) RTD_MT_CASE(35) RTD_MT_CASE(36) RTD_MT_CASE(37)
    RTD_MT_CASE(38) RTD_MT_CASE(39) RTD_MT_CASE(40)
#undef RTD_MT_CASE
    default: throw std::string("matmul_tma: p out of range");
  }
  RTD_LAUNCHED();
}

namespace {

template <int P, int V>
void dist_tma_launch_v(const CUtensorMap& map, long long m, const int* pairs, int npairs, const int* inst, int nstart,
                       const double* cstage, int cstride, double* d2_all, cudaStream_t st) {
  using C = DistTmaCfg<P, V>;
  const long long ntiles = (m + C::TR - 1) / C::TR;
  // C::MINB CTAs per SM; the items share one wave of 148 * MINB CTAs (floor: no straggler wave), the CTAs of
  // an item split its tiles evenly
  const long long per_item = std::max<long long>(1, 148LL * C::MINB / npairs);
  const int tpc = (int)std::max<long long>(1, (ntiles + per_item - 1) / per_item);
  const unsigned gx = (unsigned)((ntiles + tpc - 1) / tpc);
  set_max_dyn_smem(reinterpret_cast<const void*>(k_dist_tma<P, V>), (int)C::SMEM);
  k_dist_tma<P, V><<<dim3(gx, npairs), (C::NCW + 1) * 32, C::SMEM, st>>>(map, m, pairs, inst, nstart, cstage, cstride,
                                                                         d2_all, tpc);
}

template <int P>
void dist_tma_launch(const double* Zall, long long m, int nblk, const int* pairs, int npairs, const int* inst,
                     int nstart, const double* cstage, int cstride, double* d2_all, cudaStream_t st) {
  static const int variant = getenv("RTD_DIST_TMA_VARIANT") ? atoi(getenv("RTD_DIST_TMA_VARIANT")) : 2;
  const int tr = variant == 1 ? DistTmaCfg<P, 1>::TR : (variant == 2 ? DistTmaCfg<P, 2>::TR : DistTmaCfg<P, 0>::TR);
  CUtensorMap map;
  if (!encode_blocks(&map, Zall, m, P, nblk, tr)) throw std::string("cuTensorMapEncodeTiled failed for the distance pass");
  if (variant == 0) dist_tma_launch_v<P, 0>(map, m, pairs, npairs, inst, nstart, cstage, cstride, d2_all, st);
  else if (variant == 1) dist_tma_launch_v<P, 1>(map, m, pairs, npairs, inst, nstart, cstage, cstride, d2_all, st);
  else dist_tma_launch_v<P, 2>(map, m, pairs, npairs, inst, nstart, cstage, cstride, d2_all, st);
}

}  // namespace

bool dist_tma_supported(int p, long long m) {
  static const bool off = getenv("RTD_DIST_NOTMA") != nullptr;
  return !off && p >= 8 && p <= RTD_MAXP && m % 2 == 0 && m >= 8192 && encode_fn() != nullptr;
}

void launch_dist_tma(int p, const double* Zall, long long m, int nblk, const int* pairs, int npairs, const int* inst,
                     int nstart, const double* cstage, int cstride, double* d2_all, cudaStream_t st) {
  switch (p) {
#define RTD_TMA_CASE(P) \
  case P: dist_tma_launch<P>(Zall, m, nblk, pairs, npairs, inst, nstart, cstage, cstride, d2_all, st); break;
    RTD_TMA_CASE(8) RTD_TMA_CASE(9) RTD_TMA_CASE(10) RTD_TMA_CASE(11) RTD_TMA_CASE(12) RTD_TMA_CASE(13)
    RTD_TMA_CASE(14) RTD_TMA_CASE(15) RTD_TMA_CASE(16) RTD_TMA_CASE(17) RTD_TMA_CASE(18) RTD_TMA_CASE(19)
    RTD_TMA_CASE(20) RTD_TMA_CASE(21) RTD_TMA_CASE(22) RTD_TMA_CASE(23) RTD_TMA_CASE(24) RTD_TMA_CASE(25)
    RTD_TMA_CASE(26) RTD_TMA_CASE(27) RTD_TMA_CASE(28) RTD_TMA_CASE(29) RTD_TMA_CASE(30) RTD_TMA_CASE(31)
    RTD_TMA_CASE(32) RTD_TMA_CASE(33) RTD_TMA_CASE(34) RTD_TMA_CASE(35) RTD_TMA_CASE(36) RTD_TMA_CASE(37)
    RTD_TMA_CASE(38) RTD_TMA_CASE(39) RTD_TMA_CASE(40)
#undef RTD_TMA_CASE
    default: throw std::string("dist_tma: p out of range");
  }
  RTD_LAUNCHED();
}

}  // namespace rtd
