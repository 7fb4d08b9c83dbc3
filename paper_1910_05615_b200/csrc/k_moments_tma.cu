// Dense moment passes fed by TMA: S2 = sum_r w_r u_r u_r^T (lower 8x8 blocks), S1 = sum_r w_r u_r,
// count = sum_r w_r over a block's rows, for the dense modes of k_moments.cu:
//   MOM_WRAP     u = psi(z) (the wrapping function of PAPER.md:467-503, S~1), w = 1; also writes the
//                row norms ||z_i|| of S~2 from the same tile;
//   MOM_XI       u = z, w = xi(||z_i||)^2 (LR-GSSCM weights, S~2);
//   MOM_MEMBER   u = z - c, w = [i in H] (C-step moments);
//   MOM_REWEIGHT u = z - c, w = [d_i^2 <= chi2] (reweighting);
//   MOM_WRAPXI   MOM_WRAP (warps [0, split), into partial) and MOM_XI (the other warps, into partial2) on
//                the same tiles: S~1 and S~2 from one read of Z once the norms and cutoffs are known.
//
// Lane 0 of warp 0 streams TR-row tiles of the block's column-major Z through an NS-stage
// shared-memory ring with cp.async.bulk.tensor (3-D tensor map [blocks][columns][rows]) and
// per-stage full / empty mbarriers; 8 consumer warps contract 4-row groups on DMMA m8n8k4: lane
// (g, t) holds u[row t][column 8b + g] of every column block b and feeds it as the A operand (times
// w) of block row b and as the B operand of block column b (one shared-memory read serves (NB+1)/2
// DMMAs).  TR = 100 = 4 (mod 16) doubles: the 8 columns a warp reads at once start 32 bytes apart in
// the bank space, so a fragment read fills exactly two wavefronts.  The groups of the CTA's rows are
// dealt to the warps round-robin ACROSS tiles (group q -> warp q mod 8), so no warp idles at a tile
// boundary although a tile holds an odd number (25) of groups.  Rows of a CTA: a contiguous range;
// partials are reduced in a fixed order (deterministic), as in k_moments_mma.cu.
#include <algorithm>
#include <cstdlib>

#include "rtd_internal.h"
#include "tanh_table.h"
#include "tma.cuh"

namespace rtd {

using namespace tma;

namespace {

__device__ __forceinline__ void dmma_m(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double psi_wrap(double z) {  // PAPER.md:478-486, constants verbatim (reading Q5)
  const double b = 1.5, c = 4.0, q1 = 1.541, q2 = 0.862;
  const double az = fabs(z);
  if (az <= b) return z;
  if (az <= c) {
    const double t = __dmul_rn(q1, tanh(__dmul_rn(q2, __dsub_rn(c, az))));
    return z > 0 ? t : (z < 0 ? -t : 0.0);
  }
  return 0.0;
}

// tanh on [0, 2.19) from the shared-memory copy of tools/gen_tanh_table.py's table: degree-10 Taylor
// polynomial about c_j = j W (j = rint(x / W)), Estrin's scheme (five dependent FMA levels instead of
// the library tanh's exp + Newton division chain, which left the wrap warps stalled on fixed-latency
// dependencies); <= 2 ulp (the generator's check), the library tanh 1 ulp (reading R28)
__device__ __forceinline__ double tanh_tab(double x, const double* __restrict__ tab) {
  const int j = min(__double2int_rn(__dmul_rn(x, 1.0 / RTD_TANH_W)), RTD_TANH_NI - 1);
  const double v = __dsub_rn(x, __dmul_rn((double)j, RTD_TANH_W));
  const double* a = tab + j * RTD_TANH_NC;
  const double v2 = __dmul_rn(v, v), v4 = __dmul_rn(v2, v2), v8 = __dmul_rn(v4, v4);
  const double p01 = fma(a[1], v, a[0]), p23 = fma(a[3], v, a[2]), p45 = fma(a[5], v, a[4]),
               p67 = fma(a[7], v, a[6]), p89 = fma(a[9], v, a[8]);
  const double q0 = fma(p23, v2, p01), q1 = fma(p67, v2, p45), q2 = fma(a[10], v2, p89);
  return fma(q2, v8, fma(q1, v4, q0));
}

__device__ __forceinline__ void consumer_sync() { __syncthreads(); }

// W = 8: two CTAs of 8 warps per SM, a 96 KB ring each; W = 16: one CTA of 16 warps per SM, a 192 KB ring
// (the producer runs twice as far ahead of the slowest warp)
template <int P, int W = 8>
struct MomTmaCfg {
  static constexpr int NCW = W;                  // warps (lane 0 of warp 0 also issues the TMA loads)
  static constexpr int CPS = 16 / W;             // CTAs per SM
  static constexpr int TR = 100;                 // rows per tile: 4 (mod 16) doubles, 25 groups of 4 rows
  static constexpr int G = TR / 4;
  static constexpr int TILE = TR * P;
  static constexpr int STG = (TILE + 15) / 16 * 16;
  static constexpr int NS = std::max(3, std::min(8, (96 * 1024 * (W / 8)) / (STG * 8)));
  static constexpr int NP = P + P * (P + 1) / 2 + 1;
  static constexpr size_t RING = (size_t)NS * STG * 8;
  static constexpr size_t RED = (size_t)NCW * NP * 8;  // epilogue: per-warp sums (reuses the ring)
  static constexpr size_t SCR = (size_t)NCW * 5 * 32 * 8;  // MOM_WRAP: warp-private tanh lists
  static constexpr int WST = 1024;                           // per-stage bytes of the row weights' source
  static constexpr size_t OFF_W = (std::max(RING, RED) + 127) / 128 * 128;  // weight stages (TMA destinations)
  static constexpr size_t OFF_B = OFF_W + (size_t)NS * WST;                  // full / empty barriers
  static constexpr size_t OFF_S = OFF_B + 2 * NS * 8 + 64;                    // tanh scratch
  static constexpr size_t OFF_T = OFF_S + SCR;                               // tanh table (wrap modes)
  static constexpr size_t SMEM = OFF_T + RTD_TANH_NI * RTD_TANH_NC * 8;
};

}  // namespace

template <int P, int MODE, int W>
__global__ void __launch_bounds__(W * 32, 16 / W)
    k_moments_tma(const __grid_constant__ CUtensorMap zmap, const __grid_constant__ CUtensorMap wmap, MomArgs a) {
  using C = MomTmaCfg<P, W>;
  constexpr int NB = (P + 7) / 8, NBLK = NB * (NB + 1) / 2, NCW = C::NCW, TR = C::TR, G = C::G, NS = C::NS,
                STG = C::STG, NP = C::NP;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* tiles = reinterpret_cast<double*>(smraw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + C::OFF_B);
  uint64_t* empty = full + NS;
  double* scratch = reinterpret_cast<double*>(smraw + C::OFF_S);
  // per-stage copy of the rows' weight source (norms r / distances d2 / membership bytes), loaded by TMA
  // with the tile on the same barrier
  unsigned char* wsrc = smraw + C::OFF_W;
  double* ttab = reinterpret_cast<double*>(smraw + C::OFF_T);
  constexpr bool FX = MODE == MOM_WRAPXI;
  constexpr bool WT = MODE == MOM_XI || MODE == MOM_REWEIGHT || FX;
  constexpr uint32_t WBYTES = WT ? TR * 8 : 0;
  const int slot = blockIdx.y;
  const int id = a.inst[slot];
  const int blk = id / a.nstart;
  const long long m = a.m;
  long long per = (m + a.ctas - 1) / a.ctas;
  per = (per + 3) / 4 * 4;
  const long long r_begin = (long long)blockIdx.x * per, r_end = std::min(m, r_begin + per);
  const int ntile = r_end > r_begin ? (int)((r_end - r_begin + TR - 1) / TR) : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (MODE == MOM_WRAP || FX)
    for (int i = threadIdx.x; i < RTD_TANH_NI * RTD_TANH_NC; i += W * 32) ttab[i] = rtd_tanh_coef[i];
  __syncthreads();
  // producer = lane 0 of warp 0, opportunistic: the first NS - 1 tiles now; then, between its groups, tile
  // nxt as soon as the stage's previous tile has been released by every warp (a non-blocking test, at most
  // NS - 1 tiles ahead of its own, so the parity test cannot alias an older phase); it blocks only on
  // entering a tile not yet issued
  auto issue = [&](int j) {
    const int s = j % NS;
    mbar_wait(&empty[s], (uint32_t)(((j / NS) & 1) ^ 1));
    mbar_expect_tx(&full[s], (uint32_t)(C::TILE * 8) + WBYTES);
    tma_load_3d(tiles + (size_t)s * STG, &zmap, &full[s], (int)(r_begin + (long long)j * TR), 0, blk);
    if (WT) tma_load_2d(wsrc + s * C::WST, &wmap, &full[s], (int)(r_begin + (long long)j * TR), MODE == MOM_REWEIGHT ? id : blk);
  };
  int nxt = 0;  // tiles issued so far (lane 0 of warp 0)
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&zmap)) : "memory");
    if (WT) asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
    for (; nxt < NS - 1 && nxt < ntile; nxt++) issue(nxt);
  }
  const int g = lane >> 2, t = lane & 3;
  double sh[NB];
#pragma unroll
  for (int b = 0; b < NB; b++)
    sh[b] = ((MODE == MOM_MEMBER || MODE == MOM_REWEIGHT) && 8 * b + g < P) ? a.shift[(long long)id * RTD_MAXP + 8 * b + g]
                                                                             : 0.0;
  double A = 0.0, B = 0.0, invBA = 0.0;
  if (MODE == MOM_XI || FX) {
    A = a.AB[2 * blk];
    B = a.AB[2 * blk + 1];
    invBA = B > A ? 1.0 / (B - A) : 0.0;  // (B - r) / (B - A) as a product: no division per row (reading R28)
  }
  double acc[NBLK][2];
#pragma unroll
  for (int k = 0; k < NBLK; k++) acc[k][0] = acc[k][1] = 0.0;
  double s1[NB];
#pragma unroll
  for (int b = 0; b < NB; b++) s1[b] = 0.0;
  double cnt = 0.0;
  // roles (MOM_WRAPXI): warps [0, split) take the wrapped moments, the others the xi-weighted ones; each
  // role deals the CTA's ntile * G groups round-robin across tiles: group l of tile k, then l + NWR
  // (carried into the next tile), so no warp idles at a tile boundary although a tile holds an odd
  // number (25) of groups
  const int split = a.split * (W / 8);  // a.split counts eighths of the CTA's warps
  const bool wrap_role = MODE == MOM_WRAP || (FX && warp < split);
  const int NWR = FX ? (wrap_role ? split : NCW - split) : NCW;
  const int wr = FX ? (wrap_role ? warp : warp - split) : warp;
  double* scr = scratch + warp * (5 * 32);  // wrapped moments: per-warp list of tanh-branch arguments
  int cur = -1;  // tile whose full barrier this warp has passed
  // MOM_MEMBER: the membership byte of the warp's next group is loaded one group ahead (an L2 round trip
  // per group otherwise stalls the warp before every group)
  unsigned int mb_next = 0u;
  if (MODE == MOM_MEMBER && wr < G && r_begin + 4 * wr + t < r_end)
    mb_next = a.mem_new[(long long)id * m + r_begin + 4 * wr + t];
  for (int k = 0, l = wr; k < ntile; l = (l + NWR >= G) ? (k++, l + NWR - G) : l + NWR) {
    while (cur < k) {  // release the tile left behind, enter the next one
      if (cur >= 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[cur % NS]);
      }
      cur++;
      if (warp == 0 && lane == 0)
        for (; nxt <= cur && nxt < ntile; nxt++) issue(nxt);  // blocking only for the tile entered now
      mbar_wait(&full[cur % NS], (uint32_t)((cur / NS) & 1));
    }
    if (warp == 0 && lane == 0 && nxt < ntile && nxt <= cur + NS - 1 &&
        mbar_test(&empty[nxt % NS], (uint32_t)(((nxt / NS) & 1) ^ 1))) {
      issue(nxt);  // released: does not block
      nxt++;
    }
    const long long row = r_begin + (long long)k * TR + 4 * l + t;
    unsigned int mb = 0u;
    if (MODE == MOM_MEMBER) {
      mb = mb_next;
      const int l2 = l + NWR >= G ? l + NWR - G : l + NWR, k2 = l + NWR >= G ? k + 1 : k;
      const long long row2 = r_begin + (long long)k2 * TR + 4 * l2 + t;
      mb_next = (k2 < ntile && row2 < r_end) ? a.mem_new[(long long)id * m + row2] : 0u;
    }
    double w = 0.0;
    if (row < r_end) {
      const unsigned char* ws = wsrc + (k % NS) * C::WST;
      if (wrap_role) {
        w = 1.0;
      } else if (MODE == MOM_XI || FX) {
        const double rr = reinterpret_cast<const double*>(ws)[4 * l + t];
        const double xi = rr <= A ? 1.0 : (rr <= B ? __dmul_rn(__dsub_rn(B, rr), invBA) : 0.0);
        w = __dmul_rn(xi, xi);
      } else if (MODE == MOM_MEMBER) {  // membership bytes from global memory (a UINT8 2-D TMA map of them
        // faulted with an illegal instruction on this stack; the bytes are L2-resident)
        w = (double)mb;
      } else {
        w = reinterpret_cast<const double*>(ws)[4 * l + t] <= a.c2 ? 1.0 : 0.0;
      }
    }
    if (!wrap_role && !__any_sync(0xffffffffu, w != 0.0)) continue;  // wrap_role is warp-uniform
    const double* T = tiles + (size_t)(k % NS) * STG;
    double u[NB];
#pragma unroll
    for (int b = 0; b < NB; b++) {
      const int col = 8 * b + g;
      u[b] = (col < P && w != 0.0) ? T[col * TR + 4 * l + t] : 0.0;
    }
    if (wrap_role) {
      if (MODE == MOM_WRAP && a.r_out) {  // ||z_i||: lane partial over its columns, then over the 8 column lanes
        double sq = 0.0;
#pragma unroll
        for (int b = 0; b < NB; b++) sq = __dadd_rn(sq, __dmul_rn(u[b], u[b]));
        sq = __dadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, 4));
        sq = __dadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, 8));
        sq = __dadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, 16));
        if (g == 0 && row < r_end) a.r_out[(long long)blk * m + row] = __dsqrt_rn(sq);
      }
      // psi: identity / zero branches in place; the tanh branch (1.5 < |z| <= 4, ~13 %
      // of the entries) compacted into a warp-private list, evaluated by all 32 lanes, scattered back.
      // The branch tests look at the magnitude's HIGH word only (IEEE order; integer pipe, no fp64 abs):
      // hi in [hi(1.5), hi(4)) is 1.5 <= |z| < 4, listed (|z| == 1.5 exactly, the one listed value of
      // the identity branch, is kept as is by the tanh pass); hi >= hi(4) is |z| >= 4 -> 0 (psi(4) =
      // q1 tanh(0) = 0, so |z| == 4 may take either branch).  A lane's slots in the list come from one
      // ballot per column block.
      constexpr unsigned H15 = 0x3FF80000u, H40 = 0x40100000u;  // high words of 1.5 and 4.0
      int pos[NB];
      int n = 0;
      const unsigned lt = (1u << lane) - 1u;
#pragma unroll
      for (int b = 0; b < NB; b++) {
        const unsigned ah = (unsigned)__double2hiint(u[b]) & 0x7FFFFFFFu;
        const bool need = ah - H15 < H40 - H15;
        const unsigned bal = __ballot_sync(0xffffffffu, need);
        pos[b] = need ? n + __popc(bal & lt) : -1;
        if (need) scr[pos[b]] = __hiloint2double((int)ah, __double2loint(u[b]));  // |z|
        n += __popc(bal);
        if (ah >= H40) u[b] = 0.0;
      }
      if (n) {
        __syncwarp();
        for (int i = lane; i < n; i += 32) {
          const double az = scr[i];
          if (__double_as_longlong(az) != 0x3FF8000000000000ll)  // |z| == 1.5: identity branch
            scr[i] = __dmul_rn(1.541, tanh_tab(__dmul_rn(0.862, __dsub_rn(4.0, az)), ttab));
        }
        __syncwarp();
#pragma unroll
        for (int b = 0; b < NB; b++)
          if (pos[b] >= 0) u[b] = copysign(scr[pos[b]], u[b]);  // |z| >= 1.5: the sign bit is the sign
        __syncwarp();
      }
    } else if (MODE == MOM_MEMBER || MODE == MOM_REWEIGHT) {
#pragma unroll
      for (int b = 0; b < NB; b++) u[b] = (w != 0.0 && 8 * b + g < P) ? __dsub_rn(u[b], sh[b]) : 0.0;
    }
    double wu[NB];
    // w = 1 (wrap warps; warp-uniform) or w in {0, 1} with u already 0 where w = 0 (member / reweight
    // modes): w u = u exactly, so no product on the fp64 pipe the DMMAs share
    if (wrap_role || MODE == MOM_MEMBER || MODE == MOM_REWEIGHT) {
#pragma unroll
      for (int b = 0; b < NB; b++) {
        wu[b] = u[b];
        s1[b] += u[b];
      }
    } else {
#pragma unroll
      for (int b = 0; b < NB; b++) {
        wu[b] = w * u[b];
        s1[b] += wu[b];
      }
    }
    if (g == 0) cnt += w;
    int kk = 0;
#pragma unroll
    for (int jb = 0; jb < NB; jb++)
#pragma unroll
      for (int kb = 0; kb <= jb; kb++) {
        dmma_m(acc[kk][0], acc[kk][1], wu[jb], u[kb]);
        kk++;
      }
  }
  if (cur >= 0) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[cur % NS]);
  }
  // epilogue (consumer warps only): per-warp sums into shared memory (the ring is free: every tile was
  // consumed), fixed-order sum over the warps -> this CTA's partial row
#pragma unroll
  for (int b = 0; b < NB; b++) {
    s1[b] += __shfl_xor_sync(0xffffffffu, s1[b], 1);
    s1[b] += __shfl_xor_sync(0xffffffffu, s1[b], 2);
  }
  cnt += __shfl_xor_sync(0xffffffffu, cnt, 1);
  cnt += __shfl_xor_sync(0xffffffffu, cnt, 2);
  consumer_sync();  // all warps are past their last tile read
  double* red = tiles;
  double* rw = red + warp * NP;
  for (int e = lane; e < NP; e += 32) rw[e] = 0.0;
  __syncwarp();
  if (t == 0) {
#pragma unroll
    for (int b = 0; b < NB; b++)
      if (8 * b + g < P) rw[8 * b + g] = s1[b];
  }
  if (lane == 0) rw[NP - 1] = cnt;
  {
    int kk = 0;
#pragma unroll
    for (int jb = 0; jb < NB; jb++)
#pragma unroll
      for (int kb = 0; kb <= jb; kb++) {
        const int j = 8 * jb + g;
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int c = 8 * kb + 2 * t + e;
          if (j < P && c < P && c <= j) rw[P + j * (j + 1) / 2 + c] = acc[kk][e];
        }
        kk++;
      }
  }
  consumer_sync();
  const long long po = ((long long)slot * a.ctas + blockIdx.x) * NP;
  const int q1 = FX ? split : NCW;  // warps [0, q1) -> partial, [q1, NCW) -> partial2 (fixed order)
  for (int e = threadIdx.x; e < NP; e += NCW * 32) {
    double v = 0.0;
    for (int q = 0; q < q1; q++) v += red[q * NP + e];
    a.partial[po + e] = v;
    if (FX) {
      double v2 = 0.0;
      for (int q = q1; q < NCW; q++) v2 += red[q * NP + e];
      a.partial2[po + e] = v2;
    }
  }
}

namespace {

template <int P, int W>
void moments_tma_pw(int mode, const MomArgs& a, int ninst, cudaStream_t st) {
  using C = MomTmaCfg<P, W>;
  CUtensorMap map;  // blocks addressed by the 3rd coordinate: a.nblk_hint blocks of m x p doubles at a.Z
  if (!encode_blocks(&map, a.Z, a.m, P, a.nblk_hint, C::TR))
    throw std::string("cuTensorMapEncodeTiled failed for the moment pass");
  CUtensorMap wmap = map;  // MOM_WRAP: unused
  bool ok = true;
  if (mode == MOM_XI || mode == MOM_WRAPXI)
    ok = encode_rows(&wmap, a.r, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, a.m, a.nblk_hint, C::TR);
  if (mode == MOM_REWEIGHT) ok = encode_rows(&wmap, a.d2, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, a.m, a.ninst_hint, C::TR);
  if (!ok) throw std::string("cuTensorMapEncodeTiled failed for the moment weights");
  dim3 grid(a.ctas, ninst);
#define RTD_MT_CASE(M)                                                                                        \
  case M:                                                                                                     \
    set_max_dyn_smem(reinterpret_cast<const void*>(k_moments_tma<P, M, W>), (int)C::SMEM); \
    k_moments_tma<P, M, W><<<grid, C::NCW * 32, C::SMEM, st>>>(map, wmap, a);                                   \
    break;
  switch (mode) {
    RTD_MT_CASE(MOM_WRAP)
    RTD_MT_CASE(MOM_XI)
    RTD_MT_CASE(MOM_MEMBER)
    RTD_MT_CASE(MOM_REWEIGHT)
    RTD_MT_CASE(MOM_WRAPXI)
    default: throw std::string("moments_tma: mode");
  }
#undef RTD_MT_CASE
}

// W = 16 (one CTA of 16 warps and a 192 KB ring per SM) measured slower on config 4 (wrapped + xi pass
// 1.94 -> 1.98 ms, member moments 1.36 -> 1.52 ms): two CTAs of 8 warps
template <int P>
void moments_tma_p(int mode, const MomArgs& a, int ninst, cudaStream_t st) {
  moments_tma_pw<P, 8>(mode, a, ninst, st);
}

}  // namespace

bool moments_tma_supported(int mode, const MomArgs& a) {
  static const bool off = getenv("RTD_MOM_NOTMA") != nullptr;
  if (mode == MOM_WRAPXI && (a.partial2 == nullptr || a.split < 1 || a.split >= 8 || a.r == nullptr))
    return false;
  return !off && mode != MOM_DELTA && a.p >= 8 && a.p <= RTD_MAXP && a.m % 16 == 0 && a.m >= 8192 &&
         a.blk_stride == (long long)a.p * a.m && a.nblk_hint > 0 &&
         (a.ninst_hint > 0 || mode != MOM_REWEIGHT) && encode_fn() != nullptr;
}

void launch_moments_tma(int mode, const MomArgs& a, int ninst, cudaStream_t st) {
  switch (a.p) {
#define RTD_MP(P) \
  case P: moments_tma_p<P>(mode, a, ninst, st); break;
    RTD_MP(8) RTD_MP(9) RTD_MP(10) RTD_MP(11) RTD_MP(12) RTD_MP(13) RTD_MP(14) RTD_MP(15) RTD_MP(16) RTD_MP(17)
    RTD_MP(18) RTD_MP(19) RTD_MP(20) RTD_MP(21) RTD_MP(22) RTD_MP(23) RTD_MP(24) RTD_MP(25) RTD_MP(26) RTD_MP(27)
    RTD_MP(28) RTD_MP(29) RTD_MP(30) RTD_MP(31) RTD_MP(32) RTD_MP(33) RTD_MP(34) RTD_MP(35) RTD_MP(36) RTD_MP(37)
    RTD_MP(38) RTD_MP(39) RTD_MP(40)
#undef RTD_MP
    default: throw std::string("moments_tma: p out of range");
  }
  RTD_LAUNCHED();
}

}  // namespace rtd
