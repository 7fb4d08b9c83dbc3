// Weighted first and second moments over the rows of a block (column-major Z):
//   S1 = sum_i w_i f(z_i),  S2 = sum_i w_i f(z_i) f(z_i)^T,  count = sum_i w_i
// One kernel serves every moment the method needs:
//   MOM_WRAP     f = g(z) (eq. wrapping), w = 1          -> S~1
//   MOM_XI       f = z, w = xi(||z||)^2                  -> S~2 (eq. LR)
//   MOM_MEMBER   f = z - c, w = [i in H]                 -> C-step mean/cov (eqs. cstep4a/b)
//   MOM_DELTA    f = z - c, w = delta_i in {-1,0,+1}     -> update-based C-step
//   MOM_REWEIGHT f = z - c, w = [d_i^2 <= chi2]          -> reweighting
// Row tiles of 32 whose weights are all zero are skipped without touching Z,
// so the delta path only reads the tiles that hold entering/leaving rows.
// Each CTA owns a fixed row range and writes a partial; partials are summed
// in CTA order (deterministic, no floating-point atomics).
#include "rtd_internal.h"

namespace rtd {

static constexpr int MT = 320;   // threads: 4 row groups x up to 55 (4x4 lower blocks at p=40) = 220 active
static constexpr int MTR = 32;   // rows per tile

int mom_np(int p) { return p + p * (p + 1) / 2 + 1; }

__device__ __forceinline__ double wrap_g(double z) {
  const double b = 1.5, c = 4.0, q1 = 1.541, q2 = 0.862;
  double az = fabs(z);
  if (az <= b) return z;
  if (az <= c) {
    double t = __dmul_rn(q1, tanh(__dmul_rn(q2, __dsub_rn(c, az))));
    return z > 0 ? t : (z < 0 ? -t : 0.0);
  }
  return 0.0;
}

template <int MODE>
__global__ void __launch_bounds__(MT) k_moments(MomArgs a) {
  __shared__ double U[RTD_MAXP][MTR + 1];
  __shared__ double W[MTR];
  __shared__ double red[4][RTD_MAXP + RTD_MAXP * (RTD_MAXP + 1) / 2 + 1];
  const int slot = blockIdx.y;
  const int id = a.inst[slot];
  const int blk = id / a.nstart;
  const int p = a.p;
  const long long m = a.m;
  const double* __restrict__ Z = a.Z + (long long)blk * a.blk_stride;
  const int t = threadIdx.x;
  const int NP = p + p * (p + 1) / 2 + 1;
  const int nbr = (p + 3) >> 2;
  const int nb = nbr * (nbr + 1) / 2;
  // zero padding rows of U and the reduction buffer
  for (int e = t; e < RTD_MAXP * (MTR + 1); e += MT) (&U[0][0])[e] = 0.0;
  for (int e = t; e < 4 * NP; e += MT) red[e / NP][e % NP] = 0.0;
  int grp = -1, bj = 0, bk = 0;
  if (t < 4 * nb) {
    grp = t / nb;
    int b = t - grp * nb;
    // lower-triangular block b -> (bj, bk), bj >= bk
    int r = 0;
    while (b > r) { b -= r + 1; r++; }
    bj = r;
    bk = b;
  }
  const double* shift = (MODE >= MOM_MEMBER) ? a.shift + (long long)id * RTD_MAXP : nullptr;
  double A = 0.0, B = 0.0;
  if (MODE == MOM_XI) {
    A = a.AB[2 * blk];
    B = a.AB[2 * blk + 1];
  }
  long long per = (m + a.ctas - 1) / a.ctas;
  per = (per + MTR - 1) / MTR * MTR;
  const long long r_begin = (long long)blockIdx.x * per;
  const long long r_end = min(m, r_begin + per);
  double acc[4][4];
  double s1[4];
  double cnt = 0.0;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    s1[i] = 0.0;
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = 0.0;
  }
  __syncthreads();
  for (long long ts = r_begin; ts < r_end; ts += MTR) {
    double w = 0.0;
    if (t < MTR) {
      long long row = ts + t;
      if (row < r_end) {
        if (MODE == MOM_WRAP) {
          w = 1.0;
        } else if (MODE == MOM_XI) {
          double r = a.r[(long long)blk * m + row];
          double xi = r <= A ? 1.0 : (r <= B ? __ddiv_rn(__dsub_rn(B, r), __dsub_rn(B, A)) : 0.0);
          w = __dmul_rn(xi, xi);
        } else if (MODE == MOM_MEMBER) {
          w = (double)a.mem_new[(long long)id * m + row];
        } else if (MODE == MOM_DELTA) {
          w = (double)((int)a.mem_new[(long long)id * m + row] - (int)a.mem_old[(long long)id * m + row]);
        } else {
          w = a.d2[(long long)id * m + row] <= a.c2 ? 1.0 : 0.0;
        }
      }
      W[t] = w;
    }
    if (!__syncthreads_or(w != 0.0)) continue;
    for (int e = t; e < p * MTR; e += MT) {
      int k = e / MTR, r = e - k * MTR;
      long long row = ts + r;
      double v = 0.0;
      if (row < r_end && W[r] != 0.0) {
        v = Z[(long long)k * m + row];
        if (MODE == MOM_WRAP) v = wrap_g(v);
        else if (MODE >= MOM_MEMBER) v = __dsub_rn(v, shift[k]);
      }
      U[k][r] = v;
    }
    __syncthreads();
    if (grp >= 0) {
      for (int rr = 0; rr < 8; rr++) {
        const int r = grp * 8 + rr;
        const double wr = W[r];
        if (wr == 0.0) continue;
        double av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
          av[i] = U[bj * 4 + i][r] * wr;
          bv[i] = U[bk * 4 + i][r];
        }
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
          for (int j = 0; j < 4; j++) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        if (bj == bk) {
#pragma unroll
          for (int i = 0; i < 4; i++) s1[i] += av[i];
        }
        if (bj == 0 && bk == 0) cnt += wr;
      }
    }
    __syncthreads();
  }
  // reduce the 4 row groups through shared memory (fixed order)
  for (int g = 0; g < 4; g++) {
    if (grp == g) {
      for (int i = 0; i < 4; i++) {
        int j = bj * 4 + i;
        if (j >= p) continue;
        for (int jj = 0; jj < 4; jj++) {
          int k = bk * 4 + jj;
          if (k >= p || k > j) continue;
          red[g][p + j * (j + 1) / 2 + k] = acc[i][jj];
        }
        if (bj == bk) red[g][j] = s1[i];
      }
      if (bj == 0 && bk == 0) red[g][NP - 1] = cnt;
    }
  }
  __syncthreads();
  double* out = a.partial + ((long long)slot * a.ctas + blockIdx.x) * NP;
  for (int e = t; e < NP; e += MT) out[e] = ((red[0][e] + red[1][e]) + red[2][e]) + red[3][e];
}

void launch_moments(int mode, const MomArgs& a, int ninst, cudaStream_t st) {
  dim3 grid(a.ctas, ninst);
  switch (mode) {
    case MOM_WRAP: k_moments<MOM_WRAP><<<grid, MT, 0, st>>>(a); break;
    case MOM_XI: k_moments<MOM_XI><<<grid, MT, 0, st>>>(a); break;
    case MOM_MEMBER: k_moments<MOM_MEMBER><<<grid, MT, 0, st>>>(a); break;
    case MOM_DELTA: k_moments<MOM_DELTA><<<grid, MT, 0, st>>>(a); break;
    case MOM_REWEIGHT: k_moments<MOM_REWEIGHT><<<grid, MT, 0, st>>>(a); break;
  }
  RTD_LAUNCHED();
}

// Fixed-order (deterministic) sum of the per-CTA partials: CTA (x, slot) owns 32 consecutive
// entries; warp w sums the partials of CTAs w, w+8, w+16, ... and the 8 warp sums are added in
// warp order.
__global__ void __launch_bounds__(256) k_mom_reduce(const double* __restrict__ partial, const int* __restrict__ inst,
                                                    int ctas, int np, double* __restrict__ out, int accumulate) {
  __shared__ double ws[8][32];
  const int slot = blockIdx.y;
  const int id = inst[slot];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (e < np) {
    const double* src = partial + (long long)slot * ctas * np + e;
#pragma unroll 4
    for (int c = w; c < ctas; c += 8) s += src[(long long)c * np];
  }
  ws[w][lane] = s;
  __syncthreads();
  if (w == 0 && e < np) {
    double t = ws[0][lane];
    for (int k = 1; k < 8; k++) t += ws[k][lane];
    double* o = out + (long long)id * np + e;
    *o = accumulate ? *o + t : t;
  }
}

void launch_mom_reduce(const double* partial, int ninst, const int* inst, int ctas, int np, double* out,
                       int accumulate, cudaStream_t st) {
  k_mom_reduce<<<dim3((np + 31) / 32, ninst), 256, 0, st>>>(partial, inst, ctas, np, out, accumulate);
  RTD_LAUNCHED();
}

}  // namespace rtd
