// Small helper kernels: Feistel forward map, extraction of univariate results,
// per-row outputs in original row order, scaled matrix copies; the batched
// device -> host read helper.
#include <algorithm>
#include <cstring>
#include <vector>

#include <map>
#include <mutex>
#include <utility>

#include "rtd_internal.h"

namespace rtd {

// Several device -> host reads behind ONE stream synchronisation: the copies land in a pinned staging
// buffer (a copy into pageable memory would synchronise by itself), then are unpacked.
void set_max_dyn_smem(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  RTD_CU(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  int& cur = done[{dev, func}];
  if (bytes <= cur) return;
  RTD_CU(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  cur = bytes;
}

void fetch(cudaStream_t st, std::initializer_list<Fetch> items) {
  static thread_local char* stage = nullptr;
  static thread_local size_t cap = 0;
  size_t need = 0;
  for (const Fetch& f : items) need += (f.bytes + 255) & ~size_t(255);
  if (need > cap) {
    if (stage) cudaFreeHost(stage);
    cap = std::max(need, size_t(1) << 20);
    RTD_CU(cudaMallocHost(&stage, cap));
  }
  size_t off = 0;
  for (const Fetch& f : items) {
    if (f.bytes) RTD_CU(cudaMemcpyAsync(stage + off, f.dev, f.bytes, cudaMemcpyDeviceToHost, st));
    off += (f.bytes + 255) & ~size_t(255);
  }
  RTD_CU(cudaStreamSynchronize(st));
  off = 0;
  for (const Fetch& f : items) {
    if (f.bytes) memcpy(f.host, stage + off, f.bytes);
    off += (f.bytes + 255) & ~size_t(255);
  }
}


__device__ __forceinline__ unsigned long long splitmix64_f(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ unsigned long long feistel_enc(unsigned long long x, unsigned long long seed, int half) {
  const unsigned long long mask = (1ull << half) - 1ull;
  unsigned long long L = x >> half, R = x & mask;
  for (int r = 0; r < 6; r++) {
    unsigned long long F = splitmix64_f(seed ^ ((unsigned long long)r * 0x9E3779B97F4A7C15ull) ^ R) & mask;
    unsigned long long nl = R;
    R = L ^ F;
    L = nl;
  }
  return (L << half) | R;
}

__global__ void k_feistel_fwd(long long n, unsigned long long seed, int half, long long* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long x = feistel_enc((unsigned long long)i, seed, half);
    while (x >= (unsigned long long)n) x = feistel_enc(x, seed, half);
    out[i] = (long long)x;
  }
}

void launch_feistel_fwd(long long n, unsigned long long seed, long long* out, cudaStream_t st) {
  int bits = 0;
  while ((1ll << bits) < n) bits++;
  if (bits < 2) bits = 2;
  bits += bits & 1;
  unsigned gx = (unsigned)std::min<long long>((n + 255) / 256, 148 * 16);
  k_feistel_fwd<<<gx, 256, 0, st>>>(n, seed, bits / 2, out);
  RTD_LAUNCHED();
}

// which 0: out[j] = scale_j^2 (refinement step 3); 1: out[j] = loc_j (step 4)
__global__ void k_uni_extract(const UniOut* __restrict__ uni, int p, int which, double* __restrict__ out) {
  for (int j = threadIdx.x; j < p; j += blockDim.x) out[j] = which == 0 ? uni[j].scale * uni[j].scale : uni[j].loc;
}

void launch_uni_extract(const UniOut* uni, int p, int which, double* out, cudaStream_t st) {
  k_uni_extract<<<1, 64, 0, st>>>(uni, p, which, out);
  RTD_LAUNCHED();
}

// warm start: the previous fit (mu, Sigma) in X units -> this run's standardised
// units, written as start 0 of every block: mu_z = (mu - loc) / scale, Sigma_z = Sigma / (scale scale^T)
__global__ void k_warm_start(const UniOut* __restrict__ uni, const double* __restrict__ mu_x,
                             const double* __restrict__ sig_x, int p, double* __restrict__ mu_all,
                             double* __restrict__ sig_all) {
  const int b = blockIdx.x;
  double* mu = mu_all + (long long)(2 * b) * RTD_MAXP;
  double* sg = sig_all + (long long)(2 * b) * RTD_MAXP * RTD_MAXP;
  for (int k = threadIdx.x; k < p; k += blockDim.x) mu[k] = __ddiv_rn(__dsub_rn(mu_x[k], uni[k].loc), uni[k].scale);
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int i = e / p, j = e - i * p;
    sg[e] = __ddiv_rn(sig_x[e], __dmul_rn(uni[i].scale, uni[j].scale));
  }
}

void launch_warm_start(const UniOut* uni, const double* mu_x, const double* sig_x, int p, int q, double* mu_all,
                       double* sig_all, cudaStream_t st) {
  k_warm_start<<<q, 256, 0, st>>>(uni, mu_x, sig_x, p, mu_all, sig_all);
  RTD_LAUNCHED();
}

// eq[b] = 1 iff the membership bytes of instances 2b and 2b+1 agree on all m rows (the two starts of
// block b reached the same h-subset)
__global__ void k_mem_pairs_equal(const uint8_t* __restrict__ mem_all, long long m, int* __restrict__ eq) {
  const int b = blockIdx.y;
  const uint8_t* x = mem_all + (long long)(2 * b) * m;
  const uint8_t* y = mem_all + (long long)(2 * b + 1) * m;
  int diff = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
    diff |= x[i] != y[i];
  if (__syncthreads_or(diff) && threadIdx.x == 0) eq[b] = 0;
}

void launch_mem_pairs_equal(const uint8_t* mem_all, long long m, int nblk, int* eq, cudaStream_t st) {
  std::vector<int> ones(nblk, 1);
  RTD_CU(cudaMemcpyAsync(eq, ones.data(), nblk * sizeof(int), cudaMemcpyHostToDevice, st));
  const unsigned gx = (unsigned)std::max<long long>(1, std::min<long long>((m + 255) / 256, 64));
  k_mem_pairs_equal<<<dim3(gx, nblk), 256, 0, st>>>(mem_all, m, eq);
  RTD_LAUNCHED();
}

// batched: item i (uni columns [i p, (i+1) p)) -> out_all[slot_of[i]][j]
__global__ void k_uni_extract_batch(const UniOut* __restrict__ uni, const int* __restrict__ slot_of, int p, int which,
                                    double* __restrict__ out_all) {
  const int i = blockIdx.x;
  double* out = out_all + (long long)slot_of[i] * RTD_MAXP;
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    const UniOut& u = uni[(long long)i * p + j];
    out[j] = which == 0 ? u.scale * u.scale : u.loc;
  }
}

void launch_uni_extract_batch(const UniOut* uni, const int* slot_of, int nitems, int p, int which, double* out_all,
                              cudaStream_t st) {
  k_uni_extract_batch<<<nitems, 64, 0, st>>>(uni, slot_of, p, which, out_all);
  RTD_LAUNCHED();
}

__global__ void k_weights_from_d2(const double* __restrict__ d2, long long total, double c2,
                                  const long long* __restrict__ rowmap, uint8_t* __restrict__ dst) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    long long row = rowmap ? rowmap[t] : t;
    dst[row] = d2[t] <= c2 ? 1 : 0;
  }
}

void launch_weights_from_d2(const double* d2, long long total, double c2, const long long* rowmap, uint8_t* dst,
                            cudaStream_t st) {
  unsigned gx = (unsigned)std::min<long long>((total + 255) / 256, 148 * 16);
  k_weights_from_d2<<<gx, 256, 0, st>>>(d2, total, c2, rowmap, dst);
  RTD_LAUNCHED();
}

__global__ void k_hsub_from_mem(const uint8_t* __restrict__ mem_all, const int* __restrict__ chosen_inst, long long m,
                                const long long* __restrict__ rowmap, uint8_t* __restrict__ dst) {
  const int b = blockIdx.y;
  const int id = chosen_inst[b];
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < m; s += (long long)gridDim.x * blockDim.x) {
    long long t = (long long)b * m + s;
    long long row = rowmap ? rowmap[t] : t;
    dst[row] = id >= 0 ? mem_all[(long long)id * m + s] : 0;
  }
}

void launch_hsub_from_mem(const uint8_t* mem_all, const int* chosen_inst, int q, long long m, const long long* rowmap,
                          uint8_t* dst, cudaStream_t st) {
  unsigned gx = (unsigned)std::min<long long>((m + 255) / 256, 148 * 8);
  k_hsub_from_mem<<<dim3(gx, q), 256, 0, st>>>(mem_all, chosen_inst, m, rowmap, dst);
  RTD_LAUNCHED();
}

__global__ void k_scale_copy(const double* __restrict__ src, double* __restrict__ dst, int p, double factor) {
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) dst[e] = factor * src[e];
}

void launch_scale_copy(const double* src, double* dst, int p, double factor, cudaStream_t st) {
  k_scale_copy<<<1, 256, 0, st>>>(src, dst, p, factor);
  RTD_LAUNCHED();
}

}  // namespace rtd
