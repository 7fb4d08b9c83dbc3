// Internal (non-ABI) declarations of the RT-DetMCD CUDA path.
#pragma once
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "common.cuh"

namespace rtd {

// ---------------------------------------------------------------- errors
struct CudaError {
  cudaError_t code;
  std::string where;
};
#define RTD_CU(x)                                                         \
  do {                                                                    \
    cudaError_t e__ = (x);                                                \
    if (e__ != cudaSuccess) throw ::rtd::CudaError{e__, #x};              \
  } while (0)
bool debug_sync();  // RTD_DEBUG_SYNC=1: synchronise and check after every launch
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel, size): the runtime call costs
// microseconds of host time, on the critical path of a latency-bound fit when made before every launch
void set_max_dyn_smem(const void* func, int bytes);
void count_launch(const char* file, int line);  // kernels launched by this library (hand-written kernels)
void count_sort();    // CUB radix-sort invocations
#define RTD_LAUNCHED()                                                      \
  do {                                                                      \
    ::rtd::count_launch(__FILE__, __LINE__);                                \
    RTD_CU(cudaGetLastError());                                             \
    if (::rtd::debug_sync()) {                                              \
      cudaError_t e2__ = cudaDeviceSynchronize();                           \
      if (e2__ != cudaSuccess)                                              \
        throw ::rtd::CudaError{e2__, std::string("kernel before ") + __FILE__ + ":" + std::to_string(__LINE__)}; \
    }                                                                       \
  } while (0)

// ---------------------------------------------------------------- device -> host reads
// Several device -> host copies behind one stream synchronisation (pinned staging; api.cu).
struct Fetch {
  void* host;
  const void* dev;
  size_t bytes;
};
void fetch(cudaStream_t st, std::initializer_list<Fetch> items);

// ---------------------------------------------------------------- arena
// Bump allocator over one device buffer.  A dry run (base == nullptr)
// measures the bytes a call needs; the real run carves the same offsets.
struct Arena {
  char* base = nullptr;
  size_t off = 0, cap = 0;
  template <class T>
  T* take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
    size_t o = off;
    off += bytes;
    if (base == nullptr) return nullptr;
    if (off > cap) throw std::string("workspace overflow");
    return reinterpret_cast<T*>(base + o);
  }
};

// ---------------------------------------------------------------- univariate MCD (K1)
struct UniOut {
  double loc, scale;      // reweighted estimate
  double raw_loc, raw_var;  // raw window mean, SQ/(h-1) without factor
  double var0;            // c(h/n,1) * raw_var
  long long start, kept;  // window start s*, number of kept points
  int status;             // 0 ok, 1 degenerate scale
  int pad;
};
struct UniConst {
  double c_raw;   // c(h/len, 1)
  double q1;      // chi2_{1,0.975}
  double c_rew;   // c(0.975, 1)
};
// ncols columns of length len, column-major contiguous (col j at cols + j*len).
void unimcd_batch(Arena& A, cudaStream_t st, const double* cols, long long len, int ncols, UniConst uc,
                  UniOut* out_dev);
size_t unimcd_scratch_hint(long long len, int ncols);

// ---------------------------------------------------------------- host numerics
double chi2_cdf(double x, int dof);
double chi2_quantile(double prob, int dof);
double consistency_factor(double alpha, int p);

// ---------------------------------------------------------------- constant bank
// the constant bank c_mat lives in k_dist.cu (its only reader).  It is one per device and process, so
// several contexts (streams) must not overwrite it while another's kernel reads it: a ConstLease holds a
// per-device lock from the upload until it goes out of scope (after the consuming launches are enqueued),
// makes its stream wait for the previous lease's consumers, and records their completion on release.
// Keep a lease alive exactly around the launches that read c_mat; never nest two.
class ConstLease {
 public:
  ConstLease(const double* dev_src, size_t count, cudaStream_t st);
  ~ConstLease();
  ConstLease(const ConstLease&) = delete;
  ConstLease& operator=(const ConstLease&) = delete;

 private:
  int dev_ = 0;
  cudaStream_t st_;
};

// ---------------------------------------------------------------- streaming kernels (k_dist.cu)
// X row-major n x p -> Xc column-major; nonfinite (or <= 0 when log) rows -> min index in *bad.
void launch_transpose(const double* X, long long n, int p, int log_transform, double* Xc,
                      unsigned long long* bad, cudaStream_t st);
// Z[b][k][s] = (src - loc_k)/scale_k for q blocks of m rows; perm == 0: identity from Xc,
// else row = feistel^-1(b*m+s) gathered from row-major X (with optional log).
void launch_build_Z(const double* Xc, const double* X, long long n, int p, int q, long long m, int perm,
                    unsigned long long seed, int log_transform, const UniOut* uni, double* Z, long long* rowmap,
                    double* r_out /* [q][m] row norms ||z_i|| (nullable) */,
                    cudaStream_t st);
// d2 for instances: rows of instance id = Zall + (id / nstart) * blk_stride; d2 at d2_all + id * m;
// constants in c_mat at slot*cstride:
//   [mu (p)] [M packed lower (p(p+1)/2)]
void launch_dist(int p, const double* Zall, long long m, long long blk_stride, const int* inst, int nstart, int ninst,
                 int cstride, double* d2_all, cudaStream_t st);
// out[j][i] = sum_k Z[k][i] * W[k][j], W full p x p in c_mat[0..p*p) (row-major k, j)
void launch_matmul(int p, const double* Z, long long m, double* out, cudaStream_t st);
// row-major flag pass: d2 = ||M (x - mu)||^2 with [mu][M] in c_mat slot 0
// p >= 8: the flagging pass on DMMA, rows staged per warp by cp.async; operator read from cs
void launch_flag_mma(int p, const double* X, long long n, int log_transform, const double* cs, double c2,
                     uint8_t* flags, double* rd2, cudaStream_t st);
void launch_flag(int p, const double* X, long long n, int log_transform, double c2, uint8_t* flags, double* rd2,
                 cudaStream_t st);
void launch_norms(const double* Z, long long m, int p, int nblk, long long blk_stride, double* r, cudaStream_t st);

// ---------------------------------------------------------------- norm quantiles (k_quantile.cu)
size_t quantile_scratch_bytes(int nb);
// qv[nb][6] = order statistics j, j+1 of the type-7 positions (m-1){.25,.5,.75} of r_all[b][0..m);
// fallback = blocks whose target bucket overflowed (the caller sorts them, launch_q_from_sorted)
void launch_quantiles(const double* r_all, long long m, int nb, char* scratch, double* qv, cudaStream_t st,
                      std::vector<int>& fallback);
void launch_q_from_sorted(const double* sorted, long long m, int b, double* qv, cudaStream_t st);
void launch_q_cutoffs(const double* qv, long long m, int nb, double* AB, int* ok, cudaStream_t st);

// ---------------------------------------------------------------- moments (k_moments.cu)
// MOM_WRAPXI (TMA path only): MOM_WRAP and MOM_XI from one read of Z -- warps [0, split) take the wrapped
// moments into partial, the others the xi-weighted ones into partial2 (norms r and cutoffs AB known)
enum MomMode { MOM_WRAP = 0, MOM_XI = 1, MOM_MEMBER = 2, MOM_DELTA = 3, MOM_REWEIGHT = 4, MOM_WRAPXI = 5 };
struct MomArgs {
  const double* Z;          // base of all blocks (column-major per block)
  long long m;              // rows per block
  long long blk_stride;     // doubles between blocks
  int p;
  const int* inst;          // active instance ids [ninst]
  int nstart;               // instances per block (block = inst / nstart)
  const double* shift;      // [inst][p] shift c
  const uint8_t* mem_new;   // [inst][m]
  const uint8_t* mem_old;   // [inst][m]
  const double* d2;         // [inst][m] (reweight)
  double c2;
  const double* r;          // [block][m] norms (xi mode)
  double* r_out;            // [block][m] norms written by the staged wrap pass (nullable)
  const double* AB;         // [block][2] cutoffs (xi mode)
  double* partial;          // [slot][cta][NP]
  int ctas;                 // CTAs per instance
  const int* list;          // [inst][m] changed rows per segment (+-(row+1)), MOM_DELTA on the tensor pipe
  const int* seg_cnt;       // [inst][ctas] entries per segment
  long long seg_len;        // rows per segment (segment x = CTA x)
  int nblk_hint;            // blocks of m x p doubles at Z (the TMA-fed dense passes map them; 0: unknown)
  int ninst_hint;           // instances the per-instance arrays (mem_new, d2) hold (0: unknown)
  double* partial2;         // MOM_WRAPXI: [slot][cta][NP] partials of the xi-weighted moments
  int split;                // MOM_WRAPXI: eighths of the CTA's warps on the wrapped moments (the rest: xi-weighted)
};
int mom_np(int p);  // p + p(p+1)/2 + 1
void launch_moments(int mode, const MomArgs& a, int ninst, cudaStream_t st);
// out[inst][NP] (= or +=) fixed-order sum of partials
void launch_mom_reduce(const double* partial, int ninst, const int* inst, int ctas, int np, double* out, int accumulate,
                       cudaStream_t st);

// ---------------------------------------------------------------- select (k_select.cu)
struct SelState {
  unsigned long long prefix_hi;  // composite-key prefix of the bin holding the h-th key (plen bits)
  unsigned long long prefix_lo;
  long long rank;                // rank still needed inside the current prefix
  unsigned long long base;       // centred first level: top-24-bit key of bin 1
  long long count_in;            // keys below the current prefix (diagnostic)
  int plen;                      // prefix length in bits (0..96)
  int done;
  int valid;                     // done and prefix usable to centre the next step's first level
  int centred;                   // the next level is the centred 24-bit level
  int candok;                    // not done, but the h-th key's bin (plen >= 24) holds <= SEL_CAND rows:
                                 // they are listed by k_sel_member and resolved by k_sel_fixup
  long long bincnt;              // rows in the bin of the current prefix
};
// a row of the h-th key's bin (candidate mode): its d^2 bits, row and reserved changed-list position
struct SelCand {
  unsigned long long kb;
  int row;
  int listpos;
};
// Selection of the h smallest (d^2, row) per instance + membership + ordered changed-row lists:
// list_all[id][seg x at x seg_len] (+-(row+1)), seg_cnt_all[id][nseg]; changed[id] must be zero on
// entry; changed[id] == -1 on exit means the selection needs launch_select_finish.
// st_all must be zeroed before the first step of a trajectory (no centring then).
// cand_all[inst][SEL_CAND] / cand_cnt[inst]: the candidate-mode buffers (a list entry 0 is a reserved slot of
// a candidate row that did not change: consumers skip it).
constexpr int SEL_CAND = 4096;
bool sel_cand_mode();  // RTD_SEL_NOCAND unset
void launch_select(const double* d2_all, long long m, long long h, const int* inst, int ninst, SelState* st_all,
                   unsigned int* hist_all, unsigned int* cnt_all, uint8_t* mem_new_all, const uint8_t* mem_old_all,
                   int* changed, int* list_all, int* seg_cnt_all, int nseg, long long seg_len, SelCand* cand_all,
                   int* cand_cnt, cudaStream_t st, int nfast = 3);
void launch_select_finish(const double* d2_all, long long m, const int* inst, int ninst, SelState* st_all,
                          unsigned int* hist_all, unsigned int* cnt_all, uint8_t* mem_new_all,
                          const uint8_t* mem_old_all, int* changed, int* list_all, int* seg_cnt_all, int nseg,
                          long long seg_len, SelCand* cand_all, int* cand_cnt, cudaStream_t st);

}  // namespace rtd
