// Launchers of the single-CTA dense linear algebra kernels (k_linalg.cu).
// Matrices are p x p row-major, compact, at a stride of RTD_MAXP^2 doubles per
// instance; vectors at a stride of RTD_MAXP doubles.
#pragma once
#include "rtd_internal.h"

namespace rtd {

enum InstStatus { ST_ACTIVE = 0, ST_CONVERGED = 1, ST_NOT_PD = 2, ST_COND = 3, ST_MAXSTEPS = 4, ST_REFINE = 5, ST_SKIPPED = 6 };

void launch_prepare(const int* inst, int ninst, const double* mu_all, const double* sigma_all, int p, double kappa_max,
                    double* cstage, int cstride, double* logdet_out, double* cond_out, int* status_out, double* traj,
                    int traj_stride, int step, cudaStream_t st, int full_inverse = 0, const int* skip = nullptr);
// SMW variant (single-swap inverse updates; k_linalg.cu)
void launch_smw_update(const int* inst, int ninst, const double* Zall, long long m, long long blk_stride, int nstart,
                       const double* mu_all, const int* list_all, const int* seg_cnt_all,
                       int nseg, long long seg_len, int p, long long h, double* sinv_all, double* logdet,
                       int* smw_valid, cudaStream_t st);
void launch_smw_stage(const int* inst, int ninst, const double* mu_all, const double* sigma_all, int p,
                      double kappa_max, double* cstage, int cstride, double* sinv_all, int* smw_valid,
                      double* cond_out, int* status, cudaStream_t st);
// the whole C-step loop of short blocks (m <= 20480, p <= 16) in one CTA per instance (k_linalg.cu)
// 4096 < m <= 20480, p <= 16: the same loop on a cluster of 8 CTAs per instance (DSMEM couplings)
bool csteps_cluster_supported(long long m, int p);
void launch_csteps_cluster(const double* Zall, long long m, int p, long long blk_stride, int nstart, const int* inst,
                           int ninst, long long h, double kappa_max, int max_steps, double* mu_all, double* sigma_all,
                           int* status_all, int* steps_all, double* logdet_all, double* traj, int traj_stride,
                           uint8_t* mem_all, cudaStream_t st);
bool csteps_small_supported(long long m, int p);
void launch_csteps_small(const double* Zall, long long m, int p, long long blk_stride, int nstart, const int* inst,
                         int ninst, long long h, double kappa_max, int max_steps, double* mu_all, double* sigma_all,
                         int* status_all, int* steps_all, double* logdet_all, double* traj, int traj_stride,
                         uint8_t* mem_all, cudaStream_t st);
void launch_sums_to_cov(const int* inst, int ninst, const double* sums_all, int np, const double* shift_all, int p,
                        double n_given, double factor, double* mu_all, double* sigma_all, cudaStream_t st);
void launch_sums_to_second(const double* sums_all, int nb, int np, int p, double n, double* out_all, cudaStream_t st);
void launch_copy_vec(const int* inst, int ninst, const double* src, double* dst, int p, cudaStream_t st);
void launch_jacobi(const double* A_all, int nb, int p, double kappa_max, double* V_all, double* lam_all, int* ok_all,
                   cudaStream_t st);
void launch_vdv(const double* V_all, const double* d_all, int nb, int p, int which, double* out_all, cudaStream_t st);
void launch_matvec(const double* A_all, const double* x_all, int nb, int p, double* y_all, cudaStream_t st);
void launch_lr_cutoffs(const double* rs_all, int nb, long long m, double* AB, int* ok, cudaStream_t st);
void launch_aggregate(const double* mu_base, const double* sig_base, const int* ids, int nv, int p, double m,
                      double* mu_out, double* sig_out, int* kept, double* keys, double* scratch, cudaStream_t st);
void launch_pool_sums(const double* sums_all, int nb, int np, double* out, cudaStream_t st);
void launch_destandardize(const UniOut* uni, const double* mu_z, const double* sig_z, int p, double* mu_x,
                          double* sig_x, cudaStream_t st);

}  // namespace rtd
