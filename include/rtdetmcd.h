/* rtdetmcd.h — C ABI of the B200-native RT-DetMCD hot path (libpaper_1910_05615_b200.so).
 *
 * Method: "Real-time outlier detection for large datasets by RT-DetMCD",
 * De Ketelaere, Hubert, Raymaekers, Rousseeuw, Vranckx (arXiv 1910.05615),
 * cited as PAPER.md:<line> (section / equation).
 *
 * Conventions (all entry points)
 *   - All floating point is IEEE binary64.  A data matrix X is n x p ROW-MAJOR
 *     (row = observation), 1 <= p <= 40,
 *     n > 2p.
 *   - Pointers marked [dev|host] may be device memory (cudaMalloc / torch CUDA
 *     tensor) or host memory (pageable or pinned); the library inspects each
 *     with cudaPointerGetAttributes and copies host buffers itself.  Pointers
 *     marked [host] must be host memory; [dev] must be device memory.
 *   - Ownership: the caller owns every input and output buffer.  Inputs are
 *     read-only.  No pointer is retained after a call returns.  The context
 *     owns a grow-only device workspace (or uses one handed over with
 *     rtdetmcd_set_workspace) and its CUDA stream.
 *   - Synchrony: every call enqueues its work on the context stream and
 *     returns after it completed; results are valid on return.  A context is
 *     not re-entrant (one context per thread / per rank).
 *   - Errors: a call returns a non-zero rtdetmcd_status and stores a message
 *     retrievable with rtdetmcd_last_error(); output buffers are then
 *     unspecified.  The library never calls exit/abort and never throws
 *     across the ABI.  RTD_E_CUDA means a CUDA runtime error (message names
 *     the call); the context should then be destroyed.
 */
#ifndef RTDETMCD_H
#define RTDETMCD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RTDETMCD_ABI_VERSION 3

typedef struct rtdetmcd_ctx rtdetmcd_ctx;

typedef enum {
  RTD_OK = 0,
  RTD_E_INVALID_ARG = 1,          /* sizes / options violate the preconditions below */
  RTD_E_NONFINITE = 2,            /* a NaN/Inf entry (or x <= 0 with log_transform); message names the row */
  RTD_E_DEGENERATE_COLUMN = 3,    /* univariate MCD scale is zero for a column */
  RTD_E_BOTH_STARTS_FAILED = 4,   /* q = 1: both initial estimators were dropped */
  RTD_E_TOO_FEW_VALID_BLOCKS = 5, /* q > 1: more than floor(q/2) blocks failed */
  RTD_E_NOT_PD = 6,               /* a scatter matrix that must be positive definite is not */
  RTD_E_CUDA = 7,
  RTD_E_OOM = 8,
  RTD_E_INTERNAL = 9,
  RTD_E_NCCL = 10                 /* an inter-rank exchange failed (NCCL error, or a transport callback returned != 0) */
} rtdetmcd_status;

enum { RTD_PART_PERMUTE = 0, RTD_PART_CONTIGUOUS = 1 };
/* C-step distances (the "D" of the paper's Table 1): by the Cholesky factor
 * (§3.4, default) or by the explicit inverse (variant I; needs p >= 8), or by the
 * explicit inverse kept up to date by Sherman-Morrison-Woodbury on the C-steps that interchange
 * exactly two cases (the inverse and the determinant updated directly; every other
 * step recomputes them; needs p >= 8) */
enum { RTD_DIST_CHOLESKY = 0, RTD_DIST_INVERSE = 1, RTD_DIST_SMW = 2 };
/* consistency factor of the raw scatter: c(alpha) of Croux-Haesbroeck as the text defines it
 * (default) or the median rule -- the h-subset covariance times
 * median_i d_i^2 / chi2_{p,0.5} over the rows of the block -- with which the paper's Table 2 KL
 * values are reproduced (DESIGN.md finding F1) */
enum { RTD_CONS_ALPHA = 0, RTD_CONS_MEDIAN = 1 };

/* warning bits of rtdetmcd_result.warnings (non-fatal) */
enum {
  RTD_W_H_BELOW_BOUND = 1,  /* h < [(n+p+1)/2]; accepted since h > p */
  RTD_W_MAX_CSTEPS = 2,     /* a chosen start hit max_csteps before H_new == H_old */
  RTD_W_BLOCK_FAILED = 4,   /* q > 1: at least one block had both starts dropped */
  RTD_W_START_FAILED = 8    /* at least one start was dropped (ill-conditioned / singular) */
};

typedef struct {
  int64_t h;             /* > 0: explicit coverage, p < h <= n; 0: h = floor(alpha * n) */
  double alpha;          /* used iff h == 0; default 0.5 */
  int32_t shards;        /* q >= 1 blocks; 0: q = max(floor(n/(p omega)), 1) capped by shard_cap
                            (eq. partitionsize) */
  int32_t shard_cap;     /* cap for the q rule; default 64 */
  int64_t omega;         /* minimum observations per dimension per block; default 4096 */
  double kappa_max;      /* condition threshold; default 1000 */
  double quantile;       /* cut-off quantile; default 0.975 */
  int32_t max_csteps;    /* C-step cap per start; default 100 */
  int32_t refresh_every; /* update-based C-steps: full recompute of the sums every this many steps; default 32;
                            1 = plain recompute every step (variants I / ID of Table 1) */
  uint64_t seed;         /* key of the random partition */
  int32_t partition;     /* RTD_PART_PERMUTE (keyed Feistel permutation, default) | RTD_PART_CONTIGUOUS */
  int32_t log_transform; /* 1: fit ln(x) (x must be > 0), as in BASELINE config 5 */
  int32_t distance;      /* RTD_DIST_CHOLESKY (default) | RTD_DIST_INVERSE (ablation variant I) | RTD_DIST_SMW */
  int32_t consistency;   /* RTD_CONS_ALPHA (default) | RTD_CONS_MEDIAN */
} rtdetmcd_opts;

/* Fills *o with the defaults above. */
void rtdetmcd_opts_default(rtdetmcd_opts* o);

typedef struct {
  /* [host] caller-allocated, nullable; ORIGINAL units of X (de-standardised, after ln when log_transform) */
  double* loc;        /* p: univariate reweighted MCD location per column */
  double* scale;      /* p: univariate reweighted MCD scale per column */
  double* mu_raw;     /* p: raw MCD centre (pooled when q > 1) */
  double* sigma_raw;  /* p*p row-major: c(alpha)-scaled raw scatter */
  double* mu_rew;     /* p: reweighted centre */
  double* sigma_rew;  /* p*p: reweighted scatter, scaled by c(0.975, p) */
  /* scalars written by the library */
  double logdet_raw;  /* log det of the unscaled raw scatter of the chosen start (q = 1), standardised units */
  double cutoff2;     /* chi2_{p, quantile}: a row is flagged iff RD^2 > cutoff2 */
  int64_t h;          /* coverage used */
  int64_t h_block;    /* per-block coverage floor(h m / n) */
  int64_t m;          /* rows per block floor(n/q) */
  int32_t q_used;
  int32_t warnings;   /* RTD_W_* bits */
  int32_t n_valid_blocks;
  int32_t n_kept_blocks;
  int64_t n_weighted; /* rows with weight 1 in the reweighting */
  /* [host] nullable per-block diagnostics, sized q (block_chosen) or 2q (per (block, start)) */
  int32_t* block_chosen;  /* 0 = wrapping start, 1 = GSSCM start, -1 = block failed */
  int32_t* start_steps;   /* C-steps run (distance passes) per (block, start) */
  int32_t* start_status;  /* 1 converged, 2 not PD, 3 condition >= kappa_max, 4 max steps, 5 refinement dropped,
                             6 skipped (warm start) */
  double* start_logdet;   /* log det of the converged unscaled scatter per (block, start) */
  /* [dev|host] nullable, sized n, in ORIGINAL row order */
  uint8_t* flags;    /* 1 iff RD^2 > cutoff2 under (mu_rew, sigma_rew) */
  double* rd2;       /* final squared robust distance */
  uint8_t* weights;  /* reweighting weight (0 for rows discarded by the partition) */
  uint8_t* hsubset;  /* 1 iff the row is in its block's chosen h-subset */
} rtdetmcd_result;

/* Create a context on CUDA device `device`.  cuda_stream: a cudaStream_t to
 * enqueue on (e.g. torch.cuda.current_stream().cuda_stream) or NULL for a
 * private stream. */
rtdetmcd_status rtdetmcd_create(rtdetmcd_ctx** ctx, int device, void* cuda_stream);
void rtdetmcd_destroy(rtdetmcd_ctx* ctx);
const char* rtdetmcd_last_error(const rtdetmcd_ctx* ctx);

/* Hand over a caller-owned device buffer as workspace (e.g. a torch uint8
 * tensor).  bytes must be >= rtdetmcd_fit_workspace_size(); the context then
 * never allocates device memory itself.  dev_ptr = NULL reverts to the
 * context's own grow-only allocation. */
rtdetmcd_status rtdetmcd_set_workspace(rtdetmcd_ctx* ctx, void* dev_ptr, size_t bytes);
size_t rtdetmcd_fit_workspace_size(int64_t n, int32_t p, const rtdetmcd_opts* opts);

/* The whole RT-DetMCD fit (serial IDC for q = 1, parallel IDCP_q for q > 1,
 * PAPER.md:1076-1100) followed by the flag pass over all n rows:
 *   standardise (§3.1) -> [partition, §4] -> S~1, S~2 (§3.2) -> refinement (§3.3)
 *   -> C-steps with Cholesky distances and update-based sums (§3.4-3.5)
 *   -> lowest-determinant start -> [median / KL / pooling, §4 steps 5-7]
 *   -> reweighting (§2.1, §4 steps 8-9) -> flagging (§4 step 10).
 * X [dev|host]: n x p row-major.  out: any nullable field may be NULL. */
rtdetmcd_status rtdetmcd_fit(rtdetmcd_ctx* ctx, const double* X, int64_t n, int32_t p, const rtdetmcd_opts* opts,
                             rtdetmcd_result* out);

/* Warm start (the closing note of §4): the same fit, but every block's
 * C-steps (step 3 of §4) start from (mu0, sigma0) -- typically the previous run's reweighted
 * estimate (mu_rew, sigma_rew) -- instead of from the two refined initial estimators (steps 1-2,
 * which are skipped).  mu0 [host] p, sigma0 [host] p*p row-major, in the units the fit reports
 * (ORIGINAL units of X, after ln when opts->log_transform); they are re-expressed in this run's
 * standardisation.  A warm start the C-step cannot take (not positive definite, or 1-norm
 * condition >= kappa_max) drops the block (q = 1: RTD_E_BOTH_STARTS_FAILED).  In the result,
 * block_chosen = 0 and the (block, 1) entries are unused (start_status 6 = skipped). */
rtdetmcd_status rtdetmcd_fit_warm(rtdetmcd_ctx* ctx, const double* X, int64_t n, int32_t p, const rtdetmcd_opts* opts,
                                  const double* mu0, const double* sigma0, rtdetmcd_result* out);

/* nb independent fits of the same shape and options over a sequence of HOST batches (a stream of
 * data sets, e.g. successive windows of a production line; PAPER.md:1038-1043 motivates the
 * real-time setting).  X[b] [host, pinned for full overlap]: n x p row-major.  Each batch is the
 * exact rtdetmcd_fit of X[b] (out[b] filled as there); the library copies batch b+1 to the device
 * on its own non-blocking copy stream while batch b is fitted, into two ctx-owned device buffers
 * (2 n p 8 bytes, grow-only), so the host->device transfer overlaps the compute.  Stops at the
 * first failing batch (its status is returned; later out[] are untouched).  out may be NULL. */
rtdetmcd_status rtdetmcd_fit_batches(rtdetmcd_ctx* ctx, const double* const* X, int32_t nb, int64_t n, int32_t p,
                                     const rtdetmcd_opts* opts, rtdetmcd_result* out);

/* Step 10 on its own (the paper's 8.4 ms "flagging" figure,
 * PAPER.md:1624-1627): rd2_i = (x_i - mu)^T sigma^-1 (x_i - mu) by a Cholesky
 * solve, flags_i = rd2_i > chi2_{p, quantile}.
 * X [dev|host] n x p row-major (ln applied first when log_transform);
 * mu [host] p; sigma [host] p*p row-major SPD (RTD_E_NOT_PD otherwise);
 * flags, rd2 [dev|host] n, either may be NULL. */
rtdetmcd_status rtdetmcd_flag(rtdetmcd_ctx* ctx, const double* X, int64_t n, int32_t p, const double* mu,
                              const double* sigma, double quantile, int32_t log_transform, uint8_t* flags,
                              double* rd2);

/* ---- the sharded fit: one process (rank) per GPU, rows sharded over the ranks ----
 *
 * The paper's parallel scheme (§4 steps 1-10) with the blocks spread over ranks:
 *   C2  the global standardisation needs every row of a column: columns are
 *       exchanged all-to-all, the owner of column j runs its univariate MCD over all n_global rows,
 *       the (loc, scale) records are all-gathered;
 *   --  every rank fits its own blocks (steps 1-4);
 *   C4  block records are all-gathered and every rank runs the same deterministic median / KL
 *       ranking / pooling (steps 5-7; the paper's master thread);
 *   C5  per-block reweighting sums are all-gathered and pooled in block order (steps 8-9,
 *       PAPER.md:975-995, the union of the fitted rows);
 *   --  every rank flags its own rows (step 10).
 * Every fold is a fixed-order fold by block id (never a float all-reduce), so the result is
 * bit-identical to rtdetmcd_fit with shards = q and RTD_PART_CONTIGUOUS on the concatenated rows,
 * at every world size.
 *
 * Row layout (rtdetmcd_shard_layout): q blocks of m = floor(n_global / q) consecutive rows; rank r
 * holds blocks [r q/world, (r+1) q/world) (q a multiple of world), i.e. global rows
 * [row0, row0 + n_local); the last rank also holds the n_global - q m remainder rows, which are
 * flagged but not fitted (reading R23).  The partition is the contiguous one: opts->partition must
 * be RTD_PART_CONTIGUOUS when world > 1 (RTD_E_INVALID_ARG otherwise).
 *
 * Collective: every rank calls rtdetmcd_fit_sharded with the same n_global, p and options (checked:
 * RTD_E_INVALID_ARG on every rank on a mismatch) and its own X_local.  An error detected on one rank
 * (bad rows, a failed block) is agreed on by all ranks before they leave, so no rank is left waiting in
 * a collective; RTD_E_NCCL on a failed exchange (the ranks' states are then undefined: destroy). */

/* Transport callbacks on HOST buffers (an alternative to NCCL, e.g. gloo or MPI, or ranks as threads).
 * Both are collective; return 0 on success. */
typedef struct {
  void* user;
  /* every rank contributes `bytes` bytes at send; recv (world * bytes) receives them in rank order */
  int32_t (*allgather)(void* user, const void* send, void* recv, size_t bytes);
  /* send_bytes[s] bytes at send + send_offs[s] go to rank s; recv_bytes[s] bytes from rank s land at
   * recv + recv_offs[s] (s = 0..world-1, including the rank itself) */
  int32_t (*alltoallv)(void* user, const void* send, const size_t* send_bytes, const size_t* send_offs, void* recv,
                       const size_t* recv_bytes, const size_t* recv_offs);
} rtdetmcd_transport;

/* 128-byte NCCL unique id (ncclGetUniqueId): created on one rank, shared by the caller (e.g. a
 * torch.distributed broadcast), passed to rtdetmcd_create_dist on every rank.  libnccl.so.2 is
 * loaded at run time (the copy already in the process, else the system one); RTD_E_NCCL if absent. */
rtdetmcd_status rtdetmcd_nccl_unique_id(void* id_out);
/* A context on `device` that is rank `rank` of `world` over NCCL (collective: all ranks call it).
 * nccl_unique_id NULL requires world == 1 (no communicator).  The NCCL communicator is owned by the
 * context and destroyed with it; collectives are enqueued on the context stream. */
rtdetmcd_status rtdetmcd_create_dist(rtdetmcd_ctx** ctx, int device, void* cuda_stream, const void* nccl_unique_id,
                                     int rank, int world);
/* The same with caller callbacks (copied; `user` must outlive the context). */
rtdetmcd_status rtdetmcd_create_transport(rtdetmcd_ctx** ctx, int device, void* cuda_stream,
                                          const rtdetmcd_transport* transport, int rank, int world);
/* Rows of rank `rank` (host-only arithmetic, no GPU): q blocks over world ranks as above.  Returns 0,
 * or RTD_E_INVALID_ARG when q is not a positive multiple of world or n_global < q. */
rtdetmcd_status rtdetmcd_shard_layout(int64_t n_global, int32_t q, int32_t world, int32_t rank, int64_t* row0,
                                      int64_t* n_local, int32_t* block0, int32_t* q_local);
/* The sharded fit + flag (collective).  X_local [dev|host]: this rank's n_local x p rows (row-major,
 * global rows [row0, row0 + n_local)).  q = opts->shards (a multiple of world; 0: the rule of
 * eq. partitionsize, rounded down to a multiple of world, at least world).  h = opts->h or
 * floor(alpha n_global) over ALL rows; block coverage floor(h m / n_global).
 * out: loc .. sigma_rew, scalars and the per-block arrays (sized q / 2q) are GLOBAL and identical on
 * every rank; flags, rd2, weights, hsubset are this rank's n_local rows.  A context made by
 * rtdetmcd_create (no communicator) runs it as world 1. */
rtdetmcd_status rtdetmcd_fit_sharded(rtdetmcd_ctx* ctx, const double* X_local, int64_t n_local, int64_t n_global,
                                     int32_t p, const rtdetmcd_opts* opts, rtdetmcd_result* out);
/* rank / world / transport kind ("none", "nccl", "host") of a context */
rtdetmcd_status rtdetmcd_ctx_comm(const rtdetmcd_ctx* ctx, int32_t* rank, int32_t* world, const char** kind);

/* ---- stage entry points: the same kernels, exposed for intermediate parity
 * checks and as building blocks of the multi-process driver ---- */

/* Univariate reweighted MCD with h~ = floor(len/2)+1 of
 * ncols columns.  cols [dev] column-major (column j at cols + j*len).
 * Outputs [host] sized ncols, nullable: reweighted loc/scale, raw window mean
 * and raw variance SQ/(h~-1) (no factor), window start in the sorted column.
 * RTD_E_DEGENERATE_COLUMN if a scale is zero (message names the column). */
rtdetmcd_status rtdetmcd_unimcd(rtdetmcd_ctx* ctx, const double* cols, int64_t len, int32_t ncols, double* loc,
                                double* scale, double* raw_loc, double* raw_var, int64_t* start);

/* S~1 (wrapped covariance) and S~2 (LR-GSSCM)
 * of a standardised block.  Z [dev] column-major m x p (column k at Z + k*m).
 * S1, S2 [host] p*p row-major.  *s2_ok = 0 when the norms have zero IQR. */
rtdetmcd_status rtdetmcd_initial(rtdetmcd_ctx* ctx, const double* Z, int64_t m, int32_t p, double* S1, double* S2,
                                 int32_t* s2_ok);

/* Refinement of an initial scatter S.  Z as above, S [host]
 * p*p.  Outputs [host]: mu (p), sigma (p*p), eigenvalues lam (p, nullable);
 * *ok = 0 when the start is dropped (lambda_p <= 0, lambda_1/lambda_p > kappa_max,
 * or a degenerate univariate scale). */
rtdetmcd_status rtdetmcd_refine(rtdetmcd_ctx* ctx, const double* Z, int64_t m, int32_t p, const double* S,
                                double kappa_max, double* mu, double* sigma, double* lam, int32_t* ok);

/* C-steps to convergence from (mu0, sigma0).
 * Z as above; mu0, sigma0 [host].  Outputs [host]: mu, sigma (unscaled
 * covariance of the final h-subset), logdet, steps, status (1 converged,
 * 2 not PD, 3 condition >= kappa_max, 4 max steps).  hsubset [dev|host] m
 * bytes, nullable.  logdet_traj [host] nullable, max_steps+1 entries:
 * log det of the scatter entering C-step s (s = 1..steps). */
rtdetmcd_status rtdetmcd_csteps(rtdetmcd_ctx* ctx, const double* Z, int64_t m, int32_t p, int64_t h,
                                const double* mu0, const double* sigma0, double kappa_max, int32_t max_steps,
                                int32_t refresh_every, double* mu, double* sigma, double* logdet, int32_t* steps,
                                int32_t* status, uint8_t* hsubset, double* logdet_traj);

/* Per-kernel-class timing (for bench.py's roofline).  on != 0 enables it and
 * clears the counters: every later call records a CUDA event pair on the
 * context stream around each timed kernel class ("dist" = the C-step /
 * reweight distance pass, "select", "moments_dense", "moments_delta",
 * "unimcd", "matmul", "initial", "flag", ...).  Entries accumulate the
 * device time (ms), the launch count, the ALGORITHMIC HBM bytes of those
 * launches, their algorithmic flops (0 where not meaningful) and, for the
 * distance pass, the bytes the paper's per-start C-steps would stream
 * (rows * starts * (8p + 8); the fused pass reads a block once for both
 * starts).  name [host] receives up to name_len-1 characters; every output
 * pointer is nullable. */
rtdetmcd_status rtdetmcd_set_profiling(rtdetmcd_ctx* ctx, int32_t on);
/* Process-wide counters: hand-written kernel launches and CUB radix-sort
 * invocations issued by this library so far (host pointers, nullable). */
void rtdetmcd_counters(int64_t* kernels, int64_t* sorts);
int32_t rtdetmcd_prof_count(const rtdetmcd_ctx* ctx);
rtdetmcd_status rtdetmcd_prof_entry(const rtdetmcd_ctx* ctx, int32_t i, char* name, size_t name_len, double* ms_total,
                                    int64_t* launches, double* bytes_total, double* flops_total,
                                    double* eff_bytes_total);

/* ---- distributed stages (the building blocks rtdetmcd_fit_sharded runs internally, exposed for
 * callers that move the data between ranks themselves).  Blocks are contiguous row
 * ranges; rank r holds blocks [r q/G, (r+1) q/G).  Sequence per rank:
 *   rtdetmcd_columns -> (exchange columns) -> rtdetmcd_unimcd on owned columns
 *   -> (all-gather loc/scale) -> rtdetmcd_blocks_fit -> (all-gather records)
 *   -> rtdetmcd_aggregate -> rtdetmcd_blocks_reweight -> (all-gather sums)
 *   -> rtdetmcd_pool_reweight -> rtdetmcd_flag on the local rows.
 * The results equal rtdetmcd_fit with shards = q and RTD_PART_CONTIGUOUS on
 * the concatenated rows (§4 steps 1-10).
 * rtdetmcd_blocks_fit opens a session held by the context; aggregate,
 * blocks_reweight and pool_reweight use it; any other call closes it. */

/* record layout written by rtdetmcd_blocks_fit, per block, in doubles:
 * [valid, chosen start, log det (unscaled), C-steps, mu (p), c(alpha)-scaled Sigma (p*p)] (standardised units) */
#define RTDETMCD_RECORD_DOUBLES(p) (4 + (p) + (p) * (p))
/* doubles per block of reweighting sums: p (S1) + p(p+1)/2 (S2, packed lower) + 1 (count) */
int32_t rtdetmcd_moment_doubles(int32_t p);

/* H0 alone: X [dev|host] n x p row-major -> Xc [dev] p x n column-major
 * (validated; ln applied when log_transform).  RTD_E_NONFINITE names the row. */
rtdetmcd_status rtdetmcd_columns(rtdetmcd_ctx* ctx, const double* X, int64_t n, int32_t p, int32_t log_transform,
                                 double* Xc);
/* Fit q_local contiguous blocks of m = n_local / q_local rows of X_local
 * [dev|host] with the GLOBAL standardisation loc/scale [host p] and block
 * coverage h_block (= floor(h m / n)).  records [host] q_local records.
 * q_global sizes the aggregation buffers of the session. */
rtdetmcd_status rtdetmcd_blocks_fit(rtdetmcd_ctx* ctx, const double* X_local, int64_t n_local, int32_t p,
                                    const double* loc, const double* scale, int32_t q_local, int32_t q_global,
                                    int64_t h_block, const rtdetmcd_opts* opts, double* records);
/* Entrywise median, KL ranking, ceil(q_valid/2) kept, pooling of the q_global
 * records [host] of all ranks (block order) -> raw fit [host] in standardised
 * units; identical on every rank. */
rtdetmcd_status rtdetmcd_aggregate(rtdetmcd_ctx* ctx, int32_t q, int32_t p, int64_t m, const double* records,
                                   double* mu_raw, double* sigma_raw, int32_t* n_kept);
/* Reweighting sums of the session's blocks about mu_raw -> sums [host]
 * q_local * rtdetmcd_moment_doubles(p); weights [dev|host] n_local, nullable. */
rtdetmcd_status rtdetmcd_blocks_reweight(rtdetmcd_ctx* ctx, double quantile, double* sums, uint8_t* weights);
/* Pool the q_global blocks' sums [host] (block order) -> raw and reweighted
 * fits in ORIGINAL units [host]; n_weighted [host] nullable. */
rtdetmcd_status rtdetmcd_pool_reweight(rtdetmcd_ctx* ctx, int32_t q, const double* sums, double quantile,
                                       double* mu_raw, double* sigma_raw, double* mu_rew, double* sigma_rew,
                                       int64_t* n_weighted);

/* Host numerics used by the fit, exported for checking. */
double rtdetmcd_chi2_quantile(double prob, int32_t dof);
double rtdetmcd_consistency_factor(double alpha, int32_t p);
int32_t rtdetmcd_choose_q(int64_t n, int32_t p, int64_t omega, int32_t cap); /* eq. partitionsize */
/* pi(i) of the keyed Feistel partition permutation (reading R13), for i in [0, n). out [host] n. */
rtdetmcd_status rtdetmcd_partition_perm(rtdetmcd_ctx* ctx, int64_t n, uint64_t seed, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* RTDETMCD_H */
