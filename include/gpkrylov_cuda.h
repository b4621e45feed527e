/*
 * gpkrylov_cuda.h — C-ABI of the B200-native preconditioned mBCG hot path.
 *
 * Drop-in boundary for the reference's C++ kernel-operator / preconditioner /
 * solver interface (/root/reference/proj/include/gpkrylov).  Plain pointers and
 * sizes only.  All host matrices are fp64 COLUMN-MAJOR with an explicit leading
 * dimension, matching Eigen's default layout.  Host buffers are borrowed for
 * the duration of a synchronous call; device memory is owned by the opaque
 * context.  Entry points suffixed `_device` take device pointers (same layout)
 * and leave inputs resident in HBM.
 *
 * Error convention (common.hpp:19-35): every call returns a gpk_status; the
 * message (mirroring the reference's exception text) is in gpk_last_error().
 * A context is NOT thread-safe: one host thread drives it.
 */
#ifndef GPKRYLOV_CUDA_H
#define GPKRYLOV_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gpk_ctx gpk_ctx;

/* common.hpp:19-35 — status codes map 1:1 onto the reference's exception types. */
typedef enum {
  GPK_OK = 0,
  GPK_INPUT_ERROR = 1,     /* input_error      (CLI exit 1) */
  GPK_NUMERICAL_ERROR = 2, /* numerical_error  (CLI exit 2) */
  GPK_SOLVER_ERROR = 3,    /* solver_error : numerical_error */
  GPK_CUDA_ERROR = 4,      /* device failure, reported as numerical_error by the facade */
  GPK_NCCL_ERROR = 5
} gpk_status;

/* kernels.hpp:70-87 KernelFamily (RationalQuadratic is rejected: out of scope). */
typedef enum { GPK_RBF = 0, GPK_MATERN12 = 1, GPK_MATERN32 = 2, GPK_MATERN52 = 3, GPK_RATQUAD = 4 } gpk_family;

/* Arithmetic of the fused kernel MVM.  FP64: entries and accumulation in fp64.
 * FP32: fp32 entries (direct-difference distances, SFU exp) with fp32
 * accumulation per 32-column tile and fp64 accumulation across tiles; CG state
 * and all reductions stay fp64. */
typedef enum { GPK_PREC_FP64 = 0, GPK_PREC_FP32 = 1, GPK_PREC_TF32X3 = 2 } gpk_precision;
/* GPK_PREC_TF32X3: fp32 kernel entries as in FP32, contraction on the tcgen05 tensor
 * cores in split precision (a_hi b_hi + a_hi b_lo + a_lo b_hi, tf32 parts), fp32
 * accumulation in TMEM over 128 entries and fp64 across; derivative MVMs use FP32. */

/* Kernel-entry strategy of the tensor-core (GPK_PREC_TF32X3) value MVM.
 * DIRECT: fp32 direct-difference squared distances on the CUDA cores (any family).
 * GRAM: expanded distances |x_i|^2 + |x_j|^2 - 2 x_i.x_j (the reference's own
 *   column formula, kernels.hpp:235-243) with the cross term on the tensor cores
 *   (3xTF32) from mean-centred coordinates; near pairs (s <= (|x_i|^2+|x_j|^2)/16,
 *   where cancellation would dominate) recomputed by direct differences;
 *   RBF / Matern-3/2 / Matern-5/2, d <= 32.
 * AUTO (default): GRAM when eligible, d >= 6 and max |x~|^2 of the centred
 *   pre-scaled coordinates <= 4096, else DIRECT (tf32x3 d <= 4: direct differences on the same
 *   tcgen05 pipeline). */
typedef enum { GPK_MVM_AUTO = 0, GPK_MVM_DIRECT = 1, GPK_MVM_GRAM = 2 } gpk_mvm_variant;

/* krylov.hpp:15-24 CgConfig (+ GPU fields). */
typedef struct {
  int max_iters;        /* >= 1 */
  double rel_tol;       /* in (0,1): stop when ||P^-1 r_k|| <= rel_tol ||P^-1 b|| */
  int collect_tridiag;  /* record alpha/beta for the Lanczos tridiagonal */
  int precision;        /* gpk_precision of the operator inside the iterations */
  int refine;           /* FP32 only: fp64 true-residual audit + defect correction (max passes) */
} gpk_cg_cfg;

/* gp_likelihood.hpp:26-32 MllConfig (+ GPU fields). */
typedef struct {
  gpk_cg_cfg solver;
  int share_probes;    /* reuse the forward probe batch in the backward pass (reference default 1) */
  int with_gradient;   /* evaluate_mll's with_gradient flag */
  int backward_mode;   /* 0: fused bilinear derivative pass over the forward solves
                          1: reference-faithful: mBCG over the (d+1) l right-hand sides dK_w z_i
                          2: auto (default): fused when every forward solve converged, else faithful
                             (the fused identity needs converged probe solves)
                          3: fused + per-probe backward gammas s_i' dK_w z_i - z_i' P^-1 dP_w z_i
                             from (d+1) derivative MVMs of the probe block (no backward solves) */
} gpk_mll_cfg;

/* gp_likelihood.hpp:35-46 MllEvaluation, caller-allocated arrays. */
typedef struct {
  double value;                 /* mLL estimate */
  double* gradient;             /* d+2: outputscale, lengthscales, noise (log-space) */
  int solve_iterations;         /* iterations of the K_hat u = y solve */
  double* forward_gammas;       /* l (nullable) */
  double* backward_gammas;      /* (d+2) x l row-major by parameter (nullable; NaN where unavailable) */
  double value_sample_variance; /* unbiased variance of n*gamma_i */
  int* forward_cg_iterations;   /* l (nullable) */
  int total_cg_iterations;
  /* telemetry (not in the reference struct) */
  double logdet;                /* log det K_hat estimate */
  double logdet_precond;        /* log det P_hat */
  double quad;                  /* y^T u */
  int refine_passes;            /* fp64 defect-correction passes used */
  double max_true_rel_residual; /* fp64 audit (precision != FP64, refine > 0): max over ALL solve columns of
                                   ||P^-1(b - K_hat x)|| / ||P^-1 b||, capped columns included; -1 when not
                                   audited (FP64 mode, refine = 0, or no column converged: nothing to certify) */
  double seconds_solve, seconds_backward, seconds_total;
  long long kernel_entries;     /* kernel-matrix entries evaluated by the fused kernels */
  long long mvm_flops;          /* algorithmic fused-MVM flops */
  int gpu_launches;             /* kernels this library launched in the call */
  double max_cg_rel_residual;   /* max over solve columns of the CG recurrence's last ||P^-1 r_k|| / ||P^-1 b||
                                   (krylov.hpp:102-106; what the stopping rule saw, every precision) */
  int unconverged_columns;      /* solve columns that hit max_iters (converged = false, krylov.hpp:120) */
  int backward_mode_used;       /* 0 fused, 1 faithful (what backward_mode 2 resolved to) */
} gpk_mll_result;

/* ---- context ----------------------------------------------------------- */
gpk_status gpk_create(int device, gpk_ctx** out);
void gpk_destroy(gpk_ctx* ctx);
const char* gpk_last_error(const gpk_ctx* ctx);
/* Version / build string (sm_100a). */
const char* gpk_version(void);

/* ---- row sharding across GPUs (one process or host thread per rank) ------
 * A sharded context owns rows [r0, r1) of every n-length CG / probe array (X and
 * the preconditioner factors are replicated); each CG iteration all-gathers the
 * direction block and sums per-column dot products over ranks in rank order, so
 * results are bitwise reproducible for a given world size.  Host entry points
 * take full n-row buffers; each rank reads and writes back its own rows. */
#define GPK_NCCL_ID_BYTES 128
gpk_status gpk_nccl_unique_id(void* out /* GPK_NCCL_ID_BYTES */);
/* NCCL communicator over `world` ranks, one GPU each (rank 0 creates the id, broadcasts it). */
gpk_status gpk_create_sharded(int device, int rank, int world, const void* nccl_id, gpk_ctx** out);
/* In-process rank group: host-staged collectives, one host thread per rank (any devices). */
typedef struct gpk_group gpk_group;
gpk_status gpk_group_create(int world, gpk_group** out);
void gpk_group_destroy(gpk_group* g);
gpk_status gpk_create_in_group(int device, gpk_group* g, int rank, gpk_ctx** out);
/* Total rows n and input dimension d of the data set on ctx (GPK_INPUT_ERROR before gpk_set_data). */
gpk_status gpk_data_shape(const gpk_ctx* ctx, int64_t* n, int* d);
/* This rank's rows after gpk_set_data. */
gpk_status gpk_shard_rows(const gpk_ctx* ctx, int64_t* r0, int64_t* r1);

/* KernelOperator ctor data (kernels.hpp:159-173): X is n x d, column-major, ld >= n. */
gpk_status gpk_set_data(gpk_ctx* ctx, const double* X, int64_t n, int64_t d, int64_t ldx);
gpk_status gpk_set_data_device(gpk_ctx* ctx, const double* dX, int64_t n, int64_t d, int64_t ldx);
/* Hyperparameters (kernels.hpp:17-64), log space; log_ls has d entries. */
gpk_status gpk_set_params(gpk_ctx* ctx, int family, double ratquad_alpha, double log_outputscale,
                          const double* log_lengthscales, double log_noise);

/* ---- kernel operator (kernels.hpp:184-267) ------------------------------ */
/* out = (K + sigma^2 I) V, V n x t. */
gpk_status gpk_kernel_mvm(gpk_ctx* ctx, const double* V, int64_t ldv, int t, double* out, int64_t ldo,
                          int precision);
/* out = (d K_hat / d theta_which) V, raw parameter; which in [0, d+1]. */
gpk_status gpk_kernel_deriv_mvm(gpk_ctx* ctx, int which, const double* V, int64_t ldv, int t, double* out,
                                int64_t ldo, int precision);
/* Noise-free kernel column / derivative column (reference expanded-distance formula, fp64). */
gpk_status gpk_kernel_column(gpk_ctx* ctx, int64_t i, double* out);
gpk_status gpk_kernel_deriv_column(gpk_ctx* ctx, int which, int64_t i, double* out);

/* ---- preconditioner (preconditioners.hpp:82-295) ------------------------ */
/* P_hat = I (IdentityPreconditioner, common.hpp:59-70). */
gpk_status gpk_precond_identity(gpk_ctx* ctx);
/* Greedy pivoted partial Cholesky of K (preconditioners.hpp:236-264) in fp64, then the
 * DiagPlusLowRank factorisation with sigma^2 = noise (:84-95).  pivots: rank entries
 * (nullable); achieved: achieved rank; remaining_diag: n (nullable). */
gpk_status gpk_pivoted_cholesky(gpk_ctx* ctx, int rank, double diag_tol, double noise, int64_t* pivots,
                                int* achieved, double* remaining_diag);
/* Frozen-pivot dL/dtheta factors for every non-noise parameter (preconditioners.hpp:269-295). */
gpk_status gpk_precond_deriv_factors(gpk_ctx* ctx);
/* Copy-outs for parity: L (n x k), dL_which (n x k). */
gpk_status gpk_precond_factor(gpk_ctx* ctx, double* L, int64_t ldl);
gpk_status gpk_precond_deriv_factor(gpk_ctx* ctx, int which, double* dL, int64_t ldl);
/* out = P_hat^{-1} V (Woodbury, :114-118). */
gpk_status gpk_precond_solve(gpk_ctx* ctx, const double* V, int64_t ldv, int t, double* out, int64_t ldo);
gpk_status gpk_precond_logdet(gpk_ctx* ctx, double* out);
/* tr(P_hat^{-1} dP_hat/dtheta_which) (:138-145, :168). */
gpk_status gpk_precond_trace_inv_deriv(gpk_ctx* ctx, int which, double* out);

/* ---- solver (krylov.hpp:47-153) ------------------------------------------ */
/* Batched PCG over the t columns of B; every column follows pcg_solve exactly and
 * is independent of the others (batched_pcg contract).  alpha/beta/resid_hist are
 * max_iters x t column-major (column c = history of column c), nullable. */
gpk_status gpk_mbcg(gpk_ctx* ctx, const double* B, int64_t ldb, int t, const gpk_cg_cfg* cfg, double* X,
                    int64_t ldx, int* iters, int* converged, double* alpha, double* beta, double* resid_hist);

/* ---- likelihood (gp_likelihood.hpp:51-103) -------------------------------- */
/* One mLL (+ gradient) evaluation.  Z: n x l probe block (make_probes); probe_seed
 * is recorded and used for the unshared backward batch (mix_seed(seed, 0xb2d)). */
gpk_status gpk_evaluate_mll(gpk_ctx* ctx, const double* y, const double* Z, int64_t ldz, int l,
                            uint64_t probe_seed, const gpk_mll_cfg* cfg, gpk_mll_result* res);
gpk_status gpk_evaluate_mll_device(gpk_ctx* ctx, const double* dy, const double* dZ, int64_t ldz, int l,
                                   uint64_t probe_seed, const gpk_mll_cfg* cfg, gpk_mll_result* res);

/* ---- probes (trace_estimation.hpp:27-36, common.hpp:93-98) --------------- */
gpk_status gpk_make_probes(int64_t n, int count, uint64_t seed, double* out /* n x count col-major */);
/* The same stream generated on the device (bitwise the host one), into HBM on the context's
 * stream: the n x count block of an optimizer step (optimizer.hpp:452) never crosses PCIe. */
gpk_status gpk_make_probes_device(gpk_ctx* ctx, int64_t n, int count, uint64_t seed, double* d_out);
uint64_t gpk_mix_seed(uint64_t seed, uint64_t salt);

/* ---- callers of the hot path ------------------------------ */
/* mll_exact (gp_likelihood.hpp:124-146) on the device: dense fp64 K_hat, cuSOLVER Cholesky.
 * gradient: d+2 log-space components (nullable: value only, the validation / test metric of
 * optimizer.hpp:458-459 and experiments.hpp:377-380).  Unsharded contexts only. */
gpk_status gpk_mll_exact(gpk_ctx* ctx, const double* y, double* value, double* gradient);
/* out (na) = cross_kernel(spec, params, A, X) v (kernels.hpp:339-354); A is na x d column-major
 * (ld lda), v has n entries.  fp64. */
gpk_status gpk_cross_kernel_mvm(gpk_ctx* ctx, const double* A, int64_t na, int64_t lda, const double* v,
                                double* out);
/* Predictive mean of run_training_arm (experiments.hpp:403-414): alpha = pcg_solve(K_hat, y,
 * attached preconditioner, cfg), mean = cross_kernel(A, X) alpha.  iters nullable. */
gpk_status gpk_predict_mean(gpk_ctx* ctx, const double* y, const double* A, int64_t na, int64_t lda,
                            const gpk_cg_cfg* cfg, double* mean, int* iters);

/* ---- dataset ingestion -------------------------------
 * gpk_load_csv replaces load_csv (dataset.hpp:155-242) over read_csv_table
 * (csv.hpp:91-116): header row required, rows shuffled with mt19937_64(seed) +
 * uniform_int_distribution, split train / validation / test by llround(fraction * n),
 * optional standardisation with training-split population statistics.  Host code (no
 * device needed).  Errors: GPK_INPUT_ERROR with the reference's input_error text in err
 * (errlen bytes, nullable).  Splits are stored column-major fp64, as gpk_set_data takes. */
typedef struct gpk_dataset gpk_dataset;
typedef enum { GPK_SPLIT_TRAIN = 0, GPK_SPLIT_VALIDATION = 1, GPK_SPLIT_TEST = 2 } gpk_split;
gpk_status gpk_load_csv(const char* path, const char* target_column, int standardize, double train_fraction,
                        double validation_fraction, double test_fraction, uint64_t seed, gpk_dataset** out,
                        char* err, int64_t errlen);
void gpk_dataset_free(gpk_dataset* ds);
gpk_status gpk_dataset_shape(const gpk_dataset* ds, int split, int64_t* n, int* d);
/* X: n x d column-major (ld ldx >= n), y: n; either nullable */
gpk_status gpk_dataset_copy(const gpk_dataset* ds, int split, double* X, int64_t ldx, double* y);
/* Standardizer (dataset.hpp:87-101) statistics; identity (0 / 1) when not standardised */
gpk_status gpk_dataset_stats(const gpk_dataset* ds, int* standardized, double* feature_mean, double* feature_std,
                             double* target_mean, double* target_std);
/* column < 0: the target name; 0..d-1: feature names in file order (DataSplits::feature_names) */
const char* gpk_dataset_column_name(const gpk_dataset* ds, int column);
/* Standardizer::invert_x / invert_y in place (no-op when not standardised); X or y nullable */
gpk_status gpk_dataset_invert(const gpk_dataset* ds, double* X, int64_t n, int64_t ldx, double* y);

/* optimizer.hpp:22-43 OptMethod / OptOptions */
typedef enum { GPK_OPT_LBFGS = 0, GPK_OPT_ADAM = 1 } gpk_opt_method;
typedef struct {
  int method;              /* gpk_opt_method (default L-BFGS) */
  int max_steps;           /* 20 */
  int lbfgs_memory;        /* 10 */
  double armijo_c1;        /* 1e-4 */
  double wolfe_c2;         /* 0.9 */
  double adam_lr;          /* 0.1 */
  int early_stop_patience; /* 3 */
  double grad_tol;         /* 1e-8 */
  int max_line_search;     /* 20 */
} gpk_opt_options;

/* Why the minimizer stopped (MinimizeResult.message, optimizer.hpp:236-298). */
typedef enum {
  GPK_OPT_MAX_STEPS = 0,         /* "" (ran max_steps) */
  GPK_OPT_GRAD_TOL = 1,          /* "gradient norm below tolerance" */
  GPK_OPT_LINE_SEARCH_FAILED = 2,/* "line search failed after bounded bisection; step rejected" */
  GPK_OPT_STOPPED = 3            /* "stopped by callback" (early stopping on the validation proxy) */
} gpk_opt_stop;

/* OptimizeResult (optimizer.hpp:356-361) + MinimizeResult (:205-211) + OptTrace (:45-72).
 * Arrays are caller-allocated and nullable; step arrays hold max_steps rows. */
typedef struct {
  double* best_log_params;       /* d+2: best (o, l_1..l_d, sigma^2), log space */
  double best_validation;        /* +inf without validation data */
  double final_train_neg_mll_per_point;
  double final_objective;        /* MinimizeResult.f */
  int minimizer_steps;           /* MinimizeResult.steps */
  int converged;
  int stop_reason;               /* gpk_opt_stop */
  int n_steps;                   /* OptTrace.steps.size() */
  double* step_theta;            /* max_steps x np_opt, row per step; np_opt = ard ? d+2 : 3 */
  double* step_objective;
  double* step_validation;
  double* step_wall_time;
  double* step_length;
  double* step_f_before;
  double* step_dir_derivative_before;
  double* step_dir_derivative_after;
  int* step_accepted;
  long long* step_evaluations;   /* model_evaluations_cumulative */
  int eval_capacity;             /* rows of the eval_* arrays */
  int n_evaluations;             /* OptTrace.evaluations.size() (rows beyond eval_capacity are dropped) */
  int* eval_step;
  double* eval_f;
  double* eval_grad_norm;
  long long total_cg_iterations; /* telemetry: CG iterations over every objective evaluation */
  double seconds_total;
} gpk_opt_result;

/* optimize() (optimizer.hpp:404-505) on the device path: L-BFGS (strong-Wolfe line search) or
 * Adam on the negative mLL in log space; at every step start the preconditioner is rebuilt at
 * the current iterate (precond_rank < 0: IdentityPreconditioner; >= 0: pivoted Cholesky of that
 * rank + derivative factors, experiments.hpp:30-68) and the probes are redrawn with
 * mix_seed(seed, step); trial points of the line search reuse both.  Unevaluable iterates read
 * as +inf.  train: context with the training X (gpk_set_data); validation: context with the
 * validation X or NULL (no early stopping).  dense_limit: validation / final metrics use the
 * dense mll_exact for sets of at most this size (the reference's Dense/MatrixFree switch). */
gpk_status gpk_optimize(gpk_ctx* train, const double* y, gpk_ctx* validation, const double* y_val, int family,
                        int ard, const double* init_log_params, int precond_rank, double diag_tol,
                        int probe_count, const gpk_opt_options* opts, const gpk_mll_cfg* mll_cfg, uint64_t seed,
                        int64_t dense_limit, gpk_opt_result* res);

/* Select the tensor-core MVM variant (takes effect at the next call). */
gpk_status gpk_set_mvm_variant(gpk_ctx* ctx, int variant);
/* The variant the current data/params use (DIRECT or GRAM) and max |x~|^2 of the centred coordinates. */
gpk_status gpk_get_mvm_variant(gpk_ctx* ctx, int* variant, double* max_sqnorm);

/* Number of this library's kernels launched on ctx since creation. */
long long gpk_launch_count(const gpk_ctx* ctx);

/* The CUDA stream (cudaStream_t) all of ctx's work is issued on. */
void* gpk_stream(const gpk_ctx* ctx);

/* Live per-launch timing of the two dominant kernels with CUDA events on ctx's
 * stream (off by default).  kind 0: fused kernel MVM (reduced precision), 1: fused
 * derivative pass, 2: fp64 kernel MVM (parity mode / certified residual), 3: the fused
 * single-rank CG vector phase (alpha, x/r update + Woodbury, beta, p update; its "flops"
 * field holds algorithmic HBM bytes).
 * Returns accumulated device milliseconds, launch count and algorithmic flops /
 * kernel entries since the last reset.  on: 0 off, 1 kinds 0 and 1, otherwise a bitmask of
 * kinds (bit k = kind k; each recorded launch costs two event records on the stream). */
gpk_status gpk_profile_enable(gpk_ctx* ctx, int on);
gpk_status gpk_profile_read(gpk_ctx* ctx, int kind, double* ms, long long* launches, double* flops, double* entries);
gpk_status gpk_profile_reset(gpk_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* GPKRYLOV_CUDA_H */
