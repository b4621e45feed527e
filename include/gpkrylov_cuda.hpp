// gpkrylov_cuda.hpp — header-only C++17 facade over the C-ABI (gpkrylov_cuda.h)
// with the reference's names (/root/reference/proj/include/gpkrylov):
//
//   gpkrylov::cuda::KernelOperator     ~ gpkrylov::KernelOperator   (kernels.hpp:157-336)
//   gpkrylov::cuda::DiagPlusLowRank    ~ gpkrylov::DiagPlusLowRank  (preconditioners.hpp:82-186)
//   gpkrylov::cuda::pivoted_cholesky_with_derivatives                (preconditioners.hpp:299-305)
//   gpkrylov::cuda::pcg_solve / batched_pcg                          (krylov.hpp:47-153)
//   gpkrylov::cuda::evaluate_mll                                     (gp_likelihood.hpp:51-103)
//
// Errors are thrown as input_error / numerical_error / solver_error with the
// library's message (common.hpp:19-35).  Buffers are std::vector<double>,
// column-major; when Eigen is available (the reference's own build), Eigen
// overloads with the reference signatures are enabled so optimize() and
// run_bias_variance() compile against the facade unchanged.
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "gpkrylov_cuda.h"

#if __has_include(<Eigen/Dense>)
#include <Eigen/Dense>
#define GPKRYLOV_CUDA_EIGEN 1
#endif

namespace gpkrylov {
namespace cuda {

struct input_error : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct numerical_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct solver_error : numerical_error {
  using numerical_error::numerical_error;
};

inline void check(gpk_status s, const gpk_ctx* c) {
  if (s == GPK_OK) return;
  const std::string m = c ? gpk_last_error(c) : "gpkrylov_cuda error";
  if (s == GPK_INPUT_ERROR) throw input_error(m);
  if (s == GPK_SOLVER_ERROR) throw solver_error(m);
  throw numerical_error(m);
}

enum class KernelFamily { RBF = GPK_RBF, Matern12 = GPK_MATERN12, Matern32 = GPK_MATERN32, Matern52 = GPK_MATERN52 };

struct Hyperparameters {  // kernels.hpp:17-64 (log space)
  double log_outputscale = 0.0;
  std::vector<double> log_lengthscales;
  double log_noise = -4.605170185988091;  // log(1e-2)
};

struct CgConfig {  // krylov.hpp:15-24 (+ GPU fields)
  int max_iters = 100;
  double rel_tol = 1e-6;
  bool collect_tridiag = false;
  gpk_precision precision = GPK_PREC_TF32X3;
  int refine = 2;
  gpk_cg_cfg c() const { return gpk_cg_cfg{max_iters, rel_tol, collect_tridiag ? 1 : 0, precision, refine}; }
};

struct MllConfig {  // gp_likelihood.hpp:26-32
  CgConfig solver;
  bool share_probes = true;
  int backward_mode = 2;  // 0 fused derivative pass, 1 reference-faithful per-RHS solves, 2 auto
};

struct MllEvaluation {  // gp_likelihood.hpp:35-46
  double value = 0.0;
  std::vector<double> gradient;
  int solve_iterations = 0;
  std::vector<double> forward_gammas;
  std::vector<std::vector<double>> backward_gammas;
  std::uint64_t probe_seed = 0;
  double value_sample_variance = 0.0;
  std::vector<int> forward_cg_iterations;
  int total_cg_iterations = 0;
  double logdet = 0.0;
};

struct ProbeBatch {  // trace_estimation.hpp:20-25
  std::vector<double> probes;  // n x count, column-major
  std::uint64_t seed = 0;
  int count = 0;
};

inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t salt) { return gpk_mix_seed(seed, salt); }

inline ProbeBatch make_probes(std::int64_t n, int count, std::uint64_t seed) {
  ProbeBatch b;
  b.probes.resize(static_cast<size_t>(n) * count);
  check(gpk_make_probes(n, count, seed, b.probes.data()), nullptr);
  b.seed = seed;
  b.count = count;
  return b;
}

// Owns the device context: data, packed operands, the attached preconditioner.
class KernelOperator {
 public:
  KernelOperator(KernelFamily f, const std::vector<double>& x, std::int64_t n, std::int64_t d, const Hyperparameters& p,
                 int device = 0)
      : n_(n), d_(d), fam_(f) {
    gpk_ctx* c = nullptr;
    const gpk_status s = gpk_create(device, &c);
    if (s != GPK_OK) throw numerical_error("gpk_create failed: no usable CUDA device");
    ctx_.reset(c);
    check(gpk_set_data(ctx_.get(), x.data(), n, d, n), ctx_.get());
    set_params(p);
  }
  void set_params(const Hyperparameters& p) {
    if (static_cast<std::int64_t>(p.log_lengthscales.size()) != d_)
      throw input_error("KernelOperator: lengthscale count must equal data dimension");
    check(gpk_set_params(ctx_.get(), static_cast<int>(fam_), 1.0, p.log_outputscale, p.log_lengthscales.data(),
                         p.log_noise),
          ctx_.get());
    params_ = p;
  }
  std::int64_t rows() const { return n_; }
  int dim() const { return static_cast<int>(d_); }
  int num_params() const { return dim() + 2; }
  const Hyperparameters& params() const { return params_; }
  gpk_ctx* ctx() const { return ctx_.get(); }
  KernelFamily family() const { return fam_; }

  // (K + sigma^2 I) V, t columns (kernels.hpp:184-195)
  std::vector<double> apply(const std::vector<double>& v, int t = 1, gpk_precision prec = GPK_PREC_FP64) const {
    std::vector<double> out(v.size());
    check(gpk_kernel_mvm(ctx_.get(), v.data(), n_, t, out.data(), n_, prec), ctx_.get());
    return out;
  }
  std::vector<double> deriv_apply(int which, const std::vector<double>& v, int t = 1,
                                  gpk_precision prec = GPK_PREC_FP64) const {
    std::vector<double> out(v.size());
    check(gpk_kernel_deriv_mvm(ctx_.get(), which, v.data(), n_, t, out.data(), n_, prec), ctx_.get());
    return out;
  }
  std::vector<double> kernel_column(std::int64_t i) const {
    std::vector<double> out(static_cast<size_t>(n_));
    check(gpk_kernel_column(ctx_.get(), i, out.data()), ctx_.get());
    return out;
  }

#ifdef GPKRYLOV_CUDA_EIGEN
  Eigen::VectorXd apply(const Eigen::VectorXd& v) const {
    Eigen::VectorXd out(v.size());
    check(gpk_kernel_mvm(ctx_.get(), v.data(), n_, 1, out.data(), n_, GPK_PREC_FP64), ctx_.get());
    return out;
  }
#endif

 private:
  struct Del {
    void operator()(gpk_ctx* c) const { gpk_destroy(c); }
  };
  std::unique_ptr<gpk_ctx, Del> ctx_;
  std::int64_t n_, d_;
  KernelFamily fam_;
  Hyperparameters params_;
};

// P = sigma^2 I + L L^T attached to an operator's device context.
class DiagPlusLowRank {
 public:
  DiagPlusLowRank(const KernelOperator& op, int rank, std::vector<std::int64_t> pivots)
      : op_(&op), rank_(rank), pivots_(std::move(pivots)) {}
  int rank() const { return rank_; }
  const std::vector<std::int64_t>& pivots() const { return pivots_; }
  std::vector<double> solve(const std::vector<double>& v, int t = 1) const {
    std::vector<double> out(v.size());
    check(gpk_precond_solve(op_->ctx(), v.data(), op_->rows(), t, out.data(), op_->rows()), op_->ctx());
    return out;
  }
  double logdet() const {
    double v = 0.0;
    check(gpk_precond_logdet(op_->ctx(), &v), op_->ctx());
    return v;
  }
  double trace_inv_deriv(int which) const {
    double v = 0.0;
    check(gpk_precond_trace_inv_deriv(op_->ctx(), which, &v), op_->ctx());
    return v;
  }

 private:
  const KernelOperator* op_;
  int rank_;
  std::vector<std::int64_t> pivots_;
};

// pivoted_cholesky + pivoted_cholesky_deriv_factors (preconditioners.hpp:236-305)
inline DiagPlusLowRank pivoted_cholesky_with_derivatives(const KernelOperator& op, int rank, double diag_tol = 0.0) {
  std::vector<std::int64_t> piv(static_cast<size_t>(rank > 0 ? rank : 1));
  int achieved = 0;
  double noise = 0.0;
  {
    const double ln = op.params().log_noise;
    noise = std::exp(ln);
  }
  check(gpk_pivoted_cholesky(op.ctx(), rank, diag_tol, noise, piv.data(), &achieved, nullptr), op.ctx());
  check(gpk_precond_deriv_factors(op.ctx()), op.ctx());
  piv.resize(static_cast<size_t>(achieved));
  return DiagPlusLowRank(op, achieved, std::move(piv));
}

struct CgResult {  // krylov.hpp:33-39
  std::vector<double> solution;
  int iterations_used = 0;
  bool converged = false;
};

// batched_pcg (krylov.hpp:133-153): one device solve over all columns of B (n x t, column-major)
inline std::vector<CgResult> batched_pcg(const KernelOperator& op, const std::vector<double>& B, int t,
                                         const CgConfig& cfg) {
  const std::int64_t n = op.rows();
  std::vector<double> X(B.size());
  std::vector<int> it(static_cast<size_t>(t)), cv(static_cast<size_t>(t));
  const gpk_cg_cfg c = cfg.c();
  check(gpk_mbcg(op.ctx(), B.data(), n, t, &c, X.data(), n, it.data(), cv.data(), nullptr, nullptr, nullptr),
        op.ctx());
  std::vector<CgResult> out(static_cast<size_t>(t));
  for (int q = 0; q < t; ++q) {
    out[q].solution.assign(X.begin() + q * n, X.begin() + (q + 1) * n);
    out[q].iterations_used = it[q];
    out[q].converged = cv[q] != 0;
  }
  return out;
}

// evaluate_mll (gp_likelihood.hpp:51-103)
inline MllEvaluation evaluate_mll(const std::vector<double>& y, const KernelOperator& k, const DiagPlusLowRank&,
                                  const ProbeBatch& batch, const MllConfig& cfg, bool with_gradient = true) {
  const int np = k.num_params(), l = batch.count;
  MllEvaluation out;
  out.gradient.assign(static_cast<size_t>(np), 0.0);
  out.forward_gammas.assign(static_cast<size_t>(l), 0.0);
  out.forward_cg_iterations.assign(static_cast<size_t>(l), 0);
  std::vector<double> bg(static_cast<size_t>(np) * l, 0.0);
  gpk_mll_result r{};
  r.gradient = out.gradient.data();
  r.forward_gammas = out.forward_gammas.data();
  r.backward_gammas = bg.data();
  r.forward_cg_iterations = out.forward_cg_iterations.data();
  const gpk_mll_cfg c{cfg.solver.c(), cfg.share_probes ? 1 : 0, with_gradient ? 1 : 0, cfg.backward_mode};
  check(gpk_evaluate_mll(k.ctx(), y.data(), batch.probes.data(), k.rows(), l, batch.seed, &c, &r), k.ctx());
  out.value = r.value;
  out.solve_iterations = r.solve_iterations;
  out.probe_seed = batch.seed;
  out.value_sample_variance = r.value_sample_variance;
  out.total_cg_iterations = r.total_cg_iterations;
  out.logdet = r.logdet;
  out.backward_gammas.assign(static_cast<size_t>(np), std::vector<double>(static_cast<size_t>(l)));
  for (int w = 0; w < np; ++w)
    for (int i = 0; i < l; ++i) out.backward_gammas[w][i] = bg[static_cast<size_t>(w) * l + i];
  return out;
}

// ---- the callers of the hot path ---------------------------

struct ExactMll {  // gp_likelihood.hpp:119-122
  double value = 0.0;
  std::vector<double> gradient;
};
// mll_exact (gp_likelihood.hpp:124-146): dense fp64 on the device (cuSOLVER Cholesky)
inline ExactMll mll_exact(const std::vector<double>& y, const KernelOperator& k, bool with_gradient = true) {
  ExactMll out;
  if (with_gradient) out.gradient.assign(static_cast<size_t>(k.num_params()), 0.0);
  check(gpk_mll_exact(k.ctx(), y.data(), &out.value, with_gradient ? out.gradient.data() : nullptr), k.ctx());
  return out;
}

// run_training_arm's predictive mean (experiments.hpp:403-414): cross_kernel(test, X) K_hat^{-1} y
// with the preconditioner attached to k; x_test is n_test x d column-major
inline std::vector<double> predict_mean(const KernelOperator& k, const std::vector<double>& y,
                                        const std::vector<double>& x_test, std::int64_t n_test, const CgConfig& cfg) {
  std::vector<double> mean(static_cast<size_t>(n_test));
  const gpk_cg_cfg c = cfg.c();
  check(gpk_predict_mean(k.ctx(), y.data(), x_test.data(), n_test, n_test, &c, mean.data(), nullptr), k.ctx());
  return mean;
}

struct Dataset {  // dataset.hpp:18-26 (x: n x d column-major)
  std::vector<double> x, y;
  std::int64_t n = 0;
  int d = 0;
  std::int64_t size() const { return n; }
  int dim() const { return d; }
};

struct Standardizer {  // dataset.hpp:87-101
  std::vector<double> feature_mean, feature_std;
  double target_mean = 0.0, target_std = 1.0;
};

struct DataSplits {  // dataset.hpp:103-109
  Dataset train, validation, test;
  Standardizer stats;
  bool standardized = false;
  std::vector<std::string> feature_names;
  std::string target_name;
};

struct SplitFractions {  // dataset.hpp:111-113
  double train = 0.64, validation = 0.16, test = 0.20;
};

// load_csv (dataset.hpp:155-242) over gpk_load_csv; throws input_error with the reference's text
inline DataSplits load_csv(const std::string& path, const std::string& target_column, bool standardize,
                           const SplitFractions& split, std::uint64_t seed) {
  gpk_dataset* h = nullptr;
  char err[1024];
  if (gpk_load_csv(path.c_str(), target_column.c_str(), standardize ? 1 : 0, split.train, split.validation,
                   split.test, seed, &h, err, sizeof(err)) != GPK_OK)
    throw input_error(err);
  std::unique_ptr<gpk_dataset, void (*)(gpk_dataset*)> guard(h, gpk_dataset_free);
  DataSplits out;
  Dataset* parts[3] = {&out.train, &out.validation, &out.test};
  for (int s = 0; s < 3; ++s) {
    Dataset& p = *parts[s];
    gpk_dataset_shape(h, s, &p.n, &p.d);
    p.x.resize(static_cast<size_t>(p.n) * p.d);
    p.y.resize(static_cast<size_t>(p.n));
    gpk_dataset_copy(h, s, p.x.data(), p.n > 0 ? p.n : 1, p.y.data());
  }
  const int d = out.train.d;
  int st = 0;
  out.stats.feature_mean.resize(d);
  out.stats.feature_std.resize(d);
  gpk_dataset_stats(h, &st, out.stats.feature_mean.data(), out.stats.feature_std.data(), &out.stats.target_mean,
                    &out.stats.target_std);
  out.standardized = st != 0;
  for (int j = 0; j < d; ++j) out.feature_names.emplace_back(gpk_dataset_column_name(h, j));
  out.target_name = gpk_dataset_column_name(h, -1);
  return out;
}

struct OptOptions {  // optimizer.hpp:24-43
  gpk_opt_method method = GPK_OPT_LBFGS;
  int max_steps = 20, lbfgs_memory = 10;
  double armijo_c1 = 1e-4, wolfe_c2 = 0.9, adam_lr = 0.1;
  int early_stop_patience = 3;
  double grad_tol = 1e-8;
  int max_line_search = 20;
  gpk_opt_options c() const {
    return gpk_opt_options{method, max_steps, lbfgs_memory, armijo_c1, wolfe_c2, adam_lr, early_stop_patience,
                           grad_tol, max_line_search};
  }
};

struct OptimizeResult {  // optimizer.hpp:356-361 (+ MinimizeResult, the step trace)
  Hyperparameters best;
  double best_validation = 0.0, final_train_neg_mll_per_point = 0.0, final_objective = 0.0;
  int minimizer_steps = 0, stop_reason = 0;
  bool converged = false;
  std::vector<std::vector<double>> step_theta;
  std::vector<double> step_objective, step_validation, step_wall_time;
  std::vector<int> step_accepted;
  long long model_evaluations = 0;
};

// optimize() (optimizer.hpp:404-505) on the device: train / validation are operators holding the
// data (the validation operator may be null); precond_rank < 0 selects IdentityPreconditioner.
inline OptimizeResult optimize(KernelOperator& train, const std::vector<double>& y, KernelOperator* validation,
                               const std::vector<double>* y_val, bool ard, const Hyperparameters& init,
                               int precond_rank, int probe_count, const OptOptions& opts, const MllConfig& mll,
                               std::uint64_t seed, std::int64_t dense_limit = 4096, double diag_tol = 0.0) {
  const int d = train.dim(), np = ard ? d + 2 : 3, ms = opts.max_steps;
  std::vector<double> theta0{init.log_outputscale};
  theta0.insert(theta0.end(), init.log_lengthscales.begin(), init.log_lengthscales.end());
  theta0.push_back(init.log_noise);
  std::vector<double> best(static_cast<size_t>(d + 2)), th(static_cast<size_t>(ms) * np), obj(ms), val(ms), wall(ms);
  std::vector<int> acc(ms);
  gpk_opt_result r{};
  r.best_log_params = best.data();
  r.step_theta = th.data();
  r.step_objective = obj.data();
  r.step_validation = val.data();
  r.step_wall_time = wall.data();
  r.step_accepted = acc.data();
  const gpk_opt_options oc = opts.c();
  const gpk_mll_cfg mc{mll.solver.c(), mll.share_probes ? 1 : 0, 1, mll.backward_mode};
  check(gpk_optimize(train.ctx(), y.data(), validation ? validation->ctx() : nullptr,
                     y_val ? y_val->data() : nullptr, static_cast<int>(train.family()), ard ? 1 : 0, theta0.data(),
                     precond_rank, diag_tol, probe_count, &oc, &mc, seed, dense_limit, &r),
        train.ctx());
  OptimizeResult out;
  out.best.log_outputscale = best[0];
  out.best.log_lengthscales.assign(best.begin() + 1, best.begin() + 1 + d);
  out.best.log_noise = best[static_cast<size_t>(d + 1)];
  out.best_validation = r.best_validation;
  out.final_train_neg_mll_per_point = r.final_train_neg_mll_per_point;
  out.final_objective = r.final_objective;
  out.minimizer_steps = r.minimizer_steps;
  out.stop_reason = r.stop_reason;
  out.converged = r.converged != 0;
  out.model_evaluations = r.n_evaluations;
  for (int s = 0; s < r.n_steps; ++s) {
    out.step_theta.emplace_back(th.begin() + static_cast<long>(s) * np, th.begin() + static_cast<long>(s + 1) * np);
    out.step_objective.push_back(obj[s]);
    out.step_validation.push_back(val[s]);
    out.step_wall_time.push_back(wall[s]);
    out.step_accepted.push_back(acc[s]);
  }
  return out;
}

}  // namespace cuda
}  // namespace gpkrylov
