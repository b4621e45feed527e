// gpk_optimize: the caller of the hot path —
// optimize() of /root/reference/proj/include/gpkrylov/optimizer.hpp:404-505
// restated as host C++ above the library's own C-ABI.  Every objective
// evaluation is one device evaluate_mll (gpk_evaluate_mll); the per-step
// preconditioner rebuild is the device pivoted Cholesky + derivative factors;
// the validation / final metrics are the device dense mll_exact or the
// identity-preconditioned value-only evaluate_mll.  Only O(d) vector algebra of
// the minimizer runs here.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <deque>
#include <functional>
#include <limits>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "gpkrylov_cuda.h"

extern "C" void gpk_set_error_internal(gpk_ctx* ctx, const char* msg);

namespace {

using Vec = std::vector<double>;
using Clock = std::chrono::steady_clock;

struct Fatal {  // a status that must leave the optimizer (device failure, bad arguments)
  gpk_status code;
  std::string msg;
};

double vdot(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
double vnorm(const Vec& a) { return std::sqrt(vdot(a, a)); }

struct Sample {  // detail::Evaluation (optimizer.hpp:76-79)
  double f = 0.0;
  Vec g;
};
struct StepRow {  // StepRecord (optimizer.hpp:52-66)
  Vec theta;
  double objective = 0.0, validation = 0.0, wall = 0.0, step_length = 0.0, f_before = 0.0, dd_before = 0.0,
         dd_after = 0.0;
  long long evals = 0;
  bool accepted = true;
};
struct EvalRow {  // EvalRecord (optimizer.hpp:45-50)
  int step;
  double f, gnorm;
};

class Driver {
 public:
  Driver(gpk_ctx* tr, const double* y, gpk_ctx* va, const double* yv, int family, bool ard, int d, int64_t n,
         int64_t nv, int rank, double diag_tol, int probes, const gpk_opt_options& o, const gpk_mll_cfg& mc,
         uint64_t seed, int64_t dense_limit)
      : tr_(tr), y_(y), va_(va), yv_(yv), fam_(family), ard_(ard), d_(d), n_(n), nv_(nv), rank_(rank),
        diag_tol_(diag_tol), l_(probes), o_(o), mc_(mc), seed_(seed), dense_limit_(dense_limit) {}

  // ---- parameter packing (optimizer.hpp:373-400)
  Vec full_theta(const Vec& x) const {  // (o, l_1..l_d, sigma^2)
    if (ard_) return x;
    Vec t(static_cast<size_t>(d_ + 2), x[1]);
    t[0] = x[0];
    t[static_cast<size_t>(d_ + 1)] = x[2];
    return t;
  }
  Vec collapse(const Vec& g) const {
    if (ard_) return g;
    double s = 0.0;
    for (int j = 0; j < d_; ++j) s += g[static_cast<size_t>(1 + j)];
    return {g[0], s, g[static_cast<size_t>(d_ + 1)]};
  }
  gpk_status set_params(gpk_ctx* c, const Vec& th) const {
    return gpk_set_params(c, fam_, 1.0, th[0], th.data() + 1, th[static_cast<size_t>(d_ + 1)]);
  }
  void must(gpk_status s, gpk_ctx* c) const {
    if (s != GPK_OK) throw Fatal{s, gpk_last_error(c)};
  }
  static bool recoverable(gpk_status s) {  // input_error / numerical_error (incl. solver_error)
    return s == GPK_INPUT_ERROR || s == GPK_NUMERICAL_ERROR || s == GPK_SOLVER_ERROR;
  }

  // ---- objective (optimizer.hpp:430-445): -mLL and its gradient; +inf when unevaluable
  double objective(const Vec& x, Vec& g) {
    const Vec th = full_theta(x);
    gpk_status s = set_params(tr_, th);
    if (s == GPK_OK) {
      Vec grad(static_cast<size_t>(d_ + 2), 0.0);
      gpk_mll_result r{};
      r.gradient = grad.data();
      gpk_mll_cfg c = mc_;
      c.with_gradient = 1;
      s = gpk_evaluate_mll_device(tr_, dy_.p, dprobes_.p, n_, l_, probe_seed_, &c, &r);
      if (s == GPK_OK) {
        cg_iters_ += r.total_cg_iterations;
        const Vec cg = collapse(grad);
        for (size_t i = 0; i < g.size(); ++i) g[i] = -cg[i];
        return -r.value;
      }
    }
    if (!recoverable(s)) throw Fatal{s, gpk_last_error(tr_)};
    std::fill(g.begin(), g.end(), 0.0);
    return std::numeric_limits<double>::infinity();
  }
  Sample eval(const Vec& x, int step) {  // CountingObjective (:80-89)
    Sample e;
    e.g.assign(x.size(), 0.0);
    e.f = objective(x, e.g);
    evals_.push_back({step, e.f, vnorm(e.g)});
    return e;
  }

  // ---- begin_step hook (:448-453): preconditioner at the step's iterate, fresh probes
  // The mt19937_64 probe stream (trace_estimation.hpp:27-36) is generated on the device
  // (gpk_probes.cu, bitwise the host stream) behind the preconditioner build on the context's
  // stream; y was uploaded once.  Nothing of size n crosses PCIe during the optimization.
  void begin_step(int step, const Vec& x) {
    const Vec th = full_theta(x);
    must(set_params(tr_, th), tr_);
    probe_seed_ = gpk_mix_seed(seed_, static_cast<uint64_t>(step));
    if (dy_.p == nullptr) {
      dy_.alloc(static_cast<size_t>(n_));
      if (cudaMemcpy(dy_.p, y_, sizeof(double) * static_cast<size_t>(n_), cudaMemcpyHostToDevice) != cudaSuccess)
        throw Fatal{GPK_CUDA_ERROR, "optimize: upload of y failed"};
      dprobes_.alloc(static_cast<size_t>(n_) * l_);
    }
    if (rank_ < 0) {
      must(gpk_precond_identity(tr_), tr_);
    } else {
      int achieved = 0;
      must(gpk_pivoted_cholesky(tr_, rank_, diag_tol_, std::exp(th[static_cast<size_t>(d_ + 1)]), nullptr,
                                &achieved, nullptr),
           tr_);
      must(gpk_precond_deriv_factors(tr_), tr_);
    }
    must(gpk_make_probes_device(tr_, n_, l_, probe_seed_, dprobes_.p), tr_);
  }

  // ---- validation metric (:455-471): dense mll_exact per point, or the identity-
  // preconditioned value-only estimate with probes mix_seed(seed, 0x7a11)
  double validation(const Vec& x) {
    if (va_ == nullptr || nv_ == 0) return 0.0;
    const Vec th = full_theta(x);
    must(set_params(va_, th), va_);
    double v = 0.0;
    if (nv_ <= dense_limit_) {
      must(gpk_mll_exact(va_, yv_, &v, nullptr), va_);
      return -v / static_cast<double>(nv_);
    }
    if (dvprobes_.p == nullptr) {
      vseed_ = gpk_mix_seed(seed_, 0x7a11ULL);
      dyv_.alloc(static_cast<size_t>(nv_));
      if (cudaMemcpy(dyv_.p, yv_, sizeof(double) * static_cast<size_t>(nv_), cudaMemcpyHostToDevice) != cudaSuccess)
        throw Fatal{GPK_CUDA_ERROR, "optimize: upload of the validation targets failed"};
      dvprobes_.alloc(static_cast<size_t>(nv_) * l_);
      must(gpk_make_probes_device(va_, nv_, l_, vseed_, dvprobes_.p), va_);
    }
    must(gpk_precond_identity(va_), va_);
    gpk_mll_cfg c = mc_;
    c.with_gradient = 0;
    gpk_mll_result r{};
    Vec grad(static_cast<size_t>(d_ + 2), 0.0);
    r.gradient = grad.data();
    must(gpk_evaluate_mll_device(va_, dyv_.p, dvprobes_.p, nv_, l_, vseed_, &c, &r), va_);
    return -r.value / static_cast<double>(nv_);
  }

  // ---- strong-Wolfe line search (:100-180)
  bool line_search(const Vec& x, const Vec& p, const Sample& start, int step, double* alpha_out, Sample* at) {
    const double f0 = start.f, g0 = vdot(start.g, p);
    if (!(g0 < 0.0)) return false;  // not a descent direction
    int used = 0;
    auto trial = [&](double a) {
      ++used;
      Vec xa(x.size());
      for (size_t i = 0; i < x.size(); ++i) xa[i] = x[i] + a * p[i];
      return eval(xa, step);
    };
    auto too_high = [&](double a, double f) { return f > f0 + o_.armijo_c1 * a * g0; };
    auto curvature = [&](const Sample& e) { return std::abs(vdot(e.g, p)) <= o_.wolfe_c2 * std::abs(g0); };
    double lo = 0.0, hi = 0.0, flo = f0, a = 1.0, a_prev = 0.0, f_prev = f0;
    bool bracket = false;
    while (used < o_.max_line_search) {  // expansion: double the step until bracketed
      Sample e = trial(a);
      const double ga = vdot(e.g, p);
      if (too_high(a, e.f) || (a_prev > 0.0 && e.f >= f_prev)) {
        lo = a_prev, flo = f_prev, hi = a, bracket = true;
        break;
      }
      if (curvature(e)) {
        *alpha_out = a;
        *at = std::move(e);
        return true;
      }
      if (ga >= 0.0) {
        lo = a, flo = e.f, hi = a_prev, bracket = true;
        break;
      }
      a_prev = a;
      f_prev = e.f;
      a = std::min(2.0 * a, 1e6);
    }
    if (!bracket) return false;
    while (used < o_.max_line_search) {  // zoom by bisection
      const double m = 0.5 * (lo + hi);
      Sample e = trial(m);
      if (too_high(m, e.f) || e.f >= flo) {
        hi = m;
      } else {
        if (curvature(e)) {
          *alpha_out = m;
          *at = std::move(e);
          return true;
        }
        if (vdot(e.g, p) * (hi - lo) >= 0.0) hi = lo;
        lo = m;
        flo = e.f;
      }
      if (std::abs(hi - lo) < 1e-16) break;
    }
    return false;
  }

  // after_step hook (:473-490): validation, best tracking, early stopping
  bool after_step(const Vec& x) {
    const double vm = validation(x);
    steps_.back().validation = vm;
    const bool early = va_ != nullptr && nv_ > 0;
    if (!early) {
      best_ = full_theta(x);
      return true;
    }
    if (vm < best_validation_) {
      best_validation_ = vm;
      best_ = full_theta(x);
      since_best_ = 0;
    } else if (++since_best_ >= o_.early_stop_patience) {
      return false;
    }
    return true;
  }

  // ---- L-BFGS (:215-301)
  void lbfgs(const Vec& x0) {
    x_ = x0;
    std::deque<std::pair<Vec, Vec>> hist;  // (s, y)
    const auto t0 = Clock::now();
    auto secs = [&] { return std::chrono::duration<double>(Clock::now() - t0).count(); };
    for (int step = 1; step <= o_.max_steps; ++step) {
      begin_step(step, x_);
      Sample cur = eval(x_, step);
      f_ = cur.f;
      if (vnorm(cur.g) <= o_.grad_tol) {
        converged_ = true;
        reason_ = GPK_OPT_GRAD_TOL;
        break;
      }
      Vec q = cur.g;
      std::vector<double> coef(hist.size());
      for (int i = static_cast<int>(hist.size()) - 1; i >= 0; --i) {  // two-loop recursion
        const Vec& s = hist[static_cast<size_t>(i)].first;
        const Vec& yv = hist[static_cast<size_t>(i)].second;
        const double rho = 1.0 / vdot(yv, s);
        coef[static_cast<size_t>(i)] = rho * vdot(s, q);
        for (size_t j = 0; j < q.size(); ++j) q[j] -= coef[static_cast<size_t>(i)] * yv[j];
      }
      if (!hist.empty()) {
        const double gam = vdot(hist.back().first, hist.back().second) / vdot(hist.back().second, hist.back().second);
        for (double& v : q) v *= gam;
      }
      for (size_t i = 0; i < hist.size(); ++i) {
        const double rho = 1.0 / vdot(hist[i].second, hist[i].first);
        const double b = rho * vdot(hist[i].second, q);
        for (size_t j = 0; j < q.size(); ++j) q[j] += (coef[i] - b) * hist[i].first[j];
      }
      Vec p(q.size());
      for (size_t j = 0; j < q.size(); ++j) p[j] = -q[j];
      if (vdot(p, cur.g) >= 0.0) {  // noisy curvature spoiled the direction: steepest descent
        hist.clear();
        for (size_t j = 0; j < q.size(); ++j) p[j] = -cur.g[j];
      }
      double alpha = 0.0;
      Sample at;
      const bool ok = line_search(x_, p, cur, step, &alpha, &at);
      StepRow rec;
      rec.f_before = cur.f;
      rec.dd_before = vdot(cur.g, p);
      rec.evals = static_cast<long long>(evals_.size());
      rec.wall = secs();
      if (!ok) {
        rec.theta = x_;
        rec.objective = cur.f;
        rec.accepted = false;
        steps_.push_back(rec);
        reason_ = GPK_OPT_LINE_SEARCH_FAILED;
        break;
      }
      Vec s(p.size()), yv(p.size());
      for (size_t j = 0; j < p.size(); ++j) {
        s[j] = alpha * p[j];
        yv[j] = at.g[j] - cur.g[j];
      }
      if (vdot(s, yv) > 1e-12 * vnorm(s) * vnorm(yv)) {
        hist.emplace_back(s, yv);
        if (static_cast<int>(hist.size()) > o_.lbfgs_memory) hist.pop_front();
      }
      for (size_t j = 0; j < s.size(); ++j) x_[j] += s[j];
      f_ = at.f;
      min_steps_ = step;
      rec.theta = x_;
      rec.objective = at.f;
      rec.step_length = alpha;
      rec.dd_after = vdot(at.g, p);
      rec.evals = static_cast<long long>(evals_.size());
      rec.wall = secs();
      steps_.push_back(rec);
      if (!after_step(x_)) {
        reason_ = GPK_OPT_STOPPED;
        break;
      }
    }
  }

  // ---- Adam (:305-350)
  void adam(const Vec& x0) {
    constexpr double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    x_ = x0;
    Vec m(x0.size(), 0.0), v(x0.size(), 0.0);
    const auto t0 = Clock::now();
    for (int step = 1; step <= o_.max_steps; ++step) {
      begin_step(step, x_);
      Sample cur = eval(x_, step);
      f_ = cur.f;
      if (vnorm(cur.g) <= o_.grad_tol) {
        converged_ = true;
        reason_ = GPK_OPT_GRAD_TOL;
        break;
      }
      const double bc1 = 1.0 - std::pow(b1, step), bc2 = 1.0 - std::pow(b2, step);
      for (size_t i = 0; i < x0.size(); ++i) {
        m[i] = b1 * m[i] + (1.0 - b1) * cur.g[i];
        v[i] = b2 * v[i] + (1.0 - b2) * (cur.g[i] * cur.g[i]);
        x_[i] -= (o_.adam_lr / bc1) * (m[i] / (std::sqrt(v[i] / bc2) + eps));
      }
      min_steps_ = step;
      StepRow rec;
      rec.theta = x_;
      rec.objective = cur.f;
      rec.f_before = cur.f;
      rec.step_length = o_.adam_lr;
      rec.evals = static_cast<long long>(evals_.size());
      rec.wall = std::chrono::duration<double>(Clock::now() - t0).count();
      steps_.push_back(rec);
      if (!after_step(x_)) {
        reason_ = GPK_OPT_STOPPED;
        break;
      }
    }
  }

  void run(const Vec& init_full, gpk_opt_result* res) {
    const auto t0 = Clock::now();
    best_ = init_full;
    Vec x0 = init_full;
    if (!ard_) x0 = {init_full[0], init_full[1], init_full[static_cast<size_t>(d_ + 1)]};
    if (o_.method == GPK_OPT_LBFGS) lbfgs(x0);
    else adam(x0);
    const bool early = va_ != nullptr && nv_ > 0;
    if (!early && steps_.empty()) best_ = init_full;
    double final_train = f_ / static_cast<double>(n_);
    if (n_ <= dense_limit_) {  // dense training metric (:497-502)
      double v = 0.0;
      must(set_params(tr_, best_), tr_);
      must(gpk_mll_exact(tr_, y_, &v, nullptr), tr_);
      final_train = -v / static_cast<double>(n_);
    }
    // ---- results
    if (res->best_log_params)
      for (int i = 0; i < d_ + 2; ++i) res->best_log_params[i] = best_[static_cast<size_t>(i)];
    res->best_validation = best_validation_;
    res->final_train_neg_mll_per_point = final_train;
    res->final_objective = f_;
    res->minimizer_steps = min_steps_;
    res->converged = converged_ ? 1 : 0;
    res->stop_reason = reason_;
    res->n_steps = static_cast<int>(steps_.size());
    const int npo = ard_ ? d_ + 2 : 3;
    for (size_t s = 0; s < steps_.size(); ++s) {
      const StepRow& r = steps_[s];
      if (res->step_theta)
        for (int j = 0; j < npo; ++j) res->step_theta[s * npo + j] = r.theta[static_cast<size_t>(j)];
      if (res->step_objective) res->step_objective[s] = r.objective;
      if (res->step_validation) res->step_validation[s] = r.validation;
      if (res->step_wall_time) res->step_wall_time[s] = r.wall;
      if (res->step_length) res->step_length[s] = r.step_length;
      if (res->step_f_before) res->step_f_before[s] = r.f_before;
      if (res->step_dir_derivative_before) res->step_dir_derivative_before[s] = r.dd_before;
      if (res->step_dir_derivative_after) res->step_dir_derivative_after[s] = r.dd_after;
      if (res->step_accepted) res->step_accepted[s] = r.accepted ? 1 : 0;
      if (res->step_evaluations) res->step_evaluations[s] = r.evals;
    }
    res->n_evaluations = static_cast<int>(evals_.size());
    for (size_t e = 0; e < evals_.size() && static_cast<int>(e) < res->eval_capacity; ++e) {
      if (res->eval_step) res->eval_step[e] = evals_[e].step;
      if (res->eval_f) res->eval_f[e] = evals_[e].f;
      if (res->eval_grad_norm) res->eval_grad_norm[e] = evals_[e].gnorm;
    }
    res->total_cg_iterations = cg_iters_;
    res->seconds_total = std::chrono::duration<double>(Clock::now() - t0).count();
  }

 private:
  gpk_ctx* tr_;
  const double* y_;
  gpk_ctx* va_;
  const double* yv_;
  int fam_;
  bool ard_;
  int d_;
  int64_t n_, nv_;
  int rank_;
  double diag_tol_;
  int l_;
  gpk_opt_options o_;
  gpk_mll_cfg mc_;
  uint64_t seed_;
  int64_t dense_limit_;
  struct DevBuf {  // device allocation owned by the driver
    double* p = nullptr;
    void alloc(size_t count) {
      if (cudaMalloc(reinterpret_cast<void**>(&p), sizeof(double) * count) != cudaSuccess) {
        p = nullptr;
        throw Fatal{GPK_CUDA_ERROR, "optimize: device allocation failed"};
      }
    }
    ~DevBuf() {
      if (p) cudaFree(p);
    }
  };
  DevBuf dy_, dprobes_, dyv_, dvprobes_;
  uint64_t probe_seed_ = 0, vseed_ = 0;
  std::vector<StepRow> steps_;
  std::vector<EvalRow> evals_;
  Vec x_, best_;
  double f_ = std::numeric_limits<double>::quiet_NaN();
  double best_validation_ = std::numeric_limits<double>::infinity();
  int since_best_ = 0, min_steps_ = 0, reason_ = GPK_OPT_MAX_STEPS;
  bool converged_ = false;
  long long cg_iters_ = 0;
};

}  // namespace

extern "C" gpk_status gpk_optimize(gpk_ctx* train, const double* y, gpk_ctx* validation, const double* y_val,
                                   int family, int ard, const double* init_log_params, int precond_rank,
                                   double diag_tol, int probe_count, const gpk_opt_options* opts,
                                   const gpk_mll_cfg* mll_cfg, uint64_t seed, int64_t dense_limit,
                                   gpk_opt_result* res) {
  if (train == nullptr) return GPK_INPUT_ERROR;
  auto bad = [&](const char* m) {
    gpk_set_error_internal(train, m);
    return GPK_INPUT_ERROR;
  };
  if (!y || !init_log_params || !opts || !mll_cfg || !res) return bad("gpk_optimize: null argument");
  const gpk_opt_options& o = *opts;
  // OptOptions::validate (optimizer.hpp:35-42)
  if (o.max_steps < 1) return bad("OptOptions: max_steps must be >= 1");
  if (!(o.armijo_c1 > 0.0 && o.armijo_c1 < o.wolfe_c2 && o.wolfe_c2 < 1.0))
    return bad("OptOptions: need 0 < c1 < c2 < 1");
  if (o.lbfgs_memory < 1) return bad("OptOptions: lbfgs_memory must be >= 1");
  if (o.early_stop_patience < 1) return bad("OptOptions: early_stop_patience must be >= 1");
  if (o.method != GPK_OPT_LBFGS && o.method != GPK_OPT_ADAM) return bad("OptOptions: unknown method");
  if (probe_count < 1) return bad("make_probes: need at least one probe");
  int64_t n = 0, nv = 0;
  int d = 0, dv = 0;
  if (gpk_data_shape(train, &n, &d) != GPK_OK || n < 1) return bad("optimize: empty training set");
  if (validation) {
    if (gpk_data_shape(validation, &nv, &dv) != GPK_OK) return bad("optimize: validation context has no data");
    if (dv != d) return bad("optimize: hyperparameter dimension mismatch");
    if (nv > 0 && !y_val) return bad("gpk_optimize: null validation labels");
  }
  for (int i = 0; i < d + 2; ++i) {  // Hyperparameters::validate (kernels.hpp:55-63)
    const double lv = init_log_params[i];
    if (!(std::isfinite(lv) && std::isfinite(std::exp(lv)) && std::exp(lv) > 0.0))
      return bad("Hyperparameters: initial value not positive finite");
  }
  try {
    Driver drv(train, y, validation, y_val, family, ard != 0, d, n, nv, precond_rank, diag_tol, probe_count, o,
               *mll_cfg, seed, dense_limit);
    drv.run(Vec(init_log_params, init_log_params + d + 2), res);
  } catch (const Fatal& f) {
    gpk_set_error_internal(train, f.msg.c_str());
    return f.code;
  } catch (const std::exception& e) {
    gpk_set_error_internal(train, e.what());
    return GPK_NUMERICAL_ERROR;
  }
  gpk_set_error_internal(train, "");
  return GPK_OK;
}
