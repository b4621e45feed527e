// C++ caller of the reference-named facade (include/gpkrylov_cuda.hpp) over the C-ABI.
// Prints one JSON object; tests/test_gpu_facade.py compares it with the oracle.
#include <cmath>
#include <cstdio>
#include <vector>

#include "gpkrylov_cuda.hpp"

using namespace gpkrylov::cuda;

int main() {
  const int n = 400, d = 2, l = 6, rank = 12;
  std::vector<double> x(static_cast<size_t>(n) * d), y(n);
  for (int i = 0; i < n; ++i) {
    x[i] = std::sin(0.37 * i) * 1.5;          // column 0
    x[n + i] = std::cos(0.11 * i + 0.3);      // column 1
    y[i] = std::sin(2.0 * x[i]) + 0.3 * x[n + i];
  }
  Hyperparameters p;
  p.log_outputscale = std::log(1.1);
  p.log_lengthscales = {std::log(0.8), std::log(0.8)};
  p.log_noise = std::log(0.05);
  KernelOperator op(KernelFamily::Matern52, x, n, d, p);
  DiagPlusLowRank prec = pivoted_cholesky_with_derivatives(op, rank);
  const ProbeBatch batch = make_probes(n, l, mix_seed(17, 1));
  MllConfig cfg;
  cfg.solver.max_iters = 400;
  cfg.solver.rel_tol = 1e-10;
  cfg.solver.precision = GPK_PREC_FP64;
  cfg.solver.refine = 0;
  cfg.backward_mode = 1;
  const MllEvaluation e = evaluate_mll(y, op, prec, batch, cfg);
  std::printf("{\"value\": %.17g, \"logdet\": %.17g, \"gradient\": [", e.value, e.logdet);
  for (size_t w = 0; w < e.gradient.size(); ++w) std::printf("%s%.17g", w ? ", " : "", e.gradient[w]);
  std::printf("], \"pivots\": [");
  for (size_t s = 0; s < prec.pivots().size(); ++s) std::printf("%s%lld", s ? ", " : "", (long long)prec.pivots()[s]);
  std::printf("], \"seed\": %llu", (unsigned long long)batch.seed);
  // the callers: dense exact mLL and a 3-step Adam optimize()
  const ExactMll ex = mll_exact(y, op, false);
  std::printf(", \"exact\": %.17g", ex.value);
  OptOptions oo;
  oo.method = GPK_OPT_ADAM;
  oo.max_steps = 3;
  const OptimizeResult opt = optimize(op, y, nullptr, nullptr, true, p, rank, l, oo, cfg, 17);
  std::printf(", \"opt_best\": [%.17g", opt.best.log_outputscale);
  for (double v : opt.best.log_lengthscales) std::printf(", %.17g", v);
  std::printf(", %.17g], \"opt_evals\": %lld}\n", opt.best.log_noise, opt.model_evaluations);
  // error mapping: a bad hyperparameter index is an input_error
  try {
    op.deriv_apply(7, y);
    return 2;
  } catch (const input_error&) {
  }
  return 0;
}
