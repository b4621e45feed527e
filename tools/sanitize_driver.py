"""Small invocations of every hand-written kernel family for compute-sanitizer
(tools/sanitize.sh): the tcgen05 Gram and direct MVMs (multi-unit persistent CTAs via the
GPK_TCG_CTAS hook), the fp64 DMMA MVM, the cooperative pivoted Cholesky and the derivative
factors, one evaluate_mll (fused CG iteration: pap/alpha, G1s, G2s, beta + p with the pinned
host snapshot; the bilinear derivative pass; the fp64 residual audit), the faithful backward
and a row-sharded world-2 evaluation over the in-process rank group."""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_00243_b200 as gk  # noqa: E402
from paper_2107_00243_b200.gpkrylov import RankGroup  # noqa: E402

os.environ.setdefault("GPK_TCG_CTAS", "5")
rng = np.random.default_rng(3)
n, l = 1100, 6
for fam, d, variant in (("matern32", 12, "gram"), ("rbf", 9, "gram"), ("matern52", 3, "direct")):
    x = rng.standard_normal((n, d))
    hp = gk.Hyperparameters.from_raw(d, 1.0, 1.5, 0.05)
    op = gk.KernelOperator(gk.KernelSpec(fam), x, hp).set_mvm_variant(variant)
    v = rng.standard_normal((n, 13))
    for prec in ("tf32x3", "fp32", "fp64"):
        op.apply(v, precision=prec)
    y = np.sin(x[:, 0]) + 0.1 * rng.standard_normal(n)
    pc = gk.pivoted_cholesky_with_derivatives(op, 20)
    z = gk.make_probes(n, l, gk.mix_seed(17, 1))
    for backward in ("fused", "faithful"):
        r = gk.evaluate_mll(y, op, pc, z, gk.MllConfig(gk.CgConfig(300, 1e-6, False, "tf32x3", 2), True, backward))
        print(fam, variant, backward, r.value, r.max_true_rel_residual)

x = rng.standard_normal((n, 4))
y = np.cos(x[:, 1])
hp = gk.Hyperparameters.from_raw(4, 1.0, 1.2, 0.05)
z = gk.make_probes(n, l, 5)
group = RankGroup(2)
out = [None, None]


def rank(rk):
    op = gk.KernelOperator(gk.KernelSpec("matern32"), x, hp, shard=(group, rk))
    pc = gk.pivoted_cholesky_with_derivatives(op, 12)
    out[rk] = gk.evaluate_mll(y, op, pc, z, gk.MllConfig(gk.CgConfig(300, 1e-6, False, "tf32x3", 2), True, "fused"))


th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
for t in th:
    t.start()
for t in th:
    t.join()
print("sharded", out[0].value, out[1].value)
