"""bench.py's multi-rank launcher: `--gpus N` runs ONE row-sharded evaluation over N ranks and
prints one line from rank 0 with n_gpus N and strong scaling.  On a one-GPU box the test-only
`--comm group` transport runs the N ranks as threads over the library's host-staged rank
group, so the spawn, sharding, rank-ordered reductions and max-over-ranks timing run end to
end; the NCCL transport is the same code behind gpk_create_sharded."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*extra):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "3", "--no-sweep",
           "--no-cpu", "--workload", "C2", *extra]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_bench_group_world2_matches_single():
    one = run_bench()
    two = run_bench("--gpus", "2", "--comm", "group")
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["scaling"] == "strong" and "row-sharded x2" in two["config"]["parallelism"]
    t1, t2 = one["telemetry"], two["telemetry"]
    assert t2["value"] == pytest.approx(t1["value"], rel=1e-6)
    assert t2["logdet"] == pytest.approx(t1["logdet"], rel=1e-6)
    assert t2["unconverged_columns"] == 0
    assert two["gpu_launches"] > 0


def test_bench_refuses_more_gpus_than_visible():
    import torch

    n = torch.cuda.device_count() + 1
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert p.returncode == 2 and "visible" in p.stderr
