"""world_size-2 gloo tests (CPU) of the row-sharding host logic of the multi-GPU
design: balanced shards, deterministic rank-order reductions, the global
(max, lowest index) pivot reduction, and a sharded PCG that reproduces the
unsharded oracle PCG."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import sharding_model as sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out[rank] = fn(rank, world, dist)
    finally:
        dist.destroy_process_group()


def run(fn, world=2):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), fn, out), nprocs=world, join=True)
    return [out[r] for r in range(world)]


def test_shard_ranges_partition_and_balance():
    # the product's rule (gpk_host.cu shard_of): contiguous runs of whole 128-row blocks, block
    # counts balanced to within one -- a fused-MVM row block never straddles two ranks
    for n in (1, 7, 1100, 16384, 45730, 1048576):
        for world in (1, 2, 3, 8):
            rs = [sharding.shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert all(a % 128 == 0 or a == n for a, _ in rs)
            blocks = [(b - a + 127) // 128 for a, b in rs]
            assert max(blocks) - min(blocks) <= 1
    assert [sharding.shard_range(1100, r, 2) for r in range(2)] == [(0, 640), (640, 1100)]


def _reduce_fn(rank, world, dist):
    rng = np.random.default_rng(100 + rank)
    x = rng.standard_normal(5) * 10.0 ** rng.integers(-8, 8, 5)
    s1 = sharding.allreduce_sum_fixed(x, dist)
    s2 = sharding.allreduce_sum_fixed(x, dist)
    return s1.tolist(), s2.tolist(), x.tolist()


def test_fixed_order_allreduce_is_deterministic_and_identical_on_ranks():
    res = run(_reduce_fn)
    (a0, b0, x0), (a1, b1, x1) = res
    assert a0 == b0 == a1 == b1  # bitwise, on every rank
    assert a0 == (np.array(x0) + np.array(x1)).tolist()  # rank order 0 then 1


def _argmax_fn(rank, world, dist):
    n = 10
    lo, hi = sharding.shard_range(n, rank, world)
    vals = np.zeros(n)
    vals[[2, 7]] = 5.0  # a tie across the two shards -> lowest global index wins
    return sharding.global_argmax(vals[lo:hi], lo, dist)


def test_global_argmax_ties_to_lowest_index():
    for v, i in run(_argmax_fn):
        assert v == 5.0 and i == 2


def _pcg_fn(rank, world, dist):
    import oracle

    n, d, t = 300, 2, 5
    x = oracle.random_matrix(n, d, 11)
    p = oracle.Params(d, 1.0, 0.6, 0.05)
    K = oracle.dense(oracle.RBF, x, p)  # K_hat (dense rows stand in for the fused MVM)
    B = oracle.random_matrix(n, t, 12)
    lo, hi = sharding.shard_range(n, rank, world)
    xs, it, cv = sharding.sharded_pcg(lambda P: K[lo:hi] @ P, B[lo:hi], n, lambda R: R / 0.05, dist,
                                      max_iters=300, rel_tol=1e-8)
    full = sharding.allgather_rows(xs, n, dist)
    return full, it, cv


def test_sharded_pcg_matches_oracle(orc):
    res = run(_pcg_fn)
    full0, it0, cv0 = res[0]
    full1, it1, cv1 = res[1]
    assert np.array_equal(full0, full1) and list(it0) == list(it1)
    n, d = 300, 2
    x = orc.random_matrix(n, d, 11)
    p = orc.Params(d, 1.0, 0.6, 0.05)
    B = orc.random_matrix(n, 5, 12)
    # rank-0 pivoted Cholesky == sigma^2 I preconditioner, the same as the sharded run
    want, wit, wcv = orc.pcg_kernel(orc.RBF, x, p, B, rank=0, max_iters=300, rel_tol=1e-8)
    for c in range(5):
        assert abs(int(it0[c]) - int(wit[c])) <= max(1, int(0.1 * wit[c]))
        assert np.linalg.norm(full0[:, c] - want[:, c]) / np.linalg.norm(want[:, c]) < 1e-6
    assert all(cv0) and all(wcv)
