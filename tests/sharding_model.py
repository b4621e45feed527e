"""TEST MODEL (not product code): numpy / torch.distributed restatement of the row sharding
that the C++ driver implements (gpk_host.cu shard_of / apply_kernel / psolve / the sharded
pivoted Cholesky), so that the decomposition can be exercised at world size 2 over gloo on CPU.

Host-side logic of the multi-GPU design, expressed with
torch.distributed collectives so it runs over NCCL on B200s and over gloo on
CPU (tests/test_sharding_gloo.py):

* every n-length array (CG state, L, C, dL) is split into contiguous row
  shards of whole 128-row blocks (the product's rule, gpk_host.cu shard_of: a fused-MVM
  row block never straddles ranks; tests/test_gpu_sharded.py checks gpk_shard_rows
  against shard_range);
* per CG iteration the direction block is all-gathered (each rank needs all
  columns' values at all rows for its K rows x all-j contraction) and the
  per-column partial dot products are all-reduced;
* cross-rank reductions are DETERMINISTIC: partials are all-gathered and summed
  in rank order (the same order for every rank and every run), never with an
  order-dependent reduction;
* the pivoted-Cholesky argmax is a global (max, lowest index) reduction so the
  pivot sequence is identical to the unsharded one (preconditioners.hpp:247-249).

The numeric per-rank work here is numpy (the reference model the NCCL path
must reproduce); on GPUs the same steps call the sm_100a kernels.
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int):
    """[start, stop) row range of `rank`: contiguous runs of 128-row blocks, block counts
    balanced to within one (gpk_host.cu shard_of, bit for bit)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    nb = (n + 127) // 128
    base, extra = divmod(nb, world)
    b0 = rank * base + min(rank, extra)
    b1 = b0 + base + (1 if rank < extra else 0)
    return min(n, b0 * 128), min(n, b1 * 128)


def allreduce_sum_fixed(x: np.ndarray, dist) -> np.ndarray:
    """Deterministic sum over ranks: all-gather the partials, add in rank order."""
    import torch

    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    out = np.zeros_like(x, dtype=np.float64)
    for p in parts:  # rank order
        out = out + p.numpy()
    return out


def allgather_rows(local: np.ndarray, n: int, dist) -> np.ndarray:
    """Concatenate the row shards (axis 0) of all ranks into the full n-row array."""
    import torch

    world = dist.get_world_size()
    sizes = [shard_range(n, r, world)[1] - shard_range(n, r, world)[0] for r in range(world)]
    maxs = max(sizes)
    pad = np.zeros((maxs,) + local.shape[1:], dtype=np.float64)
    pad[: local.shape[0]] = local
    t = torch.from_numpy(pad)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    return np.concatenate([parts[r].numpy()[: sizes[r]] for r in range(world)], axis=0)


def global_argmax(local_vals: np.ndarray, offset: int, dist):
    """(max value, lowest global index among the maxima) over all ranks."""
    import torch

    if local_vals.size:
        i = int(np.argmax(local_vals))  # numpy returns the first (lowest) index of the max
        cand = np.array([local_vals[i], float(offset + i)])
    else:
        cand = np.array([-np.inf, float(np.iinfo(np.int64).max)])
    t = torch.from_numpy(cand)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    best_v, best_i = -np.inf, np.inf
    for p in parts:
        v, idx = float(p[0]), float(p[1])
        if v > best_v or (v == best_v and idx < best_i):
            best_v, best_i = v, idx
    return best_v, int(best_i)


def sharded_pcg(kernel_rows, b_local: np.ndarray, n: int, prec_solve, dist, max_iters=100, rel_tol=1e-6):
    """Row-sharded batched PCG (krylov.hpp:47-129 per column).

    kernel_rows(P_full) -> this rank's rows of K_hat @ P_full (local x t);
    prec_solve(R_local) -> this rank's rows of P^-1 R (a row-local preconditioner, e.g. sigma^-2 I);
    b_local: this rank's rows of the right-hand sides (local x t).
    Returns (x_local, iterations per column, converged flags)."""
    t = b_local.shape[1]
    x = np.zeros_like(b_local)
    r = b_local.copy()
    z = prec_solve(r)
    rz = allreduce_sum_fixed(np.einsum("ij,ij->j", r, z), dist)
    norm0 = np.sqrt(allreduce_sum_fixed(np.einsum("ij,ij->j", z, z), dist))
    p = z.copy()
    active = norm0 > 0
    iters = np.zeros(t, dtype=int)
    conv = ~active
    for k in range(1, max_iters + 1):
        if not active.any():
            break
        p_full = allgather_rows(p, n, dist)          # all-gather of the direction block
        ap = kernel_rows(p_full)
        pap = allreduce_sum_fixed(np.einsum("ij,ij->j", p, ap), dist)
        alpha = np.where(active, rz / np.where(pap == 0, 1, pap), 0.0)
        if np.any(active & (~np.isfinite(alpha) | (alpha <= 0))):
            raise RuntimeError(f"pcg_solve: breakdown at iteration {k}")
        x += alpha * p
        r -= alpha * ap
        z = prec_solve(r)
        rz_new = allreduce_sum_fixed(np.einsum("ij,ij->j", r, z), dist)
        pres = np.sqrt(allreduce_sum_fixed(np.einsum("ij,ij->j", z, z), dist))
        iters[active] = k
        done = active & ((pres <= rel_tol * norm0) | (rz_new == 0))
        conv |= done
        active &= ~done
        beta = np.where(active, rz_new / np.where(rz == 0, 1, rz), 0.0)
        p = np.where(active, z + beta * p, p)
        rz = np.where(active, rz_new, rz)
    return x, iters, conv
