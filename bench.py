#!/usr/bin/env python
"""bench.py — seconds per mLL + gradient evaluation on the BASELINE workload.

One step = one optimizer step's hot path as optimize() runs it
(optimizer.hpp:448-453 begin_step + :437 objective):  KernelOperator at theta
(set data + params), pivoted-Cholesky preconditioner of rank k with frozen-
pivot derivative factors, and evaluate_mll (value + gradient) over [y, Z].

  value : device-resident inputs (X, y, Z already in HBM), gpk_*_device entry points
  e2e   : the reference-facing C-ABI with HOST buffers (H2D of X, y, Z and D2H of the
          result inside the timed region)

Default workload: BASELINE configs[1] (C2: n=16384, d=18, Matern-3/2, l=50,
rank 100; ranks 0 and 500 in "sweep").  --impl reference times the reference
algorithm's CPU restatement (oracle/, the reference itself cannot be built
here: Eigen is absent) on the host cores on a bounded sample, extrapolated to a
full evaluation.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2107_00243_b200 import workloads  # noqa: E402

METRIC = "s per mLL+gradient eval"
UNIT = "s/eval"


def fp64_peak():
    """Measured DMMA peak (tools/fp64_peak.py -> profiles/fp64_peak.json), else B200's nominal 40."""
    try:
        return float(json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["fp64_tflops"]), "measured"
    except Exception:
        return 40.0, "nominal B200 FP64 tensor (no measurement committed)"


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.device = device
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def __enter__(self):
        if self.device < 0:  # not the sampling rank
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for k, nm in enumerate(names):
                    if r[5 + k].strip().lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
class SingleComm:
    """N = 1: one process, one GPU."""
    rank, world, device = 0, 1, 0

    def create_ctx(self, lib, ctx):
        assert lib.gpk_create(self.device, C.byref(ctx)) == 0, "gpk_create failed"

    def barrier(self):
        pass

    def max(self, vals):
        return list(vals)


class DistComm:
    """One process per GPU (torchrun / the self-spawn below): the library's own NCCL
    communicator for the row-sharded evaluation, torch.distributed for barrier / max."""

    def __init__(self, rank, world, local):
        self.rank, self.world, self.device = rank, world, local

    def create_ctx(self, lib, ctx):
        import torch.distributed as dist

        uid = [None]
        if self.rank == 0:
            buf = C.create_string_buffer(128)
            assert lib.gpk_nccl_unique_id(buf) == 0
            uid[0] = buf.raw
        dist.broadcast_object_list(uid, src=0)
        ub = C.create_string_buffer(uid[0], 128)
        rc = lib.gpk_create_sharded(self.device, self.rank, self.world, ub, C.byref(ctx))
        assert rc == 0, f"gpk_create_sharded failed ({rc})"

    def barrier(self):
        import torch.distributed as dist

        dist.barrier()

    def max(self, vals):
        import torch
        import torch.distributed as dist

        t = torch.tensor(list(vals), dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()


class GroupComm:
    """TEST-ONLY (--comm group): the N ranks as host threads of one process on one GPU, the
    library's host-staged rank group (gpk_create_in_group) as the transport.  Exercises the
    same spawn / sharding / rank-ordered reduction / max-over-ranks logic as the NCCL path;
    its timings mean nothing (N ranks share one GPU)."""

    class Shared:
        def __init__(self, world, lib):
            g = C.c_void_p()
            assert lib.gpk_group_create(world, C.byref(g)) == 0
            self.g, self.world = g, world
            self.bar = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, shared, rank):
        self.sh, self.rank, self.world, self.device = shared, rank, shared.world, 0

    def create_ctx(self, lib, ctx):
        rc = lib.gpk_create_in_group(0, self.sh.g, self.rank, C.byref(ctx))
        assert rc == 0, f"gpk_create_in_group failed ({rc})"

    def barrier(self):
        self.sh.bar.wait()

    def max(self, vals):
        self.sh.slots[self.rank] = list(vals)
        self.sh.bar.wait()
        out = [max(s[i] for s in self.sh.slots) for i in range(len(vals))]
        self.sh.bar.wait()
        return out


def run_ours(args, comm):
    import torch

    from paper_2107_00243_b200 import capi

    rank, world, local = comm.rank, comm.world, comm.device
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = capi.lib()
    w = workloads.config(args.workload, rank=args.rank)
    x, y = workloads.generate(w)
    n, d, l = w.n, w.d, w.probes
    # replicas (N > 1): each rank evaluates with its own probe batch (optimizer step rank+1);
    # sharded: all ranks share the one evaluation's probes
    seed = int(lib.gpk_mix_seed(workloads.PROBE_SEED, 1 + (rank if args.mode == "replicas" else 0)))
    z = np.empty((n, l), order="F")
    assert lib.gpk_make_probes(n, l, C.c_uint64(seed), z.ctypes.data_as(C.POINTER(C.c_double))) == 0
    log_o, log_ls, log_noise = w.log_params
    log_ls = np.ascontiguousarray(log_ls)
    xf = np.asfortranarray(x)
    # pinned host copies for the e2e arm
    X_h = torch.from_numpy(np.ascontiguousarray(xf.T)).pin_memory()     # (d, n) == column-major n x d
    y_h = torch.from_numpy(y.copy()).pin_memory()
    Z_h = torch.from_numpy(np.ascontiguousarray(z.T)).pin_memory()      # (l, n) == column-major n x l
    X_d, y_d, Z_d = X_h.to(dev), y_h.to(dev), Z_h.to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > L2 (126 MB)

    ctx = C.c_void_p()
    if world > 1 and args.mode == "sharded":
        comm.create_ctx(lib, ctx)  # one evaluation row-sharded over all ranks
    else:
        assert lib.gpk_create(local, C.byref(ctx)) == 0, "gpk_create failed"
    stream = torch.cuda.ExternalStream(lib.gpk_stream(ctx), device=dev)
    prec = {"fp64": capi.GPK_PREC_FP64, "fp32": capi.GPK_PREC_FP32, "tf32x3": capi.GPK_PREC_TF32X3}[args.precision]
    cfg = capi.gpk_mll_cfg(capi.gpk_cg_cfg(w.max_iters, w.rel_tol, 0, prec, args.refine), 1, 1,
                           {"fused": 0, "faithful": 1, "auto": 2}[args.backward])
    grad = np.zeros(d + 2)
    fg = np.zeros(l)
    fi = np.zeros(l, dtype=np.int32)
    res = capi.gpk_mll_result()
    res.gradient = grad.ctypes.data_as(C.POINTER(C.c_double))
    res.forward_gammas = fg.ctypes.data_as(C.POINTER(C.c_double))
    res.forward_cg_iterations = fi.ctypes.data_as(C.POINTER(C.c_int))
    Dp = C.POINTER(C.c_double)

    def check(rc):
        if rc != 0:
            raise RuntimeError(lib.gpk_last_error(ctx).decode())

    def step_device(rank_k):
        check(lib.gpk_set_data_device(ctx, C.c_void_p(X_d.data_ptr()), n, d, n))
        check(lib.gpk_set_params(ctx, w.family, 1.0, log_o, log_ls.ctypes.data_as(Dp), log_noise))
        if rank_k < 0:
            check(lib.gpk_precond_identity(ctx))
        else:
            check(lib.gpk_pivoted_cholesky(ctx, rank_k, 0.0, w.noise, None, None, None))
            check(lib.gpk_precond_deriv_factors(ctx))
        check(lib.gpk_evaluate_mll_device(ctx, C.c_void_p(y_d.data_ptr()), C.c_void_p(Z_d.data_ptr()), n, l,
                                          C.c_uint64(seed), C.byref(cfg), C.byref(res)))

    def step_host(rank_k):
        check(lib.gpk_set_data(ctx, X_h.numpy().ctypes.data_as(Dp), n, d, n))
        check(lib.gpk_set_params(ctx, w.family, 1.0, log_o, log_ls.ctypes.data_as(Dp), log_noise))
        check(lib.gpk_pivoted_cholesky(ctx, rank_k, 0.0, w.noise, None, None, None))
        check(lib.gpk_precond_deriv_factors(ctx))
        check(lib.gpk_evaluate_mll(ctx, y_h.numpy().ctypes.data_as(Dp), Z_h.numpy().ctypes.data_as(Dp), n, l,
                                   C.c_uint64(seed), C.byref(cfg), C.byref(res)))

    def timed(fn, steps, warmup, rank_k):
        for _ in range(warmup):
            fn(rank_k)
        torch.cuda.synchronize()
        comm.barrier()
        times = []
        l0 = lib.gpk_launch_count(ctx)
        check(lib.gpk_profile_reset(ctx))
        for _ in range(steps):
            flush.zero_()  # flush L2 between timed iterations (outside the timed region)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn(rank_k)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        torch.cuda.synchronize()
        comm.barrier()
        launches = (lib.gpk_launch_count(ctx) - l0) // steps
        return times, launches

    # ---- headline: device-resident value, with live per-launch kernel timing
    check(lib.gpk_profile_enable(ctx, 0 if os.environ.get("GPK_BENCH_NOPROF") else 1))
    with ClockSampler(local if rank == 0 else -1) as clk:
        times, launches = timed(step_device, args.steps, args.warmup, w.rank)
    ms = C.c_double()
    cnt = C.c_longlong()
    fl = C.c_double()
    en = C.c_double()
    check(lib.gpk_profile_read(ctx, 0, C.byref(ms), C.byref(cnt), C.byref(fl), C.byref(en)))
    mvm = {"ms": ms.value, "launches": cnt.value, "flops": fl.value}
    check(lib.gpk_profile_read(ctx, 1, C.byref(ms), C.byref(cnt), C.byref(fl), C.byref(en)))
    dc = {"ms": ms.value, "launches": cnt.value, "flops": fl.value}
    # secondary kernels (fp64 MVM, CG vector phase): their events cost ~2% of the step, so they
    # are recorded in a separate diagnostic pass of the same step, not in the headline region
    check(lib.gpk_profile_enable(ctx, 12))
    timed(step_device, args.steps, 1, w.rank)
    check(lib.gpk_profile_read(ctx, 2, C.byref(ms), C.byref(cnt), C.byref(fl), C.byref(en)))
    f64 = {"ms": ms.value, "launches": cnt.value, "flops": fl.value, "entries": en.value}
    check(lib.gpk_profile_read(ctx, 3, C.byref(ms), C.byref(cnt), C.byref(fl), C.byref(en)))
    vec = {"ms": ms.value, "launches": cnt.value, "bytes": fl.value, "cols": en.value}
    check(lib.gpk_profile_enable(ctx, 0))
    var, maxnorm = C.c_int(), C.c_double()
    check(lib.gpk_get_mvm_variant(ctx, C.byref(var), C.byref(maxnorm)))
    mvm_variant = {1: "direct", 2: "gram"}.get(var.value, "direct")
    telemetry = {"value": res.value, "gradient": grad.tolist(), "logdet": res.logdet,
                 "solve_iterations": res.solve_iterations, "total_cg_iterations": res.total_cg_iterations,
                 "forward_cg_iterations_mean": float(np.mean(fi)), "refine_passes": res.refine_passes,
                 "max_true_rel_residual": res.max_true_rel_residual,
                 "max_cg_rel_residual": res.max_cg_rel_residual, "unconverged_columns": res.unconverged_columns,
                 "seconds_solve": res.seconds_solve,
                 "seconds_backward": res.seconds_backward,
                 "backward_mode_used": ("fused", "faithful")[res.backward_mode_used]}
    # ---- e2e through the host C-ABI
    e2e_times, _ = timed(step_host, max(1, args.steps), 1, w.rank)
    sweep = {}
    if not args.no_sweep and w.ranks:
        for rk in w.ranks:
            if rk == w.rank:
                continue
            tt, _ = timed(step_device, 1, 1, rk)
            sweep[str(rk)] = {"s_per_eval": tt[0], "total_cg_iterations": res.total_cg_iterations,
                              "value": res.value}
    lib.gpk_destroy(ctx)
    h2d = X_h.numel() * 8 + y_h.numel() * 8 + Z_h.numel() * 8
    d2h = 8 * (d + 2) + 8 * l + 4 * l + 8 * 8
    return dict(times=times, e2e_times=e2e_times, mean_step=float(np.mean(times)),
                mean_e2e=float(np.mean(e2e_times)), launches=launches, mvm=mvm, dc=dc, f64=f64, vec=vec,
                clocks=clk.summary(),
                mvm_variant=mvm_variant,
                telemetry=telemetry, sweep=sweep, h2d=h2d, d2h=d2h, w=w)


# ---------------------------------------------------------------------------
# CPU arm: the reference algorithm's restatement (oracle/) on the host cores
# ---------------------------------------------------------------------------
def reference_iterations(w, gpu_fwd_mean=None):
    """CG iteration counts of the REFERENCE evaluation of workload w (evaluate_mll,
    gp_likelihood.hpp:51-103): the oracle's own counts from the committed golden fixture when
    there is one (C2 ranks 0/100/500, tests/golden/c2_oracle_rank*.json); otherwise the GPU
    run's measured forward mean for every solve (C3-C5 hit the 200-iteration cap), labelled."""
    g = os.path.join(ROOT, "tests", "golden", f"{w.name.lower()}_oracle_rank{w.rank}.json")
    l, d = w.probes, w.d
    if os.path.exists(g):
        gj = json.load(open(g))
        fwd = gj["forward_cg_iterations"]
        return {"y": gj["solve_iterations"], "fwd_total": int(sum(fwd)),
                "bwd_total": int(gj["total_cg_iterations"] - gj["solve_iterations"] - sum(fwd)),
                "source": f"oracle golden {os.path.relpath(g, ROOT)} (the reference algorithm's own counts)"}
    table = os.path.join(ROOT, "profiles", "iteration_counts.json")
    m = None
    if gpu_fwd_mean:
        m, src = float(gpu_fwd_mean), "this run's GPU forward mean (every solve assumed alike)"
    elif os.path.exists(table) and w.name in json.load(open(table)):
        m, src = float(json.load(open(table))[w.name]["forward_mean"]), "profiles/iteration_counts.json (GPU-measured)"
    else:
        m, src = float(w.max_iters), "max_iters (no measured count available)"
    return {"y": m, "fwd_total": m * l, "bwd_total": m * (d + 1) * l, "source": src}


def cpu_sample(w, its, budget_s=20.0):
    """Times MatrixFree applies (kernels.hpp:184-195, 1024-row blocks) with OpenMP over
    columns (the reference's probe parallelism, krylov.hpp:141 / trace_estimation.hpp:163)
    and extrapolates the reference's apply count for one evaluate_mll from its CG iteration
    counts `its` (reference_iterations)."""
    import oracle

    cores = oracle.num_threads()
    x, y = workloads.generate(w)
    p = oracle.Params(w.d, w.outputscale, lengthscales=w.lengthscales, noise=w.noise)
    n = w.n
    # bounded sample: rows subset so that one apply on each core takes ~budget/2
    t_cols = cores
    v = np.asfortranarray(np.random.default_rng(0).standard_normal((n, t_cols)))
    rows = min(n, 2048)
    xs = x[:rows]
    t0 = time.perf_counter()
    oracle.kernel_apply_parallel(w.family, xs, p, v[:rows, :t_cols])
    t_small = time.perf_counter() - t0
    # per-apply time scales with rows^2 (n^2 entries per apply)
    t_apply = t_small * (n / rows) ** 2
    sample = f"{t_cols} concurrent MatrixFree applies on {rows} of {n} rows (oracle port), scaled by (n/rows)^2"
    if t_apply < budget_s:  # full-size sample fits the budget: measure it directly
        t0 = time.perf_counter()
        oracle.kernel_apply_parallel(w.family, x, p, v)
        t_apply = time.perf_counter() - t0
        sample = f"{t_cols} concurrent full-size MatrixFree applies (n={n}, oracle port)"
    l, d = w.probes, w.d
    par = min(cores, l)
    # wall-clock apply rounds of evaluate_mll: the y solve runs alone; the probe solves of a phase
    # run `par` at a time (OpenMP over probes); every trace_residual also applies dK_w to its l
    # probes, and deriv_apply(w, u) runs alone, for the d+1 non-noise parameters
    rounds = (its["y"] + its["fwd_total"] / par + its["bwd_total"] / par
              + (d + 1) * (math.ceil(l / par) + 1))
    return {"value": rounds * t_apply, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": sample + f"; extrapolated x{rounds:.0f} apply rounds",
            "iterations": its, "seconds_per_apply_round": t_apply, "extrapolated": True}


def cpu_c1_measured():
    """The BASELINE C1 evaluation (configs[0], the reference's CPU-runnable case) run IN FULL by
    the oracle port on the host cores: pivoted Cholesky + derivative factors + evaluate_mll,
    MatrixFree (the reference's operator, optimizer.hpp:427 picks Dense for n <= 4096; both
    modes are in the oracle), max 100 iterations as configured."""
    import oracle

    w = workloads.config("C1")
    x, y = workloads.generate(w)
    p = oracle.Params(w.d, w.outputscale, lengthscales=w.lengthscales, noise=w.noise)
    seed = oracle.mix_seed(workloads.PROBE_SEED, 1)
    z = oracle.make_probes(w.n, w.probes, seed)
    out = {}
    for mode, name in ((oracle.DENSE, "dense"), (oracle.MATRIX_FREE, "matrix_free")):
        t0 = time.perf_counter()
        r = oracle.evaluate_mll(w.family, x, p, y, z, seed=seed, prec="pivchol", rank=w.rank, mode=mode,
                                max_iters=w.max_iters, rel_tol=w.rel_tol)
        out[name] = {"seconds": time.perf_counter() - t0, "value": r["value"],
                     "total_cg_iterations": r["total_cg_iterations"]}
    return {"workload": "C1 (n=2048 d=3 rbf l=8 rank=16 max_iters=100)", "measured": True,
            "cores": oracle.num_threads(), "kind": "port", **out}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
def spawn(args):
    """--gpus N without a launcher: re-exec this script under torch.distributed.run, one rank
    per GPU (the driver's own launch form), after checking N GPUs are visible."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible", file=sys.stderr)
        return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--rank", type=int, default=None)
    ap.add_argument("--precision", default="tf32x3", choices=["tf32x3", "fp32", "fp64"])
    ap.add_argument("--backward", default="auto", choices=["auto", "fused", "faithful"])
    ap.add_argument("--refine", type=int, default=2)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--mode", default="sharded", choices=["sharded", "replicas"],
                    help="N>1: one row-sharded evaluation over N GPUs (NCCL) or N independent replicas")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "group"],
                    help="TEST ONLY 'group': the N ranks as threads on one GPU over the host-staged rank group")
    ap.add_argument("--cpu-c1", action="store_true", help="reference arm: also run the full C1 evaluation")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    env_world = os.environ.get("WORLD_SIZE")
    rank = int(os.environ.get("RANK", "0"))
    world = int(env_world or "1")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    peaks, peaks_src = load_peaks()
    w = workloads.config(args.workload, rank=args.rank)

    if args.impl == "reference":
        if rank != 0:  # under torchrun rank 0 alone runs the CPU reference arm
            return 0
        its = reference_iterations(w)
        cb = cpu_sample(w, its)
        cb["cpu_model"] = cpu_model()
        if args.cpu_c1 or w.name == "C1":
            cb["c1_full_evaluation"] = cpu_c1_measured()
        cfg = config_of(w, args, world if env_world else args.gpus)
        line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "impl": "reference", "n_gpus": 0,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["value"] * 1e3,
                "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded stand-in for the BASELINE config)", "config": cfg,
                "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                                            "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    if env_world is None and args.gpus > 1 and args.comm == "nccl":
        return spawn(args)
    if env_world is not None and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2

    if args.comm == "group" and args.gpus > 1:
        import torch  # noqa: F401  (before the library: torch's bundled NCCL must load first)

        from paper_2107_00243_b200 import capi

        shared = GroupComm.Shared(args.gpus, capi.lib())
        results, errs = [None] * args.gpus, []

        def body(r):
            try:
                results[r] = run_ours(args, GroupComm(shared, r))
            except Exception as e:  # noqa: BLE001
                errs.append(e)
                shared.bar.abort()

        th = [threading.Thread(target=body, args=(r,)) for r in range(args.gpus)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]
        comm = GroupComm(shared, 0)
        world = args.gpus
        r = results[0]
        r["max_times"] = [max(res["mean_step"] for res in results), max(res["mean_e2e"] for res in results)]
    elif world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
        comm = DistComm(rank, world, local)
        r = run_ours(args, comm)
        r["max_times"] = comm.max([r["mean_step"], r["mean_e2e"]])
    else:
        comm = SingleComm()
        r = run_ours(args, comm)
        r["max_times"] = [r["mean_step"], r["mean_e2e"]]
    per_step, e2e = r["max_times"]  # max over ranks of each rank's device-timed mean
    # replicas: N independent evaluations per step -> whole-job seconds per evaluation
    # sharded: one evaluation across all GPUs (strong scaling)
    div = world if args.mode == "replicas" else 1
    value = per_step / div
    e2e_value = e2e / div
    mvm = r["mvm"]
    mhz = float(peaks.get("sm_max_mhz", 1965.0))
    achieved = (mvm["flops"] / mvm["launches"]) / (mvm["ms"] / mvm["launches"] / 1e3) / 1e12 if mvm["launches"] else 0
    clk = r["clocks"]
    tc = args.precision == "tf32x3"
    gram = tc and r["mvm_variant"] == "gram"
    t_cols = w.probes + 1
    npad = 8 * ((t_cols + 7) // 8)
    ks = (w.d + 2 + 7) // 8  # Gram k-steps over the augmented coordinates [x~, 1, n]
    common = {"flops_per_launch": mvm["flops"] / max(mvm["launches"], 1),
              "avg_launch_ms": mvm["ms"] / max(mvm["launches"], 1),
              "launches_per_step": mvm["launches"] / max(args.steps, 1),
              "share_of_step": (mvm["ms"] / 1e3) / max(sum(r["times"]), 1e-12)}
    entries_per_s = w.n * w.n * mvm["launches"] / (mvm["ms"] / 1e3) if mvm["launches"] else 0.0
    if tc:
        # both contractions run on the 5th-gen tensor cores: the roofline is the measured dense
        # tensor peak (MEASURED_PEAKS.json bf16, the f16 kind's rate); achieved = ALGORITHMIC flops
        tpeak = float(peaks.get("bf16_tflops", 1656.1))
        roofline = {"bound": "tensor", "achieved": achieved, "peak": tpeak, "unit": "TFLOP/s",
                    "frac": achieved / tpeak, "traffic": None,
                    "kernel": ("fused_kmvm_tcg_kernel (Gram distances 3xTF32 + 3xF16 contraction on tcgen05, "
                               "kernel shape on the SFU)" if gram else
                               "fused_kmvm_tc_kernel (3xTF32 contraction on tcgen05, entries on CUDA cores)"),
                    "peak_source": f"{peaks_src} MEASURED_PEAKS.json bf16_tflops (dense, burst); achieved = "
                                   f"algorithmic flops n^2 (2t + 3d + c_fam) per launch / CUDA-event launch time",
                    **common}
        if gram:
            # hardware tensor work actually issued per entry: Gram 3 x 2 x 8 KS (tf32, half rate) and the
            # contraction 3 x 2 x NPAD (f16)
            hw_f16_equiv = 2 * (3 * 2 * 8 * ks) + 3 * 2 * npad
            roofline["tensor_issued"] = {"f16_equiv_flops_per_entry": hw_f16_equiv,
                                         "achieved": entries_per_s * hw_f16_equiv / 1e12,
                                         "frac": entries_per_s * hw_f16_equiv / 1e12 / tpeak}
            # the binding unit: the SFU evaluates the kernel shape (2 MUFU per entry; RBF 1) at 16/clk/SM
            mufu = 1 if w.family == 0 else 2
            sfu_peak = 148 * 16 * mhz * 1e6 / mufu
            roofline["sfu_bound"] = {"mufu_per_entry": mufu, "peak_entries_per_s": sfu_peak,
                                     "entries_per_s": entries_per_s, "frac": entries_per_s / sfu_peak}
            # the tensor pipe's instruction floor: every tcgen05.mma with M = 128, N <= 96 costs ~51 cycles
            # (tools/ubench_umma.cu, profiles/r2_mvm_pipeline_experiments.txt); per 128 x 64 tile the kernel
            # issues 12 contraction MMAs (4 k-steps x {hi hi, hi lo, lo hi}) + 3 KS Gram MMAs
            mmas = 12 + 3 * ks
            floor_entries = 148 * mhz * 1e6 * (128 * 64) / (mmas * 51.0)
            roofline["tensor_pipe_floor"] = {"mma_per_tile": mmas, "cycles_per_mma": 51.0,
                                             "peak_entries_per_s": floor_entries,
                                             "frac": entries_per_s / floor_entries,
                                             "source": "measured instruction cost (ubench_umma), not a vendor peak"}
    else:
        fp32_peak = 148 * 128 * 2 * mhz * 1e6 / 1e12
        roofline = {"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                    "frac": achieved / fp32_peak, "traffic": None, "kernel": "fused_kmvm_kernel (SIMT fp32)",
                    "peak_source": "FP32 CUDA-core peak = 148 SM x 128 FMA/clk x 2 x sm_max_mhz", **common}
    if clk.get("sm_mhz") and roofline["bound"] == "fp32":
        roofline["frac_at_inrun_clock"] = achieved / (148 * 128 * 2 * clk["sm_mhz"] * 1e6 / 1e12)
    roofline["entries_per_s"] = entries_per_s
    # DRAM traffic per launch of this kernel from the committed ncu --set full capture (same config)
    tfile = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "mvm_traffic.json")
    if os.path.exists(tfile):
        tr = json.load(open(tfile))
        if tr.get("workload") == w.name and tr.get("variant") == r["mvm_variant"]:
            roofline["traffic"] = tr["dram_bytes_per_launch"]
            roofline["traffic_source"] = tr.get("source")
    dcp = r["dc"]
    if dcp["launches"]:
        roofline["deriv_pass"] = {"achieved": (dcp["flops"] / dcp["ms"] * 1e3) / 1e12, "unit": "TFLOP/s",
                                  "avg_launch_ms": dcp["ms"] / dcp["launches"],
                                  "share_of_step": (dcp["ms"] / 1e3) / max(sum(r["times"]), 1e-12)}
    f64 = r.get("f64", {})
    if f64.get("launches"):
        # certified fp64 residual / fp64 parity operator: Gram + contraction on DMMA, entries on the
        # FP64 pipe; algorithmic flops n^2 (2t + 3d + c_fam)
        roofline["fp64_mvm"] = {"kernel": "fused_kmvm_f64g_kernel (DMMA 8x8x4 Gram + contraction, fp64 entries)",
                                "avg_launch_ms": f64["ms"] / f64["launches"], "launches_per_step":
                                f64["launches"] / max(args.steps, 1),
                                "achieved": (f64["flops"] / f64["ms"] * 1e3) / 1e12, "unit": "TFLOP/s",
                                "entries_per_s": f64["entries"] / (f64["ms"] / 1e3),
                                "share_of_step": (f64["ms"] / 1e3) / max(sum(r["times"]), 1e-12)}
    vec = r.get("vec", {})
    if vec.get("launches"):
        # the fused single-rank CG vector phase (alpha, x/r update + Woodbury G1, G2 + beta, p update)
        # against the measured HBM copy bandwidth; algorithmic bytes = 13 fp64 n-vectors per active
        # column + L and C per iteration (the operands are L2-resident at C2: latency-bound there)
        hbm = float(peaks.get("hbm_gbs", 6538.3))
        ach = vec["bytes"] / (vec["ms"] / 1e3) / 1e9
        # the Woodbury products G1 = L^T r and G2 = C W are 4 n k t fp64 flops per iteration on
        # the DMMA pipe; at large k they bind before HBM does (C4: 44 GFLOP vs 5.3 GB)
        f64p, f64src = fp64_peak()
        wflops = 4.0 * w.n * w.rank * vec.get("cols", 0.0)
        t_hbm = vec["bytes"] / (hbm * 1e9)
        t_f64 = wflops / (f64p * 1e12)
        roofline["cg_vector_phase"] = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                                       "frac": ach / hbm, "avg_ms_per_iteration": vec["ms"] / vec["launches"],
                                       "bytes_per_iteration": vec["bytes"] / vec["launches"],
                                       "woodbury_fp64_flops_per_iteration": wflops / vec["launches"],
                                       "fp64_tensor_peak_tflops": f64p, "fp64_peak_source": f64src,
                                       "binding": "fp64_tensor" if t_f64 > t_hbm else "hbm",
                                       "frac_of_binding_roofline": max(t_hbm, t_f64) / (vec["ms"] / 1e3),
                                       "iterations_per_step": vec["launches"] / max(args.steps, 1),
                                       "share_of_step": (vec["ms"] / 1e3) / max(sum(r["times"]), 1e-12)}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": False,
            "scaling": "weak" if (world == 1 or args.mode == "replicas") else "strong", "vs_baseline": None,
            "dtype": {"fp64": "f64", "fp32": "f32 entries+contraction / f64 CG state",
                      "tf32x3": "f32 entries; tcgen05 contraction in 3xF16 hi/lo (22 significant bits, Gram "
                                "path; 3xTF32 on the direct path) / f64 CG state"}[args.precision],
            "data": "synthetic (seeded stand-in for the BASELINE config; UCI data unavailable offline)",
            "config": config_of(w, args, world), "gpu_launches": r["launches"],
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"]},
            "roofline": roofline, "clocks": {"sm_mhz": clk.get("sm_mhz"), "sm_max_mhz": clk.get("sm_max_mhz"),
                                             "reasons": clk.get("reasons", [])},
            "telemetry": r["telemetry"], "sweep": r["sweep"]}
    if args.comm == "group":
        line["comm"] = "group (TEST ONLY: ranks are threads on one GPU, host-staged collectives)"
    if rank == 0 and world == 1 and not args.no_cpu:
        its = reference_iterations(w, None if os.path.exists(os.path.join(
            ROOT, "tests", "golden", f"{w.name.lower()}_oracle_rank{w.rank}.json")) else
            r["telemetry"]["forward_cg_iterations_mean"])
        cb = cpu_sample(w, its)
        cb["cpu_model"] = cpu_model()
        line["cpu_baseline"] = cb
    if rank == 0:
        print(json.dumps(line))
    if world > 1 and args.comm == "nccl":
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def config_of(w, args, world):
    return {"workload": f"{w.name}: n={w.n} d={w.d} {['rbf', 'matern12', 'matern32', 'matern52'][w.family]} "
                        f"l={w.probes} rank={w.rank} max_iters={w.max_iters} tol={w.rel_tol}",
            "n": w.n, "d": w.d, "probes": w.probes, "precond_rank": w.rank, "precision": args.precision,
            "backward": args.backward, "l2": "flushed between timed steps (256 MB write)",
            "step": "set_data + set_params + pivoted_cholesky(+deriv factors) + evaluate_mll(value+grad)",
            "parallelism": (f"row-sharded x{world} (NCCL)" if args.mode == "sharded" else f"replicas x{world}")
            if world > 1 else "1 GPU"}


if __name__ == "__main__":
    sys.exit(main())
