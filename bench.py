"""Benchmark: one HG cost+gradient evaluation per step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]
                    [--replicas] [--no-secondary]

A step is one full composite_grad evaluation of the workload config.  The default is c4, the
largest single-GPU configuration of BASELINE.json (two transmons x cavity 400, d = 10^4, 4 controls,
K = 32 X-gate subspace, N = 4000): BASELINE's metric is quoted on no config, so the N = 1 line is the
largest one that fits one GPU.  ``value`` is device-timed (amplitudes resident in HBM,
CUDA events on the library's launch stream); ``e2e`` goes through the public API with host buffers
(H2D of the amplitudes, D2H of cost and gradient inside the timed region).  The L2 is flushed
(256 MiB write) between timed evaluations.

``--gpus N`` (N > 1): one process per GPU.  Launched by torchrun (the driver) it reads
RANK/WORLD_SIZE; launched directly it re-executes itself under ``torch.distributed.run``.  The
default multi-GPU mode is the north star's: the K-state block SHARDED over the ranks with one NCCL
all-reduce per evaluation (distributed.ShardedEvaluator, ``scaling: strong``); ``--replicas`` runs
N independent replicas instead (``scaling: weak``).

``--impl reference`` times the reference algorithm on the host cores: the CPU oracle port
(oracle/lg_oracle.py; the reference package is pure Python and cannot travel to the GPU box), one
process per (trajectory, cost term), on a bounded sample of the same workload (a prefix of N steps
and, for large K, a subset of the trajectories, one per core), extrapolated linearly to the full
N x K (trajectories are independent; per-step cost is constant: one plan per config).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cost+gradient evals/sec"
UNIT = "evals/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 6:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def fp64_dgemm_peak():
    """Measured FP64 tensor peak of this GPU: cuBLAS DGEMM 8192^3 (best of 5, CUDA events).
    MEASURED_PEAKS.json carries no FP64 figure; this is the roofline denominator of the dense
    (DMMA) engine."""
    import torch

    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(5):
        s.record()
        a @ b
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    del a, b
    return 2 * 8192 ** 3 / (best / 1e3) / 1e12


def algorithmic_bytes(case, plan_table):
    """bytes per operator-term = S_op + 32 d K (S_op = 20 nnz + 4 (d+1)
    for CSR, 16 d^2 dense); A-terms = sum_n mu_n (fwd) + sum_n mu_n (psi adjoint) +
    sum_{n>0} mu_n n_costates + sum_{n,c} 2 mu_aux_{n,c}; A_c-terms = sum_{n,c} mu_aux_{n,c}.
    Returns (total bytes per evaluation, backward-sweep bytes per evaluation, flops)."""
    p = case.problem
    d = p.dim

    def s_op(m):
        if hasattr(m, "array"):
            return 16 * d * d, d * d
        return 20 * m.nnz + 4 * (d + 1), m.nnz

    union = None
    try:
        from paper_2304_06200_b200.sparse import linear_combine

        union = linear_combine([1.0] + [1.0] * len(p.h_controls), [p.h_static, *p.h_controls])
    except Exception:
        union = p.h_static
    sa, nnz_a = s_op(union)
    sc = [s_op(h) for h in p.h_controls]
    K = case.n_states
    n_costates = sum(1 for t in case.terms)  # one costate per term per trajectory
    mu = plan_table["m"].astype(np.int64) * plan_table["s"]
    mua = plan_table["aux_m"].astype(np.int64) * plan_table["aux_s"]
    blk = 32 * d * K
    fwd_terms = int(mu.sum())
    bwd_a = int(mu.sum() + mu[1:].sum() * n_costates + 2 * mua.sum())
    bwd_c = mua.sum(axis=0)
    bwd_bytes = bwd_a * (sa + blk) + sum(int(bwd_c[c]) * (sc[c][0] + blk) for c in range(len(sc)))
    fwd_bytes = fwd_terms * (sa + blk)
    flops = 8 * K * ((fwd_terms + bwd_a) * nnz_a + sum(int(bwd_c[c]) * sc[c][1] for c in range(len(sc))))
    return fwd_bytes + bwd_bytes, bwd_bytes, flops


def committed_traffic(workload, kernel, n_steps):
    """DRAM bytes per launch of the dominant kernel from the newest committed ncu --set full capture
    (profiles/r02_traffic.json, else r01: dram__bytes_read.sum + dram__bytes_write.sum), scaled to
    n_steps when the capture ran on a prefix.  None when no capture of this kernel/workload exists."""
    for rnd in ("r02", "r01"):
        try:
            with open(os.path.join(ROOT, "profiles", f"{rnd}_traffic.json")) as fh:
                t = json.load(fh).get(workload)
        except Exception:
            continue
        if not t or t["kernel"] not in kernel:
            continue
        return t["dram_bytes_per_launch"] * n_steps / t["n_steps_captured"], t["source"]
    return None, None


def committed_smem_wavefronts(workload, kernel, n_steps):
    """Shared-memory wavefronts per launch of the dominant kernel from the same committed capture
    (profiles/r02_traffic.json: l1tex__data_pipe_lsu_wavefronts_mem_shared.sum), scaled to n_steps."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as fh:
            t = json.load(fh).get(workload)
    except Exception:
        return None
    if not t or t["kernel"] not in kernel or "smem_wavefronts_per_launch" not in t:
        return None
    return t["smem_wavefronts_per_launch"] * n_steps / t["n_steps_captured"]


def critical_path_terms(plan_table):
    """Sequentially dependent operator-terms of one evaluation: the forward chain
    N*mu, then per backward step the adjoint chain mu plus the aux chain mu_aux (channels sharing a
    plan run as one chain)."""
    mu = plan_table["m"].astype(np.int64) * plan_table["s"]
    mua = (plan_table["aux_m"].astype(np.int64) * plan_table["aux_s"]).max(axis=1)
    return int(mu.sum() + mu.sum() + mua.sum())




def workload_config(case, world, mode):
    """The `config` object, identical in both arms for the same workload and N."""
    par = {"shard": f"trajectory shards x{world} (one NCCL all-reduce per evaluation)",
           "replicas": f"replicas x{world}", "single": "single"}[mode]
    return {"workload": case.name, "description": case.description, "n_steps": case.field.n_steps,
            "n_states": case.n_states, "parallelism": par,
            "l2": "flushed (256 MiB write) between timed evaluations"}


def _mode(args, world):
    return "single" if world == 1 else ("replicas" if args.replicas else "shard")


def cpu_reference(case, budget_s=20.0, max_items=None):
    """Time the oracle port of the reference algorithm on a bounded sample, one process per
    (trajectory, cost term): the composite is a weighted sum of per-term passes
    (src/costs.py:515-546) and the trajectories are independent, so every pass of every trajectory is
    independent work for the host cores.  The sample is a prefix of n_pref steps of the first
    trajectories (at most one item per core); the time is extrapolated linearly to all N steps and
    all trajectories.  Returns (evals_per_s_extrapolated, cores, sample description)."""
    import multiprocessing as mp

    N = case.field.n_steps
    T, nt = case.n_states, len(case.terms)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    cap = max(1, max_items or cores)
    t_sample = max(1, min(T, cap // max(nt, 1)))
    items_all = T * nt
    # probe one step to size the sample to ~budget_s of CPU work per item
    t0 = time.perf_counter()
    _ref_traj_worker((case.name, 0, 2, None))
    per_step = (time.perf_counter() - t0) / 2
    n_pref = int(max(2, min(N, budget_s / max(per_step, 1e-6))))
    items = [(case.name, t, n_pref, ti) for t in range(t_sample) for ti in range(nt)]
    procs = max(1, min(len(items), cores))
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(procs) as pool:
        pool.map(_ref_traj_worker, items, chunksize=1)
    wall = time.perf_counter() - t0
    per_eval = wall * (N / n_pref) * (items_all / len(items))
    sample = (f"oracle port of the reference (oracle/lg_oracle.py): {t_sample}/{T} trajectories x {nt} cost-term "
              f"passes x {n_pref}/{N} steps in {procs} processes, {wall:.1f}s wall, extrapolated linearly to "
              f"N={N} x K={T}")
    return 1.0 / per_eval, procs, sample


def _ref_traj_worker(arg):
    """One trajectory's forward+backward with the oracle (the reference algorithm), for one cost
    term (ti) or all of them (ti None)."""
    name, t, n_pref, ti = arg
    from oracle import lg_oracle as O
    from paper_2304_06200_b200 import models

    case = models.build_case(name, n_steps=n_pref)
    p = case.problem

    def conv(m):
        if hasattr(m, "array"):
            return O.Dense(np.asfortranarray(m.array))
        return O.Csr(m.n_rows, m.row_offsets, m.col_indices, m.values)

    states = p.initial_state if p.initial_state is not None else p.basis
    op = O.Problem(conv(p.h_static), tuple(conv(h) for h in p.h_controls), tau=p.tau,
                   initial_states=np.asarray(states)[t:t + 1],
                   basis=None if p.basis is None else np.asarray(p.basis)[t:t + 1])
    terms = []
    for term in case.terms:
        k = term.kind.value
        if term.penalty_op is not None:
            terms.append(O.Term(k, term.weight, None, conv(term.penalty_op)))
        else:
            tg = term.target_state if term.target_state is not None else term.target_images
            terms.append(O.Term(k, term.weight, np.asarray(tg)[t:t + 1]))
    if ti is not None:
        terms = [terms[ti]]
    O.composite_grad(op, case.field.amplitudes, case.field.dt, terms)
    return t


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from paper_2304_06200_b200 import models

    case = models.build_case(args.config)
    vals, cores, sample = [], 1, ""
    for i in range(args.warmup + args.steps):
        v, cores, sample = cpu_reference(case, budget_s=args.ref_budget)
        if i >= args.warmup:
            vals.append(v)
    value = float(statistics.median(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / value, "higher_is_better": True,
        "scaling": "weak" if _mode(args, world) != "shard" else "strong", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic", "config": workload_config(case, world, _mode(args, world)),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


class DeviceRun:
    """Device-timed evaluations of one case through lg_eval_device (amplitudes resident in HBM)."""

    def __init__(self, case, lib, local, shard=False):
        import torch

        from paper_2304_06200_b200 import _native
        from paper_2304_06200_b200.costs import NativeProblem
        from paper_2304_06200_b200.distributed import ShardedEvaluator

        self.case, self.lib, self._n = case, lib, _native
        p = case.problem
        N, Kc = case.field.n_steps, case.field.n_channels
        has_state = any(t.kind.value.startswith("state") for t in case.terms)
        self.stream = torch.cuda.current_stream()
        if shard:
            self.ev = ShardedEvaluator(p, case.terms, device=local)
            self.npb = self.ev.native
            self.ev._lend(N)
            self.share = (self.ev.shard[1] - self.ev.shard[0]) / max(self.ev.n_traj, 1)
            self.eval = lambda: self.ev.grad(case.field)
        else:
            self.npb = NativeProblem(p, case.terms, initial_states=p.initial_state if has_state else None,
                                     basis=p.basis, device=local)
            _native.check(lib.lg_set_stream(self.npb.handle, self.stream.cuda_stream))
            self.d_amps = torch.from_numpy(case.field.amplitudes).cuda()
            self.d_cost = torch.zeros(1, dtype=torch.float64, device="cuda")
            self.d_grad = torch.zeros((N, Kc), dtype=torch.float64, device="cuda")
            self.share = 1.0
            self.eval = lambda: _native.check(lib.lg_eval_device(
                self.npb.handle, N, case.field.dt, self.d_amps.data_ptr(), self.d_cost.data_ptr(),
                self.d_grad.data_ptr()))

    def timed(self, steps, warmup, flush, barrier=None, clocks=None):
        """Returns (per-step ms list, launches, phase ms per eval [4], n evals timed)."""
        import contextlib

        import torch

        _native = self._n
        for _ in range(warmup):
            self.eval()
        torch.cuda.synchronize()
        _native.check(self.lib.lg_set_timing(self.npb.handle, 1))
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        if barrier:
            barrier()
        torch.cuda.synchronize()
        launches0 = self.lib.lg_launch_count()
        with (clocks if clocks is not None else contextlib.nullcontext()):
            for i in range(steps):
                flush.fill_(float(i))
                starts[i].record(self.stream)
                self.eval()
                ends[i].record(self.stream)
            torch.cuda.synchronize()
        launches = int(self.lib.lg_launch_count() - launches0)
        if barrier:
            barrier()
        ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        phase = np.zeros(4)
        nev = np.zeros(1, np.int64)
        _native.check(self.lib.lg_get_timing(self.npb.handle, _native.dptr(phase), _native.i64ptr(nev)))
        _native.check(self.lib.lg_set_timing(self.npb.handle, 0))
        return ms, launches, phase, max(int(nev[0]), 1)

    def roofline(self, phase, nevals, traffic_ok=True):
        case = self.case
        table = self.npb.plan_table(case.field)
        tot_bytes, bwd_bytes, flops = algorithmic_bytes(case, table)
        bwd_bytes *= self.share
        bwd_ms = phase[2] / nevals
        peak, peak_kind = _peaks()
        achieved = bwd_bytes / (bwd_ms / 1e3) / 1e9
        crit = critical_path_terms(table)
        engine = self.lib.lg_engine_name(self.npb.handle).decode()
        traffic, traffic_src = (committed_traffic(case.name, engine, case.field.n_steps) if traffic_ok
                                else (None, None))
        roof = {"bound": "hbm", "kernel": engine, "achieved": achieved, "peak": peak, "peak_source": peak_kind,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": bwd_bytes, "algorithmic_bytes_per_eval": tot_bytes,
                "flops_per_eval": flops, "critical_path_terms": crit,
                "ns_per_critical_term": 1e6 * (phase[1] + phase[2]) / nevals / max(crit, 1)}
        if engine.startswith("dense"):
            # dense engine: every Taylor term is one complex FP64 GEMM on the DMMA pipe (tensor bound)
            sweep_ms = (phase[1] + phase[2]) / nevals
            tflops = flops * self.share / (sweep_ms / 1e3) / 1e12
            pk = fp64_dgemm_peak()
            roof.update({"bound": "tensor", "achieved": tflops, "peak": pk,
                         "peak_source": "measured (cuBLAS DGEMM 8192^3, this run)", "unit": "TFLOP/s",
                         "frac": tflops / pk, "executed_tflops_3m": 0.75 * tflops,
                         "algorithmic_flops_per_launch": flops * self.share})
        return roof


def secondary_measurements(lib, flush):
    """Driver-run evidence for the other roofline targets of the north star, on the same box in the
    same run (bounded, ~30 s): the c3 sparse evaluation (HBM roofline) and the c5 dense engine's
    dominant kernel (the DMMA ZGEMM Taylor term at d = 4096 with the c5 column counts) against the
    FP64 DGEMM peak measured here."""
    import ctypes as C

    from paper_2304_06200_b200 import models

    out = {}
    try:
        case = models.build_case("c3")
        run = DeviceRun(case, lib, 0)
        ms, _, phase, nev = run.timed(3, 1, flush)
        out["c3"] = {"evals_per_s": 3 / (sum(ms) / 1e3), "ms_per_eval": sum(ms) / 3,
                     "roofline": run.roofline(phase, nev)}
        del run
    except Exception as exc:  # noqa: BLE001 - secondary evidence must not sink the headline line
        out["c3"] = {"error": repr(exc)}
    try:
        pk = fp64_dgemm_peak()
        z = {}
        for cols in (64, 128):
            msl = C.c_double()
            rc = lib.lg_bench_zgemm(4096, cols, 20, C.byref(msl))
            if rc:
                raise RuntimeError(lib.lg_last_error().decode())
            alg = 8.0 * 4096 * 4096 * cols / (msl.value / 1e3) / 1e12
            z[f"C{cols}"] = {"ms_per_term": msl.value, "algorithmic_tflops": alg, "executed_tflops_3m": 0.75 * alg,
                             "frac_algorithmic": alg / pk, "frac_executed": 0.75 * alg / pk}
        out["c5_dense_term"] = {"kernel": "lg_k_zgemm_taylor_n32 (split-k 8)", "d": 4096,
                                "fp64_peak_tflops": pk, "peak_source": "measured (cuBLAS DGEMM 8192^3, this run)",
                                **z}
    except Exception as exc:  # noqa: BLE001
        out["c5_dense_term"] = {"error": repr(exc)}
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2304_06200_b200 import _native, composite_grad, models

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    mode = _mode(args, world)
    lib = _native.load()
    case = models.build_case(args.config)
    N, Kc = case.field.n_steps, case.field.n_channels
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    run = DeviceRun(case, lib, local, shard=(mode == "shard"))
    barrier = dist.barrier if world > 1 else None
    clk = ClockSampler(local)  # sampled during the timed region only
    ms, launches, phase, nevals = run.timed(args.steps, args.warmup, flush, barrier=barrier, clocks=clk)
    total_ms = float(sum(ms))
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    jobs = world if mode == "replicas" else 1  # evaluations the whole job completes per step
    value = jobs * args.steps / (total_ms / 1e3)

    # end to end through the public API with host buffers (its own untimed warm-up: the first call
    # builds the API's cached device problem); bounded to a few evaluations for slow configs
    if mode == "shard":
        e2e_eval = lambda: run.ev.grad(case.field)  # noqa: E731 - the sharded public API object
    else:
        e2e_eval = lambda: composite_grad(case.problem, case.field, case.terms)  # noqa: E731
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    for _ in range(max(1, min(args.warmup, 1))):
        e2e_eval()
    e2e_ms = []
    for i in range(e2e_steps):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        if barrier:
            barrier()
        t0 = time.perf_counter()
        res = e2e_eval()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    te = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = jobs * e2e_steps / (float(te.item()) / 1e3)

    roofline = run.roofline(phase, nevals, traffic_ok=(mode != "shard"))
    clocks = clk.summary()
    wf = committed_smem_wavefronts(case.name, roofline["kernel"], N) if mode != "shard" else None
    if wf and clocks.get("sm_mhz"):
        # what actually bounds the sparse cluster kernels (state windows live in shared memory): the
        # shared-memory pipe, 1 wavefront per cycle per SM, over all SMs of the device at the clock
        # sampled during the timed region; wavefront count from the committed ncu capture
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        per_clk = wf / ((phase[2] / nevals / 1e3) * clocks["sm_mhz"] * 1e6 * sms)
        roofline["onchip"] = {"bound": "shared-memory pipe", "wavefronts_per_launch": wf, "sms": sms,
                              "achieved": per_clk, "peak": 1.0, "unit": "wavefronts/clk/SM", "frac": per_clk,
                              "source": "profiles/r02_c4_final_ncu.md"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if mode == "shard" else "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded BASELINE configs, SURVEY §8d)",
        "config": workload_config(case, world, mode),
        "state_steps_per_sec": value * case.n_states * N,
        "phase_ms_per_eval": {k: float(v / nevals) for k, v in
                              zip(["prep_plans", "forward", "backward", "finalize"], phase)},
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * N * Kc,
                "d2h_bytes_per_step": 8 * N * Kc + 8, "steps": e2e_steps},
        "gpu_launches": launches,
        "clocks": clocks,
        "cost": res.cost,
    }
    if mode == "shard":
        line["shard"] = {"trajectories_per_rank": int(run.ev.shard[1] - run.ev.shard[0]),
                         "allreduce_calls_per_eval": run.ev.calls,
                         "allreduce_bytes_per_eval": 8 * int(run.npb.raw_size(N))}
    if rank == 0 and world == 1 and not args.no_cpu:
        v, cores, sample = cpu_reference(case, budget_s=args.ref_budget)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}
    if rank == 0 and world == 1 and not args.no_secondary and args.config == "c4":
        del run
        line["secondary"] = secondary_measurements(lib, flush)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-budget", type=float, default=None,
                    help="CPU seconds per reference sample item (default: ~100 s over all steps)")
    ap.add_argument("--e2e-steps", type=int, default=5, help="timed end-to-end evaluations (<= --steps)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas (weak scaling) instead of the sharded K-state block")
    ap.add_argument("--shard", action="store_true", help="(default for N > 1; kept for old command lines)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launched directly: one process per GPU under torch.distributed.run (NCCL over NVLink)
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd, env=env))
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.ref_budget is None:
        args.ref_budget = 12.0 if args.impl == "ours" else max(2.0, 100.0 / (args.steps + args.warmup))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
