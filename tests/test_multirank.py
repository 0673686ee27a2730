"""Multi-rank combine on CPU (gloo, world_size 2).

Each rank owns half of the trajectories, produces the raw per-trajectory
scalars of its shard (here with the CPU oracle standing in for the GPU sweeps,
which need a B200), the raw arrays are sum-allreduced, and every rank runs the
library's host combine `lg_finalize_raw`.  The result must equal the oracle's
single-process composite_grad -- this exercises the shard layout, the raw-slot
format and the cross-rank reduction the GPU path uses.
"""

import ctypes as C
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import _golden as G
from oracle import lg_oracle as O

KINDS = [O.STATE_INFIDELITY, O.STATE_PENALTY, O.STATE_RUNNING_INFIDELITY, O.GATE_INFIDELITY]
CODE = {O.STATE_INFIDELITY: 0, O.STATE_PENALTY: 1, O.STATE_RUNNING_INFIDELITY: 2, O.GATE_INFIDELITY: 3}
WEIGHTS = [0.7, 0.2, 0.4, 1.0]


def _case(n_steps=6):
    z = G.sub(G.load("stress"), "s_csr60")
    hs, hc = G.mats(z, "oracle")
    om = G.penalty(z, "oracle")
    p = O.Problem(hs, tuple(hc), initial_states=z["psi0"], basis=z["basis"])
    return p, z["amps"][:n_steps], float(z["dt"]), z, om


def _raw_shard(p, amps, dt, z, om, lo, hi):
    """Raw scalars (ip, fin, trp, run) of global trajectories [lo, hi); zeros elsewhere.
    Trajectories 0..K-1: state set (psi0); K..2K-1: gate set (basis)."""
    N, Kc = amps.shape
    K = z["psi0"].shape[0]
    T, S = 2 * K, len(KINDS)
    ip = np.zeros((N, S, Kc, T), np.complex128)
    fin = np.zeros((S, T), np.complex128)
    trp = np.zeros((S, N, T), np.complex128)
    run = np.zeros((S, T))
    for t in range(lo, hi):
        gate = t >= K
        h = t - K if gate else t
        psi = np.array((z["basis"] if gate else z["psi0"])[h])
        specs = [3] if gate else [0, 1, 2]
        steps = [O.Step(p.h_static, p.h_controls, amps[n], dt, p.tau) for n in range(N)]
        for n in range(N):
            psi = steps[n].forward(psi)
            for s in specs:
                if KINDS[s] == O.STATE_PENALTY:
                    run[s, t] += np.vdot(psi, O.matvec(om, psi)).real
                elif KINDS[s] == O.STATE_RUNNING_INFIDELITY:
                    run[s, t] += abs(np.vdot(z["targets"][h], psi)) ** 2
        lam = {}
        for s in specs:
            k = KINDS[s]
            if k == O.STATE_INFIDELITY:
                fin[s, t] = np.vdot(psi, z["targets"][h])
                lam[s] = np.array(z["targets"][h])
            elif k == O.STATE_PENALTY:
                lam[s] = O.matvec(om, psi)
            elif k == O.STATE_RUNNING_INFIDELITY:
                lam[s] = z["targets"][h] * np.vdot(z["targets"][h], psi)
            else:
                fin[s, t] = np.vdot(z["images"][h], psi)
                lam[s] = np.array(z["images"][h])
        for n in range(N - 1, -1, -1):
            st = steps[n]
            psi = st.adjoint(psi)
            for k in range(Kc):
                du = st.dU(k, psi)
                for s in specs:
                    ip[n, s, k, t] = np.vdot(lam[s], du)
            if n > 0:
                for s in specs:
                    moved = st.adjoint(lam[s])
                    if KINDS[s] == O.STATE_PENALTY:
                        moved += O.matvec(om, psi)
                    elif KINDS[s] == O.STATE_RUNNING_INFIDELITY:
                        moved += z["targets"][h] * np.vdot(z["targets"][h], psi)
                    lam[s] = moved
    return np.concatenate([ip.ravel().view(np.float64), fin.ravel().view(np.float64),
                           trp.ravel().view(np.float64), run.ravel()])


def _finalize(raw, N, Kc, T, K):
    from paper_2304_06200_b200 import _native

    lib = _native.load()
    kinds = np.array([CODE[k] for k in KINDS], np.int32)
    w = np.array(WEIGHTS)
    t0 = np.array([0, 0, 0, K], np.int32)
    kk = np.array([K, K, K, K], np.int32)
    cost, grad = C.c_double(), np.zeros((N, Kc))
    raw = np.ascontiguousarray(raw)
    _native.check(lib.lg_finalize_raw(len(KINDS), _native.i32ptr(kinds), _native.dptr(w), _native.i32ptr(t0),
                                      _native.i32ptr(kk), N, Kc, T, _native.dptr(raw), C.byref(cost),
                                      _native.dptr(grad)))
    return cost.value, grad


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p, amps, dt, z, om = _case()
    K = z["psi0"].shape[0]
    T = 2 * K
    per = (T + world - 1) // world
    raw = _raw_shard(p, amps, dt, z, om, rank * per, min(T, (rank + 1) * per))
    t = torch.from_numpy(raw)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    cost, grad = _finalize(t.numpy(), amps.shape[0], amps.shape[1], T, K)
    np.savez(os.path.join(out, f"rank{rank}.npz"), cost=cost, grad=grad)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_shard_combine_matches_single_process():
    p, amps, dt, z, om = _case()
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
        r0 = np.load(os.path.join(out, "rank0.npz"))
        r1 = np.load(os.path.join(out, "rank1.npz"))
    assert float(r0["cost"]) == float(r1["cost"]) and np.array_equal(r0["grad"], r1["grad"])
    terms = [O.Term(O.STATE_INFIDELITY, 0.7, z["targets"]), O.Term(O.STATE_PENALTY, 0.2, None, om),
             O.Term(O.STATE_RUNNING_INFIDELITY, 0.4, z["targets"]), O.Term(O.GATE_INFIDELITY, 1.0, z["images"])]
    c_ref, g_ref = O.composite_grad(p, amps, dt, terms)
    assert abs(float(r0["cost"]) - c_ref) <= 1e-13
    assert np.linalg.norm(r0["grad"] - g_ref) <= 1e-12 * np.linalg.norm(g_ref)


def test_single_rank_raw_equals_sum_of_shards():
    p, amps, dt, z, om = _case(n_steps=3)
    K = z["psi0"].shape[0]
    full = _raw_shard(p, amps, dt, z, om, 0, 2 * K)
    parts = _raw_shard(p, amps, dt, z, om, 0, 2) + _raw_shard(p, amps, dt, z, om, 2, 2 * K)
    assert np.array_equal(full, parts)  # x + 0 = x: sharding is exact
