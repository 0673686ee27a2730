"""Sharded evaluation over a process group on CPU (gloo): paper_2304_06200_b200.distributed.

The device library needs a B200, so each rank drives a stand-in (`OracleShard`) that follows the
library's lg_eval_sharded protocol exactly: it writes its shard's raw per-trajectory scalars into
the buffer the evaluator lends it ([ip | fin | trp | run], the lg_raw_get layout), calls the
evaluator's all-reduce hook between the sweeps when a running gate cost is present (its costate
source needs the global trace, src/costs.py:462,477-478) and once more before the combine, and
combines with the library's host `lg_finalize_raw`.  The per-trajectory propagation is the CPU
oracle's.  What is under test is the real `ShardedEvaluator` (shard bounds, hook -> all_reduce on
views of the lent buffer, call sequence, empty shards) and the cross-rank result: it must equal the
single-process oracle `composite_grad` -- and the reference's golden values for the C3^g term --
and be bit-identical across world sizes (every raw slot has one writer, so x + 0 sums are exact).
"""

import ctypes as C
import os
import socket
import tempfile

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

import _golden as G
from oracle import lg_oracle as O

KINDS = [O.STATE_INFIDELITY, O.STATE_PENALTY, O.STATE_RUNNING_INFIDELITY, O.GATE_INFIDELITY,
         O.GATE_RUNNING_INFIDELITY]
CODE = {k: i for i, k in enumerate(KINDS)}  # include/leangrape_b200.h LG_* kind codes
WEIGHTS = [0.7, 0.2, 0.4, 1.0, 0.5]


def _case(n_steps=8):
    z = G.sub(G.load("stress"), "s_csr60")
    hs, hc = G.mats(z, "oracle")
    om = G.penalty(z, "oracle")
    return z, hs, hc, om, z["amps"][:n_steps], float(z["dt"])


class OracleShard:
    """Host stand-in for a sharded device problem (costs.NativeProblem's sharded interface)."""

    def __init__(self, kinds, shard):
        self.kinds = list(kinds)
        self.z, self.hs, self.hc, self.om, _, _ = _case(1)
        self.K = self.z["psi0"].shape[0]
        self.T = 2 * self.K  # state set 0..K-1, gate set K..2K-1
        self.lo, self.hi = shard
        self.buf = None

    def raw_size(self, N):
        S, T, Kc = len(self.kinds), self.T, len(self.hc)
        return 2 * (N * S * Kc * T + S * T + S * N * T) + S * T

    def set_raw_buffer(self, ptr, length):
        self.ptr = ptr
        self.buf = np.ctypeslib.as_array((C.c_double * length).from_address(ptr))

    def set_stream(self, stream):
        pass

    def _views(self, N):
        S, T, Kc = len(self.kinds), self.T, len(self.hc)
        n_ip, n_fin, n_trp = 2 * N * S * Kc * T, 2 * S * T, 2 * S * N * T
        b = self.buf
        ip = b[:n_ip].view(np.complex128).reshape(N, S, Kc, T)
        fin = b[n_ip:n_ip + n_fin].view(np.complex128).reshape(S, T)
        trp = b[n_ip + n_fin:n_ip + n_fin + n_trp].view(np.complex128).reshape(S, N, T)
        run = b[n_ip + n_fin + n_trp:].reshape(S, T)
        return (n_ip, n_fin, n_trp), ip, fin, trp, run

    def grad_sharded(self, a, hook):
        return self._eval(a, hook, grad=True)

    def cost_sharded(self, a, hook):
        return self._eval(a, hook, grad=False)[0]

    def _eval(self, a, hook, grad):
        amps, dt = np.asarray(a.amplitudes), float(a.dt)
        N, Kc = amps.shape
        z, K = self.z, self.K
        (n_ip, n_fin, n_trp), ip, fin, trp, run = self._views(N)
        self.buf[:] = 0.0
        steps = [O.Step(self.hs, tuple(self.hc), amps[n], dt, 1e-8) for n in range(N)]
        local = [t for t in range(self.T) if self.lo <= (t - K if t >= K else t) < self.hi]
        specs_of = {t: [s for s, k in enumerate(self.kinds) if (k in O.STATE_KINDS) == (t < K)] for t in local}
        psiN = {}
        for t in local:  # forward sweep (src/costs.py:286-297, 433-445)
            gate, h = t >= K, (t - K if t >= K else t)
            psi = np.array((z["basis"] if gate else z["psi0"])[h])
            for n in range(N):
                psi = steps[n].forward(psi)
                for s in specs_of[t]:
                    k = self.kinds[s]
                    if k == O.STATE_PENALTY:
                        run[s, t] += np.vdot(psi, O.matvec(self.om, psi)).real
                    elif k == O.STATE_RUNNING_INFIDELITY:
                        run[s, t] += abs(np.vdot(z["targets"][h], psi)) ** 2
                    elif k == O.GATE_RUNNING_INFIDELITY:
                        trp[s, n, t] = np.vdot(z["images"][h], psi)
            for s in specs_of[t]:
                if self.kinds[s] == O.STATE_INFIDELITY:
                    fin[s, t] = np.vdot(psi, z["targets"][h])
                elif self.kinds[s] == O.GATE_INFIDELITY:
                    fin[s, t] = np.vdot(z["images"][h], psi)
            psiN[t] = psi
        gate_run = O.GATE_RUNNING_INFIDELITY in self.kinds
        reduced = False
        if grad and gate_run:  # library: hook_traces
            assert hook(self.ptr + 8 * (n_ip + n_fin), n_trp) == 0
            reduced = True
        if grad:
            tr = trp[:, :, K:].sum(axis=2)  # global running traces (every rank holds them now)
            for t in local:  # backward sweep (src/costs.py:312-353, 452-482)
                h = t - K if t >= K else t
                psi = psiN[t]
                lam = {}
                for s in specs_of[t]:
                    k = self.kinds[s]
                    if k == O.STATE_INFIDELITY:
                        lam[s] = np.array(z["targets"][h])
                    elif k == O.STATE_PENALTY:
                        lam[s] = O.matvec(self.om, psi)
                    elif k == O.STATE_RUNNING_INFIDELITY:
                        lam[s] = z["targets"][h] * np.vdot(z["targets"][h], psi)
                    elif k == O.GATE_INFIDELITY:
                        lam[s] = np.array(z["images"][h])
                    else:
                        lam[s] = z["images"][h] * tr[s, N - 1]
                for n in range(N - 1, -1, -1):
                    st = steps[n]
                    psi = st.adjoint(psi)
                    for kc in range(Kc):
                        du = st.dU(kc, psi)
                        for s in specs_of[t]:
                            ip[n, s, kc, t] = np.vdot(lam[s], du)
                    if n > 0:
                        for s in specs_of[t]:
                            k = self.kinds[s]
                            moved = st.adjoint(lam[s])
                            if k == O.STATE_PENALTY:
                                moved += O.matvec(self.om, psi)
                            elif k == O.STATE_RUNNING_INFIDELITY:
                                moved += z["targets"][h] * np.vdot(z["targets"][h], psi)
                            elif k == O.GATE_RUNNING_INFIDELITY:
                                moved += z["images"][h] * tr[s, n - 1]
                            lam[s] = moved
        if reduced:  # library: hook_raw
            assert hook(self.ptr, n_ip + n_fin) == 0
            assert hook(self.ptr + 8 * (n_ip + n_fin + n_trp), self.buf.size - (n_ip + n_fin + n_trp)) == 0
        else:
            assert hook(self.ptr, self.buf.size) == 0
        return self._combine(N, Kc)

    def _combine(self, N, Kc):
        from paper_2304_06200_b200 import _native

        lib = _native.load()
        kinds = np.array([CODE[k] for k in self.kinds], np.int32)
        w = np.array([WEIGHTS[KINDS.index(k)] for k in self.kinds])
        t0 = np.array([0 if k in O.STATE_KINDS else self.K for k in self.kinds], np.int32)
        kk = np.full(len(self.kinds), self.K, np.int32)
        cost, g = C.c_double(), np.zeros((N, Kc))
        raw = np.ascontiguousarray(self.buf)
        _native.check(lib.lg_finalize_raw(len(self.kinds), _native.i32ptr(kinds), _native.dptr(w),
                                          _native.i32ptr(t0), _native.i32ptr(kk), N, Kc, self.T,
                                          _native.dptr(raw), C.byref(cost), _native.dptr(g)))
        return cost.value, g


def _problem_and_terms(z, kinds):
    """Product-side objects: only used by ShardedEvaluator for set sizes and validation."""
    from paper_2304_06200_b200 import ControlProblem, CostKind, CostTerm

    hs, hc = G.mats(z, "product")
    pk = {O.STATE_INFIDELITY: CostKind.STATE_INFIDELITY, O.STATE_PENALTY: CostKind.STATE_PENALTY,
          O.STATE_RUNNING_INFIDELITY: CostKind.STATE_RUNNING_INFIDELITY,
          O.GATE_INFIDELITY: CostKind.GATE_INFIDELITY, O.GATE_RUNNING_INFIDELITY: CostKind.GATE_RUNNING_INFIDELITY}
    terms = []
    for k in kinds:
        w = WEIGHTS[KINDS.index(k)]
        if k == O.STATE_PENALTY:
            terms.append(CostTerm(pk[k], w, penalty_op=G.penalty(z, "product")))
        elif k in O.STATE_KINDS:
            terms.append(CostTerm(pk[k], w, target_state=z["targets"]))
        else:
            terms.append(CostTerm(pk[k], w, target_images=z["images"]))
    prob = ControlProblem(hs, tuple(hc), initial_state=z["psi0"], basis=z["basis"])
    return prob, terms


def _worker(rank, world, port, out, kinds, n_steps):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2304_06200_b200 import ControlField
    from paper_2304_06200_b200.distributed import ShardedEvaluator

    z, _, _, _, amps, dt = _case(n_steps)
    prob, terms = _problem_and_terms(z, kinds)
    ev = ShardedEvaluator(prob, terms, native=OracleShard(kinds, _bounds(prob, terms, rank, world)),
                          buffer_device="cpu")
    field = ControlField(amps.shape[0], amps.shape[1], dt, amps)
    cost, grad = ev.grad(field)
    calls = ev.calls
    c_only = ev.cost(field)
    np.savez(os.path.join(out, f"rank{rank}.npz"), cost=cost, grad=grad, calls=calls, c_only=c_only,
             shard=np.array(ev.shard))
    dist.destroy_process_group()


def _bounds(prob, terms, rank, world):
    from paper_2304_06200_b200.distributed import _set_sizes, shard_bounds

    return shard_bounds(max(_set_sizes(prob, terms)), rank, world)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, kinds, n_steps=8):
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_worker, args=(world, _free_port(), out, kinds, n_steps), nprocs=world, join=True)
        return [dict(np.load(os.path.join(out, f"rank{r}.npz"))) for r in range(world)]


def _oracle(kinds):
    z, hs, hc, om, amps, dt = _case()
    p = O.Problem(hs, tuple(hc), initial_states=z["psi0"], basis=z["basis"])
    terms = []
    for k in kinds:
        w = WEIGHTS[KINDS.index(k)]
        if k == O.STATE_PENALTY:
            terms.append(O.Term(k, w, None, om))
        elif k in O.STATE_KINDS:
            terms.append(O.Term(k, w, z["targets"]))
        else:
            terms.append(O.Term(k, w, z["images"]))
    return O.composite_grad(p, amps, dt, terms), O.composite_cost(p, amps, dt, terms)


def test_sharded_all_kinds_two_and_four_ranks():
    (c_ref, g_ref), cc_ref = _oracle(KINDS)
    res = {w: _run(w, KINDS) for w in (1, 2, 4)}
    for w, rs in res.items():
        for r in rs:  # identical on every rank, and bit-identical across world sizes
            assert float(r["cost"]) == float(res[1][0]["cost"])
            assert np.array_equal(r["grad"], res[1][0]["grad"])
            assert float(r["c_only"]) == float(res[1][0]["c_only"])
            assert int(r["calls"]) == 3  # traces between sweeps + (ip|fin) + run
    assert [tuple(r["shard"]) for r in res[4]] == [(0, 1), (1, 2), (2, 3), (3, 3)]  # rank 3: empty shard
    r0 = res[2][0]
    assert abs(float(r0["cost"]) - c_ref) <= 1e-13
    assert np.linalg.norm(r0["grad"] - g_ref) <= 1e-12 * np.linalg.norm(g_ref)
    assert abs(float(r0["c_only"]) - cc_ref) <= 1e-13


def test_sharded_running_gate_matches_reference_golden():
    z = G.sub(G.load("stress"), "s_csr60")
    rs = _run(2, [O.GATE_RUNNING_INFIDELITY], n_steps=z["grad_g3"].shape[0])
    w = WEIGHTS[KINDS.index(O.GATE_RUNNING_INFIDELITY)]
    assert abs(float(rs[0]["cost"]) / w - float(z["cost_g3"])) <= 1e-12
    g = rs[0]["grad"] / w
    assert np.linalg.norm(g - z["grad_g3"]) <= 1e-9 * np.linalg.norm(z["grad_g3"])
    assert int(rs[0]["calls"]) == 3


def test_sharded_without_running_gate_uses_one_allreduce():
    kinds = [O.STATE_INFIDELITY, O.GATE_INFIDELITY]
    (c_ref, g_ref), _ = _oracle(kinds)
    rs = _run(2, kinds)
    assert all(int(r["calls"]) == 1 for r in rs)
    assert abs(float(rs[0]["cost"]) - c_ref) <= 1e-13
    assert np.linalg.norm(rs[0]["grad"] - g_ref) <= 1e-12 * np.linalg.norm(g_ref)
