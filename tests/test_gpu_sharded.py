"""GPU: sharded evaluation through the C ABI (lg_set_raw_buffer / lg_eval_sharded / lg_cost_sharded).

Two shards of one problem are evaluated by two host threads on the one GPU of the test box; their
all-reduce hook is a host-side sum between the threads (stream-synchronised, so no kernel ever waits
on another shard's kernel).  This drives the library's exchange points exactly as NCCL ranks would:
the running-gate traces between the sweeps and the raw scalars before the device combine.  Every raw
slot has one writer, so the sharded result must be bit-identical to the unsharded evaluation; both
are checked against the CPU oracle too.  Covers the ws, cluster/CTA and dense engines.
"""

import threading

import numpy as np
import pytest
import torch

import _golden as G
from oracle import lg_oracle as O
from paper_2304_06200_b200 import ControlField, ControlProblem, CostKind, CostTerm
from paper_2304_06200_b200.costs import NativeProblem
from paper_2304_06200_b200.distributed import ShardedEvaluator, shard_bounds

pytestmark = pytest.mark.gpu

W = [0.7, 0.2, 0.4, 1.0, 0.5]


def _setup(tag, n_steps=12):
    z = G.sub(G.load("stress"), tag)
    hs, hc = G.mats(z)
    N, Kc = min(n_steps, z["amps"].shape[0]), z["amps"].shape[1]
    a = ControlField(N, Kc, float(z["dt"]), z["amps"][:N])
    prob = ControlProblem(hs, tuple(hc), initial_state=z["psi0"], basis=z["basis"])
    terms = [CostTerm(CostKind.STATE_INFIDELITY, W[0], target_state=z["targets"]),
             CostTerm(CostKind.STATE_PENALTY, W[1], penalty_op=G.penalty(z)),
             CostTerm(CostKind.STATE_RUNNING_INFIDELITY, W[2], target_state=z["targets"]),
             CostTerm(CostKind.GATE_INFIDELITY, W[3], target_images=z["images"]),
             CostTerm(CostKind.GATE_RUNNING_INFIDELITY, W[4], target_images=z["images"])]
    return z, a, prob, terms


def _oracle(z, a):
    hs, hc = G.mats(z, "oracle")
    om = G.penalty(z, "oracle")
    p = O.Problem(hs, tuple(hc), initial_states=z["psi0"], basis=z["basis"])
    terms = [O.Term(O.STATE_INFIDELITY, W[0], z["targets"]), O.Term(O.STATE_PENALTY, W[1], None, om),
             O.Term(O.STATE_RUNNING_INFIDELITY, W[2], z["targets"]), O.Term(O.GATE_INFIDELITY, W[3], z["images"]),
             O.Term(O.GATE_RUNNING_INFIDELITY, W[4], z["images"])]
    return O.composite_grad(p, a.amplitudes, a.dt, terms), O.composite_cost(p, a.amplitudes, a.dt, terms)


class _ThreadSum:
    """All-reduce between host threads: each contributes a copy, all read back the sum in rank order."""

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.parts = [None] * world

    def __call__(self, rank, view):
        torch.cuda.current_stream().synchronize()
        self.parts[rank] = view.clone()
        self.bar.wait()
        total = self.parts[0].clone()
        for r in range(1, self.world):
            total += self.parts[r]
        self.bar.wait()
        view.copy_(total)
        torch.cuda.current_stream().synchronize()


class _ThreadShard(ShardedEvaluator):
    def __init__(self, prob, terms, rank, world, reducer):
        n = prob.dim if prob.basis is None else np.asarray(prob.basis).shape[0]
        n = max(n, np.asarray(prob.initial_state).reshape(-1, prob.dim).shape[0])
        shard = shard_bounds(n, rank, world)
        native = NativeProblem(prob, terms, prob.initial_state, prob.basis, shard=shard)
        super().__init__(prob, terms, native=native)
        self.rank_, self.reducer = rank, reducer

    def _allreduce(self, view):
        self.reducer(self.rank_, view)


@pytest.mark.parametrize("tag", ["s_csr60", "s_block160", "s_dense24", "s_denseblk160"])
def test_sharded_matches_unsharded_bitwise(tag):
    z, a, prob, terms = _setup(tag)
    full = NativeProblem(prob, terms, prob.initial_state, prob.basis)
    ref = full.grad(a)
    ref_cost = full.cost(a)
    # world 1 through the real evaluator: lent buffer, stream, hook sequence
    ev = ShardedEvaluator(prob, terms)
    r1 = ev.grad(a)
    assert ev.calls == 3  # running gate traces between the sweeps + (ip|fin) + run
    assert r1.cost == ref.cost and np.array_equal(r1.grad, ref.grad)
    assert r1.live_vector_peak == ref.live_vector_peak > 0
    assert ev.cost(a) == ref_cost and ev.calls == 1
    # two shards on two host threads
    world = 2
    red = _ThreadSum(world)
    evs = [_ThreadShard(prob, terms, r, world, red) for r in range(world)]
    out = [None] * world

    def run(r):
        torch.cuda.set_device(0)
        out[r] = (evs[r].grad(a), evs[r].cost(a))

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for r in range(world):
        g, c = out[r]
        assert g.cost == ref.cost and np.array_equal(g.grad, ref.grad), r
        assert c == ref_cost, r
    (c_o, g_o), cc_o = _oracle(z, a)
    assert abs(ref.cost - c_o) <= 1e-12
    assert G.grad_rel(ref.grad, g_o) <= 1e-9
    assert abs(ref_cost - cc_o) <= 1e-12


def test_unhooked_sharded_running_gate_is_refused():
    z, a, prob, terms = _setup("s_csr60", 4)
    npb = NativeProblem(prob, terms, prob.initial_state, prob.basis, shard=(0, 1))
    with pytest.raises(NotImplementedError):
        npb.grad(a)


@pytest.mark.parametrize("tag", ["s_csr60", "s_block160", "s_denseblk160"])
def test_host_combine_of_raw_scalars_is_bitwise_the_device_combine(tag):
    """lg_raw_get + lg_finalize_host (the multi-rank combine) == lg_eval bit for bit:
    lg_k_finalize is built -fmad=false and both sides share lg_final.cuh (numpy's |z|)."""
    z, a, prob, terms = _setup(tag)
    terms = terms[:4]  # no running gate term: a plain lg_eval works on any problem
    npb = NativeProblem(prob, terms, prob.initial_state, prob.basis)
    res = npb.grad(a)
    cost, grad = npb.finalize(a.n_steps, npb.raw(a.n_steps))
    assert cost == res.cost
    assert np.array_equal(grad, res.grad)
