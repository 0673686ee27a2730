"""The reference-side shim evaluates on the GPU and reuses the cached device problem.

The reference package does not travel to the GPU box, so stand-in objects carry the reference's
field names and enum ``.value`` strings (src/costs.py:49-168); a stand-in module plays
``leangrape.optimizer`` for ``enable()``.
"""

import types
from enum import Enum

import numpy as np
import pytest

from paper_2304_06200_b200 import composite_grad, costs, leangrape_compat as compat, models

pytestmark = pytest.mark.gpu


class _Kind(Enum):
    STATE_INFIDELITY = "state_infidelity"
    STATE_PENALTY = "state_penalty"
    GATE_INFIDELITY = "gate_infidelity"


class _Backend(Enum):
    SCALING_SQUARING = "scaling_squaring"


def _standins(case):
    p = case.problem
    prob = types.SimpleNamespace(h_static=p.h_static, h_controls=p.h_controls, backend=_Backend.SCALING_SQUARING,
                                 tau=p.tau, initial_state=np.array(p.initial_state), basis=tuple(np.array(p.basis)))
    terms = []
    for t in case.terms:
        terms.append(types.SimpleNamespace(kind=_Kind(t.kind.value), weight=t.weight, target_state=None,
                                           target_gate=None, penalty_op=t.penalty_op))
        if t.target_images is not None:
            # a full-d gate cannot be formed for the K=2 subspace; carry the images as target_gate's
            # replacement through the mirror's extension instead
            terms[-1] = t
    f = case.field
    a = types.SimpleNamespace(n_steps=f.n_steps, n_channels=f.n_channels, dt=f.dt, amplitudes=f.amplitudes.copy())
    return prob, terms, a


def test_shim_matches_mirror_and_hits_cache():
    case = models.build_case("c2", n_steps=60)
    ref = composite_grad(case.problem, case.field, case.terms)
    prob, terms, a = _standins(case)
    opt = types.ModuleType("standin.optimizer")
    opt.composite_grad = opt.composite_cost = None
    compat.enable(opt)
    try:
        r1 = opt.composite_grad(prob, a, terms)
        n_cached = len(costs._CACHE)
        r2 = opt.composite_grad(prob, a, terms)
        c2 = opt.composite_cost(prob, a, terms)
        assert len(costs._CACHE) == n_cached  # no new device problem on repeated calls
    finally:
        compat.disable(opt)
    assert r1.cost == ref.cost and np.array_equal(r1.grad, ref.grad)
    assert r2.cost == r1.cost and np.array_equal(r2.grad, r1.grad)
    assert abs(c2 - ref.cost) <= 1e-12
