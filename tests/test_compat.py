"""The reference-side shim (paper_2304_06200_b200.leangrape_compat) on the reference's own objects.

CPU only: conversion of real ``leangrape`` objects (imported from /root/reference when present --
the build container; skipped elsewhere), memoisation per reference object, and the rebinding of
``leangrape.optimizer.composite_grad/composite_cost`` (src/optimizer.py:18).  The GPU evaluation
through the shim is tests/test_gpu_compat.py.
"""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


@pytest.fixture(scope="module")
def lg():
    sys.path.insert(0, REF)
    try:
        import leangrape.costs as costs
        import leangrape.models as models
        import leangrape.optimizer as optimizer
        import leangrape.sparse as sparse
    finally:
        sys.path.remove(REF)
    return costs, models, optimizer, sparse


def _ref_case(lg):
    costs, models, _, sparse = lg
    p = models.TransmonCavityParams(delta=0.1, anharmonicity=-0.225, g=0.05, d_transmon=3, d_cavity=4)
    h_s, ctrls = models.build_transmon_cavity(p)
    d = h_s.n_rows
    psi0 = models.fock_state(d, 0)
    phi = models.fock_state(d, 1)
    prob = costs.ControlProblem(h_s, tuple(ctrls), initial_state=psi0)
    terms = [costs.CostTerm(costs.CostKind.STATE_INFIDELITY, 1.0, target_state=phi),
             costs.CostTerm(costs.CostKind.STATE_PENALTY, 0.1, penalty_op=sparse.identity_csr(d))]
    a = costs.ControlField(5, len(ctrls), 0.5, np.full((5, len(ctrls)), 0.01))
    return prob, terms, a


def test_conversion_fields_and_memo(lg):
    from paper_2304_06200_b200 import costs as B
    from paper_2304_06200_b200 import leangrape_compat as compat

    prob, terms, a = _ref_case(lg)
    cp = compat.convert_problem(prob)
    assert isinstance(cp, B.ControlProblem)
    assert cp.backend is B.Backend.SCALING_SQUARING and cp.tau == prob.tau
    assert np.array_equal(cp.h_static.values, prob.h_static.values)
    assert np.array_equal(cp.initial_state, prob.initial_state)
    assert not cp.initial_state.flags.writeable  # private read-only copy
    assert compat.convert_problem(prob) is cp  # memoised per reference object
    ct = compat.convert_terms(terms)
    assert [t.kind.value for t in ct] == [t.kind.value for t in terms]
    assert compat.convert_terms(terms) is ct
    assert all(x is y for x, y in zip(compat.convert_terms(list(terms)), ct))
    cf = compat.convert_field(a)
    assert np.array_equal(cf.amplitudes, a.amplitudes) and cf.dt == a.dt


def test_enable_rebinds_reference_optimizer(lg):
    from paper_2304_06200_b200 import leangrape_compat as compat

    _, _, optimizer, _ = lg
    orig = (optimizer.composite_grad, optimizer.composite_cost)
    compat.enable(optimizer)
    try:
        assert optimizer.composite_grad is compat.composite_grad
        assert optimizer.composite_cost is compat.composite_cost
    finally:
        compat.disable(optimizer)
    assert (optimizer.composite_grad, optimizer.composite_cost) == orig
