"""Pin the CPU oracle (oracle/lg_oracle.py) to the reference's own outputs.

Golden vectors come from running the reference package itself
(tests/golden/make_golden.py).  Planner results and plan tables must match
bit-for-bit; costs/gradients to the parity tolerances (they are in fact
identical to ~1e-16 because the oracle performs the same numpy operations).
"""

import math

import numpy as np
import pytest

from oracle import lg_oracle as O
import _golden as G


def test_planner_matches_reference_exactly():
    z = G.load("planner")
    for norm, sp, tau, m, s, b, st in zip(z["norm"], z["sp"], z["tau"], z["m"], z["s"], z["bound"], z["status"]):
        if st:
            with pytest.raises(O.PlanningError):
                O.make_plan(float(norm), int(sp), float(tau))
        else:
            pm, ps, pb = O.make_plan(float(norm), int(sp), float(tau))
            assert (pm, ps) == (m, s), (norm, sp, tau)
            assert pb == b


def test_frozen_bound_constants():
    z = G.load("planner")
    assert O.remainder_rm(1.0, 5) == z["remainder_1_5"]
    assert O.gamma_n(3) == z["gamma_3"]
    assert O.rounding_bound(0.5, 10, 2, 4) == z["rounding_05_10_2_4"]
    assert O.truncation_bound(0.5, 15, 4) == z["truncation_05_15_4"]
    # the reference's 60-digit mpmath literals (tests/test_expm_bounds.py:62,105,110,133)
    assert O.remainder_rm(1.0, 5) == pytest.approx(0.001615161792378568693620805, rel=1e-14)
    assert O.gamma_n(3) == pytest.approx(9.420554752102661e-16, rel=1e-14)
    assert O.rounding_bound(0.5, 10, 2, 4) == pytest.approx(1.553186900115791e-14, rel=1e-12)
    assert O.truncation_bound(0.5, 15, 4) == pytest.approx(3.005407950636189e-18, rel=1e-12)


def test_planner_refusal_and_validation():
    with pytest.raises(O.PlanningError, match="norm1=1000"):
        O.make_plan(1000.0, 5, 1e-12, s_max=100)
    with pytest.raises(ValueError):
        O.make_plan(1.0, 1, 0.0)
    with pytest.raises(ValueError):
        O.make_plan(float("nan"), 1, 1e-8)


def _oracle_problem(z, kind_states=None):
    hs, hc = G.mats(z, "oracle")
    return hs, hc


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_plan_tables_bit_exact(name):
    z = G.load(name)
    hs, hc = G.mats(z, "oracle")
    amps = z["amps"]
    t = O.plan_table(hs, hc, amps, float(z["dt"]), 1e-8)
    for k in G.plan_keys():
        assert np.array_equal(t[k], z["plan_" + k]), k


@pytest.mark.parametrize("tag", ["s_csr60", "s_block160", "s_dense24", "s_denseblk160"])
def test_stress_plan_tables_bit_exact(tag):
    z = G.sub(G.load("stress"), tag)
    hs, hc = G.mats(z, "oracle")
    t = O.plan_table(hs, hc, z["amps"], float(z["dt"]), 1e-8)
    for k in G.plan_keys():
        assert np.array_equal(t[k], z["plan_" + k]), k


def test_c1_cost_grad_full_size():
    z = G.load("c1")
    hs, hc = G.mats(z, "oracle")
    p = O.Problem(hs, tuple(hc), initial_states=z["psi0"])
    cost, grad = O.composite_grad(p, z["amps"], float(z["dt"]), [O.Term(O.STATE_INFIDELITY, 1.0, z["targets"])])
    assert abs(cost - float(z["cost"])) <= 1e-14
    assert G.grad_rel(grad, z["grad"]) <= 1e-13
    c = O.composite_cost(p, z["amps"], float(z["dt"]), [O.Term(O.STATE_INFIDELITY, 1.0, z["targets"])])
    assert abs(c - float(z["cost_only"])) <= 1e-14


def test_full_basis_gate_matches_reference():
    z = G.load("fullbasis")
    hs, hc = G.mats(z, "oracle")
    u = z["target_gate"]
    d = u.shape[0]
    images = (u @ np.eye(d)).T.copy()
    p = O.Problem(hs, tuple(hc))
    for kind, ck, gk in [(O.GATE_INFIDELITY, "cost_g1", "grad_g1"), (O.GATE_RUNNING_INFIDELITY, "cost_g3", "grad_g3")]:
        cost, grad = O.composite_grad(p, z["amps"], float(z["dt"]), [O.Term(kind, 1.0, images)])
        assert abs(cost - float(z[ck])) <= 1e-15
        assert G.grad_rel(grad, z[gk]) <= 1e-13


@pytest.mark.parametrize("tag", ["s_csr60", "s_block160", "s_dense24", "s_denseblk160"])
def test_stress_cost_grad(tag):
    z = G.sub(G.load("stress"), tag)
    hs, hc = G.mats(z, "oracle")
    om = G.penalty(z, "oracle")
    p = O.Problem(hs, tuple(hc), initial_states=z["psi0"], basis=z["basis"])
    dt = float(z["dt"])
    terms = [O.Term(O.STATE_INFIDELITY, 0.7, z["targets"]), O.Term(O.STATE_PENALTY, 0.2, None, om),
             O.Term(O.STATE_RUNNING_INFIDELITY, 0.4, z["targets"])]
    cost, grad = O.composite_grad(p, z["amps"], dt, terms)
    assert abs(cost - float(z["cost_state"])) <= 1e-13
    assert G.grad_rel(grad, z["grad_state"]) <= 1e-12
    assert abs(O.composite_cost(p, z["amps"], dt, terms) - float(z["cost_state_only"])) <= 1e-13
    for kind, ck, gk in [(O.GATE_INFIDELITY, "cost_g1", "grad_g1"), (O.GATE_RUNNING_INFIDELITY, "cost_g3", "grad_g3")]:
        cost, grad = O.composite_grad(p, z["amps"], dt, [O.Term(kind, 1.0, z["images"])])
        assert abs(cost - float(z[ck])) <= 1e-13
        assert G.grad_rel(grad, z[gk]) <= 1e-12


@pytest.mark.parametrize("golden,tag", [("diag", "d_dense40"), ("diag", "d_csr24"), ("diag", "d_csr60"),
                                        ("diag_big", "d_csr180"), ("diag_big", "d_dense256")])
def test_diagonalization_backend_cost_grad(golden, tag):
    """The oracle's DIAGONALIZATION restatement against the reference's own backend."""
    z = G.sub(G.load(golden), tag)
    hs, hc = G.mats(z, "oracle")
    om = G.penalty(z, "oracle")
    p = O.Problem(hs, tuple(hc), initial_states=z["psi0"], basis=z["basis"], backend="diagonalization")
    dt = float(z["dt"])
    terms = [O.Term(O.STATE_INFIDELITY, 0.7, z["targets"]), O.Term(O.STATE_PENALTY, 0.2, None, om),
             O.Term(O.STATE_RUNNING_INFIDELITY, 0.4, z["targets"])]
    cost, grad = O.composite_grad(p, z["amps"], dt, terms)
    assert abs(cost - float(z["cost_state"])) <= 1e-13
    assert G.grad_rel(grad, z["grad_state"]) <= 1e-12
    assert abs(O.composite_cost(p, z["amps"], dt, terms) - float(z["cost_state_only"])) <= 1e-13
    for kind, ck, gk in [(O.GATE_INFIDELITY, "cost_g1", "grad_g1"), (O.GATE_RUNNING_INFIDELITY, "cost_g3", "grad_g3")]:
        cost, grad = O.composite_grad(p, z["amps"], dt, [O.Term(kind, 1.0, z["images"])])
        assert abs(cost - float(z[ck])) <= 1e-13
        assert G.grad_rel(grad, z[gk]) <= 1e-12


@pytest.mark.slow
def test_c2_cost_grad_full_size():
    z = G.load("c2")
    hs, hc = G.mats(z, "oracle")
    om = G.penalty(z, "oracle")
    p = O.Problem(hs, tuple(hc), initial_states=z["basis"], basis=z["basis"])
    terms = [O.Term(O.GATE_INFIDELITY, 1.0, z["images"]), O.Term(O.STATE_PENALTY, 0.1, None, om)]
    cost, grad = O.composite_grad(p, z["amps"], float(z["dt"]), terms)
    assert abs(cost - float(z["cost"])) <= 1e-13
    assert G.grad_rel(grad, z["grad"]) <= 1e-12


def test_numpy_abs_rule_restated():
    """|z| = larger * sqrt(fma(r, r, 1)), r = smaller/larger (numpy SIMD cabs)."""
    from fractions import Fraction

    z = G.load("numpy_rules")
    zz, ref = z["z"][:3000], z["absz"][:3000]
    for v, a in zip(zz, ref):
        re, im = abs(v.real), abs(v.imag)
        big, small = max(re, im), min(re, im)
        if big == 0:
            assert a == 0
            continue
        r = small / big
        f = float(Fraction(r) * Fraction(r) + 1)
        assert big * math.sqrt(f) == a or math.sqrt(f) * big == a
