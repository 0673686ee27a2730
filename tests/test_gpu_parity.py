"""GPU parity: the sm_100a path vs the reference's golden vectors and the CPU oracle.

Bars (BASELINE.json north_star): plans bit-identical; cost within 1e-12 absolute;
gradient within 1e-9 relative (norm-wise, as tests/test_costs.py:39-42 measures).
Everything here calls through the C ABI (include/leangrape_b200.h).
"""

import os

import numpy as np
import pytest

import _golden as G
from paper_2304_06200_b200 import (
    ControlField,
    ControlProblem,
    CostKind,
    CostTerm,
    c1_gate_grad,
    c3_gate_grad,
    composite_cost,
    composite_grad,
    forward_propagate,
    models,
)
from paper_2304_06200_b200.costs import NativeProblem
from paper_2304_06200_b200.expm import make_plans_device

pytestmark = pytest.mark.gpu

COST_TOL = 1e-12
GRAD_TOL = 1e-9


def _check(res, cost, grad, ctol=COST_TOL, gtol=GRAD_TOL):
    assert abs(res.cost - float(cost)) <= ctol, (res.cost, float(cost))
    assert G.grad_rel(res.grad, grad) <= gtol, G.grad_rel(res.grad, grad)


def _plans_equal(t, z, prefix="plan_"):
    for k in G.plan_keys():
        ref = z[prefix + k]
        got = t[k]
        assert np.array_equal(got, ref), (k, np.argwhere(got != ref)[:5])


# ----------------------------------------------------------------------------- planner


def test_device_planner_matches_reference():
    z = G.load("planner")
    for tau in np.unique(z["tau"]):
        sel = z["tau"] == tau
        m, s, st, unc = make_plans_device(z["norm"][sel], z["sp"][sel], float(tau))
        assert np.array_equal(st != 0, z["status"][sel] != 0)
        ok = st == 0
        assert np.array_equal(m[ok], z["m"][sel][ok])
        assert np.array_equal(s[ok], z["s"][sel][ok])


# ----------------------------------------------------------------------------- configs


def _c2_problem(z):
    hs, hc = G.mats(z)
    om = G.penalty(z)
    prob = ControlProblem(hs, tuple(hc), initial_state=z["basis"], basis=z["basis"])
    terms = [CostTerm(CostKind.GATE_INFIDELITY, 1.0, target_images=z["images"]),
             CostTerm(CostKind.STATE_PENALTY, 0.1, penalty_op=om)]
    return prob, terms


def test_c1_full_size():
    z = G.load("c1")
    hs, hc = G.mats(z)
    prob = ControlProblem(hs, tuple(hc), initial_state=z["psi0"])
    a = ControlField(1000, 1, float(z["dt"]), z["amps"])
    terms = [CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=z["targets"])]
    _check(composite_grad(prob, a, terms), z["cost"], z["grad"])
    assert abs(composite_cost(prob, a, terms) - float(z["cost_only"])) <= COST_TOL
    _plans_equal(NativeProblem(prob, terms, initial_states=z["psi0"]).plan_table(a), z)


def test_c2_full_size():
    z = G.load("c2")
    prob, terms = _c2_problem(z)
    a = ControlField(2000, 2, float(z["dt"]), z["amps"])
    _check(composite_grad(prob, a, terms), z["cost"], z["grad"])
    assert abs(composite_grad(prob, a, terms[:1]).cost - float(z["cost_gate"])) <= COST_TOL
    assert abs(composite_cost(prob, a, terms[1:]) - float(z["cost_only_pen"])) <= COST_TOL
    _plans_equal(NativeProblem(prob, terms, initial_states=z["basis"], basis=z["basis"]).plan_table(a), z)


def test_c3_prefix():
    z = G.load("c3")
    hs, hc = G.mats(z)
    N = z["amps"].shape[0]
    prob = ControlProblem(hs, tuple(hc), initial_state=z["psi0"])
    a = ControlField(N, 2, float(z["dt"]), z["amps"])
    terms = [CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=z["targets"])]
    _check(composite_grad(prob, a, terms), z["cost"], z["grad"])
    _plans_equal(NativeProblem(prob, terms, initial_states=z["psi0"]).plan_table(a), z)


def test_c4_prefix():
    z = G.load("c4")
    case = models.build_case("c4", n_steps=z["amps"].shape[0])
    _check(composite_grad(case.problem, case.field, case.terms), z["cost"], z["grad"])
    a32 = ControlField(32, 4, float(z["dt"]), z["amps_full"][:32])
    t = NativeProblem(case.problem, case.terms, basis=case.problem.basis).plan_table(a32)
    _plans_equal(t, z)


# ----------------------------------------------------------------------------- stress variants


@pytest.mark.parametrize("tag", ["s_csr60", "s_block160", "s_dense24", "s_denseblk160"])
@pytest.mark.parametrize("engine", ["auto", "multi"])
def test_stress_all_cost_kinds(tag, engine, monkeypatch):
    if engine == "multi":
        monkeypatch.setenv("LG_ENGINE", "multi")
    z = G.sub(G.load("stress"), tag)
    hs, hc = G.mats(z)
    om = G.penalty(z)
    N, Kc = z["amps"].shape
    a = ControlField(N, Kc, float(z["dt"]), z["amps"])
    prob = ControlProblem(hs, tuple(hc), initial_state=z["psi0"], basis=z["basis"])
    terms = [CostTerm(CostKind.STATE_INFIDELITY, 0.7, target_state=z["targets"]),
             CostTerm(CostKind.STATE_PENALTY, 0.2, penalty_op=om),
             CostTerm(CostKind.STATE_RUNNING_INFIDELITY, 0.4, target_state=z["targets"])]
    _check(NativeProblem(prob, terms, initial_states=z["psi0"]).grad(a), z["cost_state"], z["grad_state"])
    assert abs(NativeProblem(prob, terms, initial_states=z["psi0"]).cost(a) - float(z["cost_state_only"])) <= COST_TOL
    for kind, ck, gk in [(CostKind.GATE_INFIDELITY, "cost_g1", "grad_g1"),
                         (CostKind.GATE_RUNNING_INFIDELITY, "cost_g3", "grad_g3")]:
        t = [CostTerm(kind, 1.0, target_images=z["images"])]
        _check(NativeProblem(prob, t, basis=z["basis"]).grad(a), z[ck], z[gk])
    _plans_equal(NativeProblem(prob, terms, initial_states=z["psi0"]).plan_table(a), z)


def test_full_basis_gates_match_reference_functions():
    z = G.load("fullbasis")
    hs, hc = G.mats(z)
    N, Kc = z["amps"].shape
    a = ControlField(N, Kc, float(z["dt"]), z["amps"])
    prob = ControlProblem(hs, tuple(hc))
    _check(c1_gate_grad(prob, a, z["target_gate"]), z["cost_g1"], z["grad_g1"])
    _check(c3_gate_grad(prob, a, z["target_gate"]), z["cost_g3"], z["grad_g3"])


# ----------------------------------------------------------------------------- oracle + properties


def test_against_live_oracle_random_problem():
    from oracle import lg_oracle as O

    rng = np.random.default_rng(77)
    h_s, hx, hy = models.transmon_cavity_ops(3, 6)
    d = 18
    N = 9
    amps = rng.uniform(-0.8, 0.8, (N, 2))
    psi0 = models.rand_states(rng, 2, d)
    phi = models.rand_states(rng, 2, d)
    prob = ControlProblem(h_s, (hx, hy), initial_state=psi0)
    terms = [CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=phi),
             CostTerm(CostKind.STATE_RUNNING_INFIDELITY, 0.5, target_state=phi)]
    a = ControlField(N, 2, 0.4, amps)
    res = composite_grad(prob, a, terms)
    oc = lambda m: O.Csr(m.n_rows, m.row_offsets, m.col_indices, m.values)
    op = O.Problem(oc(h_s), (oc(hx), oc(hy)), initial_states=psi0)
    c, g = O.composite_grad(op, amps, 0.4, [O.Term(O.STATE_INFIDELITY, 1.0, phi),
                                            O.Term(O.STATE_RUNNING_INFIDELITY, 0.5, phi)])
    _check(res, c, g)


def test_determinism_and_forward_unitarity():
    case = models.build_case("c2", n_steps=300)
    r1 = composite_grad(case.problem, case.field, case.terms)
    r2 = composite_grad(case.problem, case.field, case.terms)
    assert r1.cost == r2.cost and np.array_equal(r1.grad, r2.grad)
    psi = forward_propagate(case.problem, case.field, case.problem.initial_state)
    assert np.allclose(np.linalg.norm(psi, axis=1), 1.0, atol=1e-10)


def test_live_vector_peak_independent_of_steps():
    p1 = composite_grad(*_args(models.build_case("c2", n_steps=10)))
    p2 = composite_grad(*_args(models.build_case("c2", n_steps=200)))
    assert p1.live_vector_peak == p2.live_vector_peak > 0


def _args(case):
    return case.problem, case.field, case.terms


def test_c3_full_size_finite_difference():
    """Size-independent property at BASELINE's full c3 size: dC/da against central FD."""
    case = models.build_case("c3")
    res = composite_grad(*_args(case))
    rng = np.random.default_rng(3)
    eps = 1e-6
    for _ in range(3):
        n, k = int(rng.integers(0, case.field.n_steps)), int(rng.integers(0, 2))
        ap = case.field.amplitudes.copy()
        am = ap.copy()
        ap[n, k] += eps
        am[n, k] -= eps
        cp = composite_cost(case.problem, case.field.replace_amplitudes(ap), case.terms)
        cm = composite_cost(case.problem, case.field.replace_amplitudes(am), case.terms)
        fd = (cp - cm) / (2 * eps)
        assert abs(fd - res.grad[n, k]) <= 1e-6 * max(1e-3, np.abs(res.grad).max())


def test_optimizer_decreases_cost():
    from paper_2304_06200_b200 import OptimizerConfig, grape_optimize

    case = models.build_case("c2", n_steps=100)
    tr = grape_optimize(case.problem, case.terms, case.field, OptimizerConfig(max_iters=4, eta0=0.05))
    costs = [r.cost for r in tr.records]
    assert len(costs) >= 2 and all(b <= a for a, b in zip(costs, costs[1:]))


def test_c5_prefix_dense_dmma():
    """config 5 (dense d=4096, DMMA GEMM path): N'=4 steps, K'=4 of the 64 transfers."""
    z = G.load("c5")
    case = models.build_case("c5", n_steps=int(z["amps"].shape[0]), n_states=int(z["k_sub"]))
    assert np.sum(np.abs(case.problem.h_static.array)) == float(z["hs_checksum"])
    _check(composite_grad(case.problem, case.field, case.terms), z["cost"], z["grad"])
    a8 = ControlField(8, 1, float(z["dt"]), models.controls(105, 1000, 1, 1.0)[:8])
    t = NativeProblem(case.problem, case.terms, initial_states=case.problem.initial_state).plan_table(a8)
    _plans_equal(t, z)


# ----------------------------------------------------------------------------- cluster-engine variants


@pytest.mark.parametrize("size,q,nosmall,fused", [(16, 1, 0, 0), (16, 3, 0, 0), (16, 6, 0, 0), (8, 3, 0, 0),
                                                  (16, 3, 1, 0), (8, 2, 1, 0), (16, 1, 2, 0), (8, 1, 2, 0),
                                                  (16, 3, 0, 1), (8, 3, 0, 1), (16, 3, 1, 1), (16, 1, 2, 1)])
def test_cluster_engine_variants(size, q, nosmall, fused, monkeypatch):
    """Every cluster-engine layout (cluster size, ghost-zone block length Q, SMALL, generic or
    LARGE (two rows per thread, nosmall == 2) kernels), with the two-phase backward (adjoint sweep
    + derivative-product items, the default) and the fused one (split backward for the SMALL
    kernels) against the golden c3 prefix and the plan-sensitive block-aux stress variant."""
    monkeypatch.setenv("LG_CL_SIZE", str(size))
    monkeypatch.setenv("LG_CL_Q", str(q))
    if fused:
        monkeypatch.setenv("LG_CL_FUSED", "1")
    if nosmall == 1:
        monkeypatch.setenv("LG_CL_NOSMALL", "1")
    if nosmall == 2:
        monkeypatch.setenv("LG_CL_LARGE", "1")
    z = G.load("c3")
    hs, hc = G.mats(z)
    prob = ControlProblem(hs, tuple(hc), initial_state=z["psi0"])
    a = ControlField(z["amps"].shape[0], 2, float(z["dt"]), z["amps"])
    terms = [CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=z["targets"])]
    npb = NativeProblem(prob, terms, initial_states=z["psi0"])
    for _ in range(4):  # repeated gradient and forward-only calls on one problem (intermittent-race guard)
        _check(npb.grad(a), z["cost"], z["grad"])
        assert abs(npb.cost(a) - float(z["cost"])) <= COST_TOL
    assert npb.engine.startswith("cluster-large" if nosmall == 2 else "cluster"), npb.engine
    assert ("adjoint" in npb.engine) == (not fused), npb.engine
    zs = G.sub(G.load("stress"), "s_block160")
    hs, hc = G.mats(zs)
    om = G.penalty(zs)
    N, Kc = zs["amps"].shape
    a = ControlField(N, Kc, float(zs["dt"]), zs["amps"])
    prob = ControlProblem(hs, tuple(hc), initial_state=zs["psi0"], basis=zs["basis"])
    terms = [CostTerm(CostKind.STATE_INFIDELITY, 0.7, target_state=zs["targets"]),
             CostTerm(CostKind.STATE_PENALTY, 0.2, penalty_op=om),
             CostTerm(CostKind.STATE_RUNNING_INFIDELITY, 0.4, target_state=zs["targets"])]
    _check(NativeProblem(prob, terms, initial_states=zs["psi0"]).grad(a), zs["cost_state"], zs["grad_state"])
    t = [CostTerm(CostKind.GATE_RUNNING_INFIDELITY, 1.0, target_images=zs["images"])]
    _check(NativeProblem(prob, t, basis=zs["basis"]).grad(a), zs["cost_g3"], zs["grad_g3"])
