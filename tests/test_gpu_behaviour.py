"""Behavioural checks of the device path through the public API, after the reference's own test
strategy for this path (pkg/tests/test_costs.py, test_optimizer.py, test_derivatives.py):
closed forms on a single qubit, central finite differences for every cost kind on both derivative
backends, identity / stationary cases with EMPTY operators (no stored entries), single-step
reductions, composite identities, argument validation, range / gauge / determinism invariants, and
the steepest-descent driver's stopping rules.  Nothing here needs the oracle: every expectation is
analytic or self-consistent, so these also hold at sizes no golden covers.

Tolerances: closed forms 1e-10 (cost) / 1e-9 (gradient) at tau = 1e-12; finite differences 1e-6
relative (step 1e-6, truncation-limited); identities between two device evaluations 1e-12."""

import numpy as np
import pytest

from paper_2304_06200_b200 import costs, optimizer, sparse
from paper_2304_06200_b200.costs import Backend, ControlField, ControlProblem, CostKind, CostTerm

pytestmark = pytest.mark.gpu

PAULI_X = np.array([[0.0, 1.0], [1.0, 0.0]], np.complex128)
BOTH_BACKENDS = [Backend.SCALING_SQUARING, Backend.DIAGONALIZATION]


# ------------------------------------------------------------------------------------------ helpers
def _herm(g, d, scale=1.0):
    z = g.standard_normal((d, d)) + 1j * g.standard_normal((d, d))
    return scale * (z + z.conj().T) / 2


def _ket(g, d):
    v = g.standard_normal(d) + 1j * g.standard_normal(d)
    return v / np.linalg.norm(v)


def _unitary(g, d):
    q, _ = np.linalg.qr(g.standard_normal((d, d)) + 1j * g.standard_normal((d, d)))
    return q


def _empty(d):
    return sparse.build_csr([], d, d)


def _random_problem(g, d, channels, backend=Backend.SCALING_SQUARING, tau=1e-12, psi0=None):
    return ControlProblem(sparse.from_dense(_herm(g, d)), tuple(sparse.from_dense(_herm(g, d)) for _ in range(channels)),
                          backend, tau, initial_state=psi0)


def _random_field(g, n, channels, dt, scale=0.5):
    return ControlField(n, channels, dt, g.normal(scale=scale, size=(n, channels)))


def _central_differences(cost_of, field, h=1e-6):
    base = field.amplitudes
    out = np.empty_like(base)
    for idx in np.ndindex(*base.shape):
        hi, lo = base.copy(), base.copy()
        hi[idx] += h
        lo[idx] -= h
        out[idx] = (cost_of(field.replace_amplitudes(hi)) - cost_of(field.replace_amplitudes(lo))) / (2 * h)
    return out


def _check_against_differences(result, cost_of, field, rtol=1e-6):
    fd = _central_differences(cost_of, field)
    assert np.linalg.norm(result.grad - fd) <= rtol * max(np.linalg.norm(fd), 1e-300)


@pytest.fixture
def g():
    return np.random.default_rng(4182)


# ------------------------------------------------------------------------------- forward propagation
def test_propagation_with_no_stored_entries_is_identity(g):
    d = 4
    problem = ControlProblem(_empty(d), (sparse.identity_csr(d),))
    psi0 = _ket(g, d)
    out = costs.forward_propagate(problem, ControlField.constant(0.0, 1, 1, 0.5), psi0)
    assert np.allclose(out, psi0, atol=1e-12)


def test_pi_pulse_flips_the_qubit():
    problem = ControlProblem(_empty(2), (sparse.from_dense(PAULI_X),), tau=1e-12)
    out = costs.forward_propagate(problem, ControlField.constant(np.pi / 2, 1, 1, 1.0), np.array([1.0, 0.0], complex))
    assert abs(abs(out[1]) - 1.0) <= 1e-10
    assert abs(out[0]) <= 1e-10


def test_propagation_keeps_the_norm_within_the_certified_error(g):
    d, n, tau = 8, 12, 1e-10
    problem = _random_problem(g, d, 2, tau=tau)
    out = costs.forward_propagate(problem, _random_field(g, n, 2, 0.2, 0.4), _ket(g, d))
    assert abs(np.linalg.norm(out) - 1.0) <= 2 * n * tau


# ------------------------------------------------------------------------ state-transfer infidelity
def test_state_infidelity_vanishes_when_nothing_moves(g):
    d = 4
    psi = _ket(g, d)
    problem = ControlProblem(_empty(d), (_empty(d),))
    res = costs.c1_state_grad(problem, ControlField.constant(0.0, 3, 1, 0.4), psi, psi)
    assert res.cost <= 1e-12
    assert np.abs(res.grad).max() <= 1e-12


@pytest.mark.parametrize("backend", BOTH_BACKENDS)
def test_state_infidelity_single_qubit_closed_form(backend):
    # H = a X from |0> to |1>: C = cos^2(a dt), dC/da = -dt sin(2 a dt)
    a, dt = np.pi / 7, 0.9
    problem = ControlProblem(_empty(2), (sparse.from_dense(PAULI_X),), backend, 1e-12)
    res = costs.c1_state_grad(problem, ControlField.constant(a, 1, 1, dt), np.array([1, 0], complex),
                              np.array([0, 1], complex))
    assert res.cost == pytest.approx(np.cos(a * dt) ** 2, abs=1e-10)
    assert res.grad[0, 0] == pytest.approx(-dt * np.sin(2 * a * dt), abs=1e-9)


@pytest.mark.parametrize("backend", BOTH_BACKENDS)
def test_state_infidelity_gradient_matches_differences(g, backend):
    d, n, k = 8, 5, 2
    psi0, phi = _ket(g, d), _ket(g, d)
    problem = _random_problem(g, d, k, backend)
    field = _random_field(g, n, k, 0.3)
    res = costs.c1_state_grad(problem, field, psi0, phi)
    _check_against_differences(res, lambda f: costs.c1_state_grad(problem, f, psi0, phi).cost, field)


# ------------------------------------------------------------------------------- occupation penalty
def test_identity_penalty_is_one_with_zero_gradient(g):
    d, n = 5, 4
    problem = _random_problem(g, d, 1)
    res = costs.c2_state_grad(problem, _random_field(g, n, 1, 0.2, 1.0), _ket(g, d), sparse.identity_csr(d))
    assert res.cost == pytest.approx(1.0, abs=1e-9)
    assert np.abs(res.grad).max() <= 1e-8


def test_empty_penalty_gives_exact_zeros(g):
    d, n = 4, 3
    problem = _random_problem(g, d, 1)
    res = costs.c2_state_grad(problem, _random_field(g, n, 1, 0.2, 1.0), _ket(g, d), _empty(d))
    assert res.cost == 0.0
    assert np.abs(res.grad).max() == 0.0


@pytest.mark.parametrize("backend", BOTH_BACKENDS)
def test_penalty_gradient_matches_differences(g, backend):
    d, n, k = 8, 4, 2
    psi0 = _ket(g, d)
    omega = sparse.from_dense(_herm(g, d))
    problem = _random_problem(g, d, k, backend)
    field = _random_field(g, n, k, 0.25)
    res = costs.c2_state_grad(problem, field, psi0, omega)
    _check_against_differences(res, lambda f: costs.c2_state_grad(problem, f, psi0, omega).cost, field)


def test_penalty_must_be_hermitian(g):
    d = 3
    problem = _random_problem(g, d, 1)
    lopsided = sparse.build_csr([(0, 1, 1.0)], d, d)
    with pytest.raises(ValueError, match="Hermitian"):
        costs.c2_state_grad(problem, ControlField.constant(0.1, 2, 1, 0.2), _ket(g, d), lopsided)


# ------------------------------------------------------------------ time-integrated state infidelity
def test_running_state_cost_vanishes_at_a_stationary_target(g):
    d = 4
    psi = _ket(g, d)
    problem = ControlProblem(_empty(d), (_empty(d),))
    assert costs.c3_state_grad(problem, ControlField.constant(0.0, 4, 1, 0.3), psi, psi).cost <= 1e-12


def test_running_state_cost_of_one_step_is_the_final_cost(g):
    d, k = 6, 2
    psi0, phi = _ket(g, d), _ket(g, d)
    problem = _random_problem(g, d, k)
    field = _random_field(g, 1, k, 0.4, 1.0)
    final, running = costs.c1_state_grad(problem, field, psi0, phi), costs.c3_state_grad(problem, field, psi0, phi)
    assert running.cost == pytest.approx(final.cost, abs=1e-12)
    assert np.abs(running.grad - final.grad).max() <= 1e-12


@pytest.mark.parametrize("backend", BOTH_BACKENDS)
def test_running_state_gradient_matches_differences(g, backend):
    d, n, k = 8, 4, 2
    psi0, phi = _ket(g, d), _ket(g, d)
    problem = _random_problem(g, d, k, backend)
    field = _random_field(g, n, k, 0.3)
    res = costs.c3_state_grad(problem, field, psi0, phi)
    _check_against_differences(res, lambda f: costs.c3_state_grad(problem, f, psi0, phi).cost, field)


# ----------------------------------------------------------------------------------- gate infidelity
def test_gate_infidelity_of_identity_dynamics_against_identity(g):
    d = 3
    problem = ControlProblem(_empty(d), (_empty(d),))
    assert costs.c1_gate_grad(problem, ControlField.constant(0.0, 2, 1, 0.3), np.eye(d, dtype=complex)).cost <= 1e-12


@pytest.mark.parametrize("backend", BOTH_BACKENDS)
def test_gate_infidelity_single_qubit_closed_form(backend):
    # U = exp(-i a dt X), target X: |tr(X^dagger U)|^2 / 4 = sin^2(a dt)
    a, dt = np.pi / 7, 0.9
    problem = ControlProblem(_empty(2), (sparse.from_dense(PAULI_X),), backend, 1e-12)
    res = costs.c1_gate_grad(problem, ControlField.constant(a, 1, 1, dt), PAULI_X.copy())
    assert res.cost == pytest.approx(np.cos(a * dt) ** 2, abs=1e-10)
    assert res.grad[0, 0] == pytest.approx(-dt * np.sin(2 * a * dt), abs=1e-9)


@pytest.mark.parametrize("backend", BOTH_BACKENDS)
def test_gate_infidelity_gradient_matches_differences(g, backend):
    d, n, k = 6, 3, 2
    problem = _random_problem(g, d, k, backend)
    target = _unitary(g, d)
    field = _random_field(g, n, k, 0.3)
    res = costs.c1_gate_grad(problem, field, target)
    _check_against_differences(res, lambda f: costs.c1_gate_grad(problem, f, target).cost, field)


def test_gate_basis_must_be_orthonormal(g):
    d = 3
    problem = _random_problem(g, d, 1)
    skewed = [_ket(g, d) for _ in range(d)]
    with pytest.raises(ValueError, match="orthonormal"):
        costs.c1_gate_grad(problem, ControlField.constant(0.1, 1, 1, 0.2), np.eye(d, dtype=complex), skewed)


# ------------------------------------------------------------------- time-integrated gate infidelity
def test_running_gate_cost_of_identity_dynamics(g):
    d = 3
    problem = ControlProblem(_empty(d), (_empty(d),))
    assert costs.c3_gate_grad(problem, ControlField.constant(0.0, 3, 1, 0.3), np.eye(d, dtype=complex)).cost <= 1e-12


def test_running_gate_cost_of_one_step_is_the_gate_infidelity(g):
    d, k = 4, 2
    problem = _random_problem(g, d, k)
    target = _unitary(g, d)
    field = _random_field(g, 1, k, 0.35, 1.0)
    final, running = costs.c1_gate_grad(problem, field, target), costs.c3_gate_grad(problem, field, target)
    assert running.cost == pytest.approx(final.cost, abs=1e-12)
    assert np.abs(running.grad - final.grad).max() <= 1e-12


@pytest.mark.parametrize("backend", BOTH_BACKENDS)
def test_running_gate_gradient_matches_differences(g, backend):
    d, n, k = 4, 3, 2
    problem = _random_problem(g, d, k, backend)
    target = _unitary(g, d)
    field = _random_field(g, n, k, 0.3)
    res = costs.c3_gate_grad(problem, field, target)
    _check_against_differences(res, lambda f: costs.c3_gate_grad(problem, f, target).cost, field)


# ---------------------------------------------------------------------------------------- composites
def test_one_term_composite_equals_the_direct_function(g):
    d, n, k = 5, 3, 2
    psi0, phi = _ket(g, d), _ket(g, d)
    problem = _random_problem(g, d, k, psi0=psi0)
    field = _random_field(g, n, k, 0.3, 1.0)
    direct = costs.c1_state_grad(problem, field, psi0, phi)
    combo = costs.composite_grad(problem, field, [CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=phi)])
    assert combo.cost == pytest.approx(direct.cost, abs=1e-14)
    assert np.abs(combo.grad - direct.grad).max() <= 1e-14


def test_zero_weight_term_drops_out(g):
    d, n = 5, 3
    psi0, phi = _ket(g, d), _ket(g, d)
    omega = sparse.from_dense(_herm(g, d))
    problem = _random_problem(g, d, 1, psi0=psi0)
    field = _random_field(g, n, 1, 0.3, 1.0)
    combo = costs.composite_grad(problem, field, [CostTerm(CostKind.STATE_INFIDELITY, 0.0, target_state=phi),
                                                  CostTerm(CostKind.STATE_PENALTY, 1.0, penalty_op=omega)])
    alone = costs.c2_state_grad(problem, field, psi0, omega)
    assert combo.cost == pytest.approx(alone.cost, abs=1e-13)
    assert np.abs(combo.grad - alone.grad).max() <= 1e-13


def test_fused_pass_equals_the_weighted_sum_of_separate_passes(g):
    d, n, k = 6, 4, 2
    psi0, phi = _ket(g, d), _ket(g, d)
    omega = sparse.from_dense(_herm(g, d))
    problem = _random_problem(g, d, k, psi0=psi0)
    field = _random_field(g, n, k, 0.25, 1.0)
    wa, wb = 0.7, 0.4
    fused = costs.composite_grad(problem, field, [CostTerm(CostKind.STATE_INFIDELITY, wa, target_state=phi),
                                                  CostTerm(CostKind.STATE_PENALTY, wb, penalty_op=omega)])
    ra, rb = costs.c1_state_grad(problem, field, psi0, phi), costs.c2_state_grad(problem, field, psi0, omega)
    assert fused.cost == pytest.approx(wa * ra.cost + wb * rb.cost, abs=1e-12)
    assert np.abs(fused.grad - (wa * ra.grad + wb * rb.grad)).max() <= 1e-12


def test_cost_only_pass_agrees_with_the_gradient_pass(g):
    d, n, k = 5, 3, 2
    psi0, phi = _ket(g, d), _ket(g, d)
    problem = _random_problem(g, d, k, psi0=psi0)
    field = _random_field(g, n, k, 0.3, 1.0)
    terms = [CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=phi)]
    assert costs.composite_cost(problem, field, terms) == pytest.approx(costs.composite_grad(problem, field, terms).cost,
                                                                        abs=1e-13)


def test_composite_needs_a_term(g):
    problem = _random_problem(g, 3, 1)
    with pytest.raises(ValueError):
        costs.composite_grad(problem, ControlField.constant(0.1, 2, 1, 0.2), [])


# ---------------------------------------------------------------------------------------- validation
def test_term_without_payload_is_rejected():
    with pytest.raises(ValueError, match="target_state"):
        CostTerm(CostKind.STATE_INFIDELITY, 1.0)


def test_non_unitary_gate_is_rejected(g):
    with pytest.raises(ValueError, match="unitary"):
        CostTerm(CostKind.GATE_INFIDELITY, 1.0, target_gate=g.standard_normal((3, 3)).astype(complex))


def test_negative_weight_is_rejected(g):
    with pytest.raises(ValueError, match="weight"):
        CostTerm(CostKind.STATE_INFIDELITY, -0.5, target_state=_ket(g, 3))


# ---------------------------------------------------------------------------------------- invariants
def test_normalised_costs_stay_in_the_unit_interval(g):
    tau = 1e-10
    for _ in range(8):
        d = int(g.integers(3, 9))
        n, k = int(g.integers(1, 5)), int(g.integers(1, 3))
        psi0, phi, target = _ket(g, d), _ket(g, d), _unitary(g, d)
        problem = _random_problem(g, d, k, tau=tau)
        field = _random_field(g, n, k, 0.3, 0.3)
        for res in (costs.c1_state_grad(problem, field, psi0, phi), costs.c3_state_grad(problem, field, psi0, phi),
                    costs.c1_gate_grad(problem, field, target), costs.c3_gate_grad(problem, field, target)):
            assert -10 * tau <= res.cost <= 1.0 + 10 * tau


def test_gate_cost_ignores_a_global_phase_of_the_target(g):
    d, n = 4, 2
    problem = _random_problem(g, d, 1)
    target = _unitary(g, d)
    field = _random_field(g, n, 1, 0.3, 1.0)
    plain = costs.c1_gate_grad(problem, field, target)
    rotated = costs.c1_gate_grad(problem, field, np.exp(0.7j) * target)
    assert rotated.cost == pytest.approx(plain.cost, abs=1e-10)
    assert np.abs(rotated.grad - plain.grad).max() <= 1e-10


def test_live_vector_peak_does_not_grow_with_the_step_count(g):
    d = 6
    psi0, phi = _ket(g, d), _ket(g, d)
    problem = _random_problem(g, d, 1)
    peaks = [costs.c1_state_grad(problem, _random_field(g, n, 1, 0.05, 0.2), psi0, phi).live_vector_peak
             for n in (5, 50)]
    assert peaks[0] == peaks[1] and peaks[0] >= 1


def test_repeated_evaluations_are_bit_identical(g):
    d, n, k = 5, 3, 2
    psi0, phi = _ket(g, d), _ket(g, d)
    problem = _random_problem(g, d, k)
    field = _random_field(g, n, k, 0.3, 1.0)
    first, second = costs.c1_state_grad(problem, field, psi0, phi), costs.c1_state_grad(problem, field, psi0, phi)
    assert first.cost == second.cost
    assert np.array_equal(first.grad, second.grad)


# ------------------------------------------------------------------------------- steepest descent
def _qubit_transfer(tau=1e-10):
    problem = ControlProblem(_empty(2), (sparse.from_dense(PAULI_X),), tau=tau, initial_state=np.array([1.0, 0.0], complex))
    return problem, [CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=np.array([0.0, 1.0], complex))]


def test_descent_stops_at_once_on_a_zero_gradient(g):
    d = 3
    problem = ControlProblem(sparse.from_dense(_herm(g, d)), (_empty(d),), initial_state=_ket(g, d))
    terms = [CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=_ket(g, d))]
    start = ControlField.constant(0.3, 4, 1, 0.2)
    trace = optimizer.grape_optimize(problem, terms, start, optimizer.OptimizerConfig(max_iters=10, stop_grad_norm=1e-12))
    assert trace.stop_reason == "stop_grad_norm" and len(trace.records) == 1
    assert np.array_equal(trace.final_field.amplitudes, start.amplitudes)


def test_descent_reaches_the_pi_pulse():
    problem, terms = _qubit_transfer()
    cfg = optimizer.OptimizerConfig(max_iters=200, eta0=0.1, eta_schedule="backtracking", stop_cost=1e-7)
    trace = optimizer.grape_optimize(problem, terms, ControlField.constant(0.1, 10, 1, 0.1), cfg)
    assert trace.stop_reason == "stop_cost" and trace.final_cost <= 1e-6


def test_backtracking_never_raises_the_cost():
    for seed in range(12):
        r = np.random.default_rng(900 + seed)
        d, n, k = 4, 5, 2
        problem = ControlProblem(sparse.from_dense(_herm(r, d)), tuple(sparse.from_dense(_herm(r, d)) for _ in range(k)),
                                 tau=1e-10, initial_state=_ket(r, d))
        terms = [CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=_ket(r, d))]
        trace = optimizer.grape_optimize(problem, terms, _random_field(r, n, k, 0.2, 0.3),
                                         optimizer.OptimizerConfig(max_iters=15, eta0=0.5))
        seq = [rec.cost for rec in trace.records]
        assert all(b <= a + 1e-15 for a, b in zip(seq, seq[1:]))


def test_constant_schedule_uses_the_whole_budget():
    problem, terms = _qubit_transfer()
    trace = optimizer.grape_optimize(problem, terms, ControlField.constant(0.1, 5, 1, 0.1),
                                     optimizer.OptimizerConfig(max_iters=5, eta0=0.05, eta_schedule="constant"))
    assert len(trace.records) == 5 and trace.stop_reason == "max_iters"


def test_descent_traces_repeat_exactly():
    problem, terms = _qubit_transfer()
    start, cfg = ControlField.constant(0.1, 8, 1, 0.1), optimizer.OptimizerConfig(max_iters=30, eta0=0.2)
    one, two = optimizer.grape_optimize(problem, terms, start, cfg), optimizer.grape_optimize(problem, terms, start, cfg)
    assert [r.cost for r in one.records] == [r.cost for r in two.records]
    assert [r.grad_inf_norm for r in one.records] == [r.grad_inf_norm for r in two.records]
    assert np.array_equal(one.final_field.amplitudes, two.final_field.amplitudes)


def test_trace_csv_has_a_header_and_one_line_per_record():
    problem, terms = _qubit_transfer()
    trace = optimizer.grape_optimize(problem, terms, ControlField.constant(0.1, 4, 1, 0.1),
                                     optimizer.OptimizerConfig(max_iters=3))
    lines = trace.to_csv_lines()
    assert lines[0] == "iter,cost,grad_inf_norm,eta,wall_ms" and len(lines) == len(trace.records) + 1


def test_optimizer_config_rejects_bad_values():
    for bad in (dict(eta0=-1.0), dict(eta_schedule="adam"), dict(shrink=1.5)):
        with pytest.raises(ValueError):
            optimizer.OptimizerConfig(**bad)


def test_runaway_step_returns_the_partial_trace():
    # an absurd constant step blows the amplitudes up: the driver must hand back what it recorded
    problem, terms = _qubit_transfer()
    trace = optimizer.grape_optimize(problem, terms, ControlField.constant(0.1, 5, 1, 0.1),
                                     optimizer.OptimizerConfig(max_iters=400, eta0=1e9, eta_schedule="constant"))
    assert trace.records
    assert trace.stop_reason.startswith("evaluation_failure") or trace.stop_reason in ("max_iters", "stop_cost")
