"""GPU: the line-search path (src/optimizer.py:153-170).  composite_cost_batch evaluates
all candidate fields in ONE forward launch on the warp-specialised and cluster engines
(lg_cost_batch); every cost matches the oracle's composite_cost and is bit-identical to
composite_cost of that field, and the optimizer with a batched line search reproduces the
sequential trace exactly."""

import time

import numpy as np
import pytest

from oracle import lg_oracle as O
from paper_2304_06200_b200 import composite_cost, composite_cost_batch, models
from paper_2304_06200_b200.costs import CostKind, _native_for, _split
from paper_2304_06200_b200.optimizer import OptimizerConfig, grape_optimize
from paper_2304_06200_b200.sparse import DenseMatrix

pytestmark = pytest.mark.gpu

COST_TOL = 1e-12


def _om(m):
    if isinstance(m, DenseMatrix):
        return O.Dense(np.asfortranarray(m.array))
    return O.Csr(m.n_rows, m.row_offsets, m.col_indices, m.values)


def _oracle_cost(case, field):
    p = case.problem
    op = O.Problem(_om(p.h_static), tuple(_om(h) for h in p.h_controls), initial_states=p.initial_state,
                   basis=p.basis)
    kinds = {CostKind.STATE_INFIDELITY: O.STATE_INFIDELITY, CostKind.GATE_INFIDELITY: O.GATE_INFIDELITY,
             CostKind.STATE_PENALTY: O.STATE_PENALTY}
    terms = []
    for t in case.terms:
        tg = t.target_state if t.kind == CostKind.STATE_INFIDELITY else t.target_images
        terms.append(O.Term(kinds[t.kind], t.weight, tg, _om(t.penalty_op) if t.penalty_op is not None else None))
    return O.composite_cost(op, field.amplitudes, field.dt, terms)


@pytest.mark.parametrize("name,n_steps,n_states,k,engine", [("c2", 60, None, 6, "ws"), ("c3", 12, 3, 4, "cluster"),
                                                             ("c4", 3, 2, 3, "cluster-large")])
def test_batch_costs_one_launch_against_oracle(name, n_steps, n_states, k, engine):
    case = models.build_case(name, n_steps=n_steps, n_states=n_states)
    rng = np.random.default_rng(9)
    amp = 0.02 if name == "c2" else 0.005
    fields = [case.field.replace_amplitudes(case.field.amplitudes + rng.uniform(-amp, amp, case.field.amplitudes.shape))
              for _ in range(k)]
    terms, has_state = _split(case.terms)
    npb = _native_for(case.problem, terms, case.problem.initial_state if has_state else None, case.problem.basis)
    assert npb.engine.startswith(engine), npb.engine
    one_launch = npb.cost_batch(fields)  # the batched kernel itself (raises if the engine has none)
    batch = composite_cost_batch(case.problem, fields, case.terms)
    single = [composite_cost(case.problem, f, case.terms) for f in fields]
    assert batch == single == one_launch
    for f, c in zip(fields, batch):
        assert abs(c - _oracle_cost(case, f)) <= COST_TOL
    assert len(set(batch)) == k  # the candidates really differ


def test_batch_faster_than_sequential():
    case = models.build_case("c2", n_steps=400)
    rng = np.random.default_rng(3)
    fields = [case.field.replace_amplitudes(case.field.amplitudes + rng.uniform(-0.02, 0.02, case.field.amplitudes.shape))
              for _ in range(8)]
    composite_cost_batch(case.problem, fields, case.terms)  # warm (device buffers)
    t0 = time.perf_counter()
    batch = composite_cost_batch(case.problem, fields, case.terms)
    t_batch = time.perf_counter() - t0
    t0 = time.perf_counter()
    single = [composite_cost(case.problem, f, case.terms) for f in fields]
    t_single = time.perf_counter() - t0
    assert batch == single
    print(f"8 c2 costs (N=400, warm): one launch {1e3 * t_batch:.2f} ms, sequential {1e3 * t_single:.2f} ms")
    assert t_batch < t_single


def test_batched_line_search_trace_identical():
    case = models.build_case("c2", n_steps=40)
    runs = []
    for b in (1, 6):
        cfg = OptimizerConfig(max_iters=5, eta0=50.0, line_search_batch=b)
        runs.append(grape_optimize(case.problem, case.terms, case.field, cfg))
    ref, got = runs
    assert [(r.cost, r.eta_used) for r in got.records] == [(r.cost, r.eta_used) for r in ref.records]
    assert np.array_equal(got.final_field.amplitudes, ref.final_field.amplitudes)
    assert ref.records[-1].cost < ref.records[0].cost
