"""GPU: composite_cost_batch is bit-identical to composite_cost per field, and the optimizer with a
batched line search reproduces the sequential trace exactly (src/optimizer.py:153-170)."""

import time

import numpy as np
import pytest

from paper_2304_06200_b200 import composite_cost, composite_cost_batch, models
from paper_2304_06200_b200.optimizer import OptimizerConfig, grape_optimize

pytestmark = pytest.mark.gpu


def test_batch_costs_bit_identical():
    case = models.build_case("c2", n_steps=60)
    rng = np.random.default_rng(9)
    fields = [case.field.replace_amplitudes(case.field.amplitudes + rng.uniform(-0.02, 0.02, case.field.amplitudes.shape))
              for _ in range(6)]
    composite_cost_batch(case.problem, fields, case.terms)  # builds the per-slot device problems
    t0 = time.perf_counter()
    batch = composite_cost_batch(case.problem, fields, case.terms)
    t_batch = time.perf_counter() - t0
    t0 = time.perf_counter()
    single = [composite_cost(case.problem, f, case.terms) for f in fields]
    t_single = time.perf_counter() - t0
    assert batch == single
    print(f"6 costs (warm): batched {1e3 * t_batch:.2f} ms, sequential {1e3 * t_single:.2f} ms")


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
