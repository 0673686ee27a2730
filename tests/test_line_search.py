"""Batched backtracking line search (src/optimizer.py:153-170): evaluating several
candidates per batch must reproduce the sequential loop's trace exactly (accepted eta, fields,
stall behaviour).  CPU: an analytic cost; the GPU version is in test_gpu_line_search.py."""

import numpy as np
import pytest

from paper_2304_06200_b200 import ControlField
from paper_2304_06200_b200.costs import GradientResult
from paper_2304_06200_b200.optimizer import OptimizerConfig, grape_optimize

TARGET = np.linspace(-0.3, 0.4, 12).reshape(6, 2)


def cost(_p, a, _t):
    x = a.amplitudes - TARGET
    return float(np.sum(x ** 4) + 0.3 * np.sum(np.sin(3 * x) ** 2))


def grad(_p, a, _t):
    x = a.amplitudes - TARGET
    return GradientResult(cost=cost(None, a, None), grad=4 * x ** 3 + 0.9 * np.sin(6 * x), live_vector_peak=0)


class _P:
    n_channels = 2


def run(batch, eta0=3.0, shrink=0.5, max_backtracks=60, iters=25):
    calls = []

    def cost_batch(p, fields, t):
        calls.append(len(fields))
        return [cost(p, f, t) for f in fields]

    a0 = ControlField(6, 2, 0.5, np.zeros((6, 2)))
    cfg = OptimizerConfig(max_iters=iters, eta0=eta0, shrink=shrink, max_backtracks=max_backtracks,
                          line_search_batch=batch)
    tr = grape_optimize(_P(), [], a0, cfg, grad_fn=grad, cost_fn=cost, cost_batch_fn=cost_batch)
    return tr, calls


@pytest.mark.parametrize("batch", [2, 3, 8, 60])
def test_batched_trace_equals_sequential(batch):
    ref, _ = run(1)
    got, calls = run(batch)
    assert got.stop_reason == ref.stop_reason
    assert [(r.cost, r.eta_used) for r in got.records] == [(r.cost, r.eta_used) for r in ref.records]
    assert np.array_equal(got.final_field.amplitudes, ref.final_field.amplitudes)
    assert calls and max(calls) <= batch


def test_stall_is_reported_identically():
    # the cost cannot decrease with a tiny backtracking budget and a huge first step
    ref, _ = run(1, eta0=1e6, shrink=0.9, max_backtracks=5, iters=5)
    got, _ = run(4, eta0=1e6, shrink=0.9, max_backtracks=5, iters=5)
    assert ref.stop_reason == got.stop_reason == "line_search_stalled"
    assert [(r.cost, r.eta_used) for r in got.records] == [(r.cost, r.eta_used) for r in ref.records]


def test_bad_batch_rejected():
    with pytest.raises(ValueError):
        OptimizerConfig(line_search_batch=0)
