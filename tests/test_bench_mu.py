"""Planning sweeps (the reference's bench-mu, src/bench.py:169-193, 281-313):
every record of ``bench_mu.measure_mu`` -- dimension, planner inputs (one-norm, sigma'), matvec
count, stored elements -- equals the reference's for every model family, size, time step and
tolerance in tests/golden/bench_mu.npz (bitwise: the norms follow numpy's reduction order and the
planner is the exact host port), including infeasible plans, and the sweep / fit helpers agree."""

import numpy as np
import pytest

import _golden as G
from paper_2304_06200_b200 import bench_mu as B


def _cases():
    z = G.load("bench_mu")
    return [(str(m), tuple(r)) for m, r in zip(z["models"], z["rows"])]


@pytest.mark.parametrize("model,row", _cases())
def test_measure_mu_matches_reference(model, row):
    d, norm1, sp, mu, kappa, tau, dt, size = row
    r = B.measure_mu(model, int(size), float(dt), float(tau))
    assert r.d == int(d) and r.sigma_prime == int(sp) and r.kappa == int(kappa)
    assert r.norm1 == norm1  # bitwise
    assert (-1 if r.matvecs is None else r.matvecs) == int(mu)


def test_dimension_sweep_csv_and_power_law():
    z = G.load("bench_mu")
    sweep = B.mu_vs_dim_sweep("transmon_cavity", [10, 20, 40, 80, 160], 1e-8)
    assert [r.to_csv_row() for r in sweep] == [str(c) for c in z["csv"]]
    fit = B.fit_power_law([(r.d, r.matvecs) for r in sweep])
    assert np.allclose([fit.exponent, fit.log_prefactor, fit.r_squared], z["fit"], rtol=0, atol=1e-12)
    norm = B.mu_vs_norm_sweep("transmon_cavity", 20, [0.1, 0.2, 0.4], 1e-8)
    assert [r.norm1 for r in norm] == sorted(r.norm1 for r in norm)


def test_unknown_model_and_fit_errors():
    with pytest.raises(ValueError):
        B.build_model("nope", 3)
    with pytest.raises(ValueError):
        B.fit_power_law([(1, 1), (2, 2), (3, 3)])
