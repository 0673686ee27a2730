"""Host-side checks of the C-ABI library that need no GPU.

* the library loads and exports every entry point include/leangrape_b200.h declares;
* the exact host planner (used for guarded device plans) is bit-identical to the
  reference's make_plan on the golden table;
* the numpy-order reductions that feed the planner (lg_numpy.cuh) are bit-exact;
* the raw-scalar combine (lg_finalize_raw) reproduces the reference formulas.
"""

import ctypes as C
import os
import re

import numpy as np
import pytest

import _golden as G
from paper_2304_06200_b200 import _native
from paper_2304_06200_b200.expm import PlanningError, make_plan

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "leangrape_b200.h")


def test_library_exports_every_declared_symbol(lib):
    text = open(HEADER).read()
    declared = set(re.findall(r"\b(lg_[a-z0-9_]+)\s*\(", text))
    assert declared, "no declarations parsed"
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_native.EXPORTED) <= declared
    assert b"sm_100a" in lib.lg_version()


def test_host_planner_bit_identical_to_reference():
    z = G.load("planner")
    for norm, sp, tau, m, s, b, st in zip(z["norm"], z["sp"], z["tau"], z["m"], z["s"], z["bound"], z["status"]):
        if st:
            with pytest.raises(PlanningError):
                make_plan(float(norm), int(sp), float(tau))
            continue
        p = make_plan(float(norm), int(sp), float(tau))
        assert (p.order, p.scaling) == (m, s), (norm, sp, tau)
        assert p.bound == b, (norm, sp, tau)


def test_planner_errors_map_to_reference_exceptions():
    with pytest.raises(PlanningError, match="norm1=1000"):
        make_plan(1000.0, 5, 1e-12, s_max=100)
    with pytest.raises(ValueError):
        make_plan(1.0, 1, 0.0)
    with pytest.raises(ValueError, match="non-negative"):
        make_plan(float("nan"), 1, 1e-8)
    p = make_plan(0.0, 5, 1e-8)
    assert (p.order, p.scaling, p.matvecs) == (1, 1, 1)


def test_numpy_abs_bit_exact(lib):
    z = G.load("numpy_rules")
    zz = np.ascontiguousarray(z["z"])
    out = np.zeros(zz.size)
    lib.lg_np_cabs_host(zz.size, _native.dptr(zz.view(np.float64)), _native.dptr(out))
    assert np.array_equal(out, z["absz"])
    assert np.array_equal(out, np.abs(zz))


@pytest.mark.parametrize("n", [1, 2, 3, 5, 7, 8, 9, 15, 16, 17, 40, 80, 127, 128, 129, 200, 256, 1000, 4096, 4097])
def test_numpy_reduction_orders_bit_exact(lib, n):
    rng = np.random.default_rng(n)
    for _ in range(20):
        a = np.ascontiguousarray(np.abs(rng.standard_normal(n)) * np.exp(rng.uniform(-8, 8, n)))
        # reduceat segment (CSR row sums): a0 + pairwise(rest)
        assert lib.lg_np_reduce_host(n, _native.dptr(a)) == np.add.reduceat(a, [0])[0]
        # plain 1-D sum: pairwise over everything
        assert lib.lg_np_pairwise_host(n, _native.dptr(a)) == a.sum()
        # dense column sum of an F-ordered matrix: pairwise over the whole column
        m = np.asfortranarray(np.stack([a, a[::-1]], axis=1))
        assert lib.lg_np_pairwise_host(n, _native.dptr(a)) == m.sum(axis=0)[0]


def _final_py(kinds, weights, t0, K, N, Kc, T, ip, fin, trp, run):
    """The reference's cost/grad formulas on raw per-trajectory scalars."""
    cost, grad = 0.0, np.zeros((N, Kc))
    for s, kind in enumerate(kinds):
        sl = slice(t0[s], t0[s] + K[s])
        w = weights[s]
        if kind == 0:
            z = fin[s, sl]
            cost += w * np.mean(1 - np.abs(z) ** 2)
            grad += w * np.mean(-2 * (ip[:, s, :, sl] * z).real, axis=-1)
        elif kind == 1:
            cost += w * np.mean(run[s, sl] / N)
            grad += w * np.mean(2.0 / N * ip[:, s, :, sl].real, axis=-1)
        elif kind == 2:
            cost += w * np.mean(1 - run[s, sl] / N)
            grad += w * np.mean(-2.0 / N * ip[:, s, :, sl].real, axis=-1)
        elif kind == 3:
            tr = fin[s, sl].sum()
            cost += w * (1 - abs(tr) ** 2 / K[s] ** 2)
            grad += w * (-2.0 / K[s] ** 2 * (ip[:, s, :, sl].sum(-1) * np.conj(tr)).real)
        else:
            tr = trp[s, :, sl].sum(-1)
            cost += w * (1 - np.sum(np.abs(tr) ** 2) / (N * K[s] ** 2))
            grad += w * (-2.0 / (N * K[s] ** 2) * ip[:, s, :, sl].sum(-1).real)
    return cost, grad


def test_finalize_raw_matches_reference_formulas(lib):
    rng = np.random.default_rng(5)
    N, Kc, T = 7, 3, 5
    kinds = np.array([0, 1, 2, 3, 4], np.int32)
    weights = np.array([0.7, 0.2, 0.4, 1.0, 0.3])
    t0 = np.array([0, 0, 0, 2, 2], np.int32)
    K = np.array([2, 2, 2, 3, 3], np.int32)
    S = kinds.size
    cz = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)
    ip, fin, trp, run = cz(N, S, Kc, T), cz(S, T), cz(S, N, T), rng.random((S, T))
    raw = np.concatenate([ip.ravel().view(np.float64), fin.ravel().view(np.float64),
                          trp.ravel().view(np.float64), run.ravel()])
    cost, grad = C.c_double(), np.zeros((N, Kc))
    _native.check(lib.lg_finalize_raw(S, _native.i32ptr(kinds), _native.dptr(weights), _native.i32ptr(t0),
                                      _native.i32ptr(K), N, Kc, T, _native.dptr(raw), C.byref(cost),
                                      _native.dptr(grad)))
    c_ref, g_ref = _final_py(kinds, weights, t0, K, N, Kc, T, ip, fin, trp, run)
    assert abs(cost.value - c_ref) <= 1e-14
    assert np.allclose(grad, g_ref, rtol=1e-13, atol=1e-15)


def test_no_cpu_fallback_without_device(lib):
    """With no CUDA device the product raises instead of computing on the host."""
    if lib.lg_device_count() > 0:
        pytest.skip("a CUDA device is present")
    from paper_2304_06200_b200 import models

    case = models.build_case("c2", n_steps=4)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        from paper_2304_06200_b200.costs import composite_grad

        composite_grad(case.problem, case.field, case.terms)
