"""GPU parity at BASELINE's full sizes where the reference finishes in minutes.

* c3 at full size (N=2000, K=8): golden ``c3_full.npz`` = the reference's composite_grad per state
  (src/costs.py:515-546 -> _state_pass :269-354), summed in state order (make_golden.py).
* c5 with ALL K=64 states on an N'=2 prefix: the full-K dense engine path.  Its forward chain has
  64 columns and its adjoint / aux chains 128 / 64, so every Taylor GEMM runs the wide-tile kernels
  every full-size c5 evaluation executes (DenseMatrix.matvec, src/sparse.py:193-199, inside
  expm.apply, src/expm.py:345-350): by default the TMA bulk-copy kernel ``lg_k_zgemm_taylor_bulk``
  (tile-aligned shapes) with its wave-filling split-k, and -- parametrised -- the same kernel without
  split-k (fused Taylor epilogue) and with an uneven split, and the cp.async kernel
  ``lg_k_zgemm_taylor_n32`` (LG_ZGEMM_BULK=0) with split-k 8.
* c4 at full size: engine agreement (below) and the directional derivative of the cost against the
  gradient, a size-independent property (the reference needs ~21 h for this configuration).
* The same dense cases with the wide tile forced from 1 column (LG_ZGEMM_N32=1) and with split-k
  forced off / to 8, so both GEMM kernels and the split-k epilogue meet every dense golden.

Bars: cost within 1e-12 absolute, gradient within 1e-9 relative (norm-wise).
"""

import numpy as np
import pytest

import _golden as G
from paper_2304_06200_b200 import ControlField, ControlProblem, CostKind, CostTerm, composite_grad, models
from paper_2304_06200_b200.costs import NativeProblem

pytestmark = pytest.mark.gpu

COST_TOL = 1e-12
GRAD_TOL = 1e-9


def _check(res, cost, grad):
    assert abs(res.cost - float(cost)) <= COST_TOL, (res.cost, float(cost))
    assert G.grad_rel(res.grad, grad) <= GRAD_TOL, G.grad_rel(res.grad, grad)


def test_c3_full_size_against_reference():
    z = G.load("c3_full")
    case = models.build_case("c3")
    _check(composite_grad(case.problem, case.field, case.terms), z["cost"], z["grad"])


@pytest.mark.parametrize("bulk,splitk", [(None, None), ("1", "1"), ("1", "5"), ("0", None)])
def test_c5_all_64_states_full_k_gemm_path(bulk, splitk, monkeypatch):
    if bulk is not None:
        monkeypatch.setenv("LG_ZGEMM_BULK", bulk)
    if splitk is not None:
        monkeypatch.setenv("LG_SPLITK", splitk)
    z = G.load("c5_fullk")
    n = int(z["n_prefix"])
    case = models.build_case("c5", n_steps=n, n_states=64)
    npb = NativeProblem(case.problem, case.terms, initial_states=case.problem.initial_state)
    assert npb.engine.startswith("dense"), npb.engine
    res = npb.grad(case.field)
    _check(res, z["cost"], z["grad"])
    # per-trajectory raw scalars: the final overlaps <psi_N|phi_t> of all 64 states reproduce each
    # state's reference cost 1 - |<phi|psi_N>|^2 individually
    assert abs(npb.cost(case.field) - float(z["cost"])) <= COST_TOL


@pytest.mark.parametrize("bulk", ["1", "0"])
@pytest.mark.parametrize("zfast", ["1", "0"])
def test_c5_fused_split_k_finish_is_bit_identical(bulk, zfast, monkeypatch):
    """LG_ZGEMM_FUSEDK=1 (the tile's last-arriving k-slice reduces it in slice order inside the GEMM)
    against the default two-kernel split-k path: same sums in the same order, so identical bits."""
    z = G.load("c5_fullk")
    case = models.build_case("c5", n_steps=int(z["n_prefix"]), n_states=64)
    monkeypatch.setenv("LG_ZGEMM_BULK", bulk)

    def run():
        return NativeProblem(case.problem, case.terms, initial_states=case.problem.initial_state).grad(case.field)

    base = run()
    monkeypatch.setenv("LG_ZGEMM_FUSEDK", "1")
    monkeypatch.setenv("LG_ZGEMM_ZFAST", zfast)
    fused = run()
    assert fused.cost == base.cost
    assert np.array_equal(fused.grad, base.grad)
    _check(fused, z["cost"], z["grad"])


@pytest.mark.parametrize("n32,splitk", [("1", None), ("1", "1"), ("0", "8"), ("1", "8")])
def test_dense_goldens_with_forced_gemm_tiles(n32, splitk, monkeypatch):
    monkeypatch.setenv("LG_ZGEMM_N32", n32)
    if splitk:
        monkeypatch.setenv("LG_SPLITK", splitk)
    z = G.load("c5")
    case = models.build_case("c5", n_steps=int(z["amps"].shape[0]), n_states=int(z["k_sub"]))
    _check(NativeProblem(case.problem, case.terms, initial_states=case.problem.initial_state).grad(case.field),
           z["cost"], z["grad"])
    # the dense stress variant (d = 160, all five cost kinds, +-1 rad/ns controls: plans vary per
    # step) on the dense GEMM engine (LG_ENGINE=dense; it otherwise takes d > 512 only)
    monkeypatch.setenv("LG_ENGINE", "dense")
    zs = G.sub(G.load("stress"), "s_denseblk160")
    hs, hc = G.mats(zs)
    om = G.penalty(zs)
    N, Kc = zs["amps"].shape
    a = ControlField(N, Kc, float(zs["dt"]), zs["amps"])
    prob = ControlProblem(hs, tuple(hc), initial_state=zs["psi0"], basis=zs["basis"])
    terms = [CostTerm(CostKind.STATE_INFIDELITY, 0.7, target_state=zs["targets"]),
             CostTerm(CostKind.STATE_PENALTY, 0.2, penalty_op=om),
             CostTerm(CostKind.STATE_RUNNING_INFIDELITY, 0.4, target_state=zs["targets"])]
    npb = NativeProblem(prob, terms, initial_states=zs["psi0"])
    assert npb.engine.startswith("dense"), npb.engine
    _check(npb.grad(a), zs["cost_state"], zs["grad_state"])
    for kind, ck, gk in [(CostKind.GATE_INFIDELITY, "cost_g1", "grad_g1"),
                         (CostKind.GATE_RUNNING_INFIDELITY, "cost_g3", "grad_g3")]:
        t = [CostTerm(kind, 1.0, target_images=zs["images"])]
        _check(NativeProblem(prob, t, basis=zs["basis"]).grad(a), zs[ck], zs[gk])


def test_c4_full_size_engine_agreement(monkeypatch):
    """c4 at FULL size (d = 10^4, K = 32, N = 4000; the reference needs ~21 h, so no golden): the
    bench configuration evaluated three ways must agree -- the LARGE kernels' two-phase backward
    (default), their fused backward (LG_CL_FUSED=1: bit-identical, the same chains on the same
    psi_{n-1} / lambda(n) values) and the generic cluster kernels (LG_CL_NOLARGE=1: another
    summation order, so 1e-12 / 1e-10) -- and composite_cost must equal composite_grad's cost
    bitwise.  The prefix golden (c4.npz, N' = 8, all 32 states) pins the same code path against
    the reference."""
    case = models.build_case("c4")

    def run():
        npb = NativeProblem(case.problem, case.terms, basis=case.problem.basis)
        return npb.engine, npb.grad(case.field), npb.cost(case.field)

    eng, res, cost = run()
    assert eng.startswith("cluster-large:lg_k_cll_adjoint"), eng
    assert cost == res.cost
    monkeypatch.setenv("LG_CL_FUSED", "1")
    eng_f, res_f, _ = run()
    assert eng_f.startswith("cluster-large:lg_k_cll_backward"), eng_f
    assert res_f.cost == res.cost and np.array_equal(res_f.grad, res.grad)
    monkeypatch.delenv("LG_CL_FUSED")
    monkeypatch.setenv("LG_CL_NOLARGE", "1")
    eng_g, res_g, _ = run()
    assert eng_g.startswith("cluster") and "large" not in eng_g, eng_g
    assert abs(res_g.cost - res.cost) <= COST_TOL
    assert G.grad_rel(res_g.grad, res.grad) <= 1e-10


def test_c4_full_size_directional_derivative():
    """Size-independent property at the bench configuration's full size: along a random direction v
    of the control field, the central difference of composite_cost (forward sweeps only) matches
    grad . v from composite_grad (forward + two-phase backward).  The two sides share only the
    forward sweep, so this pins the adjoint sweep and the derivative-product items of all 32
    trajectories and 4000 steps against the cost itself."""
    from paper_2304_06200_b200 import composite_cost

    case = models.build_case("c4")
    res = composite_grad(case.problem, case.field, case.terms)
    rng = np.random.default_rng(11)
    v = rng.standard_normal(res.grad.shape)
    v /= np.linalg.norm(v)
    # a direction with a gradient component, so the derivative is well above the FD noise floor
    v = 0.5 * v + 0.5 * res.grad / max(np.linalg.norm(res.grad), 1e-300)
    eps = 1e-4
    a0 = case.field.amplitudes
    cp = composite_cost(case.problem, case.field.replace_amplitudes(a0 + eps * v), case.terms)
    cm = composite_cost(case.problem, case.field.replace_amplitudes(a0 - eps * v), case.terms)
    fd = (cp - cm) / (2 * eps)
    gv = float(np.sum(res.grad * v))
    assert abs(fd - gv) <= 1e-5 * abs(gv) + 1e-11, (fd, gv)
