"""GPU edge cases through the C ABI, each engine: a single step, exactly-zero amplitudes (the
reference drops exact zeros from H_n, src/sparse.py:261-263, which changes sigma' and the norms),
three control channels, every cost kind at once, forward-only cost, and the error conventions
(PlanningError for an infeasible tau, ValueError for non-finite amplitudes / bad shapes).
Bars as tests/test_gpu_parity.py: cost 1e-12 absolute, gradient 1e-9 relative (norm-wise)."""

import numpy as np
import pytest

import _golden as G
from oracle import lg_oracle as O
from paper_2304_06200_b200 import (
    ControlField,
    ControlProblem,
    CostKind,
    CostTerm,
    CsrMatrix,
    DenseMatrix,
    PlanningError,
    composite_cost,
    composite_grad,
)
from paper_2304_06200_b200.costs import NativeProblem

pytestmark = pytest.mark.gpu

W = [0.7, 0.2, 0.4, 1.0, 0.5]


def _herm_sparse(rng, d, offsets, scale):
    """Hermitian banded matrix with the given diagonal offsets (complex entries, real diagonal)."""
    m = np.zeros((d, d), np.complex128)
    for o in offsets:
        n = d - abs(o)
        v = scale * (rng.standard_normal(n) + (1j * rng.standard_normal(n) if o else 0))
        if o >= 0:
            m[np.arange(n), np.arange(n) + o] += v
            if o:
                m[np.arange(n) + o, np.arange(n)] += np.conj(v)
    return m


def _csr(m):
    rows, cols = np.nonzero(m)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    indptr = np.zeros(m.shape[0] + 1, np.int64)
    np.add.at(indptr, rows + 1, 1)
    return np.cumsum(indptr), cols.astype(np.int64), m[rows, cols]


def _states(rng, k, d):
    s = rng.standard_normal((k, d)) + 1j * rng.standard_normal((k, d))
    return s / np.linalg.norm(s, axis=1, keepdims=True)


def _case(kind, seed=7, n_steps=6, kc=3):
    """kind: 'ws' (sparse d=48), 'wsdense' (dense d=40), 'cl' (sparse d=320), 'cta' (dense d=24, engine
    forced), 'dense' (dense d=600)."""
    rng = np.random.default_rng(seed)
    d = {"ws": 48, "wsdense": 40, "cl": 320, "cta": 24, "dense": 600}[kind]
    dense = kind in ("wsdense", "cta", "dense")
    if dense:
        hs = _herm_sparse(rng, d, range(d), 1.0 / d)
        hc = [_herm_sparse(rng, d, range(d), 0.3 / d) for _ in range(kc)]
    else:
        hs = _herm_sparse(rng, d, (0, 1, 7), 0.6)
        hc = [_herm_sparse(rng, d, (1,) if c % 2 == 0 else (7,), 0.4) for c in range(kc)]
    K = 3
    psi0, tgt, basis, img = _states(rng, K, d), _states(rng, K, d), None, None
    q, _ = np.linalg.qr(rng.standard_normal((d, K)) + 1j * rng.standard_normal((d, K)))
    basis = q.T.copy()
    img = _states(rng, K, d)
    pen = np.zeros((d, d), np.complex128)
    pen[np.arange(0, d, 5), np.arange(0, d, 5)] = 1.0
    amps = rng.uniform(-0.5, 0.5, (n_steps, kc))
    return dict(d=d, dense=dense, hs=hs, hc=hc, psi0=psi0, tgt=tgt, basis=basis, img=img, pen=pen, amps=amps,
                dt=0.3)


def _product(c, kinds):
    if c["dense"]:
        mk = lambda m: DenseMatrix(np.asfortranarray(m))  # noqa: E731
    else:
        mk = lambda m: CsrMatrix(m.shape[0], m.shape[1], *_csr(m))  # noqa: E731
    prob = ControlProblem(mk(c["hs"]), tuple(mk(h) for h in c["hc"]), initial_state=c["psi0"], basis=c["basis"])
    pen = CsrMatrix(c["d"], c["d"], *_csr(c["pen"]))
    terms = []
    for k in kinds:
        w = W[k]
        if k == 0:
            terms.append(CostTerm(CostKind.STATE_INFIDELITY, w, target_state=c["tgt"]))
        elif k == 1:
            terms.append(CostTerm(CostKind.STATE_PENALTY, w, penalty_op=pen))
        elif k == 2:
            terms.append(CostTerm(CostKind.STATE_RUNNING_INFIDELITY, w, target_state=c["tgt"]))
        elif k == 3:
            terms.append(CostTerm(CostKind.GATE_INFIDELITY, w, target_images=c["img"]))
        else:
            terms.append(CostTerm(CostKind.GATE_RUNNING_INFIDELITY, w, target_images=c["img"]))
    return prob, terms


def _oracle(c, kinds, amps):
    if c["dense"]:
        mk = lambda m: O.Dense(np.asfortranarray(m))  # noqa: E731
    else:
        mk = lambda m: O.Csr(m.shape[0], *_csr(m))  # noqa: E731
    p = O.Problem(mk(c["hs"]), tuple(mk(h) for h in c["hc"]), initial_states=c["psi0"], basis=c["basis"])
    pen = O.Csr(c["d"], *_csr(c["pen"]))
    kmap = [O.STATE_INFIDELITY, O.STATE_PENALTY, O.STATE_RUNNING_INFIDELITY, O.GATE_INFIDELITY,
            O.GATE_RUNNING_INFIDELITY]
    terms = []
    for k in kinds:
        if k == 1:
            terms.append(O.Term(kmap[k], W[k], None, pen))
        else:
            terms.append(O.Term(kmap[k], W[k], c["img"] if k >= 3 else c["tgt"]))
    return O.composite_grad(p, amps, c["dt"], terms), O.composite_cost(p, amps, c["dt"], terms)


ENGINES = ["ws", "wsdense", "cl", "cta", "dense"]


@pytest.fixture(autouse=True)
def _force_engine(request, monkeypatch):
    """The 'cta' cases force the single-CTA engine (small dense problems default to the ws engine)."""
    if "engine" in request.fixturenames and request.getfixturevalue("engine") == "cta":
        monkeypatch.setenv("LG_ENGINE", "cta")


@pytest.mark.parametrize("engine", ENGINES)
def test_all_kinds_three_channels(engine):
    c = _case(engine)
    kinds = [0, 1, 2, 3, 4]
    prob, terms = _product(c, kinds)
    a = ControlField(*c["amps"].shape, c["dt"], c["amps"])
    res = composite_grad(prob, a, terms)
    (co, go), cc = _oracle(c, kinds, c["amps"])
    assert abs(res.cost - co) <= 1e-12
    assert G.grad_rel(res.grad, go) <= 1e-9
    assert abs(composite_cost(prob, a, terms) - cc) <= 1e-12
    npb = NativeProblem(prob, terms, prob.initial_state, prob.basis)
    name = npb._lib.lg_engine_name(npb.handle).decode()
    assert name.startswith({"ws": "ws", "wsdense": "ws", "cl": "cluster", "cta": "cta", "dense": "dense"}[engine]), name


@pytest.mark.parametrize("engine", ENGINES)
def test_single_step(engine):
    c = _case(engine, seed=11, n_steps=1)
    kinds = [0, 3, 4]
    prob, terms = _product(c, kinds)
    a = ControlField(1, c["amps"].shape[1], c["dt"], c["amps"])
    res = composite_grad(prob, a, terms)
    (co, go), _ = _oracle(c, kinds, c["amps"])
    assert res.grad.shape == (1, c["amps"].shape[1])
    assert abs(res.cost - co) <= 1e-12
    assert G.grad_rel(res.grad, go) <= 1e-9


@pytest.mark.parametrize("engine", ENGINES)
def test_exact_zero_amplitudes(engine):
    """Zero controls drop their entries from H_n: plans and sparsity change from step to step."""
    c = _case(engine, seed=13, n_steps=8)
    amps = c["amps"].copy()
    amps[1] = 0.0
    amps[3, 0] = 0.0
    amps[5, 1:] = 0.0
    kinds = [0, 1, 3]
    prob, terms = _product(c, kinds)
    a = ControlField(*amps.shape, c["dt"], amps)
    res = composite_grad(prob, a, terms)
    (co, go), _ = _oracle(c, kinds, amps)
    assert abs(res.cost - co) <= 1e-12
    assert G.grad_rel(res.grad, go) <= 1e-9


def test_planning_error_and_bad_inputs():
    c = _case("ws", seed=17, n_steps=4)
    prob, terms = _product(c, [0])
    tight = ControlProblem(prob.h_static, prob.h_controls, tau=1e-300, initial_state=c["psi0"], basis=c["basis"])
    a = ControlField(*c["amps"].shape, c["dt"], c["amps"])
    with pytest.raises(PlanningError):
        NativeProblem(tight, terms, initial_states=c["psi0"]).grad(a)
    bad = c["amps"].copy()
    bad[2, 1] = np.nan
    with pytest.raises(ValueError):
        composite_grad(prob, ControlField(*bad.shape, c["dt"], bad), terms)
    with pytest.raises(ValueError):
        composite_grad(prob, ControlField(4, 2, c["dt"], c["amps"][:, :2]), terms)


def test_interleaved_problems_sharing_kernels():
    """Problems that share a kernel with different shared-memory sizes (and engines), evaluated
    alternately: each launch must carry its own dynamic shared-memory limit."""
    import _golden as G2
    from paper_2304_06200_b200 import models

    z3 = G2.load("c3")
    hs, hc = G2.mats(z3)
    p3 = ControlProblem(hs, tuple(hc), initial_state=z3["psi0"])
    a3 = ControlField(z3["amps"].shape[0], 2, float(z3["dt"]), z3["amps"])
    t3 = [CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=z3["targets"])]
    zs = G2.sub(G2.load("stress"), "s_block160")
    hs2, hc2 = G2.mats(zs)
    N, Kc = zs["amps"].shape
    a2 = ControlField(N, Kc, float(zs["dt"]), zs["amps"])
    p2 = ControlProblem(hs2, tuple(hc2), initial_state=zs["psi0"])
    t2 = [CostTerm(CostKind.STATE_INFIDELITY, 0.7, target_state=zs["targets"]),
          CostTerm(CostKind.STATE_PENALTY, 0.2, penalty_op=G2.penalty(zs)),
          CostTerm(CostKind.STATE_RUNNING_INFIDELITY, 0.4, target_state=zs["targets"])]
    c2 = models.build_case("c2", n_steps=50)
    n3 = NativeProblem(p3, t3, initial_states=z3["psi0"])
    n2 = NativeProblem(p2, t2, initial_states=zs["psi0"])
    r_c2 = composite_grad(c2.problem, c2.field, c2.terms)
    for _ in range(2):
        r = n3.grad(a3)
        assert abs(r.cost - float(z3["cost"])) <= 1e-12 and G2.grad_rel(r.grad, z3["grad"]) <= 1e-9
        r = n2.grad(a2)
        assert abs(r.cost - float(zs["cost_state"])) <= 1e-12 and G2.grad_rel(r.grad, zs["grad_state"]) <= 1e-9
        r = composite_grad(c2.problem, c2.field, c2.terms)
        assert r.cost == r_c2.cost and np.array_equal(r.grad, r_c2.grad)
