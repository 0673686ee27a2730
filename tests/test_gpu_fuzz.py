"""GPU vs the CPU oracle on seeded random problems (every engine the library picks, every cost kind).

Random banded sparse and dense Hermitian problems, 1-3 controls, random trajectories, gate
subspaces and penalty operators, amplitudes large enough that the (m, s) plans vary from step
to step.  Bars as everywhere: cost 1e-12 absolute, gradient 1e-9 relative (norm-wise).
"""

import numpy as np
import pytest

import _golden as G
from oracle import lg_oracle as O
from paper_2304_06200_b200 import ControlField, ControlProblem, CostKind, CostTerm
from paper_2304_06200_b200.costs import NativeProblem
from paper_2304_06200_b200.sparse import CsrMatrix, DenseMatrix

pytestmark = pytest.mark.gpu


def _banded(rng, d, offsets, scale):
    """Hermitian CSR with the given (positive) off-diagonal offsets plus a diagonal."""
    rows, cols, vals = [], [], []
    for i in range(d):
        rows.append(i), cols.append(i), vals.append(complex(scale * rng.standard_normal(), 0.0))
        for o in offsets:
            if i + o < d:
                v = scale * (rng.standard_normal() + 1j * rng.standard_normal())
                rows += [i, i + o]
                cols += [i + o, i]
                vals += [v, np.conj(v)]
    a = np.zeros((d, d), np.complex128)
    a[rows, cols] = vals
    return a


def _csr(a):
    d = a.shape[0]
    ptr, idx, val = [0], [], []
    for i in range(d):
        nz = np.nonzero(a[i])[0]
        idx += list(nz)
        val += list(a[i, nz])
        ptr.append(len(idx))
    return CsrMatrix(d, d, np.array(ptr, np.int64), np.array(idx, np.int64), np.array(val, np.complex128))


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    dense = seed % 4 == 3
    d = int(rng.choice([6, 12, 24, 40])) if dense else int(rng.choice([8, 20, 48, 64, 90, 130]))
    kc = int(rng.integers(1, 4))
    offs = sorted({int(x) for x in rng.integers(1, max(2, d // 3), size=2)})
    hs = _banded(rng, d, offs, 1.0)
    hcs = [_banded(rng, d, [offs[0]], 0.3) for _ in range(kc)]
    mk = (lambda a: DenseMatrix(np.asfortranarray(a))) if dense else _csr
    N = int(rng.integers(3, 21))
    dt = float(rng.uniform(0.1, 0.5))
    amps = rng.uniform(-1.5, 1.5, (N, kc))
    K = int(rng.integers(1, 4))
    psi0 = G_states(rng, K, d)
    phi = G_states(rng, K, d)
    q, _ = np.linalg.qr(rng.standard_normal((d, K)) + 1j * rng.standard_normal((d, K)))
    basis = q.T.copy()
    u, _ = np.linalg.qr(rng.standard_normal((K, K)) + 1j * rng.standard_normal((K, K)))
    images = (u.T @ basis).copy()
    pen = _csr(np.diag((np.arange(d) % 3) / 3.0).astype(np.complex128))
    return dict(hs=mk(hs), hcs=[mk(h) for h in hcs], N=N, dt=dt, amps=amps, psi0=psi0, phi=phi, basis=basis,
                images=images, pen=pen, hs_a=hs, hcs_a=hcs, dense=dense)


def G_states(rng, k, d):
    z = rng.standard_normal((k, d)) + 1j * rng.standard_normal((k, d))
    return z / np.linalg.norm(z, axis=1, keepdims=True)


def _oracle_mat(m):
    if isinstance(m, DenseMatrix):
        return O.Dense(np.asfortranarray(m.array))
    return O.Csr(m.n_rows, m.row_offsets, m.col_indices, m.values)


@pytest.mark.parametrize("seed", range(40))
def test_random_problem_against_oracle(seed):
    c = _case(seed)
    a = ControlField(c["N"], len(c["hcs"]), c["dt"], c["amps"])
    prob = ControlProblem(c["hs"], tuple(c["hcs"]), initial_state=c["psi0"], basis=c["basis"])
    op = O.Problem(_oracle_mat(c["hs"]), tuple(_oracle_mat(h) for h in c["hcs"]), initial_states=c["psi0"],
                   basis=c["basis"])
    rng = np.random.default_rng(seed)
    w = rng.uniform(0.2, 1.0, 3)
    st = [CostTerm(CostKind.STATE_INFIDELITY, w[0], target_state=c["phi"]),
          CostTerm(CostKind.STATE_PENALTY, w[1], penalty_op=c["pen"]),
          CostTerm(CostKind.STATE_RUNNING_INFIDELITY, w[2], target_state=c["phi"])]
    ost = [O.Term(O.STATE_INFIDELITY, w[0], c["phi"]), O.Term(O.STATE_PENALTY, w[1], None, _oracle_mat(c["pen"])),
           O.Term(O.STATE_RUNNING_INFIDELITY, w[2], c["phi"])]
    npb = NativeProblem(prob, st, initial_states=c["psi0"])
    res = npb.grad(a)
    cost, grad = O.composite_grad(op, c["amps"], c["dt"], ost)
    assert abs(res.cost - cost) <= 1e-12, (npb.engine, res.cost, cost)
    assert G.grad_rel(res.grad, grad) <= 1e-9, (npb.engine, G.grad_rel(res.grad, grad))
    assert abs(npb.cost(a) - cost) <= 1e-12
    for kind, ok in [(CostKind.GATE_INFIDELITY, O.GATE_INFIDELITY),
                     (CostKind.GATE_RUNNING_INFIDELITY, O.GATE_RUNNING_INFIDELITY)]:
        gp = NativeProblem(prob, [CostTerm(kind, 1.0, target_images=c["images"])], basis=c["basis"])
        res = gp.grad(a)
        cost, grad = O.composite_grad(op, c["amps"], c["dt"], [O.Term(ok, 1.0, c["images"])])
        assert abs(res.cost - cost) <= 1e-12, (gp.engine, kind, res.cost, cost)
        assert G.grad_rel(res.grad, grad) <= 1e-9, (gp.engine, kind, G.grad_rel(res.grad, grad))


@pytest.mark.parametrize("seed", range(12))
def test_random_problem_diagonalization_backend(seed):
    """The DIAGONALIZATION backend on the same random problems against the oracle's restatement."""
    from paper_2304_06200_b200 import Backend

    c = _case(seed)
    if c["hs"].n_rows > 128 if hasattr(c["hs"], "n_rows") else False:
        pytest.skip("the device DIAGONALIZATION backend covers d <= 128")
    a = ControlField(c["N"], len(c["hcs"]), c["dt"], c["amps"])
    prob = ControlProblem(c["hs"], tuple(c["hcs"]), backend=Backend.DIAGONALIZATION, initial_state=c["psi0"],
                          basis=c["basis"])
    op = O.Problem(_oracle_mat(c["hs"]), tuple(_oracle_mat(h) for h in c["hcs"]), initial_states=c["psi0"],
                   basis=c["basis"], backend="diagonalization")
    st = [CostTerm(CostKind.STATE_INFIDELITY, 0.6, target_state=c["phi"]),
          CostTerm(CostKind.STATE_PENALTY, 0.3, penalty_op=c["pen"]),
          CostTerm(CostKind.STATE_RUNNING_INFIDELITY, 0.5, target_state=c["phi"])]
    ost = [O.Term(O.STATE_INFIDELITY, 0.6, c["phi"]), O.Term(O.STATE_PENALTY, 0.3, None, _oracle_mat(c["pen"])),
           O.Term(O.STATE_RUNNING_INFIDELITY, 0.5, c["phi"])]
    res = NativeProblem(prob, st, initial_states=c["psi0"]).grad(a)
    cost, grad = O.composite_grad(op, c["amps"], c["dt"], ost)
    assert abs(res.cost - cost) <= 1e-12, (res.cost, cost)
    assert G.grad_rel(res.grad, grad) <= 1e-9, G.grad_rel(res.grad, grad)
    gp = NativeProblem(prob, [CostTerm(CostKind.GATE_RUNNING_INFIDELITY, 1.0, target_images=c["images"])],
                       basis=c["basis"])
    res = gp.grad(a)
    cost, grad = O.composite_grad(op, c["amps"], c["dt"], [O.Term(O.GATE_RUNNING_INFIDELITY, 1.0, c["images"])])
    assert abs(res.cost - cost) <= 1e-12, (res.cost, cost)
    assert G.grad_rel(res.grad, grad) <= 1e-9, G.grad_rel(res.grad, grad)
