"""Synthetic benchmark problems: the five BASELINE.json configurations.

Host-side input construction only (restates the reference's builders,
src/models.py:49-86,149-175, with the parameter choices of SURVEY.md §8d).
Parameters are in GHz and converted x 2 pi to rad/ns; basis index
n_t * d_c + n_c (transmon (x) cavity).  Controls are seeded
``default_rng(seed).uniform(-A, A, (N, K_c))`` (src/cli.py:367).  The matrices
are bit-identical to the ones the reference's own builders produce
(tests/test_models.py checks them against tests/golden).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .costs import ControlField, ControlProblem, CostKind, CostTerm
from .sparse import DenseMatrix, build_csr_arrays, identity_csr, kron_csr, linear_combine

TWO_PI = 2.0 * math.pi

__all__ = ["Case", "build_case", "CONFIGS", "transmon_cavity_ops", "two_transmon_cavity_ops"]


def _lowering(dim):
    n = np.arange(1, dim, dtype=np.int64)
    return build_csr_arrays(n - 1, n, np.sqrt(n).astype(np.complex128), dim, dim)


def _raising(dim):
    n = np.arange(1, dim, dtype=np.int64)
    return build_csr_arrays(n, n - 1, np.sqrt(n).astype(np.complex128), dim, dim)


def _number(dim):
    n = np.arange(dim, dtype=np.int64)
    return build_csr_arrays(n, n, n.astype(np.complex128), dim, dim)


def _anharmonic(dim):
    n = np.arange(dim, dtype=np.int64)
    return build_csr_arrays(n, n, (n * (n - 1)).astype(np.complex128), dim, dim)


def transmon_cavity_ops(d_t, d_c, delta=0.1, alpha=-0.225, g=0.05):
    """H_s = D b'b + a/2 b'b(b'b-1) + g(c b' + c' b); controls (b+b') (x) I, i(b'-b) (x) I."""
    b, bd = _lowering(d_t), _raising(d_t)
    ic = identity_csr(d_c)
    c, cd = _lowering(d_c), _raising(d_c)
    nt = kron_csr(_number(d_t), ic)
    anh = kron_csr(_anharmonic(d_t), ic)
    exchange = linear_combine([1.0, 1.0], [kron_csr(bd, c), kron_csr(b, cd)])
    h_s = linear_combine([TWO_PI * delta, 0.5 * (TWO_PI * alpha), TWO_PI * g], [nt, anh, exchange])
    hx = kron_csr(linear_combine([1.0, 1.0], [b, bd]), ic)
    hy = kron_csr(linear_combine([1j, -1j], [bd, b]), ic)
    return h_s, hx, hy


def two_transmon_cavity_ops(d_t=5, d_c=400, d1=0.1, d2=0.15, alpha=-0.225, g=0.05):
    """sum_j [D_j n_j + a/2 n_j(n_j-1) + g(c b_j' + c' b_j)], controls x/y per transmon.
    Basis index (t1 d_t + t2) d_c + n."""
    it, ic = identity_csr(d_t), identity_csr(d_c)
    b, bd = _lowering(d_t), _raising(d_t)
    c, cd = _lowering(d_c), _raising(d_c)

    def k3(x, y, z):
        return kron_csr(kron_csr(x, y), z)

    n1, n2 = k3(_number(d_t), it, ic), k3(it, _number(d_t), ic)
    a1, a2 = k3(_anharmonic(d_t), it, ic), k3(it, _anharmonic(d_t), ic)
    ex1 = linear_combine([1.0, 1.0], [k3(bd, it, c), k3(b, it, cd)])
    ex2 = linear_combine([1.0, 1.0], [k3(it, bd, c), k3(it, b, cd)])
    h_s = linear_combine(
        [TWO_PI * d1, TWO_PI * d2, 0.5 * TWO_PI * alpha, 0.5 * TWO_PI * alpha, TWO_PI * g, TWO_PI * g],
        [n1, n2, a1, a2, ex1, ex2])
    x = linear_combine([1.0, 1.0], [b, bd])
    y = linear_combine([1j, -1j], [bd, b])
    return h_s, [k3(x, it, ic), k3(y, it, ic), k3(it, x, ic), k3(it, y, ic)]


def gue(rng, d, norm, scale=None):
    """(G + G^dagger)/2 of a complex Gaussian G, scaled to spectral norm ``norm``
    (the scale may be supplied to skip the O(d^3) eigvalsh)."""
    g = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
    h = (g + g.conj().T) / 2
    if scale is None:
        scale = norm / float(np.max(np.abs(np.linalg.eigvalsh(h))))
    return h, scale


def rand_states(rng, k, d):
    z = rng.standard_normal((k, d)) + 1j * rng.standard_normal((k, d))
    return z / np.linalg.norm(z, axis=1, keepdims=True)


def controls(seed, n, kc, amp):
    return np.random.default_rng(seed).uniform(-amp, amp, (n, kc))


def fock(d, n):
    v = np.zeros(d, np.complex128)
    v[n] = 1.0
    return v


@dataclass
class Case:
    name: str
    problem: ControlProblem
    field: ControlField
    terms: list
    n_states: int
    description: str


# scale factors of config 5 (computed once with eigvalsh by tests/golden/make_golden.py; stored
# so the GPU box does not need an O(d^3) eigensolve)
C5_SCALES = (0.007819919487427133, 0.0007828317290088312)


def build_case(name: str, n_steps: int | None = None, n_states: int | None = None) -> Case:
    """Build config ``c1`` .. ``c5`` (optionally truncated to the first n_steps / n_states)."""
    if name == "c1":
        h_s, hx, _ = transmon_cavity_ops(4, 10)
        h_s, hx = DenseMatrix(h_s.to_dense()), DenseMatrix(hx.to_dense())
        N, dt = 1000, 0.5
        amps = controls(101, N, 1, 0.01)
        psi0, phi = fock(40, 0)[None], fock(40, 1)[None]
        n_states = 1
        problem = ControlProblem(h_s, (hx,), initial_state=psi0)
        terms = [CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=phi)]
        desc = "dense transmon 4 x cavity 10 (d=40), 1 control, C1 state transfer |g,0>->|g,1>"
    elif name == "c2":
        h_s, hx, hy = transmon_cavity_ops(3, 20)
        d = 60
        N, dt = 2000, 0.25
        amps = controls(102, N, 2, 0.01)
        basis = np.array([fock(d, 0), fock(d, 20)])
        images = np.array([fock(d, 20), fock(d, 0)])
        proj = build_csr_arrays(np.arange(40, 60), np.arange(40, 60), np.ones(20, np.complex128), d, d)
        n_states = 2
        problem = ControlProblem(h_s, (hx, hy), initial_state=basis, basis=basis)
        terms = [CostTerm(CostKind.GATE_INFIDELITY, 1.0, target_images=images),
                 CostTerm(CostKind.STATE_PENALTY, 0.1, penalty_op=proj)]
        desc = "CSR transmon 3 x cavity 20 (d=60), 2 controls, K=2 X-gate + 0.1 x forbidden-level penalty"
    elif name == "c3":
        h_s, hx, hy = transmon_cavity_ops(6, 200)
        d = 1200
        N, dt = 2000, 0.5
        amps = controls(103, N, 2, 0.01)
        K = 8 if n_states is None else n_states
        psi0 = np.array([fock(d, n) for n in range(K)])
        phis = np.array([fock(d, n + 1) for n in range(K)])
        n_states = K
        problem = ControlProblem(h_s, (hx, hy), initial_state=psi0)
        terms = [CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=phis)]
        desc = "CSR transmon 6 x cavity 200 (d=1200), 2 controls, K=8 Fock transfers"
    elif name == "c4":
        h_s, ctrls = two_transmon_cavity_ops()
        d = 10000
        N, dt = 4000, 0.25
        amps = controls(104, N, 4, 0.01)

        def idx(t1, t2, n):
            return (t1 * 5 + t2) * 400 + n

        bi = [idx(t1, t2, n) for t1 in (0, 1) for t2 in (0, 1) for n in range(8)]
        ii = [idx(1 - t1, t2, n) for t1 in (0, 1) for t2 in (0, 1) for n in range(8)]
        K = 32 if n_states is None else n_states
        basis = np.zeros((K, d), np.complex128)
        images = np.zeros((K, d), np.complex128)
        basis[np.arange(K), bi[:K]] = 1.0
        images[np.arange(K), ii[:K]] = 1.0
        n_states = K
        problem = ControlProblem(h_s, tuple(ctrls), basis=basis)
        terms = [CostTerm(CostKind.GATE_INFIDELITY, 1.0, target_images=images)]
        desc = "CSR 2 transmons (5) x cavity 400 (d=10000), 4 controls, K=32 X(t1) gate subspace"
    elif name == "c5":
        d = 4096
        rng = np.random.default_rng(5005)
        hs_arr, s1 = gue(rng, d, 1.0, C5_SCALES[0])
        hc_arr, s2 = gue(rng, d, 0.1, C5_SCALES[1])
        K = 64 if n_states is None else n_states
        psi0 = rand_states(rng, 64, d)[:K]
        phis = rand_states(rng, 64, d)[:K]
        N, dt = 1000, 0.1
        amps = controls(105, N, 1, 1.0)
        n_states = K
        problem = ControlProblem(DenseMatrix(hs_arr * s1), (DenseMatrix(hc_arr * s2),), initial_state=psi0)
        terms = [CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=phis)]
        desc = "dense GUE d=4096 (|H_s|=1, |h_c|=0.1), 1 control, K=64 random transfers"
    else:
        raise KeyError(name)
    if n_steps is not None:
        N = n_steps
        amps = amps[:N]
    field = ControlField(N, amps.shape[1], dt, amps)
    return Case(name, problem, field, terms, n_states, desc)


CONFIGS = ("c1", "c2", "c3", "c4", "c5")
