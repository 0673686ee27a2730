"""CPU oracle for the HG cost+gradient evaluation -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``leangrape``
(``/root/reference/pkg/src/leangrape``; paths below are relative to that
package).  It exists so that ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` leg of ``bench.py`` can check / time the product path; the
product (``paper_2304_06200_b200``) never imports it.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by the reference itself (``tests/golden/make_golden.py``
imports ``/root/reference`` in the build container and writes
``tests/golden/*.npz``), and against the reference's own frozen constants
(``tests/test_expm_bounds.py:16-49,61-65,104-113,132-136``).

Everything is IEEE binary64.  Quantities that feed the (m, s) planner -- the
generator one-norm, sigma' and the auxiliary-matrix norms -- are computed with
exactly the numpy operations the reference uses, so they are bit-identical;
matvec and reduction orders are free (they only need to meet the 1e-12 / 1e-9
parity tolerances).

Block extension (documented in DESIGN.md): the reference carries one
``initial_state`` and a full ``d``-state gate basis.  The oracle accepts a
K-state block: state costs are averaged over the K transfers, gate costs
use a K-state subspace basis with 1/K normalisation (identical to the
reference's ``d``-state formulas when K == d).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

# ----------------------------------------------------------------------------
# operators  (restates src/sparse.py)


@dataclass(frozen=True, eq=False)
class Csr:
    """CSR complex matrix; invariants of src/sparse.py:42-60 (no stored zeros)."""

    n: int
    indptr: np.ndarray
    indices: np.ndarray
    data: np.ndarray

    kind = "csr"

    @property
    def nnz(self):
        return int(self.data.size)


@dataclass(frozen=True, eq=False)
class Dense:
    """Dense complex matrix, column-major (src/sparse.py:152-231)."""

    arr: np.ndarray

    kind = "dense"

    @property
    def n(self):
        return self.arr.shape[0]


def csr_from_coo(rows, cols, vals, n):
    """Sum duplicates, drop exact zeros (src/sparse.py:237-270)."""
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    vals = np.asarray(vals, np.complex128)
    key = rows * np.int64(n) + cols
    uniq, inv = np.unique(key, return_inverse=True)
    acc = np.zeros(uniq.size, np.complex128)
    np.add.at(acc, inv, vals)  # accumulation in input order
    keep = acc != 0
    uniq, acc = uniq[keep], acc[keep]
    r = uniq // n
    indptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=indptr[1:])
    return Csr(n, indptr, (uniq % n).astype(np.int64), acc)


def csr_from_any(m):
    """Accept this oracle's Csr, or any object exposing the reference's CSR fields."""
    if isinstance(m, (Csr, Dense)):
        return m
    if hasattr(m, "row_offsets"):
        return Csr(int(m.n_rows), np.asarray(m.row_offsets, np.int64),
                   np.asarray(m.col_indices, np.int64), np.asarray(m.values, np.complex128))
    if hasattr(m, "array"):
        return Dense(np.asfortranarray(np.asarray(m.array, np.complex128)))
    arr = np.asarray(m)
    return Dense(np.asfortranarray(arr.astype(np.complex128)))


def triplets(m: Csr):
    return np.repeat(np.arange(m.n), np.diff(m.indptr)), m.indices, m.data


def to_dense(m):
    if m.kind == "dense":
        return m.arr
    out = np.zeros((m.n, m.n), np.complex128, order="F")
    r, c, v = triplets(m)
    out[r, c] = v
    return out


def combine(coeffs, mats):
    """sum_i coeffs[i] * mats[i] (src/sparse.py:313-349): products rounded
    separately, accumulated in operand order, zero coefficients skipped."""
    coeffs = [complex(c) for c in coeffs]
    if any(m.kind == "dense" for m in mats):
        n = mats[0].n
        total = np.zeros((n, n), np.complex128, order="F")
        for c, m in zip(coeffs, mats):
            if c == 0:
                continue
            total += to_dense(m) * c
        return Dense(total)
    rs, cs, vs = [], [], []
    for c, m in zip(coeffs, mats):
        if c == 0 or m.nnz == 0:
            continue
        r, k, v = triplets(m)
        rs.append(r)
        cs.append(k)
        vs.append(c * v)
    n = mats[0].n
    if not rs:
        return Csr(n, np.zeros(n + 1, np.int64), np.zeros(0, np.int64), np.zeros(0, np.complex128))
    return csr_from_coo(np.concatenate(rs), np.concatenate(cs), np.concatenate(vs), n)


def scale(m, factor):
    """factor * m, pattern kept (src/sparse.py:123-133, 226-227)."""
    if m.kind == "dense":
        return Dense(m.arr * complex(factor))
    return Csr(m.n, m.indptr, m.indices, m.data * complex(factor))


def matvec(m, v):
    """src/sparse.py:69-88 (CSR reduceat) and :193-199 (dense matmul)."""
    if m.kind == "dense":
        return m.arr @ v
    out = np.zeros(m.n, np.complex128)
    if m.nnz == 0:
        return out
    prod = m.data * v[m.indices]
    starts = m.indptr[:-1]
    np.add.reduceat(prod, np.minimum(starts, prod.size - 1), out=out)
    out[starts == m.indptr[1:]] = 0.0
    return out


def col_abs_sums(m):
    if m.kind == "dense":
        return np.abs(m.arr).sum(axis=0)  # pairwise per contiguous column
    return np.bincount(m.indices, weights=np.abs(m.data), minlength=m.n)  # sequential, CSR order


def row_abs_sums(m):
    if m.kind == "dense":
        return np.abs(m.arr).sum(axis=1)  # sequential across columns
    out = np.zeros(m.n)
    if m.nnz:
        out = np.add.reduceat(np.abs(m.data), np.minimum(m.indptr[:-1], m.nnz - 1))  # a0 + pairwise(rest)
        out[m.indptr[:-1] == m.indptr[1:]] = 0.0
    return out


def row_nnz(m):
    if m.kind == "dense":
        return np.full(m.n, m.n, np.int64)
    return np.diff(m.indptr)


def one_norm(m):
    if (m.kind == "dense" and m.arr.size == 0) or (m.kind == "csr" and m.nnz == 0):
        return 0.0
    return float(col_abs_sums(m).max())


def inf_norm(m):
    if (m.kind == "dense" and m.arr.size == 0) or (m.kind == "csr" and m.nnz == 0):
        return 0.0
    return float(row_abs_sums(m).max())


def sigma_prime(m):
    """max_row_nnz (src/sparse.py:117-121); dense reports n_cols (:220-222)."""
    if m.kind == "dense":
        return m.n
    return int(row_nnz(m).max()) if m.n else 0


def embed_aux(h_step, h_ctrl, dt):
    """Materialised [[A, A_c], [0, A]] (src/sparse.py:352-380)."""
    d = h_step.n
    sc = -1j * dt
    if h_step.kind == "dense" or h_ctrl.kind == "dense":
        e = np.zeros((2 * d, 2 * d), np.complex128, order="F")
        e[:d, :d] = sc * to_dense(h_step)
        e[:d, d:] = sc * to_dense(h_ctrl)
        e[d:, d:] = e[:d, :d]
        return Dense(e)
    hr, hc, hv = triplets(h_step)
    cr, cc, cv = triplets(h_ctrl)
    rows = np.concatenate([hr, cr, hr + d])
    cols = np.concatenate([hc, cc + d, hc + d])
    return csr_from_coo(rows, cols, sc * np.concatenate([hv, cv, hv]), 2 * d)


class BlockAux:
    """Matrix-free [[A, A_c], [0, A]] (src/derivatives.py:133-184)."""

    kind = "block"

    def __init__(self, gen, h_ctrl, dt):
        self.gen = gen
        self.ctrl = scale(h_ctrl, -1j * dt)
        self.n = 2 * gen.n

    def matvec(self, v):
        d = self.gen.n
        top = matvec(self.gen, v[:d])
        top += matvec(self.ctrl, v[d:])
        return np.concatenate([top, matvec(self.gen, v[d:])])

    def one_norm(self):
        g, c = col_abs_sums(self.gen), col_abs_sums(self.ctrl)
        return float(max(g.max(), (g + c).max())) if g.size else 0.0

    def inf_norm(self):
        g, c = row_abs_sums(self.gen), row_abs_sums(self.ctrl)
        return float(max((g + c).max(), g.max())) if g.size else 0.0

    def sigma_prime(self):
        return int((row_nnz(self.gen) + row_nnz(self.ctrl)).max()) + 1


AUX_MATERIALISE_DIM = 256  # 2d at or below which aux is materialised (src/derivatives.py:29)

# ----------------------------------------------------------------------------
# certified planner  (restates src/expm.py:69-303)

M_MAX, S_MAX = 60, 10_000
U = 2.0 ** -53
U_PRIME = 2.0 * math.sqrt(2.0) * U / (1.0 - 2.0 * U)


class PlanningError(RuntimeError):
    pass


class _Infeasible(ArithmeticError):
    pass


def remainder_rm(x, m):
    """sum_{q>m} x^q/q!, ascending, geometric tail after 500 terms (src/expm.py:110-143)."""
    if x < 0:
        raise ValueError("negative argument")
    if x == 0.0:
        return 0.0
    t = 1.0
    for q in range(1, m + 2):
        t *= x / q
        if math.isinf(t):
            return math.inf
    acc, q = t, m + 1
    for _ in range(500):
        q += 1
        t *= x / q
        acc += t
        if t < 1e-20 * acc:
            return acc
    ratio = x / (q + 1)
    if ratio >= 1.0:
        return math.inf
    return acc + t * ratio / (1.0 - ratio)


def gamma_n(n):
    """n u' / (1 - n u') (src/expm.py:146-153)."""
    nu = n * U_PRIME
    if nu >= 1.0:
        raise _Infeasible
    return nu / (1.0 - nu)


def beta_sum(xb, m, sp):
    """sum_k gamma_{k(sp+2)+m+2} xb^k/k! (src/expm.py:156-169)."""
    b, p = 0.0, 1.0
    for k in range(m + 1):
        if k:
            p *= xb / k
        b += gamma_n(k * (sp + 2) + m + 2) * p
    return b


def rounding_bound(xb, m, s, sp):
    """alpha^s expm1(s log1p(beta/alpha)) (src/expm.py:172-196)."""
    rm = remainder_rm(xb, m)
    if math.isinf(rm):
        return math.inf
    alpha = 1.0 + rm
    try:
        b = beta_sum(xb, m, sp)
    except _Infeasible:
        return math.inf
    try:
        return alpha ** s * math.expm1(s * math.log1p(b / alpha))
    except OverflowError:
        return math.inf


def truncation_bound(xb, m, s):
    """x(1-x^s)/(1-x) with x = s R_m (src/expm.py:199-211)."""
    x = s * remainder_rm(xb, m)
    if math.isinf(x) or x >= 1.0:
        return math.inf
    if x == 0.0:
        return 0.0
    return x * (1.0 - x ** s) / (1.0 - x)


def error_bound(xa, m, s, sp):
    xb = xa / s
    t = truncation_bound(xb, m, s)
    if math.isinf(t):
        return math.inf
    return t + rounding_bound(xb, m, s, sp)


@lru_cache(maxsize=1 << 16)
def _plan(xa, sp, tau, m_max, s_max):
    g3 = gamma_n(3)
    for s in range(1, s_max + 1):
        if s * g3 > tau:
            raise PlanningError(f"tolerance {tau:g} is below the rounding floor for norm1={xa:g}")
        xb = xa / s
        if truncation_bound(xb, m_max, s) > tau:
            continue
        for m in range(1, m_max + 1):
            try:
                if s * beta_sum(xb, m, sp) > tau:
                    break
            except _Infeasible:
                break
            b = error_bound(xa, m, s, sp)
            if b <= tau:
                return (m, s, b)
    raise PlanningError(f"no feasible (order, scaling) pair for norm1={xa:g}, sigma_prime={sp}, tau={tau:g}")


def make_plan(norm1, sp, tau, m_max=M_MAX, s_max=S_MAX):
    """(order, scaling, bound): smallest scaling, then smallest order (src/expm.py:229-303)."""
    if not norm1 >= 0.0:
        raise ValueError(f"norm1_a must be non-negative, got {norm1}")
    if sp < 0 or not tau > 0.0:
        raise ValueError("bad sigma_prime / tau")
    return _plan(float(norm1), int(sp), float(tau), int(m_max), int(s_max))


def taylor_apply(mv, psi, m, s):
    """((T_m(A/s))^s psi) with term <- (A term) * (1/(s j)) (src/expm.py:306-351)."""
    cur = np.array(psi, np.complex128, copy=True)
    for _ in range(s):
        term = cur.copy()
        for j in range(1, m + 1):
            term = mv(term) * (1.0 / (s * j))
            cur += term
    return cur


# ----------------------------------------------------------------------------
# one time step  (restates src/derivatives.py:105-110,187-202,278-331 and
# ControlProblem.step_evaluator, src/costs.py:131-138)


class Step:
    def __init__(self, h_static, h_controls, amps_n, dt, tau):
        self.h_controls = h_controls
        self.dt = dt
        self.tau = tau
        self.h = combine([1.0] + [complex(x) for x in amps_n], [h_static, *h_controls])
        self.gen = scale(self.h, -1j * dt)
        self.norm1 = one_norm(self.gen)
        self.sp = sigma_prime(self.gen)
        self.m, self.s, _ = make_plan(self.norm1, self.sp, tau)
        self.neg = scale(self.gen, -1.0)
        self._aux = {}

    def aux(self, k):
        if k not in self._aux:
            d = self.h.n
            if 2 * d <= AUX_MATERIALISE_DIM:
                op = embed_aux(self.h, self.h_controls[k], self.dt)
                one, inf, sp = one_norm(op), inf_norm(op), sigma_prime(op)
                mv = lambda v, op=op: matvec(op, v)
            else:
                op = BlockAux(self.gen, self.h_controls[k], self.dt)
                one, inf, sp = op.one_norm(), op.inf_norm(), op.sigma_prime()
                mv = op.matvec
            arg = math.sqrt(one * inf)
            m, s, _ = make_plan(arg, sp, self.tau)
            self._aux[k] = (mv, m, s, arg, sp)
        return self._aux[k]

    def forward(self, psi):
        return taylor_apply(lambda v: matvec(self.gen, v), psi, self.m, self.s)

    def adjoint(self, psi):
        return taylor_apply(lambda v: matvec(self.neg, v), psi, self.m, self.s)

    def dU(self, k, psi):
        mv, m, s, _, _ = self.aux(k)
        d = psi.size
        stacked = np.zeros(2 * d, np.complex128)
        stacked[d:] = psi
        return taylor_apply(mv, stacked, m, s)[:d]


DEGENERACY_RTOL = 1e-12  # src/derivatives.py:45


class DiagStep:
    """DIAGONALIZATION backend step (src/derivatives.py:228-275): eigenfactorisation of the
    dense step matrix H_n dt, exact propagators and the divided-difference derivative."""

    def __init__(self, h_static, h_controls, amps_n, dt, tau):
        self.h_controls = h_controls
        self.dt = dt
        h = combine([1.0] + [complex(x) for x in amps_n], [h_static, *h_controls])
        w, self.vecs = np.linalg.eigh(to_dense(h) * dt)  # src/derivatives.py:230-231
        self.eig = -1j * w.astype(np.complex128)
        self.exp = np.exp(self.eig)
        gaps = self.eig[None, :] - self.eig[:, None]
        scale_ = float(np.abs(w).max()) if w.size else 0.0
        degenerate = np.abs(gaps) <= DEGENERACY_RTOL * max(scale_, 1e-300)
        inv = np.zeros_like(gaps)
        np.divide(1.0, gaps, out=inv, where=~degenerate)
        self.hadamard = (self.exp[None, :] - self.exp[:, None]) * inv + np.diag(self.exp)

    def _prop(self, psi, adjoint):
        c = self.vecs.conj().T @ psi
        return self.vecs @ ((np.conj(self.exp) if adjoint else self.exp) * c)

    def forward(self, psi):
        return self._prop(psi, False)

    def adjoint(self, psi):
        return self._prop(psi, True)

    def dU(self, k, psi):  # src/derivatives.py:249-275
        da = to_dense(self.h_controls[k]) * (-1j * self.dt)
        s = self.vecs
        inner = s.conj().T @ da @ s
        return s @ ((self.hadamard * inner) @ (s.conj().T @ psi))


def plan_table(h_static, h_controls, amps, dt, tau):
    """Per-step planner inputs and plans: returns dict of arrays
    norm1[N], sp[N], m[N], s[N], aux_arg[N,Kc], aux_sp[N,Kc], aux_m, aux_s."""
    N, Kc = amps.shape
    out = {k: [] for k in ("norm1", "sp", "m", "s", "aux_arg", "aux_sp", "aux_m", "aux_s")}
    for n in range(N):
        st = Step(h_static, h_controls, amps[n], dt, tau)
        out["norm1"].append(st.norm1)
        out["sp"].append(st.sp)
        out["m"].append(st.m)
        out["s"].append(st.s)
        row = [st.aux(k) for k in range(Kc)]
        out["aux_arg"].append([r[3] for r in row])
        out["aux_sp"].append([r[4] for r in row])
        out["aux_m"].append([r[1] for r in row])
        out["aux_s"].append([r[2] for r in row])
    return {k: np.asarray(v) for k, v in out.items()}


# ----------------------------------------------------------------------------
# costs and forward-backward gradients  (restates src/costs.py)

STATE_INFIDELITY = "state_infidelity"
STATE_PENALTY = "state_penalty"
STATE_RUNNING_INFIDELITY = "state_running_infidelity"
GATE_INFIDELITY = "gate_infidelity"
GATE_RUNNING_INFIDELITY = "gate_running_infidelity"
STATE_KINDS = (STATE_INFIDELITY, STATE_PENALTY, STATE_RUNNING_INFIDELITY)


@dataclass
class Term:
    """One weighted cost term.  ``targets``: (K, d) target states (state
    infidelities) or target images U_T psi_0^h (gate terms); ``penalty``: Csr/Dense."""

    kind: str
    weight: float = 1.0
    targets: np.ndarray | None = None
    penalty: object = None


@dataclass
class Problem:
    h_static: object
    h_controls: tuple
    tau: float = 1e-8
    initial_states: np.ndarray | None = None  # (K, d) state-transfer trajectories
    basis: np.ndarray | None = None  # (K, d) gate basis (computational basis if None)
    backend: str = "scaling_squaring"  # or "diagonalization" (src/derivatives.py:48-51)


class _Memo:
    """Capacity-one step cache (src/costs.py:227-247)."""

    def __init__(self, p, amps, dt):
        self.p, self.amps, self.dt = p, amps, dt
        self.n, self.st = -1, None

    def get(self, n):
        if n != self.n:
            cls = DiagStep if self.p.backend == "diagonalization" else Step
            self.st = cls(self.p.h_static, self.p.h_controls, self.amps[n], self.dt, self.p.tau)
            self.n = n
        return self.st


def _state_pass_one(p, amps, dt, psi0, specs):
    """Fused state-cost pass for one trajectory (src/costs.py:269-354).
    specs: list of (kind, weight, target (d,) | None, penalty | None)."""
    N, Kc = amps.shape
    memo = _Memo(p, amps, dt)
    pen, ovs = {}, {}
    psi = np.array(psi0, np.complex128)
    for n in range(N):
        psi = memo.get(n).forward(psi)
        for i, (kind, w, tgt, om) in enumerate(specs):
            if kind == STATE_PENALTY:
                pen[i] = pen.get(i, 0.0) + np.vdot(psi, matvec(om, psi)).real
            elif kind == STATE_RUNNING_INFIDELITY:
                ovs[i] = ovs.get(i, 0.0) + abs(np.vdot(tgt, psi)) ** 2
    cost, z = 0.0, {}
    for i, (kind, w, tgt, om) in enumerate(specs):
        if kind == STATE_INFIDELITY:
            z[i] = np.vdot(psi, tgt)
            cost += w * (1.0 - abs(z[i]) ** 2)
        elif kind == STATE_PENALTY:
            cost += w * pen[i] / N
        else:
            cost += w * (1.0 - ovs[i] / N)
    lam = {}
    for i, (kind, w, tgt, om) in enumerate(specs):
        if kind == STATE_INFIDELITY:
            lam[i] = np.array(tgt, np.complex128)
        elif kind == STATE_PENALTY:
            lam[i] = matvec(om, psi)
        else:
            lam[i] = tgt * np.vdot(tgt, psi)
    grad = np.zeros((N, Kc))
    for n in range(N - 1, -1, -1):
        st = memo.get(n)
        psi = st.adjoint(psi)
        for k in range(Kc):
            du = st.dU(k, psi)
            for i, (kind, w, tgt, om) in enumerate(specs):
                ip = np.vdot(lam[i], du)
                if kind == STATE_INFIDELITY:
                    c = -2.0 * (ip * z[i]).real
                elif kind == STATE_PENALTY:
                    c = 2.0 / N * ip.real
                else:
                    c = -2.0 / N * ip.real
                grad[n, k] += w * c
        if n > 0:
            for i, (kind, w, tgt, om) in enumerate(specs):
                moved = st.adjoint(lam[i])
                if kind == STATE_PENALTY:
                    moved += matvec(om, psi)
                elif kind == STATE_RUNNING_INFIDELITY:
                    moved += tgt * np.vdot(tgt, psi)
                lam[i] = moved
    return cost, grad


def _gate_pass(p, amps, dt, states, images, running):
    """Two-sweep gate pass over a K-state basis (src/costs.py:407-488) with
    1/K normalisation (== the reference's 1/d when K == d)."""
    N, Kc = amps.shape
    K = len(states)
    memo = _Memo(p, amps, dt)
    tr = np.zeros(N, np.complex128)
    for h in range(K):
        psi = np.array(states[h], np.complex128)
        for n in range(N):
            psi = memo.get(n).forward(psi)
            if running or n == N - 1:
                tr[n] += np.vdot(images[h], psi)
    if running:
        cost = 1.0 - float(np.sum(np.abs(tr) ** 2)) / (N * K * K)
    else:
        cost = 1.0 - abs(tr[-1]) ** 2 / (K * K)
    acc = np.zeros((N, Kc), np.complex128)
    for h in range(K):
        psi = np.array(states[h], np.complex128)
        for n in range(N):
            psi = memo.get(n).forward(psi)
        lam = images[h] * tr[N - 1] if running else np.array(images[h], np.complex128)
        for n in range(N - 1, -1, -1):
            st = memo.get(n)
            psi = st.adjoint(psi)
            for k in range(Kc):
                acc[n, k] += np.vdot(lam, st.dU(k, psi))
            if n > 0:
                moved = st.adjoint(lam)
                if running:
                    moved += images[h] * tr[n - 1]
                lam = moved
    if running:
        grad = -2.0 / (N * K * K) * acc.real
    else:
        grad = -2.0 / (K * K) * (acc * np.conj(tr[-1])).real
    return cost, grad


def _rows(x, d):
    x = np.asarray(x, np.complex128)
    return x.reshape(1, d) if x.ndim == 1 else x


def _basis(p):
    d = p.h_static.n
    if p.basis is None:
        return np.eye(d, dtype=np.complex128)
    return _rows(p.basis, d)


def composite_grad(p: Problem, amps, dt, terms):
    """Weighted cost and gradient (src/costs.py:515-546), K-block extension."""
    amps = np.asarray(amps, np.float64)
    N, Kc = amps.shape
    d = p.h_static.n
    cost, grad = 0.0, np.zeros((N, Kc))
    st_terms = [t for t in terms if t.kind in STATE_KINDS]
    if st_terms:
        psi0 = _rows(p.initial_states, d)
        K = psi0.shape[0]
        for h in range(K):
            specs = [(t.kind, t.weight, None if t.targets is None else _rows(t.targets, d)[h], t.penalty)
                     for t in st_terms]
            c, g = _state_pass_one(p, amps, dt, psi0[h], specs)
            cost += c / K
            grad += g / K
    for t in terms:
        if t.kind in STATE_KINDS:
            continue
        c, g = _gate_pass(p, amps, dt, _basis(p), _rows(t.targets, d),
                          t.kind == GATE_RUNNING_INFIDELITY)
        cost += t.weight * c
        grad += t.weight * g
    return cost, grad


def composite_cost(p: Problem, amps, dt, terms):
    """Forward-only weighted cost (src/costs.py:549-597), K-block extension."""
    amps = np.asarray(amps, np.float64)
    N, Kc = amps.shape
    d = p.h_static.n
    total = 0.0
    st_terms = [t for t in terms if t.kind in STATE_KINDS]
    if st_terms:
        psi0 = _rows(p.initial_states, d)
        K = psi0.shape[0]
        for h in range(K):
            memo = _Memo(p, amps, dt)
            psi = np.array(psi0[h])
            pen = [0.0] * len(st_terms)
            ovs = [0.0] * len(st_terms)
            for n in range(N):
                psi = memo.get(n).forward(psi)
                for i, t in enumerate(st_terms):
                    if t.kind == STATE_PENALTY:
                        pen[i] += np.vdot(psi, matvec(t.penalty, psi)).real
                    elif t.kind == STATE_RUNNING_INFIDELITY:
                        ovs[i] += abs(np.vdot(_rows(t.targets, d)[h], psi)) ** 2
            for i, t in enumerate(st_terms):
                if t.kind == STATE_INFIDELITY:
                    total += t.weight * (1.0 - abs(np.vdot(psi, _rows(t.targets, d)[h])) ** 2) / K
                elif t.kind == STATE_PENALTY:
                    total += t.weight * pen[i] / N / K
                else:
                    total += t.weight * (1.0 - ovs[i] / N) / K
    for t in terms:
        if t.kind in STATE_KINDS:
            continue
        running = t.kind == GATE_RUNNING_INFIDELITY
        states, images = _basis(p), _rows(t.targets, d)
        K = len(states)
        memo = _Memo(p, amps, dt)
        tr = np.zeros(N, np.complex128)
        for h in range(K):
            psi = np.array(states[h])
            for n in range(N):
                psi = memo.get(n).forward(psi)
                if running or n == N - 1:
                    tr[n] += np.vdot(images[h], psi)
        if running:
            total += t.weight * (1.0 - float(np.sum(np.abs(tr) ** 2)) / (N * K * K))
        else:
            total += t.weight * (1.0 - abs(tr[-1]) ** 2 / (K * K))
    return float(total)


def forward_propagate(p: Problem, amps, dt, psi0):
    """src/costs.py:209-217."""
    amps = np.asarray(amps, np.float64)
    memo = _Memo(p, amps, dt)
    psi = np.array(psi0, np.complex128)
    for n in range(amps.shape[0]):
        psi = memo.get(n).forward(psi)
    return psi
