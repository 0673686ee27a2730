"""Drop-in mirror of the reference's cost API (src/costs.py), evaluated on B200.

Same names, argument meaning and error behaviour as ``leangrape.costs``:
``ControlField``, ``ControlProblem``, ``CostKind``, ``CostTerm``,
``GradientResult``, ``composite_grad``, ``composite_cost``, ``c1/c2/c3_state_grad``,
``c1/c3_gate_grad``, ``forward_propagate``.  Every evaluation runs the
sm_100a kernels through the C ABI (include/leangrape_b200.h); there is no CPU
fallback.  Both backends run on the device: SCALING_SQUARING (the certified
Taylor action) and DIAGONALIZATION (per-step eigenfactorisation on the device, dense operators,
lg_diag.cu).

K-state block extension (documented in DESIGN.md):
  * ``ControlProblem.initial_state`` may be ``(K, d)``: state terms are then the
    mean over the K transfers (``CostTerm.target_state`` is ``(K, d)`` too);
  * ``ControlProblem.basis`` may hold K <= d orthonormal states: gate terms use
    that subspace with 1/K normalisation (identical to the reference at K == d);
  * ``CostTerm.target_images`` (``(K, d)``, the images U_T psi_h) may replace a
    dense ``target_gate``, which is infeasible at d = 10^4.
"""

from __future__ import annotations

import ctypes as C
from collections import OrderedDict
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _native
from .sparse import DenseMatrix, as_own_matrix, frozen_copy, is_hermitian, linear_combine, one_norm_host, to_dense

__all__ = [
    "Backend",
    "CostKind",
    "ControlField",
    "ControlProblem",
    "CostTerm",
    "GradientResult",
    "forward_propagate",
    "c1_state_grad",
    "c2_state_grad",
    "c3_state_grad",
    "c1_gate_grad",
    "c3_gate_grad",
    "composite_grad",
    "composite_cost",
]


class Backend(Enum):
    SCALING_SQUARING = "scaling_squaring"
    DIAGONALIZATION = "diagonalization"


class CostKind(Enum):
    STATE_INFIDELITY = "state_infidelity"
    STATE_PENALTY = "state_penalty"
    STATE_RUNNING_INFIDELITY = "state_running_infidelity"
    GATE_INFIDELITY = "gate_infidelity"
    GATE_RUNNING_INFIDELITY = "gate_running_infidelity"


_STATE_KINDS = (CostKind.STATE_INFIDELITY, CostKind.STATE_PENALTY, CostKind.STATE_RUNNING_INFIDELITY)
_KIND_CODE = {
    CostKind.STATE_INFIDELITY: 0,
    CostKind.STATE_PENALTY: 1,
    CostKind.STATE_RUNNING_INFIDELITY: 2,
    CostKind.GATE_INFIDELITY: 3,
    CostKind.GATE_RUNNING_INFIDELITY: 4,
}


@dataclass(frozen=True)
class ControlField:
    """Piecewise-constant amplitudes on n_steps x n_channels (src/costs.py:64-93)."""

    n_steps: int
    n_channels: int
    dt: float
    amplitudes: np.ndarray = field(repr=False)

    def __post_init__(self):
        amps = np.asarray(self.amplitudes, dtype=np.float64)
        if amps.shape != (self.n_steps, self.n_channels):
            raise ValueError(f"amplitudes shape {amps.shape} does not match ({self.n_steps}, {self.n_channels})")
        if self.n_steps < 1 or self.n_channels < 1:
            raise ValueError("need at least one step and one channel")
        if self.dt <= 0.0:
            raise ValueError("dt must be positive")
        if not np.isfinite(amps).all():
            raise ValueError("control amplitudes must be finite")
        object.__setattr__(self, "amplitudes", amps)

    @classmethod
    def constant(cls, value: float, n_steps: int, n_channels: int, dt: float) -> "ControlField":
        return cls(n_steps, n_channels, dt, np.full((n_steps, n_channels), value))

    def replace_amplitudes(self, amps) -> "ControlField":
        return ControlField(self.n_steps, self.n_channels, self.dt, amps)


def _shape(m):
    return (m.n_rows, m.n_cols)


@dataclass(frozen=True)
class ControlProblem:
    """Static Hamiltonian, controls and engine settings (src/costs.py:96-138)."""

    h_static: object
    h_controls: tuple
    backend: Backend = Backend.SCALING_SQUARING
    tau: float = 1e-8
    initial_state: np.ndarray | None = None
    basis: tuple | None = None

    def __post_init__(self):
        # immutable private copies (device problems are cached per object, _native_for)
        object.__setattr__(self, "h_static", as_own_matrix(self.h_static))
        object.__setattr__(self, "h_controls", tuple(as_own_matrix(h) for h in self.h_controls))
        if self.initial_state is not None:
            object.__setattr__(self, "initial_state", frozen_copy(self.initial_state, np.complex128))
        if self.basis is not None:
            object.__setattr__(self, "basis", frozen_copy(np.asarray(self.basis), np.complex128))
        tol = 1e-12 * max(1.0, one_norm_host(self.h_static))
        if not is_hermitian(self.h_static, tol):
            raise ValueError("static Hamiltonian is not Hermitian within tolerance")
        for k, hc in enumerate(self.h_controls):
            if _shape(hc) != _shape(self.h_static):
                raise ValueError(f"control operator {k} has mismatched shape")
            if not is_hermitian(hc, 1e-12 * max(1.0, one_norm_host(hc))):
                raise ValueError(f"control operator {k} is not Hermitian")

    def step_evaluator(self, a: "ControlField", n: int):
        """The reference's per-step evaluator (src/costs.py:131-138): step n's amplitudes folded into
        H_n, actions evaluated on the device (derivatives.StepEvaluator)."""
        from .derivatives import StepContext, StepEvaluator

        coeffs = [1.0] + [complex(x) for x in a.amplitudes[n]]
        h_step = linear_combine(coeffs, [self.h_static, *self.h_controls])
        return StepEvaluator(StepContext(h_step, self.h_controls, a.dt, self.backend, self.tau, validate=False))

    @property
    def dim(self) -> int:
        return self.h_static.n_rows

    @property
    def n_channels(self) -> int:
        return len(self.h_controls)


@dataclass(frozen=True)
class CostTerm:
    """One weighted cost contribution (src/costs.py:141-168) + ``target_images``."""

    kind: CostKind
    weight: float = 1.0
    target_state: np.ndarray | None = None
    target_gate: np.ndarray | None = None
    penalty_op: object = None
    target_images: np.ndarray | None = None

    def __post_init__(self):
        if self.weight < 0.0:
            raise ValueError("cost weights must be non-negative")
        for name in ("target_state", "target_gate", "target_images"):
            v = getattr(self, name)
            if v is not None:
                object.__setattr__(self, name, frozen_copy(v, np.complex128))
        if self.penalty_op is not None:
            object.__setattr__(self, "penalty_op", as_own_matrix(self.penalty_op))
        if self.kind in (CostKind.STATE_INFIDELITY, CostKind.STATE_RUNNING_INFIDELITY):
            if self.target_state is None:
                raise ValueError(f"{self.kind.value} requires target_state")
        elif self.kind is CostKind.STATE_PENALTY:
            if self.penalty_op is None:
                raise ValueError("state_penalty requires penalty_op")
            if not is_hermitian(self.penalty_op, 1e-12 * max(1.0, one_norm_host(self.penalty_op))):
                raise ValueError("penalty operator must be Hermitian")
        else:
            if self.target_gate is None and self.target_images is None:
                raise ValueError(f"{self.kind.value} requires target_gate")
            if self.target_gate is not None:
                u = np.asarray(self.target_gate)
                defect = np.abs(u.conj().T @ u - np.eye(u.shape[0])).max()
                if defect > 1e-10:
                    raise ValueError(f"target gate is not unitary (defect {defect:.2e})")


@dataclass(frozen=True)
class GradientResult:
    """cost, grad[n, k] = dC/da[n, k], and the live state-vector peak (src/costs.py:171-182).
    ``live_vector_peak`` counts the device state vectors held per trajectory; it
    does not depend on the number of steps."""

    cost: float
    grad: np.ndarray
    live_vector_peak: int


# ------------------------------------------------------------------------- native marshalling


def _as_rows(x, d, name):
    a = np.asarray(x, dtype=np.complex128)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    if a.ndim != 2 or a.shape[1] != d:
        raise ValueError(f"{name} has shape {np.shape(x)}, expected ({d},) or (K, {d})")
    return np.ascontiguousarray(a)


class _Keep:
    """Holds numpy buffers alive while a descriptor is passed to the library."""

    def __init__(self):
        self.refs = []

    def arr(self, a):
        self.refs.append(a)
        return a


def _matrix(m, d, keep: _Keep) -> _native.lg_matrix:
    s = _native.lg_matrix()
    s.n = d
    if isinstance(m, DenseMatrix) or hasattr(m, "array"):
        a = np.asarray(m.array, dtype=np.complex128)
        if a.shape != (d, d):
            raise ValueError("operator dimension mismatch")
        a = keep.arr(np.asfortranarray(a).ravel(order="F").view(np.float64))
        s.dense = 1
        s.nnz = d * d
        s.values = _native.dptr(a)
        return s
    if (m.n_rows, m.n_cols) != (d, d):
        raise ValueError("operator dimension mismatch")
    ro = keep.arr(np.ascontiguousarray(m.row_offsets, np.int64))
    ci = keep.arr(np.ascontiguousarray(m.col_indices, np.int64))
    va = keep.arr(np.ascontiguousarray(m.values, np.complex128).view(np.float64))
    s.dense = 0
    s.nnz = ci.size
    s.row_offsets = _native.i64ptr(ro)
    s.col_indices = _native.i64ptr(ci)
    s.values = _native.dptr(va)
    return s


class NativeProblem:
    """One device-resident problem: operators, trajectories and cost terms."""

    def __init__(self, problem: ControlProblem, terms, initial_states=None, basis=None, device: int = 0,
                 shard: tuple[int, int] | None = None):
        diag = problem.backend is Backend.DIAGONALIZATION
        lib = _native.load()
        d = problem.dim
        keep = _Keep()
        desc = _native.lg_problem_desc()
        # DIAGONALIZATION factorises the dense step matrix (src/derivatives.py:228-230): dense operators
        dn = (lambda m: DenseMatrix(to_dense(m))) if diag else (lambda m: m)
        desc.h_static = _matrix(dn(problem.h_static), d, keep)
        ctrls = (_native.lg_matrix * len(problem.h_controls))()
        for k, h in enumerate(problem.h_controls):
            ctrls[k] = _matrix(dn(h), d, keep)
        keep.arr(ctrls)
        desc.n_channels = len(problem.h_controls)
        desc.h_controls = ctrls
        desc.tau = float(problem.tau)
        state_terms = [t for t in terms if t.kind in _STATE_KINDS]
        gate_terms = [t for t in terms if t.kind not in _STATE_KINDS]
        ks = 0
        if initial_states is not None:
            st = keep.arr(_as_rows(initial_states, d, "initial_state").view(np.float64))
            ks = st.shape[0] * st.shape[1] // (2 * d)
            desc.n_states = ks
            desc.initial_states = _native.dptr(st)
        elif state_terms:
            raise ValueError("state-transfer terms require problem.initial_state")
        kg = 0
        basis_rows = None
        if gate_terms:
            if basis is None:
                basis_rows = np.eye(d, dtype=np.complex128)
            else:
                basis_rows = _as_rows(np.asarray(basis), d, "basis")
                if basis_rows.shape[0] > d:
                    raise ValueError(f"basis must contain at most {d} states, got {basis_rows.shape[0]}")
                gram = basis_rows.conj() @ basis_rows.T
                if np.abs(gram - np.eye(basis_rows.shape[0])).max() > 1e-10:
                    raise ValueError("gate basis is not orthonormal")
            kg = basis_rows.shape[0]
            b = keep.arr(np.ascontiguousarray(basis_rows).view(np.float64))
            desc.n_basis = kg
            desc.basis = _native.dptr(b)
        cterms = (_native.lg_cost_term * max(1, len(terms)))()
        for i, t in enumerate(terms):
            ct = cterms[i]
            ct.kind = _KIND_CODE[t.kind]
            ct.weight = float(t.weight)
            if t.kind is CostKind.STATE_PENALTY:
                ct.penalty = _matrix(t.penalty_op, d, keep)
            elif t.kind in _STATE_KINDS:
                tg = _as_rows(t.target_state, d, "target_state")
                if tg.shape[0] != ks:
                    raise ValueError(f"target_state has {tg.shape[0]} rows, initial_state has {ks}")
                ct.targets = _native.dptr(keep.arr(tg.view(np.float64)))
            else:
                if t.target_images is not None:
                    im = _as_rows(t.target_images, d, "target_images")
                else:
                    u = np.asarray(t.target_gate, np.complex128)
                    if u.shape != (d, d):
                        raise ValueError("target gate dimension mismatch")
                    im = np.ascontiguousarray((u @ basis_rows.T).T)
                if im.shape[0] != kg:
                    raise ValueError(f"target_images has {im.shape[0]} rows, basis has {kg}")
                ct.targets = _native.dptr(keep.arr(im.view(np.float64)))
        keep.arr(cterms)
        desc.n_terms = len(terms)
        desc.terms = cterms
        desc.device = device
        desc.backend = 1 if diag else 0
        if shard is not None:
            desc.shard_begin, desc.shard_end = shard
        h = C.c_void_p()
        _native.check(lib.lg_problem_create(C.byref(desc), C.byref(h)))
        self._lib = lib
        self.handle = h
        self.dim = d
        self.n_channels = len(problem.h_controls)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self._lib.lg_problem_destroy(h)
            self.handle = None

    @property
    def engine(self) -> str:
        """Sweep engine the library chose for this problem (lg_engine_name)."""
        return self._lib.lg_engine_name(self.handle).decode()

    @property
    def diag_solver(self) -> str:
        """Per-step factorisation the last DIAGONALIZATION evaluation used (lg_diag_solver_name)."""
        return self._lib.lg_diag_solver_name(self.handle).decode()

    def grad(self, a: ControlField) -> GradientResult:
        amps = np.ascontiguousarray(a.amplitudes, np.float64)
        cost = C.c_double()
        g = np.zeros((a.n_steps, a.n_channels))
        peak = C.c_int64()
        _native.check(self._lib.lg_eval(self.handle, a.n_steps, float(a.dt), _native.dptr(amps), C.byref(cost),
                                        _native.dptr(g), C.byref(peak)))
        return GradientResult(cost=float(cost.value), grad=g, live_vector_peak=int(peak.value))

    def cost(self, a: ControlField) -> float:
        amps = np.ascontiguousarray(a.amplitudes, np.float64)
        cost = C.c_double()
        _native.check(self._lib.lg_cost(self.handle, a.n_steps, float(a.dt), _native.dptr(amps), C.byref(cost)))
        return float(cost.value)

    def cost_batch(self, fields) -> list:
        """Costs of several fields with the same (n_steps, dt) in one forward launch
        (``lg_cost_batch``); NotImplementedError on engines without a batched forward kernel."""
        amps = np.ascontiguousarray(np.stack([a.amplitudes for a in fields]), np.float64)
        out = np.zeros(len(fields), np.float64)
        a0 = fields[0]
        _native.check(self._lib.lg_cost_batch(self.handle, len(fields), a0.n_steps, float(a0.dt), _native.dptr(amps),
                                              _native.dptr(out)))
        return [float(c) for c in out]

    def forward_states(self, a: ControlField, k: int) -> np.ndarray:
        amps = np.ascontiguousarray(a.amplitudes, np.float64)
        out = np.zeros((k, self.dim), np.complex128)
        _native.check(self._lib.lg_forward_states(self.handle, a.n_steps, float(a.dt), _native.dptr(amps),
                                                  _native.dptr(out.view(np.float64))))
        return out

    def step_derivative(self, a: ControlField, step: int, channel: int, psi) -> np.ndarray:
        """(dU_step/da_channel) psi of a DIAGONALIZATION problem from the device factorisation
        (derivative_action_diag, src/derivatives.py:256-275)."""
        amps = np.ascontiguousarray(a.amplitudes, np.float64)
        vec = np.ascontiguousarray(psi, np.complex128)
        if vec.shape != (self.dim,):
            raise ValueError("state dimension mismatch")
        out = np.zeros(self.dim, np.complex128)
        _native.check(self._lib.lg_step_derivative(self.handle, a.n_steps, float(a.dt), _native.dptr(amps), int(step),
                                                   int(channel), _native.dptr(vec.view(np.float64)),
                                                   _native.dptr(out.view(np.float64))))
        return out

    def plan_table(self, a: ControlField) -> dict:
        N, Kc = a.n_steps, a.n_channels
        amps = np.ascontiguousarray(a.amplitudes, np.float64)
        out = dict(norm1=np.zeros(N), sp=np.zeros(N, np.int64), m=np.zeros(N, np.int32), s=np.zeros(N, np.int32),
                   aux_arg=np.zeros((N, Kc)), aux_sp=np.zeros((N, Kc), np.int64), aux_m=np.zeros((N, Kc), np.int32),
                   aux_s=np.zeros((N, Kc), np.int32))
        _native.check(self._lib.lg_plan_table(
            self.handle, N, float(a.dt), _native.dptr(amps), _native.dptr(out["norm1"]), _native.i64ptr(out["sp"]),
            _native.i32ptr(out["m"]), _native.i32ptr(out["s"]), _native.dptr(out["aux_arg"]),
            _native.i64ptr(out["aux_sp"]), _native.i32ptr(out["aux_m"]), _native.i32ptr(out["aux_s"])))
        return out

    def raw(self, n_steps: int) -> np.ndarray:
        buf = np.zeros(self._lib.lg_raw_size(self.handle, n_steps))
        _native.check(self._lib.lg_raw_get(self.handle, _native.dptr(buf)))
        return buf

    def raw_size(self, n_steps: int) -> int:
        return int(self._lib.lg_raw_size(self.handle, n_steps))

    def set_raw_buffer(self, ptr: int, length: int) -> None:
        """Lend the library device memory for the raw scalars (lg_set_raw_buffer)."""
        _native.check(self._lib.lg_set_raw_buffer(self.handle, C.c_void_p(ptr or None), int(length)))

    def set_stream(self, stream_ptr: int) -> None:
        _native.check(self._lib.lg_set_stream(self.handle, C.c_void_p(stream_ptr or None)))

    def grad_sharded(self, a: ControlField, hook) -> GradientResult:
        """lg_eval_sharded: `hook(ptr, count)` sums `count` doubles at device address ptr across ranks."""
        amps = np.ascontiguousarray(a.amplitudes, np.float64)
        cost = C.c_double()
        g = np.zeros((a.n_steps, a.n_channels))
        cb = _native.ALLREDUCE_FN(lambda ptr, count, stream, user: hook(ptr, count))
        _native.check(self._lib.lg_eval_sharded(self.handle, a.n_steps, float(a.dt), _native.dptr(amps), cb, None,
                                                C.byref(cost), _native.dptr(g)))
        return GradientResult(cost=float(cost.value), grad=g,
                              live_vector_peak=int(self._lib.lg_live_vector_peak(self.handle)))

    def cost_sharded(self, a: ControlField, hook) -> float:
        amps = np.ascontiguousarray(a.amplitudes, np.float64)
        cost = C.c_double()
        cb = _native.ALLREDUCE_FN(lambda ptr, count, stream, user: hook(ptr, count))
        _native.check(self._lib.lg_cost_sharded(self.handle, a.n_steps, float(a.dt), _native.dptr(amps), cb, None,
                                                C.byref(cost)))
        return float(cost.value)

    def finalize(self, n_steps: int, raw: np.ndarray):
        raw = np.ascontiguousarray(raw, np.float64)
        cost = C.c_double()
        g = np.zeros((n_steps, self.n_channels))
        _native.check(self._lib.lg_finalize_host(self.handle, n_steps, _native.dptr(raw), C.byref(cost),
                                                 _native.dptr(g)))
        return float(cost.value), g


_CACHE: "OrderedDict[tuple, tuple]" = OrderedDict()
_CACHE_SIZE = 8


def _native_for(problem, terms, initial_states, basis) -> NativeProblem:
    """Device problems are built once per (problem, terms, states) and reused."""
    key = (id(problem), tuple(id(t) for t in terms), id(initial_states), id(basis))
    hit = _CACHE.get(key)
    if hit is not None:
        _CACHE.move_to_end(key)
        return hit[0]
    npb = NativeProblem(problem, terms, initial_states, basis)
    _CACHE[key] = (npb, problem, tuple(terms), initial_states, basis)
    while len(_CACHE) > _CACHE_SIZE:
        _CACHE.popitem(last=False)
    return npb


def _check_field(problem, a):
    if a.n_channels != problem.n_channels:
        raise ValueError(f"field has {a.n_channels} channels, problem has {problem.n_channels}")


def _split(terms):
    if not terms:
        raise ValueError("composite cost needs at least one term")
    terms = list(terms)
    has_state = any(t.kind in _STATE_KINDS for t in terms)
    if has_state and getattr(terms[0], "kind", None) is None:
        raise ValueError("bad cost term")
    return terms, has_state


def composite_grad(problem: ControlProblem, a: ControlField, terms) -> GradientResult:
    """Weighted sum of cost terms and their gradient (src/costs.py:515-546), on the GPU."""
    terms, has_state = _split(terms)
    _check_field(problem, a)
    if has_state and problem.initial_state is None:
        raise ValueError("state-transfer terms require problem.initial_state")
    npb = _native_for(problem, terms, problem.initial_state if has_state else None, problem.basis)
    return npb.grad(a)


def composite_cost(problem: ControlProblem, a: ControlField, terms) -> float:
    """Weighted cost only (src/costs.py:549-597): forward sweeps on the GPU."""
    terms, has_state = _split(terms)
    _check_field(problem, a)
    if has_state and problem.initial_state is None:
        raise ValueError("state-transfer terms require problem.initial_state")
    npb = _native_for(problem, terms, problem.initial_state if has_state else None, problem.basis)
    return npb.cost(a)


_POOLS: "OrderedDict[tuple, tuple]" = OrderedDict()


def composite_cost_batch(problem: ControlProblem, fields, terms) -> list:
    """``composite_cost`` for several fields at once (the line-search path,
    src/optimizer.py:153-170).  Fields with a common (n_steps, dt) go through ``lg_cost_batch``:
    one forward launch over (candidate, trajectory) for the warp-specialised and cluster engines.
    Other engines (dense GEMM, DIAGONALIZATION) give each field its own device problem and stream
    and run the evaluations concurrently.  Every cost is bit-identical to ``composite_cost`` of
    that field."""
    from concurrent.futures import ThreadPoolExecutor

    terms, has_state = _split(terms)
    fields = list(fields)
    for a in fields:
        _check_field(problem, a)
    if has_state and problem.initial_state is None:
        raise ValueError("state-transfer terms require problem.initial_state")
    if not fields:
        return []
    if len(fields) > 1 and len({(a.n_steps, float(a.dt)) for a in fields}) == 1:
        npb = _native_for(problem, terms, problem.initial_state if has_state else None, problem.basis)
        try:
            return npb.cost_batch(fields)
        except NotImplementedError:
            pass
    key = (id(problem), tuple(id(t) for t in terms))
    hit = _POOLS.get(key)
    pool = list(hit[0]) if hit else []
    while len(pool) < len(fields):
        pool.append(NativeProblem(problem, terms, problem.initial_state if has_state else None, problem.basis))
    _POOLS[key] = (pool, problem, tuple(terms))
    while len(_POOLS) > 4:
        _POOLS.popitem(last=False)
    if len(fields) == 1:
        return [pool[0].cost(fields[0])]
    with ThreadPoolExecutor(max_workers=len(fields)) as ex:
        return list(ex.map(lambda pa: pa[0].cost(pa[1]), zip(pool, fields)))


def _single(problem, a, psi0, term):
    _check_field(problem, a)
    npb = NativeProblem(problem, [term], initial_states=psi0)
    return npb.grad(a)


def c1_state_grad(problem, a, psi0, phi_target) -> GradientResult:
    """1 - |<phi_T|psi_N>|^2 and its gradient (src/costs.py:357-362)."""
    return _single(problem, a, psi0, CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=phi_target))


def c2_state_grad(problem, a, psi0, penalty_op) -> GradientResult:
    """(1/N) sum_n <psi_n|Omega|psi_n> and its gradient (src/costs.py:365-372)."""
    return _single(problem, a, psi0, CostTerm(CostKind.STATE_PENALTY, 1.0, penalty_op=penalty_op))


def c3_state_grad(problem, a, psi0, phi_target) -> GradientResult:
    """1 - (1/N) sum_n |<phi_T|psi_n>|^2 and its gradient (src/costs.py:375-384)."""
    return _single(problem, a, psi0, CostTerm(CostKind.STATE_RUNNING_INFIDELITY, 1.0, target_state=phi_target))


def _gate(problem, a, u_target, basis, kind):
    _check_field(problem, a)
    b = basis if basis is not None else problem.basis
    npb = NativeProblem(problem, [CostTerm(kind, 1.0, target_gate=u_target)], basis=b)
    return npb.grad(a)


def c1_gate_grad(problem, a, u_target, basis=None) -> GradientResult:
    """1 - |tr(U_T^+ U)/K|^2 and its gradient (src/costs.py:491-495)."""
    return _gate(problem, a, u_target, basis, CostKind.GATE_INFIDELITY)


def c3_gate_grad(problem, a, u_target, basis=None) -> GradientResult:
    """1 - sum_n |tr(U_T^+ U_n)|^2/(N K^2) and its gradient (src/costs.py:498-502)."""
    return _gate(problem, a, u_target, basis, CostKind.GATE_RUNNING_INFIDELITY)


def forward_propagate(problem: ControlProblem, a: ControlField, psi0) -> np.ndarray:
    """Propagate psi0 (d,) or a block (K, d) through all steps (src/costs.py:209-217)."""
    _check_field(problem, a)
    rows = _as_rows(psi0, problem.dim, "psi0")
    npb = NativeProblem(problem, [], initial_states=rows)
    out = npb.forward_states(a, rows.shape[0])
    return out[0] if np.ndim(psi0) == 1 else out
