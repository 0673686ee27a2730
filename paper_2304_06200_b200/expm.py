"""Certified planner surface (mirror of src/expm.py:87-107,279-303).

``make_plan`` runs the library's exact host port of the reference planner
(csrc/lg_planner.cuh, bit-identical to ``leangrape.expm.make_plan``).  During an
evaluation the same planner runs on the GPU for every (step, operator) at once;
entries that fall inside its libm guard band are recomputed with this exact
host path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native

__all__ = ["ExpmPlan", "PlanningError", "BoundInfeasibleError", "make_plan", "make_plans_device", "plan_inputs", "apply", "expm_multiply",
           "is_anti_hermitian", "DEFAULT_M_MAX", "DEFAULT_S_MAX"]

DEFAULT_M_MAX = 60
DEFAULT_S_MAX = 10_000


class PlanningError(RuntimeError):
    """No feasible (order, scaling) pair within the search limits."""


class BoundInfeasibleError(ArithmeticError):
    """The rounding model is outside its validity range (n u' >= 1, src/expm.py:65-67,146-153).
    The planner handles it internally (such plans are skipped, as the reference's loop does);
    exported for API parity."""


@dataclass(frozen=True)
class ExpmPlan:
    order: int
    scaling: int
    tau: float
    norm1: float
    sigma_prime: int
    bound: float

    @property
    def matvecs(self) -> int:
        return self.order * self.scaling


def make_plan(norm1_a: float, sigma_prime: int, tau: float, *, m_max: int = DEFAULT_M_MAX,
              s_max: int = DEFAULT_S_MAX) -> ExpmPlan:
    lib = _native.load()
    m, s, b = C.c_int32(), C.c_int32(), C.c_double()
    _native.check(lib.lg_make_plan(float(norm1_a), int(sigma_prime), float(tau), int(m_max), int(s_max),
                                   C.byref(m), C.byref(s), C.byref(b)))
    return ExpmPlan(m.value, s.value, float(tau), float(norm1_a), int(sigma_prime), b.value)


def make_plans_device(norm1, sigma, tau: float):
    """Device planner over arrays (guarded; uncertain entries re-planned on the host).
    Returns (order, scaling, status, n_uncertain); status 1 marks PlanningError entries."""
    lib = _native.load()
    norm1 = np.ascontiguousarray(norm1, np.float64)
    sigma = np.ascontiguousarray(sigma, np.int64)
    n = norm1.size
    order = np.zeros(n, np.int32)
    scaling = np.zeros(n, np.int32)
    status = np.zeros(n, np.int32)
    unc = C.c_int32()
    _native.check(lib.lg_make_plans_device(n, _native.dptr(norm1), _native.i64ptr(sigma), float(tau),
                                           _native.i32ptr(order), _native.i32ptr(scaling), _native.i32ptr(status),
                                           C.byref(unc)))
    return order, scaling, status, unc.value


# ----------------------------------------------------------------------------------------------
# Standalone certified action (src/expm.py:306-369): exp(A) psi on the GPU.


def _shape(a):
    return (a.n_rows, a.n_cols) if hasattr(a, "n_rows") else np.asarray(a.array).shape


def plan_inputs(a) -> tuple[float, int]:
    """(A.one_norm(), A.max_row_nnz()) exactly as the reference computes them (numpy's reduction
    order; DenseMatrix reports n_cols), via the library's host path."""
    from .costs import _Keep, _matrix

    n, m = _shape(a)
    if n != m:
        raise ValueError("generator must be square")
    keep = _Keep()
    desc = _matrix(a, n, keep)
    norm1, sp = C.c_double(), C.c_int64()
    _native.check(_native.load().lg_expm_plan_inputs(C.byref(desc), C.byref(norm1), C.byref(sp)))
    return float(norm1.value), int(sp.value)


def is_anti_hermitian(a, tol: float) -> bool:
    """max |A + A^dagger| <= tol (src/sparse.py:400-404); host-side input validation."""
    n, m = _shape(a)
    if n != m:
        return False
    dense = np.asarray(a.array) if hasattr(a, "array") else a.to_dense()
    return float(np.max(np.abs(dense + dense.conj().T), initial=0.0)) <= tol


def apply(a, psi, plan: ExpmPlan, *, validate: bool = True, out: np.ndarray | None = None,
          device: int = 0) -> np.ndarray:
    """exp(A) @ psi under a previously selected plan (src/expm.py:306-351), evaluated on the GPU:
    ``plan.matvecs`` fused Taylor terms ``term <- (A term) * (1/(s j)); current += term``.
    ``psi`` may also be a (K, d) block of states (one launch per term for all of them)."""
    from .costs import _Keep, _matrix

    n, m = _shape(a)
    psi_arr = np.asarray(psi, dtype=np.complex128)
    if n != m or psi_arr.ndim not in (1, 2) or psi_arr.shape[-1] != m:
        raise ValueError("apply expects a square matrix and a matching vector")
    if validate:
        norm1, _ = plan_inputs(a)
        if not is_anti_hermitian(a, 1e-12 * max(norm1, 1.0)):
            raise ValueError("generator is not anti-Hermitian within tolerance")
    rows = np.ascontiguousarray(psi_arr.reshape(-1, m))
    res = np.empty_like(rows)
    keep = _Keep()
    desc = _matrix(a, n, keep)
    _native.check(_native.load().lg_expm_apply(C.byref(desc), rows.shape[0], _native.dptr(rows.view(np.float64)),
                                               int(plan.order), int(plan.scaling),
                                               _native.dptr(res.view(np.float64)), int(device)))
    res = res.reshape(psi_arr.shape)
    if out is not None:
        if out.shape != psi_arr.shape:
            raise ValueError("out has the wrong shape")
        np.copyto(out, res)
        return out
    return res


def expm_multiply(a, psi, tau: float, *, validate: bool = True, m_max: int = DEFAULT_M_MAX,
                  s_max: int = DEFAULT_S_MAX, device: int = 0):
    """Plan-and-apply convenience (src/expm.py:354-369): returns (exp(A) psi, matvecs used)."""
    norm1, sp = plan_inputs(a)
    plan = make_plan(norm1, sp, tau, m_max=m_max, s_max=s_max)
    return apply(a, psi, plan, validate=validate, device=device), plan.matvecs
