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

__all__ = ["ExpmPlan", "PlanningError", "make_plan", "make_plans_device", "DEFAULT_M_MAX", "DEFAULT_S_MAX"]

DEFAULT_M_MAX = 60
DEFAULT_S_MAX = 10_000


class PlanningError(RuntimeError):
    """No feasible (order, scaling) pair within the search limits."""


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
