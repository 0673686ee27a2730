"""B200-native hard-coded-gradient (HG) GRAPE evaluation.

Drop-in for the hot path of the reference package ``leangrape`` (arXiv
2304.06200): ``composite_grad`` / ``composite_cost`` and the cost objects they
consume, evaluated by hand-written sm_100a CUDA kernels behind the C ABI in
``include/leangrape_b200.h``.
"""

from .costs import (
    Backend,
    ControlField,
    ControlProblem,
    CostKind,
    CostTerm,
    GradientResult,
    c1_gate_grad,
    c1_state_grad,
    c2_state_grad,
    c3_gate_grad,
    c3_state_grad,
    composite_cost,
    composite_cost_batch,
    composite_grad,
    forward_propagate,
)
from .expm import ExpmPlan, PlanningError, make_plan
from .optimizer import OptimizationTrace, OptimizerConfig, grape_optimize
from .sparse import CsrMatrix, DenseMatrix, build_csr, build_csr_arrays, from_dense, identity_csr, linear_combine

__all__ = [
    "Backend", "ControlField", "ControlProblem", "CostKind", "CostTerm", "GradientResult",
    "c1_gate_grad", "c1_state_grad", "c2_state_grad", "c3_gate_grad", "c3_state_grad",
    "composite_cost", "composite_cost_batch", "composite_grad", "forward_propagate", "ExpmPlan", "PlanningError", "make_plan",
    "OptimizationTrace", "OptimizerConfig", "grape_optimize", "CsrMatrix", "DenseMatrix", "build_csr",
    "build_csr_arrays", "from_dense", "identity_csr", "linear_combine",
]
