"""Per-step propagator actions (mirror of src/derivatives.py:54-84,105-225,278-330).

The reference's ``StepEvaluator`` serves one time step: ``forward`` (exp(-i H_n dt) psi), ``adjoint``
(exp(+i H_n dt) psi) and ``control_derivative`` ((dU_n/da_k) psi through the block embedding
``exp([[A, A_c], [0, A]]) (0, psi)``).  Inside ``composite_grad`` these run fused in the sweep kernels;
this module exposes the same three actions one step at a time for callers that use the reference's
``ControlProblem.step_evaluator`` / ``derivatives.propagate`` surface directly.  Every action is a
certified Taylor action evaluated on the GPU (``expm.apply`` -> ``lg_expm_apply``) under the plan the
reference would select: the generator's numpy-order one-norm and sigma' for the propagators, the
two-norm surrogate sqrt(norm_1 norm_inf) and the embedding's sigma' for the derivative (the
materialised embedding up to 2 d = 256, the block operator's assembled bounds with its extra unit
above, src/derivatives.py:133-196).  There is no host evaluation path.

DIAGONALIZATION: ``forward`` / ``adjoint`` / ``control_derivative`` run a one-step device problem on
that backend (hand-written Jacobi factorisation and the eigenbasis derivative formula of
src/derivatives.py:256-275 in csrc/lg_diag.cu; the product through the C ABI's
``lg_step_derivative``).  The host objects ``diag_prepare`` / ``DiagFactorization`` are not offered:
the factorisation never leaves the device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import expm
from .costs import Backend
from .sparse import DenseMatrix, as_own_matrix, aux_embed, build_csr, build_csr_arrays, is_hermitian, to_dense

__all__ = ["Backend", "StepContext", "BlockDerivativeOperator", "StepEvaluator", "propagate", "propagate_adjoint",
           "aux_embed", "aux_plan", "derivative_action_aux", "MATERIALIZE_DIM_LIMIT"]

MATERIALIZE_DIM_LIMIT = 256  # src/derivatives.py: embeddings up to this dimension are materialised


@dataclass(frozen=True)
class StepContext:
    """One step: H_n = H_s + sum_k a_k h_k with the amplitudes folded in, the control operators, dt."""

    h_step: object
    h_controls: tuple
    dt: float
    backend: Backend = Backend.SCALING_SQUARING
    tau: float = 1e-8
    validate: bool = True

    def __post_init__(self):
        object.__setattr__(self, "h_step", as_own_matrix(self.h_step))
        object.__setattr__(self, "h_controls", tuple(as_own_matrix(h) for h in self.h_controls))
        if self.dt <= 0.0:
            raise ValueError("dt must be positive")
        if self.validate:
            if not is_hermitian(self.h_step, 1e-12 * max(1.0, self.h_step.one_norm())):
                raise ValueError("step Hamiltonian is not Hermitian within tolerance")
            for k, hc in enumerate(self.h_controls):
                if not is_hermitian(hc, 1e-12 * max(1.0, hc.one_norm())):
                    raise ValueError(f"control operator {k} is not Hermitian")

    @property
    def dim(self) -> int:
        return self.h_step.shape[0]


def _generator(ctx: StepContext):
    return ctx.h_step.scaled(-1j * ctx.dt)


def _plan_for(ctx: StepContext, gen) -> expm.ExpmPlan:
    norm1, sp = expm.plan_inputs(gen)
    return expm.make_plan(norm1, sp, ctx.tau)


def _state(ctx: StepContext, psi) -> np.ndarray:
    v = np.asarray(psi, dtype=np.complex128)
    if v.shape != (ctx.dim,):
        raise ValueError("state dimension mismatch")
    return v


def _diag_action(ctx: StepContext, psi, sign: float) -> np.ndarray:
    """exp(-i sign H dt) psi on the device DIAGONALIZATION backend: a one-step problem whose static
    Hamiltonian is sign * H_n and whose (required) control channel carries amplitude zero."""
    from .costs import ControlField, ControlProblem, forward_propagate

    d = ctx.dim
    ctrl = ctx.h_controls[0] if ctx.h_controls else build_csr([], d, d)
    problem = ControlProblem(ctx.h_step.scaled(sign), (ctrl,), ctx.backend, ctx.tau)
    return forward_propagate(problem, ControlField.constant(0.0, 1, 1, ctx.dt), _state(ctx, psi))


def _diag_derivative(ctx: StepContext, channel: int, psi) -> np.ndarray:
    """(dU/da_channel) psi on the device DIAGONALIZATION backend: the one-step problem H_n + 0 * h_c
    (amplitudes already folded into h_step), product by lg_step_derivative."""
    from .costs import ControlField, ControlProblem, NativeProblem

    problem = ControlProblem(ctx.h_step, (ctx.h_controls[channel],), ctx.backend, ctx.tau)
    npb = NativeProblem(problem, [], initial_states=_state(ctx, psi).reshape(1, -1))
    return npb.step_derivative(ControlField.constant(0.0, 1, 1, ctx.dt), 0, 0, psi)


def propagate(ctx: StepContext, psi) -> np.ndarray:
    """exp(-i H dt) psi (src/derivatives.py:113-118)."""
    if ctx.backend is Backend.DIAGONALIZATION:
        return _diag_action(ctx, psi, 1.0)
    gen = _generator(ctx)
    return expm.apply(gen, _state(ctx, psi), _plan_for(ctx, gen), validate=False)


def propagate_adjoint(ctx: StepContext, psi) -> np.ndarray:
    """exp(+i H dt) psi under the forward plan: negation keeps the norms (src/derivatives.py:121-130)."""
    if ctx.backend is Backend.DIAGONALIZATION:
        return _diag_action(ctx, psi, -1.0)
    gen = _generator(ctx)
    return expm.apply(gen.scaled(-1.0), _state(ctx, psi), _plan_for(ctx, gen), validate=False)


class BlockDerivativeOperator:
    """The embedded derivative generator described by its blocks (src/derivatives.py:133-184): norms
    and the per-row count assembled from A = -i H dt and A_c = -i h_c dt exactly as the reference
    does, including the extra sigma' unit of its two-part top block.  ``stored()`` gives the device
    the entrywise identical stored matrix."""

    def __init__(self, generator, h_control, dt: float):
        self.generator = as_own_matrix(generator)
        self.control_gen = as_own_matrix(h_control).scaled(-1j * dt)
        d = self.generator.shape[0]
        self.n_rows = self.n_cols = 2 * d
        self.shape = (2 * d, 2 * d)
        self.nnz = 2 * self.generator.nnz + self.control_gen.nnz

    def one_norm(self) -> float:
        g, c = self.generator.col_abs_sums(), self.control_gen.col_abs_sums()
        return float(max(g.max(), (g + c).max())) if g.size else 0.0

    def inf_norm(self) -> float:
        g, c = self.generator.row_abs_sums(), self.control_gen.row_abs_sums()
        return float(max((g + c).max(), g.max())) if g.size else 0.0

    def max_row_nnz(self) -> int:
        counts = self.generator.row_nnz_counts() + self.control_gen.row_nnz_counts()
        return (int(counts.max()) if counts.size else 0) + 1

    def stored(self):
        d = self.generator.shape[0]
        if isinstance(self.generator, DenseMatrix) or isinstance(self.control_gen, DenseMatrix):
            big = np.zeros((2 * d, 2 * d), np.complex128, order="F")
            big[:d, :d] = to_dense(self.generator)
            big[:d, d:] = to_dense(self.control_gen)
            big[d:, d:] = big[:d, :d]
            return DenseMatrix(big)
        gr, gc, gv = self.generator.triplets()
        cr, cc, cv = self.control_gen.triplets()
        return build_csr_arrays(np.concatenate([gr, cr, gr + d]), np.concatenate([gc, cc + d, gc + d]),
                                np.concatenate([gv, cv, gv]), 2 * d, 2 * d)


def aux_plan(aux, tau: float) -> expm.ExpmPlan:
    """Plan of the (non-normal) embedding from the two-norm surrogate (src/derivatives.py:187-196)."""
    return expm.make_plan(math.sqrt(aux.one_norm() * aux.inf_norm()), aux.max_row_nnz(), tau)


def _embedded(ctx: StepContext, channel: int, gen):
    """(matrix the device applies, object whose bounds select the plan)."""
    if 2 * ctx.dim <= MATERIALIZE_DIM_LIMIT:
        m = aux_embed(ctx.h_step, ctx.h_controls[channel], ctx.dt)
        return m, m
    blk = BlockDerivativeOperator(gen, ctx.h_controls[channel], ctx.dt)
    return blk.stored(), blk


def _aux_action(ctx: StepContext, matrix, plan, psi):
    d = ctx.dim
    stacked = np.zeros(2 * d, np.complex128)
    stacked[d:] = _state(ctx, psi)
    res = expm.apply(matrix, stacked, plan, validate=False)
    return res[:d].copy(), res[d:].copy()


def derivative_action_aux(ctx: StepContext, channel: int, psi):
    """((dU/da_channel) psi, U psi) via the block embedding (src/derivatives.py:205-225)."""
    if not 0 <= channel < len(ctx.h_controls):
        raise IndexError(f"control channel {channel} out of range")
    matrix, bounds = _embedded(ctx, channel, _generator(ctx))
    return _aux_action(ctx, matrix, aux_plan(bounds, ctx.tau), psi)


class StepEvaluator:
    """One step's generator, plan and embeddings, built once and reused by the three actions
    (src/derivatives.py:278-330)."""

    def __init__(self, ctx: StepContext):
        self.ctx = ctx
        self._gen = None
        self._plan = None
        self._aux = {}

    def _generator_plan(self):
        if self._gen is None:
            self._gen = _generator(self.ctx)
            self._plan = _plan_for(self.ctx, self._gen)
        return self._gen, self._plan

    def forward(self, psi) -> np.ndarray:
        if self.ctx.backend is Backend.DIAGONALIZATION:
            return _diag_action(self.ctx, psi, 1.0)
        gen, plan = self._generator_plan()
        return expm.apply(gen, _state(self.ctx, psi), plan, validate=False)

    def adjoint(self, psi) -> np.ndarray:
        if self.ctx.backend is Backend.DIAGONALIZATION:
            return _diag_action(self.ctx, psi, -1.0)
        gen, plan = self._generator_plan()
        return expm.apply(gen.scaled(-1.0), _state(self.ctx, psi), plan, validate=False)

    def control_derivative(self, channel: int, psi) -> np.ndarray:
        if not 0 <= channel < len(self.ctx.h_controls):
            raise IndexError(f"control channel {channel} out of range")
        if self.ctx.backend is Backend.DIAGONALIZATION:
            return _diag_derivative(self.ctx, channel, psi)
        if channel not in self._aux:
            gen, _ = self._generator_plan()
            matrix, bounds = _embedded(self.ctx, channel, gen)
            self._aux[channel] = (matrix, aux_plan(bounds, self.ctx.tau))
        matrix, plan = self._aux[channel]
        return _aux_action(self.ctx, matrix, plan, psi)[0]
