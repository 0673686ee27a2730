"""Multi-GPU ``composite_grad`` / ``composite_cost``: the trajectory block sharded over ranks.

SURVEY.md section 8(e); north_star: "The K-state block shards across the 8 GPUs of one box, with
one NCCL allreduce over NVLink per evaluation for the overlaps and gradients."

One process per GPU (``torchrun``).  Rank r builds the device problem with trajectories
``[lo_r, hi_r)`` of each trajectory set -- the initial states (src/costs.py:109, K-state block)
and the gate basis (src/costs.py:110, 399-400) -- and lends the library a device tensor for its
raw per-trajectory scalars (``lg_set_raw_buffer``).  During ``lg_eval_sharded`` the library calls
back at the exchange points and the callback sums views of that tensor across ranks with
``torch.distributed.all_reduce`` (NCCL over NVLink/NVSwitch), on the stream the kernels run on:

* once per evaluation, the raw scalars (``<lambda|dU/da|psi>`` overlaps, final overlaps, running
  sums) before the device combine, so every rank ends with the same cost and gradient;
* only with a running gate cost (C3^g), also the per-step traces between the sweeps, because its
  costate source needs the global trace (src/costs.py:462, 477-478).

Every raw slot is indexed by trajectory and written by exactly one rank (the others hold 0), so
the sum is exact in any reduction order: results are bit-identical to the single-GPU evaluation
at every world size.
"""

from __future__ import annotations

from collections import OrderedDict

import torch
import torch.distributed as dist

from . import costs as _costs
from .costs import ControlField, ControlProblem, GradientResult


def shard_bounds(n_traj: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of trajectory indices for `rank` (the same range is taken from each set).
    Ranks past the end get an empty range at n_traj (still a sharded problem)."""
    per = -(-n_traj // world)
    lo = min(n_traj, rank * per)
    return lo, min(n_traj, lo + per)


def _set_sizes(problem: ControlProblem, terms) -> tuple[int, int]:
    has_state = any(t.kind in _costs._STATE_KINDS for t in terms)
    has_gate = any(t.kind not in _costs._STATE_KINDS for t in terms)
    ks = 0
    if has_state and problem.initial_state is not None:
        ks = _costs._as_rows(problem.initial_state, problem.dim, "initial_state").shape[0]
    kg = 0
    if has_gate:
        kg = problem.dim if problem.basis is None else _costs._as_rows(problem.basis, problem.dim, "basis").shape[0]
    return ks, kg


class ShardedEvaluator:
    """Evaluates one (problem, terms) pair with its trajectories sharded over a process group.

    ``native`` and ``buffer_device`` exist for host-side tests (gloo on CPU with a stand-in for the
    device library); production use leaves them at their defaults (the C-ABI library, CUDA)."""

    def __init__(self, problem: ControlProblem, terms, group=None, device: int | None = None, native=None,
                 buffer_device: str | None = None):
        terms, has_state = _costs._split(terms)
        if has_state and problem.initial_state is None:
            raise ValueError("state-transfer terms require problem.initial_state")
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        ks, kg = _set_sizes(problem, terms)
        self.n_traj = max(ks, kg)
        self.shard = shard_bounds(self.n_traj, self.rank, self.world)
        if device is None:
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        self.device = device
        if native is None:
            native = _costs.NativeProblem(problem, terms, problem.initial_state if has_state else None,
                                          problem.basis, device=device, shard=self.shard)
        self.native = native
        self.buffer_device = buffer_device or f"cuda:{device}"
        self._buf: torch.Tensor | None = None
        self._n_steps = -1
        self.calls = 0  # all-reduce calls made by the last evaluation

    def _lend(self, n_steps: int) -> torch.Tensor:
        if self._buf is None or n_steps != self._n_steps:
            self._buf = torch.zeros(self.native.raw_size(n_steps), dtype=torch.float64, device=self.buffer_device)
            self._n_steps = n_steps
            self.native.set_raw_buffer(self._buf.data_ptr(), self._buf.numel())
        if self._buf.is_cuda:
            self.native.set_stream(torch.cuda.current_stream(self._buf.device).cuda_stream)
        return self._buf

    def _hook(self, ptr: int, count: int) -> int:
        """Sum `count` doubles at `ptr` (inside the lent buffer) across the group, in place."""
        try:
            off = (ptr - self._buf.data_ptr()) // 8
            if off < 0 or off + count > self._buf.numel():
                return 1
            self._allreduce(self._buf[off:off + count])
            self.calls += 1
            return 0
        except Exception:  # noqa: BLE001 - reported to the library as a failed hook
            return 1

    def _allreduce(self, view: torch.Tensor) -> None:
        if self.world > 1:
            dist.all_reduce(view, op=dist.ReduceOp.SUM, group=self.group)

    def grad(self, a: ControlField) -> GradientResult:
        self._lend(a.n_steps)
        self.calls = 0
        return self.native.grad_sharded(a, self._hook)

    def cost(self, a: ControlField) -> float:
        self._lend(a.n_steps)
        self.calls = 0
        return self.native.cost_sharded(a, self._hook)


_CACHE: "OrderedDict[tuple, tuple]" = OrderedDict()


def _evaluator(problem, terms, group) -> ShardedEvaluator:
    key = (id(problem), tuple(id(t) for t in terms), id(group))
    hit = _CACHE.get(key)
    if hit is None:
        hit = (ShardedEvaluator(problem, terms, group), problem, tuple(terms))
        _CACHE[key] = hit
        while len(_CACHE) > 8:
            _CACHE.popitem(last=False)
    return hit[0]


def composite_grad_sharded(problem: ControlProblem, a: ControlField, terms, group=None) -> GradientResult:
    """``composite_grad`` (src/costs.py:515-546) with the trajectory block sharded over `group`.
    Collective: every rank of the group must call it with the same arguments."""
    _costs._check_field(problem, a)
    return _evaluator(problem, list(terms), group).grad(a)


def composite_cost_sharded(problem: ControlProblem, a: ControlField, terms, group=None) -> float:
    """``composite_cost`` (src/costs.py:549-597), sharded like composite_grad_sharded."""
    _costs._check_field(problem, a)
    return _evaluator(problem, list(terms), group).cost(a)


__all__ = ["ShardedEvaluator", "composite_cost_sharded", "composite_grad_sharded", "shard_bounds"]
