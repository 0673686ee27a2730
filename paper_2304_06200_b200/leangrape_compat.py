"""Drop-in shim for the reference package ``leangrape``: its optimiser evaluates on the B200.

The reference binds ``composite_grad`` / ``composite_cost`` at import
(``src/optimizer.py:18``) and calls them at ``src/optimizer.py:117,150,159,169``.
``enable()`` rebinds those two names in ``leangrape.optimizer`` to the functions
below, which convert the reference's objects (``ControlProblem``, ``ControlField``,
``CostTerm`` -- field names identical to this package's mirror classes,
``src/costs.py:64-168``) and evaluate through the C ABI.

Conversions are memoised per reference object (the object is kept alive next to
its conversion, so its ``id`` cannot be reused), so repeated calls on one problem
hit the device-problem cache (``costs._native_for``) instead of re-uploading the
operators on every call.  The converted objects hold private read-only copies of
the arrays (``sparse.frozen_copy``): an in-place edit of a reference array after
the first call is not seen -- build a new reference object instead, as the
reference's frozen dataclasses intend.
"""

from __future__ import annotations

from collections import OrderedDict

from . import costs as _b

__all__ = ["convert_problem", "convert_terms", "convert_field", "composite_grad", "composite_cost", "enable",
           "disable"]

_MEMO: "OrderedDict[tuple, tuple]" = OrderedDict()
_MEMO_SIZE = 32


def _memo(key, keep, build):
    hit = _MEMO.get(key)
    if hit is not None:
        _MEMO.move_to_end(key)
        return hit[1]
    val = build()
    _MEMO[key] = (keep, val)
    while len(_MEMO) > _MEMO_SIZE:
        _MEMO.popitem(last=False)
    return val


def convert_problem(p) -> _b.ControlProblem:
    """leangrape ControlProblem -> mirror ControlProblem (src/costs.py:96-138)."""
    if isinstance(p, _b.ControlProblem):
        return p
    return _memo(("problem", id(p)), p, lambda: _b.ControlProblem(
        p.h_static, tuple(p.h_controls), _b.Backend(p.backend.value), float(p.tau), p.initial_state,
        None if p.basis is None else tuple(p.basis)))


def convert_terms(terms) -> list:
    """leangrape CostTerm list -> mirror CostTerm list (src/costs.py:141-168)."""
    terms = list(terms)
    if all(isinstance(t, _b.CostTerm) for t in terms):
        return terms

    def one(t):
        if isinstance(t, _b.CostTerm):
            return t
        return _memo(("term", id(t)), t, lambda: _b.CostTerm(
            _b.CostKind(t.kind.value), float(t.weight), t.target_state, t.target_gate, t.penalty_op))

    # the same list of converted objects every time, so _native_for's key (ids of the terms) repeats
    return _memo(("terms",) + tuple(id(t) for t in terms), tuple(terms), lambda: [one(t) for t in terms])


def convert_field(a) -> _b.ControlField:
    """leangrape ControlField -> mirror ControlField (cheap; not memoised: fields change every step)."""
    if isinstance(a, _b.ControlField):
        return a
    return _b.ControlField(int(a.n_steps), int(a.n_channels), float(a.dt), a.amplitudes)


def _to_reference_result(res, ref_result_type):
    if ref_result_type is None:
        return res
    return ref_result_type(cost=res.cost, grad=res.grad, live_vector_peak=res.live_vector_peak)


_RESULT_TYPE = None  # leangrape.costs.GradientResult once enable() has seen the module


def composite_grad(problem, a, terms):
    """``leangrape.costs.composite_grad`` (src/costs.py:515-546) on the GPU."""
    res = _b.composite_grad(convert_problem(problem), convert_field(a), convert_terms(terms))
    return _to_reference_result(res, _RESULT_TYPE)


def composite_cost(problem, a, terms) -> float:
    """``leangrape.costs.composite_cost`` (src/costs.py:549-597) on the GPU."""
    return _b.composite_cost(convert_problem(problem), convert_field(a), convert_terms(terms))


_SAVED: dict = {}


def enable(optimizer_module=None):
    """Rebind ``composite_grad`` / ``composite_cost`` in ``leangrape.optimizer`` (or the given
    module): ``grape_optimize`` then evaluates every cost and gradient on the GPU."""
    global _RESULT_TYPE
    if optimizer_module is None:
        import leangrape.optimizer as optimizer_module  # noqa: PLC0415 - the reference, when installed
    costs_mod = None
    try:
        import sys

        costs_mod = sys.modules.get(optimizer_module.__name__.rsplit(".", 1)[0] + ".costs")
    except Exception:  # noqa: BLE001
        costs_mod = None
    _RESULT_TYPE = getattr(costs_mod, "GradientResult", None)
    _SAVED[id(optimizer_module)] = (optimizer_module, optimizer_module.composite_grad,
                                    optimizer_module.composite_cost)
    optimizer_module.composite_grad = composite_grad
    optimizer_module.composite_cost = composite_cost
    return optimizer_module


def disable(optimizer_module=None):
    """Undo ``enable``."""
    global _RESULT_TYPE
    if optimizer_module is None:
        import leangrape.optimizer as optimizer_module  # noqa: PLC0415
    saved = _SAVED.pop(id(optimizer_module), None)
    if saved is not None:
        optimizer_module.composite_grad, optimizer_module.composite_cost = saved[1], saved[2]
    if not _SAVED:
        _RESULT_TYPE = None
