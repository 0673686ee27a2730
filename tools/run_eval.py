"""Run a few evaluations of one config (for ncu / timing runs on the GPU box).

    python tools/run_eval.py c2 [n_steps|full] [repeats] [n_states]

Prints wall time per evaluation, the engine the library chose and the device
phase split (CUDA events on the library stream) of the timed repeats.
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2304_06200_b200 import _native, composite_grad, models  # noqa: E402
from paper_2304_06200_b200.costs import _native_for, _split  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "full" else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
ns = int(sys.argv[4]) if len(sys.argv) > 4 else None
case = models.build_case(name, n_steps=n, n_states=ns)
p = case.problem
npb = None
for r in range(reps):
    t0 = time.perf_counter()
    res = composite_grad(case.problem, case.field, case.terms)
    ms = 1e3 * (time.perf_counter() - t0)
    if npb is None:
        terms, has_state = _split(case.terms)
        npb = _native_for(p, terms, p.initial_state if has_state else None, p.basis)
        lib = _native.load()
        lib.lg_set_timing(npb.handle, 1)
    print(f"{name} N={case.field.n_steps} eval {r}: {ms:.2f} ms cost={res.cost:.15f}")
if npb is not None and reps > 1:
    phase = np.zeros(4)
    nev = np.zeros(1, np.int64)
    _native.check(lib.lg_get_timing(npb.handle, _native.dptr(phase), _native.i64ptr(nev)))
    k = max(int(nev[0]), 1)
    print(f"{name} engine={lib.lg_engine_name(npb.handle).decode()} phases ms/eval: prep_plans {phase[0] / k:.3f} "
          f"forward {phase[1] / k:.3f} backward {phase[2] / k:.3f} finalize {phase[3] / k:.3f}")
