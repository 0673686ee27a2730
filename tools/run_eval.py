"""Run a few evaluations of one config (for ncu / timing runs on the GPU box).

    python tools/run_eval.py c2 [n_steps] [repeats]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2304_06200_b200 import composite_grad, models  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "full" else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
case = models.build_case(name, n_steps=n)
for r in range(reps):
    t0 = time.perf_counter()
    res = composite_grad(case.problem, case.field, case.terms)
    print(f"{name} N={case.field.n_steps} eval {r}: {1e3 * (time.perf_counter() - t0):.2f} ms cost={res.cost:.15f}")
