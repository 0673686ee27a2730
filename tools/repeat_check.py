"""Repeat one config's evaluation and count results that differ bit-wise from the first (race hunting).

    python tools/repeat_check.py [c2] [repeats] [n_steps|full]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_06200_b200 import composite_grad, models  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
n = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "full" else None
case = models.build_case(name, n_steps=n)
ref = composite_grad(case.problem, case.field, case.terms)
bad = 0
for _ in range(reps):
    r = composite_grad(case.problem, case.field, case.terms)
    if r.cost != ref.cost or not np.array_equal(r.grad, ref.grad) or not np.isfinite(r.grad).all():
        bad += 1
print(f"{name}: {bad} of {reps} repeats differ from the first (cost {ref.cost!r})")
