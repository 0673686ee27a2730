"""Time the DIAGONALIZATION backend on config c1's model (dense d = 40, N = 1000) next to the
Taylor path (CUDA-synchronised wall clock of composite_grad, median of 5)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dataclasses import replace  # noqa: E402

from paper_2304_06200_b200 import Backend, composite_grad, models  # noqa: E402

case = models.build_case("c1")
for backend in (Backend.SCALING_SQUARING, Backend.DIAGONALIZATION):
    prob = replace(case.problem, backend=backend)
    ts = []
    for _ in range(6):
        t0 = time.perf_counter()
        res = composite_grad(prob, case.field, case.terms)
        ts.append(time.perf_counter() - t0)
    print(f"{backend.value}: cost {res.cost:.15f}  median {1e3 * statistics.median(ts[1:]):.2f} ms")
