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

# Above d = 64: the global-memory Jacobi + batched products against the cuSOLVER / cuBLAS A/B path
# (LG_DIAG_LIB=1) on the transmon-cavity model, one control, C1^st.
import numpy as np  # noqa: E402

from paper_2304_06200_b200 import ControlField, ControlProblem, CostKind, CostTerm  # noqa: E402
from paper_2304_06200_b200.costs import NativeProblem  # noqa: E402

for nt, nc, N in ((4, 24, 200), (4, 64, 100)):
    h_s, hx, _ = models.transmon_cavity_ops(nt, nc)
    d = nt * nc
    rng = np.random.default_rng(5)
    amps = rng.uniform(-0.5, 0.5, (N, 1))
    psi0 = np.zeros(d, complex)
    psi0[0] = 1.0
    tgt = np.zeros(d, complex)
    tgt[1] = 1.0
    prob = ControlProblem(h_s, (hx,), backend=Backend.DIAGONALIZATION, initial_state=psi0)
    terms = [CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=tgt)]
    a = ControlField(N, 1, 0.5, amps)
    for lib in (False, True):
        if lib:
            os.environ["LG_DIAG_LIB"] = "1"
        else:
            os.environ.pop("LG_DIAG_LIB", None)
        npb = NativeProblem(prob, terms, initial_states=psi0[None])
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            res = npb.grad(a)
            ts.append(time.perf_counter() - t0)
        print(f"d={d} N={N} {npb.diag_solver} [{npb.engine}]: cost {res.cost:.15f}  median "
              f"{1e3 * statistics.median(ts[1:]):.2f} ms")
os.environ.pop("LG_DIAG_LIB", None)
