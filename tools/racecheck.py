"""Repeat the c3 golden-prefix gradient and count non-finite / mismatching results (race hunting)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import _golden as G  # noqa: E402
from paper_2304_06200_b200 import ControlField, ControlProblem, CostKind, CostTerm  # noqa: E402
from paper_2304_06200_b200.costs import NativeProblem  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
z = G.load("c3")
hs, hc = G.mats(z)
prob = ControlProblem(hs, tuple(hc), initial_state=z["psi0"])
a = ControlField(z["amps"].shape[0], 2, float(z["dt"]), z["amps"])
terms = [CostTerm(CostKind.STATE_INFIDELITY, 1.0, target_state=z["targets"])]
bad = bad_c = bad_gc = bad_g = 0
for r in range(reps):
    npb = NativeProblem(prob, terms, initial_states=z["psi0"])
    res = npb.grad(a)
    c = npb.cost(a)
    e_c = abs(c - float(z["cost"])) > 1e-12 or not np.isfinite(c)
    e_gc = abs(res.cost - float(z["cost"])) > 1e-12 or not np.isfinite(res.cost)
    e_g = not (G.grad_rel(res.grad, z["grad"]) <= 1e-9)
    bad_c += e_c
    bad_gc += e_gc
    bad_g += e_g
    bad += e_c or e_gc or e_g
    del npb
print(f"{os.environ.get('TAG', '')}: {bad} bad of {reps} (forward-only cost {bad_c}, grad-call cost {bad_gc}, grad {bad_g})")
