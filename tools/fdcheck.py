import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2304_06200_b200 import composite_grad, composite_cost, models
case = models.build_case("c3")
for rep in range(3):
    c = composite_cost(case.problem, case.field, case.terms)
    r = composite_grad(case.problem, case.field, case.terms)
    print(rep, c, r.cost, np.isnan(r.grad).sum(), flush=True)
