"""Standalone certified action, host side (no GPU): the planner inputs the library computes for a
generator (lg_expm_plan_inputs: A.one_norm() in numpy's reduction order, A.max_row_nnz()) and the
resulting plans are bit-identical to the reference's (tests/golden/expm.npz, written by
make_golden.py from leangrape.expm), and the oracle's Taylor recursion reproduces the reference's
expm_multiply outputs."""

import numpy as np
import pytest

import _golden as G
from oracle import lg_oracle as O
from paper_2304_06200_b200 import CsrMatrix, DenseMatrix
from paper_2304_06200_b200.expm import make_plan, plan_inputs

TAGS = ["csr16", "dense12", "rot", "zero", "band1200"]


def golden_matrix(z, kind="product"):
    if "a_dense" in z:
        a = np.asfortranarray(z["a_dense"])
        return DenseMatrix(a) if kind == "product" else O.Dense(a)
    ip, ix, dv = z["a_indptr"], z["a_indices"], z["a_data"]
    n = ip.size - 1
    return CsrMatrix(n, n, ip, ix, dv) if kind == "product" else O.Csr(n, ip, ix, dv)


def n_taus(z):
    return sum(1 for k in z if k.startswith("tau"))


@pytest.mark.parametrize("tag", TAGS)
def test_plan_inputs_and_plans_bit_exact(tag):
    z = G.sub(G.load("expm"), tag)
    norm1, sp = plan_inputs(golden_matrix(z))
    assert norm1 == float(z["norm1"]) and sp == int(z["sp"])
    for i in range(n_taus(z)):
        p = make_plan(norm1, sp, float(z[f"tau{i}"]))
        assert (p.order, p.scaling) == (int(z[f"m{i}"]), int(z[f"s{i}"]))
        assert p.matvecs == int(z[f"mu{i}"])


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_action_matches_reference(tag):
    z = G.sub(G.load("expm"), tag)
    a = golden_matrix(z, "oracle")
    for i in range(n_taus(z)):
        m, s = int(z[f"m{i}"]), int(z[f"s{i}"])
        for h in range(z["psi"].shape[0]):
            got = O.taylor_apply(lambda v: O.matvec(a, v), z["psi"][h], m, s)
            want = z[f"out{i}"][h]
            assert np.linalg.norm(got - want) <= 1e-14 * max(np.linalg.norm(want), 1.0)
