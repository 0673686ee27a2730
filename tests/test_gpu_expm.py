"""GPU: standalone certified action exp(A) psi (expm.apply / expm.expm_multiply, src/expm.py:306-369)
through the C ABI (lg_expm_apply), against the reference's own outputs (tests/golden/expm.npz) and the
properties the reference tests check (tests/test_expm_apply.py): identity for the zero generator, the
sigma_x rotation, certified accuracy against a diagonalisation oracle over a tau panel, unitarity,
the inverse property, and input validation."""

import numpy as np
import pytest
import scipy.linalg

import _golden as G
from paper_2304_06200_b200 import expm, sparse
from test_expm_host import TAGS, golden_matrix, n_taus

pytestmark = pytest.mark.gpu


def anti(rng, d, scale=1.0):
    g = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
    return scale * (g - g.conj().T) / 2.0


def state(rng, d):
    z = rng.standard_normal(d) + 1j * rng.standard_normal(d)
    return z / np.linalg.norm(z)


@pytest.mark.parametrize("tag", TAGS)
def test_matches_reference_expm_multiply(tag):
    z = G.sub(G.load("expm"), tag)
    a = golden_matrix(z)
    for i in range(n_taus(z)):
        tau = float(z[f"tau{i}"])
        for h in range(z["psi"].shape[0]):
            out, mu = expm.expm_multiply(a, z["psi"][h], tau)
            want = z[f"out{i}"][h]
            assert mu == int(z[f"mu{i}"])
            assert np.linalg.norm(out - want) <= 1e-13 * max(np.linalg.norm(want), 1.0)
        # the whole block in one call
        plan = expm.make_plan(*expm.plan_inputs(a), tau)
        blk = expm.apply(a, z["psi"], plan)
        assert np.linalg.norm(blk - z[f"out{i}"]) <= 1e-13 * max(np.linalg.norm(z[f"out{i}"]), 1.0)


def test_zero_generator_and_rotation():
    rng = np.random.default_rng(1)
    a = sparse.build_csr([], 6, 6)
    psi = state(rng, 6)
    out, mu = expm.expm_multiply(a, psi, 1e-8)
    assert mu == 1 and np.allclose(out, psi, atol=1e-14)
    rot = sparse.build_csr([(0, 1, -1j * np.pi / 2), (1, 0, -1j * np.pi / 2)], 2, 2)
    out, mu = expm.expm_multiply(rot, np.array([1.0, 0.0], complex), 1e-10)
    assert np.linalg.norm(out - np.array([0.0, -1j])) <= 1e-10 and mu >= 1


@pytest.mark.parametrize("tau", [1e-4, 1e-8, 1e-12])
def test_certified_accuracy_panel(tau):
    rng = np.random.default_rng(int(-np.log10(tau)))
    for _ in range(10):
        d = int(rng.integers(4, 33))
        dense = anti(rng, d)
        a = sparse.from_dense(dense)
        dense *= float(rng.uniform(0.5, 18.0)) / expm.plan_inputs(a)[0]
        a = sparse.from_dense(dense)
        psi = state(rng, d)
        plan = expm.make_plan(*expm.plan_inputs(a), tau)
        out = expm.apply(a, psi, plan)
        want = scipy.linalg.expm(dense) @ psi
        assert np.linalg.norm(out - want) / np.linalg.norm(want) <= tau


def test_unitarity_and_inverse():
    rng = np.random.default_rng(3)
    for _ in range(10):
        d = int(rng.integers(4, 25))
        dense = anti(rng, d, 1.2)
        a, neg = sparse.from_dense(dense), sparse.from_dense(-dense)
        psi = state(rng, d)
        out, _ = expm.expm_multiply(a, psi, 1e-9)
        assert abs(np.linalg.norm(out) - 1.0) <= 2e-9
        plan = expm.make_plan(*expm.plan_inputs(a), 1e-10)
        back = expm.apply(neg, expm.apply(a, psi, plan), plan)
        assert np.linalg.norm(back - psi) <= 4e-10


def test_dense_generator_and_validation():
    rng = np.random.default_rng(5)
    dense = anti(rng, 20, 0.7)
    a = sparse.DenseMatrix(np.asfortranarray(dense))
    psi = state(rng, 20)
    out, _ = expm.expm_multiply(a, psi, 1e-12)
    assert np.linalg.norm(out - scipy.linalg.expm(dense) @ psi) <= 1e-12
    bad = sparse.from_dense(rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4)))
    plan = expm.make_plan(*expm.plan_inputs(bad), 1e-8)
    with pytest.raises(ValueError, match="anti-Hermitian"):
        expm.apply(bad, state(rng, 4), plan)
    with pytest.raises(ValueError):
        expm.apply(sparse.from_dense(anti(rng, 4)), np.zeros(5, complex), plan)
