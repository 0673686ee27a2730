"""``sparse.matvec`` / ``CsrMatrix.matvec`` / ``DenseMatrix.matvec`` (src/sparse.py:69-88,193-199,
297-298) on the device through the C ABI's ``lg_matvec``: against numpy's dense product (1e-13
relative: the row sums run in ELL slot order, not numpy's), with blocks of vectors, ``out=``, an empty
matrix, more than 64 vectors (one launch handles 64) and the error conventions."""

import numpy as np
import pytest

from paper_2304_06200_b200 import sparse as S

pytestmark = pytest.mark.gpu


def _cvec(g, *shape):
    return g.standard_normal(shape) + 1j * g.standard_normal(shape)


@pytest.mark.parametrize("n,density", [(1, 1.0), (17, 0.3), (300, 0.02)])
def test_csr_matvec_matches_dense_product(n, density):
    g = np.random.default_rng(n)
    a = _cvec(g, n, n) * (g.random((n, n)) < density)
    m = S.from_dense(a)
    x = _cvec(g, n)
    want = a @ x
    got = m.matvec(x)
    assert np.abs(got - want).max() <= 1e-13 * max(1.0, np.abs(want).max())
    assert np.array_equal(S.matvec(m, x), got)
    out = np.empty(n, complex)
    assert m.matvec(x, out=out) is out and np.array_equal(out, got)


def test_dense_matvec_and_blocks_of_vectors():
    g = np.random.default_rng(3)
    n, k = 48, 70  # more than the 64 vectors of one launch
    a = _cvec(g, n, n)
    xs = _cvec(g, k, n)
    got = S.DenseMatrix(a).matvec(xs)
    want = xs @ a.T
    assert got.shape == (k, n)
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()


def test_empty_matrix_gives_zeros_and_shapes_are_checked():
    g = np.random.default_rng(4)
    assert np.array_equal(S.build_csr([], 5, 5).matvec(_cvec(g, 5)), np.zeros(5, complex))
    with pytest.raises(ValueError):
        S.identity_csr(4).matvec(_cvec(g, 5))
    with pytest.raises(ValueError):
        S.identity_csr(4).matvec(_cvec(g, 4), out=np.empty(3, complex))
    with pytest.raises(NotImplementedError):
        S.build_csr([(0, 1, 1.0)], 2, 3).matvec(_cvec(g, 3))
