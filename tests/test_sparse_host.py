"""Host-side matrix helpers of the mirror (paper_2304_06200_b200.sparse) against the reference's own
(src/sparse.py, imported from /root/reference when present -- the build container; skipped
elsewhere): these are the data formats either side of the device path, and the norms among them feed
the planner, so stored patterns, values and descriptors must be the reference's bit for bit.  CPU only."""

import os
import sys

import numpy as np
import pytest

from paper_2304_06200_b200 import sparse as S

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


@pytest.fixture(scope="module")
def R():
    sys.path.insert(0, REF)
    try:
        import leangrape.sparse as sparse
    finally:
        sys.path.remove(REF)
    return sparse


def _same_csr(mine, theirs):
    assert (mine.n_rows, mine.n_cols) == (theirs.n_rows, theirs.n_cols)
    assert np.array_equal(mine.row_offsets, theirs.row_offsets)
    assert np.array_equal(mine.col_indices, theirs.col_indices)
    assert np.array_equal(mine.values, theirs.values)


def _random_triplets(g, n_rows, n_cols, count):
    rows = g.integers(0, n_rows, count)
    cols = g.integers(0, n_cols, count)
    vals = g.standard_normal(count) + 1j * g.standard_normal(count)
    return rows, cols, vals


@pytest.mark.parametrize("seed", range(4))
def test_builders_sum_duplicates_and_order_like_the_reference(R, seed):
    g = np.random.default_rng(seed)
    n_rows, n_cols = int(g.integers(1, 9)), int(g.integers(1, 9))
    rows, cols, vals = _random_triplets(g, n_rows, n_cols, int(g.integers(0, 40)))
    _same_csr(S.build_csr_arrays(rows, cols, vals, n_rows, n_cols), R.build_csr_arrays(rows, cols, vals, n_rows, n_cols))
    trip = list(zip(rows.tolist(), cols.tolist(), vals.tolist()))
    _same_csr(S.build_csr(trip, n_rows, n_cols), R.build_csr(trip, n_rows, n_cols))
    dense = g.standard_normal((n_rows, n_cols)) * (g.random((n_rows, n_cols)) < 0.4)
    _same_csr(S.from_dense(dense), R.from_dense(dense))
    _same_csr(S.identity_csr(n_rows), R.identity_csr(n_rows))


@pytest.mark.parametrize("seed", range(4))
def test_descriptors_scaling_transpose_and_combination(R, seed):
    g = np.random.default_rng(100 + seed)
    n = int(g.integers(2, 12))
    rows, cols, vals = _random_triplets(g, n, n, int(g.integers(1, 5 * n)))
    mine, theirs = S.build_csr_arrays(rows, cols, vals, n, n), R.build_csr_arrays(rows, cols, vals, n, n)
    for name in ("col_abs_sums", "row_abs_sums", "row_nnz_counts"):
        assert np.array_equal(getattr(mine, name)(), getattr(theirs, name)()), name
    assert (mine.one_norm(), mine.inf_norm(), mine.max_row_nnz()) == (theirs.one_norm(), theirs.inf_norm(),
                                                                     theirs.max_row_nnz())
    assert (S.one_norm(mine), S.inf_norm(mine), S.max_row_nnz(mine)) == (R.one_norm(theirs), R.inf_norm(theirs),
                                                                        R.max_row_nnz(theirs))
    _same_csr(mine.scaled(-0.3j), theirs.scaled(-0.3j))
    _same_csr(mine.scaled(0.0), theirs.scaled(0.0))
    _same_csr(mine.conj_transpose(), theirs.conj_transpose())
    assert np.array_equal(mine.to_dense(), theirs.to_dense())
    r2, c2, v2 = _random_triplets(g, n, n, 2 * n)
    other_m, other_t = S.build_csr_arrays(r2, c2, v2, n, n), R.build_csr_arrays(r2, c2, v2, n, n)
    for coeffs in ([1.0, 0.25], [1.0, 0.0], [0.0, 0.0], [-1.5, 2.0 + 0.5j]):
        _same_csr(S.linear_combine(coeffs, [mine, other_m]), R.linear_combine(coeffs, [theirs, other_t]))
    _same_csr(S.kron_csr(mine, other_m), R.kron_csr(theirs, other_t)) if hasattr(R, "kron_csr") else None
    herm = mine.to_dense() + mine.to_dense().conj().T
    hm, ht = S.from_dense(herm), R.from_dense(herm)
    assert S.is_hermitian(hm, 1e-12) == R.is_hermitian(ht, 1e-12) is True
    assert S.is_hermitian(mine, 1e-12) == R.is_hermitian(theirs, 1e-12)
    assert S.is_anti_hermitian(hm.scaled(1j), 1e-12) == R.is_anti_hermitian(ht.scaled(1j), 1e-12) is True
    assert S.is_anti_hermitian(hm, 1e-12) == R.is_anti_hermitian(ht, 1e-12)


def test_dense_matrix_descriptors_and_embedding(R):
    g = np.random.default_rng(9)
    n = 7
    a = g.standard_normal((n, n)) + 1j * g.standard_normal((n, n))
    a = a + a.conj().T
    mine, theirs = S.DenseMatrix(a), R.DenseMatrix(np.asfortranarray(a))
    assert np.array_equal(mine.col_abs_sums(), theirs.col_abs_sums())
    assert np.array_equal(mine.row_abs_sums(), theirs.row_abs_sums())
    assert (mine.one_norm(), mine.inf_norm(), mine.max_row_nnz(), mine.nnz) == (theirs.one_norm(), theirs.inf_norm(),
                                                                               theirs.max_row_nnz(), theirs.nnz)
    assert np.array_equal(mine.scaled(-0.2j).to_dense(), theirs.scaled(-0.2j).to_dense())
    ctrl = g.standard_normal((n, n)) * (g.random((n, n)) < 0.3)
    ctrl = ctrl + ctrl.T
    em = S.aux_embed(mine, S.from_dense(ctrl), 0.3)
    et = R.aux_embed(theirs, R.from_dense(ctrl), 0.3)
    assert np.array_equal(S.to_dense(em), et.to_dense())
    assert (em.one_norm(), em.inf_norm(), em.max_row_nnz()) == (et.one_norm(), et.inf_norm(), et.max_row_nnz())
    mixed = S.linear_combine([1.0, 0.5], [mine, S.from_dense(ctrl)])
    mixed_t = R.linear_combine([1.0, 0.5], [theirs, R.from_dense(ctrl)])
    assert np.array_equal(S.to_dense(mixed), mixed_t.to_dense())


def test_shape_errors_are_value_errors(R):
    with pytest.raises(ValueError):
        S.linear_combine([1.0], [S.identity_csr(2), S.identity_csr(2)])
    with pytest.raises(ValueError):
        S.linear_combine([1.0, 1.0], [S.identity_csr(2), S.identity_csr(3)])
    with pytest.raises(ValueError):
        S.aux_embed(S.identity_csr(2), S.identity_csr(3), 0.1)
    assert issubclass(S.SparseMatrixError, ValueError) and issubclass(R.SparseMatrixError, ValueError)
