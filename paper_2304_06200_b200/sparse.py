"""Host-side operator containers (mirror of the reference's src/sparse.py API).

These are plain data holders used to *describe* a problem to the device
library: the layouts are exactly the reference's (CSR with int64 offsets and
indices, complex128 values, exact zeros dropped and duplicates summed at
construction, src/sparse.py:237-270; column-major dense, :152-170).  Every
numerical operation of an evaluation happens on the GPU; the helpers here
(construction, linear_combine, kron, Hermiticity checks) only build and
validate inputs, as ControlProblem does in the reference.

Objects that merely expose the reference's field names (``row_offsets``,
``col_indices``, ``values`` / ``array``) -- e.g. the reference's own
CsrMatrix -- are accepted everywhere too.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "SparseMatrixError",
    "CsrMatrix",
    "DenseMatrix",
    "build_csr_arrays",
    "build_csr",
    "from_dense",
    "identity_csr",
    "linear_combine",
    "matvec",
    "one_norm",
    "inf_norm",
    "max_row_nnz",
    "aux_embed",
    "is_anti_hermitian",
    "kron_csr",
    "is_hermitian",
    "to_dense",
    "frozen_copy",
    "as_own_matrix",
]


class SparseMatrixError(ValueError):
    """Malformed construction input or shape mismatch (src/sparse.py:37-38)."""


def frozen_copy(a, dtype=None, order="C"):
    """A private read-only copy: device problems are cached per Python object, so the arrays an
    object describes must not change behind the cache (in-place edits raise instead)."""
    out = np.array(a, dtype=dtype, order=order, copy=True)
    out.setflags(write=False)
    return out


@dataclass(frozen=True, eq=False)
class CsrMatrix:
    n_rows: int
    n_cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "row_offsets", frozen_copy(self.row_offsets, np.int64))
        object.__setattr__(self, "col_indices", frozen_copy(self.col_indices, np.int64))
        object.__setattr__(self, "values", frozen_copy(self.values, np.complex128))

    @property
    def nnz(self) -> int:
        return int(self.values.size)

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    # --- host-side descriptors with the reference's semantics (src/sparse.py:90-133); validation
    # and planning helpers, not the hot path (every matvec of an evaluation runs fused on the GPU)
    def col_abs_sums(self) -> np.ndarray:
        return np.bincount(self.col_indices, weights=np.abs(self.values), minlength=self.n_cols)

    def row_abs_sums(self) -> np.ndarray:
        sums = np.zeros(self.n_rows)
        if self.nnz:
            sums = np.add.reduceat(np.abs(self.values), np.minimum(self.row_offsets[:-1], self.nnz - 1))
            sums[self.row_offsets[:-1] == self.row_offsets[1:]] = 0.0
        return sums

    def row_nnz_counts(self) -> np.ndarray:
        return np.diff(self.row_offsets)

    def one_norm(self) -> float:
        return 0.0 if self.nnz == 0 else float(self.col_abs_sums().max())

    def inf_norm(self) -> float:
        return 0.0 if self.nnz == 0 else float(self.row_abs_sums().max())

    def max_row_nnz(self) -> int:
        return 0 if self.n_rows == 0 else int(self.row_nnz_counts().max())

    def scaled(self, factor: complex) -> "CsrMatrix":
        if factor == 0:
            return build_csr([], self.n_rows, self.n_cols)
        return CsrMatrix(self.n_rows, self.n_cols, self.row_offsets, self.col_indices, self.values * complex(factor))

    def matvec(self, v, out=None):
        """A v on the GPU (src/sparse.py:69-88); there is no host matvec."""
        return matvec(self, v, out)

    def triplets(self):
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_offsets))
        return rows, self.col_indices.copy(), self.values.copy()

    def conj_transpose(self) -> "CsrMatrix":
        r, c, v = self.triplets()
        return build_csr_arrays(c, r, np.conj(v), self.n_cols, self.n_rows)

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n_rows, self.n_cols), np.complex128, order="F")
        r, c, v = self.triplets()
        out[r, c] = v
        return out


@dataclass(frozen=True, eq=False)
class DenseMatrix:
    array: np.ndarray = field(repr=False)

    def __post_init__(self):
        arr = frozen_copy(self.array, np.complex128, order="F")
        if arr.ndim != 2:
            raise SparseMatrixError("DenseMatrix expects a 2-d array")
        if not np.isfinite(arr).all():
            raise SparseMatrixError("matrix entries must be finite")
        object.__setattr__(self, "array", arr)

    @property
    def n_rows(self):
        return self.array.shape[0]

    @property
    def n_cols(self):
        return self.array.shape[1]

    @property
    def shape(self):
        return self.array.shape

    @property
    def nnz(self):
        return self.array.size

    # --- host-side descriptors (src/sparse.py:201-227); Dense max_row_nnz is n_cols (:220-222)
    def col_abs_sums(self) -> np.ndarray:
        return np.abs(self.array).sum(axis=0)

    def row_abs_sums(self) -> np.ndarray:
        return np.abs(self.array).sum(axis=1)

    def row_nnz_counts(self) -> np.ndarray:
        return np.full(self.n_rows, self.n_cols, dtype=np.int64)

    def one_norm(self) -> float:
        return float(self.col_abs_sums().max()) if self.array.size else 0.0

    def inf_norm(self) -> float:
        return float(self.row_abs_sums().max()) if self.array.size else 0.0

    def max_row_nnz(self) -> int:
        return int(self.n_cols)

    def scaled(self, factor: complex) -> "DenseMatrix":
        return DenseMatrix(self.array * complex(factor))

    def matvec(self, v, out=None):
        """A v on the GPU (src/sparse.py:193-199); there is no host matvec."""
        return matvec(self, v, out)

    def to_dense(self) -> np.ndarray:
        return self.array.copy(order="F")

    def conj_transpose(self) -> "DenseMatrix":
        return DenseMatrix(self.array.conj().T)


def build_csr_arrays(rows, cols, vals, n_rows: int, n_cols: int) -> CsrMatrix:
    """COO -> CSR, duplicates summed in input order, exact zeros dropped."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.complex128)
    if not (rows.shape == cols.shape == vals.shape):
        raise SparseMatrixError("rows, cols and values must have equal length")
    if rows.size:
        if rows.min() < 0 or rows.max() >= n_rows or cols.min() < 0 or cols.max() >= n_cols:
            raise SparseMatrixError("index out of range")
        if not np.isfinite(vals).all():
            raise SparseMatrixError("matrix entries must be finite")
    keys = rows * np.int64(n_cols) + cols
    uniq, inv = np.unique(keys, return_inverse=True)
    summed = np.zeros(uniq.size, np.complex128)
    np.add.at(summed, inv, vals)
    keep = summed != 0
    uniq, summed = uniq[keep], summed[keep]
    offsets = np.zeros(n_rows + 1, np.int64)
    np.cumsum(np.bincount(uniq // n_cols, minlength=n_rows), out=offsets[1:])
    return CsrMatrix(n_rows, n_cols, offsets, (uniq % n_cols).astype(np.int64), summed)


def build_csr(triplets, n_rows: int, n_cols: int) -> CsrMatrix:
    entries = list(triplets)
    if not entries:
        return build_csr_arrays(np.empty(0), np.empty(0), np.empty(0), n_rows, n_cols)
    r, c, v = zip(*entries)
    return build_csr_arrays(r, c, v, n_rows, n_cols)


def from_dense(array) -> CsrMatrix:
    a = np.asarray(array, np.complex128)
    r, c = np.nonzero(a)
    return build_csr_arrays(r, c, a[r, c], a.shape[0], a.shape[1])


def identity_csr(n: int) -> CsrMatrix:
    i = np.arange(n, dtype=np.int64)
    return build_csr_arrays(i, i, np.ones(n, np.complex128), n, n)


def as_own_matrix(m):
    """This package's (immutable) matrix type for any object with the reference's field names."""
    if isinstance(m, (CsrMatrix, DenseMatrix)):
        return m
    if hasattr(m, "array"):
        return DenseMatrix(m.array)
    return CsrMatrix(int(m.n_rows), int(m.n_cols), m.row_offsets, m.col_indices, m.values)


def to_dense(m) -> np.ndarray:
    if hasattr(m, "array"):
        return np.asarray(m.array)
    return m.to_dense()


def linear_combine(coeffs, mats):
    """sum_i coeffs[i] mats[i] with the reference's operand order (src/sparse.py:313-349)."""
    mats = list(mats)
    coeffs = [complex(c) for c in coeffs]
    if len(coeffs) != len(mats) or not mats:
        raise SparseMatrixError("need one coefficient per matrix")
    shape = mats[0].shape
    if any(m.shape != shape for m in mats):
        raise SparseMatrixError("shape mismatch in linear_combine")
    if any(isinstance(m, DenseMatrix) for m in mats):
        total = np.zeros(shape, np.complex128, order="F")
        for c, m in zip(coeffs, mats):
            if c != 0:
                total += to_dense(m) * c
        return DenseMatrix(total)
    rs, cs, vs = [], [], []
    for c, m in zip(coeffs, mats):
        if c == 0 or m.nnz == 0:
            continue
        r, k, v = m.triplets()
        rs.append(r)
        cs.append(k)
        vs.append(c * v)
    if not rs:
        return build_csr([], *shape)
    return build_csr_arrays(np.concatenate(rs), np.concatenate(cs), np.concatenate(vs), *shape)


def matvec(m, v, out=None):
    """A v (or A applied to every row of a (K, n) block) evaluated on the GPU through the C ABI's
    ``lg_matvec`` -- the ELL row kernel of the sweeps; mirrors ``sparse.matvec`` / ``CsrMatrix.matvec`` /
    ``DenseMatrix.matvec`` (src/sparse.py:69-88,193-199,297-298).  Square matrices (the library's
    descriptor); raises without the library or a GPU -- there is no host product."""
    import ctypes as C

    from . import _native
    from .costs import _Keep, _matrix

    m = as_own_matrix(m)
    n_rows, n_cols = m.shape
    x = np.asarray(v, dtype=np.complex128)
    if x.ndim not in (1, 2) or x.shape[-1] != n_cols:
        raise SparseMatrixError("matvec dimension mismatch")
    if n_rows != n_cols:
        raise NotImplementedError("device matvec serves square matrices (lg_matrix)")
    rows = np.ascontiguousarray(x.reshape(-1, n_cols))
    res = np.empty_like(rows)
    keep = _Keep()
    desc = _matrix(m, n_rows, keep)
    _native.check(_native.load().lg_matvec(C.byref(desc), rows.shape[0], _native.dptr(rows.view(np.float64)),
                                           _native.dptr(res.view(np.float64)), 0))
    res = res.reshape(x.shape)
    if out is not None:
        if out.shape != res.shape:
            raise SparseMatrixError("out has the wrong shape")
        np.copyto(out, res)
        return out
    return res


def one_norm(m) -> float:
    """Module-level accessors of the reference (src/sparse.py:301-310)."""
    return as_own_matrix(m).one_norm()


def inf_norm(m) -> float:
    return as_own_matrix(m).inf_norm()


def max_row_nnz(m) -> int:
    return as_own_matrix(m).max_row_nnz()


def aux_embed(h_step, h_control, dt: float):
    """[[-i dt H, -i dt h_c], [0, -i dt H]] as a stored matrix (src/sparse.py:352-380): dense when
    either block is dense, CSR otherwise, entries scaled by -i dt in one multiplication each."""
    h_step, h_control = as_own_matrix(h_step), as_own_matrix(h_control)
    d = h_step.shape[0]
    if h_step.shape != h_control.shape or h_step.shape[1] != d:
        raise SparseMatrixError("aux_embed expects two square matrices of equal dimension")
    scale = -1j * dt
    if isinstance(h_step, DenseMatrix) or isinstance(h_control, DenseMatrix):
        big = np.zeros((2 * d, 2 * d), np.complex128, order="F")
        big[:d, :d] = scale * to_dense(h_step)
        big[:d, d:] = scale * to_dense(h_control)
        big[d:, d:] = big[:d, :d]
        return DenseMatrix(big)
    hr, hc, hv = h_step.triplets()
    cr, cc, cv = h_control.triplets()
    return build_csr_arrays(np.concatenate([hr, cr, hr + d]), np.concatenate([hc, cc + d, hc + d]),
                            scale * np.concatenate([hv, cv, hv]), 2 * d, 2 * d)


def is_anti_hermitian(m, tol: float) -> bool:
    """max |M + M^dagger| <= tol (src/sparse.py:400-404)."""
    m = as_own_matrix(m)
    if m.shape[0] != m.shape[1]:
        return False
    dense = to_dense(m)
    return float(np.max(np.abs(dense + dense.conj().T), initial=0.0)) <= tol


def kron_csr(a: CsrMatrix, b: CsrMatrix) -> CsrMatrix:
    ra, ca, va = a.triplets()
    rb, cb, vb = b.triplets()
    rows = (ra[:, None] * b.n_rows + rb[None, :]).ravel()
    cols = (ca[:, None] * b.n_cols + cb[None, :]).ravel()
    vals = (va[:, None] * vb[None, :]).ravel()
    return build_csr_arrays(rows, cols, vals, a.n_rows * b.n_rows, a.n_cols * b.n_cols)


def is_hermitian(m, tol: float) -> bool:
    """max |M - M^dagger| <= tol (src/sparse.py:393-397)."""
    if m.shape[0] != m.shape[1]:
        return False
    if isinstance(m, DenseMatrix) or hasattr(m, "array"):
        a = np.asarray(m.array)
        return float(np.abs(a - a.conj().T).max()) <= tol if a.size else True
    diff = linear_combine([1.0, -1.0], [m, m.conj_transpose()])
    return (float(np.abs(diff.values).max()) if diff.nnz else 0.0) <= tol


def one_norm_host(m) -> float:
    """max column abs sum, for host-side validation tolerances only."""
    if isinstance(m, DenseMatrix) or hasattr(m, "array"):
        a = np.asarray(m.array)
        return float(np.abs(a).sum(axis=0).max()) if a.size else 0.0
    if m.nnz == 0:
        return 0.0
    return float(np.bincount(m.col_indices, weights=np.abs(m.values), minlength=m.n_cols).max())
