"""The package's config builders reproduce the reference-built matrices bit-for-bit,
and the Python API validates inputs like the reference (src/costs.py:64-168)."""

import numpy as np
import pytest

import _golden as G
from paper_2304_06200_b200 import CostKind, CostTerm, ControlField, ControlProblem, models
from paper_2304_06200_b200.sparse import CsrMatrix, DenseMatrix, build_csr_arrays


def _same(m, z, prefix):
    if isinstance(m, DenseMatrix):
        assert np.array_equal(m.array, z[prefix + "_dense"])
    else:
        assert np.array_equal(m.row_offsets, z[prefix + "_indptr"])
        assert np.array_equal(m.col_indices, z[prefix + "_indices"])
        assert np.array_equal(m.values, z[prefix + "_data"])


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_builders_bit_identical(name):
    z = G.load(name)
    case = models.build_case(name, n_steps=int(z["amps"].shape[0]))
    _same(case.problem.h_static, z, "hs")
    for k, h in enumerate(case.problem.h_controls):
        _same(h, z, f"hc{k}")
    assert np.array_equal(case.field.amplitudes, z["amps"])
    assert case.field.dt == float(z["dt"])


def test_c5_scales_reproduce_reference():
    z = G.load("c5")
    assert models.C5_SCALES == (float(z["scale_hs"]), float(z["scale_hc"]))


def test_control_field_validation():
    with pytest.raises(ValueError):
        ControlField(3, 1, 0.1, np.zeros((2, 1)))
    with pytest.raises(ValueError):
        ControlField(1, 1, 0.0, np.zeros((1, 1)))
    with pytest.raises(ValueError):
        ControlField(1, 1, 0.1, np.array([[np.nan]]))
    f = ControlField.constant(0.5, 4, 2, 0.1)
    assert f.replace_amplitudes(np.ones((4, 2))).amplitudes.sum() == 8


def test_problem_and_term_validation():
    d = 4
    h = build_csr_arrays([0, 1], [1, 0], [1.0, 1.0], d, d)
    bad = build_csr_arrays([0], [1], [1.0], d, d)
    with pytest.raises(ValueError, match="Hermitian"):
        ControlProblem(bad, (h,))
    with pytest.raises(ValueError, match="Hermitian"):
        ControlProblem(h, (bad,))
    with pytest.raises(ValueError):
        CostTerm(CostKind.STATE_INFIDELITY)
    with pytest.raises(ValueError):
        CostTerm(CostKind.STATE_PENALTY)
    with pytest.raises(ValueError, match="unitary"):
        CostTerm(CostKind.GATE_INFIDELITY, target_gate=np.ones((d, d)))
    with pytest.raises(ValueError):
        CostTerm(CostKind.STATE_INFIDELITY, weight=-1.0, target_state=np.ones(d))
