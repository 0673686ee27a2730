"""Host side of the per-step surface (paper_2304_06200_b200.derivatives) against the reference's own
objects (imported from /root/reference when present -- the build container; skipped elsewhere): the
embedded generator, the block operator's assembled bounds and the derivative plans must be the
reference's, bit for bit, because they select the Taylor plan the device runs
(src/derivatives.py:133-203, src/sparse.py:352-380).  CPU only: no device calls besides the host
planner of the C library.  The actions themselves are tests/test_gpu_step_evaluator.py."""

import os
import sys

import numpy as np
import pytest

from paper_2304_06200_b200 import derivatives as D
from paper_2304_06200_b200 import sparse as S
from paper_2304_06200_b200.costs import ControlField, ControlProblem

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF)
    try:
        import leangrape.costs as costs
        import leangrape.derivatives as derivatives
        import leangrape.sparse as sparse
    finally:
        sys.path.remove(REF)
    return costs, derivatives, sparse


def _banded(g, d, offsets, dense=False):
    m = np.zeros((d, d), complex)
    for o in offsets:
        v = g.standard_normal(d - o) + (1j * g.standard_normal(d - o) if o else 0)
        m[np.arange(d - o), np.arange(d - o) + o] = v
        if o:
            m[np.arange(d - o) + o, np.arange(d - o)] = np.conj(v)
    return m


@pytest.mark.parametrize("d,dense", [(12, False), (12, True), (150, False)])
def test_embedding_bounds_and_plans_are_the_references(ref, d, dense):
    rcosts, rder, rsp = ref
    g = np.random.default_rng(31 + d)
    hs, hc = _banded(g, d, (0, 1, 4)), _banded(g, d, (2,))
    dt, tau = 0.3, 1e-9
    mine_s = S.DenseMatrix(hs) if dense else S.from_dense(hs)
    mine_c = S.from_dense(hc)
    theirs_s = rsp.DenseMatrix(np.asfortranarray(hs)) if dense else rsp.from_dense(hs)
    theirs_c = rsp.from_dense(hc)
    # materialised embedding: same stored entries
    em, et = D.aux_embed(mine_s, mine_c, dt), rsp.aux_embed(theirs_s, theirs_c, dt)
    assert np.array_equal(S.to_dense(em), et.to_dense())
    # block operator: same assembled bounds and the same plan as the reference selects
    bm = D.BlockDerivativeOperator(mine_s.scaled(-1j * dt), mine_c, dt)
    bt = rder.BlockDerivativeOperator(theirs_s.scaled(-1j * dt), theirs_c, dt)
    assert bm.one_norm() == bt.one_norm() and bm.inf_norm() == bt.inf_norm()
    assert bm.max_row_nnz() == bt.max_row_nnz() and bm.nnz == bt.nnz
    pm, pt = D.aux_plan(bm, tau), rder.aux_plan(bt, tau)
    assert (pm.order, pm.scaling, pm.norm1, pm.sigma_prime, pm.bound) == (pt.order, pt.scaling, pt.norm1,
                                                                         pt.sigma_prime, pt.bound)
    assert np.array_equal(S.to_dense(bm.stored()), et.to_dense())
    # the path the evaluator takes at this size (materialised up to 2 d = 256, block bounds above)
    ctx_m = D.StepContext(mine_s, (mine_c,), dt, tau=tau)
    ctx_t = rder.StepContext(theirs_s, (theirs_c,), dt, tau=tau)
    _, bounds = D._embedded(ctx_m, 0, D._generator(ctx_m))
    theirs = rder._embedded_generator(ctx_t, 0, rder._generator(ctx_t))
    assert type(theirs).__name__ == ("BlockDerivativeOperator" if 2 * d > 256 else type(et).__name__)
    pm, pt = D.aux_plan(bounds, tau), rder.aux_plan(theirs, tau)
    assert (pm.order, pm.scaling, pm.bound) == (pt.order, pt.scaling, pt.bound)


def test_step_evaluator_folds_the_amplitudes_like_the_reference(ref):
    rcosts, rder, rsp = ref
    g = np.random.default_rng(5)
    d, n, k = 9, 3, 2
    hs, hcs = _banded(g, d, (0, 1)), [_banded(g, d, (1,)), _banded(g, d, (2,))]
    amps = g.normal(size=(n, k))
    amps[1, 0] = 0.0  # an exactly-zero amplitude drops its operator from H_n (src/sparse.py:261-263)
    mine = ControlProblem(S.from_dense(hs), tuple(S.from_dense(h) for h in hcs), tau=1e-9)
    theirs = rcosts.ControlProblem(rsp.from_dense(hs), tuple(rsp.from_dense(h) for h in hcs), tau=1e-9)
    for i in range(n):
        em = mine.step_evaluator(ControlField(n, k, 0.2, amps), i)
        et = theirs.step_evaluator(rcosts.ControlField(n, k, 0.2, amps), i)
        hm, ht = em.ctx.h_step, et.ctx.h_step
        assert np.array_equal(hm.row_offsets, ht.row_offsets) and np.array_equal(hm.col_indices, ht.col_indices)
        assert np.array_equal(hm.values, ht.values)
        gm, pm = em._generator_plan()
        gt, pt = et._generator_plan()
        assert np.array_equal(gm.values, gt.values)
        assert (pm.order, pm.scaling, pm.norm1, pm.sigma_prime, pm.bound) == (pt.order, pt.scaling, pt.norm1,
                                                                             pt.sigma_prime, pt.bound)
