"""Load tests/golden/*.npz (generated from the reference by make_golden.py) into
both the oracle's objects and the product's Python API objects."""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def sub(z, tag):
    p = tag + "__"
    return {k[len(p):]: v for k, v in z.items() if k.startswith(p)}


def mats(z, kind="product"):
    """(h_static, [h_c...]) as product CsrMatrix/DenseMatrix or oracle Csr/Dense."""
    from paper_2304_06200_b200.sparse import CsrMatrix, DenseMatrix

    def one(prefix):
        if prefix + "_dense" in z:
            a = np.asfortranarray(z[prefix + "_dense"])
            if kind == "product":
                return DenseMatrix(a)
            from oracle import lg_oracle as O

            return O.Dense(a)
        ip, ix, dv = z[prefix + "_indptr"], z[prefix + "_indices"], z[prefix + "_data"]
        n = ip.size - 1
        if kind == "product":
            return CsrMatrix(n, n, ip, ix, dv)
        from oracle import lg_oracle as O

        return O.Csr(n, ip, ix, dv)

    kc = int(z["n_channels"])
    return one("hs"), [one(f"hc{k}") for k in range(kc)]


def penalty(z, kind="product"):
    ip, ix, dv = z["pen_indptr"], z["pen_indices"], z["pen_data"]
    n = ip.size - 1
    if kind == "product":
        from paper_2304_06200_b200.sparse import CsrMatrix

        return CsrMatrix(n, n, ip, ix, dv)
    from oracle import lg_oracle as O

    return O.Csr(n, ip, ix, dv)


def plan_keys():
    return ("norm1", "sp", "m", "s", "aux_arg", "aux_sp", "aux_m", "aux_s")


def grad_rel(g, g_ref):
    """Norm-wise relative gradient error (tests/test_costs.py:39-42 style)."""
    den = np.linalg.norm(g_ref)
    return float(np.linalg.norm(g - g_ref) / den) if den > 0 else float(np.linalg.norm(g))
