"""Planning sweeps of the certified action (the reference's ``bench-mu``:
src/bench.py:57-193, 281-323): how many matvecs (mu = order x scaling of the certified Taylor
plan) one propagator-state product needs, across time steps (norm) and dimensions.

Host-side planning only -- the same bit-exact planner inputs (``expm.plan_inputs``: numpy's
one-norm and sigma' rules) and the same native planner (``expm.make_plan``, lg_planner.cuh) the
device evaluations use -- over the reference's four benchmark model families, built here with the
reference's parameters (src/models.py:98-140, 147-286) so the records match its ``measure_mu``
field for field (tests/test_bench_mu.py against tests/golden/bench_mu.npz).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import expm
from .models import _anharmonic, _lowering, _number, _raising
from .sparse import build_csr_arrays, from_dense, identity_csr, kron_csr, linear_combine

__all__ = ["BenchRecord", "PowerLawFit", "MODEL_NAMES", "DEFAULT_SWEEP_DT", "build_model", "measure_mu",
           "mu_vs_norm_sweep", "mu_vs_dim_sweep", "fit_power_law"]

TWO_PI = 2.0 * math.pi
DEFAULT_SWEEP_DT = 0.1  # src/bench.py:57


@dataclass(frozen=True)
class BenchRecord:
    """One point of a scaling study (src/bench.py:65-85)."""

    model: str
    d: int
    n_steps: int
    tau: float
    norm1: float
    sigma_prime: int
    matvecs: int | None  # None: no feasible plan at this tolerance
    kappa: int  # stored Hamiltonian elements, static plus every control
    wall_ns: int = 0
    live_vector_peak: int = 0

    def to_csv_row(self) -> str:
        mu = "" if self.matvecs is None else str(self.matvecs)
        return (f"{self.model},{self.d},{self.n_steps},{self.tau:.17g},{self.norm1:.17g},"
                f"{self.sigma_prime},{mu},{self.kappa},{self.wall_ns},{self.live_vector_peak}")


@dataclass(frozen=True)
class PowerLawFit:
    """Least squares of log y = exponent log x + log_prefactor (src/bench.py:88-95)."""

    exponent: float
    log_prefactor: float
    r_squared: float


# ------------------------------------------------------------------------------- model families
# (reference defaults, linear frequencies in GHz converted to rad/ns)

def _embed(op, site: int, dims):
    out = op if site == 0 else identity_csr(dims[0])
    for k in range(1, len(dims)):
        out = kron_csr(out, op if k == site else identity_csr(dims[k]))
    return out


def _transmon_cavity(size: int):
    """delta b'b + alpha/2 b'b(b'b-1) + g(c b' + c' b); controls b'b, b + b' (src/models.py:147-176)."""
    d_t, d_c, delta, alpha, g = 6, size, 3.0, -0.225, 0.1
    if d_c < 2:
        raise ValueError("mode dimensions must be at least 2")
    b, bd, c, cd, ic = _lowering(d_t), _raising(d_t), _lowering(d_c), _raising(d_c), identity_csr(d_c)
    nt = kron_csr(_number(d_t), ic)
    exchange = linear_combine([1.0, 1.0], [kron_csr(bd, c), kron_csr(b, cd)])
    h = linear_combine([TWO_PI * delta, 0.5 * (TWO_PI * alpha), TWO_PI * g],
                       [nt, kron_csr(_anharmonic(d_t), ic), exchange])
    return h, [nt, kron_csr(linear_combine([1.0, 1.0], [b, bd]), ic)], [TWO_PI * 0.1, TWO_PI * 0.1]


def _three_transmons(size: int):
    """Three transmons, anharmonic, nearest-neighbour hopping; one drive each (src/models.py:179-202)."""
    if size < 2:
        raise ValueError("transmon dimension must be at least 2")
    dims, b, bd, ident = [size] * 3, _lowering(size), _raising(size), identity_csr(size)
    alpha, g = TWO_PI * -0.225, TWO_PI * 0.1
    terms = [_embed(_anharmonic(size), s, dims) for s in range(3)]
    coeffs = [0.5 * alpha] * 3
    for hop in (kron_csr(kron_csr(b, bd), ident), kron_csr(ident, kron_csr(b, bd))):
        terms.append(linear_combine([1.0, 1.0], [hop, hop.conj_transpose()]))
        coeffs.append(g)
    ctrls = [_embed(linear_combine([1.0, 1.0], [b, bd]), s, dims) for s in range(3)]
    return linear_combine(coeffs, terms), ctrls, [TWO_PI * 0.1] * 3


def _qubit_chain(size: int):
    """sigma_z sigma_z chain, x / y drive per qubit, qubit 1 leftmost (src/models.py:205-236)."""
    if size < 1:
        raise ValueError("need at least one qubit")
    dim = 2 ** size
    idx = np.arange(dim, dtype=np.int64)
    g = TWO_PI * 0.1
    diag = np.zeros(dim)
    for nu in range(size - 1):
        diag += g * (1.0 - 2.0 * ((idx >> (size - 1 - nu)) & 1)) * (1.0 - 2.0 * ((idx >> (size - 2 - nu)) & 1))
    h = build_csr_arrays(idx, idx, diag.astype(np.complex128), dim, dim)
    ctrls = []
    for nu in range(size):
        mask = 1 << (size - 1 - nu)
        flip = idx ^ mask
        ctrls.append(build_csr_arrays(idx, flip, np.ones(dim, np.complex128), dim, dim))
        ctrls.append(build_csr_arrays(idx, flip, np.where((idx & mask) != 0, 1j, -1j).astype(np.complex128), dim, dim))
    return h, ctrls, [TWO_PI * 0.5] * len(ctrls)


def _fluxonium(e_c, e_j, e_l, ext_flux, dim):
    """Dense single fluxonium in the oscillator basis: (h, phi, n) in rad/ns (src/models.py:239-266)."""
    ec, ej, el = TWO_PI * e_c, TWO_PI * e_j, TWO_PI * e_l
    a = np.zeros((dim, dim), dtype=np.complex128)
    a[np.arange(dim - 1), np.arange(1, dim)] = np.sqrt(np.arange(1, dim))
    ad = a.conj().T
    phi = (8.0 * ec / el) ** 0.25 / math.sqrt(2.0) * (a + ad)
    n_op = 1j * ((el / (8.0 * ec)) ** 0.25 / math.sqrt(2.0)) * (ad - a)
    w, v = np.linalg.eigh(phi)
    cos_phi = (v * np.cos(w)) @ v.conj().T
    shifted = phi - ext_flux * np.eye(dim)
    return 4.0 * ec * (n_op @ n_op) - ej * cos_phi + 0.5 * el * (shifted @ shifted), phi, n_op


def _fluxonium_pair(size: int):
    """Two capacitively coupled fluxoniums, flux drives -E_L phi (src/models.py:269-305); no drive
    amplitude in the fixture: the static Hamiltonian alone sets the norm."""
    if size < 4:
        raise ValueError("fluxonium oscillator basis needs at least 4 levels")
    h1, phi1, n1 = _fluxonium(2.5, 8.9, 0.5, 0.33, size)
    h2, phi2, n2 = _fluxonium(2.5, 8.9, 0.5, 0.33, size)
    ident = identity_csr(size)
    h = linear_combine([1.0, 1.0, TWO_PI * 0.1],
                       [kron_csr(from_dense(0.5 * (h1 + h1.conj().T)), ident),
                        kron_csr(ident, from_dense(0.5 * (h2 + h2.conj().T))),
                        kron_csr(from_dense(n1), from_dense(n2))])
    el = TWO_PI * 0.5
    return h, [kron_csr(from_dense(-el * phi1), ident), kron_csr(ident, from_dense(-el * phi2))], [0.0, 0.0]


def _zero(size: int):
    return build_csr_arrays(np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0, np.complex128), size, size), [], []


_BUILDERS = {"transmon_cavity": _transmon_cavity, "three_transmons": _three_transmons, "qubit_chain": _qubit_chain,
             "fluxonium_pair": _fluxonium_pair, "zero": _zero}
MODEL_NAMES = tuple(sorted(_BUILDERS))


def build_model(model: str, size: int):
    """(h_static, controls, fixture drive amplitudes) of a family at its sweep parameter ``size``
    (cavity dimension, per-mode dimension or qubit count; src/bench.py:143-153)."""
    try:
        return _BUILDERS[model](size)
    except KeyError:
        raise ValueError(f"unknown model {model!r}; choose from {MODEL_NAMES}") from None


def measure_mu(model: str, size: int, dt: float, tau: float) -> BenchRecord:
    """Plan one propagator-state product of the fixture generator -i dt (H_s + sum a_c h_c) and
    record its matvec count (src/bench.py:169-193); an infeasible tolerance gives matvecs=None."""
    h, ctrls, amps = build_model(model, size)
    gen = (linear_combine([1.0, *amps], [h, *ctrls]) if ctrls else h).scaled(-1j * dt)
    norm1, sigma = expm.plan_inputs(gen)
    try:
        mu = expm.make_plan(norm1, sigma, tau).matvecs
    except expm.PlanningError:
        mu = None
    return BenchRecord(model=model, d=h.n_rows, n_steps=1, tau=tau, norm1=norm1, sigma_prime=sigma, matvecs=mu,
                       kappa=h.nnz + sum(c.nnz for c in ctrls))


def mu_vs_norm_sweep(model: str, size: int, dts, tau: float) -> list:
    """Matvec counts across time steps (the norm grows linearly in dt; src/bench.py:281-283)."""
    return [measure_mu(model, size, float(dt), tau) for dt in dts]


def mu_vs_dim_sweep(model: str, sizes, tau: float, dt: float = DEFAULT_SWEEP_DT) -> list:
    """Matvec counts across dimensions at a fixed time step (src/bench.py:286-290)."""
    return [measure_mu(model, int(s), dt, tau) for s in sizes]


def fit_power_law(points) -> PowerLawFit:
    """log-log least squares over >= 4 positive (x, y) points (src/bench.py:293-313)."""
    pts = [(float(x), float(y)) for x, y in points]
    if len(pts) < 4:
        raise ValueError("power-law fit needs at least 4 points")
    if any(x <= 0 or y <= 0 for x, y in pts):
        raise ValueError("power-law fit needs positive data")
    lx, ly = np.log([x for x, _ in pts]), np.log([y for _, y in pts])
    slope, icept = np.polyfit(lx, ly, 1)
    res = ly - (slope * lx + icept)
    ss_tot = float(((ly - ly.mean()) ** 2).sum())
    return PowerLawFit(float(slope), float(icept), 1.0 if ss_tot == 0.0 else 1.0 - float((res ** 2).sum()) / ss_tot)
