"""Generate golden vectors by running the REFERENCE package (build container only).

Run once in the container that has ``/root/reference`` mounted:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything here is computed by the reference ``leangrape`` code (its model
builders, sparse primitives, planner, StepEvaluator and cost functions).  The
only code not taken from the reference is the K-state *subspace* gate pass
(``ref_gate_pass_subspace``), which the reference cannot express (it demands a
full d-state basis, src/costs.py:399-400).  It is assembled from the
reference's own ``_EvaluatorMemo``/``StepEvaluator`` primitives and checked
here to be bit-identical to ``c1_gate_grad``/``c3_gate_grad`` at K == d.

Outputs ``tests/golden/*.npz`` (small; committed).  Nothing at test time
reads ``/root/reference``.
"""

from __future__ import annotations

import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from leangrape import costs, derivatives, expm, models, sparse  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
TWO_PI = 2.0 * math.pi

# ----------------------------------------------------------------------------- builders
# (the same parameter choices as paper_2304_06200_b200.models)


def tc_ops(d_t, d_c, delta=0.1, alpha=-0.225, g=0.05):
    p = models.TransmonCavityParams(delta=delta, anharmonicity=alpha, g=g, d_transmon=d_t, d_cavity=d_c)
    h_s, _ = models.build_transmon_cavity(p)
    b, bd = models._lowering(d_t), models._raising(d_t)
    ic = sparse.identity_csr(d_c)
    hx = models.kron_csr(sparse.linear_combine([1.0, 1.0], [b, bd]), ic)
    hy = models.kron_csr(sparse.linear_combine([1j, -1j], [bd, b]), ic)
    return h_s, hx, hy


def two_transmon_cavity(d_t=5, d_c=400, d1=0.1, d2=0.15, alpha=-0.225, g=0.05):
    """Two transmons (t1, t2) coupled to one cavity: sum_j [D_j n_j + a/2 n_j(n_j-1) + g(c b_j' + c' b_j)].
    Basis index (t1 * d_t + t2) * d_c + n."""
    it, ic = sparse.identity_csr(d_t), sparse.identity_csr(d_c)
    b, bd = models._lowering(d_t), models._raising(d_t)
    c, cd = models._lowering(d_c), models._raising(d_c)
    k3 = lambda x, y, z: models.kron_csr(models.kron_csr(x, y), z)
    n1, n2 = k3(models._number(d_t), it, ic), k3(it, models._number(d_t), ic)
    a1, a2 = k3(models._anharmonic(d_t), it, ic), k3(it, models._anharmonic(d_t), ic)
    ex1 = sparse.linear_combine([1.0, 1.0], [k3(bd, it, c), k3(b, it, cd)])
    ex2 = sparse.linear_combine([1.0, 1.0], [k3(it, bd, c), k3(it, b, cd)])
    h_s = sparse.linear_combine(
        [TWO_PI * d1, TWO_PI * d2, 0.5 * TWO_PI * alpha, 0.5 * TWO_PI * alpha, TWO_PI * g, TWO_PI * g],
        [n1, n2, a1, a2, ex1, ex2])
    x = sparse.linear_combine([1.0, 1.0], [b, bd])
    y = sparse.linear_combine([1j, -1j], [bd, b])
    ctrls = [k3(x, it, ic), k3(y, it, ic), k3(it, x, ic), k3(it, y, ic)]
    return h_s, ctrls


def gue(rng, d, norm):
    g = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
    h = (g + g.conj().T) / 2
    s = norm / float(np.max(np.abs(np.linalg.eigvalsh(h))))
    return h, s


def rand_states(rng, k, d):
    z = rng.standard_normal((k, d)) + 1j * rng.standard_normal((k, d))
    return z / np.linalg.norm(z, axis=1, keepdims=True)


def controls(seed, n, kc, amp):
    return np.random.default_rng(seed).uniform(-amp, amp, (n, kc))


# ----------------------------------------------------------------------------- reference-side evaluation


def ref_gate_pass_subspace(problem, a, states, images, running):
    """_gate_pass (src/costs.py:407-488) over K given states with 1/K normalisation,
    built from the reference's _EvaluatorMemo / StepEvaluator."""
    n_steps, kc = a.n_steps, a.n_channels
    K = len(states)
    ev = costs._EvaluatorMemo(problem, a)
    traces = np.zeros(n_steps, np.complex128)
    for h in range(K):
        psi = states[h].copy()
        for n in range(n_steps):
            psi = ev.get(n).forward(psi)
            if running or n == n_steps - 1:
                traces[n] += np.vdot(images[h], psi)
    if running:
        cost = 1.0 - float(np.sum(np.abs(traces) ** 2)) / (n_steps * K * K)
    else:
        cost = 1.0 - abs(traces[-1]) ** 2 / (K * K)
    accum = np.zeros((n_steps, kc), np.complex128)
    for h in range(K):
        psi = states[h].copy()
        for n in range(n_steps):
            psi = ev.get(n).forward(psi)
        lam = images[h] * traces[n_steps - 1] if running else images[h].copy()
        for n in range(n_steps - 1, -1, -1):
            e = ev.get(n)
            psi = e.adjoint(psi)
            for k in range(kc):
                accum[n, k] += np.vdot(lam, e.control_derivative(k, psi))
            if n > 0:
                moved = e.adjoint(lam)
                if running:
                    moved += images[h] * traces[n - 1]
                lam = moved
    if running:
        grad = -2.0 / (n_steps * K * K) * accum.real
    else:
        grad = -2.0 / (K * K) * (accum * np.conj(traces[-1])).real
    return float(cost), grad


def ref_state_block(problem_kw, a, psi0s, make_terms):
    """Mean over K of the reference's fused state pass (composite_grad with state terms)."""
    K = len(psi0s)
    c_tot, g_tot = 0.0, np.zeros((a.n_steps, a.n_channels))
    for h in range(K):
        pr = costs.ControlProblem(initial_state=psi0s[h], **problem_kw)
        r = costs.composite_grad(pr, a, make_terms(h))
        c_tot += r.cost / K
        g_tot += r.grad / K
    return c_tot, g_tot


def ref_cost_block(problem_kw, a, psi0s, make_terms):
    K = len(psi0s)
    c = 0.0
    for h in range(K):
        pr = costs.ControlProblem(initial_state=psi0s[h], **problem_kw)
        c += costs.composite_cost(pr, a, make_terms(h)) / K
    return c


def ref_plan_table(h_s, ctrls, amps, dt, tau=1e-8):
    """Per-step planner inputs/plans through the reference's StepEvaluator internals."""
    problem = costs.ControlProblem(h_s, tuple(ctrls), tau=tau)
    a = costs.ControlField(amps.shape[0], amps.shape[1], dt, amps)
    out = {k: [] for k in ("norm1", "sp", "m", "s", "aux_arg", "aux_sp", "aux_m", "aux_s")}
    for n in range(amps.shape[0]):
        ev = problem.step_evaluator(a, n)
        gen, plan = ev._generator_plan()
        out["norm1"].append(gen.one_norm())
        out["sp"].append(gen.max_row_nnz())
        out["m"].append(plan.order)
        out["s"].append(plan.scaling)
        row = []
        for k in range(len(ctrls)):
            aux = derivatives._embedded_generator(ev.ctx, k, gen)
            ap = derivatives.aux_plan(aux, tau)
            row.append((math.sqrt(aux.one_norm() * aux.inf_norm()), aux.max_row_nnz(), ap.order, ap.scaling))
        out["aux_arg"].append([r[0] for r in row])
        out["aux_sp"].append([r[1] for r in row])
        out["aux_m"].append([r[2] for r in row])
        out["aux_s"].append([r[3] for r in row])
    return {k: np.asarray(v) for k, v in out.items()}


def csr_arrays(prefix, m):
    if isinstance(m, sparse.DenseMatrix):
        return {prefix + "_dense": np.asarray(m.array)}
    return {prefix + "_indptr": m.row_offsets, prefix + "_indices": m.col_indices, prefix + "_data": m.values}


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"  wrote {name}.npz ({os.path.getsize(path) / 1024:.0f} KiB)", flush=True)


def mats_payload(h_s, ctrls):
    out = dict(csr_arrays("hs", h_s))
    for k, c in enumerate(ctrls):
        out.update(csr_arrays(f"hc{k}", c))
    out["n_channels"] = np.int64(len(ctrls))
    return out


# ----------------------------------------------------------------------------- cases


def golden_planner():
    """make_plan on random and structured inputs (src/expm.py:279-303)."""
    rng = np.random.default_rng(777)
    rows = []
    taus = [1e-4, 1e-6, 1e-8, 1e-10, 1e-12]
    for _ in range(3000):
        norm = float(np.exp(rng.uniform(np.log(1e-4), np.log(60.0))))
        sp = int(rng.integers(0, 40))
        tau = float(rng.choice(taus))
        rows.append((norm, sp, tau))
    for norm in np.linspace(0.0, 40.0, 401):
        rows.append((float(norm), 5, 1e-8))
    # plan breakpoints around the config norms (SURVEY §8 sizing table)
    for base, sp in [(2.0, 40), (3.1, 80), (0.976, 5), (1.58, 7), (12.38, 5), (14.5, 8), (12.66, 9),
                     (13.59, 12), (2.93, 4096), (3.217, 8193), (12.342397, 5), (12.641749, 5),
                     (12.641380, 9), (13.303916, 9)]:
        for rel in np.linspace(-2e-3, 2e-3, 41):
            rows.append((base * (1 + rel), sp, 1e-8))
    rows.append((0.0, 0, 1e-8))
    rows.append((1e-300, 3, 1e-8))
    norms, sps, taus_, ms, ss, bounds, status = [], [], [], [], [], [], []
    for norm, sp, tau in rows:
        try:
            p = expm.make_plan(norm, sp, tau)
            ms.append(p.order), ss.append(p.scaling), bounds.append(p.bound), status.append(0)
        except expm.PlanningError:
            ms.append(0), ss.append(0), bounds.append(np.nan), status.append(1)
        norms.append(norm), sps.append(sp), taus_.append(tau)
    consts = dict(
        remainder_1_5=expm.remainder_rm(1.0, 5),
        gamma_3=expm.gamma_n(3),
        rounding_05_10_2_4=expm.rounding_bound(0.5, 10, 2, 4),
        truncation_05_15_4=expm.truncation_bound(0.5, 15, 4),
    )
    save("planner", norm=np.array(norms), sp=np.array(sps), tau=np.array(taus_), m=np.array(ms),
         s=np.array(ss), bound=np.array(bounds), status=np.array(status),
         **{k: np.float64(v) for k, v in consts.items()})


def golden_numpy_rules():
    """np.abs / bincount / reduceat / dense sums on adversarial data (plan-input recipe)."""
    rng = np.random.default_rng(4242)
    z = (rng.standard_normal(12000) + 1j * rng.standard_normal(12000)) * np.exp(rng.uniform(-30, 30, 12000))
    z[:100] = rng.standard_normal(100)  # purely real
    z[100:200] = 1j * rng.standard_normal(100)  # purely imaginary
    z[200:210] = 0
    save("numpy_rules", z=z, absz=np.abs(z))


def golden_c1():
    """config 1: dense transmon-cavity 4x10, C1^st, N=1000 (full size)."""
    h_s, hx, _ = tc_ops(4, 10)
    h_s, hx = sparse.DenseMatrix(h_s.to_dense()), sparse.DenseMatrix(hx.to_dense())
    N, dt = 1000, 0.5
    amps = controls(101, N, 1, 0.01)
    psi0, phi = models.fock_state(40, 0), models.fock_state(40, 1)
    pr = costs.ControlProblem(h_s, (hx,), initial_state=psi0)
    a = costs.ControlField(N, 1, dt, amps)
    t0 = time.time()
    r = costs.c1_state_grad(pr, a, psi0, phi)
    cost_only = costs.composite_cost(pr, a, [costs.CostTerm(costs.CostKind.STATE_INFIDELITY, 1.0, target_state=phi)])
    pt = ref_plan_table(h_s, [hx], amps, dt)
    print(f"c1 {time.time() - t0:.1f}s cost={r.cost}")
    save("c1", **mats_payload(h_s, [hx]), amps=amps, dt=dt, psi0=psi0[None], targets=phi[None],
         cost=r.cost, grad=r.grad, cost_only=cost_only, live_peak=r.live_vector_peak,
         **{"plan_" + k: v for k, v in pt.items()})


def golden_c2():
    """config 2: CSR 3x20, K=2 X-gate subspace + 0.1 x penalty on top transmon level."""
    h_s, hx, hy = tc_ops(3, 20)
    N, dt = 2000, 0.25
    amps = controls(102, N, 2, 0.01)
    d = 60
    basis = [models.fock_state(d, 0), models.fock_state(d, 20)]
    images = [basis[1], basis[0]]
    proj = sparse.build_csr_arrays(np.arange(40, 60), np.arange(40, 60), np.ones(20, np.complex128), d, d)
    kw = dict(h_static=h_s, h_controls=(hx, hy))
    a = costs.ControlField(N, 2, dt, amps)
    t0 = time.time()
    pr = costs.ControlProblem(h_s, (hx, hy))
    cg, gg = ref_gate_pass_subspace(pr, a, basis, images, running=False)
    cp, gp = ref_state_block(kw, a, basis, lambda h: [costs.CostTerm(costs.CostKind.STATE_PENALTY, 0.1, penalty_op=proj)])
    cost, grad = cg + cp, gg + gp
    cc = ref_cost_block(kw, a, basis, lambda h: [costs.CostTerm(costs.CostKind.STATE_PENALTY, 0.1, penalty_op=proj)])
    pt = ref_plan_table(h_s, [hx, hy], amps, dt)
    print(f"c2 {time.time() - t0:.1f}s cost={cost}")
    save("c2", **mats_payload(h_s, [hx, hy]), amps=amps, dt=dt, basis=np.array(basis), images=np.array(images),
         pen_indptr=proj.row_offsets, pen_indices=proj.col_indices, pen_data=proj.values,
         cost=cost, grad=grad, cost_gate=cg, cost_pen=cp, cost_only_pen=cc,
         **{"plan_" + k: v for k, v in pt.items()})


def golden_c3(n_prefix=200):
    """config 3: CSR 6x200, K=8 Fock transfers |g,n> -> |g,n+1>, prefix N' of N=2000."""
    h_s, hx, hy = tc_ops(6, 200)
    N, dt = 2000, 0.5
    amps_full = controls(103, N, 2, 0.01)
    amps = amps_full[:n_prefix]
    d = 1200
    psi0s = [models.fock_state(d, n) for n in range(8)]
    phis = [models.fock_state(d, n + 1) for n in range(8)]
    kw = dict(h_static=h_s, h_controls=(hx, hy))
    a = costs.ControlField(n_prefix, 2, dt, amps)
    t0 = time.time()
    cost, grad = ref_state_block(kw, a, psi0s, lambda h: [costs.CostTerm(costs.CostKind.STATE_INFIDELITY, 1.0, target_state=phis[h])])
    pt = ref_plan_table(h_s, [hx, hy], amps, dt)
    print(f"c3 prefix {n_prefix}: {time.time() - t0:.1f}s cost={cost}")
    save("c3", **mats_payload(h_s, [hx, hy]), amps=amps, amps_full=amps_full, dt=dt, psi0=np.array(psi0s),
         targets=np.array(phis), cost=cost, grad=grad, **{"plan_" + k: v for k, v in pt.items()})


def golden_c4(n_prefix=8):
    """config 4: CSR two transmons (5) x cavity 400, 4 controls, K=32 X(t1) gate subspace, prefix N'."""
    h_s, ctrls = two_transmon_cavity()
    N, dt = 4000, 0.25
    amps_full = controls(104, N, 4, 0.01)
    amps = amps_full[:n_prefix]
    d = 10000
    idx = lambda t1, t2, n: (t1 * 5 + t2) * 400 + n
    basis_idx = [idx(t1, t2, n) for t1 in (0, 1) for t2 in (0, 1) for n in range(8)]
    image_idx = [idx(1 - t1, t2, n) for t1 in (0, 1) for t2 in (0, 1) for n in range(8)]
    basis = [models.fock_state(d, i) for i in basis_idx]
    images = [models.fock_state(d, i) for i in image_idx]
    a = costs.ControlField(n_prefix, 4, dt, amps)
    t0 = time.time()
    pr = costs.ControlProblem(h_s, tuple(ctrls))
    cost, grad = ref_gate_pass_subspace(pr, a, basis, images, running=False)
    pt = ref_plan_table(h_s, ctrls, amps_full[:32], dt)
    print(f"c4 prefix {n_prefix}: {time.time() - t0:.1f}s cost={cost}")
    save("c4", **mats_payload(h_s, ctrls), amps=amps, amps_full=amps_full, dt=dt,
         basis_idx=np.array(basis_idx), image_idx=np.array(image_idx), cost=cost, grad=grad,
         **{"plan_" + k: v for k, v in pt.items()})


def golden_c5(n_prefix=4, k_sub=4):
    """config 5: dense GUE 4096, K'=4 of 64 random transfers, prefix N'=4 of N=1000."""
    d = 4096
    rng = np.random.default_rng(5005)
    hs_arr, s1 = gue(rng, d, 1.0)
    hc_arr, s2 = gue(rng, d, 0.1)
    psi0s = rand_states(rng, 64, d)
    phis = rand_states(rng, 64, d)
    h_s = sparse.DenseMatrix(hs_arr * s1)
    hc = sparse.DenseMatrix(hc_arr * s2)
    N, dt = 1000, 0.1
    amps_full = controls(105, N, 1, 1.0)
    amps = amps_full[:n_prefix]
    kw = dict(h_static=h_s, h_controls=(hc,))
    a = costs.ControlField(n_prefix, 1, dt, amps)
    t0 = time.time()
    cost, grad = ref_state_block(kw, a, list(psi0s[:k_sub]),
                                 lambda h: [costs.CostTerm(costs.CostKind.STATE_INFIDELITY, 1.0, target_state=phis[h])])
    pt = ref_plan_table(h_s, [hc], amps_full[:8], dt)
    print(f"c5 prefix {n_prefix} K'={k_sub}: {time.time() - t0:.1f}s cost={cost}")
    save("c5", seed=np.int64(5005), scale_hs=s1, scale_hc=s2, amps=amps, dt=dt, k_sub=np.int64(k_sub),
         cost=cost, grad=grad, hs_checksum=np.sum(np.abs(h_s.array)), **{"plan_" + k: v for k, v in pt.items()})


def _c3_state(h):
    """One state of the full-size c3 block (worker process)."""
    h_s, hx, hy = tc_ops(6, 200)
    amps = controls(103, 2000, 2, 0.01)
    a = costs.ControlField(2000, 2, 0.5, amps)
    pr = costs.ControlProblem(h_s, (hx, hy), initial_state=models.fock_state(1200, h))
    r = costs.composite_grad(pr, a, [costs.CostTerm(costs.CostKind.STATE_INFIDELITY, 1.0,
                                                    target_state=models.fock_state(1200, h + 1))])
    return r.cost, r.grad


def _c5_parts():
    d = 4096
    rng = np.random.default_rng(5005)
    hs_arr, s1 = gue(rng, d, 1.0)
    hc_arr, s2 = gue(rng, d, 0.1)
    psi0s = rand_states(rng, 64, d)
    phis = rand_states(rng, 64, d)
    return sparse.DenseMatrix(hs_arr * s1), sparse.DenseMatrix(hc_arr * s2), psi0s, phis, s1, s2


_C5 = None


def _c5_state(arg):
    """One state of the full-K c5 prefix (worker process; the matrices are built once per worker)."""
    global _C5
    h, n_prefix = arg
    if _C5 is None:
        _C5 = _c5_parts()
    h_s, hc, psi0s, phis, _, _ = _C5
    a = costs.ControlField(n_prefix, 1, 0.1, controls(105, 1000, 1, 1.0)[:n_prefix])
    pr = costs.ControlProblem(h_s, (hc,), initial_state=psi0s[h])
    r = costs.composite_grad(pr, a, [costs.CostTerm(costs.CostKind.STATE_INFIDELITY, 1.0, target_state=phis[h])])
    return r.cost, r.grad


def _pool(fn, items, procs=8):
    import multiprocessing as mp

    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    with mp.get_context("fork").Pool(procs) as pool:
        return pool.map(fn, items, chunksize=1)


def golden_c3_full():
    """config 3 at FULL size (N=2000, K=8): the reference's composite_grad per state, one process
    per state, summed in state order exactly as ref_state_block does (c_tot += cost/K)."""
    t0 = time.time()
    parts = _pool(_c3_state, list(range(8)))
    cost, grad = 0.0, np.zeros((2000, 2))
    for c, g in parts:
        cost += c / 8
        grad += g / 8
    print(f"c3 full: {time.time() - t0:.1f}s cost={cost}")
    save("c3_full", cost=cost, grad=grad, state_costs=np.array([c for c, _ in parts]))


def golden_c5_fullk(n_prefix=2):
    """config 5 with ALL K=64 states (the full-K dense GEMM path: 64/128-column Taylor terms), prefix
    N' of N=1000; per-state composite_grad summed in state order."""
    t0 = time.time()
    parts = _pool(_c5_state, [(h, n_prefix) for h in range(64)])
    cost, grad = 0.0, np.zeros((n_prefix, 1))
    for c, g in parts:
        cost += c / 64
        grad += g / 64
    print(f"c5 full-K prefix {n_prefix}: {time.time() - t0:.1f}s cost={cost}")
    save("c5_fullk", cost=cost, grad=grad, n_prefix=np.int64(n_prefix),
         state_costs=np.array([c for c, _ in parts]), state_grads=np.array([g for _, g in parts]))


def golden_stress():
    """Random-state / large-amplitude variants with every cost kind (plans vary per step)."""
    out = {}
    rng = np.random.default_rng(9090)

    def one(tag, h_s, ctrls, N, dt, amp, K, seed, dense=False):
        d = h_s.n_rows
        if dense:
            h_s = sparse.DenseMatrix(h_s.to_dense())
            ctrls = [sparse.DenseMatrix(c.to_dense()) for c in ctrls]
        amps = controls(seed, N, len(ctrls), amp)
        a = costs.ControlField(N, len(ctrls), dt, amps)
        psi0s = rand_states(rng, K, d)
        phis = rand_states(rng, K, d)
        # penalty: number operator of the "slow" factor (diagonal, Hermitian) -- CSR
        om = sparse.build_csr_arrays(np.arange(d), np.arange(d), (np.arange(d) % 7).astype(np.complex128) / 7.0, d, d)
        kw = dict(h_static=h_s, h_controls=tuple(ctrls))
        mk = lambda h: [costs.CostTerm(costs.CostKind.STATE_INFIDELITY, 0.7, target_state=phis[h]),
                        costs.CostTerm(costs.CostKind.STATE_PENALTY, 0.2, penalty_op=om),
                        costs.CostTerm(costs.CostKind.STATE_RUNNING_INFIDELITY, 0.4, target_state=phis[h])]
        cs, gs = ref_state_block(kw, a, list(psi0s), mk)
        css = ref_cost_block(kw, a, list(psi0s), mk)
        # gate subspace over K orthonormal states with a random unitary on them
        q, _ = np.linalg.qr(rng.standard_normal((d, K)) + 1j * rng.standard_normal((d, K)))
        basis = [q[:, h].copy() for h in range(K)]
        u, _ = np.linalg.qr(rng.standard_normal((K, K)) + 1j * rng.standard_normal((K, K)))
        images = [sum(u[j, h] * basis[j] for j in range(K)) for h in range(K)]
        pr = costs.ControlProblem(h_s, tuple(ctrls))
        cg1, gg1 = ref_gate_pass_subspace(pr, a, basis, images, running=False)
        cg3, gg3 = ref_gate_pass_subspace(pr, a, basis, images, running=True)
        pt = ref_plan_table(h_s, ctrls, amps, dt)
        print(f"stress {tag}: d={d} N={N} K={K} plans m={sorted(set(pt['m']))} aux_m={sorted(set(pt['aux_m'].ravel()))}")
        pay = mats_payload(h_s, ctrls)
        out.update({f"{tag}__{k}": v for k, v in pay.items()})
        out.update({f"{tag}__{k}": v for k, v in dict(
            amps=amps, dt=dt, psi0=psi0s, targets=phis, pen_indptr=om.row_offsets, pen_indices=om.col_indices,
            pen_data=om.values, basis=np.array(basis), images=np.array(images),
            cost_state=cs, grad_state=gs, cost_state_only=css, cost_g1=cg1, grad_g1=gg1, cost_g3=cg3, grad_g3=gg3,
            **{"plan_" + k: v for k, v in pt.items()}).items()})

    h_s, hx, hy = tc_ops(3, 20)
    one("s_csr60", h_s, [hx, hy], 30, 0.25, 1.0, 3, 201)
    h_s, hx, hy = tc_ops(4, 40)
    one("s_block160", h_s, [hx, hy], 10, 0.5, 0.5, 2, 202)
    h_s, hx, hy = tc_ops(3, 8)
    one("s_dense24", h_s, [hx, hy], 12, 0.5, 1.0, 3, 203, dense=True)
    h_s, hx, _ = tc_ops(4, 40)
    one("s_denseblk160", h_s, [hx], 5, 0.5, 0.5, 2, 204, dense=True)
    save("stress", **out)


def golden_diag(big=False, mid=False):
    """The reference's DIAGONALIZATION backend (src/derivatives.py:228-275): every cost kind on a
    dense d = 40 problem (c1's model), a CSR d = 24 and a CSR d = 60 problem, random states,
    large amplitudes.  Sparse inputs stay CSR here: the reference densifies each step.
    big=True (``diag_big``): a CSR d = 180 problem (transmon 6 x cavity 30) and a dense d = 256
    one, above the device CTA engine's d <= 128 (the dense GEMM engine applies the propagators).
    mid=True (``diag_mid``): a CSR d = 96 problem (transmon 4 x cavity 24): above the in-shared-memory
    factorisation's d <= 64, still on the CTA engine."""
    out = {}
    rng = np.random.default_rng(7171)
    DIAG = derivatives.Backend.DIAGONALIZATION

    def one(tag, h_s, ctrls, N, dt, amp, K, seed):
        d = h_s.n_rows
        amps = controls(seed, N, len(ctrls), amp)
        a = costs.ControlField(N, len(ctrls), dt, amps)
        psi0s = rand_states(rng, K, d)
        phis = rand_states(rng, K, d)
        om = sparse.build_csr_arrays(np.arange(d), np.arange(d), (np.arange(d) % 5).astype(np.complex128) / 5.0, d, d)
        kw = dict(h_static=h_s, h_controls=tuple(ctrls), backend=DIAG)
        mk = lambda h: [costs.CostTerm(costs.CostKind.STATE_INFIDELITY, 0.7, target_state=phis[h]),
                        costs.CostTerm(costs.CostKind.STATE_PENALTY, 0.2, penalty_op=om),
                        costs.CostTerm(costs.CostKind.STATE_RUNNING_INFIDELITY, 0.4, target_state=phis[h])]
        cs, gs = ref_state_block(kw, a, list(psi0s), mk)
        css = ref_cost_block(kw, a, list(psi0s), mk)
        q, _ = np.linalg.qr(rng.standard_normal((d, K)) + 1j * rng.standard_normal((d, K)))
        basis = [q[:, h].copy() for h in range(K)]
        u, _ = np.linalg.qr(rng.standard_normal((K, K)) + 1j * rng.standard_normal((K, K)))
        images = [sum(u[j, h] * basis[j] for j in range(K)) for h in range(K)]
        pr = costs.ControlProblem(h_s, tuple(ctrls), backend=DIAG)
        cg1, gg1 = ref_gate_pass_subspace(pr, a, basis, images, running=False)
        cg3, gg3 = ref_gate_pass_subspace(pr, a, basis, images, running=True)
        print(f"diag {tag}: d={d} N={N} K={K} cost_state={cs:.6f} cost_g1={cg1:.6f}")
        pay = mats_payload(h_s, ctrls)
        out.update({f"{tag}__{k}": v for k, v in pay.items()})
        out.update({f"{tag}__{k}": v for k, v in dict(
            amps=amps, dt=dt, psi0=psi0s, targets=phis, pen_indptr=om.row_offsets, pen_indices=om.col_indices,
            pen_data=om.values, basis=np.array(basis), images=np.array(images),
            cost_state=cs, grad_state=gs, cost_state_only=css, cost_g1=cg1, grad_g1=gg1, cost_g3=cg3,
            grad_g3=gg3).items()})

    if mid:
        h_s, hx, hy = tc_ops(4, 24)
        one("d_csr96", h_s, [hx, hy], 12, 0.5, 0.8, 2, 406)
        save("diag_mid", **out)
        return
    if big:
        h_s, hx, hy = tc_ops(6, 30)
        one("d_csr180", h_s, [hx, hy], 10, 0.5, 0.5, 2, 404)
        h_s, hx, _ = tc_ops(4, 64)
        one("d_dense256", sparse.DenseMatrix(h_s.to_dense()), [sparse.DenseMatrix(hx.to_dense())], 8, 0.5, 0.5, 2, 405)
        save("diag_big", **out)
        return
    h_s, hx, _ = tc_ops(4, 10)
    one("d_dense40", sparse.DenseMatrix(h_s.to_dense()), [sparse.DenseMatrix(hx.to_dense())], 40, 0.5, 1.0, 2, 401)
    h_s, hx, hy = tc_ops(3, 8)
    one("d_csr24", h_s, [hx, hy], 20, 0.5, 1.0, 3, 402)
    h_s, hx, hy = tc_ops(3, 20)
    one("d_csr60", h_s, [hx, hy], 16, 0.25, 1.0, 2, 403)
    save("diag", **out)


def golden_diag_big():
    golden_diag(big=True)


def golden_diag_mid():
    golden_diag(mid=True)


BENCH_MU_CASES = [("transmon_cavity", 10, 0.1), ("transmon_cavity", 40, 0.5), ("transmon_cavity", 80, 2.0),
                  ("three_transmons", 3, 0.1), ("three_transmons", 5, 1.0), ("qubit_chain", 3, 0.1),
                  ("qubit_chain", 6, 0.7), ("fluxonium_pair", 6, 0.1), ("fluxonium_pair", 12, 0.05),
                  ("zero", 4, 0.1), ("transmon_cavity", 20, 1e4)]


def golden_bench_mu():
    """The reference's planning sweep records (src/bench.py:169-193, measure_mu) for every model
    family at several sizes / time steps, tau 1e-8 and 1e-14 (the latter makes large norms
    infeasible: matvecs None -> -1 here), plus one power-law fit of a dimension sweep."""
    from leangrape import bench as rb

    rows = []
    for tau in (1e-8, 1e-14):
        for m, size, dt in BENCH_MU_CASES:
            r = rb.measure_mu(m, size, dt, tau)
            rows.append((r.d, r.norm1, r.sigma_prime, -1 if r.matvecs is None else r.matvecs, r.kappa, tau, dt, size))
    sweep = rb.mu_vs_dim_sweep("transmon_cavity", [10, 20, 40, 80, 160], 1e-8)
    fit = rb.fit_power_law([(r.d, r.matvecs) for r in sweep])
    save("bench_mu", rows=np.array(rows, dtype=np.float64), models=np.array([m for _ in (0, 1) for m, _, _ in BENCH_MU_CASES]),
         csv=np.array([r.to_csv_row() for r in sweep]), fit=np.array([fit.exponent, fit.log_prefactor, fit.r_squared]))


def golden_full_basis_check():
    """Restated subspace gate pass == reference c1/c3_gate_grad at K == d (bitwise)."""
    rng = np.random.default_rng(31)
    h_s, hx, hy = tc_ops(2, 3)
    N, dt = 4, 0.5
    amps = controls(301, N, 2, 0.3)
    a = costs.ControlField(N, 2, dt, amps)
    pr = costs.ControlProblem(h_s, (hx, hy))
    d = 6
    u, _ = np.linalg.qr(rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d)))
    eye = np.eye(d, dtype=np.complex128)
    basis = [eye[:, h] for h in range(d)]
    images = [u @ basis[h] for h in range(d)]
    r1 = costs.c1_gate_grad(pr, a, u)
    r3 = costs.c3_gate_grad(pr, a, u)
    c1, g1 = ref_gate_pass_subspace(pr, a, basis, images, False)
    c3, g3 = ref_gate_pass_subspace(pr, a, basis, images, True)
    assert c1 == r1.cost and np.array_equal(g1, r1.grad), "restated C1^g != reference"
    assert c3 == r3.cost and np.array_equal(g3, r3.grad), "restated C3^g != reference"
    print("full-basis restatement: bit-identical to c1_gate_grad / c3_gate_grad")
    save("fullbasis", **mats_payload(h_s, [hx, hy]), amps=amps, dt=dt, target_gate=u,
         cost_g1=r1.cost, grad_g1=r1.grad, cost_g3=r3.cost, grad_g3=r3.grad,
         live_g1=r1.live_vector_peak)


def golden_expm():
    """Standalone certified action: reference expm.make_plan / expm.expm_multiply (src/expm.py:279-369)
    on random anti-Hermitian CSR and dense generators, the sigma_x rotation, the zero generator and a
    banded transmon-cavity generator; three states each (the reference takes one vector at a time)."""
    rng = np.random.default_rng(4242)

    def anti(d, scale):
        g = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
        return scale * (g - g.conj().T) / 2.0

    h_s, hx, hy = tc_ops(6, 200)
    hn = sparse.linear_combine([1.0, 0.01, -0.007], [h_s, hx, hy])
    cases = {
        "csr16": (sparse.from_dense(anti(16, 1.5)), (1e-8, 1e-12)),
        "dense12": (sparse.DenseMatrix(np.asfortranarray(anti(12, 0.8))), (1e-10,)),
        "rot": (sparse.build_csr([(0, 1, -1j * np.pi / 2), (1, 0, -1j * np.pi / 2)], 2, 2), (1e-10,)),
        "zero": (sparse.build_csr([], 5, 5), (1e-8,)),
        "band1200": (hn.scaled(-1j * 0.5), (1e-8,)),
    }
    out = {}
    for tag, (a, taus) in cases.items():
        d = a.n_rows
        psi = rand_states(rng, 3, d)
        out.update({f"{tag}__{k}": v for k, v in csr_arrays("a", a).items()})
        out[f"{tag}__psi"] = psi
        out[f"{tag}__norm1"] = np.float64(a.one_norm())
        out[f"{tag}__sp"] = np.int64(a.max_row_nnz())
        for i, tau in enumerate(taus):
            plan = expm.make_plan(a.one_norm(), a.max_row_nnz(), tau)
            res = [expm.expm_multiply(a, psi[h], tau) for h in range(3)]
            out[f"{tag}__tau{i}"] = np.float64(tau)
            out[f"{tag}__m{i}"] = np.int64(plan.order)
            out[f"{tag}__s{i}"] = np.int64(plan.scaling)
            out[f"{tag}__mu{i}"] = np.int64(res[0][1])
            out[f"{tag}__out{i}"] = np.array([r[0] for r in res])
    save("expm", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["planner", "numpy_rules", "full_basis_check", "c1", "c2", "stress", "c3", "c4", "c5",
                             "expm", "diag"]
    for w in which:
        globals()["golden_" + w]()
