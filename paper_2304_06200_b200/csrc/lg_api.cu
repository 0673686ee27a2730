// Host orchestration and the C ABI (include/leangrape_b200.h).
//
// lg_problem_create  ~ ControlProblem + CostTerm validation + device upload
//                      (src/costs.py:96-168); builds the union ELL pattern of
//                      H_s and every h_c so that all N step generators share
//                      one index structure.
// lg_eval            ~ composite_grad (src/costs.py:515-546):
//   1. lg_k_prep_*     all N step generators A_n + bit-exact planner inputs
//   2. lg_k_plans      all N x (1 + K_c) plans on the device; guarded entries
//                      re-planned exactly on the host (lg_planner.cuh)
//   3. lg_k_forward    forward sweep (all trajectories, all steps)
//   4. lg_k_trsum      running gate traces (between sweeps)
//   5. lg_k_backward   backward sweep: adjoint, derivative products, costates
//   6. lg_k_finalize   cost + gradient
#include "lg_host.h"

namespace lgi {

// Steps 3-6 with amplitudes already on the device.
// Point ip/fin/trp/run at the raw buffer with the exact layout of lg_raw_get for N steps
// (the caller-lent buffer of lg_set_raw_buffer when one is set).
int raw_views(lg_problem* p, long N) {
  const long S = std::max<long>((long)p->specs.size(), 1), T = std::max(p->T_total, 1), Kc = p->Kc;
  const long need = 2 * (N * S * Kc * T + S * T + S * N * T) + S * T;
  double* base = p->d_raw;
  if (p->ext_raw) {
    if (p->ext_raw_len < need) return fail(LG_INVALID_ARG, "lent raw buffer is smaller than lg_raw_size");
    base = p->ext_raw;
  }
  p->d_ip = reinterpret_cast<double2*>(base);
  p->d_fin = p->d_ip + N * S * Kc * T;
  p->d_trp = p->d_fin + S * T;
  p->d_run = reinterpret_cast<double*>(p->d_trp + S * N * T);
  return LG_OK;
}

// Sharded evaluation hook points.  Every rank reaches them in the same order.
int hook_traces(lg_problem* p, long N) {  // between the sweeps: global running gate traces
  p->trp_reduced = false;
  if (!p->hook || !p->has_gate_run) return LG_OK;
  const long S = (long)p->specs.size(), T = p->T_total;
  if (p->hook(reinterpret_cast<double*>(p->d_trp), 2 * S * N * T, p->stream, p->hook_user) != 0)
    return fail(LG_CUDA_ERROR, "all-reduce hook failed (traces)");
  p->trp_reduced = true;
  return LG_OK;
}
int hook_raw(lg_problem* p, long N) {  // before the combine: every shard's raw scalars
  if (!p->hook) return LG_OK;
  const long S = (long)p->specs.size(), T = p->T_total, Kc = p->Kc;
  const long nipfin = 2 * (N * S * Kc * T + S * T), ntrp = 2 * S * N * T, nrun = S * T;
  double* base = reinterpret_cast<double*>(p->d_ip);
  int e = 0;
  if (p->trp_reduced) {
    e |= p->hook(base, nipfin, p->stream, p->hook_user);
    e |= p->hook(base + nipfin + ntrp, nrun, p->stream, p->hook_user);
  } else {
    e |= p->hook(base, nipfin + ntrp + nrun, p->stream, p->hook_user);
  }
  if (e) return fail(LG_CUDA_ERROR, "all-reduce hook failed (raw scalars)");
  return LG_OK;
}

int run_sweeps(lg_problem* p, long N, bool grad) {
  const int S = (int)p->specs.size(), T = p->T_total;
  if (int rv = raw_views(p, N)) return rv;
  p->trp_reduced = false;
  if (p->engine == 3) {
    p->mark(1);
    p->dense_bwd_marked = false;
    int rc = run_dense(p, N, p->cached_dt, grad);  // records the forward / backward boundary itself
    if (rc) return rc;
    if (!p->dense_bwd_marked) p->mark(2);
    rc = hook_raw(p, N);
    if (rc) return rc;
    p->mark(3);
    LgFinalArgs F = final_args(p, N, p->d_ip, p->d_fin, p->d_run, p->d_trp, p->d_grad, p->d_cost);
    void* fargs[] = {&F};
    rc = launch(lg_finalize_kernel(), dim3((unsigned)std::min<long>((N * p->Kc + 255) / 256 + 1, 1024)), dim3(256),
                fargs, 0, p->stream);
    if (rc) return rc;
    p->mark(4);
    p->lastN = N;
    return LG_OK;
  }
  CK(cudaMemsetAsync(p->d_run, 0, sizeof(double) * std::max(S, 1) * std::max(T, 1), p->stream));
  CK(cudaMemsetAsync(p->d_fin, 0, sizeof(double2) * std::max(S, 1) * std::max(T, 1), p->stream));
  if (grad) CK(cudaMemsetAsync(p->d_ip, 0, sizeof(double2) * N * std::max(S, 1) * p->Kc * std::max(T, 1), p->stream));
  CK(cudaMemsetAsync(p->d_trp, 0, sizeof(double2) * std::max(S, 1) * N * std::max(T, 1), p->stream));
  CK(cudaMemsetAsync(p->d_bar, 0, sizeof(unsigned) * 4 * std::max(p->n_groups, 1), p->stream));
  LgEngineArgs E = engine_args(p, N);
  void* eargs[] = {&E};
  const dim3 grid(p->n_groups * p->n_slabs), block(p->threads);
  int rc = LG_OK;
  p->mark(1);
  void* fwd = p->engine == 2 ? lg_cta_kernel(0, p->cta_maxr, p->cta_maxc, p->cta_wreg) : lg_forward_kernel(p->multi);
  void* bwd = p->engine == 2 ? lg_cta_kernel(1, p->cta_maxr, p->cta_maxc, p->cta_wreg) : lg_backward_kernel(p->multi);
  int fsm = p->smem_bytes, bsm = p->smem_bytes;
  dim3 bblock = block;
  if (p->engine == 4) {
    fwd = lg_ws_kernel(0, p->dense ? -lg_ws_dense_width((int)p->d) : p->W, p->ws_rpl);
    bwd = lg_ws_kernel(1, p->dense ? -lg_ws_dense_width((int)p->d) : p->W, p->ws_rpl);
    fsm = p->ws_fwd_smem;
    bsm = p->ws_bwd_smem;
    bblock = dim3(p->ws_bwd_threads);
  }
  auto cl_launch = [&](void* f, bool backward, int clusters = 0, bool allow_split = true,
                       cudaStream_t st = nullptr) -> int {
    E.cl_acs = backward ? p->cl_acs : 0;
    const bool split = backward && p->cl_split && allow_split;
    E.cl_R = split ? p->cl_R_b : p->cl_R;
    E.cl_Q = split ? p->cl_Q_b : p->cl_Q;
    E.cl_E = split ? p->cl_E_b : p->cl_E;
    if (split) f = lg_cl_kernel(1, p->W, p->cl_maxc, 2);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((clusters ? clusters : p->n_groups) * p->cl_CS);
    cfg.blockDim = dim3(split ? p->cl_T_b : p->threads);
    cfg.dynamicSmemBytes = split ? p->cl_smem_split : (backward ? p->cl_smem_b : p->cl_smem);
    cfg.stream = st ? st : p->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = p->cl_CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ++g_launches;
    ensure_smem(f, cfg.dynamicSmemBytes);
    cudaError_t e = cudaLaunchKernelExC(&cfg, f, eargs);
    if (e != cudaSuccess) return fail(LG_CUDA_ERROR, std::string("cluster launch: ") + cudaGetErrorString(e));
    return LG_OK;
  };
  if (p->engine == 5) {
    fwd = lg_cl_kernel(0, p->W, p->cl_maxc, p->cl_small);
    bwd = lg_cl_kernel(1, p->W, p->cl_maxc, p->cl_small);
  }
  if (p->n_groups > 0) rc = p->engine == 5 ? cl_launch(fwd, false) : launch(fwd, grid, block, eargs, fsm, p->stream, p->multi);
  if (rc) return rc;
  p->mark(2);
  if (grad) {
    rc = hook_traces(p, N);
    if (rc) return rc;
  }
  if (grad && S > 0 && p->n_groups > 0) {
    int Ni = (int)N, Sv = S, Tv = T;
    long cnt = (long)S * N;
    void* targs[] = {&p->d_trp, &Sv, &Ni, &Tv, &p->d_spec_t0, &p->d_spec_K, &p->d_trsum};
    rc = launch(lg_trsum_kernel(), dim3((unsigned)((cnt + 255) / 256)), dim3(256), targs, 0, p->stream);
    if (rc) return rc;
    if (p->engine == 5) {
      // LARGE kernels: two-phase backward when the psi_{n-1} / lambda_s(n) store fits in HBM
      bool two = p->cl_aux_ncl > 0 && !std::getenv("LG_CL_FUSED");
      if (two) {
        const long need = (long)p->n_groups * N * p->d;
        if (need > p->bk_cap) {
          p->bkmem.release();
          p->bk_cap = 0;
          p->d_bk_psi = p->bkmem.alloc<double2>((size_t)need);
          p->d_bk_lam = p->bkmem.alloc<double2>((size_t)need * std::max(p->cta_Imax, 1));
          p->d_bk_flag = p->bkmem.alloc<unsigned>((size_t)p->n_groups * p->cl_CS + 3);  // + counter, error, started
          if (p->bkmem.failed) {
            p->bkmem.release();
          } else {
            p->bk_cap = need;
          }
        }
        two = p->bk_cap >= need;
      }
      if (two) {
        // adjoint sweep (n_groups clusters) and derivative-product items; when every adjoint cluster
        // and at least one item cluster fit on the GPU at once, a first item kernel runs on the spare
        // clusters CONCURRENTLY (second stream; items wait on the adjoint's per-step flags; sized so
        // both kernels are co-resident, so the waits cannot starve the adjoint), and a second one
        // takes the adjoint's clusters when it ends.  Both pull items from one atomic counter.
        E.bk_psi = p->d_bk_psi;
        E.bk_lam = p->d_bk_lam;
        E.bk_flag = p->d_bk_flag;
        E.bk_next = p->d_bk_flag + (long)p->n_groups * p->cl_CS;
        E.bk_ranks = p->cl_CS;
        E.bk_conc = 0;
        CK(cudaMemsetAsync(p->d_bk_flag, 0, sizeof(unsigned) * ((size_t)p->n_groups * p->cl_CS + 3), p->stream));
        const long items = (long)p->n_groups * N;
        const bool ilay = p->cli_CS > 0;  // items on their own (LARGE, smaller-cluster) layout
        const int incl = ilay ? p->cli_ncl : p->cl_aux_ncl;
        void* fa = lg_cl_kernel(4, p->W, p->cl_maxc, p->cl_small);
        void* fi = lg_cl_kernel(5, p->W, p->cl_maxc, ilay ? 3 : p->cl_small);
        auto item_launch = [&](int clusters, cudaStream_t st) -> int {
          if (!ilay) return cl_launch(fi, true, clusters, false, st);
          LgEngineArgs Ei = E;
          Ei.cl_acs = 1;
          Ei.cl_R = p->cli_R;
          Ei.cl_Q = 1;
          Ei.cl_E = 0;
          void* iargs[] = {&Ei};
          cudaLaunchConfig_t cfg{};
          cfg.gridDim = dim3(clusters * p->cli_CS);
          cfg.blockDim = dim3(p->cli_T);
          cfg.dynamicSmemBytes = p->cli_smem;
          cfg.stream = st ? st : p->stream;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = p->cli_CS;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          ++g_launches;
          ensure_smem(fi, cfg.dynamicSmemBytes);
          cudaError_t e = cudaLaunchKernelExC(&cfg, fi, iargs);
          if (e != cudaSuccess) return fail(LG_CUDA_ERROR, std::string("item launch: ") + cudaGetErrorString(e));
          return LG_OK;
        };
        // concurrent item kernel: only when the adjoint sweep fits the GPU at once (its clusters then
        // all start; the item kernel checks that and otherwise exits at once, lg_sweep_cl.cuh bk_may_run)
        // More trajectories than cluster slots (c4: 32 on 7): the adjoint sweep's last wave leaves
        // slots free (4 of 7 used).  A concurrent item kernel of that many clusters, launched behind the
        // adjoint sweep, is dispatched once the sweep has no cluster left to issue -- i.e. into those
        // slots -- and bk_may_run makes a cluster that was placed earlier leave at once (LG_CL_TAIL=0: off).
        const int tail_free = !ilay && p->cl_aux_ncl > 0 && p->n_groups > p->cl_aux_ncl && p->n_groups % p->cl_aux_ncl
                                  ? p->cl_aux_ncl - p->n_groups % p->cl_aux_ncl
                                  : 0;
        const char* etail = std::getenv("LG_CL_TAIL");
        const bool tail = tail_free > 0 && !(etail && std::atoi(etail) == 0);
        const bool conc = (p->n_groups < p->cl_aux_ncl || tail) && !std::getenv("LG_CL_SERIAL");
        if (conc) {
          if (!p->stream2) CK(cudaStreamCreateWithFlags(&p->stream2, cudaStreamNonBlocking));
          if (!p->ev_fork) CK(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
          if (!p->ev_join) CK(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
          CK(cudaEventRecord(p->ev_fork, p->stream));
        }
        rc = cl_launch(fa, true, 0, false);
        if (rc) return rc;
        if (conc) {
          CK(cudaStreamWaitEvent(p->stream2, p->ev_fork, 0));
          E.bk_conc = 1;
          rc = item_launch(p->n_groups < p->cl_aux_ncl ? (int)std::min<long>(incl, items) : tail_free, p->stream2);
          E.bk_conc = 0;
          if (rc) return rc;
        }
        rc = item_launch((int)std::min<long>(incl, items), nullptr);
        if (rc) return rc;
        if (conc) {
          CK(cudaEventRecord(p->ev_join, p->stream2));
          CK(cudaStreamWaitEvent(p->stream, p->ev_join, 0));
        }
        unsigned werr = 0;  // item-kernel watchdog (lg_sweep_cl.cuh bk_wait)
        CK(cudaMemcpyAsync(&werr, E.bk_next + 1, sizeof(unsigned), cudaMemcpyDeviceToHost, p->stream));
        CK(cudaStreamSynchronize(p->stream));
        if (werr) return fail(LG_CUDA_ERROR, "two-phase backward: derivative items timed out waiting on the adjoint sweep");
      } else {
        rc = cl_launch(bwd, true);
      }
      if (rc) return rc;
    } else if (p->engine == 4 && p->ws_cluster) {
      cudaLaunchConfig_t cfg{};
      const int csz = 1 + p->cta_Imax + p->Kc * p->ws_nw;
      cfg.gridDim = dim3(p->n_groups * csz);
      cfg.blockDim = bblock;
      cfg.dynamicSmemBytes = bsm;
      cfg.stream = p->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csz;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      ++g_launches;
      void* wsc = lg_ws_kernel(2, p->dense ? -lg_ws_dense_width((int)p->d) : p->W, p->ws_rpl);
      ensure_smem(wsc, cfg.dynamicSmemBytes);
      cudaError_t e = cudaLaunchKernelExC(&cfg, wsc, eargs);
      if (e != cudaSuccess) return fail(LG_CUDA_ERROR, std::string("cluster launch: ") + cudaGetErrorString(e));
    } else {
      rc = launch(bwd, grid, bblock, eargs, bsm, p->stream, p->multi);
      if (rc) return rc;
    }
    if (E.trace) {
      const size_t need = (size_t)p->n_groups * 8 * N * 4;
      std::vector<long long> h(need);
      cudaStreamSynchronize(p->stream);
      cudaMemcpy(h.data(), E.trace, need * sizeof(long long), cudaMemcpyDeviceToHost);
      if (FILE* f = std::fopen(std::getenv("LG_TRACE"), "wb")) {
        std::fwrite(h.data(), sizeof(long long), need, f);
        std::fclose(f);
      }
    }
  }
  rc = hook_raw(p, N);
  if (rc) return rc;
  p->mark(3);
  LgFinalArgs F = final_args(p, N, p->d_ip, p->d_fin, p->d_run, p->d_trp, p->d_grad, p->d_cost);
  void* fargs[] = {&F};
  rc = launch(lg_finalize_kernel(), dim3((unsigned)std::min<long>((N * p->Kc + 255) / 256 + 1, 1024)), dim3(256),
              fargs, 0, p->stream);
  if (rc) return rc;
  p->mark(4);
  p->lastN = N;
  return LG_OK;
}

int check_field(lg_problem* p, long N, double dt, const double* amps) {
  if (!p) return fail(LG_INVALID_ARG, "null problem handle");
  if (p->has_gate_run && p->shard_e < (1L << 40) && !p->hook)
    return fail(LG_UNSUPPORTED, "a sharded running gate cost needs lg_eval_sharded (global traces between sweeps)");
  if (N < 1) return fail(LG_INVALID_ARG, "need at least one step and one channel");
  if (!(dt > 0.0)) return fail(LG_INVALID_ARG, "dt must be positive");
  if (amps)
    for (long q = 0; q < N * p->Kc; ++q)
      if (!std::isfinite(amps[q])) return fail(LG_INVALID_ARG, "control amplitudes must be finite");
  return LG_OK;
}

}  // namespace lgi

using namespace lgi;

// ============================================================================ C ABI

extern "C" {

const char* lg_last_error(void) { return g_err.c_str(); }
const char* lg_version(void) { return "paper_2304_06200_b200 0.1 (sm_100a)"; }

int lg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int lg_make_plan(double norm1, int64_t sigma_prime, double tau, int32_t m_max, int32_t s_max, int32_t* order,
                 int32_t* scaling, double* bound) {
  LgPlannerCtx cx{lg_u_prime(), 0};
  LgPlan p = lg_make_plan(cx, norm1, (long)sigma_prime, tau, m_max, s_max);
  if (p.status == LG_PLAN_BADARG) {
    if (!(norm1 >= 0.0)) {
      char buf[96];
      std::snprintf(buf, sizeof buf, "norm1_a must be non-negative, got %g", norm1);
      return fail(LG_INVALID_ARG, buf);
    }
    return fail(LG_INVALID_ARG, sigma_prime < 0 ? "sigma_prime must be non-negative" : "tau must be positive");
  }
  if (p.status == LG_PLAN_INFEASIBLE) {
    char buf[256];
    std::snprintf(buf, sizeof buf,
                  "no feasible (order, scaling) pair for norm1=%g, sigma_prime=%lld, tau=%g within order<=%d, "
                  "scaling<=%d",
                  norm1, (long long)sigma_prime, tau, m_max, s_max);
    return fail(LG_PLANNING_INFEASIBLE, buf);
  }
  *order = p.order;
  *scaling = p.scaling;
  *bound = p.bound;
  return LG_OK;
}

int lg_make_plans_device(int64_t count, const double* norm1, const int64_t* sigma, double tau, int32_t* order,
                         int32_t* scaling, int32_t* status, int32_t* n_uncertain) {
  DevMem m;
  double* a = m.alloc<double>(count);
  long long* s = m.alloc<long long>(count);
  int4* pl = m.alloc<int4>(count);
  int* fl = m.alloc<int>(1);
  if (!a || !s || !pl || !fl) {
    m.release();
    return fail(LG_CUDA_ERROR, "device allocation failed");
  }
  cudaMemcpy(a, norm1, sizeof(double) * count, cudaMemcpyHostToDevice);
  cudaMemcpy(s, sigma, sizeof(long long) * count, cudaMemcpyHostToDevice);
  cudaMemset(fl, 0, sizeof(int));
  int cnt = (int)count;
  double up = lg_u_prime();
  void* args[] = {&a, &s, &cnt, &tau, &up, &pl, &fl};
  int rc = launch(lg_plans_kernel(), dim3((cnt + 127) / 128), dim3(128), args, 0, 0);
  std::vector<int4> h(count);
  if (!rc) {
    cudaError_t e = cudaMemcpy(h.data(), pl, sizeof(int4) * count, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = fail(LG_CUDA_ERROR, cudaGetErrorString(e));
  }
  m.release();
  if (rc) return rc;
  int unc = 0;
  for (long q = 0; q < count; ++q) {
    if (h[q].z & LG_PLAN_UNCERTAIN) {
      ++unc;
      LgPlannerCtx cx{lg_u_prime(), 0};
      LgPlan hp = lg_make_plan(cx, norm1[q], (long)sigma[q], tau, 60, 10000);
      h[q] = make_int4(hp.order, hp.scaling, hp.status, 0);
    }
    order[q] = h[q].x;
    scaling[q] = h[q].y;
    status[q] = h[q].z;
  }
  *n_uncertain = unc;
  return LG_OK;
}

int lg_problem_create(const lg_problem_desc* desc, lg_problem** out) {
  if (!out) return fail(LG_INVALID_ARG, "null output pointer");
  *out = nullptr;
  int ndev = lg_device_count();
  if (ndev <= 0) return fail(LG_CUDA_ERROR, "no CUDA device available (this library has no CPU fallback)");
  lg_problem* p = new lg_problem();
  int rc = build_problem(desc, p);
  if (rc) {
    std::string keep = g_err;
    delete p;
    g_err = keep;
    return rc;
  }
  *out = p;
  return LG_OK;
}

void lg_problem_destroy(lg_problem* p) { delete p; }

int lg_bench_zgemm(int32_t d, int32_t C, int32_t iters, double* ms) {
  lg_problem tmp;
  tmp.d = d;
  CK(cudaStreamCreate(&tmp.stream));
  DevMem m;
  double2* Ad = m.alloc<double2>((size_t)d * d);
  double2* X = m.alloc<double2>((size_t)d * C);
  double2* cur = m.alloc<double2>((size_t)d * C);
  double2* T = m.alloc<double2>((size_t)d * C);
  if (m.failed) {
    m.release();
    return fail(LG_CUDA_ERROR, "allocation failed");
  }
  cudaMemset(Ad, 0, sizeof(double2) * d * d);
  cudaMemset(X, 0, sizeof(double2) * d * C);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int rc = LG_OK;
  for (int it = 0; it < 3 && !rc; ++it) rc = dense_gemm(&tmp, Ad, X, nullptr, nullptr, C, 0.5, false, false, nullptr, cur, T);
  cudaEventRecord(e0, tmp.stream);
  for (int it = 0; it < iters && !rc; ++it) rc = dense_gemm(&tmp, Ad, X, nullptr, nullptr, C, 0.5, false, false, nullptr, cur, T);
  cudaEventRecord(e1, tmp.stream);
  cudaEventSynchronize(e1);
  float t = 0.f;
  cudaEventElapsedTime(&t, e0, e1);
  *ms = t / iters;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  m.release();
  return rc;
}

int lg_set_stream(lg_problem* p, void* stream) {
  if (!p) return fail(LG_INVALID_ARG, "null problem handle");
  CK(cudaStreamSynchronize(p->stream));
  if (p->own_stream && p->stream) CK(cudaStreamDestroy(p->stream));
  p->stream = (cudaStream_t)stream;
  p->own_stream = false;
  return LG_OK;
}

int64_t lg_launch_count(void) { return g_launches; }

int64_t lg_live_vector_peak(lg_problem* p) { return p ? (int64_t)p->live_peak : 0; }

const char* lg_engine_name(lg_problem* p) {
  if (!p) return "none";
  switch (p->engine) {
    case 0: return "grid:lg_k_backward";
    case 1: return "grid-multi:lg_k_backward";
    case 2: return "cta:lg_k_cta_backward";
    case 3: return p->backend == 1 ? "dense-diag:lg_k_zgemm_taylor" : "dense:lg_k_zgemm_taylor";
    case 4: return p->ws_cluster ? "ws-cluster:lg_k_wsc_backward" : "ws:lg_k_ws_backward";
    case 5: {
      const bool two = p->cl_aux_ncl > 0 && !std::getenv("LG_CL_FUSED");
      if (p->cl_small >= 3)
        return two ? "cluster-large:lg_k_cll_adjoint+lg_k_cll_aux" : "cluster-large:lg_k_cll_backward";
      if (two) return p->cli_CS > 0 ? "cluster-2phase:lg_k_cl_adjoint+lg_k_cll_aux" : "cluster-2phase:lg_k_cl_adjoint+lg_k_cl_aux";
      return p->cl_split ? "cluster-split:lg_k_cl_backward" : "cluster:lg_k_cl_backward";
    }
    default: return "unknown";
  }
}

const char* lg_diag_solver_name(lg_problem* p) { return p ? p->diag_solver : ""; }

int lg_set_timing(lg_problem* p, int enable) {
  if (!p) return fail(LG_INVALID_ARG, "null problem handle");
  if (enable && !p->ev[0])
    for (auto& e : p->ev) CK(cudaEventCreate(&e));
  p->timing = enable != 0;
  for (double& v : p->phase_ms) v = 0.0;
  p->timed_evals = 0;
  return LG_OK;
}

int lg_get_timing(lg_problem* p, double* phase_ms, int64_t* evals) {
  if (!p) return fail(LG_INVALID_ARG, "null problem handle");
  for (int i = 0; i < 4; ++i) phase_ms[i] = p->phase_ms[i];
  *evals = p->timed_evals;
  return LG_OK;
}

int lg_eval_device(lg_problem* p, int64_t n_steps, double dt, const double* d_amps, double* d_cost, double* d_grad) {
  int rc = check_field(p, n_steps, dt, nullptr);
  if (rc) return rc;
  CK(cudaSetDevice(p->device));
  rc = ensure_N(p, n_steps);
  if (rc) return rc;
  if (d_amps != p->d_amps)
    CK(cudaMemcpyAsync(p->d_amps, d_amps, sizeof(double) * n_steps * p->Kc, cudaMemcpyDeviceToDevice, p->stream));
  rc = prepare_steps(p, n_steps, dt, true);
  if (rc) return rc;
  rc = run_sweeps(p, n_steps, true);
  if (rc) return rc;
  if (d_cost) CK(cudaMemcpyAsync(d_cost, p->d_cost, sizeof(double), cudaMemcpyDeviceToDevice, p->stream));
  if (d_grad)
    CK(cudaMemcpyAsync(d_grad, p->d_grad, sizeof(double) * n_steps * p->Kc, cudaMemcpyDeviceToDevice, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  p->collect();
  return LG_OK;
}

int lg_eval(lg_problem* p, int64_t n_steps, double dt, const double* amps, double* cost, double* grad,
            int64_t* live_vector_peak) {
  int rc = check_field(p, n_steps, dt, amps);
  if (rc) return rc;
  if (p->specs.empty()) return fail(LG_INVALID_ARG, "composite cost needs at least one term");
  CK(cudaSetDevice(p->device));
  rc = ensure_N(p, n_steps);
  if (rc) return rc;
  CK(cudaMemcpyAsync(p->d_amps, amps, sizeof(double) * n_steps * p->Kc, cudaMemcpyHostToDevice, p->stream));
  rc = prepare_steps(p, n_steps, dt, true);
  if (rc) return rc;
  rc = run_sweeps(p, n_steps, true);
  if (rc) return rc;
  CK(cudaMemcpyAsync(cost, p->d_cost, sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  CK(cudaMemcpyAsync(grad, p->d_grad, sizeof(double) * n_steps * p->Kc, cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  p->collect();
  if (live_vector_peak) *live_vector_peak = p->live_peak;
  return LG_OK;
}

int lg_set_raw_buffer(lg_problem* p, double* d_raw, int64_t len) {
  if (!p) return fail(LG_INVALID_ARG, "null problem handle");
  if ((d_raw == nullptr) != (len == 0)) return fail(LG_INVALID_ARG, "raw buffer and length must both be set or both 0");
  p->ext_raw = d_raw;
  p->ext_raw_len = len;
  return LG_OK;
}

namespace {
struct HookScope {  // installs the caller's all-reduce hook for one call
  lg_problem* p;
  HookScope(lg_problem* p_, lg_allreduce_fn fn, void* user) : p(p_) {
    p->hook = fn;
    p->hook_user = user;
  }
  ~HookScope() {
    p->hook = nullptr;
    p->hook_user = nullptr;
  }
};
}  // namespace

int lg_eval_sharded(lg_problem* p, int64_t n_steps, double dt, const double* amps, lg_allreduce_fn allreduce,
                    void* user, double* cost, double* grad) {
  if (!allreduce) return fail(LG_INVALID_ARG, "lg_eval_sharded needs an all-reduce hook");
  if (!p) return fail(LG_INVALID_ARG, "null problem handle");
  HookScope hs(p, allreduce, user);
  return lg_eval(p, n_steps, dt, amps, cost, grad, nullptr);
}

int lg_cost_sharded(lg_problem* p, int64_t n_steps, double dt, const double* amps, lg_allreduce_fn allreduce,
                    void* user, double* cost) {
  if (!allreduce) return fail(LG_INVALID_ARG, "lg_cost_sharded needs an all-reduce hook");
  if (!p) return fail(LG_INVALID_ARG, "null problem handle");
  HookScope hs(p, allreduce, user);
  return lg_cost(p, n_steps, dt, amps, cost);
}

int lg_cost(lg_problem* p, int64_t n_steps, double dt, const double* amps, double* cost) {
  int rc = check_field(p, n_steps, dt, amps);
  if (rc) return rc;
  if (p->specs.empty()) return fail(LG_INVALID_ARG, "composite cost needs at least one term");
  CK(cudaSetDevice(p->device));
  rc = ensure_N(p, n_steps);
  if (rc) return rc;
  CK(cudaMemcpyAsync(p->d_amps, amps, sizeof(double) * n_steps * p->Kc, cudaMemcpyHostToDevice, p->stream));
  rc = prepare_steps(p, n_steps, dt, false);
  if (rc) return rc;
  rc = run_sweeps(p, n_steps, false);
  if (rc) return rc;
  CK(cudaMemcpyAsync(cost, p->d_cost, sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  return LG_OK;
}

// composite_cost for k candidate fields in one forward launch (src/optimizer.py:153-170: the
// backtracking line search's trial fields): the k x N step generators and plans are prepared as
// one batch of steps, and the forward kernel takes candidate c from blockIdx.y with its own
// slice of generators, plans and raw outputs.  Costs are bit-identical to k lg_cost calls.
int lg_cost_batch(lg_problem* p, int32_t n_fields, int64_t n_steps, double dt, const double* amps, double* costs) {
  const long k = n_fields, N = n_steps;
  if (!p) return fail(LG_INVALID_ARG, "null problem handle");
  if (k < 1) return fail(LG_INVALID_ARG, "need at least one candidate field");
  int rc = check_field(p, k * N, dt, amps);
  if (rc) return rc;
  if (p->specs.empty()) return fail(LG_INVALID_ARG, "composite cost needs at least one term");
  if (p->backend == 1 || !(p->engine == 4 || p->engine == 5) || p->shard_e < (1L << 40) || p->n_groups < 1)
    return fail(LG_UNSUPPORTED, "batched candidates need the warp-specialised or cluster engine on an unsharded problem");
  if (k > 65535) return fail(LG_INVALID_ARG, "too many candidate fields");
  CK(cudaSetDevice(p->device));
  rc = ensure_N(p, k * N);
  if (rc) return rc;
  CK(cudaMemcpyAsync(p->d_amps, amps, sizeof(double) * k * N * p->Kc, cudaMemcpyHostToDevice, p->stream));
  rc = prepare_steps(p, k * N, dt, false);
  if (rc) return rc;
  const long S = std::max<long>((long)p->specs.size(), 1), T = std::max(p->T_total, 1);
  const long runsz = (S * T + 1) / 2 * 2;  // keeps trp (complex) 16-byte aligned
  const long per = 2 * S * T + runsz + 2 * S * N * T;  // doubles: fin (complex), run, trp (complex)
  if (k > p->bcap_k || N > p->bcap_N) {
    p->bmem.release();
    p->bcap_k = p->bcap_N = 0;
    p->d_bat = p->bmem.alloc<double>((size_t)k * per);
    p->d_bpsi = p->bmem.alloc<double2>((size_t)k * T * p->d);
    p->d_bcost = p->bmem.alloc<double>((size_t)k);
    p->d_bEA = p->bmem.alloc<LgEngineArgs>((size_t)k);
    if (p->bmem.failed) {
      p->bmem.release();
      return fail(LG_CUDA_ERROR, "device allocation failed (candidate batch)");
    }
    p->bcap_k = k;
    p->bcap_N = N;
  }
  CK(cudaMemsetAsync(p->d_bat, 0, sizeof(double) * k * per, p->stream));
  std::vector<LgEngineArgs> ea((size_t)k);
  const long Wst = p->dense ? p->d : p->W;  // generator row width of the step table A[N][W][d]
  for (long c = 0; c < k; ++c) {
    LgEngineArgs E = engine_args(p, N);
    double* b = p->d_bat + c * per;
    E.A = p->d_A + c * N * Wst * p->d;
    E.plan = p->d_plan + c * N * (p->Kc + 1);
    E.rtab = p->d_rtab ? p->d_rtab + c * N * 64 : nullptr;
    E.fin = reinterpret_cast<double2*>(b);
    E.run = b + 2 * S * T;
    E.trp = reinterpret_cast<double2*>(b + 2 * S * T + runsz);
    E.psiN = p->d_bpsi + c * T * p->d;
    E.cl_acs = 0;
    E.trace = nullptr;
    ea[c] = E;
  }
  CK(cudaMemcpyAsync(p->d_bEA, ea.data(), sizeof(LgEngineArgs) * k, cudaMemcpyHostToDevice, p->stream));
  void* bargs[] = {&p->d_bEA};
  cudaError_t e;
  if (p->engine == 5) {
    void* f = lg_cl_kernel(3, p->W, p->cl_maxc, p->cl_small);
    if (!f) return fail(LG_UNSUPPORTED, "no batched forward kernel for this cluster layout");
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p->n_groups * p->cl_CS, (unsigned)k);
    cfg.blockDim = dim3(p->threads);
    cfg.dynamicSmemBytes = p->cl_smem;
    cfg.stream = p->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = p->cl_CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ensure_smem(f, cfg.dynamicSmemBytes);
    if (p->cl_CS > 8) cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    ++g_launches;
    e = cudaLaunchKernelExC(&cfg, f, bargs);
  } else {
    void* f = lg_ws_kernel(3, p->dense ? -lg_ws_dense_width((int)p->d) : p->W, p->ws_rpl);
    if (!f) return fail(LG_UNSUPPORTED, "no batched forward kernel for this problem");
    ensure_smem(f, p->ws_fwd_smem);
    ++g_launches;
    e = cudaLaunchKernel(f, dim3(p->n_groups * p->n_slabs, (unsigned)k), dim3(p->threads), bargs, p->ws_fwd_smem,
                         p->stream);
  }
  if (e != cudaSuccess) return fail(LG_CUDA_ERROR, std::string("batched forward launch: ") + cudaGetErrorString(e));
  for (long c = 0; c < k; ++c) {
    const double* b = p->d_bat + c * per;
    LgFinalArgs F = final_args(p, N, p->d_ip, reinterpret_cast<const double2*>(b), b + 2 * S * T,
                               reinterpret_cast<const double2*>(b + 2 * S * T + runsz), p->d_grad, p->d_bcost + c);
    F.Kc = 0;  // cost only
    void* fargs[] = {&F};
    rc = launch(lg_finalize_kernel(), dim3(1), dim3(32), fargs, 0, p->stream);
    if (rc) return rc;
  }
  CK(cudaMemcpyAsync(costs, p->d_bcost, sizeof(double) * k, cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  return LG_OK;
}

int lg_forward_states(lg_problem* p, int64_t n_steps, double dt, const double* amps, double* out) {
  int rc = check_field(p, n_steps, dt, amps);
  if (rc) return rc;
  if (p->set_T[0] == 0) return fail(LG_INVALID_ARG, "problem has no initial states");
  CK(cudaSetDevice(p->device));
  rc = ensure_N(p, n_steps);
  if (rc) return rc;
  CK(cudaMemcpyAsync(p->d_amps, amps, sizeof(double) * n_steps * p->Kc, cudaMemcpyHostToDevice, p->stream));
  rc = prepare_steps(p, n_steps, dt, false);
  if (rc) return rc;
  rc = run_sweeps(p, n_steps, false);
  if (rc) return rc;
  CK(cudaMemcpyAsync(out, p->d_psiN + (size_t)p->set_t0[0] * p->d, sizeof(double2) * p->set_T[0] * p->d,
                     cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  return LG_OK;
}

// y = M x for one column-major d x d complex matrix (one CTA; rows over the threads)
__global__ void lg_k_zgemv_one(const double2* __restrict__ M, const double2* __restrict__ x, int d, double2* __restrict__ y) {
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int j = 0; j < d; ++j) {
      const double2 m = M[(long)j * d + i], v = x[j];
      acc.x += m.x * v.x - m.y * v.y;
      acc.y += m.x * v.y + m.y * v.x;
    }
    y[i] = acc;
  }
}

int lg_step_derivative(lg_problem* p, int64_t n_steps, double dt, const double* amps, int64_t step, int32_t channel,
                       const double* psi, double* out) {
  int rc = check_field(p, n_steps, dt, amps);
  if (rc) return rc;
  if (!psi || !out) return fail(LG_INVALID_ARG, "null state pointer");
  if (p->backend != 1)
    return fail(LG_UNSUPPORTED, "lg_step_derivative serves the DIAGONALIZATION backend (Taylor problems: lg_expm_apply "
                                "on the embedded generator)");
  if (step < 0 || step >= n_steps) return fail(LG_INDEX_ERROR, "step out of range");
  if (channel < 0 || channel >= p->Kc) return fail(LG_INDEX_ERROR, "control channel out of range");
  CK(cudaSetDevice(p->device));
  rc = ensure_N(p, n_steps);
  if (rc) return rc;
  CK(cudaMemcpyAsync(p->d_amps, amps, sizeof(double) * n_steps * p->Kc, cudaMemcpyHostToDevice, p->stream));
  rc = prepare_steps(p, n_steps, dt, true);  // factorises every step and forms dU_n/da_k in p->d_D
  if (rc) return rc;
  const long d = p->d, dd = d * d;
  double2* buf = nullptr;
  CK(cudaMallocAsync(&buf, sizeof(double2) * 2 * d, p->stream));
  cudaError_t e = cudaMemcpyAsync(buf, psi, sizeof(double2) * d, cudaMemcpyHostToDevice, p->stream);
  if (e == cudaSuccess) {
    lg_k_zgemv_one<<<1, 256, 0, p->stream>>>(p->d_D + ((long)step * p->Kc + channel) * dd, buf, (int)d, buf + d);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, buf + d, sizeof(double2) * d, cudaMemcpyDeviceToHost, p->stream);
  cudaFreeAsync(buf, p->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
  if (e != cudaSuccess) return fail(LG_CUDA_ERROR, std::string("lg_step_derivative: ") + cudaGetErrorString(e));
  return LG_OK;
}

int lg_plan_table(lg_problem* p, int64_t n_steps, double dt, const double* amps, double* norm1, int64_t* sigma,
                  int32_t* order, int32_t* scaling, double* aux_arg, int64_t* aux_sigma, int32_t* aux_order,
                  int32_t* aux_scaling) {
  int rc = check_field(p, n_steps, dt, amps);
  if (rc) return rc;
  if (p->backend == 1) return fail(LG_UNSUPPORTED, "the DIAGONALIZATION backend has no Taylor plans");
  CK(cudaSetDevice(p->device));
  rc = ensure_N(p, n_steps);
  if (rc) return rc;
  CK(cudaMemcpyAsync(p->d_amps, amps, sizeof(double) * n_steps * p->Kc, cudaMemcpyHostToDevice, p->stream));
  rc = prepare_steps(p, n_steps, dt, true);
  if (rc) return rc;
  const long N = n_steps, Kc = p->Kc;
  std::vector<int4> pl((size_t)N * (Kc + 1));
  std::vector<long long> sp(N), asp((size_t)N * Kc);
  CK(cudaMemcpy(norm1, p->d_norm1, sizeof(double) * N, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(sp.data(), p->d_sp, sizeof(long long) * N, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(aux_arg, p->d_aux_arg, sizeof(double) * N * Kc, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(asp.data(), p->d_aux_sp, sizeof(long long) * N * Kc, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(pl.data(), p->d_plan, sizeof(int4) * pl.size(), cudaMemcpyDeviceToHost));
  for (long n = 0; n < N; ++n) {
    sigma[n] = sp[n];
    order[n] = pl[n * (Kc + 1)].x;
    scaling[n] = pl[n * (Kc + 1)].y;
    for (long c = 0; c < Kc; ++c) {
      aux_sigma[n * Kc + c] = asp[n * Kc + c];
      aux_order[n * Kc + c] = pl[n * (Kc + 1) + 1 + c].x;
      aux_scaling[n * Kc + c] = pl[n * (Kc + 1) + 1 + c].y;
    }
  }
  return LG_OK;
}

int64_t lg_raw_size(lg_problem* p, int64_t N) {
  const long S = (long)p->specs.size(), T = p->T_total, Kc = p->Kc;
  // ip, fin, trp (complex) + run (real)
  return 2 * (N * S * Kc * T + S * T + S * N * T) + S * T;
}

int lg_raw_get(lg_problem* p, double* raw) {
  const long N = p->lastN, S = (long)p->specs.size(), T = p->T_total, Kc = p->Kc;
  double* q = raw;
  CK(cudaMemcpy(q, p->d_ip, sizeof(double2) * N * S * Kc * T, cudaMemcpyDeviceToHost));
  q += 2 * N * S * Kc * T;
  CK(cudaMemcpy(q, p->d_fin, sizeof(double2) * S * T, cudaMemcpyDeviceToHost));
  q += 2 * S * T;
  CK(cudaMemcpy(q, p->d_trp, sizeof(double2) * S * N * T, cudaMemcpyDeviceToHost));
  q += 2 * S * N * T;
  CK(cudaMemcpy(q, p->d_run, sizeof(double) * S * T, cudaMemcpyDeviceToHost));
  return LG_OK;
}

int lg_finalize_raw(int32_t n_terms, const int32_t* kinds, const double* weights, const int32_t* t0, const int32_t* K,
                    int64_t N, int32_t Kc, int32_t T, const double* raw, double* cost, double* grad) {
  if (n_terms < 0 || n_terms > LG_MAX_SPECS || N < 1 || Kc < 1 || T < 0) return fail(LG_INVALID_ARG, "bad sizes");
  const long S = n_terms;
  LgFinalArgs F{};
  F.N = (int)N;
  F.Kc = Kc;
  F.n_specs = n_terms;
  F.T_total = T;
  for (int s = 0; s < n_terms; ++s) {
    F.kind[s] = kinds[s];
    F.weight[s] = weights[s];
    F.t0[s] = t0[s];
    F.K[s] = K[s];
  }
  F.ip = (const double2*)raw;
  F.fin = F.ip + N * S * Kc * T;
  F.trp = F.fin + S * T;
  F.run = (const double*)(F.trp + S * N * T);
  for (long q = 0; q < N * Kc; ++q) grad[q] = lg_final_grad(F, q);
  *cost = lg_final_cost(F);
  return LG_OK;
}

void lg_np_cabs_host(int64_t n, const double* z, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = lg_np_cabs(z[2 * i], z[2 * i + 1]);
}
double lg_np_pairwise_host(int64_t n, const double* a) {
  auto get = [&](long k) { return a[k]; };
  return lg_np_pairwise(get, 0, (long)n);
}
double lg_np_reduce_host(int64_t n, const double* a) {
  auto get = [&](long k) { return a[k]; };
  return lg_np_reduce(get, 0, (long)n);
}

int lg_expm_plan_inputs(const lg_matrix* a, double* norm1, int64_t* sigma_prime) {
  if (!a || !norm1 || !sigma_prime || a->n < 0) return fail(LG_INVALID_ARG, "null argument");
  Mat m;
  int rc = parse_mat(*a, a->n, &m, "generator");
  if (rc) return rc;
  const long n = m.n;
  double best = 0.0;
  if (m.dense) {
    // abs(F-array).sum(axis=0).max(): numpy pairwise per contiguous column (src/sparse.py:201-222)
    std::vector<double> col((size_t)n);
    for (long j = 0; j < n; ++j) {
      for (long i = 0; i < n; ++i) col[i] = lg_np_cabs(m.vals[(size_t)j * n + i].x, m.vals[(size_t)j * n + i].y);
      auto get = [&](long k) { return col[k]; };
      const double sj = lg_np_pairwise(get, 0, n);
      best = (j == 0 || sj > best) ? sj : best;
    }
    *sigma_prime = n;  // DenseMatrix.max_row_nnz returns n_cols
  } else {
    // np.bincount(col, |v|, minlength=n).max(): sequential per column in CSR order (src/sparse.py:90-121)
    std::vector<double> cs((size_t)n, 0.0);
    for (size_t k = 0; k < m.indices.size(); ++k) cs[m.indices[k]] += lg_np_cabs(m.vals[k].x, m.vals[k].y);
    for (long j = 0; j < n; ++j) best = (j == 0 || cs[j] > best) ? cs[j] : best;
    long sp = 0;
    for (long i = 0; i < n; ++i) sp = std::max(sp, m.indptr[i + 1] - m.indptr[i]);
    *sigma_prime = sp;
  }
  *norm1 = best;
  return LG_OK;
}

int lg_expm_apply(const lg_matrix* a, int64_t n_vec, const double* psi, int32_t order, int32_t scaling,
                  double* out, int32_t device) {
  if (!a || !psi || !out || n_vec < 1 || order < 0 || scaling < 1) return fail(LG_INVALID_ARG, "bad arguments");
  Mat m;
  int rc = parse_mat(*a, a->n, &m, "generator");
  if (rc) return rc;
  const long d = m.n;
  if (d < 1) return fail(LG_INVALID_ARG, "empty generator");
  if (order == 0) {  // zero generator plan: exp(A) psi = psi
    std::memcpy(out, psi, sizeof(double2) * d * n_vec);
    return LG_OK;
  }
  int W = 1;
  std::vector<int> cols;
  std::vector<double2> vals;
  to_ell(m, &W, cols, vals, nullptr);
  CK(cudaSetDevice(device));
  DevMem mem;
  const int* dcols = mem.upload(cols);
  const double2* dvals = mem.upload(vals);
  std::vector<double2> h((size_t)d * n_vec);
  std::memcpy(h.data(), psi, sizeof(double2) * h.size());
  const double2* dpsi = mem.upload(h);
  double2* cur = mem.alloc<double2>(h.size());
  double2* t0 = mem.alloc<double2>(h.size());
  double2* t1 = mem.alloc<double2>(h.size());
  if (!dcols || !dvals || !dpsi || !cur || !t0 || !t1) return fail(LG_CUDA_ERROR, "device allocation failed");
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  LgEllTaylorArgs A{};
  A.d = (int)d;
  A.W = W;
  A.ncol = (int)n_vec;
  A.cols = dcols;
  A.vals = dvals;
  A.xin = dpsi;
  A.cur = cur;
  const double2* x = dpsi;
  double2* outs[2] = {t0, t1};
  int k = 0;
  const dim3 grid((unsigned)std::min<long>((d + 255) / 256, 1024), (unsigned)n_vec);
  for (int s = 0; s < scaling; ++s)
    for (int j = 1; j <= order && rc == LG_OK; ++j) {
      A.first = s == 0 && j == 1;
      A.last = j == order;
      A.r = 1.0 / ((double)scaling * j);  // multiply by the reciprocal, src/expm.py:349
      A.X = x;
      A.T = outs[k];
      void* args[] = {&A};
      rc = launch(lg_ell_taylor_kernel(), grid, dim3(256), args, 0, st);
      x = outs[k];
      k ^= 1;
    }
  if (rc == LG_OK) {
    cudaMemcpyAsync(out, cur, sizeof(double2) * h.size(), cudaMemcpyDeviceToHost, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(LG_CUDA_ERROR, cudaGetErrorString(e));
  }
  cudaStreamDestroy(st);
  return rc;
}

int lg_matvec(const lg_matrix* a, int64_t n_vec, const double* x, double* y, int32_t device) {
  if (!a || !x || !y || n_vec < 1) return fail(LG_INVALID_ARG, "bad arguments");
  Mat m;
  int rc = parse_mat(*a, a->n, &m, "matrix");
  if (rc) return rc;
  const long d = m.n;
  if (d < 1) return fail(LG_INVALID_ARG, "empty matrix");
  int W = 1;
  std::vector<int> cols;
  std::vector<double2> vals;
  to_ell(m, &W, cols, vals, nullptr);
  CK(cudaSetDevice(device));
  DevMem mem;
  const int* dcols = mem.upload(cols);
  const double2* dvals = mem.upload(vals);
  std::vector<double2> h((size_t)d * n_vec);
  std::memcpy(h.data(), x, sizeof(double2) * h.size());
  const double2* dx = mem.upload(h);
  double2* dy = mem.alloc<double2>(h.size());
  if (!dcols || !dvals || !dx || !dy) return fail(LG_CUDA_ERROR, "device allocation failed");
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  for (int64_t b0 = 0; b0 < n_vec && rc == LG_OK; b0 += 64) {
    LgEllArgs A{};
    A.d = (int)d;
    A.W = W;
    A.ncol = (int)std::min<int64_t>(64, n_vec - b0);
    A.accumulate = 0;
    A.cols = dcols;
    A.vals = dvals;
    for (int q = 0; q < A.ncol; ++q) {
      A.x[q] = dx + (b0 + q) * d;
      A.y[q] = dy + (b0 + q) * d;
    }
    void* args[] = {&A};
    rc = launch(lg_ell_kernel(), dim3((unsigned)((d + 255) / 256), (unsigned)A.ncol), dim3(256), args, 0, st);
  }
  if (rc == LG_OK) {
    cudaMemcpyAsync(y, dy, sizeof(double2) * h.size(), cudaMemcpyDeviceToHost, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(LG_CUDA_ERROR, cudaGetErrorString(e));
  }
  cudaStreamDestroy(st);
  return rc;
}

int lg_finalize_host(lg_problem* p, int64_t N, const double* raw, double* cost, double* grad) {
  const long S = (long)p->specs.size(), T = p->T_total, Kc = p->Kc;
  const double2* ip = (const double2*)raw;
  const double2* fin = ip + N * S * Kc * T;
  const double2* trp = fin + S * T;
  const double* run = (const double*)(trp + S * N * T);
  LgFinalArgs F = final_args(p, N, ip, fin, run, trp, grad, cost);
  for (long q = 0; q < N * Kc; ++q) grad[q] = lg_final_grad(F, q);
  *cost = lg_final_cost(F);
  return LG_OK;
}

}  // extern "C"
