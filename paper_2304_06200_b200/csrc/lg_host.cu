// Host units, part 1: problem ingestion (lg_problem_create: ControlProblem + CostTerm validation
// and device upload, src/costs.py:96-168 -- the union ELL pattern of H_s and every h_c shared by
// all N step generators) and the per-evaluation preparation (all generators, planner inputs and
// plans, src/derivatives.py:105-110, src/expm.py:279-303) that every engine consumes.
#include "lg_host.h"

namespace lgi {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int parse_mat(const lg_matrix& m, long d, Mat* out, const char* what) {
  if (m.n != d) return fail(LG_INVALID_ARG, std::string(what) + " has mismatched shape");
  out->dense = m.dense != 0;
  out->n = d;
  if (out->dense) {
    if (!m.values) return fail(LG_INVALID_ARG, std::string(what) + ": missing dense values");
    out->vals.resize((size_t)d * d);
    std::memcpy(out->vals.data(), m.values, sizeof(double2) * d * d);
  } else {
    if (!m.row_offsets || (m.nnz && (!m.col_indices || !m.values)))
      return fail(LG_INVALID_ARG, std::string(what) + ": missing CSR arrays");
    out->indptr.assign(m.row_offsets, m.row_offsets + d + 1);
    out->indices.assign(m.col_indices, m.col_indices + m.nnz);
    out->vals.resize(m.nnz);
    if (m.nnz) std::memcpy(out->vals.data(), m.values, sizeof(double2) * m.nnz);
    if (out->indptr[0] != 0 || out->indptr[d] != m.nnz)
      return fail(LG_INVALID_ARG, std::string(what) + ": malformed row offsets");
    for (long i = 0; i < d; ++i) {
      if (out->indptr[i + 1] < out->indptr[i]) return fail(LG_INVALID_ARG, std::string(what) + ": malformed row offsets");
      for (long k = out->indptr[i]; k < out->indptr[i + 1]; ++k) {
        if (out->indices[k] < 0 || out->indices[k] >= d)
          return fail(LG_INVALID_ARG, std::string(what) + ": column index out of range");
        if (k > out->indptr[i] && out->indices[k] <= out->indices[k - 1])
          return fail(LG_INVALID_ARG, std::string(what) + ": columns must be strictly increasing per row");
      }
    }
  }
  return LG_OK;
}

// ELL of one operator (for the engine): W = widest row, padded with (col = row, value 0).
void to_ell(const Mat& m, int* W_out, std::vector<int>& cols, std::vector<double2>& vals, std::vector<int>* rowlen) {
  const long d = m.n;
  int W = 0;
  if (m.dense) {
    W = (int)d;
  } else {
    for (long i = 0; i < d; ++i) W = std::max<int>(W, (int)(m.indptr[i + 1] - m.indptr[i]));
  }
  W = std::max(W, 1);
  *W_out = W;
  cols.assign((size_t)W * d, 0);
  vals.assign((size_t)W * d, make_double2(0.0, 0.0));
  if (rowlen) rowlen->assign(d, 0);
  for (long i = 0; i < d; ++i) {
    if (m.dense) {
      for (long w = 0; w < d; ++w) {
        cols[w * d + i] = (int)w;
        vals[w * d + i] = m.vals[w * d + i];
      }
      if (rowlen) (*rowlen)[i] = (int)d;
    } else {
      long L = m.indptr[i + 1] - m.indptr[i];
      for (long w = 0; w < W; ++w) {
        if (w < L) {
          cols[w * d + i] = (int)m.indices[m.indptr[i] + w];
          vals[w * d + i] = m.vals[m.indptr[i] + w];
        } else {
          cols[w * d + i] = (int)i;
        }
      }
      if (rowlen) (*rowlen)[i] = (int)L;
    }
  }
}

// numpy-exact statistics of A_c = -i dt h_c (src/derivatives.py:148,166-184; src/sparse.py:90-121,201-222)
int prepare_dt(lg_problem* p, double dt) {
  if (p->cached_dt == dt) return LG_OK;
  p->dtmem.release();
  const long d = p->d;
  const int Kc = p->Kc;
  std::vector<double> ccol((size_t)Kc * d, 0.0), crow((size_t)Kc * d, 0.0), acabs, acabs_dense;
  std::vector<int> cnnz((size_t)Kc * d, 0), acrow((size_t)Kc * d, 0);
  std::vector<double2> Ac((size_t)Kc * p->Wc * d, make_double2(0.0, 0.0));
  if (!p->dense && p->materialise) acabs.assign((size_t)Kc * p->Wc * d, 0.0);
  if (p->dense && p->materialise) acabs_dense.assign((size_t)Kc * d * d, 0.0);
  for (int c = 0; c < Kc; ++c) {
    const Mat& m = p->hc[c];
    if (!p->dense_large)
      for (size_t q = 0; q < (size_t)p->Wc * d; ++q)
        Ac[(size_t)c * p->Wc * d + q] = gen_host(p->cvals[(size_t)c * p->Wc * d + q], dt);
    if (m.dense) {
      std::vector<double> a((size_t)d * d);
      for (size_t q = 0; q < a.size(); ++q) {
        double2 g = gen_host(m.vals[q], dt);
        a[q] = lg_np_cabs(g.x, g.y);
      }
      for (long j = 0; j < d; ++j) {
        auto get = [&](long k) { return a[(size_t)j * d + k]; };
        ccol[(size_t)c * d + j] = lg_np_pairwise(get, 0, d);
      }
      for (long i = 0; i < d; ++i) {
        double r = 0.0;
        for (long j = 0; j < d; ++j) r = r + a[(size_t)j * d + i];
        crow[(size_t)c * d + i] = r;
        cnnz[(size_t)c * d + i] = (int)d;
      }
      if (!acabs_dense.empty()) std::copy(a.begin(), a.end(), acabs_dense.begin() + (size_t)c * d * d);
    } else {
      std::vector<double> colsum(d, 0.0);
      for (long i = 0; i < d; ++i) {
        const long k0 = m.indptr[i], k1 = m.indptr[i + 1];
        std::vector<double> av;
        for (long k = k0; k < k1; ++k) {
          double2 g = gen_host(m.vals[k], dt);
          double a = lg_np_cabs(g.x, g.y);
          av.push_back(a);
          colsum[m.indices[k]] = colsum[m.indices[k]] + a;  // bincount: sequential, CSR order
        }
        auto get = [&](long k) { return av[k]; };
        crow[(size_t)c * d + i] = lg_np_reduce(get, 0, (long)av.size());
        cnnz[(size_t)c * d + i] = (int)av.size();
        acrow[(size_t)c * d + i] = (int)av.size();
        if (!acabs.empty())
          for (size_t k = 0; k < av.size(); ++k) acabs[((size_t)c * p->Wc + k) * d + i] = av[k];
        if (!acabs_dense.empty())
          for (long k = k0; k < k1; ++k) acabs_dense[(size_t)c * d * d + (size_t)m.indices[k] * d + i] = av[k - k0];
      }
      std::copy(colsum.begin(), colsum.end(), ccol.begin() + (size_t)c * d);
    }
  }
  p->d_Ac = p->dtmem.upload(Ac);
  p->d_ctrl_col = p->dtmem.upload(ccol);
  p->d_ctrl_row = p->dtmem.upload(crow);
  p->d_ctrl_nnz = p->dtmem.upload(cnnz);
  p->d_ac_rowlen = p->dtmem.upload(acrow);
  p->d_ac_abs = acabs.empty() ? nullptr : p->dtmem.upload(acabs);
  p->d_ac_abs_dense = acabs_dense.empty() ? nullptr : p->dtmem.upload(acabs_dense);
  if (p->dtmem.failed) {
    p->dtmem.release();
    return fail(LG_CUDA_ERROR, "device allocation failed (per-dt data)");
  }
  p->cached_dt = dt;
  return LG_OK;
}

int ensure_N(lg_problem* p, long N) {
  if (N <= p->capN) return LG_OK;
  p->nmem.release();
  const long d = p->d;
  const int Kc = p->Kc, S = (int)p->specs.size(), T = p->T_total;
  DevMem& m = p->nmem;
  p->d_amps = m.alloc<double>((size_t)N * Kc);
  p->d_A = p->dense_large ? m.alloc<double2>(1) : m.alloc<double2>((size_t)N * p->W * d);
  p->d_norm1 = m.alloc<double>(N);
  p->d_sp = m.alloc<long long>(N);
  p->d_aux_arg = m.alloc<double>((size_t)N * Kc);
  p->d_aux_sp = m.alloc<long long>((size_t)N * Kc);
  p->d_parg = m.alloc<double>((size_t)N * (Kc + 1));
  p->d_psp = m.alloc<long long>((size_t)N * (Kc + 1));
  p->d_plan = m.alloc<int4>((size_t)N * (Kc + 1));
  p->d_rtab = m.alloc<double>((size_t)N * 64);
  p->d_flag = m.alloc<int>(1);
  {
    // [ip | fin | trp | run], the lg_raw_get layout, so one all-reduce covers a shard's scalars
    const size_t Sx = std::max(S, 1), Tx = std::max(T, 1);
    const size_t nip = (size_t)N * Sx * Kc * Tx, nfin = Sx * Tx, ntrp = Sx * N * Tx, nrun = Sx * Tx;
    p->d_raw = m.alloc<double>(2 * (nip + nfin + ntrp) + nrun);
  }
  p->d_trsum = m.alloc<double2>((size_t)std::max(S, 1) * N);
  p->d_psiN = m.alloc<double2>((size_t)std::max(T, 1) * d);
  p->d_grad = m.alloc<double>((size_t)N * Kc);
  p->d_cost = m.alloc<double>(1);
  std::vector<int> st0(std::max(S, 1), 0), sK(std::max(S, 1), 0);
  for (int s = 0; s < S; ++s) {
    st0[s] = p->set_t0[p->specs[s].set];
    sK[s] = p->set_T[p->specs[s].set];
  }
  p->d_spec_t0 = m.upload(st0);
  p->d_spec_K = m.upload(sK);
  if (m.failed) {  // every buffer or none: a partial set would leave null pointers for the kernels
    m.release();
    p->capN = 0;
    return fail(LG_CUDA_ERROR, "device allocation failed (per-step buffers)");
  }
  p->capN = N;
  return LG_OK;
}

long long g_launches = 0;  // kernels this library launched (lg_launch_count)

// The dynamic shared-memory limit is a per-function (per-device) attribute: problems that share a
// kernel but not its size set it before each launch, so one problem's setting never truncates
// another's.
void ensure_smem(void* f, size_t smem) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

int launch(void* f, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t st, bool coop) {
  ++g_launches;
  ensure_smem(f, smem);
  cudaError_t e = coop ? cudaLaunchCooperativeKernel(f, grid, block, args, smem, st)
                       : cudaLaunchKernel(f, grid, block, args, smem, st);
  if (e != cudaSuccess) return fail(LG_CUDA_ERROR, std::string("kernel launch: ") + cudaGetErrorString(e));
  return LG_OK;
}

// Steps 1-2: generators, planner inputs, plans (all steps at once).
int prepare_steps(lg_problem* p, long N, double dt, bool need_aux) {
  if (p->backend == 1) return prepare_diag(p, N, dt, need_aux);
  p->mark(0);
  int rc = prepare_dt(p, dt);
  if (rc) return rc;
  LgPrepArgs P{};
  P.d = (int)p->d;
  P.Kc = p->Kc;
  P.N = (int)N;
  P.dt = dt;
  P.amps = p->d_amps;
  P.dense = p->dense;
  P.materialise = p->materialise;
  P.W = p->W;
  P.rowlen = p->d_rowlen;
  P.src_s = p->d_src_s;
  P.src_c = p->d_src_c;
  P.hs_vals = p->d_hs;
  P.hc_vals = p->d_hc_ptrs;
  P.colptr = p->d_colptr;
  P.colent = p->d_colent;
  P.hs_dense = p->d_hs_dense;
  P.hc_dense = p->d_hc_dense_ptrs;
  P.ctrl_col = p->d_ctrl_col;
  P.ctrl_row = p->d_ctrl_row;
  P.ctrl_nnz = p->d_ctrl_nnz;
  P.Wc = p->Wc;
  P.ac_rowlen = p->d_ac_rowlen;
  P.ac_abs = p->d_ac_abs;
  P.ac_abs_dense = p->d_ac_abs_dense;
  P.A = p->dense_large ? nullptr : p->d_A;
  P.norm1 = p->d_norm1;
  P.sp = p->d_sp;
  P.aux_arg = p->d_aux_arg;
  P.aux_sp = p->d_aux_sp;
  void* args[] = {&P};
  rc = launch(p->dense ? lg_prep_dense_kernel() : lg_prep_sparse_kernel(), dim3((unsigned)N), dim3(256), args, 0,
              p->stream);
  if (rc) return rc;
  int Kc = p->Kc;
  int count = (int)(N * (Kc + 1));
  int Ni = (int)N;
  void* gargs[] = {&p->d_norm1, &p->d_sp, &p->d_aux_arg, &p->d_aux_sp, &Ni, &Kc, &p->d_parg, &p->d_psp};
  rc = launch(lg_gather_kernel(), dim3((count + 255) / 256), dim3(256), gargs, 0, p->stream);
  if (rc) return rc;
  CK(cudaMemsetAsync(p->d_flag, 0, sizeof(int), p->stream));
  double tau = p->tau, up = lg_u_prime();
  void* pargs[] = {&p->d_parg, &p->d_psp, &count, &tau, &up, &p->d_plan, &p->d_flag};
  rc = launch(lg_plans_kernel(), dim3((count + 127) / 128), dim3(128), pargs, 0, p->stream);
  if (rc) return rc;
  int flagged = 0;
  CK(cudaMemcpyAsync(&flagged, p->d_flag, sizeof(int), cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  if (flagged) {
    std::vector<int4> plans(count);
    std::vector<double> arg(count);
    std::vector<long long> sp(count);
    CK(cudaMemcpy(plans.data(), p->d_plan, sizeof(int4) * count, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(arg.data(), p->d_parg, sizeof(double) * count, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sp.data(), p->d_psp, sizeof(long long) * count, cudaMemcpyDeviceToHost));
    bool changed = false;
    for (int q = 0; q < count; ++q) {
      if (plans[q].z == 0) continue;
      const bool aux = (q % (Kc + 1)) != 0;
      if (plans[q].z & LG_PLAN_UNCERTAIN) {
        LgPlannerCtx cx{lg_u_prime(), 0};
        LgPlan hp = lg_make_plan(cx, arg[q], (long)sp[q], p->tau, 60, 10000);
        plans[q] = make_int4(hp.order, hp.scaling, hp.status, 0);
        changed = true;
      }
      if (plans[q].z == LG_PLAN_BADARG) {
        char buf[128];
        std::snprintf(buf, sizeof buf, "norm1_a must be non-negative, got %g", arg[q]);
        return fail(LG_INVALID_ARG, buf);
      }
      if (plans[q].z == LG_PLAN_INFEASIBLE && (need_aux || !aux)) {
        char buf[256];
        std::snprintf(buf, sizeof buf,
                      "no feasible (order, scaling) pair for norm1=%g, sigma_prime=%lld, tau=%g within order<=60, "
                      "scaling<=10000",
                      arg[q], (long long)sp[q], p->tau);
        return fail(LG_PLANNING_INFEASIBLE, buf);
      }
    }
    if (changed) CK(cudaMemcpy(p->d_plan, plans.data(), sizeof(int4) * count, cudaMemcpyHostToDevice));
  }
  if (p->engine == 4 && !p->dense) {  // the ws chains read their per-step Taylor coefficients from this table
    void* rargs[] = {&p->d_plan, &Kc, &Ni, &p->d_rtab};
    rc = launch(lg_rtab_kernel(), dim3((unsigned)N), dim3(64), rargs, 0, p->stream);
    if (rc) return rc;
  }
  return LG_OK;
}

LgEngineArgs engine_args(lg_problem* p, long N) {
  LgEngineArgs E{};
  E.d = (int)p->d;
  E.N = (int)N;
  E.Kc = p->Kc;
  E.W = p->W;
  E.Wc = p->Wc;
  E.n_specs = (int)p->specs.size();
  for (int s = 0; s < E.n_specs; ++s) {
    const Spec& sp = p->specs[s];
    E.spec[s].kind = sp.kind;
    E.spec[s].weight = sp.weight;
    E.spec[s].set = sp.set;
    E.spec[s].pen_W = sp.pen_W;
    E.spec[s].pen_cols = sp.d_pen_cols;
    E.spec[s].pen_vals = sp.d_pen_vals;
    E.spec[s].tgt = sp.d_tgt;
    E.set_spec[sp.set][E.set_nspec[sp.set]++] = s;
  }
  for (int k = 0; k < 2; ++k) {
    E.set_t0[k] = p->set_t0[k];
    E.set_T[k] = p->set_T[k];
  }
  E.T_total = p->T_total;
  E.n_groups = p->n_groups;
  E.n_slabs = p->n_slabs;
  for (int g = 0; g < p->n_groups; ++g) {
    E.grp_set[g] = p->grp_set[g];
    E.grp_t0[g] = p->grp_t0[g];
    E.grp_nT[g] = p->grp_nT[g];
  }
  E.A_cols = p->d_cols;
  E.A = p->d_A;
  E.Ac_cols = p->d_ccols;
  E.Ac = p->d_Ac;
  E.plan = p->d_plan;
  E.rtab = p->d_rtab;
  E.psi0 = p->d_traj;
  E.scratch = p->d_scratch;
  E.scratch_per_group = p->scratch_per_group;
  E.bar = p->d_bar;
  E.red = p->d_red;
  E.red_cap = p->red_cap;
  E.smem_bytes = p->smem_bytes;
  E.smem_mode = p->smem_mode;
  E.row_lanes = p->row_lanes;
  E.cta_Imax = p->cta_Imax;
  E.grp_T = 1;
  for (int g = 0; g < p->n_groups; ++g) E.grp_T = std::max(E.grp_T, p->grp_nT[g]);
  E.ip = p->d_ip;
  E.fin = p->d_fin;
  E.run = p->d_run;
  E.trp = p->d_trp;
  E.psiN = p->d_psiN;
  E.trsum = p->d_trsum;
  E.trace = nullptr;
  E.cl_R = p->cl_R;
  E.cl_H = p->cl_H;
  E.cl_Q = p->cl_Q;
  E.cl_E = p->cl_E;
  E.diag = p->backend == 1 ? 1 : 0;
  E.diag_Ud = p->d_Ud;
  E.diag_D = p->d_D;
  E.cl_acs = 0;
  E.dbg = std::getenv("LG_DBG") ? std::atoi(std::getenv("LG_DBG")) : 0;
  E.ws_nw = p->ws_nw;
  E.dense_rows = (p->dense && p->W == p->d && p->Wc == p->d) ? 1 : 0;
  E.cl_perm = p->d_cl_perm;
  E.cl_inv = p->d_cl_inv;
  E.cl_cols = p->d_cl_cols;
  E.cl_slot = p->d_cl_slot;
  E.cl_accols = p->d_cl_accols;
  E.cl_cshare = p->cl_cshare;
  if (std::getenv("LG_TRACE") && p->engine == 4) {
    static long long* tbuf = nullptr;
    static size_t tcap = 0;
    const size_t need = (size_t)p->n_groups * 8 * N * 4;
    if (need > tcap) {
      if (tbuf) cudaFree(tbuf);
      cudaMalloc(&tbuf, need * sizeof(long long));
      tcap = need;
    }
    cudaMemset(tbuf, 0, need * sizeof(long long));
    E.trace = tbuf;
  }
  return E;
}

LgFinalArgs final_args(lg_problem* p, long N, const double2* ip, const double2* fin, const double* run,
                       const double2* trp, double* grad, double* cost) {
  LgFinalArgs F{};
  F.N = (int)N;
  F.Kc = p->Kc;
  F.n_specs = (int)p->specs.size();
  F.T_total = p->T_total;
  for (int s = 0; s < F.n_specs; ++s) {
    F.kind[s] = p->specs[s].kind;
    F.weight[s] = p->specs[s].weight;
    F.t0[s] = p->set_t0[p->specs[s].set];
    F.K[s] = p->set_T[p->specs[s].set];
  }
  F.ip = ip;
  F.fin = fin;
  F.run = run;
  F.trp = trp;
  F.grad = grad;
  F.cost = cost;
  return F;
}


// ============================================================================ dense GEMM engine
// Host-orchestrated: every Taylor term is one DMMA complex GEMM over all the
// chain's columns (lg_dense.cu); per-step scalars via deterministic dot kernels.

int build_problem(const lg_problem_desc* D, lg_problem* p) {
  if (!D) return fail(LG_INVALID_ARG, "null descriptor");
  const long d = D->h_static.n;
  if (d < 1) return fail(LG_INVALID_ARG, "empty Hamiltonian");
  if (D->n_channels < 1) return fail(LG_INVALID_ARG, "need at least one control channel");
  if (D->n_channels > LG_MAX_CHANNELS) return fail(LG_UNSUPPORTED, "more than 16 control channels");
  if (!(D->tau > 0.0)) return fail(LG_INVALID_ARG, "tau must be positive");
  p->d = d;
  p->Kc = D->n_channels;
  p->tau = D->tau;
  p->device = D->device;
  int rc = parse_mat(D->h_static, d, &p->hs, "static Hamiltonian");
  if (rc) return rc;
  p->hc.resize(p->Kc);
  for (int c = 0; c < p->Kc; ++c) {
    rc = parse_mat(D->h_controls[c], d, &p->hc[c], "control operator");
    if (rc) return rc;
  }
  p->dense = p->hs.dense;
  for (auto& m : p->hc) p->dense = p->dense || m.dense;
  p->materialise = 2 * d <= 256;  // src/derivatives.py:29,199-202
  // per-term DMMA GEMM engine (lg_dense.cu); LG_ENGINE=dense forces it for smaller dense problems
  // (tests exercise its kernels against the dense goldens below d = 512)
  const char* fe = std::getenv("LG_ENGINE");
  p->dense_large = p->dense && D->backend == 0 && (d > 512 || (fe && std::string(fe) == "dense"));
  // DIAGONALIZATION above the CTA engine's d <= 128 (or LG_ENGINE=dense): the propagators
  // U_n, U_n^dagger, dU_n/da_k are applied by the dense GEMM engine, one GEMM per application
  p->diag_dense = p->dense && D->backend == 1 && (d > 128 || (fe && std::string(fe) == "dense"));
  // ---- terms and trajectory sets
  if (D->n_terms > LG_MAX_SPECS) return fail(LG_UNSUPPORTED, "more than 8 cost terms");
  bool has_state = false, has_gate = false;
  for (int t = 0; t < D->n_terms; ++t) {
    const lg_cost_term& ct = D->terms[t];
    if (ct.kind < 0 || ct.kind > 4) return fail(LG_INVALID_ARG, "unknown cost kind");
    if (ct.weight < 0.0) return fail(LG_INVALID_ARG, "cost weights must be non-negative");
    (ct.kind <= LG_STATE_RUNNING_INFIDELITY ? has_state : has_gate) = true;
  }
  const long Ks = D->n_states, Kg = D->n_basis;
  if ((has_state || D->n_terms == 0) && (Ks < 1 || !D->initial_states))
    return fail(LG_INVALID_ARG, "state-transfer terms require problem.initial_state");
  std::vector<double2> basis_v;
  long Kgate = 0;
  if (has_gate) {
    if (Kg > 0 && D->basis) {
      Kgate = Kg;
      basis_v.resize((size_t)Kg * d);
      std::memcpy(basis_v.data(), D->basis, sizeof(double2) * Kg * d);
    } else {
      Kgate = d;  // computational basis (src/costs.py:393-397)
      basis_v.assign((size_t)d * d, make_double2(0.0, 0.0));
      for (long h = 0; h < d; ++h) basis_v[(size_t)h * d + h] = make_double2(1.0, 0.0);
    }
  }
  std::vector<double2> states_v;
  if (Ks > 0 && D->initial_states && (has_state || D->n_terms == 0)) {
    states_v.resize((size_t)Ks * d);
    std::memcpy(states_v.data(), D->initial_states, sizeof(double2) * Ks * d);
  }
  // merge identical sets (same trajectories drive both kinds of term)
  bool merged = has_gate && !states_v.empty() && states_v.size() == basis_v.size() &&
                std::memcmp(states_v.data(), basis_v.data(), sizeof(double2) * states_v.size()) == 0;
  p->traj.clear();
  if (!states_v.empty()) {
    p->set_t0[0] = 0;
    p->set_T[0] = (int)Ks;
    p->traj.insert(p->traj.end(), states_v.begin(), states_v.end());
  }
  if (has_gate) {
    if (merged) {
      p->set_t0[1] = 0;
      p->set_T[1] = 0;  // gate terms ride on set 0's trajectories
    } else {
      p->set_t0[1] = (int)(p->traj.size() / d);
      p->set_T[1] = (int)Kgate;
      p->traj.insert(p->traj.end(), basis_v.begin(), basis_v.end());
    }
  }
  p->T_total = (int)(p->traj.size() / d);
  // sharding (multi-GPU): each set propagates only trajectories [shard_begin, shard_end) of itself
  p->backend = D->backend;
  if (p->backend < 0 || p->backend > 1) return fail(LG_INVALID_ARG, "unknown backend");
  if (p->backend == 1 && !p->dense)
    return fail(LG_UNSUPPORTED, "the DIAGONALIZATION backend runs dense operators on the device");
  p->shard_b = D->shard_end > 0 ? D->shard_begin : 0;
  p->shard_e = D->shard_end > 0 ? D->shard_end : (1L << 40);
  for (int t = 0; t < D->n_terms; ++t) {
    const lg_cost_term& ct = D->terms[t];
    Spec sp;
    sp.kind = ct.kind;
    sp.weight = ct.weight;
    sp.set = (ct.kind <= LG_STATE_RUNNING_INFIDELITY || merged) ? 0 : 1;
    if (sp.kind == LG_GATE_RUNNING_INFIDELITY) p->has_gate_run = true;
    const int K = p->set_T[sp.set];
    if (ct.kind == LG_STATE_PENALTY) {
      rc = parse_mat(ct.penalty, d, &sp.pen, "penalty operator");
      if (rc) return rc;
    } else {
      if (!ct.targets) return fail(LG_INVALID_ARG, "cost term requires target states / images");
      sp.tgt.resize((size_t)K * d);
      std::memcpy(sp.tgt.data(), ct.targets, sizeof(double2) * K * d);
    }
    p->specs.push_back(std::move(sp));
  }
  // ---- union ELL pattern (sparse) or full pattern (dense)
  if (p->dense_large) {
    p->W = 1;
  } else if (p->dense) {
    p->W = (int)d;
    p->rowlen.assign(d, (int)d);
    p->cols.resize((size_t)d * d);
    for (long w = 0; w < d; ++w)
      for (long i = 0; i < d; ++i) p->cols[w * d + i] = (int)w;
  } else {
    std::vector<std::vector<int>> rows(d);
    for (long i = 0; i < d; ++i) {
      std::vector<int>& r = rows[i];
      for (long k = p->hs.indptr[i]; k < p->hs.indptr[i + 1]; ++k) r.push_back((int)p->hs.indices[k]);
      for (auto& m : p->hc)
        for (long k = m.indptr[i]; k < m.indptr[i + 1]; ++k) r.push_back((int)m.indices[k]);
      std::sort(r.begin(), r.end());
      r.erase(std::unique(r.begin(), r.end()), r.end());
      p->W = std::max<int>(p->W, (int)r.size());
    }
    p->W = std::max(p->W, 1);
    if (p->W > LG_MAXW) return fail(LG_UNSUPPORTED, "more than 64 stored elements per row");
    const int W = p->W;
    p->rowlen.assign(d, 0);
    p->cols.assign((size_t)W * d, 0);
    p->src_s.assign((size_t)W * d, -1);
    p->src_c.assign((size_t)p->Kc * W * d, -1);
    for (long i = 0; i < d; ++i) {
      const auto& r = rows[i];
      p->rowlen[i] = (int)r.size();
      for (int w = 0; w < W; ++w) p->cols[(size_t)w * d + i] = w < (int)r.size() ? r[w] : (int)i;
      auto fill = [&](const Mat& m, int* dst) {
        size_t w = 0;
        for (long k = m.indptr[i]; k < m.indptr[i + 1]; ++k) {
          while (r[w] != m.indices[k]) ++w;
          dst[w * d + i] = (int)k;
        }
      };
      fill(p->hs, p->src_s.data());
      for (int c = 0; c < p->Kc; ++c) fill(p->hc[c], p->src_c.data() + (size_t)c * W * d);
    }
    // transposed slot lists: for each column, slots in ascending row order
    p->colptr.assign(d + 1, 0);
    for (long i = 0; i < d; ++i)
      for (int w = 0; w < p->rowlen[i]; ++w) p->colptr[p->cols[(size_t)w * d + i] + 1]++;
    for (long j = 0; j < d; ++j) p->colptr[j + 1] += p->colptr[j];
    p->colent.assign(p->colptr[d], 0);
    std::vector<int> fillp(p->colptr.begin(), p->colptr.end() - 1);
    for (long i = 0; i < d; ++i)
      for (int w = 0; w < p->rowlen[i]; ++w) p->colent[fillp[p->cols[(size_t)w * d + i]]++] = (int)(w * d + i);
  }
  // ---- control ELL (engine) — raw h_c values; A_c is formed per dt
  if (p->dense_large) {
    p->Wc = 1;
  } else {
    int Wc = 1;
    for (auto& m : p->hc) {
      if (m.dense) Wc = std::max<int>(Wc, (int)d);
      else
        for (long i = 0; i < d; ++i) Wc = std::max<int>(Wc, (int)(m.indptr[i + 1] - m.indptr[i]));
    }
    if (!p->dense && Wc > LG_MAXW) return fail(LG_UNSUPPORTED, "more than 64 stored elements per control row");
    p->Wc = Wc;
    p->ccols.assign((size_t)p->Kc * Wc * d, 0);
    p->cvals.assign((size_t)p->Kc * Wc * d, make_double2(0.0, 0.0));
    for (int c = 0; c < p->Kc; ++c) {
      const Mat& m = p->hc[c];
      for (long i = 0; i < d; ++i) {
        for (int w = 0; w < Wc; ++w) {
          size_t q = ((size_t)c * Wc + w) * d + i;
          if (m.dense) {
            p->ccols[q] = w;
            p->cvals[q] = m.vals[(size_t)w * d + i];
          } else {
            long L = m.indptr[i + 1] - m.indptr[i];
            if (w < L) {
              p->ccols[q] = (int)m.indices[m.indptr[i] + w];
              p->cvals[q] = m.vals[m.indptr[i] + w];
            } else {
              p->ccols[q] = (int)i;
            }
          }
        }
      }
    }
  }
  // ---- device upload
  CK(cudaSetDevice(p->device));
  CK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
  DevMem& M = p->mem;
  p->d_rowlen = M.upload(p->rowlen);
  p->d_cols = M.upload(p->cols);
  p->d_ccols = M.upload(p->ccols);
  p->d_traj = M.upload(p->traj);
  if (p->dense) {
    std::vector<double2> hsd = p->hs.dense ? p->hs.vals : std::vector<double2>((size_t)d * d, make_double2(0, 0));
    if (!p->hs.dense)
      for (long i = 0; i < d; ++i)
        for (long k = p->hs.indptr[i]; k < p->hs.indptr[i + 1]; ++k) hsd[(size_t)p->hs.indices[k] * d + i] = p->hs.vals[k];
    p->d_hs_dense = M.upload(hsd);
    std::vector<double2*> ptrs(p->Kc);
    for (int c = 0; c < p->Kc; ++c) {
      const Mat& m = p->hc[c];
      std::vector<double2> v = m.dense ? m.vals : std::vector<double2>((size_t)d * d, make_double2(0, 0));
      (void)0;
      if (!m.dense)
        for (long i = 0; i < d; ++i)
          for (long k = m.indptr[i]; k < m.indptr[i + 1]; ++k) v[(size_t)m.indices[k] * d + i] = m.vals[k];
      ptrs[c] = M.upload(v);
    }
    p->d_hc_dense_ptrs = M.upload(ptrs);
    p->d_hc_dense_host = ptrs;
  } else {
    p->d_src_s = M.upload(p->src_s);
    p->d_src_c = M.upload(p->src_c);
    p->d_colptr = M.upload(p->colptr);
    p->d_colent = M.upload(p->colent);
    p->d_hs = M.upload(p->hs.vals);
    std::vector<double2*> ptrs(p->Kc);
    for (int c = 0; c < p->Kc; ++c) ptrs[c] = M.upload(p->hc[c].vals);
    p->d_hc_ptrs = M.upload(ptrs);
  }
  for (auto& sp : p->specs) {
    if (sp.kind == LG_STATE_PENALTY) {
      std::vector<int> pc;
      std::vector<double2> pv;
      to_ell(sp.pen, &sp.pen_W, pc, pv, nullptr);
      sp.d_pen_cols = M.upload(pc);
      sp.d_pen_vals = M.upload(pv);
    } else {
      sp.d_tgt = M.upload(sp.tgt);
    }
  }
  if (M.failed) return fail(LG_CUDA_ERROR, "device allocation failed (problem data)");
  const int rc_cfg = configure(p);
  if (rc_cfg == LG_OK && p->mem.failed) return fail(LG_CUDA_ERROR, "device allocation failed (engine buffers)");
  return rc_cfg;
}

}  // namespace lgi
