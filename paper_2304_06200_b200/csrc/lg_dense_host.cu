// Host units, part 3: the dense (DMMA) engine driver -- per-step host loop over the dense Taylor
// GEMMs (lg_dense.cu), derivative chains, costate sources and per-step scalars.
#include "lg_host.h"

namespace lgi {

int dense_gemm(lg_problem* p, const double2* A, const double2* X, const double2* B, const double2* Xb, int C,
               double r, bool first, bool last, const double2* xin, double2* cur, double2* tout) {
  LgGemmArgs G{};
  const int d = (int)p->d;
  G.M = d;
  G.C = C;
  G.seg[0] = LgGemmSeg{A, d, X, d, d};
  G.nseg = 1;
  if (B) {
    G.seg[1] = LgGemmSeg{B, d, Xb, d, d};
    G.nseg = 2;
  }
  G.xin = xin;
  G.ldxin = d;
  G.cur = cur;
  G.ldc = d;
  G.tout = tout;
  G.ldt = d;
  G.r = r;
  G.first = first;
  G.last = last;
  // split-k when the output tiles alone cannot fill the GPU (tall-skinny Taylor terms, 4 warps per
  // 64 x 16 tile): deterministic, slices summed in order by lg_k_taylor_epi.  Measured at d = 4096:
  // C = 64: 22.6 (1 slice) -> 29.7 TF/s (4); C = 128: 25.8 -> 31.2 TF/s (4) (tools/bench_zgemm.py).
  // wide tile (4 warps of 16 x 32) from 64 columns: half the A-fragment loads per DMMA
  // (tools/bench_zgemm.py, d = 4096: C = 64 33.0 -> 34.3, C = 128 35.0 -> 35.9 TF/s, split-k 8)
  // ... and from 32 columns since the bulk-copy kernel: d = 4096, C = 32: 0.155 ms with the 16 x 16 warp
  // tiles, 0.120 ms with the bulk kernel's 16 x 32 (36.0 TF/s; a shard of 32 trajectories)
  const char* ev = std::getenv("LG_ZGEMM_N32");
  const int n32_from = ev ? std::atoi(ev) : 32;
  const int ntt = n32_from > 0 && C >= n32_from ? 4 : 2;
  const int bn = 8 * ntt;
  int smem = lg_zgemm_smem_bytes(ntt);
  void* kern = ntt == 4 ? lg_zgemm_n32_kernel() : lg_zgemm_kernel();
  // aligned shapes (c5): the warp-specialised kernel whose tiles move by TMA bulk copies through a
  // 4-stage mbarrier ring (producer warp + 4 MMA warps); LG_ZGEMM_BULK=0 keeps the cp.async kernel
  const char* eb = std::getenv("LG_ZGEMM_BULK");
  const bool bulk_on = !(eb && std::atoi(eb) == 0);
  const bool bulk = bulk_on && ntt == 4 && d % 64 == 0 && C % 32 == 0;  // every segment has K = lda = d
  int threads = 128;
  if (bulk) {
    kern = lg_zgemm_bulk_kernel();
    smem = lg_zgemm_bulk_smem_bytes();
    threads = 160;
  }
  // (launch() raises the kernel's dynamic shared-memory limit to `smem` when it exceeds 48 KB)
  const long nct = (long)((C + bn - 1) / bn) * ((d + 63) / 64);
  // narrow chains (8 - 16 columns: small shards) stream the operator from HBM for little arithmetic: more
  // k-slices keep more copies in flight (d = 4096, C = 8 / 16: 0.082 / 0.085 ms with 4 slices, 0.073 /
  // 0.076 ms with 16, 0.079 / 0.084 ms with 32; tools/bench_zgemm.py)
  const long ktiles = (long)((d + 15) / 16) * (B ? 2 : 1);
  int ks = (int)std::max<long>(1, std::min<long>({ntt == 4 ? 8L : 16L, 2048L / std::max<long>(nct, 1), ktiles}));
  if (bulk) {
    // the k-slices that fill whole waves of co-resident CTAs: minimise waves x (k-tiles per slice + ~2
    // tiles of pipeline fill and epilogue); d = 4096: C = 64 -> 9 slices (37.1 vs 35.1 TF/s with 8),
    // C = 128 -> 8 (LG_SPLITK sweep, tools/bench_zgemm.py)
    static int slots = 0;
    if (!slots) {
      int dev = 0, sms = 148, occ = 2;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      ensure_smem(kern, smem);
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess || occ < 1) occ = 2;
      slots = sms * occ;
    }
    const long tiles = (long)(d / 16) * (B ? 2 : 1);
    long best = -1;
    for (int k = 1; k <= 16; ++k) {
      const long cost = ((nct * k + slots - 1) / slots) * ((tiles + k - 1) / k + 2);
      if (best < 0 || cost < best) best = cost, ks = k;
    }
  }
  if (const char* e = std::getenv("LG_SPLITK")) ks = std::max(1, std::atoi(e));
  G.ksplit = ks;
  if (ks > 1) {
    const size_t need = (size_t)ks * d * C;
    if (need > p->splitws_cap) {
      if (p->d_splitws) cudaFree(p->d_splitws);
      p->d_splitws = nullptr;
      p->splitws_cap = 0;
      if (cudaMalloc(&p->d_splitws, need * sizeof(double2)) != cudaSuccess) return fail(LG_CUDA_ERROR, "split-k workspace");
      p->splitws_cap = need;
    }
    G.partial = p->d_splitws;
  }
  // LG_ZGEMM_FUSEDK=1 (A/B knob, off by default): fused split-k finish -- every slice counts itself on
  // its tile's counter and the last one to arrive reduces the tile and applies the Taylor update, so
  // lg_k_taylor_epi's launch disappears; LG_ZGEMM_ZFAST=0 keeps the slice index on blockIdx.z instead
  // of co-scheduling a tile's slices.  Measured at d = 4096 (tools/bench_zgemm.py, same box): 0.267 /
  // 0.482 ms (slices co-scheduled) and 0.252 / 0.455 ms (slice index slowest) against 0.2275 / 0.4375 ms
  // for the two-kernel path at 64 / 128 columns: the per-slice fence + counter round trip and the
  // reduction on the tail of the last CTAs cost more than the 16 us epilogue kernel they replace.
  constexpr int kCtrCap = 4096;
  const char* ef = std::getenv("LG_ZGEMM_FUSEDK");
  const bool fused = ks > 1 && nct <= kCtrCap && ef && std::atoi(ef) == 1;
  if (fused && !p->d_tilectr) {
    if (cudaMalloc(&p->d_tilectr, kCtrCap * sizeof(int)) != cudaSuccess) return fail(LG_CUDA_ERROR, "split-k tile counters");
    if (cudaMemsetAsync(p->d_tilectr, 0, kCtrCap * sizeof(int), p->stream) != cudaSuccess)
      return fail(LG_CUDA_ERROR, "split-k tile counters");
  }
  G.tile_ctr = fused ? p->d_tilectr : nullptr;
  const char* ez = std::getenv("LG_ZGEMM_ZFAST");
  G.zfast = fused && !(ez && std::atoi(ez) == 0) ? 1 : 0;
  void* args[] = {&G};
  const dim3 grid = G.zfast ? dim3(ks, (C + bn - 1) / bn, (d + 63) / 64) : dim3((C + bn - 1) / bn, (d + 63) / 64, ks);
  int rc = launch(kern, grid, dim3(threads), args, smem, p->stream);
  if (rc || ks == 1 || fused) return rc;
  const long mc = (long)d * C;
  return launch(lg_taylor_epi_kernel(), dim3((unsigned)std::min<long>((mc + 255) / 256, 148 * 8)), dim3(256), args, 0,
                p->stream);
}

// Y <- Op X over C columns: one GEMM, no Taylor recursion (DIAGONALIZATION backend: Op = U_n,
// U_n^dagger or dU_n/da_k as formed by prepare_diag, column-major d x d)
int dense_apply(lg_problem* p, const double2* op, int C, const double2* X, double2* Y) {
  return dense_gemm(p, op, X, nullptr, nullptr, C, 1.0, true, true, nullptr, Y, p->dd_tb0);
}

// cur <- (T_m(sgn A / s))^s x over C columns (columns contiguous, stride d)
int dense_chain(lg_problem* p, int C, double sgn, int m, int s, const double2* x, double2* cur) {
  const double2* prev = x;
  double2* bufs[2] = {p->dd_tb0, p->dd_tb1};
  int b = 0;
  for (int si = 0; si < s; ++si)
    for (int j = 1; j <= m; ++j) {
      const bool first = si == 0 && j == 1;
      int rc = dense_gemm(p, p->d_Ad, prev, nullptr, nullptr, C, sgn * (1.0 / (double)(s * j)), first, j == m,
                          first ? x : nullptr, cur, bufs[b]);
      if (rc) return rc;
      prev = bufs[b];
      b ^= 1;
    }
  return LG_OK;
}

// aux embedding chain for channels gch[0..G): tops (G*T columns) then bottoms (T columns)
int dense_aux_chain(lg_problem* p, int T, const int* gch, int G, int m, int s, const double2* psi) {
  const long d = p->d;
  double2* bufs[2] = {p->dd_xtb0, p->dd_xtb1};
  const double2* prev = nullptr;
  int b = 0;
  // Narrow chains (a small shard of the K-state block: T <= LG_AUX_MERGE columns, default 8) are bound by
  // streaming the d x d operators from HBM, not by the MMAs: a single-channel chain then runs tops and
  // bottoms as ONE two-segment GEMM per term (2 operator reads instead of 3, full 16-column tiles).
  // The T columns behind the bottoms of both term buffers are zeroed per chain (another trajectory set
  // or channel group may have used them).
  static const int merge_T = [] {
    const char* e = std::getenv("LG_AUX_MERGE");
    return e ? std::atoi(e) : 8;
  }();
  const bool merged = G == 1 && T <= merge_T && m * s > 1;
  if (merged)
    for (double2* tb : bufs)
      CK(cudaMemsetAsync(tb + 2L * T * d, 0, sizeof(double2) * (size_t)T * d, p->stream));
  for (int si = 0; si < s; ++si)
    for (int j = 1; j <= m; ++j) {
      const bool first = si == 0 && j == 1, last = j == m;
      const double r = 1.0 / (double)(s * j);
      double2* out = bufs[b];
      if (merged && !first) {
        // one pass [A | A_c] [[X_top, X_bot], [X_bot, 0]] over the 2 T columns [top | bottom]: A and A_c are
        // each read once per term instead of A twice and A_c once (the zero columns behind the bottoms
        // add exact zeros)
        int rc = dense_gemm(p, p->d_Ad, prev, p->d_Acd[gch[0]], prev + (long)T * d, 2 * T, r, false, last, nullptr,
                            p->dd_xcur, out);
        if (rc) return rc;
        prev = out;
        b ^= 1;
        continue;
      }
      for (int gi = 0; gi < G; ++gi) {
        const int k = gch[gi];
        int rc;
        if (first)
          rc = dense_gemm(p, p->d_Acd[k], psi, nullptr, nullptr, T, r, true, last, nullptr, p->dd_xcur + gi * T * d,
                          out + gi * T * d);
        else
          rc = dense_gemm(p, p->d_Ad, prev + gi * T * d, p->d_Acd[k], prev + (long)G * T * d, T, r, false, last,
                          nullptr, p->dd_xcur + gi * T * d, out + gi * T * d);
        if (rc) return rc;
      }
      int rc = dense_gemm(p, p->d_Ad, first ? psi : prev + (long)G * T * d, nullptr, nullptr, T, r, first, last,
                          first ? psi : nullptr, p->dd_xcur + (long)G * T * d, out + (long)G * T * d);
      if (rc) return rc;
      prev = out;
      b ^= 1;
    }
  return LG_OK;
}

int dense_form(lg_problem* p, const double2* hs, double2** hc_dev, const double* amps, int kc, double dt, double2* A) {
  long count = p->d * p->d;
  void* args[] = {&hs, &hc_dev, &amps, &kc, &dt, &count, &A};
  return launch(lg_dense_form_kernel(), dim3(148 * 8), dim3(256), args, 0, p->stream);
}

// deterministic dots over pairs, written (mode 0) or accumulated (modes 1, 2: running costs, in step
// order) straight into the device-side raw scalars: no host round trip inside the sweeps
struct DotOut {
  double2* out;
  int mode;
};
int dense_dots(lg_problem* p, const std::vector<std::pair<const double2*, const double2*>>& pr,
               const std::vector<DotOut>& to) {
  for (size_t b0 = 0; b0 < pr.size(); b0 += 64) {
    LgDotArgs D{};
    D.d = (int)p->d;
    D.n = (int)std::min<size_t>(64, pr.size() - b0);
    for (int q = 0; q < D.n; ++q) {
      D.u[q] = pr[b0 + q].first;
      D.v[q] = pr[b0 + q].second;
      D.out[q] = to[b0 + q].out;
      D.mode[q] = to[b0 + q].mode;
    }
    void* args[] = {&D};
    int rc = launch(lg_dots_kernel(), dim3(D.n), dim3(256), args, 0, p->stream);
    if (rc) return rc;
  }
  return LG_OK;
}

int dense_ell(lg_problem* p, const Spec& sp, const std::vector<const double2*>& x, const std::vector<double2*>& y,
              bool acc) {
  for (size_t b0 = 0; b0 < x.size(); b0 += 64) {
    LgEllArgs A{};
    A.d = (int)p->d;
    A.W = sp.pen_W;
    A.ncol = (int)std::min<size_t>(64, x.size() - b0);
    A.accumulate = acc;
    A.cols = sp.d_pen_cols;
    A.vals = sp.d_pen_vals;
    for (int q = 0; q < A.ncol; ++q) {
      A.x[q] = x[b0 + q];
      A.y[q] = y[b0 + q];
    }
    void* args[] = {&A};
    int rc = launch(lg_ell_kernel(), dim3((unsigned)((p->d + 255) / 256), A.ncol), dim3(256), args, 0, p->stream);
    if (rc) return rc;
  }
  return LG_OK;
}

// y_q (+)= alpha_q u_q; alpha_q from the device (alpha_ptr[q]) when given, else the host value
int dense_axpy(lg_problem* p, const std::vector<const double2*>& u, const std::vector<double2*>& y,
               const std::vector<double2>& alpha, const std::vector<const double2*>& alpha_ptr, bool acc) {
  for (size_t b0 = 0; b0 < u.size(); b0 += 64) {
    LgAxpyArgs A{};
    A.d = (int)p->d;
    A.ncol = (int)std::min<size_t>(64, u.size() - b0);
    for (int q = 0; q < A.ncol; ++q) {
      A.u[q] = u[b0 + q];
      A.y[q] = y[b0 + q];
      A.alpha[q] = alpha[b0 + q];
      A.alpha_ptr[q] = alpha_ptr[b0 + q];
      A.accumulate[q] = acc;
    }
    void* args[] = {&A};
    int rc = launch(lg_axpy_kernel(), dim3((unsigned)((p->d + 255) / 256), A.ncol), dim3(256), args, 0, p->stream);
    if (rc) return rc;
  }
  return LG_OK;
}

int configure_dense(lg_problem* p) {
  const long d = p->d;
  int nspec[2] = {0, 0};
  for (auto& s : p->specs) nspec[s.set]++;
  const int Imax = std::max({1, nspec[0], nspec[1]});
  int Tmax = 1;
  for (int s = 0; s < 2; ++s) {
    const int lo = (int)std::min<long>(p->shard_b, p->set_T[s]), hi = (int)std::min<long>(p->shard_e, p->set_T[s]);
    Tmax = std::max(Tmax, hi - lo);
  }
  // aux term buffers: K_c T tops + T bottoms + T columns that stay zero (merged aux pass, dense_aux_chain)
  const long cst = (long)Tmax * (1 + Imax), cx = (long)(p->Kc + 2) * Tmax;
  DevMem& M = p->mem;
  p->d_Ad = M.alloc<double2>((size_t)d * d);
  p->d_Acd.assign(p->Kc, nullptr);
  for (int c = 0; c < p->Kc; ++c) p->d_Acd[c] = M.alloc<double2>((size_t)d * d);
  p->dd_st = M.alloc<double2>((size_t)cst * d);
  p->dd_nx = M.alloc<double2>((size_t)cst * d);
  p->dd_cur = M.alloc<double2>((size_t)cst * d);
  p->dd_tb0 = M.alloc<double2>((size_t)cst * d);
  p->dd_tb1 = M.alloc<double2>((size_t)cst * d);
  p->dd_xcur = M.alloc<double2>((size_t)cx * d);
  p->dd_xtb0 = M.alloc<double2>((size_t)cx * d);
  p->dd_xtb1 = M.alloc<double2>((size_t)cx * d);
  p->dd_tmp = M.alloc<double2>((size_t)Tmax * d);
  p->dd_dots = M.alloc<double2>((size_t)std::max<long>(64, (long)Imax * p->Kc * Tmax + 2 * cst));
  p->engine = 3;
  p->n_groups = 0;
  p->live_peak = (int)((3 * cst + 3 * cx + Tmax - 1) / Tmax);
  p->d_bar = M.alloc<unsigned>(4);
  p->d_scratch = M.alloc<double2>(1);
  p->d_red = M.alloc<double2>(1);
  if (M.failed) return fail(LG_CUDA_ERROR, "device allocation failed (dense engine)");
  return LG_OK;
}

// One evaluation on the dense engine.  The host drives the per-step GEMM chains (the Taylor
// plans are read back once, before the sweeps); every per-step scalar -- overlaps, running
// costs, traces, <lambda|dU/da psi> -- is produced and accumulated on the device, in the raw
// layout the finalize kernel and the sharded all-reduce hook read (lg_raw_get).
int run_dense(lg_problem* p, long N, double dt, bool grad) {
  const long d = p->d;
  const int Kc = p->Kc, S = (int)p->specs.size(), Tt = p->T_total;
  int rc;
  std::vector<int4> pl((size_t)N * (Kc + 1));
  CK(cudaMemcpyAsync(pl.data(), p->d_plan, sizeof(int4) * pl.size(), cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  const bool diag = p->backend == 1;  // propagators formed by prepare_diag (lg_diag.cu)
  const long dd = d * d;
  if (!diag && !(p->dense_dt == dt)) {
    for (int c = 0; c < Kc; ++c) {
      double2** none = nullptr;
      rc = dense_form(p, p->d_hc_dense_host[c], none, nullptr, 0, dt, p->d_Acd[c]);
      if (rc) return rc;
    }
    p->dense_dt = dt;
  }
  const size_t Sx = std::max(S, 1), Tx = std::max(Tt, 1);
  CK(cudaMemsetAsync(p->d_run, 0, sizeof(double) * Sx * Tx, p->stream));
  CK(cudaMemsetAsync(p->d_fin, 0, sizeof(double2) * Sx * Tx, p->stream));
  if (grad) CK(cudaMemsetAsync(p->d_ip, 0, sizeof(double2) * N * Sx * Kc * Tx, p->stream));
  CK(cudaMemsetAsync(p->d_trp, 0, sizeof(double2) * Sx * N * Tx, p->stream));
  auto runp = [&](long o) { return reinterpret_cast<double2*>(p->d_run + o); };
  // sharded running gate costs: every rank all-reduces the traces between its sweeps
  auto trace_hook = [&](int set) -> int {
    if (!grad || !p->hook) return LG_OK;
    bool any = false;
    for (int s = 0; s < S; ++s) any |= p->specs[s].set == set && p->specs[s].kind == LGK_GATE_RUN;
    if (!any) return LG_OK;
    if (p->hook(reinterpret_cast<double*>(p->d_trp), 2 * (long)Sx * N * Tx, p->stream, p->hook_user) != 0)
      return fail(LG_CUDA_ERROR, "all-reduce hook failed (traces)");
    p->trp_reduced = true;
    return LG_OK;
  };
  for (int set = 0; set < 2; ++set) {
    const int lo = (int)std::min<long>(p->shard_b, p->set_T[set]), hi = (int)std::min<long>(p->shard_e, p->set_T[set]);
    const int T = hi - lo;
    if (T <= 0) {
      if (int rh = trace_hook(set)) return rh;
      continue;
    }
    const int t0 = p->set_t0[set] + lo;  // global trajectory index of column 0
    std::vector<int> sp_idx;
    for (int s = 0; s < S; ++s)
      if (p->specs[s].set == set) sp_idx.push_back(s);
    const int I = (int)sp_idx.size();
    auto col = [&](double2* base, int c) { return base + (long)c * d; };
    auto tgt = [&](int s, int t) { return p->specs[s].d_tgt + (long)(lo + t) * d; };
    CK(cudaMemcpyAsync(p->dd_st, p->d_traj + (long)t0 * d, sizeof(double2) * T * d, cudaMemcpyDeviceToDevice, p->stream));
    // ---- forward sweep
    for (long n = 0; n < N; ++n) {
      const int4 q = pl[(size_t)n * (Kc + 1)];
      if (diag) {
        rc = dense_apply(p, p->d_A + n * dd, T, p->dd_st, p->dd_cur);
      } else {
        rc = dense_form(p, p->d_hs_dense, p->d_hc_dense_ptrs, p->d_amps + n * Kc, Kc, dt, p->d_Ad);
        if (rc) return rc;
        rc = dense_chain(p, T, 1.0, q.x, q.y, p->dd_st, p->dd_cur);
      }
      if (rc) return rc;
      CK(cudaMemcpyAsync(p->dd_st, p->dd_cur, sizeof(double2) * T * d, cudaMemcpyDeviceToDevice, p->stream));
      const bool fin_step = n == N - 1;
      std::vector<std::pair<const double2*, const double2*>> pr;
      std::vector<DotOut> to;
      for (int s : sp_idx) {
        const int kind = p->specs[s].kind;
        for (int t = 0; t < T; ++t) {
          const long o = (long)s * Tt + t0 + t;
          if (kind == LGK_STATE_PEN) {
            pr.push_back({col(p->dd_st, t), col(p->dd_tmp, t)});
            to.push_back({runp(o), 1});
          } else if (kind == LGK_STATE_RUN) {
            pr.push_back({tgt(s, t), col(p->dd_st, t)});
            to.push_back({runp(o), 2});
          } else if (kind == LGK_GATE_RUN) {
            pr.push_back({tgt(s, t), col(p->dd_st, t)});
            to.push_back({p->d_trp + ((long)s * N + n) * Tt + t0 + t, 0});
          } else if (fin_step && kind == LGK_GATE) {
            pr.push_back({tgt(s, t), col(p->dd_st, t)});
            to.push_back({p->d_fin + o, 0});
          } else if (fin_step && kind == LGK_STATE_INF) {
            pr.push_back({col(p->dd_st, t), tgt(s, t)});
            to.push_back({p->d_fin + o, 0});
          }
        }
        if (kind == LGK_STATE_PEN) {
          // Omega psi_n into tmp, and the penalty dots taken before tmp is reused by another penalty term
          std::vector<const double2*> x;
          std::vector<double2*> y;
          for (int t = 0; t < T; ++t) x.push_back(col(p->dd_st, t)), y.push_back(col(p->dd_tmp, t));
          rc = dense_ell(p, p->specs[s], x, y, false);
          if (rc) return rc;
          rc = dense_dots(p, pr, to);
          if (rc) return rc;
          pr.clear();
          to.clear();
        }
      }
      rc = dense_dots(p, pr, to);
      if (rc) return rc;
    }
    CK(cudaMemcpyAsync(p->d_psiN + (long)t0 * d, p->dd_st, sizeof(double2) * T * d, cudaMemcpyDeviceToDevice, p->stream));
    if (int rh = trace_hook(set)) return rh;
    if (!grad || I == 0) continue;
    bool gate_run = false;
    for (int s : sp_idx) gate_run |= p->specs[s].kind == LGK_GATE_RUN;
    if (gate_run) {  // running gate traces summed over the set (trajectory order), on the device
      int Ni = (int)N, Sv = S, Tv = Tt;
      long cnt = (long)S * N;
      void* targs[] = {&p->d_trp, &Sv, &Ni, &Tv, &p->d_spec_t0, &p->d_spec_K, &p->d_trsum};
      rc = launch(lg_trsum_kernel(), dim3((unsigned)((cnt + 255) / 256)), dim3(256), targs, 0, p->stream);
      if (rc) return rc;
    }
    auto lam = [&](double2* base, int si, int t) { return col(base, T + si * T + t); };
    // overlaps <phi|psi> of the running state costs: device scratch read by the axpy kernel
    auto run_overlaps = [&](double2* psi_base) -> int {
      std::vector<std::pair<const double2*, const double2*>> pr;
      std::vector<DotOut> to;
      for (int si = 0; si < I; ++si)
        if (p->specs[sp_idx[si]].kind == LGK_STATE_RUN)
          for (int t = 0; t < T; ++t) {
            pr.push_back({tgt(sp_idx[si], t), col(psi_base, t)});
            to.push_back({p->dd_dots + si * T + t, 0});
          }
      return dense_dots(p, pr, to);
    };
    // ---- costate initialisation (src/costs.py:312-321, :457-460)
    rc = run_overlaps(p->dd_st);
    if (rc) return rc;
    for (int si = 0; si < I; ++si) {
      const int s = sp_idx[si];
      const Spec& sp = p->specs[s];
      if (sp.kind == LGK_STATE_PEN) {
        std::vector<const double2*> x;
        std::vector<double2*> yy;
        for (int t = 0; t < T; ++t) x.push_back(col(p->dd_st, t)), yy.push_back(lam(p->dd_st, si, t));
        rc = dense_ell(p, sp, x, yy, false);
      } else {
        std::vector<const double2*> u, ap;
        std::vector<double2*> y;
        std::vector<double2> al;
        for (int t = 0; t < T; ++t) {
          u.push_back(tgt(s, t));
          y.push_back(lam(p->dd_st, si, t));
          al.push_back(make_double2(1.0, 0.0));
          ap.push_back(sp.kind == LGK_STATE_RUN   ? p->dd_dots + si * T + t
                       : sp.kind == LGK_GATE_RUN ? p->d_trsum + (long)s * N + N - 1
                                                 : nullptr);
        }
        rc = dense_axpy(p, u, y, al, ap, false);
      }
      if (rc) return rc;
    }
    // ---- backward sweep (phase event: with several trajectory sets the last set's boundary is kept)
    p->mark(2);
    p->dense_bwd_marked = true;
    int gch[LG_MAX_CHANNELS];
    for (long n = N - 1; n >= 0; --n) {
      const int4* pn = &pl[(size_t)n * (Kc + 1)];
      const int cadj = n > 0 ? T * (1 + I) : T;
      if (diag) {
        rc = dense_apply(p, p->d_Ud + n * dd, cadj, p->dd_st, p->dd_nx);
      } else {
        rc = dense_form(p, p->d_hs_dense, p->d_hc_dense_ptrs, p->d_amps + n * Kc, Kc, dt, p->d_Ad);
        if (rc) return rc;
        rc = dense_chain(p, cadj, -1.0, pn[0].x, pn[0].y, p->dd_st, p->dd_nx);
      }
      if (rc) return rc;
      unsigned done = 0;
      for (int kc = 0; kc < Kc && diag; ++kc) {  // <lambda_s(n)| dU_n/da_k psi_{n-1}>, one GEMM per channel
        rc = dense_apply(p, p->d_D + (n * Kc + kc) * dd, T, p->dd_nx, p->dd_xcur);
        if (rc) return rc;
        std::vector<std::pair<const double2*, const double2*>> pr;
        std::vector<DotOut> to;
        for (int si = 0; si < I; ++si)
          for (int t = 0; t < T; ++t) {
            pr.push_back({lam(p->dd_st, si, t), p->dd_xcur + (long)t * d});
            to.push_back({p->d_ip + (((long)n * S + sp_idx[si]) * Kc + kc) * Tt + t0 + t, 0});
          }
        rc = dense_dots(p, pr, to);
        if (rc) return rc;
      }
      for (int kc = 0; kc < Kc && !diag; ++kc) {
        if (done & (1u << kc)) continue;
        int G = 0;
        for (int k2 = kc; k2 < Kc; ++k2)
          if (!(done & (1u << k2)) && pn[1 + k2].x == pn[1 + kc].x && pn[1 + k2].y == pn[1 + kc].y) {
            gch[G++] = k2;
            done |= 1u << k2;
          }
        rc = dense_aux_chain(p, T, gch, G, pn[1 + kc].x, pn[1 + kc].y, p->dd_nx);
        if (rc) return rc;
        // <lambda_s(n)| dU_n/da_k psi_{n-1}> straight into ip (src/costs.py:328-339)
        std::vector<std::pair<const double2*, const double2*>> pr;
        std::vector<DotOut> to;
        for (int gi = 0; gi < G; ++gi)
          for (int si = 0; si < I; ++si)
            for (int t = 0; t < T; ++t) {
              pr.push_back({lam(p->dd_st, si, t), p->dd_xcur + ((long)gi * T + t) * d});
              to.push_back({p->d_ip + (((long)n * S + sp_idx[si]) * Kc + gch[gi]) * Tt + t0 + t, 0});
            }
        rc = dense_dots(p, pr, to);
        if (rc) return rc;
      }
      if (n == 0) break;
      // costate sources at psi_{n-1} (src/costs.py:341-353, :474-479)
      rc = run_overlaps(p->dd_nx);
      if (rc) return rc;
      for (int si = 0; si < I; ++si) {
        const int s = sp_idx[si];
        const Spec& sp = p->specs[s];
        if (sp.kind == LGK_STATE_PEN) {
          std::vector<const double2*> x;
          std::vector<double2*> yy;
          for (int t = 0; t < T; ++t) x.push_back(col(p->dd_nx, t)), yy.push_back(lam(p->dd_nx, si, t));
          rc = dense_ell(p, sp, x, yy, true);
        } else if (sp.kind == LGK_STATE_RUN || sp.kind == LGK_GATE_RUN) {
          std::vector<const double2*> u, ap;
          std::vector<double2*> y;
          std::vector<double2> al;
          for (int t = 0; t < T; ++t) {
            u.push_back(tgt(s, t));
            y.push_back(lam(p->dd_nx, si, t));
            al.push_back(make_double2(0.0, 0.0));
            ap.push_back(sp.kind == LGK_STATE_RUN ? p->dd_dots + si * T + t : p->d_trsum + (long)s * N + n - 1);
          }
          rc = dense_axpy(p, u, y, al, ap, true);
        } else {
          rc = LG_OK;
        }
        if (rc) return rc;
      }
      CK(cudaMemcpyAsync(p->dd_st, p->dd_nx, sizeof(double2) * T * (1 + I) * d, cudaMemcpyDeviceToDevice, p->stream));
    }
  }
  return LG_OK;
}

}  // namespace lgi
