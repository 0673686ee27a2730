// Internal host-side declarations shared by the library's host units (lg_host.cu,
// lg_configure.cu, lg_dense_host.cu, lg_api.cu).  Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/leangrape_b200.h"
#include "lg_final.cuh"
#include "lg_numpy.cuh"
#include "lg_planner.cuh"
#include "lg_types.h"

// kernel getters of the device units
extern "C" void* lg_forward_kernel(int multi);
extern "C" void* lg_backward_kernel(int multi);
extern "C" void* lg_trsum_kernel();
extern "C" void* lg_ell_taylor_kernel();
extern "C" void* lg_finalize_kernel();
extern "C" void* lg_prep_sparse_kernel();
extern "C" void* lg_prep_dense_kernel();
extern "C" void* lg_plans_kernel();
extern "C" void* lg_gather_kernel();
extern "C" void* lg_cta_kernel(int backward, int maxr, int maxc, int wreg);
extern "C" void* lg_zgemm_kernel();
extern "C" void* lg_zgemm_n32_kernel();
extern "C" int lg_zgemm_smem_bytes(int ntt);
extern "C" void* lg_zgemm_bulk_kernel();
extern "C" int lg_zgemm_bulk_smem_bytes();
extern "C" void* lg_taylor_epi_kernel();
extern "C" void* lg_cl_kernel(int backward, int W, int maxc, int small);
extern "C" int lg_cl_smem_words(int R, int H, int Q, int E, int cmax, int W, int acw);
extern "C" void* lg_ws_kernel(int backward, int W, int rpl);
extern "C" void* lg_rtab_kernel();
extern "C" int lg_ws_dense_width(int d);
extern "C" int lg_ws_layout_words(int d, int nteams, int I, int Wp, int extra_bars, int dense);
extern "C" void* lg_dense_form_kernel();
extern "C" void* lg_dots_kernel();
extern "C" void* lg_ell_kernel();
extern "C" void* lg_axpy_kernel();

namespace lgi {

extern thread_local std::string g_err;
int fail(int code, const std::string& msg);

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) return fail(LG_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct Mat {
  bool dense = false;
  long n = 0;
  std::vector<long> indptr, indices;  // CSR
  std::vector<double2> vals;          // CSR values or dense column-major
  long nnz() const { return dense ? n * n : (long)indices.size(); }
};

int parse_mat(const lg_matrix& m, long d, Mat* out, const char* what);
// ELL of one operator (for the engine): W = widest row, padded with (col = row, value 0).
void to_ell(const Mat& m, int* W_out, std::vector<int>& cols, std::vector<double2>& vals, std::vector<int>* rowlen);

inline double2 gen_host(double2 h, double dt) { return make_double2(dt * h.y, -(dt * h.x)); }

struct DevMem {
  std::vector<void*> ptrs;
  bool failed = false;  // some alloc() since the last release() failed: callers check this once
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    if (cudaMalloc(&p, count * sizeof(T)) != cudaSuccess) {
      cudaGetLastError();  // clear the (non-sticky) allocation error
      failed = true;
      return nullptr;
    }
    ptrs.push_back(p);
    return (T*)p;
  }
  template <class T>
  T* upload(const std::vector<T>& v) {
    T* p = alloc<T>(v.size());
    if (p && !v.empty()) cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
    return p;
  }
  void release() {
    for (void* p : ptrs) cudaFree(p);
    ptrs.clear();
    failed = false;
  }
};

struct Spec {
  int kind;
  double weight;
  int set;
  std::vector<double2> tgt;  // [K_set][d]
  Mat pen;
  int pen_W = 0;
  int* d_pen_cols = nullptr;
  double2* d_pen_vals = nullptr;
  double2* d_tgt = nullptr;
};

void release_diag(lg_problem* p);  // lg_diag.cu

}  // namespace lgi

using lgi::DevMem;
using lgi::Mat;
using lgi::Spec;

struct lg_problem {
  int device = 0;
  long d = 0;
  int Kc = 0;
  bool dense = false, materialise = false;
  double tau = 1e-8;
  Mat hs;
  std::vector<Mat> hc;
  std::vector<Spec> specs;
  // trajectories
  int set_t0[2] = {0, 0}, set_T[2] = {0, 0};
  int T_total = 0;
  std::vector<double2> traj;
  // union ELL
  int W = 0;
  std::vector<int> rowlen, cols, src_s, src_c, colptr, colent;
  // control ELL
  int Wc = 0;
  std::vector<int> ccols, crowlen;
  std::vector<double2> cvals;
  // engine configuration
  bool multi = false;
  int engine = 0;  // 0 legacy single-CTA, 1 legacy multi-CTA (grid barrier), 2 cta engine, 3 dense GEMM
  bool dense_large = false;
  bool diag_dense = false;  // DIAGONALIZATION backend on the dense GEMM engine (d > 128)
  bool dense_bwd_marked = false;  // run_dense recorded the forward / backward phase event of this evaluation
  // dense GEMM engine buffers
  double2* d_Ad = nullptr;           // dense engine: A_n = -i dt H_n, interleaved, column-major
  std::vector<double2*> d_Acd;       // A_c = -i dt h_c per channel
  double2 *dd_st = nullptr, *dd_nx = nullptr, *dd_cur = nullptr, *dd_tb0 = nullptr, *dd_tb1 = nullptr,
          *dd_xcur = nullptr, *dd_xtb0 = nullptr, *dd_xtb1 = nullptr, *dd_tmp = nullptr;
  double2* dd_dots = nullptr;
  double dense_dt = NAN;
  std::vector<double2*> d_hc_dense_host;
  int cta_maxr = 1, cta_maxc = 1, cta_wreg = 0, row_lanes = 32, cta_Imax = 1;
  int ws_rpl = 1, ws_fwd_smem = 0, ws_bwd_smem = 0, ws_bwd_threads = 0;
  bool ws_cluster = false;
  int ws_nw = 1;  // derivative workers per channel in the cluster backward
  double2* d_splitws = nullptr;  // dense engine split-k workspace (cudaMalloc'd, freed in ~lg_problem)
  size_t splitws_cap = 0;
  int* d_tilectr = nullptr;  // dense engine: per-tile arrival counters of the fused split-k finish
  // cluster engine
  int cl_split = 0, cl_R_b = 0, cl_Q_b = 1, cl_E_b = 0, cl_T_b = 0, cl_smem_split = 0;  // split backward
  int cl_CS = 0, cl_R = 0, cl_H = 0, cl_Q = 1, cl_E = 0, cl_small = 0, cl_maxc = 0, cl_smem = 0, cl_smem_b = 0, cl_acs = 0;
  unsigned cl_cshare = 0;  // bit k: control channel k has channel k-1's (renumbered) column pattern
  int cl_aux_ncl = 0;  // two-phase backward: co-resident clusters of the item kernel (0: fused backward)
  // item layout: the derivative-product items on smaller clusters of the LARGE kernels (0: the sweep layout)
  int cli_CS = 0, cli_R = 0, cli_smem = 0, cli_ncl = 0, cli_T = 320;
  DevMem bkmem;        // ... its psi_{n-1} / lambda_s(n) store
  long bk_cap = 0;
  double2 *d_bk_psi = nullptr, *d_bk_lam = nullptr;
  unsigned* d_bk_flag = nullptr;  // [n_groups][CS] steps stored, then [1] item counter
  cudaStream_t stream2 = nullptr;  // concurrent derivative-product items (two-phase backward)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int *d_cl_perm = nullptr, *d_cl_inv = nullptr, *d_cl_cols = nullptr, *d_cl_accols = nullptr;
  unsigned char* d_cl_slot = nullptr;
  int n_groups = 0, n_slabs = 1, threads = 512, smem_mode = 0, smem_bytes = 0, red_cap = 64;
  long scratch_per_group = 0;
  std::vector<int> grp_set, grp_t0, grp_nT;
  int live_peak = 0;
  long shard_b = 0, shard_e = 1L << 40;
  // device: static
  // line-search batch (lg_cost_batch): per-candidate raw outputs [k][fin | run | trp], final
  // states, costs and engine arguments
  DevMem bmem;
  long bcap_k = 0, bcap_N = 0;
  double* d_bat = nullptr;
  double2* d_bpsi = nullptr;
  double* d_bcost = nullptr;
  LgEngineArgs* d_bEA = nullptr;
  DevMem mem;
  cudaStream_t stream = nullptr;
  int *d_rowlen = nullptr, *d_cols = nullptr, *d_src_s = nullptr, *d_src_c = nullptr, *d_colptr = nullptr,
      *d_colent = nullptr;
  double2* d_hs = nullptr;
  double2** d_hc_ptrs = nullptr;
  double2* d_hs_dense = nullptr;
  double2** d_hc_dense_ptrs = nullptr;
  int* d_ccols = nullptr;
  double2* d_traj = nullptr;
  double2* d_scratch = nullptr;
  unsigned* d_bar = nullptr;
  double2* d_red = nullptr;
  // per-dt control data
  double cached_dt = NAN;
  DevMem dtmem;
  double2* d_Ac = nullptr;
  double *d_ctrl_col = nullptr, *d_ctrl_row = nullptr, *d_ac_abs = nullptr, *d_ac_abs_dense = nullptr;
  int *d_ctrl_nnz = nullptr, *d_ac_rowlen = nullptr;
  // per-N buffers
  long capN = 0;
  DevMem nmem;
  double* d_amps = nullptr;
  double2* d_A = nullptr;
  double *d_norm1 = nullptr, *d_aux_arg = nullptr, *d_parg = nullptr;
  long long *d_sp = nullptr, *d_aux_sp = nullptr, *d_psp = nullptr;
  int4* d_plan = nullptr;
  double* d_rtab = nullptr;  // [N][64] Taylor coefficient table (ws engine)
  int* d_flag = nullptr;
  double2 *d_ip = nullptr, *d_fin = nullptr, *d_trp = nullptr, *d_trsum = nullptr, *d_psiN = nullptr;
  // sharded evaluation: raw scalars [ip | fin | trp | run] in one (optionally caller-lent) buffer and
  // the caller's all-reduce hook (lg_eval_sharded)
  double* d_raw = nullptr;
  double* ext_raw = nullptr;
  long ext_raw_len = 0;
  lg_allreduce_fn hook = nullptr;
  void* hook_user = nullptr;
  bool trp_reduced = false;
  bool has_gate_run = false;
  double *d_run = nullptr, *d_grad = nullptr, *d_cost = nullptr;
  int *d_spec_t0 = nullptr, *d_spec_K = nullptr;
  long lastN = 0;
  bool own_stream = true;
  bool timing = false;
  // DIAGONALIZATION backend (lg_diag.cu): per-step exact propagators and derivative operators
  int backend = 0;                 // 0 scaling-and-squaring (Taylor), 1 diagonalization
  DevMem diagmem;                  // per-N: U^dagger, D, eigen workspace
  long diag_capN = 0;
  bool diag_need_aux = false;
  double2 *d_Ud = nullptr, *d_D = nullptr, *d_V = nullptr, *d_wk0 = nullptr, *d_wk1 = nullptr, *d_ph = nullptr;
  double* d_w = nullptr;
  int* d_info = nullptr;
  void* cublas = nullptr;          // cublasHandle_t
  void* cusolver = nullptr;        // cusolverDnHandle_t
  const char* diag_solver = "";
  cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  double phase_ms[4] = {0, 0, 0, 0};
  long timed_evals = 0;

  ~lg_problem() {
    lgi::release_diag(this);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    nmem.release();
    dtmem.release();
    bmem.release();
    bkmem.release();
    mem.release();
    if (d_splitws) cudaFree(d_splitws);
    if (d_tilectr) cudaFree(d_tilectr);
    if (stream2) cudaStreamDestroy(stream2);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (stream && own_stream) cudaStreamDestroy(stream);
  }
  void mark(int i) {
    if (timing) cudaEventRecord(ev[i], stream);
  }
  void collect() {
    if (!timing) return;
    cudaEventSynchronize(ev[4]);
    for (int i = 0; i < 4; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      phase_ms[i] += ms;
    }
    ++timed_evals;
  }
};

namespace lgi {

extern long long g_launches;  // kernels launched by this library (lg_launch_count)

// lg_host.cu: problem ingestion and per-evaluation preparation
int build_problem(const lg_problem_desc* D, lg_problem* p);
int prepare_dt(lg_problem* p, double dt);
int ensure_N(lg_problem* p, long N);
int launch(void* f, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t st, bool coop = false);
void ensure_smem(void* f, size_t smem);
int prepare_steps(lg_problem* p, long N, double dt, bool need_aux);
int prepare_diag(lg_problem* p, long N, double dt, bool need_aux);  // lg_diag.cu
LgEngineArgs engine_args(lg_problem* p, long N);
LgFinalArgs final_args(lg_problem* p, long N, const double2* ip, const double2* fin, const double* run,
                       const double2* trp, double* grad, double* cost);

// lg_configure.cu: engine selection
int configure(lg_problem* p);
std::vector<int> rcm_order(long d, const std::vector<std::vector<int>>& adj);
void cl_color_slots(long d, int W, int R, const std::vector<int>& perm, const std::vector<int>& rowlen,
                    const std::vector<int>& cp, std::vector<int>& ncol, std::vector<unsigned char>& nslot);

// lg_dense_host.cu: dense (DMMA) engine driver
int configure_dense(lg_problem* p);
int run_dense(lg_problem* p, long N, double dt, bool grad);
int dense_gemm(lg_problem* p, const double2* A, const double2* X, const double2* B, const double2* Xb, int C,
               double r, bool first, bool last, const double2* xin, double2* cur, double2* tout);

}  // namespace lgi
