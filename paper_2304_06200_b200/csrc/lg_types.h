// Device-side data descriptors shared by the host orchestration (lg_api.cu),
// the step-preparation kernels (lg_prep.cu) and the sweep engine (lg_engine.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define LG_MAX_CHANNELS 16
#define LG_MAX_SPECS 8
#define LG_MAXW 64  // widest ELL row handled by the bit-exact row-sum path

// Cluster engine (lg_sweep_cl.cuh) shared-memory layout, in 16-byte words, up to the word
// holding the two exchange mbarriers (reduction scratch, 1/(s j) table, 2 or 4 window
// buffers of cmax columns, packed slot columns, staged control rows acw = Kc * Wc).
__host__ __device__ inline int lg_cl_mb_word(int R, int H, int Q, int E, int cmax, int W, int acw) {
  const int T = 32 * ((R + 2 * E + 31) / 32);
  return 16 * 32 + 16 * 16 + 72 + (Q > 1 ? 4 : 2) * cmax * (R + 2 * (E + H)) + ((W + 3) / 4 * T + 3) / 4 + acw * T +
         (acw * T + 3) / 4;
}

// LARGE cluster kernels (lg_sweep_cl_large.cuh): two rows per thread (T threads, R <= 2 T),
// one Taylor term per exchange.  Reduction scratch, 1/(s j) table, two window buffers of cmax
// columns, staged control rows [acw][2 T] (values, then int columns), then the two exchange
// mbarriers (one 16-byte word).
// Entries per staged control row table: one per OWN row (rows past R are never touched), not one per
// thread slot, so the thread count can exceed R / rpt without growing shared memory.
__host__ __device__ inline int lg_cll_as(int R, int T, int rpt) {
  const int r8 = (R + 7) & ~7;
  return r8 < rpt * T ? r8 : rpt * T;
}
__host__ __device__ inline int lg_cll_mb_word(int R, int H, int T, int cmax, int acw, int rpt) {
  const int as = lg_cll_as(R, T, rpt);
  return 16 * 32 + 16 * 16 + 72 + 2 * cmax * (R + 2 * H) + acw * as + (acw * as + 3) / 4;
}

// Cost kinds (src/costs.py:49-61)
enum LgKind { LGK_STATE_INF = 0, LGK_STATE_PEN = 1, LGK_STATE_RUN = 2, LGK_GATE = 3, LGK_GATE_RUN = 4 };

// ---------------------------------------------------------------- step preparation (G1)
struct LgPrepArgs {
  int d, Kc, N;
  double dt;
  const double* amps;  // [N][Kc]
  int dense;           // storage of H_n (any input dense -> dense, src/sparse.py:322-334)
  int materialise;     // 2d <= 256 (src/derivatives.py:29,199-202)
  // sparse: union ELL pattern of H_s and all h_c (CSR column order per row)
  int W;
  const int* rowlen;   // [d]
  const int* src_s;    // [W][d] index into hs_vals or -1
  const int* src_c;    // [Kc][W][d] index into hc_vals[c] or -1
  const double2* hs_vals;
  const double2* const* hc_vals;  // device array of Kc pointers
  const int* colptr;   // [d+1] union pattern transposed (slots w*d+i sorted by row)
  const int* colent;   // [nnz_union]
  // dense inputs (column-major)
  const double2* hs_dense;              // [d*d]
  const double2* const* hc_dense;       // Kc pointers [d*d]
  // control-generator statistics for A_c = -i dt h_c (host-computed, numpy rules)
  const double* ctrl_col;   // [Kc][d] column abs sums
  const double* ctrl_row;   // [Kc][d] row abs sums
  const int* ctrl_nnz;      // [Kc][d] stored entries per row
  int Wc;                   // sparse materialised aux needs A_c row entries in column order
  const int* ac_rowlen;     // [Kc][d]
  const double* ac_abs;     // [Kc][Wc][d] |A_c| entries in column order (slot w of row i)
  const double* ac_abs_dense;  // dense materialised: [Kc][d*d] |A_c| column-major
  // outputs
  double2* A;               // [N][W][d] step generators (nullptr: do not store)
  double* norm1;            // [N]
  long long* sp;            // [N]
  double* aux_arg;          // [N][Kc] sqrt(||aux||_1 ||aux||_inf)
  long long* aux_sp;        // [N][Kc]
};

// ---------------------------------------------------------------- sweep engine
struct LgSpecDev {
  int kind;
  double weight;
  int set;                 // 0 = state trajectories, 1 = gate basis
  int pen_W;               // STATE_PEN: ELL width of the penalty operator
  const int* pen_cols;     // [W][d]
  const double2* pen_vals; // [W][d]
  const double2* tgt;      // [T_set][d] targets (state) / images U_T psi_h (gate), rows = set order
};

struct LgEngineArgs {
  int d, N, Kc, W, Wc;
  int n_specs;
  LgSpecDev spec[LG_MAX_SPECS];
  int set_nspec[2];
  int set_spec[2][LG_MAX_SPECS];
  int set_t0[2], set_T[2];   // global trajectory index range of each set
  int T_total;
  // groups: blockIdx.x / n_slabs = group; each group = trajectory range in one set
  int n_groups, n_slabs, grp_T;   // trajectories per group (last may be short)
  int grp_set[64], grp_t0[64], grp_nT[64];
  // operators
  const int* A_cols;        // [W][d]
  const double2* A;         // [N][W][d]
  const int* Ac_cols;       // [Kc][Wc][d]
  const double2* Ac;        // [Kc][Wc][d]
  const int4* plan;         // [N][1+Kc] (order, scaling, status, -)
  const double* rtab;       // [N][64] 1/(s (j+1)), j < order, of the propagation plans (ws engine, sparse)
  const double2* psi0;      // [T_total][d] initial trajectories
  // scratch
  double2* scratch;         // per group: scratch_per_group d-vectors
  long long scratch_per_group;  // in double2 units
  unsigned* bar;            // per group [4]
  double2* red;             // per group [2][red_cap][n_slabs]
  int red_cap;
  int smem_bytes;           // dynamic shared memory provided
  int smem_mode;            // legacy engine: bit0 state in smem, bit1 term buffers, bit2 A_n; cta engine: bit2 A_n, bit3 A_c
  int row_lanes;            // cta engine: row lanes (multiple of 32); blockDim = row_lanes x column slots
  int cta_Imax;             // cta engine: max specs per set (state layout stride)
  // raw outputs (indexed by global trajectory)
  double2* ip;              // [N][n_specs][Kc][T_total]
  double2* fin;             // [n_specs][T_total]
  double* run;              // [n_specs][T_total]
  double2* trp;             // [n_specs][N][T_total]
  double2* psiN;            // [T_total][d] final states (forward -> backward)
  const double2* trsum;     // [n_specs][N] trace sums (GATE_RUN), filled between sweeps
  long long* trace;         // optional: per-team clock64 trace [group][team][N][4] (LG_TRACE)
  // cluster engine (lg_sweep_cl.cu): RCM renumbering of the rows
  int cl_R, cl_H;           // rows per CTA, bandwidth of the renumbered pattern
  int cl_Q, cl_E;           // Taylor terms per cluster exchange; ghost rows computed beyond the own rows per side
  // DIAGONALIZATION backend (CTA engine): A holds U_n = exp(-i H_n dt) column-major per step,
  // diag_Ud U_n^dagger, diag_D [N][Kc] the derivative operators dU_n/da_k (src/derivatives.py:251-275)
  int diag;
  const double2* diag_Ud;
  const double2* diag_D;
  int cl_acs;               // backward stages the control-generator rows in shared memory
  int dbg;                  // LG_DBG bits (timing experiments only; results are wrong when set)
  unsigned cl_cshare;       // bit k: control channel k has channel k-1's column pattern (LARGE aux chains)
  double2* bk_psi;          // cluster LARGE two-phase backward: psi_{n-1} [group][N][d] (renumbered rows)
  double2* bk_lam;          // ... lambda_s(n) [group][N][cta_Imax][d]
  unsigned* bk_flag;        // ... steps stored so far per (group, cluster rank) (release / acquire, gpu scope)
  unsigned* bk_next;        // ... [0] next derivative-product item (atomic work counter), [1] watchdog error,
                            //     [2] adjoint clusters started
  int bk_ranks;             // ... cluster size of the adjoint sweep (flags per trajectory)
  int bk_conc;              // ... this item kernel runs concurrently with the adjoint sweep
  int ws_nw;                // ws cluster backward: derivative workers per control channel
  int dense_rows;           // every operator row stores all d columns in order (dense H): slot w == column w
  const int* cl_perm;       // [d] renumbered row -> original row
  const int* cl_inv;        // [d] original row -> renumbered row
  const int* cl_cols;       // [W][d] renumbered column of slot w of renumbered row i
  const unsigned char* cl_slot;  // [W][d] source ELL slot of engine slot w (bank-conflict-free order)
  const int* cl_accols;     // [Kc][Wc][d] same for the control generators
};

struct LgFinalArgs {
  int N, Kc, n_specs, T_total;
  int kind[LG_MAX_SPECS];
  double weight[LG_MAX_SPECS];
  int t0[LG_MAX_SPECS], K[LG_MAX_SPECS];
  const double2* ip;
  const double2* fin;
  const double* run;
  const double2* trp;
  double* grad;   // [N][Kc]
  double* cost;   // [1]
};

// ---- host <-> dense-path kernel arguments (lg_dense.cu; filled by the host units)
struct LgGemmSeg {
  const double2* A;  // interleaved complex, column-major
  int lda;
  const double2* X;
  int ldx;
  int K;
};
struct LgGemmArgs {
  int M, C;
  LgGemmSeg seg[2];
  int nseg;
  const double2* xin;
  int ldxin;
  double2* cur;
  int ldc;
  double2* tout;
  int ldt;
  double r;
  int first, last;
  int ksplit;  // lg_dense.cu: split-k slices (partial products in `partial`)
  double2* partial;
  int* tile_ctr;  // per-output-tile arrival counters (zeroed; the last slice resets): fused split-k finish
  int zfast;      // k-slice index on blockIdx.x (slices of a tile co-scheduled) instead of blockIdx.z
};
struct LgDotArgs {
  int d, n;
  const double2* u[64];
  const double2* v[64];
  double2* out[64];
  int mode[64];  // 0: *out = <u|v>; 1: ((double*)out)[0] += Re<u|v>; 2: ((double*)out)[0] += |<u|v>|^2
};
struct LgEllArgs {
  int d, W, ncol, accumulate;
  const int* cols;
  const double2* vals;
  const double2* x[64];
  double2* y[64];
};
struct LgAxpyArgs {
  int d, ncol;
  const double2* u[64];
  double2* y[64];
  double2 alpha[64];
  const double2* alpha_ptr[64];
  int accumulate[64];
};
struct LgEllTaylorArgs {  // lg_dense.cu
  int d, W, ncol, first, last;
  double r;
  const int* cols;
  const double2* vals;
  const double2* X;
  const double2* xin;
  double2* cur;
  double2* T;
};
