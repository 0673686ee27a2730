/* leangrape_b200.h -- C ABI of the B200-native HG cost+gradient evaluation.
 *
 * The reference (`leangrape`, pure Python) has no FFI layer; its drop-in
 * boundary is the function pair the optimiser binds
 *     composite_grad(problem, a, terms) -> GradientResult   (src/costs.py:515-546)
 *     composite_cost(problem, a, terms) -> float            (src/costs.py:549-597)
 * called from grape_optimize (src/optimizer.py:18,117,150,159,169).  Every
 * entry point below replaces one piece of that surface; the Python mirror
 * (paper_2304_06200_b200/costs.py) binds them with ctypes exactly as
 * INTEGRATION.md shows.  Plain pointers and sizes only: complex numbers are
 * interleaved (re, im) float64 pairs, matrices are CSR (int64 offsets/indices)
 * or column-major dense, exactly the reference's CsrMatrix / DenseMatrix
 * layouts (src/sparse.py:42-60,152-170).
 *
 * Status codes map onto the reference's exception types (see lg_last_error()).
 * A handle is not thread-safe; calls are synchronous like the Python API.
 */
#ifndef LEANGRAPE_B200_H
#define LEANGRAPE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------- */
#define LG_OK 0
#define LG_INVALID_ARG 1         /* ValueError   (src/costs.py:75-85,112-121,151-168) */
#define LG_PLANNING_INFEASIBLE 2 /* PlanningError(RuntimeError) (src/expm.py:61-62,244-249,273-276) */
#define LG_CUDA_ERROR 3          /* RuntimeError */
#define LG_NCCL_ERROR 4          /* RuntimeError */
#define LG_INDEX_ERROR 5         /* IndexError   (src/derivatives.py:214-215) */
#define LG_UNSUPPORTED 6         /* NotImplementedError (e.g. DIAGONALIZATION backend) */

/* ---- cost kinds: CostKind (src/costs.py:49-61) -------------------------- */
#define LG_STATE_INFIDELITY 0
#define LG_STATE_PENALTY 1
#define LG_STATE_RUNNING_INFIDELITY 2
#define LG_GATE_INFIDELITY 3
#define LG_GATE_RUNNING_INFIDELITY 4

/* One square operator: CsrMatrix (dense == 0) or DenseMatrix (dense == 1). */
typedef struct {
  int32_t dense;
  int64_t n;
  int64_t nnz;                /* CSR: stored elements                          */
  const int64_t* row_offsets; /* CSR: [n + 1]                                   */
  const int64_t* col_indices; /* CSR: [nnz], strictly increasing per row        */
  const double* values;       /* CSR: [2 nnz]; dense: [2 n n] column-major      */
} lg_matrix;

/* One CostTerm (src/costs.py:141-168).  `targets` holds one complex vector
 * of length d per trajectory of the term's set: the target states (state
 * kinds) or the target images U_T |psi_0^h> (gate kinds; the images replace a
 * dense d x d target_gate, which at d = 10^4 would not fit the host). */
typedef struct {
  int32_t kind;
  double weight;
  const double* targets; /* [K][2 d] or NULL for STATE_PENALTY */
  lg_matrix penalty;     /* STATE_PENALTY only */
} lg_cost_term;

/* ControlProblem (src/costs.py:96-138) plus the K-state block:
 *   initial_states : the K_s state-transfer trajectories (reference: one initial_state)
 *   basis          : the K_g gate basis states (reference: d states; here K_g <= d,
 *                    subspace costs normalised by K_g, == reference at K_g == d).
 * shard_begin/shard_end select the trajectories this process owns (multi-GPU);
 * shard_end <= 0 means all. */
typedef struct {
  lg_matrix h_static;
  int32_t n_channels;
  const lg_matrix* h_controls;
  double tau;
  int64_t n_states;
  const double* initial_states; /* [K_s][2 d] */
  int64_t n_basis;
  const double* basis; /* [K_g][2 d] */
  int32_t n_terms;
  const lg_cost_term* terms;
  int32_t device;
  int64_t shard_begin, shard_end;
  /* Backend (src/derivatives.py:48-51): 0 SCALING_SQUARING (certified Taylor action),
   * 1 DIAGONALIZATION (per-step eigenfactorisation, src/derivatives.py:228-275; dense
   * operators: the CTA engine applies the propagators for d <= 128, the dense GEMM engine above). */
  int32_t backend;
} lg_problem_desc;

typedef struct lg_problem lg_problem;

/* Copy operators, trajectories and targets to the device once per problem. */
int lg_problem_create(const lg_problem_desc* desc, lg_problem** out);
void lg_problem_destroy(lg_problem* p);

/* composite_grad: cost and gradient grad[n * n_channels + k] = dC/da[n, k]
 * for the ControlField (n_steps, n_channels, dt, amps[n_steps][n_channels]). */
int lg_eval(lg_problem* p, int64_t n_steps, double dt, const double* amps, double* cost, double* grad,
            int64_t* live_vector_peak);

/* composite_cost: forward sweeps only (line search, src/optimizer.py:153-170). */
int lg_cost(lg_problem* p, int64_t n_steps, double dt, const double* amps, double* cost);

/* composite_cost of n_fields candidate fields in ONE forward launch (the line search's trial
 * fields, src/optimizer.py:153-170): amps[c][n_steps][n_channels], costs[c].  Each cost is
 * bit-identical to lg_cost on that field.  LG_UNSUPPORTED on engines without a batched forward
 * kernel (dense GEMM, DIAGONALIZATION backend) and on sharded problems. */
int lg_cost_batch(lg_problem* p, int32_t n_fields, int64_t n_steps, double dt, const double* amps, double* costs);

/* Same as lg_eval, but with amplitudes already resident on the device and the
 * results left on the device (benchmarking the kernels without host copies). */
int lg_eval_device(lg_problem* p, int64_t n_steps, double dt, const double* d_amps, double* d_cost, double* d_grad);

/* Per-step planner inputs and plans exactly as the reference's StepEvaluator
 * computes them (src/derivatives.py:105-110,187-196): for debugging and the
 * bit-exact plan-parity tests.  aux_* arrays are [n_steps][n_channels]. */
int lg_plan_table(lg_problem* p, int64_t n_steps, double dt, const double* amps, double* norm1, int64_t* sigma,
                  int32_t* order, int32_t* scaling, double* aux_arg, int64_t* aux_sigma, int32_t* aux_order,
                  int32_t* aux_scaling);

/* Forward-propagated final states of the state trajectories, [K_s][2 d]
 * (forward_propagate, src/costs.py:209-217). */
int lg_forward_states(lg_problem* p, int64_t n_steps, double dt, const double* amps, double* out);

/* (dU_step / da_channel) psi of a DIAGONALIZATION problem, [2 d]: the per-step derivative product of
 * the reference's eigenbasis formula (derivative_action_diag, src/derivatives.py:256-275, as
 * StepEvaluator.control_derivative calls it, :317-320), from the device factorisation of the
 * field's steps.  LG_UNSUPPORTED for Taylor problems (their product is lg_expm_apply on the embedded
 * generator), LG_INDEX_ERROR for a step or channel out of range. */
int lg_step_derivative(lg_problem* p, int64_t n_steps, double dt, const double* amps, int64_t step, int32_t channel,
                       const double* psi, double* out);

/* Raw per-trajectory scalars of the last evaluation (for sharded runs: the
 * partial sums every rank contributes; summing them across ranks and calling
 * lg_finalize_host reproduces the single-process result exactly). */
int64_t lg_raw_size(lg_problem* p, int64_t n_steps);
int lg_raw_get(lg_problem* p, double* raw);
int lg_finalize_host(lg_problem* p, int64_t n_steps, const double* raw, double* cost, double* grad);

/* Multi-GPU: one process per GPU, each holding the problem created with its
 * shard [shard_begin, shard_end) of the trajectory block (north_star: "the
 * K-state block shards across the GPUs ... one allreduce per evaluation").
 * The library calls `allreduce` (sum, in place, on device memory, ordered on
 * `stream`) at the points where the shards exchange data:
 *   - between the sweeps, the running gate traces (only if a
 *     LG_GATE_RUNNING_INFIDELITY term is present: its costate source needs the
 *     global traces, src/costs.py:462,477-478);
 *   - after the backward sweep, the raw per-trajectory scalars, before the
 *     device combine (src/costs.py:484-487, 543-544).
 * Every rank must make the same sequence of calls.  Returns 0 on success.
 * With lg_set_raw_buffer the raw scalars live in caller-owned device memory
 * (e.g. a torch tensor of lg_raw_size doubles), so the hook can hand views of
 * it straight to NCCL. */
typedef int (*lg_allreduce_fn)(double* d_buf, int64_t count, void* stream, void* user);
int lg_set_raw_buffer(lg_problem* p, double* d_raw, int64_t len);
int lg_eval_sharded(lg_problem* p, int64_t n_steps, double dt, const double* amps, lg_allreduce_fn allreduce,
                    void* user, double* cost, double* grad);
int lg_cost_sharded(lg_problem* p, int64_t n_steps, double dt, const double* amps, lg_allreduce_fn allreduce,
                    void* user, double* cost);

/* Standalone certified action (src/expm.py:306-369).
 * lg_expm_plan_inputs: the planner inputs of a generator A exactly as the reference computes them
 *   (A.one_norm() with numpy's reduction order, A.max_row_nnz(); DenseMatrix -> n), host only.
 * lg_expm_apply: exp(A) applied to n_vec vectors (psi: [n_vec][2n], interleaved complex) under the
 *   plan (order, scaling) -- the Taylor recursion of expm.apply on the GPU; out may alias psi. */
int lg_expm_plan_inputs(const lg_matrix* a, double* norm1, int64_t* sigma_prime);
int lg_expm_apply(const lg_matrix* a, int64_t n_vec, const double* psi, int32_t order, int32_t scaling,
                  double* out, int32_t device);

/* y_k = A x_k for n_vec vectors [n_vec][2 n] on the device (CsrMatrix.matvec / DenseMatrix.matvec /
 * sparse.matvec, src/sparse.py:69-88,193-199,297-298): the stored matrix goes through the same ELL
 * layout and row kernel the sweeps use for penalty operators. */
int lg_matvec(const lg_matrix* a, int64_t n_vec, const double* x, double* y, int32_t device);

/* make_plan (src/expm.py:279-303) on the host: bit-identical to the reference. */
int lg_make_plan(double norm1, int64_t sigma_prime, double tau, int32_t m_max, int32_t s_max, int32_t* order,
                 int32_t* scaling, double* bound);

/* Evaluate a batch of plans with the DEVICE planner (guarded; uncertain ones
 * fixed on the host) -- exposed for the planner parity test. */
int lg_make_plans_device(int64_t count, const double* norm1, const int64_t* sigma, double tau, int32_t* order,
                         int32_t* scaling, int32_t* status, int32_t* n_uncertain);

/* Handle-free combine of raw per-trajectory scalars (layout of lg_raw_get):
 * what every rank runs after the cross-rank sum.  kinds/weights/t0/K per term. */
int lg_finalize_raw(int32_t n_terms, const int32_t* kinds, const double* weights, const int32_t* t0,
                    const int32_t* K, int64_t n_steps, int32_t n_channels, int32_t n_traj, const double* raw,
                    double* cost, double* grad);

/* Host restatements of the numpy reductions that feed the planner
 * (lg_numpy.cuh) -- test hooks for the bit-exactness rules. */
void lg_np_cabs_host(int64_t n, const double* z /* [2n] */, double* out);
double lg_np_pairwise_host(int64_t n, const double* a);
double lg_np_reduce_host(int64_t n, const double* a);

/* Launch on a caller-owned stream (e.g. torch.cuda.current_stream()) and/or
 * record CUDA events around every phase of every evaluation:
 * phase_ms = {prep+plans, forward sweep, backward sweep, finalize}, summed
 * over `evals` evaluations since the last reset. */
int lg_set_stream(lg_problem* p, void* stream);
int lg_set_timing(lg_problem* p, int enable);
int lg_get_timing(lg_problem* p, double* phase_ms /* [4] */, int64_t* evals);

/* Benchmark hook: time the dense Taylor-term GEMM (lg_k_zgemm_taylor, the c5
 * operator-term) on random data, d x d times d x C complex; ms per launch. */
int lg_bench_zgemm(int32_t d, int32_t C, int32_t iters, double* ms_per_launch);

/* "<engine>:<dominant backward kernel>" chosen for this problem (diagnostics, bench.py roofline). */
const char* lg_engine_name(lg_problem* p);

/* DIAGONALIZATION backend (src/derivatives.py:228-246, the np.linalg.eigh call): which per-step
 * factorisation the last evaluation used -- "jacobi ..." (in shared memory, d <= 64),
 * "jacobi-global ..." (hand-written, any d), "syevBatched" / "syevd" (LG_DIAG_LIB=1 A/B path);
 * "" before the first evaluation or on the Taylor backend. */
const char* lg_diag_solver_name(lg_problem* p);
/* Device state vectors held per trajectory by this problem's engine (GradientResult.live_vector_peak,
 * src/costs.py:171-199); the same value lg_eval reports, also for sharded problems. */
int64_t lg_live_vector_peak(lg_problem* p);
/* Kernels launched by this library since load (all problems, all threads; diagnostics). */
int64_t lg_launch_count(void);
int lg_device_count(void);
const char* lg_last_error(void);
const char* lg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LEANGRAPE_B200_H */
