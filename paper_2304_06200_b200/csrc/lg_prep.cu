// Step preparation: all N step generators, their bit-exact planner inputs (G1)
// and the device planner (G2), for every step of one evaluation at once.
//
// Replaces, per step, ControlProblem.step_evaluator -> linear_combine ->
// build_csr_arrays (src/costs.py:131-138, src/sparse.py:237-270,313-349),
// _generator/_plan_for (src/derivatives.py:105-110), the aux embedding norms
// (src/derivatives.py:166-202, src/sparse.py:352-380) and make_plan
// (src/expm.py:279-303).  The reference does this serially, one step at a time,
// inside the sweep; here every step is independent, so one CTA per step.
//
// This translation unit is compiled with -fmad=false: the arithmetic below
// must round exactly like numpy (see lg_numpy.cuh).
#include "lg_final.cuh"
#include "lg_numpy.cuh"
#include "lg_planner.cuh"
#include "lg_types.h"

namespace {

__device__ __forceinline__ double2 h_entry_sparse(const LgPrepArgs& P, const double* amps, int w, int i) {
  // ((0 + v_s) + a_1 v_1) + a_2 v_2 ... in operand order, products rounded
  // separately; a zero amplitude skips its operand (src/sparse.py:336-349,257-263).
  const int idx = P.W * 0 + w * P.d + i;
  double hr = 0.0, hi = 0.0;
  int s = P.src_s[idx];
  if (s >= 0) {
    double2 v = P.hs_vals[s];
    hr = LG_ADD(hr, v.x);
    hi = LG_ADD(hi, v.y);
  }
  for (int c = 0; c < P.Kc; ++c) {
    double a = amps[c];
    if (a == 0.0) continue;
    int sc = P.src_c[(long)c * P.W * P.d + idx];
    if (sc < 0) continue;
    double2 v = P.hc_vals[c][sc];
    hr = LG_ADD(hr, LG_MUL(a, v.x));
    hi = LG_ADD(hi, LG_MUL(a, v.y));
  }
  return make_double2(hr, hi);
}

// A = H.scaled(-1j dt): (dt Im h, -dt Re h), each one rounded product.
__device__ __forceinline__ double2 gen_of(double2 h, double dt) {
  return make_double2(LG_MUL(dt, h.y), -LG_MUL(dt, h.x));
}

__device__ __forceinline__ double2 h_entry_dense(const LgPrepArgs& P, const double* amps, long pos) {
  double hr = LG_ADD(0.0, P.hs_dense[pos].x), hi = LG_ADD(0.0, P.hs_dense[pos].y);
  for (int c = 0; c < P.Kc; ++c) {
    double a = amps[c];
    if (a == 0.0) continue;
    double2 v = P.hc_dense[c][pos];
    hr = LG_ADD(hr, LG_MUL(v.x, a));
    hi = LG_ADD(hi, LG_MUL(v.y, a));
  }
  return make_double2(hr, hi);
}

template <class T>
__device__ T block_max(T v, T* sm) {
  for (int o = 16; o > 0; o >>= 1) {
    T u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    T r = sm[0];
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) r = sm[k] > r ? sm[k] : r;
    sm[32] = r;
  }
  __syncthreads();
  T r = sm[32];
  __syncthreads();
  return r;
}

}  // namespace

// One CTA per step: sparse (all-CSR) problems.
extern "C" __global__ void lg_k_prep_sparse(LgPrepArgs P) {
  __shared__ double smd[33];
  __shared__ long long sml[33];
  const int n = blockIdx.x;
  const int d = P.d, W = P.W, Kc = P.Kc;
  const double* amps = P.amps + (long)n * Kc;
  double2* A = P.A ? P.A + (long)n * W * d : nullptr;

  long long sp = 0;
  double gen_inf = 0.0;
  double aux_inf[LG_MAX_CHANNELS];
  long long aux_nz[LG_MAX_CHANNELS];
  for (int c = 0; c < Kc; ++c) aux_inf[c] = 0.0, aux_nz[c] = 0;

  // ---- row phase: generator values, sigma', row sums (a0 + pairwise, nonzeros only)
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    double av[LG_MAXW * 2];
    int nz = 0;
    const int L = P.rowlen[i];
    for (int w = 0; w < W; ++w) {
      double2 a = make_double2(0.0, 0.0);
      if (w < L) {
        double2 h = h_entry_sparse(P, amps, w, i);
        if (h.x != 0.0 || h.y != 0.0) {  // exact zeros are dropped (src/sparse.py:261-263)
          a = gen_of(h, P.dt);
          av[nz++] = lg_np_cabs(a.x, a.y);
        }
      }
      if (A) A[(long)w * d + i] = a;
    }
    auto get = [&](long k) { return av[k]; };
    double grow = lg_np_reduce(get, 0, nz);
    sp = nz > sp ? nz : sp;
    gen_inf = grow > gen_inf ? grow : gen_inf;
    for (int c = 0; c < Kc; ++c) {
      const long ci = (long)c * d + i;
      long long z = nz + P.ctrl_nnz[ci];
      aux_nz[c] = z > aux_nz[c] ? z : aux_nz[c];
      double r;
      if (P.materialise) {
        // top row i of aux_embed: A's entries then A_c's (columns + d)
        const int Lc = P.ac_rowlen[ci];
        for (int k = 0; k < Lc; ++k) av[nz + k] = P.ac_abs[((long)c * P.Wc + k) * d + i];
        r = lg_np_reduce(get, 0, nz + Lc);
      } else {
        r = LG_ADD(grow, P.ctrl_row[ci]);  // gen_rows + ctrl_rows (src/derivatives.py:175-178)
      }
      aux_inf[c] = r > aux_inf[c] ? r : aux_inf[c];
    }
  }
  sp = block_max(sp, sml);
  gen_inf = block_max(gen_inf, smd);
  for (int c = 0; c < Kc; ++c) {
    aux_inf[c] = block_max(aux_inf[c], smd);
    aux_nz[c] = block_max(aux_nz[c], sml);
  }
  __syncthreads();

  // ---- column phase: bincount order = ascending row within each column
  double gen_one = 0.0;
  double aux_one[LG_MAX_CHANNELS];
  for (int c = 0; c < Kc; ++c) aux_one[c] = 0.0;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double cs = 0.0;
    const int k0 = P.colptr[j], k1 = P.colptr[j + 1];
    for (int k = k0; k < k1; ++k) {
      int slot = P.colent[k];
      double2 a;
      if (A) {
        a = A[slot];
      } else {
        int w = slot / d, i = slot - w * d;
        double2 h = h_entry_sparse(P, amps, w, i);
        a = gen_of(h, P.dt);
      }
      cs = LG_ADD(cs, lg_np_cabs(a.x, a.y));
    }
    gen_one = cs > gen_one ? cs : gen_one;
    for (int c = 0; c < Kc; ++c) {
      const long cj = (long)c * d + j;
      double v;
      if (P.materialise) {
        // column d + j of aux_embed: A_c's entries (top rows) then A's (bottom rows)
        v = P.ctrl_col[cj];
        for (int k = k0; k < k1; ++k) {
          int slot = P.colent[k];
          double2 a;
          if (A) {
            a = A[slot];
          } else {
            int w = slot / d, i = slot - w * d;
            a = gen_of(h_entry_sparse(P, amps, w, i), P.dt);
          }
          v = LG_ADD(v, lg_np_cabs(a.x, a.y));
        }
      } else {
        v = LG_ADD(cs, P.ctrl_col[cj]);  // gen_cols + ctrl_cols (src/derivatives.py:166-171)
      }
      double m2 = v > cs ? v : cs;
      aux_one[c] = m2 > aux_one[c] ? m2 : aux_one[c];
    }
  }
  gen_one = block_max(gen_one, smd);
  for (int c = 0; c < Kc; ++c) aux_one[c] = block_max(aux_one[c], smd);
  if (threadIdx.x == 0) {
    P.norm1[n] = gen_one;
    P.sp[n] = sp;
    for (int c = 0; c < Kc; ++c) {
      double inf = aux_inf[c] > gen_inf ? aux_inf[c] : gen_inf;
      P.aux_arg[(long)n * Kc + c] = LG_SQRT(LG_MUL(aux_one[c], inf));
      P.aux_sp[(long)n * Kc + c] = P.materialise ? aux_nz[c] : aux_nz[c] + 1;
    }
  }
}

// One CTA per step: dense problems (DenseMatrix storage, src/sparse.py:152-231).
extern "C" __global__ void lg_k_prep_dense(LgPrepArgs P) {
  __shared__ double smd[33];
  const int n = blockIdx.x;
  const int d = P.d, Kc = P.Kc;
  const double* amps = P.amps + (long)n * Kc;
  double2* A = P.A ? P.A + (long)n * d * d : nullptr;
  const double dt = P.dt;

  auto absA = [&](long pos) {
    double2 a = gen_of(h_entry_dense(P, amps, pos), dt);
    return lg_np_cabs(a.x, a.y);
  };
  if (A) {
    for (long pos = threadIdx.x; pos < (long)d * d; pos += blockDim.x) A[pos] = gen_of(h_entry_dense(P, amps, pos), dt);
  }
  // ---- columns: pairwise over each contiguous column
  double gen_one = 0.0;
  double aux_one[LG_MAX_CHANNELS];
  for (int c = 0; c < Kc; ++c) aux_one[c] = 0.0;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    const long base = (long)j * d;
    auto col = [&](long k) { return absA(base + k); };
    double cs = lg_np_pairwise(col, 0, d);
    gen_one = cs > gen_one ? cs : gen_one;
    for (int c = 0; c < Kc; ++c) {
      double v;
      if (P.materialise) {
        // 2d x 2d dense aux_embed: column j -> [|A(:,j)|; 0], column d+j -> [|A_c(:,j)|; |A(:,j)|]
        const double* ac = P.ac_abs_dense + (long)c * d * d + base;
        auto lo = [&](long k) { return k < d ? absA(base + k) : 0.0; };
        auto hi = [&](long k) { return k < d ? ac[k] : absA(base + k - d); };
        double v0 = lg_np_pairwise(lo, 0, 2 * d);
        double v1 = lg_np_pairwise(hi, 0, 2 * d);
        v = v0 > v1 ? v0 : v1;
      } else {
        double t = LG_ADD(cs, P.ctrl_col[(long)c * d + j]);
        v = t > cs ? t : cs;
      }
      aux_one[c] = v > aux_one[c] ? v : aux_one[c];
    }
  }
  gen_one = block_max(gen_one, smd);
  for (int c = 0; c < Kc; ++c) aux_one[c] = block_max(aux_one[c], smd);
  // ---- rows: sequential across columns
  double gen_inf = 0.0;
  double aux_inf[LG_MAX_CHANNELS];
  for (int c = 0; c < Kc; ++c) aux_inf[c] = 0.0;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    double rs = 0.0;
    for (int j = 0; j < d; ++j) rs = LG_ADD(rs, absA((long)j * d + i));
    gen_inf = rs > gen_inf ? rs : gen_inf;
    for (int c = 0; c < Kc; ++c) {
      double v;
      if (P.materialise) {
        const double* ac = P.ac_abs_dense + (long)c * d * d;
        v = rs;
        for (int j = 0; j < d; ++j) v = LG_ADD(v, ac[(long)j * d + i]);
      } else {
        v = LG_ADD(rs, P.ctrl_row[(long)c * d + i]);
      }
      aux_inf[c] = v > aux_inf[c] ? v : aux_inf[c];
    }
  }
  gen_inf = block_max(gen_inf, smd);
  for (int c = 0; c < Kc; ++c) aux_inf[c] = block_max(aux_inf[c], smd);
  if (threadIdx.x == 0) {
    P.norm1[n] = gen_one;
    P.sp[n] = d;  // dense: every entry counts as stored
    for (int c = 0; c < Kc; ++c) {
      double inf = aux_inf[c] > gen_inf ? aux_inf[c] : gen_inf;
      P.aux_arg[(long)n * Kc + c] = LG_SQRT(LG_MUL(aux_one[c], inf));
      long long z = 0;
      if (P.materialise) {
        z = 2 * (long long)d;
      } else {
        for (int i = 0; i < d; ++i) {
          long long t = d + P.ctrl_nnz[(long)c * d + i];
          z = t > z ? t : z;
        }
        z += 1;
      }
      P.aux_sp[(long)n * Kc + c] = z;
    }
  }
}

// G2: one thread per (step, operator) plan.
extern "C" __global__ void lg_k_plans(const double* arg, const long long* sp, int count, double tau, double u_prime,
                                      int4* plan_out, int* n_flagged) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  LgPlannerCtx cx{u_prime, 0};
  LgPlan p = lg_make_plan(cx, arg[t], (long)sp[t], tau, 60, 10000);
  if (cx.uncertain) p.status |= LG_PLAN_UNCERTAIN;
  plan_out[t] = make_int4(p.order, p.scaling, p.status, 0);
  if (p.status) atomicAdd(n_flagged, 1);
}

// Gather planner inputs into one [N][1+Kc] array layout.
extern "C" __global__ void lg_k_gather_plan_inputs(const double* norm1, const long long* sp, const double* aux_arg,
                                                   const long long* aux_sp, int N, int Kc, double* arg,
                                                   long long* asp) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N * (Kc + 1)) return;
  int n = t / (Kc + 1), o = t - n * (Kc + 1);
  if (o == 0) {
    arg[t] = norm1[n];
    asp[t] = sp[n];
  } else {
    arg[t] = aux_arg[(long)n * Kc + o - 1];
    asp[t] = aux_sp[(long)n * Kc + o - 1];
  }
}

extern "C" void* lg_prep_sparse_kernel() { return (void*)lg_k_prep_sparse; }
extern "C" void* lg_prep_dense_kernel() { return (void*)lg_k_prep_dense; }
extern "C" void* lg_plans_kernel() { return (void*)lg_k_plans; }

// Per-step Taylor coefficients 1 / (s (j + 1)) of the propagation plans, one row of 64 per step
// (order <= 60), the same IEEE division the chains performed at the start of every step.
extern "C" __global__ void lg_k_rtab(const int4* plan, int Kc, int N, double* rtab) {
  const int n = blockIdx.x, j = threadIdx.x;
  if (n >= N) return;
  const int4 pl = plan[(long)n * (Kc + 1)];
  rtab[(long)n * 64 + j] = j < pl.x ? 1.0 / (double)(pl.y * (j + 1)) : 0.0;
}
extern "C" void* lg_rtab_kernel() { return (void*)lg_k_rtab; }
extern "C" void* lg_gather_kernel() { return (void*)lg_k_gather_plan_inputs; }

// cost and gradient from the raw per-trajectory scalars (lg_final.cuh).  Built here, in the
// -fmad=false unit, so it rounds exactly like the host combine lg_finalize_host.
extern "C" __global__ void lg_k_finalize(const __grid_constant__ LgFinalArgs F) {
  for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < (long)F.N * F.Kc; q += (long)gridDim.x * blockDim.x)
    F.grad[q] = lg_final_grad(F, q);
  if (blockIdx.x == 0 && threadIdx.x == 0) *F.cost = lg_final_cost(F);
}
extern "C" void* lg_finalize_kernel() { return (void*)lg_k_finalize; }
