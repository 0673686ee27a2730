// Single-CTA sweep engine: one CTA owns one trajectory group for the whole
// evaluation (forward and backward sweeps of src/costs.py:269-354, :407-488).
//
// Every Taylor term (src/expm.py:345-350) is one fused step over the chain's
// columns with a FIXED thread <-> (row, column) ownership for the whole chain:
//   * the Taylor accumulator `cur` of each owned (row, column) stays in registers;
//   * narrow operators (ELL width <= WREG) keep the thread's rows of A_n in
//     registers for the whole step; wide ones read A_n from shared memory;
//   * the term vectors live in shared memory (double-buffered) -> ONE
//     __syncthreads per Taylor term and no global traffic inside a chain.
// Thread layout: blockDim = RL row lanes x CS column slots, RL a multiple of 32,
// so every warp belongs to exactly one column slot and column reductions are
// warp-shuffle trees (deterministic, fixed order).
#include "lg_final.cuh"
#include "lg_types.h"

extern __shared__ double2 lg_smem[];

#ifdef LG_DEBUG
#include <cstdio>
__device__ __forceinline__ unsigned lg_dyn_smem() {
  unsigned r;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
  return r;
}
__device__ __forceinline__ double2& lg_smx(double2* sm, long idx, int line) {
  const long n = lg_dyn_smem() / 16;
  if (idx < 0 || idx >= n) {
    printf("LG_DEBUG smem OOB idx=%ld words=%ld line=%d block=%d thread=%d\n", idx, n, line, blockIdx.x, threadIdx.x);
    return sm[0];
  }
  return sm[idx];
}
#define SMX(i) lg_smx(lg_smem, (long)(i), __LINE__)
#else
#define SMX(i) lg_smem[i]
#endif

namespace {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cdot(double2 a, double2 b) {  // conj(a) b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 warp_sum(double2 v) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// Shared-memory layout (offsets in double2 units), filled by init().
struct Lay {
  int red;      // [64] reduction scratch
  int res;      // [64] reduction results
  int rt;       // [64] 1/(s j) table (x component)
  int a;        // A_n [W][d] (smem-A mode)
  int acols;    // int view: A cols [W][d] (smem-A mode)
  int ac;       // A_c [Kc][Wc][d] (if in smem) else -1
  int accols;   // int view
  int state;    // [T(1+I)][d]   psi | lambda
  int next;     // [T(1+I)][d]   adjoint results
  int tb0, tb1; // [Cmax][d]
};

struct Ctx {
  const LgEngineArgs* E;
  int d, T, I, t0, set, trel;
  int rl, cs, lane, slot;
  int W, Wc;
  bool a_smem, ac_smem;
  bool dense;            // dense rows: slot w is column w (no index loads)
  const double2* astep;  // global A_n of the current step (global-A mode)
  int n;                 // current step (DIAGONALIZATION operators)
  Lay L;
};

// WREG > 0: the operator has exactly WREG stored slots per row (ELL width) and
// the thread's rows of A_n live in registers; WREG == 0: A_n read from memory.
template <int MAXR, int MAXC, int WREG>
struct Regs {
  double2 cur[MAXC][MAXR];
  double2 a[MAXR][WREG > 0 ? WREG : 1];
  int col[MAXR][WREG > 0 ? WREG : 1];
  double2 ac[MAXC][MAXR][2];  // control-generator row of a top column (Wc <= 2)
  int accol[MAXC][MAXR][2];
};

__device__ __forceinline__ int row_of(const Ctx& c, int k) { return c.lane + k * c.rl; }

__device__ __forceinline__ void cmac(double2& p, double2& q, double2 a, double2 x) {
  // p accumulates (a.x x.x, a.x x.y), q accumulates (-a.y x.y, a.y x.x): two
  // independent dependency chains per complex product.
  p.x = fma(a.x, x.x, p.x);
  p.y = fma(a.x, x.y, p.y);
  q.x = fma(-a.y, x.y, q.x);
  q.y = fma(a.y, x.x, q.y);
}

// One Taylor chain.  mode 0: column c's input is column c of `xin` (smem
// offset, stride d).  mode 1 (aux embedding): columns [0, G*T) are tops for
// channel gch[c / T] with zero input and bottom partner G*T + c % T; columns
// [G*T, (G+1)*T) are bottoms with input xin[t].  The input is first staged into
// the term buffer so every term reads the same way; everything that does not
// change from term to term (offsets, control rows, 1/(s j)) is hoisted.
// Result: the cur registers of the owned (row, column)s.
// DIAGONALIZATION backend (lg_diag.cu): the chain is one application of the step's exact
// operator -- U_n (sgn > 0), U_n^dagger (sgn < 0), or for the aux tops dU_n/da_k acting on the
// bottom input (src/derivatives.py:249-275).  Same staging and result registers as chain().
template <int MAXR, int MAXC, int WREG>
__device__ __forceinline__ void chain_diag(Ctx& c, double2* sm, Regs<MAXR, MAXC, WREG>& R, int C, int mode,
                                           double sgn, int xin, const int* gch, int G) {
  const LgEngineArgs& E = *c.E;
  const int d = c.d, T = c.T;
  const long dd = (long)d * d;
  const int ntop = mode == 1 ? G * T : 0;
#pragma unroll
  for (int q = 0; q < MAXC; ++q) {
    const int col = c.slot + q * c.cs;
    const bool own = col < C, top = own && col < ntop;
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
      const int i = row_of(c, k);
      double2 v = make_double2(0.0, 0.0);
      if (own && i < d) {
        if (mode == 0)
          v = SMX(xin + col * d + i);
        else if (!top)
          v = SMX(xin + (col - ntop) * d + i);
        SMX(c.L.tb0 + col * d + i) = v;
      }
      R.cur[q][k] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < MAXC; ++q) {
    const int col = c.slot + q * c.cs;
    if (col >= C) continue;
    const bool top = col < ntop;
    if (mode == 1 && !top) continue;  // bottoms: not needed by the derivative
    const double2* op = mode == 0 ? (sgn > 0.0 ? c.astep : E.diag_Ud + (long)c.n * dd)
                                  : E.diag_D + ((long)c.n * E.Kc + gch[col / T]) * dd;
    const int x = c.L.tb0 + (mode == 0 ? col : ntop + col % T) * d;
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
      const int i = row_of(c, k);
      if (i >= d) continue;
      double2 p0 = make_double2(0.0, 0.0), q0 = p0, p1 = p0, q1 = p0;
      int w = 0;
      for (; w + 2 <= d; w += 2) {
        cmac(p0, q0, op[(long)w * d + i], SMX(x + w));
        cmac(p1, q1, op[(long)(w + 1) * d + i], SMX(x + w + 1));
      }
      for (; w < d; ++w) cmac(p0, q0, op[(long)w * d + i], SMX(x + w));
      R.cur[q][k] = make_double2((p0.x + q0.x) + (p1.x + q1.x), (p0.y + q0.y) + (p1.y + q1.y));
    }
  }
  __syncthreads();
}

template <int MAXR, int MAXC, int WREG>
__device__ __forceinline__ void chain(Ctx& c, double2* sm, Regs<MAXR, MAXC, WREG>& R, int C, int mode, int m, int s,
                                      double sgn, int xin, const int* gch, int G) {
  if (c.E->diag) {
    chain_diag<MAXR, MAXC, WREG>(c, sm, R, C, mode, sgn, xin, gch, G);
    return;
  }
  const int d = c.d, T = c.T, Wc = c.Wc, W = c.W;
  const int ntop = mode == 1 ? G * T : 0;
  const int* smi = reinterpret_cast<const int*>(lg_smem);
  const LgEngineArgs& E = *c.E;
  const double2* Acp = c.ac_smem ? lg_smem + c.L.ac : E.Ac;
  const int* Ccp = c.ac_smem ? smi + 4 * c.L.accols : E.Ac_cols;
  const double2* Ap = c.a_smem ? lg_smem + c.L.a : c.astep;
  const int* Cp = c.a_smem ? smi + 4 * c.L.acols : E.A_cols;
  const bool acreg = Wc <= 2;
  int coff[MAXC], poff[MAXC], kbase[MAXC];
  bool own[MAXC], top[MAXC];
#pragma unroll
  for (int q = 0; q < MAXC; ++q) {
    const int col = c.slot + q * c.cs;
    own[q] = col < C;
    top[q] = own[q] && col < ntop;
    coff[q] = col * d;
    const int t = top[q] ? col % T : 0;
    poff[q] = (ntop + t) * d;
    kbase[q] = top[q] ? gch[col / T] * Wc * d : 0;
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
      const int i = row_of(c, k);
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const bool on = top[q] && acreg && i < d && w < Wc;
        R.ac[q][k][w] = on ? Acp[kbase[q] + w * d + i] : make_double2(0.0, 0.0);
        R.accol[q][k][w] = on ? Ccp[kbase[q] + w * d + i] : 0;
      }
    }
  }
  // stage the input into tb0 and the accumulators; 1/(s j) table
#pragma unroll
  for (int q = 0; q < MAXC; ++q) {
    const int col = c.slot + q * c.cs;
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
      const int i = row_of(c, k);
      double2 v = make_double2(0.0, 0.0);
      if (own[q] && i < d) {
        if (mode == 0)
          v = SMX(xin + col * d + i);
        else if (!top[q])
          v = SMX(xin + (col - ntop) * d + i);
        SMX(c.L.tb0 + coff[q] + i) = v;
      }
      R.cur[q][k] = v;
    }
  }
  if (threadIdx.x < m) SMX(c.L.rt + threadIdx.x).x = sgn * (1.0 / (double)(s * (threadIdx.x + 1)));
  __syncthreads();
  int X = c.L.tb0, Y = c.L.tb1;
  const int rt = c.L.rt;
  int rows[MAXR];
#pragma unroll
  for (int k = 0; k < MAXR; ++k) rows[k] = row_of(c, k);
  for (int si = 0; si < s; ++si) {
    for (int j = 1; j <= m; ++j) {
      const double r = SMX(rt + j - 1).x;
      const bool last = j == m;
#pragma unroll
      for (int q = 0; q < MAXC; ++q) {
        if (!own[q]) continue;
        const int xc = X + coff[q];
#pragma unroll
        for (int k = 0; k < MAXR; ++k) {
          const int i = rows[k];
          if (i >= d) continue;
          double2 p = make_double2(0.0, 0.0), pq = make_double2(0.0, 0.0);
          if (WREG > 0) {
#pragma unroll
            for (int w = 0; w < (WREG > 0 ? WREG : 1); ++w) cmac(p, pq, R.a[k][w], SMX(xc + R.col[k][w]));
          } else if (c.dense) {
            // dense rows: x[w] is a broadcast read, four independent accumulator pairs
            double2 p1 = make_double2(0.0, 0.0), q1 = p1, p2 = p1, q2 = p1, p3 = p1, q3 = p1;
            int w = 0;
            for (; w + 4 <= W; w += 4) {
              cmac(p, pq, Ap[w * d + i], SMX(xc + w));
              cmac(p1, q1, Ap[(w + 1) * d + i], SMX(xc + w + 1));
              cmac(p2, q2, Ap[(w + 2) * d + i], SMX(xc + w + 2));
              cmac(p3, q3, Ap[(w + 3) * d + i], SMX(xc + w + 3));
            }
            for (; w < W; ++w) cmac(p, pq, Ap[w * d + i], SMX(xc + w));
            p = cadd(cadd(p, p1), cadd(p2, p3));
            pq = cadd(cadd(pq, q1), cadd(q2, q3));
          } else {
            for (int w = 0; w < W; ++w) {
              const int q2 = w * d + i;
              cmac(p, pq, Ap[q2], SMX(xc + Cp[q2]));
            }
          }
          if (top[q]) {
            const int bc = X + poff[q];
            if (acreg) {
              cmac(p, pq, R.ac[q][k][0], SMX(bc + R.accol[q][k][0]));
              cmac(p, pq, R.ac[q][k][1], SMX(bc + R.accol[q][k][1]));
            } else if (c.dense) {
              const int base = kbase[q] + i;
              double2 p1 = make_double2(0.0, 0.0), q1 = p1;
              int w = 0;
              for (; w + 2 <= Wc; w += 2) {
                cmac(p, pq, Acp[base + w * d], SMX(bc + w));
                cmac(p1, q1, Acp[base + (w + 1) * d], SMX(bc + w + 1));
              }
              for (; w < Wc; ++w) cmac(p, pq, Acp[base + w * d], SMX(bc + w));
              p = cadd(p, p1);
              pq = cadd(pq, q1);
            } else {
              const int base = kbase[q] + i;
              for (int w = 0; w < Wc; ++w) cmac(p, pq, Acp[base + w * d], SMX(bc + Ccp[base + w * d]));
            }
          }
          const double2 tt = make_double2((p.x + pq.x) * r, (p.y + pq.y) * r);
          R.cur[q][k] = cadd(R.cur[q][k], tt);
          SMX(Y + coff[q] + i) = last ? R.cur[q][k] : tt;
        }
      }
      __syncthreads();
      const int t_ = X;
      X = Y;
      Y = t_;
    }
  }
}

// Block reduction of per-thread values v[q] for "virtual columns" vc = map(q):
// each warp belongs to one column slot; lanes are rows.  out[vc] in smem res.
__device__ __forceinline__ void red_put(const Ctx& c, double2* sm, int vc, double2 v) {
  v = warp_sum(v);
  const int wpc = c.rl / 32;
  if ((threadIdx.x & 31) == 0) SMX(c.L.red + vc * wpc + (c.lane >> 5)) = v;
}
__device__ __forceinline__ void red_finish(const Ctx& c, double2* sm, int nvc) {
  __syncthreads();
  const int wpc = c.rl / 32;
  for (int vc = threadIdx.x; vc < nvc; vc += blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (int q = 0; q < wpc; ++q) s = cadd(s, SMX(c.L.red + vc * wpc + q));
    SMX(c.L.res + vc) = s;
  }
  __syncthreads();
}

__device__ __forceinline__ double2 pen_apply(const LgSpecDev& sp, int d, double2* sm, int psi, int i) {
  double2 acc = make_double2(0.0, 0.0);
  for (int w = 0; w < sp.pen_W; ++w) {
    const long q = (long)w * d + i;
    const double2 x = SMX(psi + sp.pen_cols[q]);
    const double2 a = sp.pen_vals[q];
    acc.x = fma(a.x, x.x, acc.x);
    acc.x = fma(-a.y, x.y, acc.x);
    acc.y = fma(a.x, x.y, acc.y);
    acc.y = fma(a.y, x.x, acc.y);
  }
  return acc;
}

template <int MAXR, int MAXC, int WREG>
__device__ void load_step(Ctx& c, double2* sm, Regs<MAXR, MAXC, WREG>& R, int n) {
  const LgEngineArgs& E = *c.E;
  const int d = c.d, W = c.W;
  const double2* src = E.A + (long)n * W * d;
  c.astep = src;
  c.n = n;
  if (WREG > 0) {
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
      const int i = row_of(c, k);
#pragma unroll
      for (int w = 0; w < (WREG > 0 ? WREG : 1); ++w) {
        double2 a = make_double2(0.0, 0.0);
        int cc = 0;
        if (i < d) {
          a = src[(long)w * d + i];
          cc = E.A_cols[w * d + i];
        }
        R.a[k][w] = a;
        R.col[k][w] = cc;
      }
    }
  } else if (c.a_smem) {
    __syncthreads();
    for (int q = threadIdx.x; q < W * d; q += blockDim.x) SMX(c.L.a + q) = src[q];
    __syncthreads();
  }
}

template <int MAXR, int MAXC, int WREG>
__device__ void init(Ctx& c, double2* sm, const LgEngineArgs& E) {
  c.E = &E;
  c.d = E.d;
  const int g = blockIdx.x;
  c.set = E.grp_set[g];
  c.t0 = E.grp_t0[g];
  c.T = E.grp_nT[g];
  c.I = E.set_nspec[c.set];
  c.trel = c.t0 - E.set_t0[c.set];
  c.rl = E.row_lanes;
  c.cs = blockDim.x / c.rl;
  c.lane = threadIdx.x % c.rl;
  c.slot = threadIdx.x / c.rl;
  c.W = E.W;
  c.Wc = E.Wc;
  c.a_smem = (E.smem_mode & 4) != 0;
  c.ac_smem = (E.smem_mode & 8) != 0;
  c.dense = E.dense_rows != 0;
  const int d = E.d, Tg = E.grp_T;
  const int cstate = Tg * (1 + E.cta_Imax), cx = (E.Kc + 1) * Tg, cmax = cstate > cx ? cstate : cx;
  int o = 0;
  c.L.red = o;
  o += E.red_cap * (c.rl / 32);
  c.L.res = o;
  o += E.red_cap;
  c.L.rt = o;
  o += 64;
  c.L.a = o;
  c.L.acols = o + E.W * d;  // int view: offset in double2 * 2 -> handled by 2* in use
  if (c.a_smem) o += E.W * d + (E.W * d + 1) / 2;
  c.L.ac = o;
  c.L.accols = o + E.Kc * E.Wc * d;
  if (c.ac_smem) o += E.Kc * E.Wc * d + (E.Kc * E.Wc * d + 1) / 2;
  c.L.state = o;
  o += cstate * d;
  c.L.next = o;
  o += cstate * d;
  c.L.tb0 = o;
  o += cmax * d;
  c.L.tb1 = o;
  // int views: a double2 offset o is int offset 4 o
  int* smi = reinterpret_cast<int*>(lg_smem);
  if (c.a_smem) {
    for (int q = threadIdx.x; q < E.W * d; q += blockDim.x) smi[4 * c.L.acols + q] = E.A_cols[q];
  }
  if (c.ac_smem) {
    for (int q = threadIdx.x; q < E.Kc * E.Wc * d; q += blockDim.x) {
      SMX(c.L.ac + q) = E.Ac[q];
      smi[4 * c.L.accols + q] = E.Ac_cols[q];
    }
  }
  (void)Tg;
}

}  // namespace

// ------------------------------------------------------------------------------------------- forward
template <int MAXR, int MAXC, int WREG>
__global__ void __launch_bounds__(MAXR == 1 ? 512 : 1024, 1) lg_k_cta_forward(const __grid_constant__ LgEngineArgs E) {
  double2* sm = lg_smem;
  Ctx c;
  init<MAXR, MAXC, WREG>(c, sm, E);
  Regs<MAXR, MAXC, WREG> R;
  const int d = c.d, T = c.T;
  const int psi = c.L.state;
  for (int q = threadIdx.x; q < T * d; q += blockDim.x) SMX(psi + q) = E.psi0[(long)c.t0 * d + q];
  __syncthreads();
  int qspec[LG_MAX_SPECS];
  for (int n = 0; n < E.N; ++n) {
    const int4 pl = E.plan[(long)n * (E.Kc + 1)];
    load_step<MAXR, MAXC, WREG>(c, sm, R, n);
    chain<MAXR, MAXC, WREG>(c, sm, R, T, 0, pl.x, pl.y, 1.0, psi, nullptr, 0);
    // write back psi_n
#pragma unroll
    for (int q = 0; q < MAXC; ++q) {
      const int col = c.slot + q * c.cs;
#pragma unroll
      for (int k = 0; k < MAXR; ++k) {
        const int i = row_of(c, k);
        if (col < T && i < d) SMX(psi + col * d + i) = R.cur[q][k];
      }
    }
    __syncthreads();
    const bool final_step = n == E.N - 1;
    int nq = 0;
    for (int si = 0; si < c.I; ++si) {
      const int sidx = E.set_spec[c.set][si];
      const int kind = E.spec[sidx].kind;
      if (kind == LGK_STATE_PEN || kind == LGK_STATE_RUN || kind == LGK_GATE_RUN ||
          (final_step && (kind == LGK_STATE_INF || kind == LGK_GATE)))
        qspec[nq++] = sidx;
    }
    if (nq == 0) continue;
    // per-step scalars: virtual column vc = q * T + t handled by slot (vc % cs)
    const int nvc = nq * T;
    for (int vc0 = 0; vc0 < nvc; vc0 += c.cs) {
      const int vc = vc0 + c.slot;
      double2 v = make_double2(0.0, 0.0);
      if (vc < nvc) {
        const int q = vc / T, t = vc - q * T;
        const LgSpecDev& sp = E.spec[qspec[q]];
        for (int i = c.lane; i < d; i += c.rl) {
          const double2 pv = SMX(psi + t * d + i);
          if (sp.kind == LGK_STATE_PEN) {
            v = cadd(v, cdot(pv, pen_apply(sp, d, sm, psi + t * d, i)));
          } else {
            const double2 tv = sp.tgt[(long)(c.trel + t) * d + i];
            v = cadd(v, sp.kind == LGK_STATE_INF ? cdot(pv, tv) : cdot(tv, pv));
          }
        }
      }
      if (vc0 + c.slot < nvc) red_put(c, sm, vc, v);
    }
    red_finish(c, sm, nvc);
    if (threadIdx.x == 0) {
      for (int q = 0; q < nq; ++q) {
        const int sidx = qspec[q];
        const int kind = E.spec[sidx].kind;
        for (int t = 0; t < T; ++t) {
          const double2 r = SMX(c.L.res + q * T + t);
          const long o = (long)sidx * E.T_total + c.t0 + t;
          if (kind == LGK_STATE_PEN) {
            E.run[o] += r.x;
          } else if (kind == LGK_STATE_RUN) {
            const double a = hypot(r.x, r.y);
            E.run[o] += a * a;
          } else if (kind == LGK_GATE_RUN) {
            E.trp[((long)sidx * E.N + n) * E.T_total + c.t0 + t] = r;
          } else {
            E.fin[o] = r;
          }
        }
      }
    }
    __syncthreads();
  }
  for (int q = threadIdx.x; q < T * d; q += blockDim.x) E.psiN[(long)c.t0 * d + q] = SMX(psi + q);
}

// ------------------------------------------------------------------------------------------- backward
template <int MAXR, int MAXC, int WREG>
__global__ void __launch_bounds__(MAXR == 1 ? 512 : 1024, 1) lg_k_cta_backward(const __grid_constant__ LgEngineArgs E) {
  double2* sm = lg_smem;
  Ctx c;
  init<MAXR, MAXC, WREG>(c, sm, E);
  Regs<MAXR, MAXC, WREG> R;
  const int d = c.d, T = c.T, I = c.I, Kc = E.Kc, N = E.N;
  const int st = c.L.state, nx = c.L.next;
  auto lam = [&](int si, int t) { return T + si * T + t; };  // column index in state/next
  for (int q = threadIdx.x; q < T * d; q += blockDim.x) SMX(st + q) = E.psiN[(long)c.t0 * d + q];
  __syncthreads();
  // ---- costate initialisation (src/costs.py:312-321, :457-460)
  {
    const int nvc = I * T;
    for (int vc0 = 0; vc0 < nvc; vc0 += c.cs) {
      const int vc = vc0 + c.slot;
      double2 v = make_double2(0.0, 0.0);
      if (vc < nvc) {
        const int si = vc / T, t = vc - si * T;
        const LgSpecDev& sp = E.spec[E.set_spec[c.set][si]];
        if (sp.kind == LGK_STATE_RUN)
          for (int i = c.lane; i < d; i += c.rl) v = cadd(v, cdot(sp.tgt[(long)(c.trel + t) * d + i], SMX(st + t * d + i)));
        red_put(c, sm, vc, v);
      }
    }
    red_finish(c, sm, nvc);
    for (int si = 0; si < I; ++si) {
      const int sidx = E.set_spec[c.set][si];
      const LgSpecDev& sp = E.spec[sidx];
      const double2 trN = sp.kind == LGK_GATE_RUN ? E.trsum[(long)sidx * N + N - 1] : make_double2(0.0, 0.0);
      for (int t = 0; t < T; ++t) {
        const double2 ov = SMX(c.L.res + si * T + t);
        for (int i = threadIdx.x; i < d; i += blockDim.x) {
          double2 v;
          if (sp.kind == LGK_STATE_PEN) {
            v = pen_apply(sp, d, sm, st + t * d, i);
          } else {
            const double2 tv = sp.tgt[(long)(c.trel + t) * d + i];
            v = sp.kind == LGK_STATE_RUN ? cmul(tv, ov) : (sp.kind == LGK_GATE_RUN ? cmul(tv, trN) : tv);
          }
          SMX(st + lam(si, t) * d + i) = v;
        }
      }
    }
    __syncthreads();
  }
  int gch[LG_MAX_CHANNELS];
  for (int n = N - 1; n >= 0; --n) {
    const int4* pln = E.plan + (long)n * (Kc + 1);
    const int4 pl = pln[0];
    load_step<MAXR, MAXC, WREG>(c, sm, R, n);
    // adjoint chain on [psi | lambda] (src/costs.py:326,342); costates unused at n == 0
    const int cadj = n > 0 ? T * (1 + I) : T;
    chain<MAXR, MAXC, WREG>(c, sm, R, cadj, 0, pl.x, pl.y, -1.0, st, nullptr, 0);
#pragma unroll
    for (int q = 0; q < MAXC; ++q) {
      const int col = c.slot + q * c.cs;
#pragma unroll
      for (int k = 0; k < MAXR; ++k) {
        const int i = row_of(c, k);
        if (col < cadj && i < d) SMX(nx + col * d + i) = R.cur[q][k];
      }
    }
    __syncthreads();
    // derivative products, channels grouped by identical aux plan (src/costs.py:328-339)
    unsigned done = 0;
    for (int kc = 0; kc < Kc; ++kc) {
      if (done & (1u << kc)) continue;
      const int4 pk = pln[1 + kc];
      int G = 0;
      for (int k2 = kc; k2 < Kc; ++k2) {
        const int4 p2 = pln[1 + k2];
        if (!(done & (1u << k2)) && p2.x == pk.x && p2.y == pk.y) {
          gch[G++] = k2;
          done |= 1u << k2;
        }
      }
      const int caux = (G + 1) * T;
      chain<MAXR, MAXC, WREG>(c, sm, R, caux, 1, pk.x, pk.y, 1.0, nx, gch, G);
      // <lambda_(si,t) | D_(k,t)>: the owner of top column (g, t) holds D in registers
      const int ntop = G * T;
      for (int si = 0; si < I; ++si) {
#pragma unroll
        for (int q = 0; q < MAXC; ++q) {
          const int col = c.slot + q * c.cs;
          if (col >= ntop) continue;
          const int t = col % T;
          double2 v = make_double2(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < MAXR; ++k) {
            const int i = row_of(c, k);
            if (i < d) v = cadd(v, cdot(SMX(st + lam(si, t) * d + i), R.cur[q][k]));
          }
          red_put(c, sm, si * ntop + col, v);
        }
      }
      red_finish(c, sm, I * ntop);
      if (threadIdx.x < I * ntop) {
        const int vc = threadIdx.x;
        const int si = vc / ntop, col = vc - si * ntop;
        const int t = col % T, gi = col / T;
        const int sidx = E.set_spec[c.set][si];
        E.ip[(((long)n * E.n_specs + sidx) * Kc + gch[gi]) * E.T_total + c.t0 + t] = SMX(c.L.res + vc);
      }
      __syncthreads();
    }
    if (n == 0) break;
    // costate sources at psi_{n-1} (src/costs.py:341-353, :474-479)
    {
      const int nvc = I * T;
      bool any_run = false;
      for (int si = 0; si < I; ++si) any_run |= E.spec[E.set_spec[c.set][si]].kind == LGK_STATE_RUN;
      if (any_run) {
        for (int vc0 = 0; vc0 < nvc; vc0 += c.cs) {
          const int vc = vc0 + c.slot;
          double2 v = make_double2(0.0, 0.0);
          if (vc < nvc) {
            const int si = vc / T, t = vc - si * T;
            const LgSpecDev& sp = E.spec[E.set_spec[c.set][si]];
            if (sp.kind == LGK_STATE_RUN)
              for (int i = c.lane; i < d; i += c.rl)
                v = cadd(v, cdot(sp.tgt[(long)(c.trel + t) * d + i], SMX(nx + t * d + i)));
            red_put(c, sm, vc, v);
          }
        }
        red_finish(c, sm, nvc);
      }
      for (int si = 0; si < I; ++si) {
        const int sidx = E.set_spec[c.set][si];
        const LgSpecDev& sp = E.spec[sidx];
        const double2 tr = sp.kind == LGK_GATE_RUN ? E.trsum[(long)sidx * N + n - 1] : make_double2(0.0, 0.0);
        for (int t = 0; t < T; ++t) {
          const double2 ov = any_run ? SMX(c.L.res + si * T + t) : make_double2(0.0, 0.0);
          const int col = lam(si, t);
          for (int i = threadIdx.x; i < d; i += blockDim.x) {
            double2 v = SMX(nx + col * d + i);
            if (sp.kind == LGK_STATE_PEN)
              v = cadd(v, pen_apply(sp, d, sm, nx + t * d, i));
            else if (sp.kind == LGK_STATE_RUN)
              v = cadd(v, cmul(sp.tgt[(long)(c.trel + t) * d + i], ov));
            else if (sp.kind == LGK_GATE_RUN)
              v = cadd(v, cmul(sp.tgt[(long)(c.trel + t) * d + i], tr));
            SMX(st + col * d + i) = v;
          }
        }
      }
      for (int q = threadIdx.x; q < T * d; q += blockDim.x) SMX(st + q) = SMX(nx + q);
      __syncthreads();
    }
  }
}

#define LG_CTA_W(X, R_, C_) X(R_, C_, 1) X(R_, C_, 2) X(R_, C_, 3) X(R_, C_, 4) X(R_, C_, 5) X(R_, C_, 6) X(R_, C_, 7) X(R_, C_, 8) X(R_, C_, 9)
#define LG_CTA_VARIANTS(X) LG_CTA_W(X, 1, 1) LG_CTA_W(X, 1, 2) LG_CTA_W(X, 2, 1) \
  X(1, 1, 0) X(1, 2, 0) X(2, 1, 0) X(4, 1, 0) X(2, 2, 0) X(1, 4, 0)

extern "C" void* lg_cta_kernel(int backward, int maxr, int maxc, int wreg) {
#define LG_PICK(R_, C_, W_)                                                                        \
  if (maxr == R_ && maxc == C_ && wreg == W_)                                                      \
    return backward ? (void*)lg_k_cta_backward<R_, C_, W_> : (void*)lg_k_cta_forward<R_, C_, W_>;
  LG_CTA_VARIANTS(LG_PICK)
#undef LG_PICK
  return nullptr;
}
