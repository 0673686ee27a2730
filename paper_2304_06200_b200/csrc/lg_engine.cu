// Sweep engine: the forward and backward sweeps of one HG evaluation as two
// persistent kernels (src/costs.py:269-354 state pass, :407-488 gate pass).
//
// Work decomposition.  The K trajectories (initial states of the state terms,
// or gate basis states) are split into groups; a group is owned by one CTA
// (n_slabs == 1: everything synchronises with __syncthreads and lives in
// shared memory when it fits) or by n_slabs co-resident CTAs that split the
// rows (grid-group barrier, state in L2-resident global memory).  Inside a
// group every Taylor term is ONE fused SpMM over all the group's columns:
//
//   forward   [psi_t]                          (A_n,  plan_n)
//   adjoint   [psi_t | lambda_(spec,t)]         (-A_n, plan_n)    psi and all costates batched
//   aux       [top_(k,t) | bottom_t]            (aux embedding of every channel k that shares
//                                               the same aux plan; bottom shared by those channels)
//
// fused with the Taylor scale-and-accumulate  term <- (A term)(1/(s j)); cur += term
// (src/expm.py:345-350).  Reductions (overlaps, penalty expectations, traces,
// <lambda|dU/da psi>) are deterministic fixed-order warp-shuffle trees.
//
// Outputs are raw per-trajectory complex scalars; lg_k_finalize turns them into
// cost and gradient with the reference's formulas.
#include "lg_types.h"
#include "lg_final.cuh"

namespace {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
__device__ __forceinline__ double2 cdot(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 cscale(double2 a, double r) { return make_double2(a.x * r, a.y * r); }
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 x) {
  acc.x = fma(a.x, x.x, acc.x);
  acc.x = fma(-a.y, x.y, acc.x);
  acc.y = fma(a.x, x.y, acc.y);
  acc.y = fma(a.y, x.x, acc.y);
}

template <bool M>
__device__ __forceinline__ double2 ld(const double2* p) {
  if (M) return __ldcg(p);
  return *p;
}

__device__ __forceinline__ double2 warp_sum(double2 v) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

struct Cx {
  int d, r0, r1;
  int g, slab, nslabs;
  unsigned* bar;
  double2* red;  // [2][cap][nslabs]
  int cap, par;
  double2* smred;  // shared scratch [cap]
  double2* smres;  // shared results [cap]
  bool writer;     // this CTA publishes group results
};

template <bool M>
__device__ void bar_sync(Cx& cx) {
  __syncthreads();
  if (!M) return;
  if (threadIdx.x == 0) {
    volatile unsigned* gen = cx.bar + 1;
    unsigned g0 = *gen;
    __threadfence();
    unsigned arrived = atomicAdd(cx.bar, 1u);
    if (arrived == (unsigned)cx.nslabs - 1) {
      atomicExch(cx.bar, 0u);
      __threadfence();
      atomicAdd((unsigned*)(cx.bar + 1), 1u);
    } else {
      while (*gen == g0) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// Column mapping of C columns over the slab rows: warps_per_col warps per
// column (or one warp looping over several columns when C > warps).
struct Map {
  int wpc, cslots, c0, lr, rs;
  __device__ Map(int C) {
    const int nw = blockDim.x >> 5, w = threadIdx.x >> 5, l = threadIdx.x & 31;
    wpc = nw / C;
    if (wpc < 1) wpc = 1;
    cslots = nw / wpc;
    c0 = w / wpc;
    lr = (w % wpc) * 32 + l;
    rs = 32 * wpc;
  }
};

// Deterministic sum over the group's rows of f(vc, i) for vc in [0, Cv);
// result in cx.smres[vc] for every thread of every CTA of the group.
template <bool M, class F>
__device__ void colsum(Cx& cx, int Cv, const F& f) {
  Map mp(Cv);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int c = mp.c0; c < Cv; c += mp.cslots) {
    double2 v = make_double2(0.0, 0.0);
    for (int i = cx.r0 + mp.lr; i < cx.r1; i += mp.rs) v = cadd(v, f(c, i));
    v = warp_sum(v);
    if (l == 0) cx.smred[c * mp.wpc + (w % mp.wpc)] = v;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < Cv; c += blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (int q = 0; q < mp.wpc; ++q) s = cadd(s, cx.smred[c * mp.wpc + q]);
    if (M)
      cx.red[((long)cx.par * cx.cap + c) * cx.nslabs + cx.slab] = s;
    else
      cx.smres[c] = s;
  }
  if (M) {
    bar_sync<M>(cx);
    for (int c = threadIdx.x; c < Cv; c += blockDim.x) {
      double2 s = make_double2(0.0, 0.0);
      const double2* p = cx.red + ((long)cx.par * cx.cap + c) * cx.nslabs;
      for (int q = 0; q < cx.nslabs; ++q) s = cadd(s, __ldcg(p + q));
      cx.smres[c] = s;
    }
    cx.par ^= 1;
  }
  __syncthreads();
}

// Operator views for one step.
struct Ops {
  int d, W, Wc;
  const int* cols;      // [W][d]
  const double2* A;     // [W][d]
  const int* ccols;     // [Kc][Wc][d]
  const double2* Ac;    // [Kc][Wc][d]
};

// One Taylor chain: cur <- (T_m(sgn A / s))^s x_in, over C columns.
// mode 0: column c input is xin[c].  mode 1 (aux embedding): columns
// [0, G*Tg) are tops (zero input; channel gch[c / Tg], bottom partner
// G*Tg + c % Tg) and [G*Tg, (G+1)*Tg) are bottoms with input xin[t].
template <bool M>
__device__ void chain(Cx& cx, const Ops& op, int C, int mode, int m, int s, double sgn, const double2* xin,
                      double2* cur, double2* tb0, double2* tb1, const int* gch, int G, int Tg) {
  const int d = op.d;
  Map mp(C);
  const double2* X = xin;
  double2* Y = tb0;
  double2* Yn = tb1;
  bool first = true;
  const int ntop = (mode == 1) ? G * Tg : 0;
  for (int si = 0; si < s; ++si) {
    for (int j = 1; j <= m; ++j) {
      const double r = sgn * (1.0 / (double)(s * j));
      const bool last = (j == m);
      for (int c = mp.c0; c < C; c += mp.cslots) {
        const bool top = c < ntop;
        const double2* xc;
        if (first && mode == 1)
          xc = top ? nullptr : xin + (long)(c - ntop) * d;
        else
          xc = X + (long)c * d;
        const double2* bc = nullptr;
        const int* kcols = nullptr;
        const double2* kvals = nullptr;
        if (top) {
          const int t = c % Tg, k = gch[c / Tg];
          bc = (first ? xin + (long)t * d : X + (long)(ntop + t) * d);
          kcols = op.ccols + (long)k * op.Wc * d;
          kvals = op.Ac + (long)k * op.Wc * d;
        }
        for (int i = cx.r0 + mp.lr; i < cx.r1; i += mp.rs) {
          double2 acc = make_double2(0.0, 0.0);
          if (xc) {
#pragma unroll 4
            for (int w = 0; w < op.W; ++w) {
              const long q = (long)w * d + i;
              cfma(acc, op.A[q], ld<M>(xc + op.cols[q]));
            }
          }
          if (top) {
            double2 acc2 = make_double2(0.0, 0.0);
            for (int w = 0; w < op.Wc; ++w) {
              const long q = (long)w * d + i;
              cfma(acc2, kvals[q], ld<M>(bc + kcols[q]));
            }
            acc = cadd(acc, acc2);
          }
          const double2 tt = cscale(acc, r);
          double2 base;
          if (first)
            base = top ? make_double2(0.0, 0.0) : ld<M>(xc + i);
          else
            base = cur[(long)c * d + i];
          const double2 cu = cadd(base, tt);
          cur[(long)c * d + i] = cu;
          Y[(long)c * d + i] = last ? cu : tt;
        }
      }
      bar_sync<M>(cx);
      X = Y;
      double2* t = Y;
      Y = Yn;
      Yn = t;
      first = false;
    }
  }
}

template <bool M>
__device__ __forceinline__ double2 penalty_apply(const LgSpecDev& sp, int d, const double2* psi, int i) {
  double2 acc = make_double2(0.0, 0.0);
  for (int w = 0; w < sp.pen_W; ++w) {
    const long q = (long)w * d + i;
    cfma(acc, sp.pen_vals[q], ld<M>(psi + sp.pen_cols[q]));
  }
  return acc;
}

struct Bufs {
  double2 *state, *cura, *curx, *tb0, *tb1;
};


}  // namespace

// ------------------------------------------------------------------------------------------
namespace {

struct KernelCtx {
  Cx cx;
  Bufs b;
  int Tg, t0, set, I;
  Ops op;
};

template <bool M>
__device__ void init_ctx(const LgEngineArgs& E, KernelCtx& k, double2* smem) {
  Cx& cx = k.cx;
  cx.d = E.d;
  cx.nslabs = E.n_slabs;
  cx.g = blockIdx.x / E.n_slabs;
  cx.slab = blockIdx.x % E.n_slabs;
  const int rows = (E.d + E.n_slabs - 1) / E.n_slabs;
  cx.r0 = cx.slab * rows;
  cx.r1 = min(E.d, cx.r0 + rows);
  cx.bar = E.bar + 4 * cx.g;
  cx.cap = E.red_cap;
  cx.red = E.red + (long)cx.g * 2 * E.red_cap * E.n_slabs;
  cx.par = 0;
  cx.smred = smem;
  cx.smres = smem + E.red_cap;
  cx.writer = (cx.slab == 0);
  k.set = E.grp_set[cx.g];
  k.t0 = E.grp_t0[cx.g];
  k.Tg = E.grp_nT[cx.g];
  k.I = E.set_nspec[k.set];
  const int Tg = k.Tg;
  const long d = E.d;
  const int I = k.I;
  const long cstate = (long)Tg * (1 + I), cx_cols = (long)(E.Kc + 1) * Tg;
  const long cmax = cstate > cx_cols ? cstate : cx_cols;
  double2* g = E.scratch + (long)cx.g * E.scratch_per_group;
  double2* s = smem + 2 * E.red_cap;
  if (E.smem_mode & 4) s += (long)E.W * d;  // A_n copy
  if (E.smem_mode & 1) {
    k.b.state = s;
    k.b.cura = s + cstate * d;
    k.b.curx = s + 2 * cstate * d;
    k.b.tb0 = s + (2 * cstate + cx_cols) * d;
    k.b.tb1 = k.b.tb0 + cmax * d;
  } else {
    k.b.state = g;
    k.b.cura = g + cstate * d;
    k.b.curx = g + 2 * cstate * d;
    if (E.smem_mode & 2) {
      k.b.tb0 = s;
      k.b.tb1 = s + cmax * d;
    } else {
      k.b.tb0 = g + (2 * cstate + cx_cols) * d;
      k.b.tb1 = k.b.tb0 + cmax * d;
    }
  }
  k.op.d = E.d;
  k.op.W = E.W;
  k.op.Wc = E.Wc;
  k.op.cols = E.A_cols;
  k.op.ccols = E.Ac_cols;
  k.op.Ac = E.Ac;
}

template <bool M>
__device__ void load_step_op(const LgEngineArgs& E, KernelCtx& k, double2* smem, int n) {
  const double2* src = E.A + (long)n * E.W * E.d;
  if (E.smem_mode & 4) {
    double2* dst = smem + 2 * E.red_cap;
    __syncthreads();
    const long tot = (long)E.W * E.d;
    for (long q = threadIdx.x; q < tot; q += blockDim.x) dst[q] = src[q];
    __syncthreads();
    k.op.A = dst;
  } else {
    k.op.A = src;
  }
}

}  // namespace

template <bool M>
__global__ void __launch_bounds__(1024, 1) lg_k_forward(const __grid_constant__ LgEngineArgs E) {
  extern __shared__ double2 smem[];
  KernelCtx k;
  init_ctx<M>(E, k, smem);
  Cx& cx = k.cx;
  const int d = E.d, Tg = k.Tg, t0 = k.t0, set = k.set;
  double2* psi = k.b.state;
  double2* cura = k.b.cura;
  for (int t = 0; t < Tg; ++t)
    for (int i = cx.r0 + threadIdx.x; i < cx.r1; i += blockDim.x) psi[(long)t * d + i] = E.psi0[(long)(t0 + t) * d + i];
  bar_sync<M>(cx);

  // per-step scalar quantities of this set's specs
  const int I = k.I;
  for (int n = 0; n < E.N; ++n) {
    const int4 pl = E.plan[(long)n * (E.Kc + 1)];
    load_step_op<M>(E, k, smem, n);
    chain<M>(cx, k.op, Tg, 0, pl.x, pl.y, 1.0, psi, cura, k.b.tb0, k.b.tb1, nullptr, 0, Tg);
    double2* t_ = psi;
    psi = cura;
    cura = t_;
    const bool final_step = (n == E.N - 1);
    // quantity list: q -> spec slot
    int qspec[LG_MAX_SPECS];
    int nq = 0;
    for (int si = 0; si < I; ++si) {
      const int sidx = E.set_spec[set][si];
      const int kind = E.spec[sidx].kind;
      if (kind == LGK_STATE_PEN || kind == LGK_STATE_RUN || kind == LGK_GATE_RUN ||
          (final_step && (kind == LGK_STATE_INF || kind == LGK_GATE)))
        qspec[nq++] = sidx;
    }
    if (nq == 0) continue;
    const double2* psic = psi;
    colsum<M>(cx, nq * Tg, [&](int vc, int i) {
      const int q = vc / Tg, t = vc - q * Tg;
      const LgSpecDev& sp = E.spec[qspec[q]];
      const double2* p = psic + (long)t * d;
      const double2 pv = ld<M>(p + i);
      if (sp.kind == LGK_STATE_PEN) return cdot(pv, penalty_apply<M>(sp, d, p, i));
      const double2 tv = sp.tgt[(long)(t0 - E.set_t0[set] + t) * d + i];
      if (sp.kind == LGK_STATE_INF) return cdot(pv, tv);
      return cdot(tv, pv);
    });
    if (cx.writer && threadIdx.x == 0) {
      for (int q = 0; q < nq; ++q) {
        const int sidx = qspec[q];
        const int kind = E.spec[sidx].kind;
        for (int t = 0; t < Tg; ++t) {
          const double2 r = cx.smres[q * Tg + t];
          const long o = (long)sidx * E.T_total + t0 + t;
          if (kind == LGK_STATE_PEN) {
            E.run[o] += r.x;
          } else if (kind == LGK_STATE_RUN) {
            const double a = hypot(r.x, r.y);
            E.run[o] += a * a;
          } else if (kind == LGK_GATE_RUN) {
            E.trp[((long)sidx * E.N + n) * E.T_total + t0 + t] = r;
            if (final_step) E.fin[o] = r;
          } else {
            E.fin[o] = r;
          }
        }
      }
    }
    __syncthreads();
  }
  for (int t = 0; t < Tg; ++t)
    for (int i = cx.r0 + threadIdx.x; i < cx.r1; i += blockDim.x) E.psiN[(long)(t0 + t) * d + i] = psi[(long)t * d + i];
}

template <bool M>
__global__ void __launch_bounds__(1024, 1) lg_k_backward(const __grid_constant__ LgEngineArgs E) {
  extern __shared__ double2 smem[];
  KernelCtx k;
  init_ctx<M>(E, k, smem);
  Cx& cx = k.cx;
  const int d = E.d, Tg = k.Tg, t0 = k.t0, set = k.set, I = k.I, Kc = E.Kc, N = E.N;
  double2* st = k.b.state;
  double2* cura = k.b.cura;
  double2* curx = k.b.curx;
  auto lam_col = [&](int si, int t) { return Tg + si * Tg + t; };
  const int trel = t0 - E.set_t0[set];

  for (int t = 0; t < Tg; ++t)
    for (int i = cx.r0 + threadIdx.x; i < cx.r1; i += blockDim.x) st[(long)t * d + i] = E.psiN[(long)(t0 + t) * d + i];
  bar_sync<M>(cx);
  // ---- costate initialisation (src/costs.py:312-321, :457-460)
  {
    colsum<M>(cx, I * Tg, [&](int vc, int i) {
      const int si = vc / Tg, t = vc - si * Tg;
      const LgSpecDev& sp = E.spec[E.set_spec[set][si]];
      if (sp.kind != LGK_STATE_RUN) return make_double2(0.0, 0.0);
      return cdot(sp.tgt[(long)(trel + t) * d + i], ld<M>(st + (long)t * d + i));
    });
    for (int si = 0; si < I; ++si) {
      const int sidx = E.set_spec[set][si];
      const LgSpecDev& sp = E.spec[sidx];
      for (int t = 0; t < Tg; ++t) {
        const double2 ov = cx.smres[si * Tg + t];
        const double2 trN = (sp.kind == LGK_GATE_RUN) ? E.trsum[(long)sidx * N + N - 1] : make_double2(0.0, 0.0);
        double2* lam = st + (long)lam_col(si, t) * d;
        for (int i = cx.r0 + threadIdx.x; i < cx.r1; i += blockDim.x) {
          double2 v;
          if (sp.kind == LGK_STATE_PEN) {
            v = penalty_apply<M>(sp, d, st + (long)t * d, i);
          } else {
            const double2 tv = sp.tgt[(long)(trel + t) * d + i];
            if (sp.kind == LGK_STATE_RUN)
              v = cmul(tv, ov);
            else if (sp.kind == LGK_GATE_RUN)
              v = cmul(tv, trN);
            else
              v = tv;
          }
          lam[i] = v;
        }
      }
    }
  }
  bar_sync<M>(cx);

  int gch[LG_MAX_CHANNELS];
  for (int n = N - 1; n >= 0; --n) {
    const int4* pln = E.plan + (long)n * (Kc + 1);
    const int4 pl = pln[0];
    load_step_op<M>(E, k, smem, n);
    // adjoint chain on [psi | lambda] (src/costs.py:326,342); costates not needed at n == 0
    const int cadj = (n > 0) ? Tg * (1 + I) : Tg;
    chain<M>(cx, k.op, cadj, 0, pl.x, pl.y, -1.0, st, cura, k.b.tb0, k.b.tb1, nullptr, 0, Tg);
    // derivative products for every channel, grouped by identical aux plan (src/costs.py:328-339)
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
      chain<M>(cx, k.op, (G + 1) * Tg, 1, pk.x, pk.y, 1.0, cura, curx, k.b.tb0, k.b.tb1, gch, G, Tg);
      const double2* curxc = curx;
      const double2* stc = st;
      colsum<M>(cx, G * Tg * I, [&](int vc, int i) {
        const int si = vc % I, rest = vc / I;
        const int t = rest % Tg, gi = rest / Tg;
        return cdot(ld<M>(stc + (long)lam_col(si, t) * d + i), ld<M>(curxc + (long)(gi * Tg + t) * d + i));
      });
      if (cx.writer && threadIdx.x == 0) {
        for (int vc = 0; vc < G * Tg * I; ++vc) {
          const int si = vc % I, rest = vc / I;
          const int t = rest % Tg, gi = rest / Tg;
          const int sidx = E.set_spec[set][si];
          E.ip[(((long)n * E.n_specs + sidx) * Kc + gch[gi]) * E.T_total + t0 + t] = cx.smres[vc];
        }
      }
      __syncthreads();
    }
    if (n == 0) break;
    // costate sources at psi_{n-1} (src/costs.py:341-353, :474-479)
    colsum<M>(cx, I * Tg, [&](int vc, int i) {
      const int si = vc / Tg, t = vc - si * Tg;
      const LgSpecDev& sp = E.spec[E.set_spec[set][si]];
      if (sp.kind != LGK_STATE_RUN) return make_double2(0.0, 0.0);
      return cdot(sp.tgt[(long)(trel + t) * d + i], ld<M>(cura + (long)t * d + i));
    });
    for (int si = 0; si < I; ++si) {
      const int sidx = E.set_spec[set][si];
      const LgSpecDev& sp = E.spec[sidx];
      const double2 tr = (sp.kind == LGK_GATE_RUN) ? E.trsum[(long)sidx * N + n - 1] : make_double2(0.0, 0.0);
      for (int t = 0; t < Tg; ++t) {
        const double2 ov = cx.smres[si * Tg + t];
        const long col = lam_col(si, t);
        for (int i = cx.r0 + threadIdx.x; i < cx.r1; i += blockDim.x) {
          double2 v = ld<M>(cura + col * d + i);
          if (sp.kind == LGK_STATE_PEN) {
            v = cadd(v, penalty_apply<M>(sp, d, cura + (long)t * d, i));
          } else if (sp.kind == LGK_STATE_RUN) {
            v = cadd(v, cmul(sp.tgt[(long)(trel + t) * d + i], ov));
          } else if (sp.kind == LGK_GATE_RUN) {
            v = cadd(v, cmul(sp.tgt[(long)(trel + t) * d + i], tr));
          }
          st[col * d + i] = v;
        }
      }
    }
    for (int t = 0; t < Tg; ++t)
      for (int i = cx.r0 + threadIdx.x; i < cx.r1; i += blockDim.x) st[(long)t * d + i] = ld<M>(cura + (long)t * d + i);
    bar_sync<M>(cx);
  }
}

// Sum of the per-trajectory running gate traces (fixed order), between sweeps.
extern "C" __global__ void lg_k_trsum(const double2* trp, int n_specs, int N, int T_total, const int* t0, const int* K,
                                      double2* trsum) {
  long q = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long)n_specs * N) return;
  const int s = (int)(q / N);
  const double2* p = trp + q * T_total + t0[s];
  double2 acc = make_double2(0.0, 0.0);
  for (int t = 0; t < K[s]; ++t) acc = cadd(acc, p[t]);
  trsum[q] = acc;
}

// explicit instantiations with C linkage-friendly wrappers
extern "C" void* lg_forward_kernel(int multi) {
  return multi ? (void*)lg_k_forward<true> : (void*)lg_k_forward<false>;
}
extern "C" void* lg_backward_kernel(int multi) {
  return multi ? (void*)lg_k_backward<true> : (void*)lg_k_backward<false>;
}
extern "C" void* lg_trsum_kernel() { return (void*)lg_k_trsum; }
