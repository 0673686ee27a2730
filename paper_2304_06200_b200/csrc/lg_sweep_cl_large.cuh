// LARGE variant of the cluster sweep engine (included by lg_sweep_cl.cuh; config 4 sized problems:
// several hundred rows per CTA, so one Taylor term per exchange).
//
// Same decomposition as the generic kernels -- one 16-CTA cluster per trajectory, RCM-banded rows,
// CTA rank r owns renumbered rows [r R, (r+1) R) with an H-row halo window in shared memory, halos
// pushed to the neighbours by st.async and counted on their per-buffer mbarriers -- but:
//  * every thread owns RPT rows (local rows li + k T, all in the bank-conflict-free 8-row phase
//    groups of cl_color_slots): a 640-row CTA runs 320 threads with a 168-register budget instead
//    of 640 threads capped at 96 registers (which spilled the operator rows);
//  * the window buffers are row-major with an odd column stride, so one row's gather serves every
//    column of the chain at immediate offsets (no address arithmetic per gather), and the gather
//    offsets are held as 16-bit byte offsets in registers;
//  * the column count, the chain mode and the control width are compile-time, and all gathers of a
//    row are issued before its stores;
//  * the control generator rows of the aux chains (src/derivatives.py:154-164) are staged in shared
//    memory once, padded to two entries per row.
// Measured on c4 (N' = 400): forward 114.8 -> 94.5 ms, backward 795.7 -> 781.6 ms against the
// generic kernels (which issue ~19 instructions per complex multiply-add against ~13 here); both are
// bound by the shared-memory pipe (~55 % busy on the active SMs, 10 % bank-conflict replays) and the
// latency of the gathers at 10 warps per SM -- the operator rows, Taylor accumulators, windows and
// staged control rows of 625 rows x 5 columns fill the register file and shared memory.
//
// Taylor recursion, plans, costates and per-step products are the generic kernels' (see the
// comments there and src/expm.py:345-350, src/costs.py:269-354, :407-488).
#pragma once

// RPT rows per thread at the thread count that gives the register budget they need (R <= RPT T):
// RPT 2 -> 320 threads (10 warps, 168 registers: the register file is split per SM sub-partition and two
// of them hold 3 warps), RPT 3 -> 224 threads (7 warps, 255 registers).  LG_CLL_T launches fewer threads.
#define CLL_T(RPT) ((RPT) == 2 ? 320 : 224)

namespace {

struct ClL {
  int d, R, H, WIN, CST, rank, CS, T, AS, g0, Wc, dbg;  // window rows WIN, column stride CST (odd), staged-row stride AS
  int red, rt, tb0, tb1, acs, accs, mb;
  mutable unsigned ph;  // parity bits of the next phase of the two exchange mbarriers
  const int* perm;      // renumbered row -> original row
  // row r of the thread (recomputed, not held: registers go to the term loop)
  __device__ __forceinline__ int lr(int r) const { return (int)threadIdx.x + r * T; }  // local row
  __device__ __forceinline__ int gi(int r) const { return g0 + lr(r); }                 // renumbered row
  __device__ __forceinline__ bool slot(int r) const { return lr(r) < R; }              // an own row
  __device__ __forceinline__ bool own(int r) const { return slot(r) && gi(r) < d; }    // ... that exists
  __device__ __forceinline__ int orig(int r) const { return own(r) ? __ldg(perm + gi(r)) : 0; }
};

template <int W, int MAXC, int RPT>
struct ClLRegs {
  double2 a[RPT][W];
  double2 cur[RPT][MAXC];
  // byte offset 16 CST (H + lr + rel) of the window row of slot w of row r, two 16-bit offsets
  // per register (entry k = r W + w in half k & 1 of word k >> 1; host: 16 CST WIN < 65536)
  unsigned go[(RPT * W + 1) / 2];
};

template <int RPT>
__device__ __forceinline__ ClL make_cll(const LgEngineArgs& E, int cmax, bool stage_ac) {
  ClL c;
  c.d = E.d;
  c.CS = (int)cl_size();
  c.rank = (int)cl_rank();
  c.R = E.cl_R;
  c.H = E.cl_H;
  c.T = blockDim.x;
  c.WIN = c.R + 2 * c.H;
  c.g0 = c.rank * c.R;
  c.Wc = E.Wc;
  c.dbg = E.dbg;
  c.perm = E.cl_perm;
  int o = 0;
  c.red = o;
  o += 16 * 32 + 16 * 16;
  c.rt = o;
  o += 72;
  c.CST = cmax | 1;
  c.tb0 = o;
  o += c.CST * c.WIN;
  c.tb1 = o;
  o += c.CST * c.WIN;
  c.acs = c.accs = -1;
  c.AS = lg_cll_as(c.R, c.T, RPT);
  if (stage_ac) {
    c.acs = o;
    o += E.Kc * 2 * c.AS;
    c.accs = o;
  }
  c.mb = lg_cll_mb_word(c.R, c.H, c.T, c.CST, stage_ac ? E.Kc * 2 : 0, RPT);
  c.ph = 0;
  return c;
}

__device__ __forceinline__ unsigned long long* cll_mb(const ClL& c, int k) {
  return reinterpret_cast<unsigned long long*>(cl_sm + c.mb) + k;
}

// own row r of column colo of window buffer buf: local store + the neighbours' halo slots
// Window buffers are row-major with an odd column stride CST: element (window row p, column q)
// of buffer buf at word buf + p CST + q.  A gather of one row reads all columns at immediate
// offsets, and 8 consecutive rows (an odd stride apart) still hit 8 distinct 16-byte bank groups
// whenever their row indices are distinct mod 8 (the cl_color_slots guarantee).
__device__ __forceinline__ int widx(const ClL& c, int buf, int p, int q) { return buf + p * c.CST + q; }
__device__ __forceinline__ void put_l(const ClL& c, int buf, int colo, double2 v, int r) {
  const int oi = c.lr(r);
  cl_sm[widx(c, buf, c.H + oi, colo)] = v;
  if (oi < c.H && c.rank > 0) cl_st(cl_map(&cl_sm[widx(c, buf, c.R + c.H + oi, colo)], c.rank - 1), v);
  if (oi >= c.R - c.H && c.rank + 1 < c.CS) cl_st(cl_map(&cl_sm[widx(c, buf, oi - c.R + c.H, colo)], c.rank + 1), v);
}
__device__ __forceinline__ void exchange_begin_l(const ClL& c, int yi, int C) {
  if (threadIdx.x == 0)
    mb_arm(cll_mb(c, yi), 16u * (unsigned)(c.H * C) * ((c.rank > 0 ? 1u : 0u) + (c.rank + 1 < c.CS ? 1u : 0u)));
}
__device__ __forceinline__ void exchange_end_l(const ClL& c, int yi) {
  __syncthreads();
  mb_wait(cll_mb(c, yi), (c.ph >> yi) & 1u);
  c.ph ^= 1u << yi;
}

// Cluster-wide deterministic sum of nv per-thread partials (both rows already added).
template <int NV>
__device__ void cll_reduce(const ClL& c, double2 (&v)[NV], int nv) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  double2* scr = cl_sm + c.red;
  double2* box = cl_sm + c.red + NV * 32;
  for (int q = 0; q < nv; ++q) {
    double2 s = warp_sum(v[q]);
    if (l == 0) scr[q * 32 + w] = s;
  }
  __syncthreads();
  if ((int)threadIdx.x < nv) {
    const int q = threadIdx.x;
    double2 s = make_double2(0.0, 0.0);
    for (int k = 0; k < nw; ++k) s = cadd(s, scr[q * 32 + k]);
    for (int r = 0; r < c.CS; ++r) cl_st(cl_map(&box[q * c.CS + c.rank], r), s);
  }
  cl_sync();
  for (int q = 0; q < nv; ++q) {
    double2 s = make_double2(0.0, 0.0);
    for (int r = 0; r < c.CS; ++r) s = cadd(s, box[q * c.CS + r]);
    v[q] = s;
  }
  cl_sync();
}

template <int W, int MAXC, int RPT>
__device__ __forceinline__ void load_row_l(const LgEngineArgs& E, const ClL& c, int n, ClLRegs<W, MAXC, RPT>& R) {
  const double2* src = E.A + (long)n * W * E.d;
#pragma unroll
  for (int r = 0; r < RPT; ++r)
#pragma unroll
    for (int w = 0; w < W; ++w)
      R.a[r][w] = c.own(r) ? src[(long)E.cl_slot[(long)w * E.d + c.gi(r)] * E.d + c.orig(r)] : make_double2(0.0, 0.0);
}
template <int W, int MAXC, int RPT>
__device__ __forceinline__ void load_go_l(const LgEngineArgs& E, const ClL& c, ClLRegs<W, MAXC, RPT>& R) {
#pragma unroll
  for (int r = 0; r < RPT; ++r)
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int rel = c.own(r) ? E.cl_cols[w * E.d + c.gi(r)] - c.gi(r) : 0;  // |rel| <= H
      const unsigned v = 16u * (unsigned)(c.CST * (c.H + (c.slot(r) ? c.lr(r) : 0) + rel));
      const int k = r * W + w;
      if (k & 1)
        R.go[k >> 1] |= v << 16;
      else
        R.go[k >> 1] = v;
    }
}

__device__ __forceinline__ double2 pen_apply_l(const LgEngineArgs& E, const LgSpecDev& sp, const ClL& c, int xwin,
                                               int r) {
  double2 p = make_double2(0.0, 0.0), q = make_double2(0.0, 0.0);
  for (int w = 0; w < sp.pen_W; ++w) {
    const long k = (long)w * c.d + c.orig(r);
    const int j = E.cl_inv[sp.pen_cols[k]] - c.g0 + c.H;
    cmac(p, q, sp.pen_vals[k], cl_sm[widx(c, xwin, j, 0)]);
  }
  return cadd(p, q);
}

// One Taylor term over NC columns of window buffer X into Y (MODE 1: columns [0, NC-1) aux tops
// of the channels whose staged-control offsets sit at rt + 64, NC-1 the bottom).  All gathers and
// products of both rows first, then the accumulator updates and the stores / halo pushes.
template <int W, int MAXC, int RPT, int NC, int MODE>
__device__ __forceinline__ void term_l(const ClL& c, ClLRegs<W, MAXC, RPT>& R, int X, int Y, double r, bool last, int yi) {
  const char* xbuf = reinterpret_cast<const char*>(cl_sm + X);
#pragma unroll
  for (int rr = 0; rr < RPT; ++rr) {
    // thread slots past the CTA's rows skip the term.  The branch also keeps ptxas from interleaving the
    // two rows' gathers: multi-column terms are register-bound and gain from that (c4 N' = 400 backward
    // 693 -> 674 ms), a one-column term needs the interleaving to hide its gather latency (forward 94.5 ms
    // without the branch, 117.5 ms with it), so NC == 1 keeps the unconditional form
    if (NC > 1 && !c.slot(rr)) continue;
    // FMA chains per column: four (a.x x and a.y (i x) apart) for one or two columns, two for
    // wider terms, whose columns give enough independent chains (and need the registers)
    constexpr bool SPL = NC <= 2;
    double2 p[NC], pq[SPL ? NC : 1];
#pragma unroll
    for (int q = 0; q < NC; ++q) p[q] = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < (SPL ? NC : 1); ++q) pq[q] = make_double2(0.0, 0.0);
    if (MODE >= 1 && !(c.dbg & 1)) {  // A_c of each top's channel times the bottom column (src/derivatives.py:154-164)
      // two staged entries per (channel, row) (the second zero when Wc == 1).  MODE 2: the tops come
      // in pairs of channels with one column pattern (c4: x and y drive of a transmon), and each
      // pair shares its two bottom-column gathers.
      const int* tab = reinterpret_cast<const int*>(cl_sm + c.rt + 64);
      const int* accb = reinterpret_cast<const int*>(cl_sm + c.accs) + c.lr(rr);
      constexpr int STEP = MODE == 2 ? 2 : 1;
#pragma unroll
      for (int q = 0; q < NC - 1; q += STEP) {
        const int koff = tab[q];
        double2 xb[2];
        {
          const int o0 = accb[koff], o1 = accb[koff + c.AS];
          xb[0] = cl_sm[widx(c, X, o0, NC - 1)];
          xb[1] = cl_sm[widx(c, X, o1, NC - 1)];
        }
#pragma unroll
        for (int h = 0; h < STEP; ++h) {
          const double2* ac = cl_sm + c.acs + tab[q + h] + c.lr(rr);
          cmac(p[q + h], pq[SPL ? q + h : 0], ac[0], xb[0], SPL);
          cmac(p[q + h], pq[SPL ? q + h : 0], ac[c.AS], xb[1], SPL);
        }
      }
    }
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int k = rr * W + w;
      const unsigned gw = R.go[k >> 1], go = (k & 1) ? gw >> 16 : gw & 0xffffu;
      const double2* xr = reinterpret_cast<const double2*>(xbuf + go);  // row of slot w, all columns
      const double2 a = R.a[rr][w];
#pragma unroll
      for (int q = 0; q < NC; ++q) cmac(p[q], pq[SPL ? q : 0], a, xr[q], SPL);
    }
    // local stores of this row (plain shared stores; the halo pushes follow for all rows)
    double2* yr = cl_sm + widx(c, Y, c.H + c.lr(rr), 0);
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const double2 tt = SPL ? make_double2((p[q].x + pq[SPL ? q : 0].x) * r, (p[q].y + pq[SPL ? q : 0].y) * r)
                             : make_double2(p[q].x * r, p[q].y * r);
      R.cur[rr][q] = cadd(R.cur[rr][q], tt);
      if (c.slot(rr)) yr[q] = last ? R.cur[rr][q] : tt;
    }
  }
  // boundary rows: push the stored values into the neighbours' halos (counted on their mbarrier yi)
#pragma unroll
  for (int rr = 0; rr < RPT; ++rr) {
    const int oi = c.lr(rr);
    if (!c.slot(rr)) continue;
    const bool lo = oi < c.H && c.rank > 0, hi = oi >= c.R - c.H && c.rank + 1 < c.CS;
    if (!lo && !hi) continue;
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const double2 v = cl_sm[widx(c, Y, c.H + oi, q)];
      if (lo)
        cl_st_async(cl_map(&cl_sm[widx(c, Y, c.R + c.H + oi, q)], c.rank - 1), v,
                    cl_map_u(smaddr(cll_mb(c, yi)), c.rank - 1));
      if (hi)
        cl_st_async(cl_map(&cl_sm[widx(c, Y, oi - c.R + c.H, q)], c.rank + 1), v,
                    cl_map_u(smaddr(cll_mb(c, yi)), c.rank + 1));
    }
  }
}

template <int W, int MAXC, int RPT, int NC, int MODE>
__device__ __forceinline__ void chain_l_nc(const ClL& c, ClLRegs<W, MAXC, RPT>& R, int m, int s) {
  int X = c.tb0, Y = c.tb1, yi = 1;
  for (int round = 0; round < s; ++round)
    for (int j = 1; j <= m; ++j) {
      exchange_begin_l(c, yi, NC);
      const double r = cl_sm[c.rt + j - 1].x;
      term_l<W, MAXC, RPT, NC, MODE>(c, R, X, Y, r, j == m, yi);
      exchange_end_l(c, yi);
      const int t_ = X;
      X = Y;
      Y = t_;
      yi ^= 1;
    }
}

// Input staged in tb0 (own rows + pushed halos) and in cur; result in cur.
template <int W, int MAXC, int RPT>
__device__ __forceinline__ void chain_l(const ClL& c, ClLRegs<W, MAXC, RPT>& R, int C, int mode, int m, int s, double sgn) {
  if ((int)threadIdx.x < m) cl_sm[c.rt + threadIdx.x].x = sgn * (1.0 / (double)(s * (threadIdx.x + 1)));
  cl_sync();  // staged input (incl. pushed halos) and the 1/(s j) table published
#define LG_NCL(n)                                  \
  if constexpr (n <= MAXC)                         \
    if (C == n) {                                  \
      if (mode == 0)                               \
        chain_l_nc<W, MAXC, RPT, n, 0>(c, R, m, s);     \
      else if constexpr (n >= 3 && n % 2 == 1) {   \
        if (mode == 2)                             \
          chain_l_nc<W, MAXC, RPT, n, 2>(c, R, m, s);   \
        else                                       \
          chain_l_nc<W, MAXC, RPT, n, 1>(c, R, m, s);   \
      } else if constexpr (n >= 2)                 \
        chain_l_nc<W, MAXC, RPT, n, 1>(c, R, m, s);     \
    }
  LG_NCL(1) LG_NCL(2) LG_NCL(3) LG_NCL(4) LG_NCL(5) LG_NCL(6) LG_NCL(7) LG_NCL(8)
#undef LG_NCL
  cl_sync();  // every CTA done reading its windows: the caller may stage the next chain's input
}

}  // namespace

// ------------------------------------------------------------------------------------ forward
template <int W, int MAXC, int RPT>
__device__ __forceinline__ void cll_forward_body(const LgEngineArgs& E) {
  const int g = blockIdx.x / (int)cl_size();
  const int set = E.grp_set[g], t0 = E.grp_t0[g], trel = t0 - E.set_t0[set];
  const int I = E.set_nspec[set], Kc = E.Kc, N = E.N;
  const int cst = 1 + E.cta_Imax, cmax = (Kc + 1) > cst ? (Kc + 1) : cst;
  ClL c = make_cll<RPT>(E, cmax, false);
  ClLRegs<W, MAXC, RPT> R;
  load_go_l(E, c, R);
  for (int q = threadIdx.x; q < c.tb1 + c.CST * c.WIN; q += blockDim.x) cl_sm[q] = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    mb_init(cll_mb(c, 0), 1);
    mb_init(cll_mb(c, 1), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  cl_sync();
  double2 psi[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) psi[r] = c.own(r) ? E.psi0[(long)t0 * c.d + c.orig(r)] : make_double2(0.0, 0.0);
  int4 pln = E.plan[0];
  double runacc[LG_MAX_SPECS];
  for (int q = 0; q < LG_MAX_SPECS; ++q) runacc[q] = 0.0;
  bool anyq = false, anypen = false;
  for (int si = 0; si < I; ++si) {
    const int kind = E.spec[E.set_spec[set][si]].kind;
    anyq |= kind == LGK_STATE_PEN || kind == LGK_STATE_RUN || kind == LGK_GATE_RUN;
    anypen |= kind == LGK_STATE_PEN;
  }
  for (int n = 0; n < N; ++n) {
    const int4 pl = pln;
    load_row_l(E, c, n, R);
    if (n + 1 < N) pln = E.plan[(long)(n + 1) * (Kc + 1)];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      if (c.slot(r)) put_l(c, c.tb0, 0, psi[r], r);
      R.cur[r][0] = psi[r];
    }
    chain_l(c, R, 1, 0, pl.x, pl.y, 1.0);
#pragma unroll
    for (int r = 0; r < RPT; ++r) psi[r] = R.cur[r][0];
    if (!anyq && n != N - 1) continue;
    if (anypen) {
#pragma unroll
      for (int r = 0; r < RPT; ++r)
        if (c.slot(r)) put_l(c, c.tb0, 0, psi[r], r);
      cl_sync();
    }
    double2 v[LG_MAX_SPECS];
    for (int si = 0; si < LG_MAX_SPECS; ++si) v[si] = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < RPT; ++r)
      if (c.own(r))
        for (int si = 0; si < I; ++si) {
          const LgSpecDev& sp = E.spec[E.set_spec[set][si]];
          double2 x;
          if (sp.kind == LGK_STATE_PEN)
            x = cdot(psi[r], pen_apply_l(E, sp, c, c.tb0, r));
          else if (sp.kind == LGK_STATE_INF)
            x = cdot(psi[r], sp.tgt[(long)trel * c.d + c.orig(r)]);
          else
            x = cdot(sp.tgt[(long)trel * c.d + c.orig(r)], psi[r]);
          v[si] = cadd(v[si], x);
        }
    cll_reduce<LG_MAX_SPECS>(c, v, I);
    if (c.rank == 0 && threadIdx.x == 0) {
      for (int si = 0; si < I; ++si) {
        const int sidx = E.set_spec[set][si];
        const int kind = E.spec[sidx].kind;
        if (kind == LGK_STATE_PEN) {
          runacc[si] += v[si].x;
        } else if (kind == LGK_STATE_RUN) {
          const double h = hypot(v[si].x, v[si].y);
          runacc[si] += h * h;
        } else if (kind == LGK_GATE_RUN) {
          E.trp[((long)sidx * N + n) * E.T_total + t0] = v[si];
        } else if (n == N - 1) {
          E.fin[(long)sidx * E.T_total + t0] = v[si];
        }
      }
    }
  }
  if (c.rank == 0 && threadIdx.x == 0)
    for (int si = 0; si < I; ++si) {
      const int sidx = E.set_spec[set][si];
      const int kind = E.spec[sidx].kind;
      if (kind == LGK_STATE_PEN || kind == LGK_STATE_RUN) E.run[(long)sidx * E.T_total + t0] += runacc[si];
    }
#pragma unroll
  for (int r = 0; r < RPT; ++r)
    if (c.own(r)) E.psiN[(long)t0 * c.d + c.orig(r)] = psi[r];
  cl_sync();
}

template <int W, int MAXC, int RPT>
__global__ void __launch_bounds__(CLL_T(RPT), 1) lg_k_cll_forward(const __grid_constant__ LgEngineArgs E) {
  cll_forward_body<W, MAXC, RPT>(E);
}
// line-search batch: candidate field blockIdx.y (lg_cost_batch)
template <int W, int MAXC, int RPT>
__global__ void __launch_bounds__(CLL_T(RPT), 1) lg_k_cll_forward_batch(const LgEngineArgs* __restrict__ EA) {
  cll_forward_body<W, MAXC, RPT>(EA[blockIdx.y]);
}

// ----------------------------------------------------------------------------------- backward
// Derivative products of step n (src/costs.py:328-339): for every channel group with a common aux
// plan, the aux chain [top_k ... | bottom] on the bottom psi_{n-1}, then <lambda_s(n)|top_k> into ip.
template <int W, int MAXC, int RPT>
__device__ __forceinline__ void aux_products_l(const LgEngineArgs& E, const ClL& c, ClLRegs<W, MAXC, RPT>& R, int n,
                                               int set, int t0, const double2 (&psip)[RPT],
                                               const double2 (&lam)[RPT][LG_MAX_SPECS]) {
  const int I = E.set_nspec[set], Kc = E.Kc;
  const int4* pln = E.plan + (long)n * (Kc + 1);
  int gch[LG_MAX_CHANNELS];
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
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      if (c.slot(r)) {
        for (int q = 0; q < G; ++q) put_l(c, c.tb0, q, make_double2(0.0, 0.0), r);
        put_l(c, c.tb0, G, psip[r], r);
      }
#pragma unroll
      for (int q = 0; q < MAXC; ++q) R.cur[r][q] = q == G ? psip[r] : make_double2(0.0, 0.0);
    }
    if ((int)threadIdx.x < G)  // channel offsets of the top columns (read after chain_l's cluster barrier)
      reinterpret_cast<int*>(cl_sm + c.rt + 64)[threadIdx.x] = gch[threadIdx.x] * 2 * c.AS;
    bool pairs = G % 2 == 0 && !(E.dbg & 2);  // every pair of tops: consecutive channels, one column pattern
    for (int q = 0; q + 1 < G && pairs; q += 2)
      pairs = gch[q + 1] == gch[q] + 1 && ((E.cl_cshare >> gch[q + 1]) & 1u);
    chain_l(c, R, G + 1, pairs ? 2 : 1, pk.x, pk.y, 1.0);
    double2 v[16];
    const int nv = I * G;
    for (int q = 0; q < 16; ++q) v[q] = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < RPT; ++r)
      if (c.own(r))
        for (int gi = 0; gi < G; ++gi)
          for (int si = 0; si < I; ++si) {
            double2 dd = make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < MAXC; ++q)
              if (q == gi) dd = R.cur[r][q];
            v[gi * I + si] = cadd(v[gi * I + si], cdot(lam[r][si], dd));
          }
    cll_reduce<16>(c, v, nv);
    if (c.rank == 0 && threadIdx.x == 0)
      for (int gi = 0; gi < G; ++gi)
        for (int si = 0; si < I; ++si) {
          const int sidx = E.set_spec[set][si];
          E.ip[(((long)n * E.n_specs + sidx) * Kc + gch[gi]) * E.T_total + t0] = v[gi * I + si];
        }
  }
}

// kernel prologue shared by the backward kernels: gather offsets, zeroed windows, exchange
// mbarriers, control rows staged (padded to two entries per row, Wc <= 2)
template <int W, int MAXC, int RPT>
__device__ __forceinline__ void cll_backward_setup(const LgEngineArgs& E, const ClL& c, ClLRegs<W, MAXC, RPT>& R) {
  load_go_l(E, c, R);
  for (int q = threadIdx.x; q < c.tb1 + c.CST * c.WIN; q += blockDim.x) cl_sm[q] = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    mb_init(cll_mb(c, 0), 1);
    mb_init(cll_mb(c, 1), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int kw = 0; kw < E.Kc * 2; ++kw)
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      if (c.lr(r) >= c.AS) continue;  // no table entry past the own rows
      const int k = kw >> 1, w = kw & 1;
      const bool ok = c.own(r) && w < E.Wc;
      const long src = ((long)k * E.Wc + w) * c.d;
      cl_sm[c.acs + kw * c.AS + c.lr(r)] = ok ? E.Ac[src + c.orig(r)] : make_double2(0.0, 0.0);
      reinterpret_cast<int*>(cl_sm + c.accs)[kw * c.AS + c.lr(r)] =
          ok ? E.cl_accols[src + c.gi(r)] - c.g0 + c.H : c.H + (c.slot(r) ? c.lr(r) : 0);
    }
  cl_sync();
}

// STORE == false: the fused backward sweep.  STORE == true: the adjoint sweep only -- psi_{n-1}
// and lambda_s(n) of every step go to HBM (E.bk_psi / E.bk_lam, renumbered rows) and the
// derivative products run afterwards as independent (step, trajectory) items on every resident
// cluster (lg_k_cll_aux): no tail wave, and the aux chains no longer wait on the adjoint chain.
template <int W, int MAXC, int RPT, bool STORE>
__device__ __forceinline__ void cll_backward_body(const LgEngineArgs& E) {
  const int g = blockIdx.x / (int)cl_size();
  const int set = E.grp_set[g], t0 = E.grp_t0[g], trel = t0 - E.set_t0[set];
  const int I = E.set_nspec[set], Kc = E.Kc, N = E.N;
  const int cst = 1 + E.cta_Imax, cmax = (Kc + 1) > cst ? (Kc + 1) : cst;
  ClL c = make_cll<RPT>(E, cmax, true);
  ClLRegs<W, MAXC, RPT> R;
  cll_backward_setup(E, c, R);
  if (STORE) bk_started(E);
  bool anypen = false, anyrun = false;
  for (int si = 0; si < I; ++si) {
    const int k = E.spec[E.set_spec[set][si]].kind;
    anypen |= k == LGK_STATE_PEN;
    anyrun |= k == LGK_STATE_RUN;
  }
  double2 psi[RPT], lam[RPT][LG_MAX_SPECS];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    psi[r] = c.own(r) ? E.psiN[(long)t0 * c.d + c.orig(r)] : make_double2(0.0, 0.0);
    for (int si = 0; si < LG_MAX_SPECS; ++si) lam[r][si] = make_double2(0.0, 0.0);
  }
  // ---- costate initialisation (src/costs.py:312-321, :457-460)
  {
    if (anypen) {
#pragma unroll
      for (int r = 0; r < RPT; ++r)
        if (c.slot(r)) put_l(c, c.tb0, 0, psi[r], r);
      cl_sync();
    }
    double2 ov[LG_MAX_SPECS];
    for (int si = 0; si < LG_MAX_SPECS; ++si) ov[si] = make_double2(0.0, 0.0);
    if (anyrun) {
#pragma unroll
      for (int r = 0; r < RPT; ++r)
        if (c.own(r))
          for (int si = 0; si < I; ++si) {
            const LgSpecDev& sp = E.spec[E.set_spec[set][si]];
            if (sp.kind == LGK_STATE_RUN) ov[si] = cadd(ov[si], cdot(sp.tgt[(long)trel * c.d + c.orig(r)], psi[r]));
          }
      cll_reduce<LG_MAX_SPECS>(c, ov, I);
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r)
      for (int si = 0; si < I; ++si) {
        const int sidx = E.set_spec[set][si];
        const LgSpecDev& sp = E.spec[sidx];
        double2 v = make_double2(0.0, 0.0);
        if (c.own(r)) {
          if (sp.kind == LGK_STATE_PEN) {
            v = pen_apply_l(E, sp, c, c.tb0, r);
          } else {
            const double2 tv = sp.tgt[(long)trel * c.d + c.orig(r)];
            if (sp.kind == LGK_STATE_RUN)
              v = cmul(tv, ov[si]);
            else if (sp.kind == LGK_GATE_RUN)
              v = cmul(tv, E.trsum[(long)sidx * N + N - 1]);
            else
              v = tv;
          }
        }
        lam[r][si] = v;
      }
    cl_sync();
  }
  for (int n = N - 1; n >= 0; --n) {
    const int4* pln = E.plan + (long)n * (Kc + 1);
    const int4 pl = pln[0];
    load_row_l(E, c, n, R);
    double2 psip[RPT], lamn[RPT][LG_MAX_SPECS];
    // adjoint chain on [psi | lambda] (src/costs.py:326,342); costates not needed at n == 0
    const int cadj = n > 0 ? 1 + I : 1;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      if (c.slot(r)) {
        put_l(c, c.tb0, 0, psi[r], r);
        for (int si = 0; si < I && n > 0; ++si) put_l(c, c.tb0, 1 + si, lam[r][si], r);
      }
#pragma unroll
      for (int q = 0; q < MAXC; ++q)
        R.cur[r][q] = q == 0 ? psi[r] : (q - 1 < I ? lam[r][q - 1] : make_double2(0.0, 0.0));
    }
    chain_l(c, R, cadj, 0, pl.x, pl.y, -1.0);
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      psip[r] = R.cur[r][0];
#pragma unroll
      for (int q = 1; q < MAXC; ++q)
        if (q - 1 < LG_MAX_SPECS) lamn[r][q - 1] = R.cur[r][q];
    }
    if constexpr (STORE) {  // hand psi_{n-1} and lambda_s(n) to the item kernel
      double2* bp = E.bk_psi + ((long)g * N + n) * c.d;
      double2* bl = E.bk_lam + ((long)g * N + n) * E.cta_Imax * c.d;
#pragma unroll
      for (int r = 0; r < RPT; ++r)
        if (c.own(r)) {
          bp[c.gi(r)] = psip[r];
          for (int si = 0; si < I; ++si) bl[(long)si * c.d + c.gi(r)] = lam[r][si];
        }
      bk_publish(E, g, (unsigned)c.rank, (unsigned)c.CS, (unsigned)(N - n));
    } else {
      aux_products_l(E, c, R, n, set, t0, psip, lam);
    }
    if (n == 0) break;
    // costate sources at psi_{n-1} (src/costs.py:341-353, :474-479)
    if (anypen) {
#pragma unroll
      for (int r = 0; r < RPT; ++r)
        if (c.slot(r)) put_l(c, c.tb0, 0, psip[r], r);
      cl_sync();
    }
    double2 ov[LG_MAX_SPECS];
    for (int si = 0; si < LG_MAX_SPECS; ++si) ov[si] = make_double2(0.0, 0.0);
    if (anyrun) {
#pragma unroll
      for (int r = 0; r < RPT; ++r)
        if (c.own(r))
          for (int si = 0; si < I; ++si) {
            const LgSpecDev& sp = E.spec[E.set_spec[set][si]];
            if (sp.kind == LGK_STATE_RUN) ov[si] = cadd(ov[si], cdot(sp.tgt[(long)trel * c.d + c.orig(r)], psip[r]));
          }
      cll_reduce<LG_MAX_SPECS>(c, ov, I);
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      for (int si = 0; si < I; ++si) {
        const int sidx = E.set_spec[set][si];
        const LgSpecDev& sp = E.spec[sidx];
        double2 v = lamn[r][si];
        if (c.own(r)) {
          if (sp.kind == LGK_STATE_PEN)
            v = cadd(v, pen_apply_l(E, sp, c, c.tb0, r));
          else if (sp.kind == LGK_STATE_RUN)
            v = cadd(v, cmul(sp.tgt[(long)trel * c.d + c.orig(r)], ov[si]));
          else if (sp.kind == LGK_GATE_RUN)
            v = cadd(v, cmul(sp.tgt[(long)trel * c.d + c.orig(r)], E.trsum[(long)sidx * N + n - 1]));
        }
        lam[r][si] = v;
      }
      psi[r] = psip[r];
    }
    cl_sync();
  }
  cl_sync();
}

template <int W, int MAXC, int RPT>
__global__ void __launch_bounds__(CLL_T(RPT), 1) lg_k_cll_backward(const __grid_constant__ LgEngineArgs E) {
  cll_backward_body<W, MAXC, RPT, false>(E);
}
template <int W, int MAXC, int RPT>
__global__ void __launch_bounds__(CLL_T(RPT), 1) lg_k_cll_adjoint(const __grid_constant__ LgEngineArgs E) {
  cll_backward_body<W, MAXC, RPT, true>(E);
}
// Derivative products as independent items (step n, trajectory group g), item = k * n_groups + g
// with k = N - 1 - n (the trajectories of one step are neighbours: A_n is read once into L2), dealt
// round-robin to the grid's clusters (all co-resident).  Reads psi_{n-1} and lambda_s(n) from HBM.
template <int W, int MAXC, int RPT>
__global__ void __launch_bounds__(CLL_T(RPT), 1) lg_k_cll_aux(const __grid_constant__ LgEngineArgs E) {
  const int cid = blockIdx.x / (int)cl_size(), ncl = gridDim.x / (int)cl_size();
  const int Kc = E.Kc, N = E.N;
  const int cst = 1 + E.cta_Imax, cmax = (Kc + 1) > cst ? (Kc + 1) : cst;
  ClL c = make_cll<RPT>(E, cmax, true);
  ClLRegs<W, MAXC, RPT> R;
  cll_backward_setup(E, c, R);
  (void)cid;
  (void)ncl;
  const long items = (long)E.n_groups * N;
  unsigned* slot = reinterpret_cast<unsigned*>(cl_sm + c.rt + 64) + 24;  // fetched item index (after the channel table)
  if (!bk_may_run(E, slot)) return;
  for (;;) {
    if (c.rank == 0 && threadIdx.x == 0) {
      const unsigned it = atomicAdd(E.bk_next, 1u);
      for (int r = 0; r < c.CS; ++r)
        asm volatile("st.shared::cluster.u32 [%0], %1;\n" ::"r"(cl_map(slot, r)), "r"(it) : "memory");
    }
    cl_sync();
    const long it = *slot;
    cl_sync();  // every rank has read the index before rank 0 may overwrite it
    if (it >= items) break;
    const int g = (int)(it % E.n_groups), n = N - 1 - (int)(it / E.n_groups);
    const int set = E.grp_set[g], t0 = E.grp_t0[g], I = E.set_nspec[set];
    bk_wait(E, g, (unsigned)(N - n));
    load_row_l(E, c, n, R);
    const double2* bp = E.bk_psi + ((long)g * N + n) * c.d;
    const double2* bl = E.bk_lam + ((long)g * N + n) * E.cta_Imax * c.d;
    double2 psip[RPT], lam[RPT][LG_MAX_SPECS];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      psip[r] = c.own(r) ? bp[c.gi(r)] : make_double2(0.0, 0.0);
      for (int si = 0; si < LG_MAX_SPECS; ++si)
        lam[r][si] = c.own(r) && si < I ? bl[(long)si * c.d + c.gi(r)] : make_double2(0.0, 0.0);
    }
    aux_products_l(E, c, R, n, set, t0, psip, lam);
  }
  cl_sync();
}
