// Warp-specialised sweep engine for small state dimensions (d <= 64 RPL).
//
// The backward sweep of src/costs.py:324-353 / :454-482 is a set of chains that
// are only coupled through the recovered states:
//   P   : psi_{n-1} = U_n^dagger psi_n                          (adjoint chain on psi)
//   L_s : lambda_s <- U_n^dagger lambda_s + source_s(psi_{n-1})  (one costate per cost term)
//   X_k : D_k = dU_n/da_k psi_{n-1} via the aux embedding,     (one per control channel)
//         then <lambda_s(n) | D_k> for every s
// Each chain gets its own TEAM of two warps (one row of the state per lane;
// RPL rows per lane for d > 64) that synchronises with a named barrier per
// Taylor term -- no CTA-wide barrier on the critical path.  Teams hand states
// over through shared-memory rings guarded by mbarriers (full/empty per slot),
// so P runs ahead, X_k start step n as soon as psi_{n-1} exists, and the
// critical path per step is max(mu, mu_aux) instead of mu + mu_aux.
// The forward sweep pairs the propagation team with a team that evaluates the
// per-step scalars (penalty expectations, running overlaps, gate traces).
// One CTA per trajectory; operator rows of A_n live in registers (exact ELL
// width W), prefetched one step ahead.
#include "lg_types.h"

namespace {

extern __shared__ __align__(16) double2 ws_sm[];

constexpr int TEAM = 64;  // threads per team
constexpr int RING = 4;   // ring depth (steps a producer may run ahead)

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cdot(double2 a, double2 b) {  // conj(a) b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ void cmac(double2& p, double2& q, double2 a, double2 x) {
  p.x = fma(a.x, x.x, p.x);
  p.y = fma(a.x, x.y, p.y);
  q.x = fma(-a.y, x.y, q.x);
  q.y = fma(a.y, x.x, q.y);
}
__device__ __forceinline__ double2 warp_sum(double2 v) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// ---- mbarrier helpers (shared::cta)
__device__ __forceinline__ unsigned smaddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smaddr(b)), "r"(count));
}
__device__ __forceinline__ void mb_arrive(unsigned long long* b) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smaddr(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smaddr(b)),
      "r"(parity)
      : "memory");
}
// Two phase waits with their SYNCS round trips overlapped (both try_waits issued before either is
// checked; a completed phase keeps testing true until the barrier is re-armed by this thread's writes).
__device__ __forceinline__ void mb_wait2(unsigned long long* b0, unsigned p0, unsigned long long* b1, unsigned p1) {
  asm volatile(
      "{\n .reg .pred p, q;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 q, [%2], %3;\n and.pred p, p, q;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smaddr(b0)),
      "r"(p0), "r"(smaddr(b1)), "r"(p1)
      : "memory");
}
// ---- cluster (DSMEM) helpers
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_map(const void* p, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smaddr(p)), "r"(rank));
  return r;
}
// Push 16 bytes into a peer CTA's shared memory and count them on the peer's mbarrier
// (async proxy, like a TMA store): the consumer waits with CTA-scope acquire, no L1 invalidation.
__device__ __forceinline__ void cl_st_async(unsigned addr, double2 v, unsigned mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(addr),
               "d"(v.x), "d"(v.y), "r"(mbar)
               : "memory");
}
// Arm the current phase of a local mbarrier for `bytes` of incoming st.async data (one arrival).
__device__ __forceinline__ void mb_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smaddr(b)), "r"(bytes) : "memory");
}
// "Slot free" signal to a peer's ring: carries no data (the slot's values were already consumed
// into registers), so no release fence.
__device__ __forceinline__ void cl_arrive_relaxed(unsigned addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void team_sync(int id) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(TEAM) : "memory"); }

struct Team {
  int id;    // named barrier id (1..15)
  int tl;    // thread index within team
  int tsz;   // 32 (single warp: __syncwarp) or 64 (two warps: named barrier)
  int d;
};

__device__ __forceinline__ void tsync(const Team& tm) {
  if (tm.tsz == 32)
    __syncwarp();
  else
    team_sync(tm.id);
}

// One Taylor term: Y <- (A X) r (+ cur when LAST), rows owned by this lane.
// ox/oy: shared offsets of the two term buffers; addresses of the operand
// slots are loop invariant (the caller alternates two fixed buffers).
template <int W, int RPL, int NC>
__device__ __forceinline__ void team_term(const Team& tm, double2 (&cur)[NC][RPL], const double2 (&a)[RPL][W],
                                          const int (&col)[RPL][W], const double2 (&ac)[RPL][2],
                                          const int (&accol)[RPL][2], int ox, int oy, double r, bool last) {
  const int d = tm.d;
#pragma unroll
  for (int k = 0; k < RPL; ++k) {
    const int i = tm.tl + k * tm.tsz;
    if (i >= d) continue;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double2 p = make_double2(0.0, 0.0), q = make_double2(0.0, 0.0);
#pragma unroll
      for (int w = 0; w < W; ++w) cmac(p, q, a[k][w], ws_sm[ox + c * d + col[k][w]]);
      if (NC == 2 && c == 0) {
        cmac(p, q, ac[k][0], ws_sm[ox + d + accol[k][0]]);
        cmac(p, q, ac[k][1], ws_sm[ox + d + accol[k][1]]);
      }
      const double2 tt = make_double2((p.x + q.x) * r, (p.y + q.y) * r);
      cur[c][k] = cadd(cur[c][k], tt);
      if (last)
        ws_sm[oy + c * d + i] = cur[c][k];
      else
        ws_sm[oy + c * d + i] = tt;
    }
  }
  tsync(tm);
}

// Per-team Taylor chain over NC columns (NC == 2: column 0 is the aux top with
// the control generator acting on column 1, the bottom).  Input staged in tb0;
// the chain alternates tb0 -> tb1 -> tb0 ... two terms per loop trip.
template <int W, int RPL, int NC>
__device__ __forceinline__ void team_chain(const Team& tm, double2 (&cur)[NC][RPL], const double2 (&a)[RPL][W],
                                           const int (&col)[RPL][W], const double2 (&ac)[RPL][2],
                                           const int (&accol)[RPL][2], int m, int s, double sgn, int tb0, int tb1,
                                           int rt, bool build = true) {
  if (build) {  // else the caller staged sgn / (s j) at rt from E.rtab before its last team barrier
    if (tm.tl < m) ws_sm[rt + tm.tl].x = sgn * (1.0 / (double)(s * (tm.tl + 1)));
    tsync(tm);
  }
  const int total = m * s;
  int j = 1;  // position within the current scaling round
  for (int t = 0; t < total; t += 2) {
    team_term<W, RPL, NC>(tm, cur, a, col, ac, accol, tb0, tb1, ws_sm[rt + j - 1].x, j == m);
    j = j == m ? 1 : j + 1;
    if (t + 1 == total) {
      // odd number of terms: result is in tb1; callers only use cur registers
      break;
    }
    team_term<W, RPL, NC>(tm, cur, a, col, ac, accol, tb1, tb0, ws_sm[rt + j - 1].x, j == m);
    j = j == m ? 1 : j + 1;
  }
}

// ---- dense rows (DenseMatrix problems, d <= 64): A_n is staged per step in shared memory,
// column-major like the ELL table ([w][i], slot w == column w), one step ahead with cp.async.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smaddr(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
// Issue the copy of a d x d complex block (16-byte elements) into shared memory at `dst`.
__device__ __forceinline__ void stage_block(const double2* src, int dst, int dd, int tid, int nthr) {
  for (int q = tid; q < dd; q += nthr) cp_async16(&ws_sm[dst + q], src + q);
  cp_async_commit();
}
// p = sum_w M[w][i] x[w] over a dense row, x read as a broadcast; four independent accumulators.
__device__ __forceinline__ void dense_row(double2& p, double2& q, int mop, int xo, int i, int d) {
  double2 p1 = make_double2(0.0, 0.0), q1 = p1, p2 = p1, q2 = p1, p3 = p1, q3 = p1;
  int w = 0;
  for (; w + 4 <= d; w += 4) {
    cmac(p, q, ws_sm[mop + w * d + i], ws_sm[xo + w]);
    cmac(p1, q1, ws_sm[mop + (w + 1) * d + i], ws_sm[xo + w + 1]);
    cmac(p2, q2, ws_sm[mop + (w + 2) * d + i], ws_sm[xo + w + 2]);
    cmac(p3, q3, ws_sm[mop + (w + 3) * d + i], ws_sm[xo + w + 3]);
  }
  for (; w < d; ++w) cmac(p, q, ws_sm[mop + w * d + i], ws_sm[xo + w]);
  p = cadd(cadd(p, p1), cadd(p2, p3));
  q = cadd(cadd(q, q1), cadd(q2, q3));
}
// Dense single-column team chain (propagation / adjoint / costate): operator at shared offset aop.
__device__ __forceinline__ void team_chain_dense(const Team& tm, double2& cur, int aop, int m, int s, double sgn,
                                                 int tb0, int tb1, int rt) {
  if (tm.tl < m) ws_sm[rt + tm.tl].x = sgn * (1.0 / (double)(s * (tm.tl + 1)));
  tsync(tm);
  const int total = m * s, d = tm.d, i = tm.tl;
  int X = tb0, Y = tb1, j = 1;
  for (int t = 0; t < total; ++t) {
    const double r = ws_sm[rt + j - 1].x;
    const bool last = j == m;
    if (i < d) {
      double2 p = make_double2(0.0, 0.0), q = make_double2(0.0, 0.0);
      dense_row(p, q, aop, X, i, d);
      const double2 tt = make_double2((p.x + q.x) * r, (p.y + q.y) * r);
      cur = cadd(cur, tt);
      ws_sm[Y + i] = last ? cur : tt;
    }
    tsync(tm);
    const int t_ = X;
    X = Y;
    Y = t_;
    j = last ? 1 : j + 1;
  }
}
// Same chain with the lane's operator row held in registers for the whole step (DM >= d
// columns, zero beyond d; the term buffers' second column region is zero, so the x
// broadcasts past d read zeros): per term only the d broadcast x loads go through the
// shared-memory pipe instead of d row loads + d broadcasts.
template <int DM>
__device__ __forceinline__ void team_chain_dense_r(const Team& tm, double2& cur, int aop, int m, int s, double sgn,
                                                   int tb0, int tb1, int rt) {
  if (tm.tl < m) ws_sm[rt + tm.tl].x = sgn * (1.0 / (double)(s * (tm.tl + 1)));
  tsync(tm);
  const int total = m * s, d = tm.d, i = tm.tl;
  double2 ar[DM];
#pragma unroll
  for (int w = 0; w < DM; ++w) ar[w] = (i < d && w < d) ? ws_sm[aop + w * d + i] : make_double2(0.0, 0.0);
  int j = 1;
  auto term = [&](int X, int Y) {
    const double r = ws_sm[rt + j - 1].x;
    const bool last = j == m;
    if (i < d) {
      double2 p[4], q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) p[u] = q[u] = make_double2(0.0, 0.0);
#pragma unroll
      for (int w = 0; w < DM; ++w) cmac(p[w & 3], q[w & 3], ar[w], ws_sm[X + w]);
      const double2 pp = cadd(cadd(p[0], p[1]), cadd(p[2], p[3]));
      const double2 qq = cadd(cadd(q[0], q[1]), cadd(q[2], q[3]));
      const double2 tt = make_double2((pp.x + qq.x) * r, (pp.y + qq.y) * r);
      cur = cadd(cur, tt);
      if (last)
        ws_sm[Y + i] = cur;
      else
        ws_sm[Y + i] = tt;
    }
    tsync(tm);
    j = last ? 1 : j + 1;
  };
  for (int t = 0; t < total; t += 2) {
    term(tb0, tb1);
    if (t + 1 == total) break;
    term(tb1, tb0);
  }
}
// Smallest instantiated register row width DM >= d with DM <= 2d (team_chain_dense_r reads
// the zero region past d).
extern "C" int lg_ws_dense_width(int d) {
  return d <= 8 ? 8 : d <= 16 ? 16 : d <= 32 ? 32 : d <= 40 ? 40 : d <= 48 ? 48 : 64;
}
// Register rows up to 48 columns; wider rows would spill (255 registers), so they stay in
// shared memory.
template <int DM>
__device__ __forceinline__ void team_chain_dense_w(const Team& tm, double2& cur, int aop, int m, int s, double sgn,
                                                   int tb0, int tb1, int rt) {
  if constexpr (DM <= 48)
    team_chain_dense_r<DM>(tm, cur, aop, m, s, sgn, tb0, tb1, rt);
  else
    team_chain_dense(tm, cur, aop, m, s, sgn, tb0, tb1, rt);
}
// Dense derivative chain on the four-warp team: top = A x_top + A_c x_bottom, bottom = A x_bottom.
__device__ __forceinline__ void x4_chain_dense(int bar_id, int i, int d, bool top, double2& cur, int aop, int acop,
                                               int m, int s, int tb0, int tb1, int rt, int tl) {
  if (tl < m) ws_sm[rt + tl].x = 1.0 / (double)(s * (tl + 1));
  asm volatile("bar.sync %0, 128;\n" ::"r"(bar_id) : "memory");
  const int total = m * s;
  const int c = top ? 0 : d;
  int X = tb0, Y = tb1, j = 1;
  for (int t = 0; t < total; ++t) {
    const double r = ws_sm[rt + j - 1].x;
    const bool last = j == m;
    if (i < d) {
      double2 p = make_double2(0.0, 0.0), q = make_double2(0.0, 0.0);
      dense_row(p, q, aop, X + c, i, d);
      if (top) dense_row(p, q, acop, X + d, i, d);
      const double2 tt = make_double2((p.x + q.x) * r, (p.y + q.y) * r);
      cur = cadd(cur, tt);
      ws_sm[Y + c + i] = last ? cur : tt;
    }
    asm volatile("bar.sync %0, 128;\n" ::"r"(bar_id) : "memory");
    const int t_ = X;
    X = Y;
    Y = t_;
    j = last ? 1 : j + 1;
  }
}

// Derivative team of four warps: warps 0-1 own the aux top column, warps 2-3
// the bottom column, one row per lane.  Per term every thread first loads all
// its operand slots, then accumulates, then stores (no store->load ordering
// between the two columns), and the team meets at a 128-thread named barrier.
template <int W>
__device__ __forceinline__ void x4_chain(int bar_id, int i, int d, bool top, double2& cur, const double2 (&a)[W],
                                         const int (&col)[W], const double2 (&ac)[2], const int (&accol)[2], int m,
                                         int s, int tb0, int tb1, int rt, int tl) {
  if (tl < m) ws_sm[rt + tl].x = 1.0 / (double)(s * (tl + 1));
  asm volatile("bar.sync %0, 128;\n" ::"r"(bar_id) : "memory");
  const int total = m * s;
  const int c = top ? 0 : d;  // own column offset inside a term buffer
  int X = tb0, Y = tb1, j = 1;
  for (int t = 0; t < total; ++t) {
    const double r = ws_sm[rt + j - 1].x;
    const bool last = j == m;
    if (i < d) {
      double2 x[W], y[2];
#pragma unroll
      for (int w = 0; w < W; ++w) x[w] = ws_sm[X + c + col[w]];
      if (top) {
        y[0] = ws_sm[X + d + accol[0]];
        y[1] = ws_sm[X + d + accol[1]];
      }
      double2 p0 = make_double2(0.0, 0.0), q0 = make_double2(0.0, 0.0);
      double2 p1 = make_double2(0.0, 0.0), q1 = make_double2(0.0, 0.0);
#pragma unroll
      for (int w = 0; w < W; ++w) {
        if (w & 1)
          cmac(p1, q1, a[w], x[w]);
        else
          cmac(p0, q0, a[w], x[w]);
      }
      if (top) {
        cmac(p1, q1, ac[0], y[0]);
        cmac(p0, q0, ac[1], y[1]);
      }
      const double2 tt = make_double2(((p0.x + q0.x) + (p1.x + q1.x)) * r, ((p0.y + q0.y) + (p1.y + q1.y)) * r);
      cur = cadd(cur, tt);
      ws_sm[Y + c + i] = last ? cur : tt;
    }
    asm volatile("bar.sync %0, 128;\n" ::"r"(bar_id) : "memory");
    const int t_ = X;
    X = Y;
    Y = t_;
    j = last ? 1 : j + 1;
  }
}

template <int W, int RPL>
__device__ __forceinline__ void load_rows(const LgEngineArgs& E, int n, int tl, int tsz, double2 (&a)[RPL][W],
                                          int (&col)[RPL][W]) {
  const double2* src = E.A + (long)n * W * E.d;
#pragma unroll
  for (int k = 0; k < RPL; ++k) {
    const int i = tl + k * tsz;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const bool ok = i < E.d;
      a[k][w] = ok ? src[(long)w * E.d + i] : make_double2(0.0, 0.0);
      col[k][w] = ok ? E.A_cols[w * E.d + i] : 0;
    }
  }
}

template <int W>
__device__ __forceinline__ void load_vals(const LgEngineArgs& E, int n, int i, double2 (&a)[1][W]) {
  const double2* src = E.A + (long)n * W * E.d;
#pragma unroll
  for (int w = 0; w < W; ++w) a[0][w] = i < E.d ? src[(long)w * E.d + i] : make_double2(0.0, 0.0);
}

// Team-wide deterministic sum of nv (<= NV) complex values -> v[0..nv) for all team threads.
template <int NV>
__device__ __forceinline__ void team_reduce(const Team& tm, double2 (&v)[NV], int nv, int red) {
  const int w = tm.tl >> 5, l = tm.tl & 31;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    if (q >= nv) break;
    v[q] = warp_sum(v[q]);
    if (tm.tsz == 64 && l == 0) ws_sm[red + q * 2 + w] = v[q];
  }
  if (tm.tsz == 32) return;
  team_sync(tm.id);
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    if (q >= nv) break;
    v[q] = cadd(ws_sm[red + q * 2], ws_sm[red + q * 2 + 1]);
  }
  team_sync(tm.id);
}

// Shared-memory layout (double2 units); barriers at the end (8-byte words).
struct WsLay {
  int tb;      // per team: 2 buffers x 2 columns x d   (team q at tb + q * 4d)
  int rt;      // per team: 64
  int red;     // per team: 2 * LG_MAX_SPECS
  int ring;    // psi ring: RING x d
  int lring;   // lambda rings: I x RING x d
  int tgt;     // targets: I x d
  int pen;     // penalty values: I x Wp x d ; cols as ints after
  int pencol;  // int offset (double2 units * 4 = int units)
  int dbuf;    // [2][d] derivative hand-off (cluster kernel)
  int aop;     // dense rows: A_n double buffer [2][d][d] (column-major), then A_c of one channel [d][d]
  int bars;    // mbarriers
  int words;
};

__host__ __device__ __forceinline__ WsLay ws_layout(int d, int nteams, int I, int Wp, int extra_bars = 0,
                                                    int dense = 0) {
  WsLay L;
  int o = 0;
  L.tb = o;
  o += nteams * 4 * d;
  L.rt = o;
  o += nteams * 64;
  L.red = o;
  o += nteams * 2 * LG_MAX_SPECS;
  L.ring = o;
  o += RING * d;
  L.lring = o;
  o += I * RING * d;
  L.tgt = o;
  o += I * d;
  L.pen = o;
  o += I * Wp * d;
  L.pencol = o;
  o += (I * Wp * d + 3) / 4;
  L.dbuf = o;  // [4][d] derivative columns handed from the X team to its dot warp (cluster kernel)
  o += 4 * d;
  L.aop = o;
  if (dense) o += 3 * d * d;
  L.bars = o;
  o += (2 * RING * (1 + I) + 4 + extra_bars + 1) / 2 + 1;
  L.words = o;
  return L;
}

__device__ __forceinline__ double2 pen_row(int d, int Wp, int pen, const int* pcol, int i, int psi) {
  double2 p = make_double2(0.0, 0.0), q = make_double2(0.0, 0.0);
  for (int w = 0; w < Wp; ++w) cmac(p, q, ws_sm[pen + w * d + i], ws_sm[psi + pcol[w * d + i]]);
  return cadd(p, q);
}

}  // namespace


// Stage the targets / penalty operators of this set into shared memory.
__device__ __forceinline__ void stage_specs(const LgEngineArgs& E, const WsLay& L, int set, int trel, int I, int Wp,
                                            int* pcol) {
  const int d = E.d;
  for (int si = 0; si < I; ++si) {
    const LgSpecDev& sp = E.spec[E.set_spec[set][si]];
    for (int i = threadIdx.x; i < d; i += blockDim.x)
      ws_sm[L.tgt + si * d + i] = sp.tgt ? sp.tgt[(long)trel * d + i] : make_double2(0.0, 0.0);
    for (int q = threadIdx.x; q < Wp * d; q += blockDim.x) {
      const int w = q / d;
      const bool ok = sp.kind == LGK_STATE_PEN && w < sp.pen_W;
      ws_sm[L.pen + si * Wp * d + q] = ok ? sp.pen_vals[q] : make_double2(0.0, 0.0);
      pcol[si * Wp * d + q] = ok ? sp.pen_cols[q] : (q % d);
    }
  }
}

// ------------------------------------------------------------------------------------------ forward
// warps 0-1: propagation team P; warps 2-3: per-step scalars team F.  d <= 64.
// DNS: dense rows (W unused), A_n staged in shared memory one step ahead.
template <int W, int DNS>
__device__ __forceinline__ void ws_forward_body(const LgEngineArgs& E) {
  const int d = E.d, g = blockIdx.x, N = E.N, dd = d * d;
  const int set = E.grp_set[g], t0 = E.grp_t0[g], trel = t0 - E.set_t0[set];
  const int I = E.set_nspec[set];
  int Wp = 1;
  for (int si = 0; si < I; ++si) Wp = max(Wp, E.spec[E.set_spec[set][si]].pen_W);
  const WsLay L = ws_layout(d, 2, I, Wp, 0, DNS);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(ws_sm + L.bars);
  unsigned long long* full = bars;
  unsigned long long* empty = bars + RING;
  int* pcol = reinterpret_cast<int*>(ws_sm) + 4 * L.pencol;
  const int team = threadIdx.x / 64;
  const Team tm{team + 1, (int)threadIdx.x % 64, 64, d};
  stage_specs(E, L, set, trel, I, Wp, pcol);
  for (int q = threadIdx.x; q < 2 * 4 * d; q += blockDim.x) ws_sm[L.tb + q] = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    for (int j = 0; j < RING; ++j) {
      mb_init(&full[j], 64);
      mb_init(&empty[j], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int tb0 = L.tb + team * 4 * d, tb1 = tb0 + 2 * d;
  const int i = tm.tl;
  if (team == 0) {
    // ---------------- P: forward propagation
    double2 cur[1][1];
    double2 a[1][W], an[1][W];
    int col[1][W], coln[1][W];
    const double2 ac[1][2] = {{make_double2(0.0, 0.0), make_double2(0.0, 0.0)}};
    const int accol[1][2] = {{0, 0}};
    if (i < d) ws_sm[tb0 + i] = E.psi0[(long)t0 * d + i];
    const int rt = L.rt + team * 64;
    double rnx = 0.0;  // Taylor coefficients of the next step, staged before the end-of-step barrier
    if (DNS) {
      stage_block(E.A, L.aop, dd, tm.tl, 64);
    } else {
      load_rows<W, 1>(E, 0, tm.tl, 64, an, coln);
#pragma unroll
      for (int w = 0; w < W; ++w) col[0][w] = coln[0][w];  // one ELL pattern for every step
      ws_sm[rt + tm.tl].x = E.rtab[tm.tl];
      team_sync(tm.id);
    }
    int4 pln = E.plan[0];
    for (int n = 0; n < N; ++n) {
      const int4 pl = pln;
      if (DNS) {
        cp_async_wait_all();
        tsync(tm);  // A_n staged; buffer (n + 1) & 1 no longer read (step n - 1 done)
        if (n + 1 < N) stage_block(E.A + (long)(n + 1) * dd, L.aop + ((n + 1) & 1) * dd, dd, tm.tl, 64);
      } else {
#pragma unroll
        for (int w = 0; w < W; ++w) a[0][w] = an[0][w];
        if (n + 1 < N) {
          load_vals<W>(E, n + 1, i, an);
          rnx = E.rtab[(long)(n + 1) * 64 + tm.tl];
        }
      }
      if (n + 1 < N) pln = E.plan[(long)(n + 1) * (E.Kc + 1)];
      cur[0][0] = i < d ? ws_sm[tb0 + i] : make_double2(0.0, 0.0);
      if (DNS)
        team_chain_dense_w<W>(tm, cur[0][0], L.aop + (n & 1) * dd, pl.x, pl.y, 1.0, tb0, tb1, rt);
      else
        team_chain<W, 1, 1>(tm, cur, a, col, ac, accol, pl.x, pl.y, 1.0, tb0, tb1, rt, false);
      const int slot = n % RING;
      // one slot-free wait per two steps: the scalars team consumes the ring in order, so its release
      // of step n - 3 (slot (n + 1) % RING) implies step n - 4's (slot n % RING)
      if ((n & 1) == 0 && n + 1 >= RING) mb_wait(&empty[(n + 1) % RING], (((n + 1) / RING) - 1) & 1);
      if (i < d) {
        ws_sm[L.ring + slot * d + i] = cur[0][0];
        ws_sm[tb0 + i] = cur[0][0];
      }
      if (!DNS) ws_sm[rt + tm.tl].x = rnx;  // the chain's last read of the table was before its last barrier
      mb_arrive(&full[slot]);
      team_sync(tm.id);
    }
    if (i < d) E.psiN[(long)t0 * d + i] = cur[0][0];
  } else {
    // ---------------- F: per-step scalars from the psi ring
    double runacc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int n = 0; n < N; ++n) {
      const int slot = n % RING, use = n / RING;
      mb_wait(&full[slot], use & 1);
      const int psi = L.ring + slot * d;
      double2 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = make_double2(0.0, 0.0);
      if (i < d) {
        const double2 pv = ws_sm[psi + i];
        for (int si = 0; si < I; ++si) {
          const int kind = E.spec[E.set_spec[set][si]].kind;
          if (kind == LGK_STATE_PEN)
            v[si] = cdot(pv, pen_row(d, Wp, L.pen + si * Wp * d, pcol + si * Wp * d, i, psi));
          else if (kind == LGK_STATE_INF)
            v[si] = cdot(pv, ws_sm[L.tgt + si * d + i]);
          else
            v[si] = cdot(ws_sm[L.tgt + si * d + i], pv);
        }
      }
      team_reduce<4>(tm, v, I, L.red + team * 2 * LG_MAX_SPECS);
      if (tm.tl == 0) {
        mb_arrive(&empty[slot]);
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
    if (tm.tl == 0)
      for (int si = 0; si < I; ++si) {
        const int sidx = E.set_spec[set][si];
        const int kind = E.spec[sidx].kind;
        if (kind == LGK_STATE_PEN || kind == LGK_STATE_RUN) E.run[(long)sidx * E.T_total + t0] += runacc[si];
      }
  }
}

template <int W, int DNS>
__global__ void __launch_bounds__(128, 1) lg_k_ws_forward(const __grid_constant__ LgEngineArgs E) {
  ws_forward_body<W, DNS>(E);
}
// Line-search batch (lg_cost_batch): candidate field blockIdx.y with its own step generators,
// plans and raw outputs, all candidates in one launch (src/optimizer.py:153-170).
template <int W, int DNS>
__global__ void __launch_bounds__(128, 1) lg_k_ws_forward_batch(const LgEngineArgs* __restrict__ EA) {
  ws_forward_body<W, DNS>(EA[blockIdx.y]);
}

// ------------------------------------------------------------------------------------------ backward
// teams of two warps (one row per lane): X_0..X_{Kc-1}, P, L_0..L_{I-1}.  d <= 64.
template <int W>
__global__ void __launch_bounds__(512, 1) lg_k_ws_backward(const __grid_constant__ LgEngineArgs E) {
  const int d = E.d, g = blockIdx.x, Kc = E.Kc, N = E.N;
  const int set = E.grp_set[g], t0 = E.grp_t0[g], trel = t0 - E.set_t0[set];
  const int I = E.set_nspec[set];
  int Wp = 1;
  for (int si = 0; si < I; ++si) Wp = max(Wp, E.spec[E.set_spec[set][si]].pen_W);
  const int nteams = Kc + 1 + I;
  const WsLay L = ws_layout(d, nteams, I, Wp);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(ws_sm + L.bars);
  unsigned long long* pfull = bars;               // [RING]
  unsigned long long* pempty = bars + RING;       // [RING]
  unsigned long long* lfull = bars + 2 * RING;    // [I][RING]
  unsigned long long* lempty = lfull + I * RING;  // [I][RING]
  int* pcol = reinterpret_cast<int*>(ws_sm) + 4 * L.pencol;
  const int team = threadIdx.x >> 6, tl = threadIdx.x & 63;
  const Team tm{team + 1, tl, 64, d};
  int n_lpsi = 0;
  for (int si = 0; si < I; ++si) {
    const int kind = E.spec[E.set_spec[set][si]].kind;
    n_lpsi += (kind == LGK_STATE_PEN || kind == LGK_STATE_RUN);
  }
  stage_specs(E, L, set, trel, I, Wp, pcol);
  if (threadIdx.x == 0) {
    for (int j = 0; j < RING; ++j) {
      mb_init(&pfull[j], 64);
      mb_init(&pempty[j], Kc + n_lpsi);
      for (int si = 0; si < I; ++si) {
        mb_init(&lfull[si * RING + j], 64);
        mb_init(&lempty[si * RING + j], Kc);
      }
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (team >= nteams) return;  // set with fewer cost terms than the widest set
  const int tb0 = L.tb + team * 4 * d, tb1 = tb0 + 2 * d, rt = L.rt + team * 64;
  const int red = L.red + team * 2 * LG_MAX_SPECS;

  if (team < Kc) {
    // ---------------- X_k: derivative products and inner products (one row per lane)
    const int kch = team, i = tl;
    double2 a[1][W], an[1][W];
    int col[1][W], coln[1][W];
    double2 ac[1][2];
    int accol[1][2];
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const bool ok = i < d && w < E.Wc;
      ac[0][w] = ok ? E.Ac[((long)kch * E.Wc + w) * d + i] : make_double2(0.0, 0.0);
      accol[0][w] = ok ? E.Ac_cols[((long)kch * E.Wc + w) * d + i] : 0;
    }
    load_rows<W, 1>(E, N - 1, tl, 64, an, coln);
    int4 pln = E.plan[(long)(N - 1) * (Kc + 1) + 1 + kch];
    for (int it = 0; it < N; ++it) {
      const int n = N - 1 - it;
      const int4 pl = pln;
#pragma unroll
      for (int w = 0; w < W; ++w) a[0][w] = an[0][w], col[0][w] = coln[0][w];
      if (n > 0) {
        load_rows<W, 1>(E, n - 1, tl, 64, an, coln);
        pln = E.plan[(long)(n - 1) * (Kc + 1) + 1 + kch];
      }
      const int slot = it % RING, use = it / RING;
      long long* trc = E.trace ? E.trace + (((long)g * 8 + team) * N + it) * 4 : nullptr;
      if (trc && tl == 0) trc[0] = clock64();
      mb_wait(&pfull[slot], use & 1);
      if (trc && tl == 0) trc[1] = clock64();
      double2 cur[2][1];
      const double2 v0 = i < d ? ws_sm[L.ring + slot * d + i] : make_double2(0.0, 0.0);
      cur[0][0] = make_double2(0.0, 0.0);
      cur[1][0] = v0;
      if (i < d) {
        ws_sm[tb0 + i] = make_double2(0.0, 0.0);
        ws_sm[tb0 + d + i] = v0;
      }
      team_sync(tm.id);
      if (tl == 0) mb_arrive(&pempty[slot]);
      team_chain<W, 1, 2>(tm, cur, a, col, ac, accol, pl.x, pl.y, 1.0, tb0, tb1, rt);
      if (trc && tl == 0) trc[2] = clock64();
      double2 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = make_double2(0.0, 0.0);
      for (int si = 0; si < I; ++si) {
        mb_wait(&lfull[si * RING + slot], use & 1);
        if (i < d) v[si] = cdot(ws_sm[L.lring + (si * RING + slot) * d + i], cur[0][0]);
      }
      team_reduce<4>(tm, v, I, red);
      if (trc && tl == 0) trc[3] = clock64();
      if (tl == 0) {
        for (int si = 0; si < I; ++si) {
          mb_arrive(&lempty[si * RING + slot]);
          const int sidx = E.set_spec[set][si];
          E.ip[(((long)n * E.n_specs + sidx) * Kc + kch) * E.T_total + t0] = v[si];
        }
      }
    }
  } else if (team == Kc) {
    // ---------------- P: psi recovery by adjoint propagation
    const int i = tl;
    double2 cur[1][1];
    double2 a[1][W], an[1][W];
    int col[1][W], coln[1][W];
    const double2 ac[1][2] = {};
    const int accol[1][2] = {};
    if (i < d) ws_sm[tb0 + i] = E.psiN[(long)t0 * d + i];
    load_rows<W, 1>(E, N - 1, tl, 64, an, coln);
    int4 pln = E.plan[(long)(N - 1) * (Kc + 1)];
    team_sync(tm.id);
    for (int it = 0; it < N; ++it) {
      const int n = N - 1 - it;
      const int4 pl = pln;
#pragma unroll
      for (int w = 0; w < W; ++w) a[0][w] = an[0][w], col[0][w] = coln[0][w];
      if (n > 0) {
        load_rows<W, 1>(E, n - 1, tl, 64, an, coln);
        pln = E.plan[(long)(n - 1) * (Kc + 1)];
      }
      cur[0][0] = i < d ? ws_sm[tb0 + i] : make_double2(0.0, 0.0);
      long long* trc = E.trace ? E.trace + (((long)g * 8 + team) * N + it) * 4 : nullptr;
      if (trc && tl == 0) trc[0] = clock64();
      team_chain<W, 1, 1>(tm, cur, a, col, ac, accol, pl.x, pl.y, -1.0, tb0, tb1, rt);
      if (trc && tl == 0) trc[1] = clock64();
      const int slot = it % RING, use = it / RING;
      if (use > 0) mb_wait(&pempty[slot], (use - 1) & 1);
      if (trc && tl == 0) trc[2] = clock64();
      if (i < d) {
        ws_sm[L.ring + slot * d + i] = cur[0][0];
        ws_sm[tb0 + i] = cur[0][0];
      }
      mb_arrive(&pfull[slot]);
      team_sync(tm.id);
    }
  } else {
    // ---------------- L_s: costate chain + sources 
    const int si = team - Kc - 1;
    const int sidx = E.set_spec[set][si];
    const int kind = E.spec[sidx].kind;
    const bool needs_psi = kind == LGK_STATE_PEN || kind == LGK_STATE_RUN;
    const int tg = L.tgt + si * d;
    const int pen = L.pen + si * Wp * d;
    const int* pc = pcol + si * Wp * d;
    double2 a[1][W], an[1][W];
    int col[1][W], coln[1][W];
    const double2 ac[1][2] = {};
    const int accol[1][2] = {};
    // costate initialisation from psi_N (src/costs.py:312-321, :457-460); psi_N staged in tb1
#pragma unroll
    for (int k = 0; k < 1; ++k) {
      const int i = tl;
      if (i < d) ws_sm[tb1 + i] = E.psiN[(long)t0 * d + i];
    }
    team_sync(tm.id);
    double2 ov[1] = {make_double2(0.0, 0.0)};
    if (kind == LGK_STATE_RUN) {
#pragma unroll
      for (int k = 0; k < 1; ++k) {
        const int i = tl;
        if (i < d) ov[0] = cadd(ov[0], cdot(ws_sm[tg + i], ws_sm[tb1 + i]));
      }
      team_reduce<1>(tm, ov, 1, red);
    }
    const double2 trN = kind == LGK_GATE_RUN ? E.trsum[(long)sidx * N + N - 1] : make_double2(0.0, 0.0);
    double2 cur[1][1];
#pragma unroll
    for (int k = 0; k < 1; ++k) {
      const int i = tl;
      double2 v = make_double2(0.0, 0.0);
      if (i < d) {
        if (kind == LGK_STATE_PEN)
          v = pen_row(d, Wp, pen, pc, i, tb1);
        else if (kind == LGK_STATE_RUN)
          v = cmul(ws_sm[tg + i], ov[0]);
        else if (kind == LGK_GATE_RUN)
          v = cmul(ws_sm[tg + i], trN);
        else
          v = ws_sm[tg + i];
      }
      cur[0][k] = v;
    }
    team_sync(tm.id);
    load_rows<W, 1>(E, N - 1, tl, 64, an, coln);
    int4 pln = E.plan[(long)(N - 1) * (Kc + 1)];
    for (int it = 0; it < N; ++it) {
      const int n = N - 1 - it;
      const int slot = it % RING, use = it / RING;
      long long* trc = E.trace ? E.trace + (((long)g * 8 + team) * N + it) * 4 : nullptr;
      if (trc && tl == 0) trc[0] = clock64();
      // publish lambda_s(n) for the X teams; it is also the chain input
      if (use > 0) mb_wait(&lempty[si * RING + slot], (use - 1) & 1);
      if (trc && tl == 0) trc[1] = clock64();
#pragma unroll
      for (int k = 0; k < 1; ++k) {
        const int i = tl;
        if (i < d) {
          ws_sm[L.lring + (si * RING + slot) * d + i] = cur[0][k];
          ws_sm[tb0 + i] = cur[0][k];
        }
      }
      mb_arrive(&lfull[si * RING + slot]);
      if (n == 0) break;
      const int4 pl = pln;
#pragma unroll
      for (int w = 0; w < W; ++w) a[0][w] = an[0][w], col[0][w] = coln[0][w];
      load_rows<W, 1>(E, n - 1, tl, 64, an, coln);
      pln = E.plan[(long)(n - 1) * (Kc + 1)];
      const double2 tr = kind == LGK_GATE_RUN ? E.trsum[(long)sidx * N + n - 1] : make_double2(0.0, 0.0);
      team_sync(tm.id);
      team_chain<W, 1, 1>(tm, cur, a, col, ac, accol, pl.x, pl.y, -1.0, tb0, tb1, rt);
      if (trc && tl == 0) trc[2] = clock64();
      if (needs_psi) {
        mb_wait(&pfull[slot], use & 1);
        if (trc && tl == 0) trc[3] = clock64();
        const int psi = L.ring + slot * d;
        if (kind == LGK_STATE_RUN) {
          double2 o2[1] = {make_double2(0.0, 0.0)};
#pragma unroll
          for (int k = 0; k < 1; ++k) {
            const int i = tl;
            if (i < d) o2[0] = cadd(o2[0], cdot(ws_sm[tg + i], ws_sm[psi + i]));
          }
          team_reduce<1>(tm, o2, 1, red);
#pragma unroll
          for (int k = 0; k < 1; ++k) {
            const int i = tl;
            if (i < d) cur[0][k] = cadd(cur[0][k], cmul(ws_sm[tg + i], o2[0]));
          }
        } else {
#pragma unroll
          for (int k = 0; k < 1; ++k) {
            const int i = tl;
            if (i < d) cur[0][k] = cadd(cur[0][k], pen_row(d, Wp, pen, pc, i, psi));
          }
        }
        team_sync(tm.id);
        if (tl == 0) mb_arrive(&pempty[slot]);
      } else if (kind == LGK_GATE_RUN) {
#pragma unroll
        for (int k = 0; k < 1; ++k) {
          const int i = tl;
          if (i < d) cur[0][k] = cadd(cur[0][k], cmul(ws_sm[tg + i], tr));
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------------------ backward (cluster)
// Cluster of 1 + Imax + Kc * NW CTAs per trajectory, every chain on its own SM.  Rank 0: psi-recovery
// team P (inverse propagation, src/costs.py:326).  Rank 1 + s: costate team L_s (src/costs.py:341-353).
// Rank 1 + Imax + k * NW + w: derivative worker
// of channel k for the backward steps it = w (mod NW): the aux chain of step n needs only psi_{n-1}
// and A_n (src/costs.py:328-331), so NW workers take a channel's derivative chains off the
// sequential psi / lambda critical path.  Each worker: X team (four warps: top | bottom column of
// the block operator) + a dot-product warp for <lambda_s(n)|dU_n/da_k psi_{n-1}>.  P and L_s
// st.async psi_{n-1} / lambda_s(n) rows into the responsible worker's 2-slot ring
// (mbarrier complete_tx); workers free slots with relaxed remote arrives.
constexpr int WR = 4;  // ring slots per worker (psi / lambda) and derivative hand-off depth
template <int W, int DNS>
__global__ void __launch_bounds__(192, 1) lg_k_wsc_backward(const __grid_constant__ LgEngineArgs E) {
  const int d = E.d, Kc = E.Kc, N = E.N, NW = E.ws_nw, NWK = Kc * E.ws_nw, IM = E.cta_Imax, dd = d * d;
  const unsigned rank = cl_rank();
  const int g = blockIdx.x / (1 + IM + NWK);
  const int xr0 = 1 + IM;  // first worker rank
  const int set = E.grp_set[g], t0 = E.grp_t0[g], trel = t0 - E.set_t0[set];
  const int I = E.set_nspec[set];
  int Wp = 1;
  for (int si = 0; si < I; ++si) Wp = max(Wp, E.spec[E.set_spec[set][si]].pen_W);
  const WsLay L = ws_layout(d, 1, IM, Wp, 2 * RING + NWK * WR * (1 + IM), DNS);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(ws_sm + L.bars);
  // rank 0 (P): costate ranks free psi slots; workers free their psi slots
  unsigned long long* pempty = bars;                  // [RING]
  unsigned long long* wempty = bars + RING;           // [NWK][WR]
  // costate rank 1 + s: psi_{n-1} arrived (penalty / running sources); workers free lambda slots;
  // source ring between the source warp and the costate team
  unsigned long long* pfull = bars;                   // [RING]
  unsigned long long* lempty = bars + RING;           // [NWK][WR]
  unsigned long long* sfull = lempty + NWK * WR;      // [RING]
  unsigned long long* sempty = sfull + RING;          // [RING]
  // workers
  unsigned long long* xfull = bars;                   // [WR] psi_{n-1} arrived
  unsigned long long* lfull = bars + WR;              // [I][WR] lambda_s(n) arrived
  unsigned long long* dfull = lfull + I * WR;         // [WR] X team -> dot warp
  unsigned long long* dempty = dfull + WR;            // [WR] dot warp -> X team
  int* pcol = reinterpret_cast<int*>(ws_sm) + 4 * L.pencol;
  const int team = threadIdx.x >> 6, tl = threadIdx.x & 63;
  const Team tm{team + 1, tl, 64, d};
  int n_lpsi = 0;
  for (int si = 0; si < I; ++si) {
    const int kind = E.spec[E.set_spec[set][si]].kind;
    n_lpsi += (kind == LGK_STATE_PEN || kind == LGK_STATE_RUN);
  }
  stage_specs(E, L, set, trel, I, Wp, pcol);
  for (int q = threadIdx.x; q < 4 * d; q += blockDim.x) ws_sm[L.tb + q] = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    if (rank == 0) {
      for (int j = 0; j < RING; ++j) mb_init(&pempty[j], n_lpsi > 0 ? n_lpsi : 1);
      for (int q = 0; q < NWK * WR; ++q) mb_init(&wempty[q], 1);
    } else if (rank < (unsigned)xr0) {
      for (int j = 0; j < RING; ++j) {
        mb_init(&pfull[j], 1);  // armed by expect_tx
        mb_init(&sfull[j], 32);
        mb_init(&sempty[j], 1);
      }
      for (int q = 0; q < NWK * WR; ++q) mb_init(&lempty[q], 1);
    } else {
      for (int j = 0; j < WR * (1 + I); ++j) mb_init(&xfull[j], 1);  // xfull and lfull: armed by expect_tx
      for (int b = 0; b < WR; ++b) {
        mb_init(&dfull[b], 1);
        mb_init(&dempty[b], 1);
      }
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  cl_sync();
  const int i = tl;
  const int tb0 = L.tb, tb1 = tb0 + 2 * d, rt = L.rt, red = L.red;  // one team per CTA
  if (rank >= (unsigned)xr0 && threadIdx.x < 128) {
    // ---------------- X: derivative worker (channel kch, steps it = w mod NW), four warps
    const int wi = rank - xr0, kch = wi / NW, w0 = wi % NW;
    const int t4 = threadIdx.x;
    const bool top = t4 < 64;
    const int ix = t4 & 63;
    double2 a[W], an[W];
    int col[W], coln[W];
    double2 ac[2];
    int accol[2];
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const bool ok = !DNS && top && ix < d && w < E.Wc;
      ac[w] = ok ? E.Ac[((long)kch * E.Wc + w) * d + ix] : make_double2(0.0, 0.0);
      accol[w] = ok ? E.Ac_cols[((long)kch * E.Wc + w) * d + ix] : 0;
    }
    if (DNS) stage_block(E.Ac + (long)kch * dd, L.aop + 2 * dd, dd, t4, 128);  // A_c of this channel
    auto rows = [&](int n, double2 (&aa)[W], int (&cc)[W]) {
      const double2* src = E.A + (long)n * W * d;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        aa[w] = ix < d ? src[(long)w * d + ix] : make_double2(0.0, 0.0);
        cc[w] = ix < d ? E.A_cols[w * d + ix] : 0;
      }
    };
    if (w0 < N) {
      if (DNS)
        stage_block(E.A + (long)(N - 1 - w0) * dd, L.aop, dd, t4, 128);
      else
        rows(N - 1 - w0, an, coln);
    }
    const int xb0 = L.tb, xb1 = L.tb + 2 * d, xrt = L.rt;
    for (int it = w0, u = 0; it < N; it += NW, ++u) {
      const int n = N - 1 - it;
      const int4 pl = E.plan[(long)n * (Kc + 1) + 1 + kch];
      if (DNS) {
        cp_async_wait_all();
        asm volatile("bar.sync 1, 128;\n" ::: "memory");  // A_n (and A_c) staged; the other buffer free
        if (it + NW < N) stage_block(E.A + (long)(n - NW) * dd, L.aop + ((u + 1) & 1) * dd, dd, t4, 128);
      } else {
#pragma unroll
        for (int w = 0; w < W; ++w) a[w] = an[w], col[w] = coln[w];
        if (it + NW < N) rows(n - NW, an, coln);
      }
      const int slot = u % WR;
      long long* trc = E.trace ? E.trace + (((long)g * 8 + wi) * N + it) * 4 : nullptr;
      if (trc && t4 == 0) trc[0] = clock64();
      if (t4 == 0) mb_expect_tx(&xfull[slot], (unsigned)d * 16u);
      mb_wait(&xfull[slot], (u / WR) & 1);
      if (trc && t4 == 0) trc[1] = clock64();
      double2 cur = make_double2(0.0, 0.0);
      if (ix < d) {
        const double2 v0 = ws_sm[L.ring + slot * d + ix];
        if (!top) cur = v0;
        ws_sm[xb0 + (top ? 0 : d) + ix] = top ? make_double2(0.0, 0.0) : v0;
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (t4 == 0) cl_arrive_relaxed(cl_map(&wempty[wi * WR + slot], 0));
      if (DNS)
        x4_chain_dense(1, ix, d, top, cur, L.aop + (u & 1) * dd, L.aop + 2 * dd, pl.x, pl.y, xb0, xb1, xrt, t4);
      else
        x4_chain<W>(1, ix, d, top, cur, a, col, ac, accol, pl.x, pl.y, xb0, xb1, xrt, t4);
      if (trc && t4 == 0) trc[2] = clock64();
      // hand D_k to the dot warp
      const int b = u % WR;
      if (u >= WR) mb_wait(&dempty[b], ((u / WR) - 1) & 1);
      if (top && ix < d) ws_sm[L.dbuf + b * d + ix] = cur;
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (t4 == 0) mb_arrive(&dfull[b]);
      if (trc && t4 == 0) trc[3] = clock64();
    }
  } else if (rank >= (unsigned)xr0 && threadIdx.x < 160) {
    // ---------------- dot warp of the worker: ip[n][s][k] = <lambda_s(n) | dU_n/da_k psi_{n-1}>
    const int wi = rank - xr0, kch = wi / NW, w0 = wi % NW;
    const int lane = threadIdx.x - 128;
    for (int it = w0, u = 0; it < N; it += NW, ++u) {
      const int n = N - 1 - it;
      const int slot = u % WR, b = u % WR;
      if (lane < I) mb_expect_tx(&lfull[lane * WR + slot], (unsigned)d * 16u);
      mb_wait(&dfull[b], (u / WR) & 1);
      double2 v[LG_MAX_SPECS];
      for (int si = 0; si < I; ++si) {
        mb_wait(&lfull[si * WR + slot], (u / WR) & 1);
        double2 acc = make_double2(0.0, 0.0);
        for (int i2 = lane; i2 < d; i2 += 32)
          acc = cadd(acc, cdot(ws_sm[L.lring + (si * WR + slot) * d + i2], ws_sm[L.dbuf + b * d + i2]));
        v[si] = warp_sum(acc);
      }
      __syncwarp();
      if (lane == 0) {
        mb_arrive(&dempty[b]);
        for (int si = 0; si < I; ++si) {
          cl_arrive_relaxed(cl_map(&lempty[wi * WR + slot], 1 + si));
          const int sidx = E.set_spec[set][si];
          E.ip[(((long)n * E.n_specs + sidx) * Kc + kch) * E.T_total + t0] = v[si];
        }
      }
      __syncwarp();
    }
  } else if (rank == 0 && threadIdx.x < 64) {
    // ---------------- P: psi recovery; pushes psi_{n-1} to the costate ranks that need it and to the
    // step's workers (one per channel)
    double2 cur[1][1];
    double2 a[1][W], an[1][W];
    int col[1][W], coln[1][W];
    const double2 ac[1][2] = {};
    const int accol[1][2] = {};
    unsigned lpsi = 0;  // costate ranks with psi-dependent sources
    for (int si = 0; si < I; ++si) {
      const int kind = E.spec[E.set_spec[set][si]].kind;
      if (kind == LGK_STATE_PEN || kind == LGK_STATE_RUN) lpsi |= 1u << si;
    }
    if (i < d) ws_sm[tb0 + i] = E.psiN[(long)t0 * d + i];
    double rnx = 0.0;  // Taylor coefficients of the next step, staged before the end-of-step barrier
    if (DNS) {
      stage_block(E.A + (long)(N - 1) * dd, L.aop, dd, tl, 64);
    } else {
      load_rows<W, 1>(E, N - 1, tl, 64, an, coln);
#pragma unroll
      for (int w = 0; w < W; ++w) col[0][w] = coln[0][w];  // one ELL pattern for every step
      ws_sm[rt + tl].x = -E.rtab[(long)(N - 1) * 64 + tl];
    }
    int4 pln = E.plan[(long)(N - 1) * (Kc + 1)];
    team_sync(tm.id);
    for (int it = 0; it < N; ++it) {
      const int n = N - 1 - it;
      const int4 pl = pln;
      if (DNS) {
        cp_async_wait_all();
        team_sync(tm.id);
        if (n > 0) stage_block(E.A + (long)(n - 1) * dd, L.aop + ((it + 1) & 1) * dd, dd, tl, 64);
      } else {
#pragma unroll
        for (int w = 0; w < W; ++w) a[0][w] = an[0][w];
        if (n > 0) {
          load_vals<W>(E, n - 1, i, an);
          rnx = E.rtab[(long)(n - 1) * 64 + tl];
        }
      }
      if (n > 0) pln = E.plan[(long)(n - 1) * (Kc + 1)];
      cur[0][0] = i < d ? ws_sm[tb0 + i] : make_double2(0.0, 0.0);
      long long* trc = E.trace ? E.trace + (((long)g * 8 + 7) * N + it) * 4 : nullptr;
      if (trc && tl == 0) trc[0] = clock64();
      if (DNS)
        team_chain_dense_w<W>(tm, cur[0][0], L.aop + (it & 1) * dd, pl.x, pl.y, -1.0, tb0, tb1, rt);
      else
        team_chain<W, 1, 1>(tm, cur, a, col, ac, accol, pl.x, pl.y, -1.0, tb0, tb1, rt, false);
      if (trc && tl == 0) trc[1] = clock64();
      const int w0 = it % NW, u = it / NW, wslot = u % WR;
      if (u >= WR) {  // the workers' slots are free (they took psi of step it - WR * NW)
        const unsigned par = ((u / WR) - 1) & 1;
        if (Kc == 2)
          mb_wait2(&wempty[w0 * WR + wslot], par, &wempty[(NW + w0) * WR + wslot], par);
        else
          for (int k = 0; k < Kc; ++k) mb_wait(&wempty[(k * NW + w0) * WR + wslot], par);
      }
      const int slot = it % RING, use = it / RING;
      if (lpsi && use > 0) mb_wait(&pempty[slot], (use - 1) & 1);
      if (trc && tl == 0) trc[2] = clock64();
      if (i < d) {
        ws_sm[tb0 + i] = cur[0][0];
        for (int k = 0; k < Kc; ++k) {
          const int r = xr0 + k * NW + w0;
          cl_st_async(cl_map(&ws_sm[L.ring + wslot * d + i], r), cur[0][0], cl_map(&xfull[wslot], r));
        }
        for (int si = 0; si < I; ++si)
          if (lpsi & (1u << si))
            cl_st_async(cl_map(&ws_sm[L.ring + slot * d + i], 1 + si), cur[0][0], cl_map(&pfull[slot], 1 + si));
      }
      if (!DNS) ws_sm[rt + tl].x = -rnx;  // the chain's last read of the table was before its last barrier
      team_sync(tm.id);
    }
  } else if (rank >= 1 && rank < (unsigned)(1 + I) && threadIdx.x < 64) {
    // ---------------- L_s on its own SM: costate chain + sources; pushes lambda_s(n) to the step's workers
    const int si = rank - 1;
    const int sidx = E.set_spec[set][si];
    const int kind = E.spec[sidx].kind;
    const bool needs_psi = kind == LGK_STATE_PEN || kind == LGK_STATE_RUN;
    const int tg = L.tgt + si * d;
    const int pen = L.pen + si * Wp * d;
    const int* pc = pcol + si * Wp * d;
    double2 a[1][W], an[1][W];
    int col[1][W], coln[1][W];
    const double2 ac[1][2] = {};
    const int accol[1][2] = {};
    if (i < d) ws_sm[tb1 + i] = E.psiN[(long)t0 * d + i];
    team_sync(tm.id);
    double2 ov[1] = {make_double2(0.0, 0.0)};
    if (kind == LGK_STATE_RUN) {
      if (i < d) ov[0] = cdot(ws_sm[tg + i], ws_sm[tb1 + i]);
      team_reduce<1>(tm, ov, 1, red);
    }
    const double2 trN = kind == LGK_GATE_RUN ? E.trsum[(long)sidx * N + N - 1] : make_double2(0.0, 0.0);
    double2 cur[1][1];
    {
      double2 v = make_double2(0.0, 0.0);
      if (i < d) {
        if (kind == LGK_STATE_PEN)
          v = pen_row(d, Wp, pen, pc, i, tb1);
        else if (kind == LGK_STATE_RUN)
          v = cmul(ws_sm[tg + i], ov[0]);
        else if (kind == LGK_GATE_RUN)
          v = cmul(ws_sm[tg + i], trN);
        else
          v = ws_sm[tg + i];
      }
      cur[0][0] = v;
    }
    team_sync(tm.id);
    double rnx = 0.0;  // Taylor coefficients of this iteration's chain, loaded an iteration ahead
    if (DNS) {
      stage_block(E.A + (long)(N - 1) * dd, L.aop, dd, tl, 64);
    } else {
      load_rows<W, 1>(E, N - 1, tl, 64, an, coln);
#pragma unroll
      for (int w = 0; w < W; ++w) col[0][w] = coln[0][w];  // one ELL pattern for every step
      rnx = E.rtab[(long)(N - 1) * 64 + tl];
    }
    int4 pln = E.plan[(long)(N - 1) * (Kc + 1)];
    for (int it = 0; it < N; ++it) {
      const int n = N - 1 - it;
      const int slot = it % RING, use = it / RING;
      const int w0 = it % NW, u = it / NW, wslot = u % WR;
      long long* trc = (E.trace && si < 2) ? E.trace + (((long)g * 8 + 6 - si) * N + it) * 4 : nullptr;
      if (trc && tl == 0) trc[0] = clock64();
      if (u >= WR) {
        const unsigned par = ((u / WR) - 1) & 1;
        if (Kc == 2)
          mb_wait2(&lempty[w0 * WR + wslot], par, &lempty[(NW + w0) * WR + wslot], par);
        else
          for (int k = 0; k < Kc; ++k) mb_wait(&lempty[(k * NW + w0) * WR + wslot], par);
      }
      if (trc && tl == 0) trc[1] = clock64();
      if (i < d) {
        ws_sm[tb0 + i] = cur[0][0];
        for (int k = 0; k < Kc; ++k) {
          const int r = xr0 + k * NW + w0;
          cl_st_async(cl_map(&ws_sm[L.lring + (si * WR + wslot) * d + i], r), cur[0][0],
                      cl_map(&lfull[si * WR + wslot], r));
        }
      }
      if (n == 0) break;
      const int4 pl = pln;
      if (DNS) {
        cp_async_wait_all();
        team_sync(tm.id);
        stage_block(E.A + (long)(n - 1) * dd, L.aop + ((it + 1) & 1) * dd, dd, tl, 64);
      } else {
#pragma unroll
        for (int w = 0; w < W; ++w) a[0][w] = an[0][w];
        load_vals<W>(E, n - 1, i, an);
        ws_sm[rt + tl].x = -rnx;  // the previous chain's last read of the table was before its last barrier
        rnx = E.rtab[(long)(n - 1) * 64 + tl];
      }
      pln = E.plan[(long)(n - 1) * (Kc + 1)];
      const double2 tr = kind == LGK_GATE_RUN ? E.trsum[(long)sidx * N + n - 1] : make_double2(0.0, 0.0);
      team_sync(tm.id);
      if (DNS)
        team_chain_dense_w<W>(tm, cur[0][0], L.aop + (it & 1) * dd, pl.x, pl.y, -1.0, tb0, tb1, rt);
      else
        team_chain<W, 1, 1>(tm, cur, a, col, ac, accol, pl.x, pl.y, -1.0, tb0, tb1, rt, false);
      if (trc && tl == 0) trc[2] = clock64();
      if (needs_psi) {  // source at psi_{n-1} (src/costs.py:341-353), formed by the source warp
        mb_wait(&sfull[slot], use & 1);
        if (i < d) cur[0][0] = cadd(cur[0][0], ws_sm[L.lring + slot * d + i]);
        team_sync(tm.id);
        if (tl == 0) mb_arrive(&sempty[slot]);
        if (trc && tl == 0) trc[3] = clock64();
      } else if (kind == LGK_GATE_RUN) {
        if (i < d) cur[0][0] = cadd(cur[0][0], cmul(ws_sm[tg + i], tr));
      }
    }
  } else if (rank >= 1 && rank < (unsigned)(1 + I) && threadIdx.x >= 64 && threadIdx.x < 96) {
    // ---------------- source warp of L_s: Omega psi_{n-1} or phi <phi|psi_{n-1}> as soon as P delivers
    // psi_{n-1}; the costate team adds it after its chain (same operation order as src/costs.py:341-353)
    const int si = rank - 1;
    const int sidx = E.set_spec[set][si];
    const int kind = E.spec[sidx].kind;
    if (kind == LGK_STATE_PEN || kind == LGK_STATE_RUN) {
      const int tg = L.tgt + si * d;
      const int pen = L.pen + si * Wp * d;
      const int* pc = pcol + si * Wp * d;
      const int lane = threadIdx.x - 64;
      for (int it = 0; it + 1 < N; ++it) {  // lambda(n-1) needs the source for n = N-1 .. 1
        const int slot = it % RING, use = it / RING;
        if (use > 0) mb_wait(&sempty[slot], (use - 1) & 1);
        if (lane == 0) mb_expect_tx(&pfull[slot], (unsigned)d * 16u);
        mb_wait(&pfull[slot], use & 1);
        const int psi = L.ring + slot * d;
        if (kind == LGK_STATE_RUN) {
          double2 o = make_double2(0.0, 0.0);
          for (int r = lane; r < d; r += 32) o = cadd(o, cdot(ws_sm[tg + r], ws_sm[psi + r]));
          o = warp_sum(o);
          for (int r = lane; r < d; r += 32) ws_sm[L.lring + slot * d + r] = cmul(ws_sm[tg + r], o);
        } else {
          for (int r = lane; r < d; r += 32) ws_sm[L.lring + slot * d + r] = pen_row(d, Wp, pen, pc, r, psi);
        }
        __syncwarp();
        if (lane == 0) cl_arrive_relaxed(cl_map(&pempty[slot], 0));
        mb_arrive(&sfull[slot]);
      }
    }
  }
  __syncthreads();
  cl_sync();  // no CTA leaves while its shared memory may still be addressed remotely
}

extern "C" int lg_ws_layout_words(int d, int nteams, int I, int Wp, int extra_bars, int dense) {
  return ws_layout(d, nteams, I, Wp, extra_bars, dense).words;
}

// W > 0: sparse ELL width.  W <= 0: dense rows, -W = register row width DM (lg_ws_dense_width).
extern "C" void* lg_ws_kernel(int backward, int W, int rpl) {
  (void)rpl;
#define LG_WSD(DM_) \
  if (W == -DM_)                                                                                                 \
    return backward == 3 ? (void*)lg_k_ws_forward_batch<DM_, 1>                                                  \
                         : backward == 2 ? (void*)lg_k_wsc_backward<DM_, 1> : (backward ? nullptr : (void*)lg_k_ws_forward<DM_, 1>);
  LG_WSD(8) LG_WSD(16) LG_WSD(32) LG_WSD(40) LG_WSD(48) LG_WSD(64)
#undef LG_WSD
#define LG_WS(W_)                                                                               \
  if (W == W_)                                                                                  \
    return backward == 3 ? (void*)lg_k_ws_forward_batch<W_, 0>                                  \
                         : backward == 2 ? (void*)lg_k_wsc_backward<W_, 0>                      \
                         : (backward ? (void*)lg_k_ws_backward<W_> : (void*)lg_k_ws_forward<W_, 0>);
  LG_WS(1) LG_WS(2) LG_WS(3) LG_WS(4) LG_WS(5) LG_WS(6) LG_WS(7) LG_WS(8) LG_WS(9)
#undef LG_WS
  return nullptr;
}
