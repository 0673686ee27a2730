// Cluster sweep engine for mid/large sparse problems (configs 3 and 4).
//
// One thread-block cluster per trajectory.  Rows are renumbered by reverse
// Cuthill-McKee (host) so the union pattern of H_s and the controls is a
// narrow band (c3: bandwidth 200 -> 4, c4: 2000 -> 15); CTA rank r of the
// cluster owns renumbered rows [r R, (r+1) R) and keeps every term vector as a
// window [r R - HW, (r+1) R + HW) in shared memory.  Taylor terms
// (src/expm.py:345-350) run in ghost-zone blocks of up to Q terms: after an
// exchange the window is valid everywhere, every sub-term computes the own rows
// plus E = HW - H ghost rows per side (the valid region shrinks by the
// bandwidth H per sub-term; CTA barrier between sub-terms), and the block's
// last sub-term stores the own rows, pushes the HW boundary rows into the
// neighbours' halo slots over DSMEM (st.shared::cluster) and meets at ONE
// cluster barrier.  Q = 1 (E = 0) is one cluster barrier per term.  Blocks
// never span a scaling round, so a block input is always either a Taylor term
// or the round's starting vector.  Exchange buffers alternate between blocks
// (a fast neighbour may push the next block's halo while this CTA still reads
// the current one); sub-term scratch buffers are private.  Operator rows live
// in registers (exact ELL width W); the step table is not permuted -- a thread
// gathers its original row perm[i'].  Reductions (overlaps, <lambda|dU psi>)
// are CTA trees whose partials every CTA pushes to every rank; each rank then
// sums them in rank order (identical, deterministic result everywhere).
#pragma once
#include "lg_types.h"

namespace {

extern __shared__ __align__(16) double2 cl_sm[];

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cdot(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
// p += a x with the a.y terms in q (four independent chains), or all in p when split is false
__device__ __forceinline__ void cmac(double2& p, double2& q, double2 a, double2 x, bool split = true) {
  p.x = fma(a.x, x.x, p.x);
  p.y = fma(a.x, x.y, p.y);
  if (split) {
    q.x = fma(-a.y, x.y, q.x);
    q.y = fma(a.y, x.x, q.y);
  } else {
    p.x = fma(-a.y, x.y, p.x);
    p.y = fma(a.y, x.x, p.y);
  }
}
__device__ __forceinline__ double2 warp_sum(double2 v) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}
__device__ __forceinline__ unsigned smaddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned cl_map_u(unsigned a, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ unsigned cl_map(const void* p, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smaddr(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void cl_st(unsigned addr, double2 v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};\n" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}
// Halo push of a block's last term: st.async into the neighbour's window, counted on
// the neighbour's mbarrier of that buffer (complete_tx) -- no release fence.
__device__ __forceinline__ void cl_st_async(unsigned addr, double2 v, unsigned mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(addr),
               "d"(v.x), "d"(v.y), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void mb_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smaddr(b)), "r"(count));
}
__device__ __forceinline__ void mb_arm(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smaddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smaddr(b)),
      "r"(parity)
      : "memory");
}
// Wait for a phase completed by another CTA's release-arrive (acquire at cluster scope).
__device__ __forceinline__ void mb_wait_cluster(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WC_%=:\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n @!p bra WC_%=;\n}\n" ::"r"(
          smaddr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
  return r;
}

// Two-phase backward hand-off.  The adjoint sweep publishes, per (group, cluster rank), how many
// steps it has stored (after a CTA barrier, one release store at gpu scope: cumulative over the
// CTA's stores); an item CTA waits for its own rank's count with an acquire load.  Items come from
// an atomic counter (rank 0 fetches, every rank of the cluster gets the index through DSMEM).
__device__ __forceinline__ void bk_publish(const LgEngineArgs& E, int g, unsigned rank, unsigned cs, unsigned steps) {
  __syncthreads();
  if (threadIdx.x == 0)
    asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(E.bk_flag + (long)g * cs + rank), "r"(steps) : "memory");
}
// (watchdog: a wait longer than ~20 s -- the adjoint sweep can no longer be running -- gives up and
// raises the error word after the item counter, which the host turns into LG_CUDA_ERROR; it never hangs)
// An item CTA may own rows of several adjoint CTAs (the item layout can use bigger CTAs), so it
// waits for every adjoint rank of the trajectory: thread t < bk_ranks watches rank t's flag.
__device__ __forceinline__ void bk_wait(const LgEngineArgs& E, int g, unsigned steps) {
  if ((int)threadIdx.x < E.bk_ranks) {
    unsigned v;
    const long long t0 = clock64();
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n"
                   : "=r"(v)
                   : "l"(E.bk_flag + (long)g * E.bk_ranks + threadIdx.x)
                   : "memory");
      if (v >= steps) break;
      if (clock64() - t0 > 40000000000LL) {
        atomicExch(E.bk_next + 1, 1u);
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
}
// adjoint sweep start: one count per cluster (after the cluster's first barrier)
__device__ __forceinline__ void bk_started(const LgEngineArgs& E) {
  if (cl_rank() == 0 && threadIdx.x == 0) atomicAdd(E.bk_next + 2, 1u);
}
// concurrent item kernel: run only if every adjoint cluster is already resident (so no item can wait
// on an adjoint cluster that its own residency keeps off the GPU); otherwise free the SMs at once.
// Rank 0 decides after a short spin and tells the other ranks through DSMEM.
__device__ __forceinline__ bool bk_may_run(const LgEngineArgs& E, unsigned* slot) {
  if (!E.bk_conc) return true;
  if (cl_rank() == 0 && threadIdx.x == 0) {
    unsigned v = 0, ok = 0;
    const long long t0 = clock64();
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(E.bk_next + 2) : "memory");
      if (v >= (unsigned)E.n_groups) {
        ok = 1;
        break;
      }
      if (clock64() - t0 > 200000LL) break;  // ~100 us
      __nanosleep(128);
    }
    for (unsigned r = 0; r < cl_size(); ++r)
      asm volatile("st.shared::cluster.u32 [%0], %1;\n" ::"r"(cl_map(slot, r)), "r"(ok) : "memory");
  }
  cl_sync();
  const bool ok = *slot != 0;
  cl_sync();
  return ok;
}

// Per-CTA context.  Thread li handles renumbered row gi = g0 - E + li (window
// position li + H); own rows are li in [E, E + R).
struct Cl {
  int d, R, H, E, HW, Q, T, WIN, rank, CS, li, g0;  // g0 = rank * R; HW = E + H; WIN = R + 2 HW; T = threads
  bool slot;                            // thread holds one of the R own rows (li - E in [0, R))
  bool own;                             // ... and that row exists (gi < d)
  bool ex;                              // thread's row exists (0 <= gi < d; own or ghost)
  bool act;                             // thread maps to a window row (li < R + 2E; the rest is warp padding)
  int gi;                               // renumbered global row of this thread
  int orig;                             // original row perm[gi]
  int red, rt, tb0, tb1, tb2, tb3, st, nx;  // smem offsets (double2): exchange buffers tb0/tb1, scratch tb2/tb3
  int Cmax, Cst, Wc;
  int acs, accs;                        // staged control rows: double2 [Kc][Wc][T] and int [Kc][Wc][T] (-1: not staged)
  int cols;                             // packed slot columns, unsigned [(W+3)/4][T]
  int mb;                               // mbarriers (8-byte words after the layout): [0,1] exchange buffers tb0 / tb1,
                                        // split backward: [2] group barrier, [3, 3+HR) hand-off full, [3+HR, 3+2HR) empty
  mutable unsigned ph;                  // parity bits of the next phase of mb[0], mb[1]
  // split backward (adjoint / aux CTA groups of one cluster; otherwise the group is the cluster)
  bool split;
  int group, base;                      // group index, cluster rank of the group's rank 0 (c.rank, c.CS are group-local)
  mutable unsigned gph;                 // parity of the group barrier's next phase
  int hring;                            // hand-off ring [HR][Cst][R] (double2), after the mbarriers
};
constexpr int LG_CL_HR = 2;  // hand-off ring depth (split backward)

// SMALL: the CTA has <= 256 threads (few rows per CTA, latency-bound), so the
// full register file is available: gather offsets live in registers and every
// gather of a sub-term is issued before its first store.
template <int W, int MAXC, bool SMALL>
struct ClRegs {
  double2 a[W];
  double2 cur[MAXC];
  int go[SMALL ? W : 1];  // SMALL: window offset (H + li + rel) of slot w
};
// Column of slot w relative to the own row (signed 8-bit, four per word) lives in a
// thread-private shared table [(W+3)/4][R]: kept in registers it spills (L1 is
// almost all carved out to shared memory, so spills go to L2).
__device__ __forceinline__ int slot_col(unsigned word, int w, int base) {
  return base + (int)(signed char)((word >> ((w & 3) * 8)) & 0xffu);
}

// Store a value of own row oi = li - E into column `colo` of window buffer `buf`
// locally and into the halo slots of the neighbours that need it (HW rows each).
__device__ __forceinline__ void put(const Cl& c, int buf, int colo, double2 v) {
  const int off = buf + colo * c.WIN, oi = c.li - c.E;
  cl_sm[off + c.H + c.li] = v;
  if (oi < c.HW && c.rank > 0) cl_st(cl_map(&cl_sm[off + c.R + c.HW + oi], c.base + c.rank - 1), v);
  if (oi >= c.R - c.HW && c.rank + 1 < c.CS) cl_st(cl_map(&cl_sm[off + oi - c.R + c.HW], c.base + c.rank + 1), v);
}
__device__ __forceinline__ unsigned long long* cl_mb(const Cl& c, int k) {
  return reinterpret_cast<unsigned long long*>(cl_sm + c.mb) + k;
}
// Same for a block's last term inside a chain: the halo rows travel by st.async and are
// counted on the neighbour's mbarrier of buffer yi (see exchange_begin / exchange_end).
__device__ __forceinline__ void put_async(const Cl& c, int buf, int yi, int colo, double2 v) {
  const int off = buf + colo * c.WIN, oi = c.li - c.E;
  cl_sm[off + c.H + c.li] = v;
  const unsigned mb = smaddr(cl_mb(c, yi));
  if (oi < c.HW && c.rank > 0)
    cl_st_async(cl_map(&cl_sm[off + c.R + c.HW + oi], c.base + c.rank - 1), v, cl_map_u(mb, c.base + c.rank - 1));
  if (oi >= c.R - c.HW && c.rank + 1 < c.CS)
    cl_st_async(cl_map(&cl_sm[off + oi - c.R + c.HW], c.base + c.rank + 1), v, cl_map_u(mb, c.base + c.rank + 1));
}
// Block exchange over the neighbour-only mbarriers (replaces one cluster barrier per
// block).  Buffer yi's mbarrier is armed (one arrival + the expected halo bytes) when
// a block that writes yi starts; neighbours' pushes may land before the arm (the
// transaction count then runs negative within the phase).  The block ends with a CTA
// barrier (own rows) and the wait for the halo bytes.  Write-after-read on the two
// exchange buffers needs no handshake: a neighbour overwrites buffer yi only after
// receiving this CTA's halo of the following block, i.e. after this CTA's reads of yi.
__device__ __forceinline__ void exchange_begin(const Cl& c, int yi, int C) {
  if (threadIdx.x == 0)
    mb_arm(cl_mb(c, yi), 16u * (unsigned)(c.HW * C) * ((c.rank > 0 ? 1u : 0u) + (c.rank + 1 < c.CS ? 1u : 0u)));
}
// Barrier over the CTA's group: the cluster barrier when the group is the whole cluster; in the
// split backward every CTA's threads 0..CS-1 release-arrive on the group members' barrier
// mbarriers (count CS) after a CTA barrier, and the CTA waits on its own (acquire, cluster scope).
__device__ __forceinline__ void gsync(const Cl& c) {
  if (!c.split) {
    cl_sync();
    return;
  }
  __syncthreads();
  unsigned long long* gb = cl_mb(c, 2);
  if ((int)threadIdx.x < c.CS)
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(
                     cl_map_u(smaddr(gb), c.base + threadIdx.x))
                 : "memory");
  asm volatile(
      "{\n .reg .pred p;\n GW_%=:\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n @!p bra GW_%=;\n}\n" ::"r"(
          smaddr(gb)),
      "r"(c.gph & 1u)
      : "memory");
  c.gph ^= 1u;
}
__device__ __forceinline__ void exchange_end(const Cl& c, int yi) {
  __syncthreads();
  mb_wait(cl_mb(c, yi), (c.ph >> yi) & 1u);
  c.ph ^= 1u << yi;
}

// Cluster-wide deterministic sum of nv values (per thread partials).
template <int NV>
__device__ void cl_reduce(const Cl& c, double2 (&v)[NV], int nv) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  double2* scr = cl_sm + c.red;                 // [NV][32] per-warp partials
  double2* box = cl_sm + c.red + NV * 32;       // [NV][CS] per-rank partials (pushed)
  for (int q = 0; q < nv; ++q) {
    double2 s = warp_sum(v[q]);
    if (l == 0) scr[q * 32 + w] = s;
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    const int q = threadIdx.x;
    double2 s = make_double2(0.0, 0.0);
    for (int k = 0; k < nw; ++k) s = cadd(s, scr[q * 32 + k]);
    for (int r = 0; r < c.CS; ++r) cl_st(cl_map(&box[q * c.CS + c.rank], c.base + r), s);
  }
  gsync(c);
  for (int q = 0; q < nv; ++q) {
    double2 s = make_double2(0.0, 0.0);
    for (int r = 0; r < c.CS; ++r) s = cadd(s, box[q * c.CS + r]);
    v[q] = s;
  }
  gsync(c);  // box may be rewritten by the next reduction
}

// One Taylor chain over C columns of the window buffers, input staged in tb0
// (with halos) and in cur.  mode 1: columns [0, G) tops of channels gch[], G = bottom.
// Split-phase cluster barrier per term: rows that neither read a halo slot nor
// feed a neighbour ("interior") are computed before waiting for the previous
// term's barrier; boundary rows after it, then pushed, then arrive.
// fin: last sub-term of a block -- own rows only, stored with put(); otherwise
// every thread (own and ghost rows) stores its term locally.
template <int W, int MAXC, bool SMALL>
__device__ __forceinline__ void term_row(const LgEngineArgs& E, const Cl& c, ClRegs<W, MAXC, SMALL>& R, int C, int mode, int G,
                                         int X, int Y, double r, bool last, bool fin, int yi, int vt) {
  // Ghost rows that fall out of the valid region after sub-term vt are stored as zeros: the
  // ELL pad slots (value 0) of a valid row may point up to H + 7 rows away (cl_color_slots
  // reuses another row's address), and garbage left to grow there could reach Inf (0 * Inf).
  const int pos = c.H + c.li;
  const bool keep = pos >= vt * c.H && pos < c.WIN - vt * c.H;
  // packed slot columns: loaded once per term (a store to the window between columns would
  // otherwise make the compiler reload them for every column)
  unsigned cw[(W + 3) / 4];
  {
    const unsigned* ct = reinterpret_cast<const unsigned*>(cl_sm + c.cols) + c.li;
#pragma unroll
    for (int k = 0; k < (W + 3) / 4; ++k) cw[k] = ct[k * c.T];
  }
#pragma unroll
  for (int q = 0; q < MAXC; ++q) {
    if (q >= C) break;
    double2 p = make_double2(0.0, 0.0), pq = make_double2(0.0, 0.0);
    if (c.ex && (c.slot || !fin)) {
      const int xc = X + q * c.WIN + c.H + c.li;
      double2 p1 = make_double2(0.0, 0.0), pq1 = make_double2(0.0, 0.0);
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const double2 x = cl_sm[slot_col(cw[w >> 2], w, xc)];
        if ((w & 1) && MAXC <= 3)
          cmac(p1, pq1, R.a[w], x);
        else
          cmac(p, pq, R.a[w], x);
      }
      p = cadd(p, p1);
      pq = cadd(pq, pq1);
      if (mode == 1 && q < G) {
        const int koff = reinterpret_cast<const int*>(cl_sm + c.rt + 64)[q];
        if (c.acs >= 0) {
          const int bc = X + G * c.WIN;
          const double2* ac = cl_sm + c.acs + koff + c.li;
          const int* acc = reinterpret_cast<const int*>(cl_sm + c.accs) + koff + c.li;
          for (int w = 0; w < c.Wc; ++w) cmac(p, pq, ac[w * c.T], cl_sm[bc + acc[w * c.T]]);
        } else {
          const int bc = X + G * c.WIN - c.g0 + c.HW;
          const double2* ac = E.Ac + koff + c.orig;
          const int* acc = E.cl_accols + koff + c.gi;
          for (int w = 0; w < c.Wc; ++w) cmac(p, pq, __ldg(ac + w * c.d), cl_sm[bc + __ldg(acc + w * c.d)]);
        }
      }
    }
    const double2 tt = make_double2((p.x + pq.x) * r, (p.y + pq.y) * r);
    R.cur[q] = cadd(R.cur[q], tt);
    if (fin) {
      if (c.slot) put_async(c, Y, yi, q, last ? R.cur[q] : tt);
    } else if (c.act) {
      cl_sm[Y + q * c.WIN + c.H + c.li] = keep ? tt : make_double2(0.0, 0.0);
    }
  }
}

// SMALL variant of term_row with the column count NC and the mode known at compile
// time (MODE 1: columns [0, NC-1) are aux tops, NC-1 the bottom): all gathers of
// the sub-term are issued before its first store.
template <int W, int MAXC, int NC, int MODE>
__device__ __forceinline__ void sub_term(const LgEngineArgs& E, const Cl& c, ClRegs<W, MAXC, true>& R, int X, int Y,
                                         double r, bool last, bool fin, int yi, int vt) {
  const int pos = c.H + c.li;  // see term_row
  const bool keep = pos >= vt * c.H && pos < c.WIN - vt * c.H;
  double2 tt[NC];
  if (c.ex && (c.slot || !fin)) {
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      double2 p = make_double2(0.0, 0.0), pq = make_double2(0.0, 0.0);
      double2 p1 = make_double2(0.0, 0.0), pq1 = make_double2(0.0, 0.0);
      const double2* xw = cl_sm + X + q * c.WIN;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        if (w & 1)
          cmac(p1, pq1, R.a[w], xw[R.go[w]]);
        else
          cmac(p, pq, R.a[w], xw[R.go[w]]);
      }
      if (MODE == 1 && q < NC - 1) {
        const int koff = reinterpret_cast<const int*>(cl_sm + c.rt + 64)[q];
        if (c.acs >= 0) {
          const double2* bw = cl_sm + X + (NC - 1) * c.WIN;
          const double2* ac = cl_sm + c.acs + koff + c.li;
          const int* acc = reinterpret_cast<const int*>(cl_sm + c.accs) + koff + c.li;
          for (int w = 0; w < c.Wc; ++w) cmac(p1, pq1, ac[w * c.T], bw[acc[w * c.T]]);
        } else {
          const double2* bw = cl_sm + X + (NC - 1) * c.WIN - c.g0 + c.HW;
          const double2* ac = E.Ac + koff + c.orig;
          const int* acc = E.cl_accols + koff + c.gi;
          for (int w = 0; w < c.Wc; ++w) cmac(p1, pq1, __ldg(ac + w * c.d), bw[__ldg(acc + w * c.d)]);
        }
      }
      p = cadd(p, p1);
      pq = cadd(pq, pq1);
      tt[q] = make_double2((p.x + pq.x) * r, (p.y + pq.y) * r);
    }
  } else {
#pragma unroll
    for (int q = 0; q < NC; ++q) tt[q] = make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    R.cur[q] = cadd(R.cur[q], tt[q]);
    if (fin) {
      if (c.slot) put_async(c, Y, yi, q, last ? R.cur[q] : tt[q]);
    } else if (c.act) {
      cl_sm[Y + q * c.WIN + c.H + c.li] = keep ? tt[q] : make_double2(0.0, 0.0);
    }
  }
}

template <int W, int MAXC, int NC, int MODE>
__device__ __forceinline__ void chain_nc(const LgEngineArgs& E, const Cl& c, ClRegs<W, MAXC, true>& R, int m, int s) {
  int X = c.tb0, Y = c.tb1, yi = 1;
  for (int round = 0; round < s; ++round)
    for (int j0 = 1; j0 <= m; j0 += c.Q) {
      const int b = min(c.Q, m - j0 + 1);
      exchange_begin(c, yi, NC);
      for (int t = 1; t <= b; ++t) {
        const int j = j0 + t - 1;
        const bool fin = t == b;
        const int src = t == 1 ? X : ((t & 1) ? c.tb2 : c.tb3);
        const int dst = fin ? Y : ((t & 1) ? c.tb3 : c.tb2);
        sub_term<W, MAXC, NC, MODE>(E, c, R, src, dst, cl_sm[c.rt + j - 1].x, j == m, fin, yi, t);
        if (!fin) __syncthreads();
      }
      exchange_end(c, yi);
      const int t_ = X;
      X = Y;
      Y = t_;
      yi ^= 1;
    }
}

// Input staged in tb0 (own rows + pushed halos) and in cur; result in cur.
template <int W, int MAXC, bool SMALL>
__device__ __forceinline__ void chain(const LgEngineArgs& E, const Cl& c, ClRegs<W, MAXC, SMALL>& R, int C, int mode, int G,
                                      int m, int s, double sgn) {
  if (threadIdx.x < m) cl_sm[c.rt + threadIdx.x].x = sgn * (1.0 / (double)(s * (threadIdx.x + 1)));
  gsync(c);  // staged input (incl. pushed halos) and the 1/(s j) table published
  if constexpr (SMALL) {
#define LG_NC(n)                                                            \
  if constexpr (n <= MAXC)                                                  \
    if (C == n) {                                                           \
      if (mode == 0)                                                        \
        chain_nc<W, MAXC, n, 0>(E, c, R, m, s);                             \
      else if constexpr (n >= 2)                                            \
        chain_nc<W, MAXC, n, 1>(E, c, R, m, s);                             \
    }
    LG_NC(1) LG_NC(2) LG_NC(3) LG_NC(4) LG_NC(5) LG_NC(6) LG_NC(7) LG_NC(8)
#undef LG_NC
  } else {
  int X = c.tb0, Y = c.tb1, yi = 1;  // exchange buffers: block input, block output
  for (int round = 0; round < s; ++round)
    for (int j0 = 1; j0 <= m; j0 += c.Q) {
      const int b = min(c.Q, m - j0 + 1);
      exchange_begin(c, yi, C);
      for (int t = 1; t <= b; ++t) {
        const int j = j0 + t - 1;
        const bool fin = t == b;
        const int src = t == 1 ? X : ((t & 1) ? c.tb2 : c.tb3);
        const int dst = fin ? Y : ((t & 1) ? c.tb3 : c.tb2);
        const double r = cl_sm[c.rt + j - 1].x;
        term_row<W, MAXC, SMALL>(E, c, R, C, mode, G, src, dst, r, j == m, fin, yi, t);
        if (!fin) __syncthreads();  // sub-term visible to the CTA (ghost rows are local)
      }
      exchange_end(c, yi);  // Y (own rows + halos) complete here
      const int t_ = X;
      X = Y;
      Y = t_;
      yi ^= 1;
    }
  }
  gsync(c);  // every CTA done reading its windows: the caller may stage the next chain's input
}

template <int W, int MAXC, bool SMALL>
__device__ __forceinline__ void load_row(const LgEngineArgs& E, const Cl& c, int n, ClRegs<W, MAXC, SMALL>& R) {
  const double2* src = E.A + (long)n * W * E.d;
#pragma unroll
  for (int w = 0; w < W; ++w) R.a[w] = c.ex ? src[(long)E.cl_slot[(long)w * E.d + c.gi] * E.d + c.orig] : make_double2(0.0, 0.0);
}
template <int W, int MAXC, bool SMALL>
__device__ __forceinline__ void load_cols(const LgEngineArgs& E, const Cl& c, ClRegs<W, MAXC, SMALL>& R) {
  unsigned* ct = reinterpret_cast<unsigned*>(cl_sm + c.cols) + c.li;
#pragma unroll
  for (int k = 0; k < (W + 3) / 4; ++k) {
    unsigned v = 0;
#pragma unroll
    for (int w = 4 * k; w < 4 * k + 4 && w < W; ++w) {
      const int rel = c.ex ? E.cl_cols[w * E.d + c.gi] - c.gi : 0;  // |rel| <= H <= 127 (host check)
      v |= ((unsigned)rel & 0xffu) << ((w & 3) * 8);
      if constexpr (SMALL) R.go[w] = c.H + c.li + rel;
    }
    ct[k * c.T] = v;
  }
}

__device__ __forceinline__ Cl make_cl(const LgEngineArgs& E, int Cmax, int Cst, int W, bool split = false) {
  Cl c;
  c.d = E.d;
  c.split = split;
  c.CS = (int)cl_size();
  c.rank = (int)cl_rank();
  c.group = 0;
  c.base = 0;
  c.gph = 0;
  if (split) {  // two groups of CS / 2 CTAs over the same row partition
    c.CS /= 2;
    c.group = c.rank / c.CS;
    c.base = c.group * c.CS;
    c.rank -= c.base;
  }
  c.R = E.cl_R;
  c.H = E.cl_H;
  c.Q = E.cl_Q;
  c.E = E.cl_E;
  c.HW = c.E + c.H;
  c.T = blockDim.x;
  c.WIN = c.R + 2 * c.HW;
  c.g0 = c.rank * c.R;
  c.li = threadIdx.x;
  c.gi = c.g0 - c.E + c.li;
  c.slot = c.li >= c.E && c.li < c.E + c.R;
  c.act = c.li < c.R + 2 * c.E;
  c.ex = c.act && c.gi >= 0 && c.gi < c.d;
  c.own = c.slot && c.ex;
  c.orig = c.ex ? E.cl_perm[c.gi] : 0;
  c.Cmax = Cmax;
  c.Cst = Cst;
  c.Wc = E.Wc;
  int o = 0;
  c.red = o;
  o += 16 * 32 + 16 * 16;
  c.rt = o;  // [64] 1/(s j) table, then [16] int channel offsets of the aux top columns
  o += 72;
  c.tb0 = o;
  o += Cmax * c.WIN;
  c.tb1 = o;
  o += Cmax * c.WIN;
  c.tb2 = c.tb3 = c.tb1;  // Q == 1: no sub-term scratch
  if (c.Q > 1) {
    c.tb2 = o;
    o += Cmax * c.WIN;
    c.tb3 = o;
    o += Cmax * c.WIN;
  }
  c.cols = o;
  o += ((W + 3) / 4 * c.T + 3) / 4;
  c.acs = c.accs = -1;
  if (E.cl_acs) {
    const int n = E.Kc * E.Wc * c.T;
    c.acs = o;
    o += n;
    c.accs = o;
  }
  c.st = c.nx = 0;
  c.mb = lg_cl_mb_word(c.R, c.H, c.Q, c.E, Cmax, W, E.cl_acs ? E.Kc * E.Wc : 0);
  c.ph = 0;
  c.hring = c.mb + 4;  // after 8 mbarrier words (exchange 2, group 1, hand-off 2 x HR)
  return c;
}

// ELL apply of the (renumbered) penalty operator to a window column.
__device__ __forceinline__ double2 pen_apply(const LgEngineArgs& E, const LgSpecDev& sp, const Cl& c, int xwin) {
  double2 p = make_double2(0.0, 0.0), q = make_double2(0.0, 0.0);
  for (int w = 0; w < sp.pen_W; ++w) {
    const long k = (long)w * c.d + c.orig;
    const int j = E.cl_inv[sp.pen_cols[k]] - c.g0 + c.HW;
    cmac(p, q, sp.pen_vals[k], cl_sm[xwin + j]);
  }
  return cadd(p, q);
}

}  // namespace

// ------------------------------------------------------------------------------------------ forward
template <int W, int MAXC, bool SMALL>
__device__ __forceinline__ void cl_forward_body(const LgEngineArgs& E) {
  const int g = blockIdx.x / (int)cl_size();
  const int set = E.grp_set[g], t0 = E.grp_t0[g], trel = t0 - E.set_t0[set];
  const int I = E.set_nspec[set], Kc = E.Kc, N = E.N;
  const int cst = 1 + E.cta_Imax, cmax = (Kc + 1) > cst ? (Kc + 1) : cst;
  Cl c = make_cl(E, cmax, cst, W);
  ClRegs<W, MAXC, SMALL> R;
  load_cols<W, MAXC, SMALL>(E, c, R);
  // zero everything up to the end of the window buffers (pad gathers may read a few rows past a
  // window edge, into the neighbouring column or the tables in front of tb0)
  for (int q = threadIdx.x; q < c.tb0 + (c.Q > 1 ? 4 : 2) * cmax * c.WIN; q += blockDim.x)
    cl_sm[q] = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    mb_init(cl_mb(c, 0), 1);
    mb_init(cl_mb(c, 1), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  cl_sync();
  const double2 psi0 = c.own ? E.psi0[(long)t0 * c.d + c.orig] : make_double2(0.0, 0.0);
  double2 psi = psi0;
  int4 pln = E.plan[0];
  double runacc[LG_MAX_SPECS];
  for (int q = 0; q < LG_MAX_SPECS; ++q) runacc[q] = 0.0;
  for (int n = 0; n < N; ++n) {
    const int4 pl = pln;
    load_row<W, MAXC, SMALL>(E, c, n, R);
    if (n + 1 < N) pln = E.plan[(long)(n + 1) * (Kc + 1)];
    if (c.slot) put(c, c.tb0, 0, psi);
    R.cur[0] = psi;
    chain<W, MAXC, SMALL>(E, c, R, 1, 0, 0, pl.x, pl.y, 1.0);
    psi = R.cur[0];
    // per-step scalars: the chain's result is in the window of the last-written buffer;
    // re-stage psi_n into tb0 for the penalty operator (needs neighbours' rows)
    bool anyq = false;
    for (int si = 0; si < I; ++si) {
      const int kind = E.spec[E.set_spec[set][si]].kind;
      anyq |= kind == LGK_STATE_PEN || kind == LGK_STATE_RUN || kind == LGK_GATE_RUN || n == N - 1;
    }
    if (!anyq) continue;
    bool anypen = false;
    for (int si = 0; si < I; ++si) anypen |= E.spec[E.set_spec[set][si]].kind == LGK_STATE_PEN;
    if (anypen) {
      if (c.slot) put(c, c.tb0, 0, psi);
      cl_sync();
    }
    double2 v[LG_MAX_SPECS];
    for (int si = 0; si < LG_MAX_SPECS; ++si) v[si] = make_double2(0.0, 0.0);
    if (c.own)
      for (int si = 0; si < I; ++si) {
        const LgSpecDev& sp = E.spec[E.set_spec[set][si]];
        if (sp.kind == LGK_STATE_PEN)
          v[si] = cdot(psi, pen_apply(E, sp, c, c.tb0));
        else if (sp.kind == LGK_STATE_INF)
          v[si] = cdot(psi, sp.tgt[(long)trel * c.d + c.orig]);
        else
          v[si] = cdot(sp.tgt[(long)trel * c.d + c.orig], psi);
      }
    cl_reduce<LG_MAX_SPECS>(c, v, I);
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
  if (c.own) E.psiN[(long)t0 * c.d + c.orig] = psi;
  cl_sync();
}

template <int W, int MAXC, bool SMALL>
__global__ void __launch_bounds__(SMALL ? 256 : 640, 1) lg_k_cl_forward(const __grid_constant__ LgEngineArgs E) {
  cl_forward_body<W, MAXC, SMALL>(E);
}
// line-search batch: candidate field blockIdx.y (lg_cost_batch)
template <int W, int MAXC, bool SMALL>
__global__ void __launch_bounds__(SMALL ? 256 : 640, 1) lg_k_cl_forward_batch(const LgEngineArgs* __restrict__ EA) {
  cl_forward_body<W, MAXC, SMALL>(EA[blockIdx.y]);
}

// Derivative products of step n (src/costs.py:328-339): per channel group with a common aux plan,
// the aux chain [0 ... 0 | psi_{n-1}] and <lambda_s(n)|top_k> into ip.
template <int W, int MAXC, bool SMALL>
__device__ __forceinline__ void aux_products(const LgEngineArgs& E, const Cl& c, ClRegs<W, MAXC, SMALL>& R, int n,
                                             int set, int t0, double2 psip, const double2 (&lamc)[LG_MAX_SPECS]) {
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
    // stage [0 ... 0 | psi_{n-1}]
    if (c.slot) {
      for (int q = 0; q < G; ++q) put(c, c.tb0, q, make_double2(0.0, 0.0));
      put(c, c.tb0, G, psip);
    }
#pragma unroll
    for (int q = 0; q < MAXC; ++q) R.cur[q] = q == G ? psip : make_double2(0.0, 0.0);
    if (threadIdx.x < G)  // channel offsets of the top columns (read by chain() after its cluster barrier)
      reinterpret_cast<int*>(cl_sm + c.rt + 64)[threadIdx.x] =
          gch[threadIdx.x] * E.Wc * (c.acs >= 0 ? c.T : c.d);
    chain<W, MAXC, SMALL>(E, c, R, G + 1, 1, G, pk.x, pk.y, 1.0);
    double2 v[16];
    const int nv = I * G;
    for (int q = 0; q < 16; ++q) v[q] = make_double2(0.0, 0.0);
    if (c.own)
      for (int gi = 0; gi < G; ++gi)
        for (int si = 0; si < I; ++si) {
          double2 dd = make_double2(0.0, 0.0);
#pragma unroll
          for (int q = 0; q < MAXC; ++q)
            if (q == gi) dd = R.cur[q];
          v[gi * I + si] = cdot(lamc[si], dd);
        }
    cl_reduce<16>(c, v, nv);
    if (c.rank == 0 && threadIdx.x == 0)
      for (int gi = 0; gi < G; ++gi)
        for (int si = 0; si < I; ++si) {
          const int sidx = E.set_spec[set][si];
          E.ip[(((long)n * E.n_specs + sidx) * Kc + gch[gi]) * E.T_total + t0] = v[gi * I + si];
        }
  }
}

// ------------------------------------------------------------------------------------------ backward
// SPLIT (SMALL only): the cluster's CTAs form two groups over the same row partition -- group 0
// runs the adjoint chain and the costates, group 1 the aux (derivative) chains and the inner
// products of step n while group 0 already works on step n - 1.  psi_{n-1} and lambda_s(n) go
// from each group-0 CTA to its group-1 partner through a hand-off ring (st.async + mbarriers).
// STORE (two-phase backward, not with SPLIT): the adjoint sweep only -- psi_{n-1} and lambda_s(n)
// of every step go to HBM (E.bk_psi / E.bk_lam, renumbered own rows), and lg_k_cl_aux runs the
// derivative products as independent (step, trajectory) items on every resident cluster.
template <int W, int MAXC, bool SMALL, bool SPLIT, bool STORE>
__device__ __forceinline__ void cl_backward_body(const LgEngineArgs& E) {
  const int g = blockIdx.x / (int)cl_size();
  const int set = E.grp_set[g], t0 = E.grp_t0[g], trel = t0 - E.set_t0[set];
  const int I = E.set_nspec[set], Kc = E.Kc, N = E.N;
  const int cst = 1 + E.cta_Imax, cmax = (Kc + 1) > cst ? (Kc + 1) : cst;
  Cl c = make_cl(E, cmax, cst, W, SPLIT);
  const bool doA = !SPLIT || c.group == 0, doB = (!SPLIT || c.group == 1) && !STORE;
  ClRegs<W, MAXC, SMALL> R;
  load_cols<W, MAXC, SMALL>(E, c, R);
  // zero everything up to the end of the window buffers (pad gathers may read a few rows past a
  // window edge, into the neighbouring column or the tables in front of tb0)
  for (int q = threadIdx.x; q < c.tb0 + (c.Q > 1 ? 4 : 2) * cmax * c.WIN; q += blockDim.x)
    cl_sm[q] = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    mb_init(cl_mb(c, 0), 1);
    mb_init(cl_mb(c, 1), 1);
    if (SPLIT) {
      mb_init(cl_mb(c, 2), c.CS);
      for (int h = 0; h < 2 * LG_CL_HR; ++h) mb_init(cl_mb(c, 3 + h), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (c.acs >= 0)
    for (int kw = 0; kw < Kc * E.Wc; ++kw) {
      cl_sm[c.acs + kw * c.T + c.li] = c.ex ? E.Ac[(long)kw * c.d + c.orig] : make_double2(0.0, 0.0);
      reinterpret_cast<int*>(cl_sm + c.accs)[kw * c.T + c.li] =
          c.ex ? E.cl_accols[(long)kw * c.d + c.gi] - c.g0 + c.HW : c.H + c.li;
    }
  cl_sync();
  if (STORE) bk_started(E);
  // state: psi (column 0) and the costates lambda_s (columns 1 + s), own rows in registers
  double2 psi = c.own ? E.psiN[(long)t0 * c.d + c.orig] : make_double2(0.0, 0.0);
  double2 lam[LG_MAX_SPECS];
  for (int si = 0; si < LG_MAX_SPECS; ++si) lam[si] = make_double2(0.0, 0.0);
  // ---- costate initialisation (src/costs.py:312-321, :457-460)
  if (doA) {
    bool anypen = false, anyrun = false;
    for (int si = 0; si < I; ++si) {
      const int k = E.spec[E.set_spec[set][si]].kind;
      anypen |= k == LGK_STATE_PEN;
      anyrun |= k == LGK_STATE_RUN;
    }
    if (anypen) {
      if (c.slot) put(c, c.tb0, 0, psi);
      gsync(c);
    }
    double2 ov[LG_MAX_SPECS];
    for (int si = 0; si < LG_MAX_SPECS; ++si) ov[si] = make_double2(0.0, 0.0);
    if (anyrun) {
      if (c.own)
        for (int si = 0; si < I; ++si) {
          const LgSpecDev& sp = E.spec[E.set_spec[set][si]];
          if (sp.kind == LGK_STATE_RUN) ov[si] = cdot(sp.tgt[(long)trel * c.d + c.orig], psi);
        }
      cl_reduce<LG_MAX_SPECS>(c, ov, I);
    }
    for (int si = 0; si < I; ++si) {
      const int sidx = E.set_spec[set][si];
      const LgSpecDev& sp = E.spec[sidx];
      double2 v = make_double2(0.0, 0.0);
      if (c.own) {
        if (sp.kind == LGK_STATE_PEN) {
          v = pen_apply(E, sp, c, c.tb0);
        } else {
          const double2 tv = sp.tgt[(long)trel * c.d + c.orig];
          if (sp.kind == LGK_STATE_RUN)
            v = cmul(tv, ov[si]);
          else if (sp.kind == LGK_GATE_RUN)
            v = cmul(tv, E.trsum[(long)sidx * N + N - 1]);
          else
            v = tv;
        }
      }
      lam[si] = v;
    }
    gsync(c);
  }
  int gch[LG_MAX_CHANNELS];
  for (int n = N - 1, it = 0; n >= 0; --n, ++it) {
    const int4* pln = E.plan + (long)n * (Kc + 1);
    const int4 pl = pln[0];
    load_row<W, MAXC, SMALL>(E, c, n, R);
    double2 psip = make_double2(0.0, 0.0);  // psi_{n-1}
    double2 lamn[LG_MAX_SPECS];             // U_n^dagger lambda_s(n)
    double2 lamc[LG_MAX_SPECS];             // lambda_s(n) for the inner products
    for (int si = 0; si < LG_MAX_SPECS; ++si) lamn[si] = lamc[si] = lam[si];
    const int hs = it % LG_CL_HR;
    if (doA) {
      // adjoint chain on [psi | lambda] (src/costs.py:326,342); costates not needed at n == 0
      const int cadj = n > 0 ? 1 + I : 1;
      if (c.slot) {
        put(c, c.tb0, 0, psi);
        for (int si = 0; si < I && n > 0; ++si) put(c, c.tb0, 1 + si, lam[si]);
      }
#pragma unroll
      for (int q = 0; q < MAXC; ++q) R.cur[q] = q == 0 ? psi : (q - 1 < I ? lam[q - 1] : make_double2(0.0, 0.0));
      chain<W, MAXC, SMALL>(E, c, R, cadj, 0, 0, pl.x, pl.y, -1.0);
      psip = R.cur[0];
#pragma unroll
      for (int q = 1; q < MAXC; ++q)
        if (q - 1 < LG_MAX_SPECS) lamn[q - 1] = R.cur[q];
      if (STORE) {  // hand psi_{n-1} and lambda_s(n) to the item kernel
        if (c.own) {
          E.bk_psi[((long)g * N + n) * c.d + c.gi] = psip;
          for (int si = 0; si < I; ++si) E.bk_lam[(((long)g * N + n) * E.cta_Imax + si) * c.d + c.gi] = lam[si];
        }
        bk_publish(E, g, (unsigned)(c.base + c.rank), cl_size(), (unsigned)(N - n));
      }
      if (SPLIT) {  // hand psi_{n-1} and lambda_s(n) to the partner CTA of group 1
        if (it >= LG_CL_HR) mb_wait_cluster(cl_mb(c, 3 + LG_CL_HR + hs), (unsigned)((it / LG_CL_HR) - 1) & 1u);
        if (c.slot) {
          const int oi = c.li - c.E, partner = c.CS + c.rank;
          const unsigned fb = cl_map_u(smaddr(cl_mb(c, 3 + hs)), partner);
          cl_st_async(cl_map(&cl_sm[c.hring + (hs * cst + 0) * c.R + oi], partner), psip, fb);
          for (int si = 0; si < I; ++si)
            cl_st_async(cl_map(&cl_sm[c.hring + (hs * cst + 1 + si) * c.R + oi], partner), lam[si], fb);
        }
      }
    }
    if (doB) {
      if (SPLIT) {  // take psi_{n-1} and lambda_s(n) from the partner, then free the slot
        if (threadIdx.x == 0) mb_arm(cl_mb(c, 3 + hs), 16u * (unsigned)(c.R * (1 + I)));
        mb_wait(cl_mb(c, 3 + hs), (unsigned)(it / LG_CL_HR) & 1u);
        if (c.slot) {
          const int oi = c.li - c.E;
          psip = cl_sm[c.hring + (hs * cst + 0) * c.R + oi];
          for (int si = 0; si < I; ++si) lamc[si] = cl_sm[c.hring + (hs * cst + 1 + si) * c.R + oi];
        }
        __syncthreads();
        if (threadIdx.x == 0)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(
                           cl_map_u(smaddr(cl_mb(c, 3 + LG_CL_HR + hs)), c.rank))
                       : "memory");
      }
    aux_products<W, MAXC, SMALL>(E, c, R, n, set, t0, psip, lamc);
    }  // doB
    if (n == 0) break;
    if (!doA) {
      gsync(c);
      continue;
    }
    // costate sources at psi_{n-1} (src/costs.py:341-353, :474-479)
    bool anypen = false, anyrun = false;
    for (int si = 0; si < I; ++si) {
      const int k = E.spec[E.set_spec[set][si]].kind;
      anypen |= k == LGK_STATE_PEN;
      anyrun |= k == LGK_STATE_RUN;
    }
    if (anypen) {
      if (c.slot) put(c, c.tb0, 0, psip);
      gsync(c);
    }
    double2 ov[LG_MAX_SPECS];
    for (int si = 0; si < LG_MAX_SPECS; ++si) ov[si] = make_double2(0.0, 0.0);
    if (anyrun) {
      if (c.own)
        for (int si = 0; si < I; ++si) {
          const LgSpecDev& sp = E.spec[E.set_spec[set][si]];
          if (sp.kind == LGK_STATE_RUN) ov[si] = cdot(sp.tgt[(long)trel * c.d + c.orig], psip);
        }
      cl_reduce<LG_MAX_SPECS>(c, ov, I);
    }
    for (int si = 0; si < I; ++si) {
      const int sidx = E.set_spec[set][si];
      const LgSpecDev& sp = E.spec[sidx];
      double2 v = lamn[si];
      if (c.own) {
        if (sp.kind == LGK_STATE_PEN)
          v = cadd(v, pen_apply(E, sp, c, c.tb0));
        else if (sp.kind == LGK_STATE_RUN)
          v = cadd(v, cmul(sp.tgt[(long)trel * c.d + c.orig], ov[si]));
        else if (sp.kind == LGK_GATE_RUN)
          v = cadd(v, cmul(sp.tgt[(long)trel * c.d + c.orig], E.trsum[(long)sidx * N + n - 1]));
      }
      lam[si] = v;
    }
    psi = psip;
    gsync(c);
  }
  cl_sync();
}

template <int W, int MAXC, bool SMALL, bool SPLIT = false>
__global__ void __launch_bounds__(SPLIT ? 192 : (SMALL ? 256 : 640), SPLIT ? 2 : 1)
    lg_k_cl_backward(const __grid_constant__ LgEngineArgs E) {
  cl_backward_body<W, MAXC, SMALL, SPLIT, false>(E);
}
template <int W, int MAXC, bool SMALL>
__global__ void __launch_bounds__(SMALL ? 256 : 640, 1) lg_k_cl_adjoint(const __grid_constant__ LgEngineArgs E) {
  cl_backward_body<W, MAXC, SMALL, false, true>(E);
}
// Derivative products as independent items (step n, trajectory group g), item = k * n_groups + g
// with k = N - 1 - n, dealt round-robin to the grid's co-resident clusters; psi_{n-1} and
// lambda_s(n) read from the adjoint sweep's store.
template <int W, int MAXC, bool SMALL>
__global__ void __launch_bounds__(SMALL ? 256 : 640, 1) lg_k_cl_aux(const __grid_constant__ LgEngineArgs E) {
  const int cid = blockIdx.x / (int)cl_size(), ncl = gridDim.x / (int)cl_size();
  const int Kc = E.Kc, N = E.N;
  const int cst = 1 + E.cta_Imax, cmax = (Kc + 1) > cst ? (Kc + 1) : cst;
  Cl c = make_cl(E, cmax, cst, W, false);
  ClRegs<W, MAXC, SMALL> R;
  load_cols<W, MAXC, SMALL>(E, c, R);
  for (int q = threadIdx.x; q < c.tb0 + (c.Q > 1 ? 4 : 2) * cmax * c.WIN; q += blockDim.x)
    cl_sm[q] = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    mb_init(cl_mb(c, 0), 1);
    mb_init(cl_mb(c, 1), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (c.acs >= 0)
    for (int kw = 0; kw < Kc * E.Wc; ++kw) {
      cl_sm[c.acs + kw * c.T + c.li] = c.ex ? E.Ac[(long)kw * c.d + c.orig] : make_double2(0.0, 0.0);
      reinterpret_cast<int*>(cl_sm + c.accs)[kw * c.T + c.li] =
          c.ex ? E.cl_accols[(long)kw * c.d + c.gi] - c.g0 + c.HW : c.H + c.li;
    }
  cl_sync();
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
    load_row<W, MAXC, SMALL>(E, c, n, R);
    const double2 psip = c.own ? E.bk_psi[((long)g * N + n) * c.d + c.gi] : make_double2(0.0, 0.0);
    double2 lamc[LG_MAX_SPECS];
    for (int si = 0; si < LG_MAX_SPECS; ++si)
      lamc[si] = c.own && si < I ? E.bk_lam[(((long)g * N + n) * E.cta_Imax + si) * c.d + c.gi] : make_double2(0.0, 0.0);
    aux_products<W, MAXC, SMALL>(E, c, R, n, set, t0, psip, lamc);
  }
  cl_sync();
}

#include "lg_sweep_cl_large.cuh"

// Instantiations for one ELL width per translation unit (lg_sweep_cl_w*.cu), so the
// build compiles them in parallel.
#define LG_CL_KERNELS(W_)                                                                              \
  extern "C" void* lg_cl_kernel_w##W_(int backward, int maxc, int small) {                            \
    switch (maxc * 2 + (small ? 1 : 0)) {                                                                \
      LG_CL_CASE(W_, 2) LG_CL_CASE(W_, 3) LG_CL_CASE(W_, 4) LG_CL_CASE(W_, 5) LG_CL_CASE(W_, 6)          \
      LG_CL_CASE(W_, 8)                                                                                  \
    }                                                                                                    \
    return nullptr;                                                                                      \
  }
// backward: 0 forward, 1 backward, 3 forward line-search batch, 4 adjoint sweep storing psi_{n-1} /
// lambda_s(n), 5 derivative-product items (two-phase backward)
#define LG_CL_CASE(W_, C_)                                                                                   \
  case C_ * 2:                                                                                               \
    if (backward == 3) return (void*)lg_k_cl_forward_batch<W_, C_, false>;                                  \
    if (backward == 4) return (void*)lg_k_cl_adjoint<W_, C_, false>;                                        \
    if (backward == 5) return (void*)lg_k_cl_aux<W_, C_, false>;                                            \
    return backward ? (void*)lg_k_cl_backward<W_, C_, false> : (void*)lg_k_cl_forward<W_, C_, false>;        \
  case C_ * 2 + 1:                                                                                           \
    if (small == 2) return backward == 1 ? (void*)lg_k_cl_backward<W_, C_, true, true> : nullptr;            \
    if (backward == 4 && small == 1) return (void*)lg_k_cl_adjoint<W_, C_, true>;                            \
    if (backward == 5 && small == 1) return (void*)lg_k_cl_aux<W_, C_, true>;                                \
    if (backward >= 4 && small != 3) return nullptr;                                                         \
    if (small == 3)                                                                                          \
      return backward == 3 ? (void*)lg_k_cll_forward_batch<W_, C_, 2>                                        \
           : backward == 4 ? (void*)lg_k_cll_adjoint<W_, C_, 2>                                              \
           : backward == 5 ? (void*)lg_k_cll_aux<W_, C_, 2>                                                  \
           : backward      ? (void*)lg_k_cll_backward<W_, C_, 2> : (void*)lg_k_cll_forward<W_, C_, 2>;        \
    if (backward == 3) return (void*)lg_k_cl_forward_batch<W_, C_, true>;                                   \
    return backward ? (void*)lg_k_cl_backward<W_, C_, true> : (void*)lg_k_cl_forward<W_, C_, true>;
