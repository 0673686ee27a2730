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
__device__ __forceinline__ void team_sync(int id) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(TEAM) : "memory"); }

struct Team {
  int id;    // named barrier id (1..15)
  int tl;    // thread index within team [0, 64)
  int d;
};

// Per-team Taylor chain over NC columns (NC == 2: column 0 is the aux top with
// the control generator acting on column 1, the bottom).  Input staged in tb0.
template <int W, int RPL, int NC>
__device__ __forceinline__ void team_chain(const Team& tm, double2 (&cur)[NC][RPL], const double2 (&a)[RPL][W],
                                           const int (&col)[RPL][W], const double2 (&ac)[RPL][2],
                                           const int (&accol)[RPL][2], int m, int s, double sgn, int tb0, int tb1,
                                           int rt) {
  const int d = tm.d;
  if (tm.tl < m) ws_sm[rt + tm.tl].x = sgn * (1.0 / (double)(s * (tm.tl + 1)));
  team_sync(tm.id);
  int X = tb0, Y = tb1;
  for (int si = 0; si < s; ++si) {
    for (int j = 1; j <= m; ++j) {
      const double r = ws_sm[rt + j - 1].x;
      const bool last = j == m;
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int i = tm.tl + k * TEAM;
        if (i >= d) continue;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const int xc = X + c * d;
          double2 p = make_double2(0.0, 0.0), q = make_double2(0.0, 0.0);
#pragma unroll
          for (int w = 0; w < W; ++w) cmac(p, q, a[k][w], ws_sm[xc + col[k][w]]);
          if (NC == 2 && c == 0) {
            cmac(p, q, ac[k][0], ws_sm[X + d + accol[k][0]]);
            cmac(p, q, ac[k][1], ws_sm[X + d + accol[k][1]]);
          }
          const double2 tt = make_double2((p.x + q.x) * r, (p.y + q.y) * r);
          cur[c][k] = cadd(cur[c][k], tt);
          ws_sm[Y + c * d + i] = last ? cur[c][k] : tt;
        }
      }
      team_sync(tm.id);
      const int t_ = X;
      X = Y;
      Y = t_;
    }
  }
}

template <int W, int RPL>
__device__ __forceinline__ void load_rows(const LgEngineArgs& E, int n, int tl, double2 (&a)[RPL][W], int (&col)[RPL][W]) {
  const double2* src = E.A + (long)n * W * E.d;
#pragma unroll
  for (int k = 0; k < RPL; ++k) {
    const int i = tl + k * TEAM;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const bool ok = i < E.d;
      a[k][w] = ok ? src[(long)w * E.d + i] : make_double2(0.0, 0.0);
      col[k][w] = ok ? E.A_cols[w * E.d + i] : 0;
    }
  }
}

// Team-wide deterministic sum of NV complex values (thread partials) -> res[0..NV) for all team threads.
template <int NV>
__device__ __forceinline__ void team_reduce(const Team& tm, double2 (&v)[NV], int red) {
  const int w = tm.tl >> 5, l = tm.tl & 31;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    v[q] = warp_sum(v[q]);
    if (l == 0) ws_sm[red + q * 2 + w] = v[q];
  }
  team_sync(tm.id);
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = cadd(ws_sm[red + q * 2], ws_sm[red + q * 2 + 1]);
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
  int bars;    // mbarriers
  int words;
};

__host__ __device__ __forceinline__ WsLay ws_layout(int d, int nteams, int I, int Wp) {
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
  L.bars = o;
  o += (2 * RING * (1 + I) + 1) / 2 + 1;
  L.words = o;
  return L;
}

__device__ __forceinline__ double2 pen_row(int d, int Wp, int pen, const int* pcol, int i, int psi) {
  double2 p = make_double2(0.0, 0.0), q = make_double2(0.0, 0.0);
  for (int w = 0; w < Wp; ++w) cmac(p, q, ws_sm[pen + w * d + i], ws_sm[psi + pcol[w * d + i]]);
  return cadd(p, q);
}

}  // namespace

extern "C" __global__ void lg_ws_dummy() {}

// ------------------------------------------------------------------------------------------ forward
// teams: 0 = propagation P, 1 = scalars F.   blockDim = 2 * TEAM.
template <int W, int RPL>
__global__ void __launch_bounds__(2 * TEAM, 1) lg_k_ws_forward(const __grid_constant__ LgEngineArgs E) {
  const int d = E.d, g = blockIdx.x;
  const int set = E.grp_set[g], t0 = E.grp_t0[g], trel = t0 - E.set_t0[set];
  const int I = E.set_nspec[set];
  int Wp = 1;
  for (int si = 0; si < I; ++si) Wp = max(Wp, E.spec[E.set_spec[set][si]].pen_W);
  const WsLay L = ws_layout(d, 2, I, Wp);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(ws_sm + L.bars);
  unsigned long long* full = bars;
  unsigned long long* empty = bars + RING;
  int* pcol = reinterpret_cast<int*>(ws_sm) + 4 * L.pencol;
  const int team = threadIdx.x / TEAM;
  Team tm{team + 1, (int)threadIdx.x % TEAM, d};
  // stage targets / penalty operators
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
  if (threadIdx.x == 0) {
    for (int j = 0; j < RING; ++j) {
      mb_init(&full[j], TEAM);
      mb_init(&empty[j], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int N = E.N;
  const int tb0 = L.tb + team * 4 * d, tb1 = tb0 + 2 * d;
  if (team == 0) {
    // ---------------- P: forward propagation
    double2 cur[1][RPL];
    double2 a[RPL][W], an[RPL][W];
    int col[RPL][W], coln[RPL][W];
    double2 ac[RPL][2];
    int accol[RPL][2];
#pragma unroll
    for (int k = 0; k < RPL; ++k) ac[k][0] = ac[k][1] = make_double2(0.0, 0.0), accol[k][0] = accol[k][1] = 0;
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const int i = tm.tl + k * TEAM;
      if (i < d) ws_sm[tb0 + i] = E.psi0[(long)t0 * d + i];
    }
    load_rows<W, RPL>(E, 0, tm.tl, an, coln);
    int4 pln = E.plan[0];
    team_sync(tm.id);
    for (int n = 0; n < N; ++n) {
      const int4 pl = pln;
#pragma unroll
      for (int k = 0; k < RPL; ++k)
#pragma unroll
        for (int w = 0; w < W; ++w) a[k][w] = an[k][w], col[k][w] = coln[k][w];
      if (n + 1 < N) {
        load_rows<W, RPL>(E, n + 1, tm.tl, an, coln);
        pln = E.plan[(long)(n + 1) * (E.Kc + 1)];
      }
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int i = tm.tl + k * TEAM;
        cur[0][k] = i < d ? ws_sm[tb0 + i] : make_double2(0.0, 0.0);
      }
      team_chain<W, RPL, 1>(tm, cur, a, col, ac, accol, pl.x, pl.y, 1.0, tb0, tb1, L.rt + team * 64);
      const int slot = n % RING, use = n / RING;
      if (use > 0) mb_wait(&empty[slot], (use - 1) & 1);
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int i = tm.tl + k * TEAM;
        if (i < d) {
          ws_sm[L.ring + slot * d + i] = cur[0][k];
          ws_sm[tb0 + i] = cur[0][k];
        }
      }
      mb_arrive(&full[slot]);
      team_sync(tm.id);
    }
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const int i = tm.tl + k * TEAM;
      if (i < d) E.psiN[(long)t0 * d + i] = cur[0][k];
    }
  } else {
    // ---------------- F: per-step scalars from the psi ring
    double runacc[LG_MAX_SPECS];
    for (int si = 0; si < LG_MAX_SPECS; ++si) runacc[si] = 0.0;
    for (int n = 0; n < N; ++n) {
      const int slot = n % RING, use = n / RING;
      mb_wait(&full[slot], use & 1);
      const int psi = L.ring + slot * d;
      const bool fin = n == N - 1;
      double2 v[4];
#pragma unroll
      for (int si = 0; si < 4; ++si) v[si] = make_double2(0.0, 0.0);
      for (int si = 0; si < I; ++si) {
        const int kind = E.spec[E.set_spec[set][si]].kind;
        for (int k = 0; k < RPL; ++k) {
          const int i = tm.tl + k * TEAM;
          if (i >= d) continue;
          const double2 pv = ws_sm[psi + i];
          if (kind == LGK_STATE_PEN)
            v[si] = cadd(v[si], cdot(pv, pen_row(d, Wp, L.pen + si * Wp * d, pcol + si * Wp * d, i, psi)));
          else if (kind == LGK_STATE_INF)
            v[si] = cadd(v[si], cdot(pv, ws_sm[L.tgt + si * d + i]));
          else
            v[si] = cadd(v[si], cdot(ws_sm[L.tgt + si * d + i], pv));
        }
      }
      team_reduce<4>(tm, v, L.red + team * 2 * LG_MAX_SPECS);
      if (tm.tl == 0) {
        mb_arrive(&empty[slot]);
        for (int si = 0; si < I; ++si) {
          const int sidx = E.set_spec[set][si];
          const int kind = E.spec[sidx].kind;
          const long o = (long)sidx * E.T_total + t0;
          if (kind == LGK_STATE_PEN) {
            runacc[si] += v[si].x;
          } else if (kind == LGK_STATE_RUN) {
            const double h = hypot(v[si].x, v[si].y);
            runacc[si] += h * h;
          } else if (kind == LGK_GATE_RUN) {
            E.trp[((long)sidx * N + n) * E.T_total + t0] = v[si];
          } else if (fin) {
            E.fin[o] = v[si];
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

// ------------------------------------------------------------------------------------------ backward
// teams: X_0..X_{Kc-1}, P, L_0..L_{I-1}.   blockDim = (Kc + 1 + I) * TEAM.
template <int W, int RPL>
__global__ void __launch_bounds__(8 * TEAM, 1) lg_k_ws_backward(const __grid_constant__ LgEngineArgs E) {
  const int d = E.d, g = blockIdx.x, Kc = E.Kc, N = E.N;
  const int set = E.grp_set[g], t0 = E.grp_t0[g], trel = t0 - E.set_t0[set];
  const int I = E.set_nspec[set];
  int Wp = 1;
  for (int si = 0; si < I; ++si) Wp = max(Wp, E.spec[E.set_spec[set][si]].pen_W);
  const int nteams = Kc + 1 + I;
  const WsLay L = ws_layout(d, nteams, I, Wp);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(ws_sm + L.bars);
  unsigned long long* pfull = bars;                // [RING]
  unsigned long long* pempty = bars + RING;        // [RING]
  unsigned long long* lfull = bars + 2 * RING;     // [I][RING]
  unsigned long long* lempty = lfull + I * RING;   // [I][RING]
  int* pcol = reinterpret_cast<int*>(ws_sm) + 4 * L.pencol;
  const int team = threadIdx.x / TEAM;
  Team tm{team + 1, (int)threadIdx.x % TEAM, d};
  const int Xteams = Kc, Pteam = Kc;
  // psi consumers: all X teams + L teams whose source needs psi_{n-1}
  int n_lpsi = 0;
  for (int si = 0; si < I; ++si) {
    const int kind = E.spec[E.set_spec[set][si]].kind;
    n_lpsi += (kind == LGK_STATE_PEN || kind == LGK_STATE_RUN);
  }
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
  if (threadIdx.x == 0) {
    for (int j = 0; j < RING; ++j) {
      mb_init(&pfull[j], TEAM);
      mb_init(&pempty[j], Xteams + n_lpsi);
      for (int si = 0; si < I; ++si) {
        mb_init(&lfull[si * RING + j], TEAM);
        mb_init(&lempty[si * RING + j], Xteams);
      }
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (team >= nteams) return;  // set with fewer cost terms than the widest set
  const int tb0 = L.tb + team * 4 * d, tb1 = tb0 + 2 * d, rt = L.rt + team * 64;
  const int red = L.red + team * 2 * LG_MAX_SPECS;
  double2 a[RPL][W], an[RPL][W];
  int col[RPL][W], coln[RPL][W];
  double2 ac[RPL][2];
  int accol[RPL][2];
#pragma unroll
  for (int k = 0; k < RPL; ++k) ac[k][0] = ac[k][1] = make_double2(0.0, 0.0), accol[k][0] = accol[k][1] = 0;
  load_rows<W, RPL>(E, N - 1, tm.tl, an, coln);

  if (team < Xteams) {
    // ---------------- X_k: derivative products and inner products
    const int kch = team;
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const int i = tm.tl + k * TEAM;
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const bool ok = i < d && w < E.Wc;
        ac[k][w] = ok ? E.Ac[((long)kch * E.Wc + w) * d + i] : make_double2(0.0, 0.0);
        accol[k][w] = ok ? E.Ac_cols[((long)kch * E.Wc + w) * d + i] : 0;
      }
    }
    int4 pln = E.plan[(long)(N - 1) * (Kc + 1) + 1 + kch];
    for (int it = 0; it < N; ++it) {
      const int n = N - 1 - it;
      const int4 pl = pln;
#pragma unroll
      for (int k = 0; k < RPL; ++k)
#pragma unroll
        for (int w = 0; w < W; ++w) a[k][w] = an[k][w], col[k][w] = coln[k][w];
      if (n > 0) {
        load_rows<W, RPL>(E, n - 1, tm.tl, an, coln);
        pln = E.plan[(long)(n - 1) * (Kc + 1) + 1 + kch];
      }
      const int slot = it % RING, use = it / RING;
      mb_wait(&pfull[slot], use & 1);
      double2 cur[2][RPL];
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int i = tm.tl + k * TEAM;
        const double2 v = i < d ? ws_sm[L.ring + slot * d + i] : make_double2(0.0, 0.0);
        cur[0][k] = make_double2(0.0, 0.0);
        cur[1][k] = v;
        if (i < d) {
          ws_sm[tb0 + i] = make_double2(0.0, 0.0);
          ws_sm[tb0 + d + i] = v;
        }
      }
      team_sync(tm.id);
      if (tm.tl == 0) mb_arrive(&pempty[slot]);
      team_chain<W, RPL, 2>(tm, cur, a, col, ac, accol, pl.x, pl.y, 1.0, tb0, tb1, rt);
      // inner products with lambda_s(n)
      double2 v[4];
#pragma unroll
      for (int si = 0; si < 4; ++si) v[si] = make_double2(0.0, 0.0);
      for (int si = 0; si < I; ++si) {
        mb_wait(&lfull[si * RING + slot], use & 1);
#pragma unroll
        for (int k = 0; k < RPL; ++k) {
          const int i = tm.tl + k * TEAM;
          if (i < d) v[si] = cadd(v[si], cdot(ws_sm[L.lring + (si * RING + slot) * d + i], cur[0][k]));
        }
      }
      team_reduce<4>(tm, v, red);
      if (tm.tl == 0) {
        for (int si = 0; si < I; ++si) {
          mb_arrive(&lempty[si * RING + slot]);
          const int sidx = E.set_spec[set][si];
          E.ip[(((long)n * E.n_specs + sidx) * Kc + kch) * E.T_total + t0] = v[si];
        }
      }
    }
  } else if (team == Pteam) {
    // ---------------- P: psi recovery by adjoint propagation
    double2 cur[1][RPL];
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const int i = tm.tl + k * TEAM;
      if (i < d) ws_sm[tb0 + i] = E.psiN[(long)t0 * d + i];
    }
    int4 pln = E.plan[(long)(N - 1) * (Kc + 1)];
    team_sync(tm.id);
    for (int it = 0; it < N; ++it) {
      const int n = N - 1 - it;
      const int4 pl = pln;
#pragma unroll
      for (int k = 0; k < RPL; ++k)
#pragma unroll
        for (int w = 0; w < W; ++w) a[k][w] = an[k][w], col[k][w] = coln[k][w];
      if (n > 0) {
        load_rows<W, RPL>(E, n - 1, tm.tl, an, coln);
        pln = E.plan[(long)(n - 1) * (Kc + 1)];
      }
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int i = tm.tl + k * TEAM;
        cur[0][k] = i < d ? ws_sm[tb0 + i] : make_double2(0.0, 0.0);
      }
      team_chain<W, RPL, 1>(tm, cur, a, col, ac, accol, pl.x, pl.y, -1.0, tb0, tb1, rt);
      const int slot = it % RING, use = it / RING;
      if (use > 0) mb_wait(&pempty[slot], (use - 1) & 1);
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int i = tm.tl + k * TEAM;
        if (i < d) {
          ws_sm[L.ring + slot * d + i] = cur[0][k];
          ws_sm[tb0 + i] = cur[0][k];
        }
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
    // costate initialisation from psi_N (src/costs.py:312-321, :457-460); psi_N staged in tb1
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const int i = tm.tl + k * TEAM;
      if (i < d) ws_sm[tb1 + i] = E.psiN[(long)t0 * d + i];
    }
    team_sync(tm.id);
    double2 ov[1] = {make_double2(0.0, 0.0)};
    if (kind == LGK_STATE_RUN) {
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int i = tm.tl + k * TEAM;
        if (i < d) ov[0] = cadd(ov[0], cdot(ws_sm[tg + i], ws_sm[tb1 + i]));
      }
      team_reduce<1>(tm, ov, red);
    }
    const double2 trN = kind == LGK_GATE_RUN ? E.trsum[(long)sidx * N + N - 1] : make_double2(0.0, 0.0);
    double2 cur[1][RPL];
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const int i = tm.tl + k * TEAM;
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
    int4 pln = E.plan[(long)(N - 1) * (Kc + 1)];
    for (int it = 0; it < N; ++it) {
      const int n = N - 1 - it;
      const int slot = it % RING, use = it / RING;
      // publish lambda_s(n) for the X teams; it is also the chain input
      if (use > 0) mb_wait(&lempty[si * RING + slot], (use - 1) & 1);
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int i = tm.tl + k * TEAM;
        if (i < d) {
          ws_sm[L.lring + (si * RING + slot) * d + i] = cur[0][k];
          ws_sm[tb0 + i] = cur[0][k];
        }
      }
      mb_arrive(&lfull[si * RING + slot]);
      if (n == 0) break;
      const int4 pl = pln;
#pragma unroll
      for (int k = 0; k < RPL; ++k)
#pragma unroll
        for (int w = 0; w < W; ++w) a[k][w] = an[k][w], col[k][w] = coln[k][w];
      if (n > 0) {
        load_rows<W, RPL>(E, n - 1, tm.tl, an, coln);
        pln = E.plan[(long)(n - 1) * (Kc + 1)];
      }
      const double2 tr = kind == LGK_GATE_RUN ? E.trsum[(long)sidx * N + n - 1] : make_double2(0.0, 0.0);
      team_sync(tm.id);
      team_chain<W, RPL, 1>(tm, cur, a, col, ac, accol, pl.x, pl.y, -1.0, tb0, tb1, rt);
      if (needs_psi) {
        mb_wait(&pfull[slot], use & 1);
        const int psi = L.ring + slot * d;
        if (kind == LGK_STATE_RUN) {
          double2 o2[1] = {make_double2(0.0, 0.0)};
#pragma unroll
          for (int k = 0; k < RPL; ++k) {
            const int i = tm.tl + k * TEAM;
            if (i < d) o2[0] = cadd(o2[0], cdot(ws_sm[tg + i], ws_sm[psi + i]));
          }
          team_reduce<1>(tm, o2, red);
#pragma unroll
          for (int k = 0; k < RPL; ++k) {
            const int i = tm.tl + k * TEAM;
            if (i < d) cur[0][k] = cadd(cur[0][k], cmul(ws_sm[tg + i], o2[0]));
          }
        } else {
#pragma unroll
          for (int k = 0; k < RPL; ++k) {
            const int i = tm.tl + k * TEAM;
            if (i < d) cur[0][k] = cadd(cur[0][k], pen_row(d, Wp, pen, pc, i, psi));
          }
          team_sync(tm.id);
        }
        if (tm.tl == 0) mb_arrive(&pempty[slot]);
      } else if (kind == LGK_GATE_RUN) {
#pragma unroll
        for (int k = 0; k < RPL; ++k) {
          const int i = tm.tl + k * TEAM;
          if (i < d) cur[0][k] = cadd(cur[0][k], cmul(ws_sm[tg + i], tr));
        }
      }
    }
  }
}

extern "C" int lg_ws_layout_words(int d, int nteams, int I, int Wp) { return ws_layout(d, nteams, I, Wp).words; }

extern "C" void* lg_ws_kernel(int backward, int W, int rpl) {
#define LG_WS(W_, R_) \
  if (W == W_ && rpl == R_) return backward ? (void*)lg_k_ws_backward<W_, R_> : (void*)lg_k_ws_forward<W_, R_>;
  LG_WS(1, 1) LG_WS(2, 1) LG_WS(3, 1) LG_WS(4, 1) LG_WS(5, 1) LG_WS(6, 1) LG_WS(7, 1) LG_WS(8, 1) LG_WS(9, 1)
  LG_WS(1, 2) LG_WS(2, 2) LG_WS(3, 2) LG_WS(4, 2) LG_WS(5, 2) LG_WS(6, 2) LG_WS(7, 2) LG_WS(8, 2) LG_WS(9, 2)
#undef LG_WS
  return nullptr;
}
