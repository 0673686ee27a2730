// Cost and gradient from the raw per-trajectory scalars of the two sweeps.
// Shared by the device finalize kernel and the host (sharded/multi-rank
// combine, lg_finalize_host) so both produce identical numbers: the kernel is
// built in a -fmad=false unit (lg_prep.cu) and the host with -ffp-contract=off,
// and |z| is numpy's formula (lg_np_cabs: one correctly rounded division, fma,
// sqrt) on both sides instead of the two sides' different hypot().
//
// Per cost term s over its trajectory set t in [t0, t0 + K):
//   STATE_INFIDELITY   cost 1/K sum_t (1 - |z_t|^2),  z_t = <psi_N|phi_t>     (src/costs.py:299-304)
//                      grad 1/K sum_t -2 Re(ip_t z_t)                           (:333-334)
//   STATE_PENALTY      cost 1/K sum_t P_t / N,  P_t = sum_n <psi_n|O|psi_n>   (:305-306)
//                      grad 1/K sum_t 2/N Re ip_t                               (:335-336)
//   STATE_RUNNING      cost 1/K sum_t (1 - R_t / N), R_t = sum_n |<phi|psi_n>|^2 (:307-308)
//                      grad 1/K sum_t -2/N Re ip_t                              (:337-338)
//   GATE_INFIDELITY    tr = sum_t <U_T psi_t|psi_N^t>;  cost 1 - |tr|^2/K^2       (:447-450)
//                      grad -2/K^2 Re((sum_t ip_t) conj(tr))                    (:486-487)
//   GATE_RUNNING       tr_n likewise per step; cost 1 - sum_n |tr_n|^2/(N K^2)
//                      grad -2/(N K^2) Re sum_t ip_t                            (:484-485)
// with ip_t[n][k] = <lambda_t|dU_n/da_k psi_t,n-1>.  K == 1 (state) and K == d
// (gate, full basis) are exactly the reference's formulas.
#pragma once
#include "lg_numpy.cuh"
#include "lg_types.h"

LG_HD inline double lg_final_grad(const LgFinalArgs& F, long q) {
  const int N = F.N, Kc = F.Kc, T = F.T_total;
  const int n = (int)(q / Kc), kc = (int)(q - (long)n * Kc);
  double g = 0.0;
  for (int s = 0; s < F.n_specs; ++s) {
    const int kind = F.kind[s], K = F.K[s], t0 = F.t0[s];
    if (K == 0) continue;
    const double2* ip = F.ip + (((long)n * F.n_specs + s) * Kc + kc) * T + t0;
    double gs = 0.0;
    if (kind == LGK_STATE_INF) {
      for (int t = 0; t < K; ++t) {
        const double2 z = F.fin[(long)s * T + t0 + t];
        gs += -2.0 * (ip[t].x * z.x - ip[t].y * z.y);
      }
      gs /= K;
    } else if (kind == LGK_STATE_PEN || kind == LGK_STATE_RUN) {
      for (int t = 0; t < K; ++t) gs += (kind == LGK_STATE_PEN ? 2.0 : -2.0) / N * ip[t].x;
      gs /= K;
    } else {
      double ax = 0.0, ay = 0.0;
      for (int t = 0; t < K; ++t) ax += ip[t].x, ay += ip[t].y;
      if (kind == LGK_GATE) {
        double tx = 0.0, ty = 0.0;
        for (int t = 0; t < K; ++t) tx += F.fin[(long)s * T + t0 + t].x, ty += F.fin[(long)s * T + t0 + t].y;
        gs = -2.0 / ((double)K * K) * (ax * tx + ay * ty);
      } else {
        gs = -2.0 / ((double)N * K * K) * ax;
      }
    }
    g += F.weight[s] * gs;
  }
  return g;
}

LG_HD inline double lg_final_cost(const LgFinalArgs& F) {
  const int N = F.N, T = F.T_total;
  double cost = 0.0;
  for (int s = 0; s < F.n_specs; ++s) {
    const int kind = F.kind[s], K = F.K[s], t0 = F.t0[s];
    if (K == 0) continue;
    double cs = 0.0;
    if (kind == LGK_STATE_INF) {
      for (int t = 0; t < K; ++t) {
        const double2 z = F.fin[(long)s * T + t0 + t];
        const double a = lg_np_cabs(z.x, z.y);
        cs += 1.0 - a * a;
      }
      cs /= K;
    } else if (kind == LGK_STATE_PEN) {
      for (int t = 0; t < K; ++t) cs += F.run[(long)s * T + t0 + t] / N;
      cs /= K;
    } else if (kind == LGK_STATE_RUN) {
      for (int t = 0; t < K; ++t) cs += 1.0 - F.run[(long)s * T + t0 + t] / N;
      cs /= K;
    } else if (kind == LGK_GATE) {
      double tx = 0.0, ty = 0.0;
      for (int t = 0; t < K; ++t) tx += F.fin[(long)s * T + t0 + t].x, ty += F.fin[(long)s * T + t0 + t].y;
      const double a = lg_np_cabs(tx, ty);
      cs = 1.0 - a * a / ((double)K * K);
    } else {
      double acc = 0.0;
      for (int n = 0; n < N; ++n) {
        double tx = 0.0, ty = 0.0;
        for (int t = 0; t < K; ++t) {
          const double2 v = F.trp[((long)s * N + n) * T + t0 + t];
          tx += v.x, ty += v.y;
        }
        const double a = lg_np_cabs(tx, ty);
        acc += a * a;
      }
      cs = 1.0 - acc / ((double)N * K * K);
    }
    cost += F.weight[s] * cs;
  }
  return cost;
}
