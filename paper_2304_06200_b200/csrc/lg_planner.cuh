// Certified (order, scaling) planner: restatement of src/expm.py:110-303.
//
// Host build: an exact port -- same loop bounds, early exits, evaluation order
// and glibc calls (pow, expm1, log1p) that CPython makes for `**`,
// math.expm1 and math.log1p, compiled with -ffp-contract=off, so the result
// is bit-identical to expm.make_plan on the same machine.
//
// Device build: the same arithmetic with correctly rounded __d*_rn
// intrinsics (pure arithmetic is therefore bit-identical), but CUDA's pow /
// expm1 / log1p are not glibc's.  Every comparison whose operand went through
// one of them is checked against a relative guard band of 1e-12 (the libm
// discrepancy is <~1e-15 relative); if it falls inside, the plan is flagged
// LG_PLAN_UNCERTAIN and the host recomputes it exactly.
#pragma once
#include "lg_numpy.cuh"

#define LG_PLAN_OK 0
#define LG_PLAN_INFEASIBLE 1   // PlanningError (src/expm.py:244-249,273-276)
#define LG_PLAN_BADARG 2       // ValueError (src/expm.py:295-300)
#define LG_PLAN_UNCERTAIN 4    // device only: recompute on host

struct LgPlan {
  int order, scaling, status, pad;
  double bound;
};

struct LgPlannerCtx {
  double u_prime;   // 2 sqrt(2) u / (1 - 2u), u = 2^-53 (src/expm.py:69-84)
  int uncertain;    // device: set when a guarded comparison fell in the band
};

LG_HD inline double lg_u_prime() {
  const double u = 1.1102230246251565e-16;  // 2**-53
  return LG_DIV(LG_MUL(LG_MUL(2.0, LG_SQRT(2.0)), u), LG_SUB(1.0, LG_MUL(2.0, u)));
}

LG_HD inline double lg_pow(double x, int s) {
  if (s == 1) return x;  // pow(x, 1) == x exactly in glibc and CUDA
  return pow(x, (double)s);
}

// Flags (device only) a libm-derived value that lies within the guard band of tau.
LG_HD inline double lg_guard(LgPlannerCtx& cx, double v, double tau) {
#ifdef __CUDA_ARCH__
  if (isfinite(v) && fabs(v - tau) <= 1e-12 * tau) cx.uncertain = 1;
#endif
  return v;
}

// remainder_rm: src/expm.py:110-143
LG_HD inline double lg_remainder_rm(double x, int m) {
  if (x == 0.0) return 0.0;
  double term = 1.0;
  for (int q = 1; q <= m + 1; ++q) {
    term = LG_MUL(term, LG_DIV(x, (double)q));
    if (isinf(term)) return INFINITY;
  }
  double total = term;
  int q = m + 1;
  for (int it = 0; it < 500; ++it) {
    q += 1;
    term = LG_MUL(term, LG_DIV(x, (double)q));
    total = LG_ADD(total, term);
    if (term < LG_MUL(1e-20, total)) return total;
  }
  double ratio = LG_DIV(x, (double)(q + 1));
  if (ratio < 1.0) return LG_ADD(total, LG_DIV(LG_MUL(term, ratio), LG_SUB(1.0, ratio)));
  return INFINITY;
}

// gamma_n: src/expm.py:146-153; returns false when n u' >= 1 (infeasible model).
LG_HD inline bool lg_gamma_n(const LgPlannerCtx& cx, long n, double* out) {
  double nu = LG_MUL((double)n, cx.u_prime);
  if (nu >= 1.0) return false;
  *out = LG_DIV(nu, LG_SUB(1.0, nu));
  return true;
}

// _beta_sum: src/expm.py:156-169
LG_HD inline bool lg_beta_sum(const LgPlannerCtx& cx, double xb, int m, long sp, double* out) {
  double beta = 0.0, power = 1.0;
  long step = sp + 2;
  for (int k = 0; k <= m; ++k) {
    if (k > 0) power = LG_MUL(power, LG_DIV(xb, (double)k));
    double g;
    if (!lg_gamma_n(cx, (long)k * step + m + 2, &g)) return false;
    beta = LG_ADD(beta, LG_MUL(g, power));
  }
  *out = beta;
  return true;
}

// rounding_bound: src/expm.py:172-196
LG_HD inline double lg_rounding_bound(const LgPlannerCtx& cx, double xb, int m, int s, long sp) {
  double rm = lg_remainder_rm(xb, m);
  if (isinf(rm)) return INFINITY;
  double alpha = LG_ADD(1.0, rm);
  double beta;
  if (!lg_beta_sum(cx, xb, m, sp, &beta)) return INFINITY;
  double a_s = lg_pow(alpha, s);
  if (isinf(a_s)) return INFINITY;  // Python: OverflowError -> inf
  double e = expm1(LG_MUL((double)s, log1p(LG_DIV(beta, alpha))));
  if (isinf(e)) return INFINITY;
  return LG_MUL(a_s, e);
}

// truncation_bound: src/expm.py:199-211
LG_HD inline double lg_truncation_bound(double xb, int m, int s) {
  double rm = lg_remainder_rm(xb, m);
  double x = LG_MUL((double)s, rm);
  if (isinf(x) || x >= 1.0) return INFINITY;
  if (x == 0.0) return 0.0;
  return LG_DIV(LG_MUL(x, LG_SUB(1.0, lg_pow(x, s))), LG_SUB(1.0, x));
}

// error_bound: src/expm.py:214-226
LG_HD inline double lg_error_bound(const LgPlannerCtx& cx, double xa, int m, int s, long sp) {
  double xb = LG_DIV(xa, (double)s);
  double t = lg_truncation_bound(xb, m, s);
  if (isinf(t)) return INFINITY;
  return LG_ADD(t, lg_rounding_bound(cx, xb, m, s, sp));
}

// make_plan + _cached_plan: src/expm.py:229-303
LG_HD inline LgPlan lg_make_plan(LgPlannerCtx& cx, double xa, long sp, double tau, int m_max, int s_max) {
  LgPlan p{0, 0, LG_PLAN_OK, 0, 0.0};
  if (!(xa >= 0.0) || sp < 0 || !(tau > 0.0)) {
    p.status = LG_PLAN_BADARG;
    return p;
  }
  double g3;
  lg_gamma_n(cx, 3, &g3);
  for (int s = 1; s <= s_max; ++s) {
    if (LG_MUL((double)s, g3) > tau) {
      p.status = LG_PLAN_INFEASIBLE;
      return p;
    }
    double xb = LG_DIV(xa, (double)s);
    if (lg_guard(cx, lg_truncation_bound(xb, m_max, s), tau) > tau) continue;
    for (int m = 1; m <= m_max; ++m) {
      double beta;
      if (!lg_beta_sum(cx, xb, m, sp, &beta)) break;
      if (LG_MUL((double)s, beta) > tau) break;
      double b = lg_guard(cx, lg_error_bound(cx, xa, m, s, sp), tau);
      if (b <= tau) {
        p.order = m;
        p.scaling = s;
        p.bound = b;
        return p;
      }
    }
  }
  p.status = LG_PLAN_INFEASIBLE;
  return p;
}
