// Bit-exact restatements of the numpy reductions that feed the (m, s) planner.
//
// The reference plans every step from ||A||_1, sigma' and the auxiliary-matrix
// norms (src/derivatives.py:105-110,166-196; src/sparse.py:90-121,201-222).
// Those numbers are produced by numpy, so the plan is only reproducible if the
// GPU performs exactly the same IEEE operations in exactly the same order:
//
//   * complex |z|: numpy's SIMD cabs, larger * sqrt(fma(r, r, 1)) with
//     r = smaller / larger (numpy/_core/src/umath/loops_unary_complex);
//   * np.bincount(cols, |v|): sequential per column in CSR entry order;
//   * np.add.reduceat(|v|, starts) / 1-D sum: a0 + pairwise(a[1:]);
//   * dense np.abs(F).sum(axis=0): pairwise over the whole contiguous column;
//   * dense np.abs(F).sum(axis=1): sequential across columns.
//
// pairwise() is numpy's pairwise_sum (blocks of 8 accumulators up to 128
// elements, recursive halving above).  Verified against numpy 2.3.5 in
// tests/test_numpy_rules.py.  Compile units using this header must not
// contract a*b+c into FMAs (the explicit fma below is intended).
#pragma once
#include <math.h>

#if defined(__CUDACC__)
#define LG_HD __host__ __device__
#else
#define LG_HD
#endif

#ifdef __CUDA_ARCH__
#define LG_MUL(a, b) __dmul_rn((a), (b))
#define LG_ADD(a, b) __dadd_rn((a), (b))
#define LG_SUB(a, b) __dsub_rn((a), (b))
#define LG_DIV(a, b) __ddiv_rn((a), (b))
#define LG_SQRT(a) __dsqrt_rn(a)
#define LG_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#define LG_MUL(a, b) ((a) * (b))
#define LG_ADD(a, b) ((a) + (b))
#define LG_SUB(a, b) ((a) - (b))
#define LG_DIV(a, b) ((a) / (b))
#define LG_SQRT(a) sqrt(a)
#define LG_FMA(a, b, c) fma((a), (b), (c))
#endif

// numpy complex absolute value (contiguous SIMD path).
LG_HD inline double lg_np_cabs(double re, double im) {
  double a = fabs(re), b = fabs(im);
  double larger = a > b ? a : b;
  double smaller = a > b ? b : a;
  if (isinf(larger)) return larger;
  double r = (larger == 0.0) ? 0.0 : LG_DIV(smaller, larger);
  return LG_MUL(LG_SQRT(LG_FMA(r, r, 1.0)), larger);
}

// numpy pairwise_sum leaf (n <= 128): blocks of 8 accumulators.
template <class Get>
LG_HD inline double lg_np_pairwise_leaf(const Get& get, long lo, long n) {
  if (n < 8) {
    double res = 0.0;
    for (long i = 0; i < n; ++i) res = LG_ADD(res, get(lo + i));
    return res;
  }
  double r0 = get(lo + 0), r1 = get(lo + 1), r2 = get(lo + 2), r3 = get(lo + 3);
  double r4 = get(lo + 4), r5 = get(lo + 5), r6 = get(lo + 6), r7 = get(lo + 7);
  long i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = LG_ADD(r0, get(lo + i + 0));
    r1 = LG_ADD(r1, get(lo + i + 1));
    r2 = LG_ADD(r2, get(lo + i + 2));
    r3 = LG_ADD(r3, get(lo + i + 3));
    r4 = LG_ADD(r4, get(lo + i + 4));
    r5 = LG_ADD(r5, get(lo + i + 5));
    r6 = LG_ADD(r6, get(lo + i + 6));
    r7 = LG_ADD(r7, get(lo + i + 7));
  }
  double res = LG_ADD(LG_ADD(LG_ADD(r0, r1), LG_ADD(r2, r3)), LG_ADD(LG_ADD(r4, r5), LG_ADD(r6, r7)));
  for (; i < n; ++i) res = LG_ADD(res, get(lo + i));
  return res;
}

// numpy pairwise_sum over elements get(lo) .. get(lo + n - 1): for n > 128 the
// block splits at n/2 rounded down to a multiple of 8.  Iterative (explicit
// stack, no recursion) so device stack use is static.
template <class Get>
LG_HD inline double lg_np_pairwise(const Get& get, long lo, long n) {
  if (n <= 128) return lg_np_pairwise_leaf(get, lo, n);
  struct Frame {
    long lo, n;
    int stage;
    double left;
  };
  Frame st[24];
  int sp = 0;
  st[0] = Frame{lo, n, 0, 0.0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame& f = st[sp];
    if (f.n <= 128) {
      ret = lg_np_pairwise_leaf(get, f.lo, f.n);
      --sp;
      continue;
    }
    long n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.stage == 0) {
      f.stage = 1;
      st[sp + 1] = Frame{f.lo, n2, 0, 0.0};
      ++sp;
    } else if (f.stage == 1) {
      f.left = ret;
      f.stage = 2;
      st[sp + 1] = Frame{f.lo + n2, f.n - n2, 0, 0.0};
      ++sp;
    } else {
      ret = LG_ADD(f.left, ret);
      --sp;
    }
  }
  return ret;
}

// np.add.reduceat segment / 1-D contiguous sum: a0 + pairwise(a[1:]).
template <class Get>
LG_HD inline double lg_np_reduce(const Get& get, long lo, long n) {
  if (n <= 0) return 0.0;
  if (n == 1) return get(lo);
  return LG_ADD(get(lo), lg_np_pairwise(get, lo + 1, n - 1));
}
