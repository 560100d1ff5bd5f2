// Device integrands: the reference suite f1..f8 and the reference unit-test
// integrands, with the reference's exact operation order.
//
// Two shapes:
//  * Separable (f1..f8): f(x) = fin(init (+) t_0(x_0) (+) t_1(x_1) ... (+) t_{n-1}(x_{n-1}))
//    where (+) is the reference's left fold (`s += ...` or `p *= ...`) and
//    t_a depends on x_a only.  The evaluator exploits this: the rule's points
//    only ever take 9 distinct values per axis (c, c+-l2h, c+-l3h, c+-l4h,
//    c+-l5h), so each t_a is computed once per (axis, value) and each point
//    costs only the n-1 fold steps + fin().  The fold itself is performed
//    in the same order with the same roundings, so values are bit-identical
//    to calling f(x) as the reference does (integrands.cpp:24-79).
//  * Generic (PAGANI_TEST_*): f(x, n) evaluated on the full point.
//
// f6 additionally has a per-axis cut (integrands.cpp:63): the point value is
// 0.0 as soon as any x_i >= (3+i)/10.
#pragma once

#include "fp_ops.cuh"
#include "glibc_math.cuh"

#ifndef PGN_F1_COS_BF
#define PGN_F1_COS_BF 0
#endif
#ifndef PGN_F1_PAIR
#define PGN_F1_PAIR 1  // paired cos reductions: f1 k_evaluate -5% on B200
#endif

namespace pgn {

struct MathTables {
  const uint64_t* exp_tab;  // 256 u64 (glibc __exp_data.tab)
  const double* sincos;     // 440 doubles (glibc __sincostab)
  ExpK K{};                 // exp constants (immediates unless the kernel hoists them)
  CosK KC{};                // cos constants (likewise)
  uint32_t exp_s = 0, sc_s = 0;  // shared-memory addresses of the two tables (device)
};

#if defined(__CUDACC__)
// Device tables: both tables live in shared memory.
__device__ __forceinline__ MathTables make_tables(const uint64_t* s_exp, const double* s_sc) {
  MathTables T{s_exp, s_sc};
  T.exp_s = static_cast<uint32_t>(__cvta_generic_to_shared(s_exp));
  T.sc_s = static_cast<uint32_t>(__cvta_generic_to_shared(s_sc));
  return T;
}
#endif

// exp / cos of the hot path: shared-address variants on the device.
PGN_HD double tab_exp(double x, const MathTables& T) {
#if defined(__CUDA_ARCH__)
  return gm_exp_s(x, SmemTab{T.exp_s}, T.K);
#else
  return gm_exp_k(x, T.exp_tab, T.K);
#endif
}
PGN_HD void tab_exp2(double x0, double x1, const MathTables& T, double& y0, double& y1) {
#if defined(__CUDA_ARCH__)
  gm_exp2_s(x0, x1, SmemTab{T.exp_s}, T.K, y0, y1);
#else
  y0 = gm_exp_k(x0, T.exp_tab, T.K);
  y1 = gm_exp_k(x1, T.exp_tab, T.K);
#endif
}
PGN_HD void tab_cos2(double x0, double x1, const MathTables& T, double& y0, double& y1) {
#if defined(__CUDA_ARCH__)
  gm_cos2_s(x0, x1, SmemTab{T.sc_s}, T.KC, y0, y1);
#else
  y0 = gm_cos(x0, T.sincos, T.KC);
  y1 = gm_cos(x1, T.sincos, T.KC);
#endif
}
PGN_HD double tab_cos(double x, const MathTables& T) {
#if defined(__CUDA_ARCH__)
  return gm_cos_s(x, SmemTab{T.sc_s}, T.KC);
#else
  return gm_cos(x, T.sincos, T.KC);
#endif
}

struct IntegrandParams {
  double p[32];
};

// integrands.cpp:14-22 (square-and-multiply)
PGN_HD double ipow(double base, int e) {
  double r = 1.0;
  while (e > 0) {
    if (e & 1) r = P_MUL(r, base);
    base = P_MUL(base, base);
    e >>= 1;
  }
  return r;
}

// ---- separable suite --------------------------------------------------------
// Each functor: kCut, init(), term(a, x), comb(s, t), fin(s, n, tables), cut(a, x).

struct F1 {  // cos(sum (i+1) x_i)              integrands.cpp:24-28
  static constexpr bool kSeparable = true, kCut = false;
  static constexpr bool kPrefer4CtasPerSm = true;  // evaluate.cuh eval_min_blocks
  static constexpr int kMath = 2;  // 0 none, 1 exp, 2 cos
  PGN_HD static double init() { return 0.0; }
  PGN_HD static double term(int a, double x) { return P_MUL(static_cast<double>(a + 1), x); }
  PGN_HD static double comb(double s, double t) { return P_ADD(s, t); }
  PGN_HD static double fin(double s, int, const MathTables& T) {
#if PGN_F1_COS_BF
    return gm_cos_bf(s, T.sincos);
#else
    return tab_cos(s, T);
#endif
  }
#if !PGN_F1_COS_BF && PGN_F1_PAIR
  PGN_HD static void fin2(double s0, double s1, int, const MathTables& T, double& f0, double& f1) {
    tab_cos2(s0, s1, T, f0, f1);
  }
#endif
  PGN_HD static bool cut(int, double) { return false; }
};

struct F2 {  // prod 1/(1/2500 + (x-1/2)^2)      integrands.cpp:30-37
  static constexpr bool kSeparable = true, kCut = false;
  static constexpr bool kPrefer4CtasPerSm = true;  // evaluate.cuh eval_min_blocks
  static constexpr int kMath = 0;  // 0 none, 1 exp, 2 cos
  PGN_HD static double init() { return 1.0; }
  PGN_HD static double term(int, double x) {
    const double t = P_SUB(x, 0.5);
    return P_DIV(1.0, P_ADD(0x1.a36e2eb1c432dp-12 /* 1.0/2500.0 */, P_MUL(t, t)));
  }
  PGN_HD static double comb(double s, double t) { return P_MUL(s, t); }
  PGN_HD static double fin(double s, int, const MathTables&) { return s; }
  PGN_HD static bool cut(int, double) { return false; }
};

struct F3 {  // (1 + sum (i+1) x_i)^-(n+1)       integrands.cpp:39-43
  static constexpr bool kSeparable = true, kCut = false;
  static constexpr bool kCornerRegs = true;  // evaluate.cuh corner_regs
  static constexpr int kMath = 0;  // 0 none, 1 exp, 2 cos
  PGN_HD static double init() { return 1.0; }
  PGN_HD static double term(int a, double x) { return P_MUL(static_cast<double>(a + 1), x); }
  PGN_HD static double comb(double s, double t) { return P_ADD(s, t); }
  PGN_HD static double fin(double s, int n, const MathTables&) {
    return P_DIV(1.0, ipow(s, n + 1));
  }
  PGN_HD static bool cut(int, double) { return false; }
};

#ifndef PGN_F4_UNDERFLOW_SKIP
#define PGN_F4_UNDERFLOW_SKIP 0  // A/B knob
#endif
struct F4 {  // exp(-625 sum (x-1/2)^2)          integrands.cpp:45-52
  static constexpr bool kSeparable = true, kCut = false;
  static constexpr bool kCornerRegs = true;  // evaluate.cuh corner_regs
  static constexpr int kMath = 1;  // 0 none, 1 exp, 2 cos
  PGN_HD static double init() { return 0.0; }
  PGN_HD static double term(int, double x) {
    const double t = P_SUB(x, 0.5);
    return P_MUL(t, t);
  }
  PGN_HD static double comb(double s, double t) { return P_ADD(s, t); }
  PGN_HD static double fin(double s, int, const MathTables& T) {
    return tab_exp(P_MUL(-625.0, s), T);
  }
  PGN_HD static void fin2(double s0, double s1, int, const MathTables& T, double& f0, double& f1) {
    const double x0 = P_MUL(-625.0, s0), x1 = P_MUL(-625.0, s1);
#if PGN_F4_UNDERFLOW_SKIP
    // both below -746: exp is +0 on every path of e_exp.c (tested against
    // libm), and far from the peak in 8D/10D most corner pairs are
    if (x0 < -746.0 && x1 < -746.0) {
      f0 = 0.0;
      f1 = 0.0;
      return;
    }
#endif
    tab_exp2(x0, x1, T, f0, f1);
  }
  PGN_HD static bool cut(int, double) { return false; }
};

struct F5 {  // exp(-10 sum |x-1/2|)             integrands.cpp:54-58
  static constexpr bool kSeparable = true, kCut = false;
  static constexpr bool kCornerRegs = true;  // evaluate.cuh corner_regs
  static constexpr bool kPrefer4CtasPerSm = true;  // evaluate.cuh eval_min_blocks
  static constexpr int kMath = 1;  // 0 none, 1 exp, 2 cos
  PGN_HD static double init() { return 0.0; }
  PGN_HD static double term(int, double x) { return pgn_fabs(P_SUB(x, 0.5)); }
  PGN_HD static double comb(double s, double t) { return P_ADD(s, t); }
  PGN_HD static double fin(double s, int, const MathTables& T) {
    return tab_exp(P_MUL(-10.0, s), T);
  }
  PGN_HD static void fin2(double s0, double s1, int, const MathTables& T, double& f0, double& f1) {
    tab_exp2(P_MUL(-10.0, s0), P_MUL(-10.0, s1), T, f0, f1);
  }
  PGN_HD static bool cut(int, double) { return false; }
};

struct F6 {  // exp(sum (i+5) x_i), 0 outside    integrands.cpp:60-67
  static constexpr bool kSeparable = true, kCut = true;
  static constexpr bool kCornerRegs = true;  // evaluate.cuh corner_regs
  static constexpr bool kPrefer4CtasPerSm = true;  // evaluate.cuh eval_min_blocks
  static constexpr int kMath = 1;  // 0 none, 1 exp, 2 cos
  PGN_HD static double init() { return 0.0; }
  PGN_HD static double term(int a, double x) { return P_MUL(static_cast<double>(a + 5), x); }
  PGN_HD static double comb(double s, double t) { return P_ADD(s, t); }
  PGN_HD static double fin(double s, int, const MathTables& T) {
    return tab_exp(s, T);
  }
  PGN_HD static void fin2(double s0, double s1, int, const MathTables& T, double& f0, double& f1) {
    tab_exp2(s0, s1, T, f0, f1);
  }
  PGN_HD static bool cut(int a, double x) {
    return x >= P_DIV(P_ADD(3.0, static_cast<double>(a + 1)), 10.0);
  }
};

struct F7 {  // (sum x^2)^11                     integrands.cpp:69-73
  static constexpr bool kSeparable = true, kCut = false;
  static constexpr int kMath = 0;  // 0 none, 1 exp, 2 cos
  PGN_HD static double init() { return 0.0; }
  PGN_HD static double term(int, double x) { return P_MUL(x, x); }
  PGN_HD static double comb(double s, double t) { return P_ADD(s, t); }
  PGN_HD static double fin(double s, int, const MathTables&) { return ipow(s, 11); }
  PGN_HD static bool cut(int, double) { return false; }
};

struct F8 {  // (sum x^2)^7 sqrt(sum x^2)        integrands.cpp:75-79
  static constexpr bool kSeparable = true, kCut = false;
  static constexpr int kMath = 0;  // 0 none, 1 exp, 2 cos
  PGN_HD static double init() { return 0.0; }
  PGN_HD static double term(int, double x) { return P_MUL(x, x); }
  PGN_HD static double comb(double s, double t) { return P_ADD(s, t); }
  PGN_HD static double fin(double s, int, const MathTables&) {
    return P_MUL(ipow(s, 7), P_SQRT(s));
  }
  PGN_HD static bool cut(int, double) { return false; }
};

// ---- generic: the reference unit-test lambdas (parameterised) --------------

PGN_HD double qnan() { return pgn_asf64(0x7ff8000000000000ULL); }

struct TConst {  // test_driver.cpp:22-32
  static constexpr bool kSeparable = false;
  PGN_HD static double eval(const double*, int, const IntegrandParams& P, const MathTables&) {
    return P.p[0];
  }
};
struct TMonomial {  // test_rule.cpp:40-49
  static constexpr bool kSeparable = false;
  PGN_HD static double eval(const double* x, int n, const IntegrandParams& P, const MathTables&) {
    double v = 1.0;
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < static_cast<int>(P.p[i]); ++k) v = P_MUL(v, x[i]);
    return v;
  }
};
struct TRough {  // test_driver.cpp:61-80 / :126-141
  static constexpr bool kSeparable = false;
  PGN_HD static double eval(const double* x, int n, const IntegrandParams& P,
                            const MathTables& T) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) {
      const double arg = P.p[1] == 2.0 ? P_MUL(P_MUL(P.p[0], x[i]), x[i]) : P_MUL(P.p[0], x[i]);
      s = P_ADD(s, gm_cos(arg, T.sincos));
    }
    return P_ADD(s, P_MUL(P.p[2], static_cast<double>(n)));
  }
};
struct TNanBox {  // test_rule.cpp:237-254, test_driver.cpp:111-124
  static constexpr bool kSeparable = false;
  PGN_HD static double eval(const double* x, int, const IntegrandParams& P, const MathTables&) {
    const bool in = x[0] > P.p[0] && (P.p[1] < 0.0 || x[1] > P.p[1]);
    return in ? qnan() : 1.0;
  }
};
struct TPocket {  // test_rule.cpp:217-235
  static constexpr bool kSeparable = false;
  PGN_HD static double eval(const double* x, int, const IntegrandParams& P, const MathTables&) {
    const double p = P.p[0];
    return x[0] > p && x[1] > p && x[2] > p ? 1.0 : 0.0;
  }
};
struct TCosSum {  // test_rule.cpp:191-215
  static constexpr bool kSeparable = false;
  PGN_HD static double eval(const double* x, int n, const IntegrandParams& P,
                            const MathTables& T) {
    double s = 0.0;
    for (int i = 0; i < n; ++i)
      s = P_ADD(s, gm_cos(P_MUL(P_MUL(P.p[1 + i], 3.0), x[i]), T.sincos));
    return P_MUL(P.p[0], s);
  }
};
struct TExpSq {  // test_rule.cpp:154-189
  static constexpr bool kSeparable = false;
  PGN_HD static double eval(const double* x, int n, const IntegrandParams&,
                            const MathTables& T) {
    double s = 0.0;
    for (int i = 0; i < n; ++i)
      s = P_ADD(s, P_ADD(gm_exp(P_DIV(x[i], 3.0), T.exp_tab), P_MUL(x[i], x[i])));
    return s;
  }
};

// fin() of two independent points: the integrand's paired form when it has
// one (interleaved dependency chains), else two calls.
template <class F, class = void>
struct HasFin2 { static constexpr bool value = false; };
template <class F>
struct HasFin2<F, decltype(void(&F::fin2))> { static constexpr bool value = true; };

template <class F>
PGN_HD void fin_pair(double s0, double s1, int n, const MathTables& T, double& f0, double& f1) {
  if constexpr (HasFin2<F>::value) {
    F::fin2(s0, s1, n, T, f0, f1);
  } else {
    f0 = F::fin(s0, n, T);
    f1 = F::fin(s1, n, T);
  }
}

// Full point evaluation of a separable integrand (used by the generic path
// and by pagani_call_integrand).
template <class F>
PGN_HD double eval_point(const double* x, int n, const IntegrandParams& P,
                         const MathTables& T) {
  if constexpr (F::kSeparable) {
    double s = F::init();
    for (int a = 0; a < n; ++a) {
      if constexpr (F::kCut) {
        if (F::cut(a, x[a])) return 0.0;
      }
      s = F::comb(s, F::term(a, x[a]));
    }
    return F::fin(s, n, T);
  } else {
    return F::eval(x, n, P, T);
  }
}

}  // namespace pgn
