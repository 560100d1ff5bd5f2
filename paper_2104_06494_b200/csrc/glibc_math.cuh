// glibc 2.39 `exp` and `cos`, restated for host and device, bit-for-bit.
//
// Why: the reference evaluates its integrands with the platform libm
// (`/root/reference/proj/src/integrands.cpp:27,51,57,66`).  On an FMA-capable
// x86-64 host glibc's IFUNCs select `__exp_fma` / `__cos_fma`, i.e. the C
// sources of sysdeps/ieee754/dbl-64/e_exp.c (ARM optimized-routines exp,
// N = 128 table) and s_sin.c (IBM Accurate Mathematical Library cos) compiled
// with -mfma, where GCC contracted some products into FMAs.  CUDA's libdevice
// exp/cos are different algorithms and differ in the last ulp on ~1e-3 of
// arguments.  This header restates those two routines with the
// SAME operation order and the SAME fused/unfused choices as the shipped
// machine code (read from `objdump -d libm.so.6`), and
// the same tables (glibc_tables.h, extracted by tools/extract_glibc_tables.py).
// Bit-equality with the host libm is checked by
// tests/test_host.py::test_host_glibc_restatement_matches_libm on the CPU and
// tests/test_gpu_parity.py::test_device_glibc_exp_cos_bit_exact on the B200.
//
// Attribution / licence: this is a restatement of GNU C Library code and is
// distributed under the GNU Lesser General Public License, version 2.1 or
// later (LGPL-2.1+), like its sources:
//   * sysdeps/ieee754/dbl-64/e_exp.c, e_exp_data.c -- Copyright (C) 2018-2024
//     Free Software Foundation, Inc.; originally from ARM's optimized-routines
//     (Szabolcs Nagy), contributed to glibc under the LGPL.
//   * sysdeps/ieee754/dbl-64/s_sin.c, sincostab.c, usncs.h -- IBM Accurate
//     Mathematical Library, Copyright (C) 2001-2024 Free Software Foundation,
//     Inc.; written by International Business Machines Corp.
// See https://www.gnu.org/licenses/old-licenses/lgpl-2.1.html.  The rest of
// this repository is not derived from glibc.
//
// Every arithmetic op goes through fp_ops.cuh so nvcc cannot contract it.
// Round-to-nearest is assumed (glibc switches to it when needed; CUDA always
// rounds to nearest).
#pragma once

#include "fp_ops.cuh"
#include "glibc_tables.h"

namespace pgn {

// ---- exp: sysdeps/ieee754/dbl-64/e_exp.c (glibc 2.39), __exp_fma ---------
namespace expc {
constexpr uint64_t kInvLn2N = 0x40671547652b82feULL;   // 0x1.71547652b82fep7
constexpr uint64_t kShift = 0x4338000000000000ULL;     // 0x1.8p52
constexpr uint64_t kNegLn2hiN = 0xbf762e42fefa0000ULL; // -0x1.62e42fefa0000p-8
constexpr uint64_t kNegLn2loN = 0xbd0cf79abc9e3b3aULL; // -0x1.cf79abc9e3b3ap-47
constexpr uint64_t kC2 = 0x3fdffffffffffdbdULL;
constexpr uint64_t kC3 = 0x3fc555555555543cULL;
constexpr uint64_t kC4 = 0x3fa55555cf172b91ULL;
constexpr uint64_t kC5 = 0x3f81111167a4d017ULL;
}  // namespace expc

// cos constants (s_sin.c / usncs.h)
namespace cosc {
constexpr uint64_t kBig = 0x42c8000000000000ULL;    // 0x1.8p45
constexpr uint64_t kSn3 = 0xbfc5555555555515ULL;
constexpr uint64_t kSn5 = 0x3f811110e829872fULL;
constexpr uint64_t kCs2 = 0x3fe0000000000000ULL;
constexpr uint64_t kCs4 = 0xbfa5555555555535ULL;
constexpr uint64_t kCs6 = 0x3f56c16bedd9e239ULL;
constexpr uint64_t kS1 = 0xbfc5555555555555ULL;
constexpr uint64_t kS2 = 0x3f81111111110eceULL;
constexpr uint64_t kS3 = 0xbf2a01a019db08b8ULL;
constexpr uint64_t kS4 = 0x3ec71de27b9a7ed9ULL;
constexpr uint64_t kS5 = 0xbe5addffc2fcdf59ULL;
constexpr uint64_t kHp0 = 0x3ff921fb54442d18ULL;
constexpr uint64_t kHp1 = 0x3c91a62633145c07ULL;
constexpr uint64_t kToint = 0x4338000000000000ULL;
constexpr uint64_t kHpinv = 0x3fe45f306dc9c883ULL;
constexpr uint64_t kMp1 = 0x3ff921fb58000000ULL;
constexpr uint64_t kMp2 = 0xbe4dde973c000000ULL;
constexpr uint64_t kPp3 = 0xbc8cb3b398000000ULL;
constexpr uint64_t kPp4 = 0xbacd747f23e32ed7ULL;
constexpr uint64_t kTaylorMax = 0x3fc020c49ba5e354ULL;  // 0.126
}  // namespace cosc

// Optionally (PGN_GM_CONSTANT_BANK) the device reads the constants from a
// __constant__ table as constant-bank operands instead of 64-bit immediates;
// measured neutral-to-slower on B200 (f6 8D k_evaluate +3%), so immediates are
// the default.  Same bit patterns either way.
enum GmConst {
  kGm_expc_kInvLn2N, kGm_expc_kShift, kGm_expc_kNegLn2hiN, kGm_expc_kNegLn2loN, kGm_expc_kC2, kGm_expc_kC3, kGm_expc_kC4, kGm_expc_kC5, kGm_cosc_kBig, kGm_cosc_kSn3, kGm_cosc_kSn5, kGm_cosc_kCs2, kGm_cosc_kCs4, kGm_cosc_kCs6, kGm_cosc_kS1, kGm_cosc_kS2, kGm_cosc_kS3, kGm_cosc_kS4, kGm_cosc_kS5, kGm_cosc_kHp0, kGm_cosc_kHp1, kGm_cosc_kToint, kGm_cosc_kHpinv, kGm_cosc_kMp1, kGm_cosc_kMp2, kGm_cosc_kPp3, kGm_cosc_kPp4, kGm_cosc_kTaylorMax, kGmCount
};
#if defined(__CUDACC__)
static __constant__ uint64_t c_gm[kGmCount] = {
    expc::kInvLn2N, expc::kShift, expc::kNegLn2hiN, expc::kNegLn2loN, expc::kC2, expc::kC3, expc::kC4, expc::kC5, cosc::kBig, cosc::kSn3, cosc::kSn5, cosc::kCs2, cosc::kCs4, cosc::kCs6, cosc::kS1, cosc::kS2, cosc::kS3, cosc::kS4, cosc::kS5, cosc::kHp0, cosc::kHp1, cosc::kToint, cosc::kHpinv, cosc::kMp1, cosc::kMp2, cosc::kPp3, cosc::kPp4, cosc::kTaylorMax};
#endif
#if defined(__CUDA_ARCH__) && defined(PGN_GM_CONSTANT_BANK)
#define PGN_GM(ns, name) __longlong_as_double(static_cast<long long>(c_gm[kGm_##ns##_##name]))
#else
#define PGN_GM(ns, name) pgn_asf64(ns::name)
#endif
#define PGN_C(name) PGN_GM(cosc, name)

// e_exp.c specialcase(): result near the overflow/underflow boundaries.
PGN_HD double gm_exp_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ULL) == 0) {
    // k > 0: the exponent of scale may have overflowed by <= 460.
    sbits -= 1009ULL << 52;
    const double scale = pgn_asf64(sbits);
    return P_MUL(P_FMA(scale, tmp, scale), 0x1p1009);
  }
  // k < 0: careful rounding in the subnormal range (unfused in __exp_fma:
  // the product scale*tmp is reused for `lo`).
  sbits += 1022ULL << 52;
  const double scale = pgn_asf64(sbits);
  const double st = P_MUL(scale, tmp);
  double y = P_ADD(scale, st);
  if (y < 1.0) {
    double lo = P_ADD(P_SUB(scale, y), st);
    const double hi = P_ADD(1.0, y);
    lo = P_ADD(P_ADD(P_SUB(1.0, hi), y), lo);
    y = P_SUB(P_ADD(hi, lo), 1.0);
    if (y == 0.0) y = 0.0;  // avoid -0.0
  }
  return P_MUL(0x1p-1022, y);
}

// exp's polynomial / reduction constants as values.  By default they are the
// immediates below (so nvcc folds them); the evaluator can instead load them
// once per thread into registers (PGN_HOIST_EXP) so the hot loops do not
// re-materialise 64-bit immediates (2 MOVs each) on every call.
struct ExpK {
  double inv_ln2_n = pgn_asf64(expc::kInvLn2N);
  double neg_ln2hi_n = pgn_asf64(expc::kNegLn2hiN);
  double neg_ln2lo_n = pgn_asf64(expc::kNegLn2loN);
  double c2 = pgn_asf64(expc::kC2);
  double c3 = pgn_asf64(expc::kC3);
  double c4 = pgn_asf64(expc::kC4);
  double c5 = pgn_asf64(expc::kC5);
};

PGN_HD double gm_exp_k(double x, const uint64_t* __restrict__ T, const ExpK& K);

PGN_HD double gm_exp(double x, const uint64_t* __restrict__ T) {
#if defined(PGN_GM_CONSTANT_BANK) && defined(__CUDA_ARCH__)
  using namespace expc;
  const uint64_t ix = pgn_asu64(x);
  uint32_t abstop = static_cast<uint32_t>(ix >> 52) & 0x7ff;
  if (abstop - 0x3c9u >= 0x3fu) {
    if (static_cast<int32_t>(abstop - 0x3c9u) < 0) return P_ADD(1.0, x);  // |x| < 2^-54
    if (abstop >= 0x409u) {                                               // |x| >= 1024
      if (ix == 0xfff0000000000000ULL) return 0.0;
      if (abstop >= 0x7ffu) return P_ADD(1.0, x);
      if (ix >> 63) return 0.0;                          // __math_uflow(0)
      return pgn_asf64(0x7ff0000000000000ULL);           // __math_oflow(0)
    }
    abstop = 0;  // large |x|: handled by the special case below
  }
  double kd = P_FMA(x, PGN_GM(expc, kInvLn2N), PGN_GM(expc, kShift));
  const uint64_t ki = pgn_asu64(kd);
  kd = P_SUB(kd, PGN_GM(expc, kShift));
  double r = P_FMA(kd, PGN_GM(expc, kNegLn2hiN), x);
  r = P_FMA(kd, PGN_GM(expc, kNegLn2loN), r);
  const uint64_t idx = 2 * (ki & 127);
  const uint64_t top = ki << 45;
  const double tail = pgn_asf64(T[idx]);
  const uint64_t sbits = T[idx + 1] + top;
  const double p23 = P_FMA(r, PGN_GM(expc, kC3), PGN_GM(expc, kC2));
  const double tr = P_ADD(r, tail);
  const double r2 = P_MUL(r, r);
  const double p45 = P_FMA(r, PGN_GM(expc, kC5), PGN_GM(expc, kC4));
  const double t = P_FMA(p23, r2, tr);
  const double r4 = P_MUL(r2, r2);
  const double tmp = P_FMA(r4, p45, t);
  if (abstop == 0) return gm_exp_special(tmp, sbits, ki);
  const double scale = pgn_asf64(sbits);
  return P_FMA(scale, tmp, scale);
#else
  return gm_exp_k(x, T, ExpK{});
#endif
}

PGN_HD double gm_exp_k(double x, const uint64_t* __restrict__ T, const ExpK& K) {
  using namespace expc;
  const uint64_t ix = pgn_asu64(x);
  uint32_t abstop = static_cast<uint32_t>(ix >> 52) & 0x7ff;
  if (abstop - 0x3c9u >= 0x3fu) {
    if (static_cast<int32_t>(abstop - 0x3c9u) < 0) return P_ADD(1.0, x);  // |x| < 2^-54
    if (abstop >= 0x409u) {                                               // |x| >= 1024
      if (ix == 0xfff0000000000000ULL) return 0.0;
      if (abstop >= 0x7ffu) return P_ADD(1.0, x);
      if (ix >> 63) return 0.0;                          // __math_uflow(0)
      return pgn_asf64(0x7ff0000000000000ULL);           // __math_oflow(0)
    }
    abstop = 0;  // large |x|: handled by the special case below
  }
  double kd = P_FMA(x, K.inv_ln2_n, PGN_GM(expc, kShift));
  const uint64_t ki = pgn_asu64(kd);
  kd = P_SUB(kd, PGN_GM(expc, kShift));
  double r = P_FMA(kd, K.neg_ln2hi_n, x);
  r = P_FMA(kd, K.neg_ln2lo_n, r);
  const uint64_t idx = 2 * (ki & 127);
  const uint64_t top = ki << 45;
  const double tail = pgn_asf64(T[idx]);
  const uint64_t sbits = T[idx + 1] + top;
  const double p23 = P_FMA(r, K.c3, K.c2);
  const double tr = P_ADD(r, tail);
  const double r2 = P_MUL(r, r);
  const double p45 = P_FMA(r, K.c5, K.c4);
  const double t = P_FMA(p23, r2, tr);
  const double r4 = P_MUL(r2, r2);
  const double tmp = P_FMA(r4, p45, t);
  if (abstop == 0) return gm_exp_special(tmp, sbits, ki);
  const double scale = pgn_asf64(sbits);
  return P_FMA(scale, tmp, scale);
}

// ---- cos: sysdeps/ieee754/dbl-64/s_sin.c (glibc 2.39), __cos_fma ---------

// The non-immediate cos constants of the hot path as values (see ExpK):
// hoisted into registers by the evaluator (PGN_HOIST_COS), immediates otherwise.
struct CosK {
  double hpinv = pgn_asf64(cosc::kHpinv);
  double mp1 = pgn_asf64(cosc::kMp1);
  double mp2 = pgn_asf64(cosc::kMp2);
  double pp3 = pgn_asf64(cosc::kPp3);
  double pp4 = pgn_asf64(cosc::kPp4);
  double sn3 = pgn_asf64(cosc::kSn3);
  double sn5 = pgn_asf64(cosc::kSn5);
  double cs4 = pgn_asf64(cosc::kCs4);
  double cs6 = pgn_asf64(cosc::kCs6);
  double s1 = pgn_asf64(cosc::kS1);  // TAYLOR_SIN
  double s2 = pgn_asf64(cosc::kS2);
  double s3 = pgn_asf64(cosc::kS3);
  double s4 = pgn_asf64(cosc::kS4);
  double s5 = pgn_asf64(cosc::kS5);
  double taylor_max = pgn_asf64(cosc::kTaylorMax);
};

// s_sin.c do_cos(x, dx)
PGN_HD double gm_do_cos(double x, double dx, const double* __restrict__ SC,
                         const CosK& KC = CosK{}) {
  if (x < 0) dx = -dx;
  const double ax = pgn_fabs(x);
  const double u = P_ADD(PGN_C(kBig), ax);
  const double xr = P_ADD(P_SUB(ax, P_SUB(u, PGN_C(kBig))), dx);
  const double xx = P_MUL(xr, xr);
  const double s = P_FMA(P_MUL(xr, xx), P_FMA(xx, KC.sn5, KC.sn3), xr);
  const double c =
      P_MUL(xx, P_FMA(xx, P_FMA(xx, KC.cs6, KC.cs4), PGN_C(kCs2)));
  const int k = static_cast<int>(static_cast<uint32_t>(pgn_asu64(u)) << 2);
  const double sn = SC[k], ssn = SC[k + 1], cs = SC[k + 2], ccs = SC[k + 3];
  double cor = P_FMA(-s, ssn, ccs);
  cor = P_FMA(-c, cs, cor);
  cor = P_FMA(-s, sn, cor);
  return P_ADD(cs, cor);
}

// s_sin.c do_sin(x, dx), including the TAYLOR_SIN branch.
PGN_HD double gm_do_sin(double x, double dx, const double* __restrict__ SC,
                         const CosK& KC = CosK{}) {
  if (pgn_fabs(x) < PGN_C(kTaylorMax)) {
    const double xx = P_MUL(x, x);
    double p = P_FMA(PGN_C(kS5), xx, PGN_C(kS4));
    p = P_FMA(p, xx, PGN_C(kS3));
    p = P_FMA(p, xx, PGN_C(kS2));
    p = P_FMA(p, xx, PGN_C(kS1));
    const double t = P_FMA(xx, P_FMA(p, x, -P_MUL(0.5, dx)), dx);
    return P_ADD(x, t);
  }
  const double xold = x;
  if (x <= 0) dx = -dx;
  const double ax = pgn_fabs(x);
  const double u = P_ADD(PGN_C(kBig), ax);
  const double xr = P_SUB(ax, P_SUB(u, PGN_C(kBig)));
  const double xx = P_MUL(xr, xr);
  const double s = P_ADD(xr, P_FMA(P_MUL(xr, xx), P_FMA(xx, KC.sn5, KC.sn3), dx));
  const double c = P_FMA(
      xr, dx, P_MUL(xx, P_FMA(xx, P_FMA(xx, KC.cs6, KC.cs4), PGN_C(kCs2))));
  const int k = static_cast<int>(static_cast<uint32_t>(pgn_asu64(u)) << 2);
  const double sn = SC[k], ssn = SC[k + 1], cs = SC[k + 2], ccs = SC[k + 3];
  double cor = P_FMA(s, ccs, ssn);
  cor = P_FMA(-c, sn, cor);
  cor = P_FMA(s, cs, cor);
  const double r = P_ADD(sn, cor);
  return pgn_asf64((pgn_asu64(r) & 0x7fffffffffffffffULL) |
                   (pgn_asu64(xold) & 0x8000000000000000ULL));
}

// ---- __branred: sysdeps/ieee754/dbl-64/branred.c (glibc 2.39) -------------
// Payne-Hanek style reduction of |x| >= 105414350 by pi/2 with 2/pi in 24-bit
// digits (toverp).  The shipped routine has no FMA (plain SSE2 in libm.so.6,
// checked with objdump), so every operation is rounded on its own, in the C
// source's order.  Returns the quadrant; *a + *aa is the reduced argument.
#if defined(__CUDACC__)
static __constant__ uint64_t g_pgn_toverp[75] = PGN_TOVERP_INIT;
#endif
static const uint64_t h_pgn_toverp[75] = PGN_TOVERP_INIT;

struct BranredPart {
  double b, bb, sum;
};

PGN_HD BranredPart gm_branred_part(double xp, const uint64_t* tov) {
  constexpr double big = 0x1.8p52, big1 = 0x1.8p54, tm24 = 0x1p-24;
  double r[6];
  double sum = 0.0;
  int k = static_cast<int>((pgn_asu64(xp) >> 52) & 2047);
  k = (k - 450) / 24;
  if (k < 0) k = 0;
  // gor = 2^576 with (24 k) subtracted from its exponent
  double gor = pgn_asf64(0x63f0000000000000ULL - (static_cast<uint64_t>(k * 24) << 52));
  for (int i = 0; i < 6; ++i) {
    r[i] = P_MUL(P_MUL(xp, pgn_asf64(tov[k + i])), gor);
    gor = P_MUL(gor, tm24);
  }
  for (int i = 0; i < 3; ++i) {
    const double s = P_SUB(P_ADD(r[i], big), big);
    sum = P_ADD(sum, s);
    r[i] = P_SUB(r[i], s);
  }
  double t = 0.0;
  for (int i = 0; i < 6; ++i) t = P_ADD(t, r[5 - i]);
  double bb = P_ADD(P_ADD(P_ADD(P_ADD(P_ADD(P_SUB(r[0], t), r[1]), r[2]), r[3]), r[4]), r[5]);
  double s = P_SUB(P_ADD(t, big), big);
  sum = P_ADD(sum, s);
  t = P_SUB(t, s);
  const double b = P_ADD(t, bb);
  bb = P_ADD(P_SUB(t, b), bb);
  s = P_SUB(P_ADD(sum, big1), big1);
  sum = P_SUB(sum, s);
  return {b, bb, sum};
}

PGN_HD int gm_branred(double x, double* a, double* aa) {
#if defined(__CUDA_ARCH__)
  const uint64_t* tov = g_pgn_toverp;
#else
  const uint64_t* tov = h_pgn_toverp;
#endif
  constexpr double split = 0x1.0000002p27, tm600 = 0x1p-600;
  constexpr double hp0 = 0x1.921fb54442d18p+0, hp1 = 0x1.1a62633145c07p-54;
  constexpr double mp1 = 0x1.921fb58p+0, mp2 = -0x1.dde974p-27;
  x = P_MUL(x, tm600);
  double t = P_MUL(x, split);  // split x into two 26-bit halves
  const double x1 = P_SUB(t, P_SUB(t, x));
  const double x2 = P_SUB(x, x1);
  const BranredPart p1 = gm_branred_part(x1, tov);
  const BranredPart p2 = gm_branred_part(x2, tov);
  double sum = P_ADD(p1.sum, p2.sum);
  double b = P_ADD(p1.b, p2.b);
  double bb = pgn_fabs(p1.b) > pgn_fabs(p2.b) ? P_ADD(P_SUB(p1.b, b), p2.b)
                                               : P_ADD(P_SUB(p2.b, b), p1.b);
  if (b > 0.5) {
    b = P_SUB(b, 1.0);
    sum = P_ADD(sum, 1.0);
  } else if (b < -0.5) {
    b = P_ADD(b, 1.0);
    sum = P_SUB(sum, 1.0);
  }
  double s = P_ADD(b, P_ADD(P_ADD(bb, p1.bb), p2.bb));
  t = P_ADD(P_ADD(P_SUB(b, s), bb), P_ADD(p1.bb, p2.bb));
  b = P_MUL(s, split);
  const double t1 = P_SUB(b, P_SUB(b, s));
  const double t2 = P_SUB(s, t1);
  b = P_MUL(s, hp0);
  bb = P_ADD(P_ADD(P_ADD(P_SUB(P_MUL(t1, mp1), b), P_MUL(t1, mp2)), P_MUL(t2, mp1)),
             P_ADD(P_ADD(P_MUL(t2, mp2), P_MUL(s, hp1)), P_MUL(t, hp0)));
  s = P_ADD(b, bb);
  t = P_ADD(P_SUB(b, s), bb);
  *a = s;
  *aa = t;
  return static_cast<int>(sum) & 3;  // quadrant
}

// True when |x| < 105414350 (reduce_sincos range; __branred beyond).
PGN_HD bool gm_cos_in_range(double x) {
  const uint32_t k = static_cast<uint32_t>(pgn_asu64(x) >> 32) & 0x7fffffffu;
  return k < 0x419921fbu;
}

PGN_HD double gm_cos(double x, const double* __restrict__ SC, const CosK& KC = CosK{}) {
  const uint32_t k = static_cast<uint32_t>(pgn_asu64(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;          // |x| < 2^-27
  if (k < 0x3feb6000u) return gm_do_cos(x, 0.0, SC, KC);  // |x| < 0.855469
  if (k < 0x400368fdu) {                     // |x| < 2.426265
    const double y = P_SUB(PGN_C(kHp0), pgn_fabs(x));
    const double a = P_ADD(y, PGN_C(kHp1));
    const double da = P_ADD(P_SUB(y, a), PGN_C(kHp1));
    return gm_do_sin(a, da, SC, KC);
  }
  if (k < 0x419921fbu) {                     // |x| < 105414350: reduce_sincos
    const double t = P_FMA(x, KC.hpinv, PGN_C(kToint));
    const double xn = P_SUB(t, PGN_C(kToint));
    const int n = static_cast<int>(pgn_asu64(t) & 3);
    const double y = P_FMA(-xn, KC.mp2, P_FMA(-xn, KC.mp1, x));
    const double t2 = P_FMA(-xn, KC.pp3, y);
    double db = P_FMA(-xn, KC.pp3, P_SUB(y, t2));
    const double b = P_FMA(-xn, KC.pp4, t2);
    db = P_ADD(db, P_FMA(-xn, KC.pp4, P_SUB(t2, b)));
    const double r = (n & 1) ? gm_do_sin(b, db, SC, KC) : gm_do_cos(b, db, SC, KC);
    return ((n + 1) & 2) ? -r : r;
  }
  if (k < 0x7ff00000u) {  // |x| >= 105414350: __branred, then do_sincos(a, da, n + 1)
    double a, da;
    const int m = gm_branred(x, &a, &da) + 1;
    const double r = (m & 1) ? gm_do_cos(a, da, SC, KC) : gm_do_sin(a, da, SC, KC);
    return (m & 2) ? -r : r;
  }
  return P_DIV(x, x);  // inf or nan -> nan
}

// Branch-free cos for SIMT: the same glibc arithmetic as gm_cos (every
// rounded operation identical), but with the paths merged by value selects
// so the lanes of a warp never diverge between do_sin / do_cos / TAYLOR_SIN /
// the argument-reduction branches.  Bit-equality with gm_cos (and libm) is
// checked on 1e8 samples by tests.  Operand-order notes:
//  * do_cos's s = fma(x*xx, ps, x) and do_sin's s = x + fma(x*xx, ps, dx) share
//    fma(x*xx, ps, sel) followed by a selected final add;
//  * do_cos's c = xx*pc equals fma(x, 0, xx*pc) exactly (xx*pc >= +0);
//  * the three cor fmas differ only in which table entry and sign they take.
PGN_HD double gm_sel(bool c, double a, double b) { return c ? a : b; }

PGN_HD double gm_cos_bf(double x, const double* __restrict__ SC) {
  const uint32_t k = static_cast<uint32_t>(pgn_asu64(x) >> 32) & 0x7fffffffu;
  const double ax = pgn_fabs(x);
  // path C: reduce_sincos (|x| < 105414350)
  const double t = P_FMA(x, PGN_C(kHpinv), PGN_C(kToint));
  const double xn = P_SUB(t, PGN_C(kToint));
  const int nq = static_cast<int>(pgn_asu64(t) & 3);
  const double y = P_FMA(-xn, PGN_C(kMp2), P_FMA(-xn, PGN_C(kMp1), x));
  const double t2 = P_FMA(-xn, PGN_C(kPp3), y);
  const double db0 = P_FMA(-xn, PGN_C(kPp3), P_SUB(y, t2));
  const double bC = P_FMA(-xn, PGN_C(kPp4), t2);
  const double dbC = P_ADD(db0, P_FMA(-xn, PGN_C(kPp4), P_SUB(t2, bC)));
  // path B: hp0 - |x|  (0.855469 <= |x| < 2.426265)
  const double yB = P_SUB(PGN_C(kHp0), ax);
  const double aB = P_ADD(yB, PGN_C(kHp1));
  const double daB = P_ADD(P_SUB(yB, aB), PGN_C(kHp1));
  const bool pA = k < 0x3feb6000u, pB = !pA && k < 0x400368fdu;
  const double a = pA ? x : (pB ? aB : bC);
  const double da = pA ? 0.0 : (pB ? daB : dbC);
  const bool is_cos = pA || (!pB && !(nq & 1));
  const bool neg = !pA && !pB && ((nq + 1) & 2);
  // do_sin / do_cos merged
  const double aa = pgn_fabs(a);
  const double dx = a < 0 ? -da : da;  // do_sin negates for a <= 0, but a == 0 is TAYLOR there
  const double u = P_ADD(PGN_C(kBig), aa);
  const double xr0 = P_SUB(aa, P_SUB(u, PGN_C(kBig)));
  const double xr = is_cos ? P_ADD(xr0, dx) : xr0;
  const double xx = P_MUL(xr, xr);
  const double ps = P_FMA(xx, PGN_C(kSn5), PGN_C(kSn3));
  const double pc = P_MUL(xx, P_FMA(xx, P_FMA(xx, PGN_C(kCs6), PGN_C(kCs4)), PGN_C(kCs2)));
  const double sp = P_FMA(P_MUL(xr, xx), ps, is_cos ? xr : dx);
  const double sv = is_cos ? sp : P_ADD(xr, sp);
  const double cv = P_FMA(xr, is_cos ? 0.0 : dx, pc);
  int ki = static_cast<int>(static_cast<uint32_t>(pgn_asu64(u)) << 2);
  // lanes whose result is discarded below (huge/inf/nan x) may compute any
  // index: keep the table read in bounds
  ki = (ki < 0 || ki > 436) ? 0 : ki;
  const double sn = SC[ki], ssn = SC[ki + 1], cs = SC[ki + 2], ccs = SC[ki + 3];
  const double A = is_cos ? -sv : sv;
  double cor = P_FMA(A, is_cos ? ssn : ccs, is_cos ? ccs : ssn);
  cor = P_FMA(-cv, is_cos ? cs : sn, cor);
  cor = P_FMA(A, is_cos ? sn : cs, cor);
  const double r0 = P_ADD(is_cos ? cs : sn, cor);
  double r = is_cos ? r0
                    : pgn_asf64((pgn_asu64(r0) & 0x7fffffffffffffffULL) |
                                (pgn_asu64(a) & 0x8000000000000000ULL));
  // TAYLOR_SIN branch of do_sin (|a| < 0.126)
  const double ta = P_MUL(a, a);
  double p = P_FMA(PGN_C(kS5), ta, PGN_C(kS4));
  p = P_FMA(p, ta, PGN_C(kS3));
  p = P_FMA(p, ta, PGN_C(kS2));
  p = P_FMA(p, ta, PGN_C(kS1));
  const double tt = P_FMA(ta, P_FMA(p, a, -P_MUL(0.5, da)), da);
  const double rT = P_ADD(a, tt);
  r = (!is_cos && aa < PGN_C(kTaylorMax)) ? rT : r;
  r = neg ? -r : r;
  // rare: |x| < 2^-27 -> 1; |x| >= 105414350 (__branred) / inf / nan
  if (k < 0x3e400000u) r = 1.0;
  if (k >= 0x419921fbu) r = gm_cos(x, SC);
  return r;
}

// ---------------------------------------------------------------------------
// Device hot-path variants (same arithmetic, bit-identical results; checked
// against gm_exp / gm_cos and libm by the tests).  Differences are in the
// instructions around the arithmetic only:
//  * the tables are read with 32-bit shared-memory addresses computed once per
//    kernel (a generic pointer made ptxas rebuild the shared window base --
//    S2UR + ULEA + LEA -- on every call);
//  * `-v` and copysign are sign-bit XORs (what gcc emits for the reference on
//    x86: xorpd), instead of an FP64 DADD(-0, -v) plus two FSELs;
//  * gm_cos tests the common range (2.43 <= |x| < 1.05e8, reduce_sincos)
//    first.
PGN_HD double pgn_xor_sign(double v, bool c) {
  return pgn_asf64(pgn_asu64(v) ^ (static_cast<uint64_t>(c) << 63));
}

#if defined(__CUDACC__)
struct SmemTab {  // a table in shared memory, by 32-bit shared address
  uint32_t a;
  __device__ __forceinline__ void ld2(int i, double& x, double& y) const {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a + 8u * i));
  }
  __device__ __forceinline__ void ld2u(int i, uint64_t& x, uint64_t& y) const {
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(a + 8u * i));
  }
};

__device__ __forceinline__ double gm_exp_s(double x, SmemTab T, const ExpK& K) {
  using namespace expc;
  const uint64_t ix = pgn_asu64(x);
  uint32_t abstop = static_cast<uint32_t>(ix >> 52) & 0x7ff;
  if (abstop - 0x3c9u >= 0x3fu) {
    if (static_cast<int32_t>(abstop - 0x3c9u) < 0) return P_ADD(1.0, x);  // |x| < 2^-54
    if (abstop >= 0x409u) {                                               // |x| >= 1024
      if (ix == 0xfff0000000000000ULL) return 0.0;
      if (abstop >= 0x7ffu) return P_ADD(1.0, x);
      if (ix >> 63) return 0.0;                          // __math_uflow(0)
      return pgn_asf64(0x7ff0000000000000ULL);           // __math_oflow(0)
    }
    abstop = 0;  // large |x|: handled by the special case below
  }
  double kd = P_FMA(x, K.inv_ln2_n, PGN_GM(expc, kShift));
  const uint64_t ki = pgn_asu64(kd);
  const int idx = 2 * static_cast<int>(ki & 127);
  uint64_t tail_b, sb;
  T.ld2u(idx, tail_b, sb);  // early: latency under the reduction
  kd = P_SUB(kd, PGN_GM(expc, kShift));
  double r = P_FMA(kd, K.neg_ln2hi_n, x);
  r = P_FMA(kd, K.neg_ln2lo_n, r);
  const uint64_t top = ki << 45;
  const double tail = pgn_asf64(tail_b);
  const uint64_t sbits = sb + top;
  const double p23 = P_FMA(r, K.c3, K.c2);
  const double tr = P_ADD(r, tail);
  const double r2 = P_MUL(r, r);
  const double p45 = P_FMA(r, K.c5, K.c4);
  const double t = P_FMA(p23, r2, tr);
  const double r4 = P_MUL(r2, r2);
  const double tmp = P_FMA(r4, p45, t);
  if (abstop == 0) return gm_exp_special(tmp, sbits, ki);
  const double scale = pgn_asf64(sbits);
  return P_FMA(scale, tmp, scale);
}

// exp of two independent arguments with the common path in straight-line
// code (so ptxas can interleave the two dependency chains) and the rare cases
// -- |x| < 2^-54, |x| >= 512, inf, nan -- fixed up afterwards, exactly as
// gm_exp_s computes them.  The common path is harmless on any input (the
// table index is masked), so it runs unconditionally.
__device__ __forceinline__ double gm_exp_fix(double x, uint64_t ix, uint32_t abstop, double tmp,
                                             uint64_t sbits, uint64_t ki) {
  if (static_cast<int32_t>(abstop - 0x3c9u) < 0) return P_ADD(1.0, x);  // |x| < 2^-54
  if (abstop >= 0x409u) {                                               // |x| >= 1024
    if (ix == 0xfff0000000000000ULL) return 0.0;
    if (abstop >= 0x7ffu) return P_ADD(1.0, x);
    if (ix >> 63) return 0.0;
    return pgn_asf64(0x7ff0000000000000ULL);
  }
  return gm_exp_special(tmp, sbits, ki);  // 512 <= |x| < 1024
}

// gm_exp_fix as straight-line code with selects (every case computed, the
// right one kept): the paired exp's fix-ups then cost one pass per warp
// instead of two divergent scalar passes with nested branches.  f4 in 8D/10D
// sends many points to the 512 <= |x| < 1024 special case and beyond, which
// made the divergent form the largest non-FP64 cost of k_evaluate at 10D.
__device__ __forceinline__ double gm_exp_fix_bf(double x, uint64_t ix, uint32_t abstop,
                                                double tmp, uint64_t sbits, uint64_t ki) {
  // 512 <= |x| < 1024: gm_exp_special, both signs of k
  const double sc_p = pgn_asf64(sbits - (1009ULL << 52));
  const double y_p = P_MUL(P_FMA(sc_p, tmp, sc_p), 0x1p1009);
  const double sc_n = pgn_asf64(sbits + (1022ULL << 52));
  const double st = P_MUL(sc_n, tmp);
  const double y = P_ADD(sc_n, st);
  double lo = P_ADD(P_SUB(sc_n, y), st);
  const double hi = P_ADD(1.0, y);
  lo = P_ADD(P_ADD(P_SUB(1.0, hi), y), lo);
  double y2 = P_SUB(P_ADD(hi, lo), 1.0);
  y2 = y2 == 0.0 ? 0.0 : y2;  // avoid -0.0
  const double y_n = P_MUL(0x1p-1022, y < 1.0 ? y2 : y);
  double r = (ki & 0x80000000ULL) == 0 ? y_p : y_n;
  // |x| >= 1024: -inf -> 0, inf / nan -> 1 + x, else under/overflow
  const double one_x = P_ADD(1.0, x);
  const double big = ix == 0xfff0000000000000ULL
                         ? 0.0
                         : (abstop >= 0x7ffu ? one_x
                                             : ((ix >> 63) ? 0.0
                                                           : pgn_asf64(0x7ff0000000000000ULL)));
  r = abstop >= 0x409u ? big : r;
  return static_cast<int32_t>(abstop - 0x3c9u) < 0 ? one_x : r;  // |x| < 2^-54
}

#ifndef PGN_EXP_FIX_BRANCHY
#define PGN_EXP_FIX_BRANCHY 1  // 0: straight-line gm_exp_fix_bf (measured 1-6% slower on f4 8D/10D)
#endif
__device__ __forceinline__ void gm_exp2_s(double x0, double x1, SmemTab T, const ExpK& K,
                                          double& y0, double& y1) {
  using namespace expc;
  const uint64_t ix0 = pgn_asu64(x0), ix1 = pgn_asu64(x1);
  const uint32_t at0 = static_cast<uint32_t>(ix0 >> 52) & 0x7ff;
  const uint32_t at1 = static_cast<uint32_t>(ix1 >> 52) & 0x7ff;
  double kd0 = P_FMA(x0, K.inv_ln2_n, PGN_GM(expc, kShift));
  double kd1 = P_FMA(x1, K.inv_ln2_n, PGN_GM(expc, kShift));
  const uint64_t ki0 = pgn_asu64(kd0), ki1 = pgn_asu64(kd1);
  uint64_t tb0, sb0, tb1, sb1;  // table loads first: latency under the reduction
  T.ld2u(2 * static_cast<int>(ki0 & 127), tb0, sb0);
  T.ld2u(2 * static_cast<int>(ki1 & 127), tb1, sb1);
  kd0 = P_SUB(kd0, PGN_GM(expc, kShift));
  kd1 = P_SUB(kd1, PGN_GM(expc, kShift));
  double r0 = P_FMA(kd0, K.neg_ln2hi_n, x0);
  double r1 = P_FMA(kd1, K.neg_ln2hi_n, x1);
  r0 = P_FMA(kd0, K.neg_ln2lo_n, r0);
  r1 = P_FMA(kd1, K.neg_ln2lo_n, r1);
  const uint64_t sbits0 = sb0 + (ki0 << 45), sbits1 = sb1 + (ki1 << 45);
  const double p23_0 = P_FMA(r0, K.c3, K.c2), p23_1 = P_FMA(r1, K.c3, K.c2);
  const double tr0 = P_ADD(r0, pgn_asf64(tb0)), tr1 = P_ADD(r1, pgn_asf64(tb1));
  const double r2_0 = P_MUL(r0, r0), r2_1 = P_MUL(r1, r1);
  const double p45_0 = P_FMA(r0, K.c5, K.c4), p45_1 = P_FMA(r1, K.c5, K.c4);
  const double t0 = P_FMA(p23_0, r2_0, tr0), t1 = P_FMA(p23_1, r2_1, tr1);
  const double r4_0 = P_MUL(r2_0, r2_0), r4_1 = P_MUL(r2_1, r2_1);
  const double tmp0 = P_FMA(r4_0, p45_0, t0), tmp1 = P_FMA(r4_1, p45_1, t1);
  const double sc0 = pgn_asf64(sbits0), sc1 = pgn_asf64(sbits1);
  y0 = P_FMA(sc0, tmp0, sc0);
  y1 = P_FMA(sc1, tmp1, sc1);
  // (Tried: sending x < -746 -- always +0 -- around the fix-up with a select;
  // +4% on f4 8D and +5% on f5/f6, B200.)
  const bool f0 = at0 - 0x3c9u >= 0x3fu, f1 = at1 - 0x3c9u >= 0x3fu;
#if PGN_EXP_FIX_BRANCHY
  if (f0 | f1) {
    if (f0) y0 = gm_exp_fix(x0, ix0, at0, tmp0, sbits0, ki0);
    if (f1) y1 = gm_exp_fix(x1, ix1, at1, tmp1, sbits1, ki1);
  }
#else
  if (f0 | f1) {  // one straight-line pass for both points
    const double z0 = gm_exp_fix_bf(x0, ix0, at0, tmp0, sbits0, ki0);
    const double z1 = gm_exp_fix_bf(x1, ix1, at1, tmp1, sbits1, ki1);
    y0 = f0 ? z0 : y0;
    y1 = f1 ? z1 : y1;
  }
#endif
}

__device__ __forceinline__ void gm_sc4(SmemTab SC, int k, double& sn, double& ssn, double& cs,
                                       double& ccs) {
  SC.ld2(k, sn, ssn);
  SC.ld2(k + 2, cs, ccs);
}

__device__ __forceinline__ double gm_do_cos_s(double x, double dx, SmemTab SC, const CosK& KC) {
  dx = pgn_xor_sign(dx, x < 0);
  const double ax = pgn_fabs(x);
  const double u = P_ADD(PGN_C(kBig), ax);
  // table loads issued first (the asm loads stay where they are written), so
  // their latency overlaps the polynomials instead of stalling the FMAs below
  const int k = static_cast<int>(static_cast<uint32_t>(pgn_asu64(u)) << 2);
  double sn, ssn, cs, ccs;
  gm_sc4(SC, k, sn, ssn, cs, ccs);
  const double xr = P_ADD(P_SUB(ax, P_SUB(u, PGN_C(kBig))), dx);
  const double xx = P_MUL(xr, xr);
  const double s = P_FMA(P_MUL(xr, xx), P_FMA(xx, KC.sn5, KC.sn3), xr);
  const double c = P_MUL(xx, P_FMA(xx, P_FMA(xx, KC.cs6, KC.cs4), PGN_C(kCs2)));
  double cor = P_FMA(-s, ssn, ccs);
  cor = P_FMA(-c, cs, cor);
  cor = P_FMA(-s, sn, cor);
  return P_ADD(cs, cor);
}

__device__ __forceinline__ double gm_do_sin_s(double x, double dx, SmemTab SC, const CosK& KC) {
  if (pgn_fabs(x) < KC.taylor_max) {
    const double xx = P_MUL(x, x);
    double p = P_FMA(KC.s5, xx, KC.s4);
    p = P_FMA(p, xx, KC.s3);
    p = P_FMA(p, xx, KC.s2);
    p = P_FMA(p, xx, KC.s1);
    const double t = P_FMA(xx, P_FMA(p, x, -P_MUL(0.5, dx)), dx);
    return P_ADD(x, t);
  }
  const uint64_t xsign = pgn_asu64(x) & 0x8000000000000000ULL;
  dx = pgn_xor_sign(dx, x <= 0);
  const double ax = pgn_fabs(x);
  const double u = P_ADD(PGN_C(kBig), ax);
  const int k = static_cast<int>(static_cast<uint32_t>(pgn_asu64(u)) << 2);
  double sn, ssn, cs, ccs;
  gm_sc4(SC, k, sn, ssn, cs, ccs);  // early, as in gm_do_cos_s
  const double xr = P_SUB(ax, P_SUB(u, PGN_C(kBig)));
  const double xx = P_MUL(xr, xr);
  const double s = P_ADD(xr, P_FMA(P_MUL(xr, xx), P_FMA(xx, KC.sn5, KC.sn3), dx));
  const double c =
      P_FMA(xr, dx, P_MUL(xx, P_FMA(xx, P_FMA(xx, KC.cs6, KC.cs4), PGN_C(kCs2))));
  double cor = P_FMA(s, ccs, ssn);
  cor = P_FMA(-c, sn, cor);
  cor = P_FMA(s, cs, cor);
  const double r = P_ADD(sn, cor);
  return pgn_asf64((pgn_asu64(r) & 0x7fffffffffffffffULL) | xsign);
}

// do_sin and do_cos (s_sin.c) as ONE instruction stream: q = 1 selects do_sin,
// q = 0 do_cos.  The two routines share their structure -- the same table
// lookup and polynomials, three FMAs into `cor` with the table values in a
// different arrangement -- so every operand that differs is chosen by a
// select and each operation is the one the selected routine performs
// (identical results, bit for bit).  The lanes of a warp take different
// quadrants, so the branchy form executed both routines for most warps; this
// form executes one, plus do_sin's TAYLOR_SIN (|x| < 0.126), also selected.
#ifndef PGN_COS_MERGED
#define PGN_COS_MERGED 0  // A/B knob: measured +22% k_evaluate time on f1 8D (B200)
#endif
__device__ __forceinline__ double gm_do_sc_s(double x, double dx, bool q, SmemTab SC,
                                             const CosK& KC) {
  // TAYLOR_SIN (do_sin, |x| < taylor_max)
  const double xt = P_MUL(x, x);
  double p = P_FMA(KC.s5, xt, KC.s4);
  p = P_FMA(p, xt, KC.s3);
  p = P_FMA(p, xt, KC.s2);
  p = P_FMA(p, xt, KC.s1);
  const double r_taylor = P_ADD(x, P_FMA(xt, P_FMA(p, x, -P_MUL(0.5, dx)), dx));
  // table-driven core
  const uint64_t xsign = pgn_asu64(x) & 0x8000000000000000ULL;
  const double dxs = pgn_xor_sign(dx, q ? (x <= 0) : (x < 0));
  const double ax = pgn_fabs(x);
  const double u = P_ADD(PGN_C(kBig), ax);
  const double xr0 = P_SUB(ax, P_SUB(u, PGN_C(kBig)));
  const double xr = q ? xr0 : P_ADD(xr0, dxs);              // do_cos folds dx in here
  const double xx = P_MUL(xr, xr);
  const double t = P_FMA(P_MUL(xr, xx), P_FMA(xx, KC.sn5, KC.sn3), q ? dxs : xr);
  const double s = q ? P_ADD(xr, t) : t;                    // sin: x + (dx + x^3 p)
  const double cp = P_MUL(xx, P_FMA(xx, P_FMA(xx, KC.cs6, KC.cs4), PGN_C(kCs2)));
  const double c = q ? P_FMA(xr, dxs, cp) : cp;            // sin: x dx + x^2 q
  const int k = static_cast<int>(static_cast<uint32_t>(pgn_asu64(u)) << 2);
  double sn, ssn, cs, ccs;
  gm_sc4(SC, k, sn, ssn, cs, ccs);
  const double ms = pgn_xor_sign(s, !q);                    // cos uses -s
  double cor = P_FMA(ms, q ? ccs : ssn, q ? ssn : ccs);
  cor = P_FMA(-c, q ? sn : cs, cor);
  cor = P_FMA(ms, q ? cs : sn, cor);
  const double r = P_ADD(q ? sn : cs, cor);
  const double rs = pgn_asf64((pgn_asu64(r) & 0x7fffffffffffffffULL) | xsign);  // copysign
  return q ? (pgn_fabs(x) < KC.taylor_max ? r_taylor : rs) : r;
}

// |x| >= 105414350 off the hot path: out of line, so the evaluator's register
// allocation and instruction footprint do not carry the reduction.
static __device__ __noinline__ double gm_cos_big_s(double x, SmemTab SC) {
  double a, da;
  const int m = gm_branred(x, &a, &da) + 1;
  const CosK KC{};
  const double r = (m & 1) ? gm_do_cos_s(a, da, SC, KC) : gm_do_sin_s(a, da, SC, KC);
  return (m & 2) ? -r : r;
}

__device__ __forceinline__ double gm_cos_s(double x, SmemTab SC, const CosK& KC) {
  const uint32_t k = static_cast<uint32_t>(pgn_asu64(x) >> 32) & 0x7fffffffu;
  if (k - 0x400368fdu < 0x419921fbu - 0x400368fdu) {  // 2.426265 <= |x| < 105414350
    const double t = P_FMA(x, KC.hpinv, PGN_C(kToint));
    const double xn = P_SUB(t, PGN_C(kToint));
    const int n = static_cast<int>(pgn_asu64(t) & 3);
    const double y = P_FMA(-xn, KC.mp2, P_FMA(-xn, KC.mp1, x));
    const double t2 = P_FMA(-xn, KC.pp3, y);
    double db = P_FMA(-xn, KC.pp3, P_SUB(y, t2));
    const double b = P_FMA(-xn, KC.pp4, t2);
    db = P_ADD(db, P_FMA(-xn, KC.pp4, P_SUB(t2, b)));
#if PGN_COS_MERGED
    const double r = gm_do_sc_s(b, db, (n & 1) != 0, SC, KC);
#else
    const double r = (n & 1) ? gm_do_sin_s(b, db, SC, KC) : gm_do_cos_s(b, db, SC, KC);
#endif
    return pgn_xor_sign(r, ((n + 1) & 2) != 0);
  }
  if (k < 0x3e400000u) return 1.0;                         // |x| < 2^-27
  if (k < 0x3feb6000u) return gm_do_cos_s(x, 0.0, SC, KC);  // |x| < 0.855469
  if (k < 0x400368fdu) {                                   // |x| < 2.426265
    const double y = P_SUB(PGN_C(kHp0), pgn_fabs(x));
    const double a = P_ADD(y, PGN_C(kHp1));
    const double da = P_ADD(P_SUB(y, a), PGN_C(kHp1));
    return gm_do_sin_s(a, da, SC, KC);
  }
  if (k < 0x7ff00000u) return gm_cos_big_s(x, SC);  // |x| >= 105414350: __branred
  return P_DIV(x, x);                               // inf or nan -> nan
}
// cos of two independent arguments (f1): the reduce_sincos reductions of both
// points run as straight-line code (interleaved chains); do_sin / do_cos stay
// branches per point -- the lanes of a warp hold neighbouring regions and
// rarely diverge there.  Measured on B200 (f1 8D k_evaluate): this form -5%;
// a merged branch-free sin/cos core +10% (more issued instructions for the
// same FP64 work); paired same-branch do_cos/do_sin cores +16% (code size).
__device__ __forceinline__ void gm_cos2_s(double x0, double x1, SmemTab SC, const CosK& KC,
                                          double& y0, double& y1) {
  const uint32_t k0 = static_cast<uint32_t>(pgn_asu64(x0) >> 32) & 0x7fffffffu;
  const uint32_t k1 = static_cast<uint32_t>(pgn_asu64(x1) >> 32) & 0x7fffffffu;
  if ((k0 - 0x400368fdu < 0x419921fbu - 0x400368fdu) &
      (k1 - 0x400368fdu < 0x419921fbu - 0x400368fdu)) {
    const double t0 = P_FMA(x0, KC.hpinv, PGN_C(kToint));
    const double t1 = P_FMA(x1, KC.hpinv, PGN_C(kToint));
    const double xn0 = P_SUB(t0, PGN_C(kToint)), xn1 = P_SUB(t1, PGN_C(kToint));
    const int n0 = static_cast<int>(pgn_asu64(t0) & 3), n1 = static_cast<int>(pgn_asu64(t1) & 3);
    const double ya = P_FMA(-xn0, KC.mp2, P_FMA(-xn0, KC.mp1, x0));
    const double yb = P_FMA(-xn1, KC.mp2, P_FMA(-xn1, KC.mp1, x1));
    const double t2a = P_FMA(-xn0, KC.pp3, ya), t2b = P_FMA(-xn1, KC.pp3, yb);
    double dba = P_FMA(-xn0, KC.pp3, P_SUB(ya, t2a));
    double dbb = P_FMA(-xn1, KC.pp3, P_SUB(yb, t2b));
    const double ba = P_FMA(-xn0, KC.pp4, t2a), bb = P_FMA(-xn1, KC.pp4, t2b);
    dba = P_ADD(dba, P_FMA(-xn0, KC.pp4, P_SUB(t2a, ba)));
    dbb = P_ADD(dbb, P_FMA(-xn1, KC.pp4, P_SUB(t2b, bb)));
#if PGN_COS_MERGED  // straight-line: ptxas interleaves the two cores
    const double ra = gm_do_sc_s(ba, dba, (n0 & 1) != 0, SC, KC);
    const double rb = gm_do_sc_s(bb, dbb, (n1 & 1) != 0, SC, KC);
#else
    const double ra = (n0 & 1) ? gm_do_sin_s(ba, dba, SC, KC) : gm_do_cos_s(ba, dba, SC, KC);
    const double rb = (n1 & 1) ? gm_do_sin_s(bb, dbb, SC, KC) : gm_do_cos_s(bb, dbb, SC, KC);
#endif
    y0 = pgn_xor_sign(ra, ((n0 + 1) & 2) != 0);
    y1 = pgn_xor_sign(rb, ((n1 + 1) & 2) != 0);
  } else {
    y0 = gm_cos_s(x0, SC, KC);
    y1 = gm_cos_s(x1, SC, KC);
  }
}
#endif  // __CUDACC__

#undef PGN_C

}  // namespace pgn
