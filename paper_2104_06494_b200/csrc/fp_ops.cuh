// Explicitly rounded fp64 primitives shared by host and device code.
//
// The reference is built for x86-64 without -march, so every `a*b + c` in
// rule.cpp / integrands.cpp / classify.cpp is a separately rounded DMUL then
// DADD.  nvcc contracts such expressions into DFMA by default,
// so every parity-critical expression in this project is written with these
// macros: on the device they map to the `_rn` intrinsics, which are never
// contracted; on the host the TU is compiled with -ffp-contract=off.
#pragma once

#if defined(__CUDA_ARCH__)
#define PGN_HD __host__ __device__ __forceinline__
#define P_ADD(a, b) __dadd_rn((a), (b))
#define P_SUB(a, b) __dsub_rn((a), (b))
#define P_MUL(a, b) __dmul_rn((a), (b))
#define P_DIV(a, b) __ddiv_rn((a), (b))
#define P_FMA(a, b, c) __fma_rn((a), (b), (c))
#define P_SQRT(a) __dsqrt_rn(a)
#else
#include <cmath>
#include <cstring>
#ifdef __CUDACC__
#define PGN_HD __host__ __device__ inline
#else
#define PGN_HD inline
#endif
#define P_ADD(a, b) ((a) + (b))
#define P_SUB(a, b) ((a) - (b))
#define P_MUL(a, b) ((a) * (b))
#define P_DIV(a, b) ((a) / (b))
#define P_FMA(a, b, c) std::fma((a), (b), (c))
#define P_SQRT(a) std::sqrt(a)
#endif

#include <stdint.h>

PGN_HD uint64_t pgn_asu64(double x) {
#if defined(__CUDA_ARCH__)
  return static_cast<uint64_t>(__double_as_longlong(x));
#else
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
#endif
}

PGN_HD double pgn_asf64(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(u));
#else
  double x;
  std::memcpy(&x, &u, 8);
  return x;
#endif
}

PGN_HD double pgn_fabs(double x) { return pgn_asf64(pgn_asu64(x) & 0x7fffffffffffffffULL); }

PGN_HD bool pgn_isfinite(double x) {
  return (pgn_asu64(x) & 0x7ff0000000000000ULL) != 0x7ff0000000000000ULL;
}
