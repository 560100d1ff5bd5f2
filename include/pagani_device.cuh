// pagani_device.cuh -- user-defined GPU integrands for pagani::integrate.
//
// The reference takes any integrand as a host callback {fn, ctx}
// (/root/reference/proj/include/bfcub/integrand.hpp:8-13) and calls it per
// point from OpenMP workers.  A GPU cannot call host code, so a user integrand
// is a C++ functor compiled for the device in the caller's own translation
// unit: this header instantiates the PAGANI evaluation kernel for it
// (pgn::k_evaluate_fn: the reference's point order, strict weighted folds,
// fourth-difference split axis, two-level refinement and classification) and
// hands the library a launcher (pagani_device_fn, PAGANI_DEVICE_FN).  The rest
// of the iteration -- folds, threshold search, filter, bisection, multi-GPU
// sharding -- is the library's.
//
//   #include "pagani_device.cuh"
//   struct Gauss {                       // any trivially copyable functor
//     double a;
//     __device__ double operator()(const double* x, int n) const { ... }
//   };
//   auto f = pagani::device_integrand(Gauss{625.0});
//   pagani::IntegrationResult r = pagani::integrate(f, pagani::Bounds::unit_cube(8), cfg);
//
// A functor may instead take (const double* x, int n, const pagani::Math& m)
// and call m.exp(v) / m.cos(v): glibc 2.39's exp / cos bit for bit (the
// reference's std::exp / std::cos on x86-64), so such an integrand integrates
// to the same bits as the reference given the same arithmetic.
//
// Build (CUDA 12.9, B200):
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 --expt-relaxed-constexpr \
//        -I<repo>/include user.cu -L<repo>/paper_2104_06494_b200 -lpagani_b200
// The kernel and the library must come from the same checkout: the launcher
// carries sizeof(EvalParams) and the library rejects a mismatch.
//
// The kernel is instantiated per dimension (n = 1..PAGANI_DEVICE_MAX_DIM, 16
// by default, the reference's limit) so the functor inlines with a constant n
// and its coordinates stay in registers; define PAGANI_DEVICE_MAX_DIM lower
// to cut compile time.  The kernel also runs the deterministic 2048-block
// folds in its tail (as the built-ins do), which the sharded multi-GPU path
// needs.
#ifndef PAGANI_DEVICE_CUH_
#define PAGANI_DEVICE_CUH_

#include <cuda_runtime.h>

#include <type_traits>
#include <utility>

#include "../paper_2104_06494_b200/csrc/evaluate.cuh"
#include "pagani.hpp"

namespace pagani {

// glibc-exact math inside a device integrand (shared-memory tables of the
// evaluation kernel).
struct Math {
  const pgn::MathTables& T;
  __device__ double exp(double x) const { return pgn::tab_exp(x, T); }
  __device__ double cos(double x) const { return pgn::tab_cos(x, T); }
};

namespace detail {

template <class Fn>
struct MathAdapter {  // fn(x, n, Math) seen through the kernel's (x, n, MathTables)
  Fn fn;
  __device__ double operator()(const double* x, int n, const pgn::MathTables& T) const {
    return fn(x, n, Math{T});
  }
};

#ifndef PAGANI_DEVICE_MAX_DIM
#define PAGANI_DEVICE_MAX_DIM 16
#endif
static_assert(PAGANI_DEVICE_MAX_DIM >= 1 && PAGANI_DEVICE_MAX_DIM <= 16,
              "PAGANI_DEVICE_MAX_DIM must be in [1, 16]");

template <class K, int N>
void launch_dim(const pgn::EvalParams& P, const K& k, unsigned grid, const uint64_t* te,
                const double* ts, cudaStream_t st, int32_t mode) {
  if (mode == PAGANI_MODE_FAST)
    pgn::k_evaluate_fn<K, N, 1><<<grid, pgn::kEvalThreads, pgn::kGenericSmem, st>>>(P, te, ts, k);
  else
    pgn::k_evaluate_fn<K, N, 0><<<grid, pgn::kEvalThreads, pgn::kGenericSmem, st>>>(P, te, ts, k);
}

template <class K, int... Ns>
bool dispatch_dim(int n, const pgn::EvalParams& P, const K& k, unsigned grid, const uint64_t* te,
                  const double* ts, cudaStream_t st, int32_t mode,
                  std::integer_sequence<int, Ns...>) {
  return ((n == Ns + 1 ? (launch_dim<K, Ns + 1>(P, k, grid, te, ts, st, mode), true) : false) ||
          ...);
}

template <class K>
int launch_user_kernel(const void* params, uint32_t params_size, const void* exp_table,
                       const void* sincos_table, void* stream, int64_t m, int32_t mode,
                       void* user) {
  if (params_size != sizeof(pgn::EvalParams)) return static_cast<int>(cudaErrorInvalidValue);
  if (m <= 0) return 0;
  const pgn::EvalParams& P = *static_cast<const pgn::EvalParams*>(params);
  const K& k = *static_cast<const K*>(user);
  const unsigned grid = static_cast<unsigned>((m + pgn::kEvalThreads - 1) / pgn::kEvalThreads);
  const auto* te = static_cast<const uint64_t*>(exp_table);
  const auto* ts = static_cast<const double*>(sincos_table);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!dispatch_dim(P.n, P, k, grid, te, ts, st, mode,
                    std::make_integer_sequence<int, PAGANI_DEVICE_MAX_DIM>{}))
    return static_cast<int>(cudaErrorInvalidValue);  // n > PAGANI_DEVICE_MAX_DIM
  return static_cast<int>(cudaGetLastError());
}

}  // namespace detail

// An Integrand that owns the functor and its launcher.  Not copyable (the C
// descriptor points into it); keep it alive for the integrate() call.
template <class Fn>
class DeviceIntegrand : public Integrand {
  static_assert(std::is_trivially_copyable_v<Fn>,
                "a device integrand is passed to the kernel by value");
  using K = std::conditional_t<
      std::is_invocable_v<const Fn&, const double*, int, const Math&>, detail::MathAdapter<Fn>,
      Fn>;

 public:
  explicit DeviceIntegrand(const Fn& fn) : k_(make_k(fn)) {
    dfn_.magic = PAGANI_DEVICE_FN_MAGIC;
    dfn_.params_size = static_cast<uint32_t>(sizeof(pgn::EvalParams));
    dfn_.launch = &detail::launch_user_kernel<K>;
    dfn_.user = &k_;
    desc.kind = PAGANI_DEVICE_FN;
    desc.builtin_id = 0;
    desc.device_fn = &dfn_;
  }
  DeviceIntegrand(const DeviceIntegrand&) = delete;
  DeviceIntegrand& operator=(const DeviceIntegrand&) = delete;

 private:
  static K make_k(const Fn& fn) {
    if constexpr (std::is_same_v<K, Fn>)
      return fn;
    else
      return K{fn};
  }
  K k_;
  pagani_device_fn dfn_{};
};

template <class Fn>
DeviceIntegrand<Fn> device_integrand(const Fn& fn) {
  return DeviceIntegrand<Fn>(fn);
}

}  // namespace pagani

#endif  // PAGANI_DEVICE_CUH_
