// k_evaluate instantiations for one reference integrand (f1..f8), n = 1..16,
// parity and fast modes.  The Makefile compiles this file once per integrand
// with -DPGN_FID=k (objects eval_f1.o .. eval_f8.o), and once more with
// -DPGN_LINK=1 for the deferred-bisection forms (eval_l1.o .. eval_l8.o), so
// nvcc builds the sixteen heavy instantiation sets in parallel.
#include <utility>

#include "kernels.cuh"

#ifndef PGN_FID
#error "compile with -DPGN_FID=<1..8>"
#endif

#define PGN_CAT2(a, b) a##b
#define PGN_CAT(a, b) PGN_CAT2(a, b)
#define PGN_FUNCTOR PGN_CAT(F, PGN_FID)
#define PGN_LOOKUP PGN_CAT(lookup_eval_f, PGN_FID)

namespace pgn {

#if PGN_LINK
// -DPGN_LINK=1: the deferred-bisection forms (parity mode), a separate object
// so the build runs them in parallel with the direct forms.
#define PGN_LOOKUP_LINK PGN_CAT(lookup_eval_link_f, PGN_FID)
template <int... Ns>
static EvalKernel dispatch_link(int n, std::integer_sequence<int, Ns...>) {
  EvalKernel out = nullptr;
  ((n == Ns + 1 ? (out = &k_evaluate_sep<Ns + 1, PGN_FUNCTOR, 0, true>, 0) : 0), ...);
  return out;
}

EvalKernel PGN_LOOKUP_LINK(int n) {
  return dispatch_link(n, std::make_integer_sequence<int, 16>{});
}
#else
template <int N>
static EvalLaunch pick(int mode) {
  return {mode ? &k_evaluate_sep<N, PGN_FUNCTOR, 1> : &k_evaluate_sep<N, PGN_FUNCTOR, 0>,
          eval_smem_bytes<N>(), true};
}

template <int... Ns>
static EvalLaunch dispatch(int n, int mode, std::integer_sequence<int, Ns...>) {
  EvalLaunch out{};
  ((n == Ns + 1 ? (out = pick<Ns + 1>(mode), 0) : 0), ...);
  return out;
}

EvalLaunch PGN_LOOKUP(int n, int mode) {
  return dispatch(n, mode, std::make_integer_sequence<int, 16>{});
}
#endif

}  // namespace pgn
