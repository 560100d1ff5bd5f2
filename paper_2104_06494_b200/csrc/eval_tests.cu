// k_evaluate instantiations for the reference unit-test integrands
// (generic full-point path, runtime dimension).
#include "kernels.cuh"

namespace pgn {

template <class F>
static EvalKernel pick(int mode) {
  return mode ? &k_evaluate_gen<F, 1> : &k_evaluate_gen<F, 0>;
}

EvalKernel lookup_eval_f1(int, int);
EvalKernel lookup_eval_f2(int, int);
EvalKernel lookup_eval_f3(int, int);
EvalKernel lookup_eval_f4(int, int);
EvalKernel lookup_eval_f5(int, int);
EvalKernel lookup_eval_f6(int, int);
EvalKernel lookup_eval_f7(int, int);
EvalKernel lookup_eval_f8(int, int);

EvalKernel lookup_evaluate(int fid, int n, int mode) {
  if (n < 1 || n > 16) return nullptr;
  switch (fid) {
    case 1: return lookup_eval_f1(n, mode);
    case 2: return lookup_eval_f2(n, mode);
    case 3: return lookup_eval_f3(n, mode);
    case 4: return lookup_eval_f4(n, mode);
    case 5: return lookup_eval_f5(n, mode);
    case 6: return lookup_eval_f6(n, mode);
    case 7: return lookup_eval_f7(n, mode);
    case 8: return lookup_eval_f8(n, mode);
    case 100: return pick<TConst>(mode);
    case 101: return pick<TMonomial>(mode);
    case 102: return pick<TRough>(mode);
    case 103: return pick<TNanBox>(mode);
    case 104: return pick<TPocket>(mode);
    case 105: return pick<TCosSum>(mode);
    case 106: return pick<TExpSq>(mode);
    default: return nullptr;
  }
}

}  // namespace pgn
