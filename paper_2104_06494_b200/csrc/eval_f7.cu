// k_evaluate instantiations for the reference integrand f7, n = 1..16,
// parity and fast modes (one TU per integrand so nvcc builds them in parallel).
#include "kernels.cuh"

namespace pgn {

template <int N>
static EvalLaunch pick_f7(int mode) {
  return {mode ? &k_evaluate_sep<N, F7, 1> : &k_evaluate_sep<N, F7, 0>, eval_smem_bytes<N>(), true};
}

EvalLaunch lookup_eval_f7(int n, int mode) {
  switch (n) {
    case 1: return pick_f7<1>(mode);
    case 2: return pick_f7<2>(mode);
    case 3: return pick_f7<3>(mode);
    case 4: return pick_f7<4>(mode);
    case 5: return pick_f7<5>(mode);
    case 6: return pick_f7<6>(mode);
    case 7: return pick_f7<7>(mode);
    case 8: return pick_f7<8>(mode);
    case 9: return pick_f7<9>(mode);
    case 10: return pick_f7<10>(mode);
    case 11: return pick_f7<11>(mode);
    case 12: return pick_f7<12>(mode);
    case 13: return pick_f7<13>(mode);
    case 14: return pick_f7<14>(mode);
    case 15: return pick_f7<15>(mode);
    case 16: return pick_f7<16>(mode);
    default: return {};
  }
}

}  // namespace pgn
