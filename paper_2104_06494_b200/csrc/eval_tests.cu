// k_evaluate instantiations for the reference unit-test integrands
// (generic full-point path, runtime dimension).
#include <mutex>
#include <set>
#include <utility>

#include "driver.hpp"
#include "kernels.cuh"

namespace pgn {

template <class F>
static EvalLaunch pick(int mode) {
  return {mode ? &k_evaluate_gen<F, 1> : &k_evaluate_gen<F, 0>, kGenericSmem, true};
}

EvalLaunch lookup_eval_f1(int, int);
EvalLaunch lookup_eval_f2(int, int);
EvalLaunch lookup_eval_f3(int, int);
EvalLaunch lookup_eval_f4(int, int);
EvalLaunch lookup_eval_f5(int, int);
EvalLaunch lookup_eval_f6(int, int);
EvalLaunch lookup_eval_f7(int, int);
EvalLaunch lookup_eval_f8(int, int);
EvalKernel lookup_eval_link_f1(int);
EvalKernel lookup_eval_link_f2(int);
EvalKernel lookup_eval_link_f3(int);
EvalKernel lookup_eval_link_f4(int);
EvalKernel lookup_eval_link_f5(int);
EvalKernel lookup_eval_link_f6(int);
EvalKernel lookup_eval_link_f7(int);
EvalKernel lookup_eval_link_f8(int);

EvalLaunch lookup_evaluate(int fid, int n, int mode) {
  if (n < 1 || n > 16) return {};
  // built-ins: the direct form + (parity mode) the deferred-bisection form
  using Direct = EvalLaunch (*)(int, int);
  using Linked = EvalKernel (*)(int);
  static const Direct direct[8] = {lookup_eval_f1, lookup_eval_f2, lookup_eval_f3, lookup_eval_f4,
                                   lookup_eval_f5, lookup_eval_f6, lookup_eval_f7, lookup_eval_f8};
  static const Linked linked[8] = {lookup_eval_link_f1, lookup_eval_link_f2, lookup_eval_link_f3,
                                   lookup_eval_link_f4, lookup_eval_link_f5, lookup_eval_link_f6,
                                   lookup_eval_link_f7, lookup_eval_link_f8};
  if (fid >= 1 && fid <= 8) {
    EvalLaunch k = direct[fid - 1](n, mode);
    if (mode == 0) k.fn_link = linked[fid - 1](n);
    return k;
  }
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
    default: return {};
  }
}

void launch_evaluate(const EvalLaunch& k, cudaStream_t st, const EvalParams& ep) {
  if (k.ext) {  // caller-compiled kernel (include/pagani_device.cuh)
    const int rc = k.ext->launch(&ep, static_cast<uint32_t>(sizeof(EvalParams)), device_exp_table(),
                                 device_sincos_table(), st, ep.m, k.mode, k.ext->user);
    if (rc != 0)
      throw CudaError(std::string("PAGANI_DEVICE_FN launch failed: ") +
                      cudaGetErrorString(static_cast<cudaError_t>(rc)));
    return;
  }
  const EvalKernel fn = ep.link ? k.fn_link : k.fn;
  if (!fn) throw std::logic_error("launch_evaluate: no deferred-bisection form of this kernel");
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> configured;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> g(mu);
    if (k.smem > 0 && configured.insert({dev, reinterpret_cast<const void*>(fn)}).second)
      cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                           cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(k.smem));
  }
  const unsigned grid = static_cast<unsigned>((ep.m + kEvalThreads - 1) / kEvalThreads);
  if (ep.link) {  // behind k_link: programmatic launch (pdl_wait in load_geometry)
    PGN_CK(launch_pdl(fn, dim3(grid), dim3(kEvalThreads), k.smem, st, ep, device_exp_table(),
                      device_sincos_table()));
  } else {
    fn<<<grid, kEvalThreads, k.smem, st>>>(ep, device_exp_table(), device_sincos_table());
  }
}

}  // namespace pgn
