// FP64 roofline denominator: MEASURED_PEAKS.json carries HBM and bf16
// figures only, so the FP64 CUDA-core peak is measured here with a DFMA
// microbenchmark: 8 independent dependent-DFMA chains per
// thread, 8 CTAs x 256 threads per SM, timed with CUDA events.
#include "driver.hpp"

namespace {

constexpr int kChains = 8;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256) k_dfma_peak(double* out, long long* cycles, int iters,
                                                   double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = 1.0 + 1e-3 * (threadIdx.x + c);
  const unsigned long long g0 = globaltimer_ns();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = __fma_rn(x[c], a, b);
  }
  const long long t1 = clock64();
  const unsigned long long g1 = globaltimer_ns();
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
  // SM clock of this CTA's own span (cycles / ns); the kernel may run in waves
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    cycles[0] = t1 - t0;
    cycles[1] = static_cast<long long>(g1 - g0);
  }
}

}  // namespace

extern "C" int pagani_fp64_peak(int device, double seconds, double* tflops, double* sm_mhz) {
  try {
    PGN_CK(cudaSetDevice(device));
    cudaDeviceProp prop{};
    PGN_CK(cudaGetDeviceProperties(&prop, device));
    const int blocks = prop.multiProcessorCount * 8;
    pgn::DevBuf<double> out(1);
    pgn::DevBuf<long long> cyc(2);
    cudaEvent_t e0, e1;
    PGN_CK(cudaEventCreate(&e0));
    PGN_CK(cudaEventCreate(&e1));
    int iters = 4096;
    float ms = 0.0f;
    // warm up and scale the iteration count to ~`seconds`
    for (int pass = 0; pass < 8; ++pass) {
      PGN_CK(cudaEventRecord(e0));
      k_dfma_peak<<<blocks, 256>>>(out.p, cyc.p, iters, 0.9999999, 1e-7);
      PGN_CK(cudaEventRecord(e1));
      PGN_CK(cudaEventSynchronize(e1));
      PGN_CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms > 1e3 * seconds * 0.5) break;
      const double scale = (1e3 * seconds) / (ms > 0.01f ? ms : 0.01f);
      iters = static_cast<int>(iters * (scale > 64 ? 64 : (scale < 1.1 ? 1.1 : scale)));
    }
    long long cyc_ns[2] = {0, 1};
    PGN_CK(cudaMemcpy(cyc_ns, cyc.p, sizeof cyc_ns, cudaMemcpyDeviceToHost));
    const double flops = 2.0 * kChains * static_cast<double>(iters) * blocks * 256.0;
    *tflops = flops / (ms * 1e-3) / 1e12;
    if (sm_mhz)
      *sm_mhz = cyc_ns[1] > 0 ? 1e3 * static_cast<double>(cyc_ns[0]) / static_cast<double>(cyc_ns[1])
                              : 0.0;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return PAGANI_OK;
  } catch (const std::exception&) {
    return PAGANI_E_CUDA;
  }
}
