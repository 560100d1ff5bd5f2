// FP64 dependent-chain latency and DADD/DMUL/DFMA issue rates on one SM (dev tool).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = __fma_rn(x, a, b); x = __fma_rn(x, a, b); x = __fma_rn(x, a, b); x = __fma_rn(x, a, b); }
  long long t1 = clock64();
  if (x == 1234.5) out[0] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void latadd(double* out, long long* cyc, int iters, double a) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = __dadd_rn(x, a); x = __dadd_rn(x, a); x = __dadd_rn(x, a); x = __dadd_rn(x, a); }
  long long t1 = clock64();
  if (x == 1234.5) out[0] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8);
  long long h; int it = 100000;
  lat<<<1, 32>>>(o, c, it, 0.999999, 1e-7); cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, c, it, 0.999999, 1e-7); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / (4.0 * it));
  latadd<<<1, 32>>>(o, c, it, 1e-7); cudaDeviceSynchronize();
  latadd<<<1, 32>>>(o, c, it, 1e-7); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", (double)h / (4.0 * it));
  for (int w : {1, 2, 4, 8, 16}) {
    lat<<<1, 32 * w>>>(o, c, it, 0.999999, 1e-7); cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("warps/SM=%2d: %.2f cycles per dependent DFMA step\n", w, (double)h / (4.0 * it));
  }
  return 0;
}
