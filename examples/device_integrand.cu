// Your own integrand on the GPU -- the B200 counterpart of passing a callback
// {fn, ctx} to bfcub::integrate (integrand.hpp:8-13).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 --expt-relaxed-constexpr \
//        -fmad=false -I include examples/device_integrand.cu \
//        -L paper_2104_06494_b200 -lpagani_b200 -Xlinker -rpath,paper_2104_06494_b200
//   ./a.out            # integrates an anisotropic Gaussian over [0,1]^6
#include <cmath>
#include <cstdio>

#include "pagani_device.cuh"

// exp(-sum a_i (x_i - c)^2): the "ctx" of the reference's callback becomes
// functor members (trivially copyable, passed to the kernel by value).
struct AnisoGauss {
  double c;
  double a[6];
  __device__ double operator()(const double* x, int n, const pagani::Math& m) const {
    double s = 0.0;
    for (int i = 0; i < n; ++i) {
      const double t = x[i] - c;
      s += a[i] * t * t;
    }
    return m.exp(-s);  // glibc-exact exp, like std::exp in the reference
  }
};

int main() {
  AnisoGauss g{0.5, {10.0, 20.0, 40.0, 80.0, 160.0, 320.0}};
  auto f = pagani::device_integrand(g);
  pagani::Config cfg;
  cfg.tau_rel = 1e-6;
  const pagani::IntegrationResult r = pagani::integrate(f, pagani::Bounds::unit_cube(6), cfg);
  double exact = 1.0;
  for (double a : g.a) exact *= std::sqrt(M_PI / a) * std::erf(0.5 * std::sqrt(a));
  std::printf("estimate %.16e  errorest %.3e  status %s  iterations %d  regions %lld\n",
              r.estimate, r.errorest, pagani::to_string(r.status).c_str(), r.iterations,
              static_cast<long long>(r.regions_generated));
  std::printf("true relative error %.3e\n", std::fabs(r.estimate - exact) / exact);
  return 0;
}
