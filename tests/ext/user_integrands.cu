// Test library for user-defined device integrands (include/pagani_device.cuh).
// Built by __graft_entry__.build() / tests/ext/Makefile; driven through ctypes
// by tests/test_gpu_device_fn.py.  Compiled with -fmad=false so `a * b + c`
// rounds twice, as in the reference (built without FMA).
#include <cstdint>

#include "pagani_device.cuh"

namespace {

// exp(-a * sum (x_i - c)^2): with (c, a) = (0.5, 625) the reference's f4
// (integrands.cpp:45-52) step for step.
struct Gauss {
  double c, a;
  __device__ double operator()(const double* x, int n, const pagani::Math& m) const {
    double s = 0.0;
    for (int i = 0; i < n; ++i) {
      const double t = x[i] - c;
      s += t * t;
    }
    return m.exp(-a * s);
  }
};

// cos(sum (i+1) x_i): the reference's f1 (integrands.cpp:24-28).
struct Oscillatory {
  __device__ double operator()(const double* x, int n, const pagani::Math& m) const {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += (i + 1) * x[i];
    return m.cos(s);
  }
};

// x_0 * x_1 * ... (plain (x, n) signature): the reference unit-test monomial
// with all exponents 1 (test_rule.cpp:40-49, PAGANI_TEST_MONOMIAL).
struct Product {
  __device__ double operator()(const double* x, int n) const {
    double v = 1.0;
    for (int i = 0; i < n; ++i) v *= x[i];
    return v;
  }
};

template <class Fn>
int run(const Fn& fn, int n, double tau, int relf, int mode, const double* lower,
        const double* upper, double* out_d, int64_t* out_i, void* comm = nullptr) {
  try {
    auto f = pagani::device_integrand(fn);
    pagani::Config cfg;
    cfg.comm = comm;
    cfg.tau_rel = tau;
    cfg.rel_filtering_enabled = relf != 0;
    cfg.mode = mode ? pagani::Mode::Fast : pagani::Mode::Parity;
    pagani::Bounds b = lower ? pagani::Bounds(std::vector<double>(lower, lower + n),
                                              std::vector<double>(upper, upper + n))
                             : pagani::Bounds::unit_cube(n);
    const pagani::IntegrationResult r = pagani::integrate(f, b, cfg);
    out_d[0] = r.estimate;
    out_d[1] = r.errorest;
    out_i[0] = static_cast<int>(r.status);
    out_i[1] = r.iterations;
    out_i[2] = r.regions_generated;
    out_i[3] = r.eval_count;
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

template <class Fn>
int batch(const Fn& fn, int n, int64_t m, const double* lows, const double* lens, double* est,
          double* raw, int32_t* axes) {
  auto f = pagani::device_integrand(fn);
  int64_t cnt = 0;
  return pagani_evaluate_batch(&f.desc, n, m, lows, lens, est, raw, axes, &cnt, 0);
}

}  // namespace

extern "C" {

// which: 0 Gauss(c, a) [params[0..1]], 1 Oscillatory, 2 Product
int user_integrate(int which, const double* params, int n, double tau, int relf, int mode,
                   const double* lower, const double* upper, double* out_d, int64_t* out_i) {
  switch (which) {
    case 0: return run(Gauss{params[0], params[1]}, n, tau, relf, mode, lower, upper, out_d, out_i);
    case 1: return run(Oscillatory{}, n, tau, relf, mode, lower, upper, out_d, out_i);
    case 2: return run(Product{}, n, tau, relf, mode, lower, upper, out_d, out_i);
    default: return -1;
  }
}

// The same, sharded over the ranks of `comm` (pagani_comm_init_rank / _host).
int user_integrate_comm(int which, const double* params, int n, double tau, int relf,
                        void* comm, double* out_d, int64_t* out_i) {
  switch (which) {
    case 0:
      return run(Gauss{params[0], params[1]}, n, tau, relf, 0, nullptr, nullptr, out_d, out_i,
                 comm);
    case 1: return run(Oscillatory{}, n, tau, relf, 0, nullptr, nullptr, out_d, out_i, comm);
    case 2: return run(Product{}, n, tau, relf, 0, nullptr, nullptr, out_d, out_i, comm);
    default: return -1;
  }
}

int user_evaluate_batch(int which, const double* params, int n, int64_t m, const double* lows,
                        const double* lens, double* est, double* raw, int32_t* axes) {
  switch (which) {
    case 0: return batch(Gauss{params[0], params[1]}, n, m, lows, lens, est, raw, axes);
    case 1: return batch(Oscillatory{}, n, m, lows, lens, est, raw, axes);
    case 2: return batch(Product{}, n, m, lows, lens, est, raw, axes);
    default: return -1;
  }
}

// A descriptor whose parameter-block size does not match the library's:
// pagani_integrate must reject it (PAGANI_E_INVALID) without launching.
int user_integrate_bad_abi(void) {
  auto f = pagani::device_integrand(Product{});
  pagani_device_fn bad = *f.desc.device_fn;
  bad.params_size += 8;
  pagani_integrand d = f.desc;
  d.device_fn = &bad;
  pagani_config c;
  pagani_config_default(&c);
  const double lo[2] = {0.0, 0.0}, hi[2] = {1.0, 1.0};
  pagani_result r;
  return pagani_integrate(&d, 2, lo, hi, &c, &r);
}

}  // extern "C"
