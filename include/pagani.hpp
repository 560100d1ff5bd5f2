// pagani.hpp -- C++ mirror of the reference API (bfcub, /root/reference/proj/include/bfcub)
// over the C ABI in pagani.h.  Header-only; link with -lpagani_b200.
//
// Same names, field names and exception classes as the reference:
//   Status            driver.hpp:14
//   Bounds            geometry.hpp:11-23   (validated like geometry.cpp:9-23)
//   ThresholdLimits   classify.hpp:23-29
//   Config            driver.hpp:30-45     (refiner fn-pointer -> Refiner enum)
//   ThresholdEvent    driver.hpp:47-58
//   IntegrationResult driver.hpp:60-68
//   Integrand         integrand.hpp:8-13   (a device-evaluable descriptor)
//   integrate         driver.hpp:77-79
//   integrand_by_id   integrands.hpp:31
// Errors: std::invalid_argument / std::runtime_error / std::logic_error as in
// the reference; CUDA/NCCL failures and unsupported integrands throw
// pagani::device_error (a std::runtime_error).
//
// Drop-in: `namespace bfcub = pagani;` (PAGANI_BFCUB_ALIAS) lets code written
// as `bfcub::integrate(bfcub::integrand_by_id("f4"), bfcub::Bounds::unit_cube(5), cfg)`
// compile unchanged.  The one semantic difference is the integrand: a host
// function pointer cannot run on the GPU, so Integrand is a descriptor of a
// device implementation (no CPU fallback exists).
#ifndef PAGANI_HPP_
#define PAGANI_HPP_

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "pagani.h"

namespace pagani {

inline constexpr int kMaxDim = PAGANI_MAX_DIM;

enum class Status { Converged = 0, MaxIterations = 1, MemoryExhausted = 2 };

inline std::string to_string(Status s) {
  switch (s) {
    case Status::Converged: return "converged";
    case Status::MaxIterations: return "max_iterations";
    case Status::MemoryExhausted: return "memory_exhausted";
  }
  return "unknown";
}

struct device_error : std::runtime_error {
  int code;
  device_error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void check(int rc) {
  if (rc == PAGANI_OK) return;
  const std::string msg = pagani_last_error();
  switch (rc) {
    case PAGANI_E_INVALID: throw std::invalid_argument(msg);
    case PAGANI_E_RUNTIME: throw std::runtime_error(msg);
    case PAGANI_E_LOGIC: throw std::logic_error(msg);
    default: throw device_error(rc, msg);
  }
}

struct Bounds {
  std::vector<double> lower, upper;
  Bounds() = default;
  Bounds(std::vector<double> lo, std::vector<double> hi) : lower(std::move(lo)), upper(std::move(hi)) {
    if (lower.size() != upper.size()) throw std::invalid_argument("Bounds: lower/upper size mismatch");
    const int n = dim();
    if (n < 1 || n > kMaxDim) throw std::invalid_argument("Bounds: dimension must be in [1, 16]");
    for (int a = 0; a < n; ++a) {
      if (!(lower[a] < upper[a]))
        throw std::invalid_argument("Bounds: lower must be < upper on every axis");
      if (!std::isfinite(lower[a]) || !std::isfinite(upper[a]))
        throw std::invalid_argument("Bounds: entries must be finite");
    }
  }
  static Bounds unit_cube(int n) { return Bounds(std::vector<double>(n, 0.0), std::vector<double>(n, 1.0)); }
  int dim() const { return static_cast<int>(lower.size()); }
  double volume() const {
    double v = 1.0;
    for (int a = 0; a < dim(); ++a) v *= upper[a] - lower[a];
    return v;
  }
  bool is_unit_cube() const {
    for (int a = 0; a < dim(); ++a)
      if (lower[a] != 0.0 || upper[a] != 1.0) return false;
    return true;
  }
};

struct ThresholdLimits {
  int direction_change_limit = 4;
  int attempt_limit = 40;
  double p_max_start = 0.25;
  double p_max_step = 0.10;
  double p_max_cap = 0.95;
};

enum class Refiner { TwoLevel = PAGANI_REFINER_TWO_LEVEL, Identity = PAGANI_REFINER_IDENTITY };
enum class Mode { Parity = PAGANI_MODE_PARITY, Fast = PAGANI_MODE_FAST };

struct Config {
  double tau_rel = 1e-3;
  double tau_abs = 1e-20;
  int it_max = 100;
  std::int64_t max_regions = std::int64_t{1} << 22;
  std::int64_t init_target = std::int64_t{1} << 14;
  int init_subdiv = 0;
  bool rel_filtering_enabled = true;
  int threads = 0;  // accepted for source compatibility; the GPU ignores it
  bool validate_invariants = false;
  Refiner refiner = Refiner::TwoLevel;
  ThresholdLimits threshold_limits;
  // B200 extensions
  Mode mode = Mode::Parity;
  int device = 0;
  bool profile = false;
  void* comm = nullptr;  // pagani_comm_init_rank() for multi-GPU runs

  int convergence_digits() const { return pagani_convergence_digits(tau_rel); }
  void validate() const {
    if (!(tau_rel > 0.0)) throw std::invalid_argument("Config: tau_rel must be > 0");
    if (!(tau_abs >= 0.0)) throw std::invalid_argument("Config: tau_abs must be >= 0");
    if (it_max < 1) throw std::invalid_argument("Config: it_max must be >= 1");
    if (init_subdiv == 0 && max_regions < 2 * init_target)
      throw std::invalid_argument("Config: max_regions must be >= 2 * init_target");
  }
  pagani_config to_c() const {
    pagani_config c;
    pagani_config_default(&c);
    c.tau_rel = tau_rel;
    c.tau_abs = tau_abs;
    c.it_max = it_max;
    c.init_subdiv = init_subdiv;
    c.max_regions = max_regions;
    c.init_target = init_target;
    c.rel_filtering_enabled = rel_filtering_enabled;
    c.threads = threads;
    c.validate_invariants = validate_invariants;
    c.refiner = static_cast<int32_t>(refiner);
    c.direction_change_limit = threshold_limits.direction_change_limit;
    c.attempt_limit = threshold_limits.attempt_limit;
    c.p_max_start = threshold_limits.p_max_start;
    c.p_max_step = threshold_limits.p_max_step;
    c.p_max_cap = threshold_limits.p_max_cap;
    c.mode = static_cast<int32_t>(mode);
    c.device = device;
    c.profile = profile;
    c.comm = comm;
    return c;
  }
};

struct ThresholdEvent {
  int iteration = 0;
  bool success = false;
  std::int64_t batch_size = 0;
  std::int64_t finished_count = 0;
  double discarded_error = 0.0;
  double budget_limit = 0.0;
  double retained_fraction() const {
    return batch_size ? 1.0 - static_cast<double>(finished_count) / batch_size : 1.0;
  }
};

struct IntegrationResult {
  double estimate = 0.0;
  double errorest = 0.0;
  Status status = Status::MaxIterations;
  int iterations = 0;
  std::int64_t regions_generated = 0;
  std::int64_t eval_count = 0;
  std::vector<ThresholdEvent> threshold_events;
  double device_ms = 0.0;  // B200 extension
};

// Device-evaluable integrand descriptor (replaces {fn, ctx}).
struct Integrand {
  pagani_integrand desc{};
  Integrand() { pagani_integrand_builtin(&desc, PAGANI_F1, nullptr, 0); }
  explicit Integrand(int builtin_id, const std::vector<double>& params = {}) {
    pagani_integrand_builtin(&desc, builtin_id, params.data(), static_cast<int>(params.size()));
  }
};

inline Integrand integrand_by_id(const std::string& id) {
  if (id.size() == 2 && id[0] == 'f' && id[1] >= '1' && id[1] <= '8') return Integrand(id[1] - '0');
  throw std::invalid_argument("unknown integrand id: " + id);
}

inline bool known_integrand(const std::string& id) {
  return id.size() == 2 && id[0] == 'f' && id[1] >= '1' && id[1] <= '8';
}

inline IntegrationResult integrate(const Integrand& f, const Bounds& bounds, const Config& config) {
  config.validate();
  const pagani_config c = config.to_c();
  pagani_result r;
  check(pagani_integrate(&f.desc, bounds.dim(), bounds.lower.data(), bounds.upper.data(), &c, &r));
  IntegrationResult out;
  out.estimate = r.estimate;
  out.errorest = r.errorest;
  out.status = static_cast<Status>(r.status);
  out.iterations = r.iterations;
  out.regions_generated = r.regions_generated;
  out.eval_count = r.eval_count;
  out.device_ms = r.device_ms;
  const int ne = r.n_events < PAGANI_MAX_EVENTS ? r.n_events : PAGANI_MAX_EVENTS;
  for (int i = 0; i < ne; ++i)
    out.threshold_events.push_back({r.events[i].iteration, r.events[i].success != 0,
                                    r.events[i].batch_size, r.events[i].finished_count,
                                    r.events[i].discarded_error, r.events[i].budget_limit});
  return out;
}

// sequential.hpp:15-18 -- the reference's globally adaptive comparison engine.
inline IntegrationResult integrate_sequential(const Integrand& f, const Bounds& bounds,
                                              double tau_rel, double tau_abs = 1e-20,
                                              std::int64_t max_evals = 10'000'000,
                                              bool validate_invariants = false, int device = 0) {
  pagani_result r;
  check(pagani_integrate_sequential(&f.desc, bounds.dim(), bounds.lower.data(),
                                    bounds.upper.data(), tau_rel, tau_abs, max_evals,
                                    validate_invariants ? 1 : 0, device, PAGANI_MODE_PARITY, &r));
  IntegrationResult out;
  out.estimate = r.estimate;
  out.errorest = r.errorest;
  out.status = static_cast<Status>(r.status);
  out.iterations = r.iterations;
  out.regions_generated = r.regions_generated;
  out.eval_count = r.eval_count;
  return out;
}

// integrands.hpp reference_value (integrands.cpp:178-188), long double.
inline double reference_value(const std::string& id, int dim) {
  double v = 0.0;
  check(pagani_reference_value(id.c_str(), dim, 0, &v));
  return v;
}

inline bool check_termination(double v, double e, double v_f, double e_f, double tau_rel,
                              double tau_abs) {
  return pagani_check_termination(v, e, v_f, e_f, tau_rel, tau_abs) != 0;
}
inline bool digits_converged(double v_prev, double v_curr, int digits) {
  return pagani_digits_converged(v_prev, v_curr, digits) != 0;
}
inline int initial_subdivisions(int n, std::int64_t init_target) {
  return pagani_initial_subdivisions(n, init_target);
}
inline std::int64_t rule_point_count(int n) { return pagani_rule_point_count(n); }

}  // namespace pagani

#ifdef PAGANI_BFCUB_ALIAS
namespace bfcub = pagani;
#endif

#endif  // PAGANI_HPP_
