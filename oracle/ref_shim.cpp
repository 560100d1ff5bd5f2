// TEST INFRASTRUCTURE ONLY (oracle).  Never linked into or called by the
// product path; only tests/, __graft_entry__.smoke() and bench.py's CPU
// baseline / `--impl reference` arm load the library built from this file.
//
// A thin extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libbfcub_ref.so).  It exposes the reference's public API
// (include/bfcub/*.hpp) with plain pointers so Python tests can call it via
// ctypes:
//   integrate            driver.hpp:77-79
//   evaluate_batch       rule.hpp:67-68
//   build_rule           rule.hpp:53
//   two_level_refine     errorest.hpp:20-29
//   rel_err_classify / threshold_classify / filter   classify.hpp:16-62
//   bisect / uniform_split / initial_subdivisions     geometry.hpp:50-59
//   block_sum / block_sum_where / count_flags / min_max   reduce.hpp:13-22
// plus a full-precision per-iteration trace obtained by re-driving those
// public functions in driver.cpp:124-213 order (the reference's own
// BFCUB_TRACE line prints only 4-7 digits); ref_trace's final result is
// checked against ref_integrate's by tests/test_oracle.py.
//
// Integrand ids: 1..8 = the reference suite f1..f8 (integrands.cpp:24-79);
// 100+ = the lambdas of the reference's unit tests, parameterised (see
// include/pagani.h PAGANI_TEST_* for the identical device versions).

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "bfcub/classify.hpp"
#include "bfcub/driver.hpp"
#include "bfcub/errorest.hpp"
#include "bfcub/geometry.hpp"
#include "bfcub/integrands.hpp"
#include "bfcub/reduce.hpp"
#include "bfcub/rule.hpp"
#include "bfcub/sequential.hpp"

using namespace bfcub;

namespace {

thread_local std::string g_err;

struct TestCtx {
  double p[32];
};

// ---- parameterised versions of the reference unit-test lambdas ----------
// 100: constant  (test_driver.cpp:22-32, test_rule.cpp:82-91)
double t_const(const double*, int, void* c) { return static_cast<TestCtx*>(c)->p[0]; }
// 101: monomial prod x_i^e_i by repeated multiplication (test_rule.cpp:40-49)
//      also x[0]*x[1] (test_driver.cpp:93-100) with exponents (1,1).
double t_monomial(const double* x, int n, void* c) {
  const double* e = static_cast<TestCtx*>(c)->p;
  double v = 1.0;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < static_cast<int>(e[i]); ++k) v *= x[i];
  return v;
}
// 102: rough: sum cos(p0*x) (p1 != 2) or cos((p0*x)*x) (p1 == 2), + p2*n
//      (test_driver.cpp:61-80 `cos(40.0 * x[i])`, :126-141 `cos(50.0 * x[i] * x[i])`)
double t_rough(const double* x, int n, void* c) {
  const double* p = static_cast<TestCtx*>(c)->p;
  double s = 0;
  for (int i = 0; i < n; ++i) s += std::cos(p[1] == 2.0 ? p[0] * x[i] * x[i] : p[0] * x[i]);
  return s + p[2] * n;
}
// 103: NaN box: NaN where x0 > p0 (and x1 > p1 when p1 >= 0), else 1
//      (test_rule.cpp:237-254, test_driver.cpp:111-124)
double t_nanbox(const double* x, int, void* c) {
  const double* p = static_cast<TestCtx*>(c)->p;
  const bool in = x[0] > p[0] && (p[1] < 0.0 || x[1] > p[1]);
  return in ? std::numeric_limits<double>::quiet_NaN() : 1.0;
}
// 104: corner pocket: 1 where x0,x1,x2 > p0 (test_rule.cpp:217-235)
double t_pocket(const double* x, int, void* c) {
  const double p = static_cast<TestCtx*>(c)->p[0];
  return x[0] > p && x[1] > p && x[2] > p ? 1.0 : 0.0;
}
// 105: scaled cosine sum p0 * sum cos(p[1+i]*3*x_i) (test_rule.cpp:191-215)
double t_cossum(const double* x, int n, void* c) {
  const double* p = static_cast<TestCtx*>(c)->p;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += std::cos(p[1 + i] * 3.0 * x[i]);
  return p[0] * s;
}
// 106: sum exp(x/3) + x^2 (test_rule.cpp:154-189)
double t_expsq(const double* x, int n, void*) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += std::exp(x[i] / 3.0) + x[i] * x[i];
  return s;
}

struct Fn {
  Integrand f;
  TestCtx ctx;
};

bool make_fn(int fid, const double* params, int nparams, Fn& out) {
  std::memset(&out.ctx, 0, sizeof out.ctx);
  for (int i = 0; i < nparams && i < 32; ++i) out.ctx.p[i] = params[i];
  if (fid >= 1 && fid <= 8) {
    out.f = integrand_by_id("f" + std::to_string(fid));
    return true;
  }
  double (*fn)(const double*, int, void*) = nullptr;
  switch (fid) {
    case 100: fn = t_const; break;
    case 101: fn = t_monomial; break;
    case 102: fn = t_rough; break;
    case 103: fn = t_nanbox; break;
    case 104: fn = t_pocket; break;
    case 105: fn = t_cossum; break;
    case 106: fn = t_expsq; break;
    default: g_err = "unknown integrand id " + std::to_string(fid); return false;
  }
  out.f = Integrand{fn, &out.ctx};
  return true;
}

}  // namespace

extern "C" {

struct ref_config {
  double tau_rel, tau_abs;
  int32_t it_max;
  int32_t init_subdiv;
  int64_t max_regions, init_target;
  int32_t rel_filtering_enabled, threads, validate_invariants, refiner;
  int32_t direction_change_limit, attempt_limit;
  double p_max_start, p_max_step, p_max_cap;
};

struct ref_event {
  int32_t iteration, success;
  int64_t batch_size, finished_count;
  double discarded_error, budget_limit;
};

struct ref_result {
  double estimate, errorest;
  int32_t status, iterations;
  int64_t regions_generated, eval_count;
  int32_t n_events, pad;
};

// One row per iteration, full precision, taken at the BFCUB_TRACE point
// (driver.cpp:174-182) plus the filter outcome.
struct ref_trace_row {
  int32_t it, trig_digits, trig_memory, thr_invoked;
  int64_t m, active_rel, active_final, kept;
  double v, e, v_f, e_f;        // accumulators before the filter update
  double fin_v, fin_e;          // filter finished sums
  int32_t thr_success, thr_accepted, thr_attempts, thr_dir_changes;
  double thr_threshold, thr_discarded, thr_budget;
  int64_t thr_finished;
};

const char* ref_last_error() { return g_err.c_str(); }

static Config to_cfg(const ref_config* c) {
  Config cfg;
  cfg.tau_rel = c->tau_rel;
  cfg.tau_abs = c->tau_abs;
  cfg.it_max = c->it_max;
  cfg.max_regions = c->max_regions;
  cfg.init_target = c->init_target;
  cfg.init_subdiv = c->init_subdiv;
  cfg.rel_filtering_enabled = c->rel_filtering_enabled != 0;
  cfg.threads = c->threads;
  cfg.validate_invariants = c->validate_invariants != 0;
  cfg.threshold_limits.direction_change_limit = c->direction_change_limit;
  cfg.threshold_limits.attempt_limit = c->attempt_limit;
  cfg.threshold_limits.p_max_start = c->p_max_start;
  cfg.threshold_limits.p_max_step = c->p_max_step;
  cfg.threshold_limits.p_max_cap = c->p_max_cap;
  return cfg;
}

static void no_refine(std::span<const double>, std::span<const double> raw,
                      std::span<const double>, std::span<const double>,
                      std::span<double> out) {
  for (std::size_t j = 0; j < raw.size(); ++j) out[j] = raw[j];
}

// returns 0 ok, -1 invalid_argument, -2 runtime_error, -3 logic_error, -4 other
#define REF_TRY(...)                                \
  try {                                             \
    __VA_ARGS__                                     \
  } catch (const std::invalid_argument& e) {        \
    g_err = e.what();                               \
    return -1;                                      \
  } catch (const std::logic_error& e) {             \
    g_err = e.what();                               \
    return -3;                                      \
  } catch (const std::runtime_error& e) {           \
    g_err = e.what();                               \
    return -2;                                      \
  } catch (const std::exception& e) {               \
    g_err = e.what();                               \
    return -4;                                      \
  }

int ref_integrate(int fid, const double* params, int nparams, int ndim,
                  const double* lo, const double* hi, const ref_config* c,
                  ref_result* out, ref_event* events, int max_events) {
  REF_TRY({
    Fn fn;
    if (!make_fn(fid, params, nparams, fn)) return -1;
    Config cfg = to_cfg(c);
    if (c->refiner == 1) cfg.refiner = &no_refine;
    Bounds b(std::vector<double>(lo, lo + ndim), std::vector<double>(hi, hi + ndim));
    IntegrationResult r = integrate(fn.f, b, cfg);
    out->estimate = r.estimate;
    out->errorest = r.errorest;
    out->status = static_cast<int>(r.status);
    out->iterations = r.iterations;
    out->regions_generated = r.regions_generated;
    out->eval_count = r.eval_count;
    out->n_events = static_cast<int>(r.threshold_events.size());
    for (int i = 0; i < out->n_events && i < max_events; ++i) {
      const auto& ev = r.threshold_events[i];
      events[i] = {ev.iteration, ev.success ? 1 : 0, ev.batch_size, ev.finished_count,
                   ev.discarded_error, ev.budget_limit};
    }
    return 0;
  })
}

int ref_integrate_sequential(int fid, const double* params, int nparams, int ndim,
                             const double* lo, const double* hi, double tau_rel,
                             double tau_abs, int64_t max_evals, ref_result* out) {
  REF_TRY({
    Fn fn;
    if (!make_fn(fid, params, nparams, fn)) return -1;
    Bounds b(std::vector<double>(lo, lo + ndim), std::vector<double>(hi, hi + ndim));
    IntegrationResult r = integrate_sequential(fn.f, b, tau_rel, tau_abs, max_evals);
    out->estimate = r.estimate;
    out->errorest = r.errorest;
    out->status = static_cast<int>(r.status);
    out->iterations = r.iterations;
    out->regions_generated = r.regions_generated;
    out->eval_count = r.eval_count;
    out->n_events = 0;
    return 0;
  })
}

// Re-drives driver.cpp:83-215 on the unit cube through the public batch API
// and records one ref_trace_row per iteration.  Returns the number of rows
// (<= max_rows) or a negative error code; *out gets the final result.
int ref_trace(int fid, const double* params, int nparams, int ndim,
              const ref_config* c, ref_result* out, ref_trace_row* rows,
              int max_rows) {
  REF_TRY({
    Fn fn;
    if (!make_fn(fid, params, nparams, fn)) return -1;
    Config cfg = to_cfg(c);
    cfg.validate();
    const int n = ndim;
    const RuleTable rule = build_rule(n);
    const int d = cfg.init_subdiv > 0 ? cfg.init_subdiv
                                      : initial_subdivisions(n, cfg.init_target);
    RegionBatch batch = uniform_split(Bounds::unit_cube(n), d, cfg.max_regions);
    IntegrationResult res;
    res.regions_generated = batch.count;
    Accumulators acc;
    double prev_total = std::numeric_limits<double>::quiet_NaN();
    const int digits = cfg.convergence_digits();
    int nrows = 0;
    auto finish = [&](Status s, int it) {
      out->estimate = acc.estimate();
      out->errorest = acc.errorest();
      out->status = static_cast<int>(s);
      out->iterations = it;
      out->regions_generated = res.regions_generated;
      out->eval_count = res.eval_count;
      out->n_events = static_cast<int>(res.threshold_events.size());
      return nrows;
    };
    for (int it = 1; it <= cfg.it_max; ++it) {
      EvalOutput eval = evaluate_batch(fn.f, batch, rule);
      res.eval_count += eval.eval_count;
      std::vector<double> refined;
      if (it == 1) {
        refined = std::move(eval.raw_errors);
      } else {
        refined.resize(batch.count);
        if (c->refiner == 1)
          no_refine(eval.estimates, eval.raw_errors, batch.parent_estimates,
                    batch.parent_errors, refined);
        else
          two_level_refine(eval.estimates, eval.raw_errors, batch.parent_estimates,
                           batch.parent_errors, refined);
      }
      batch.estimates = std::move(eval.estimates);
      batch.errors = std::move(refined);
      batch.split_axis = std::move(eval.split_axes);
      ClassifyFlags flags = rel_err_classify(batch.estimates, batch.errors, cfg.tau_rel,
                                             cfg.rel_filtering_enabled);
      acc.v = block_sum(batch.estimates);
      acc.e = block_sum(batch.errors);
      ref_trace_row row{};
      row.it = it;
      row.m = batch.count;
      row.active_rel = count_flags(flags, 1);
      if (check_termination(acc, cfg.tau_rel, cfg.tau_abs)) {
        row.v = acc.v; row.e = acc.e; row.v_f = acc.v_f; row.e_f = acc.e_f;
        row.active_final = row.active_rel;
        if (nrows < max_rows) rows[nrows] = row;
        ++nrows;
        return finish(Status::Converged, it);
      }
      if (it == cfg.it_max) {
        row.v = acc.v; row.e = acc.e; row.v_f = acc.v_f; row.e_f = acc.e_f;
        row.active_final = row.active_rel;
        if (nrows < max_rows) rows[nrows] = row;
        ++nrows;
        break;
      }
      const std::int64_t active_count = row.active_rel;
      const bool trig_memory = 2 * active_count > cfg.max_regions;
      const bool trig_digits = digits_converged(prev_total, acc.estimate(), digits);
      row.trig_digits = trig_digits;
      row.trig_memory = trig_memory;
      if (trig_digits || trig_memory) {
        const ThresholdResult tr =
            threshold_classify(flags, batch.errors, acc.estimate(), acc.errorest(), acc.e,
                               batch.count, cfg.tau_rel, cfg.threshold_limits);
        res.threshold_events.push_back({it, tr.success, batch.count, tr.finished_count,
                                        tr.discarded_error, tr.budget_limit});
        const bool affordable = acc.e_f + tr.discarded_error <=
                                0.25 * cfg.tau_rel * std::fabs(acc.estimate());
        row.thr_invoked = 1;
        row.thr_success = tr.success;
        row.thr_attempts = tr.attempts;
        row.thr_dir_changes = tr.direction_changes;
        row.thr_threshold = tr.threshold;
        row.thr_discarded = tr.discarded_error;
        row.thr_budget = tr.budget_limit;
        row.thr_finished = tr.finished_count;
        if (tr.success && (trig_memory || affordable)) {
          flags = tr.flags;
          row.thr_accepted = 1;
        }
      }
      row.v = acc.v; row.e = acc.e; row.v_f = acc.v_f; row.e_f = acc.e_f;
      row.active_final = count_flags(flags, 1);
      batch.active = flags;
      FilterResult filt = filter(batch, flags);
      row.fin_v = filt.finished_estimate;
      row.fin_e = filt.finished_error;
      row.kept = filt.kept.count;
      if (nrows < max_rows) rows[nrows] = row;
      ++nrows;
      acc.v_f += filt.finished_estimate;
      acc.e_f += filt.finished_error;
      acc.v -= filt.finished_estimate;
      acc.e -= filt.finished_error;
      prev_total = acc.estimate();
      if (filt.kept.count == 0) return finish(Status::MaxIterations, it);
      if (2 * filt.kept.count > cfg.max_regions) return finish(Status::MemoryExhausted, it);
      batch = bisect(filt.kept, cfg.max_regions);
      res.regions_generated += batch.count;
    }
    return finish(Status::MaxIterations, cfg.it_max);
  })
}

int64_t ref_rule_point_count(int n) { return rule_point_count(n); }

// weight_sets: 5 x N (set-major); points: N x n; probes: 4n
int ref_build_rule(int n, double* points, double* weight_sets, int* probes) {
  REF_TRY({
    const RuleTable r = build_rule(n);
    if (points) std::memcpy(points, r.points.data(), r.points.size() * 8);
    if (weight_sets)
      for (int k = 0; k < 5; ++k)
        std::memcpy(weight_sets + k * r.point_count, r.weight_sets[k].data(),
                    r.point_count * 8);
    if (probes)
      std::memcpy(probes, r.axis_probe_indices.data(), r.axis_probe_indices.size() * 4);
    return 0;
  })
}

// lows/lengths region-major (m x n), as RegionBatch stores them.
int ref_evaluate_batch(int fid, const double* params, int nparams, int n, int64_t m,
                       const double* lows, const double* lengths, double* est,
                       double* raw, int* axes, int64_t* eval_count) {
  REF_TRY({
    Fn fn;
    if (!make_fn(fid, params, nparams, fn)) return -1;
    RegionBatch b;
    b.resize(n, m);
    std::memcpy(b.lows.data(), lows, m * n * 8);
    std::memcpy(b.lengths.data(), lengths, m * n * 8);
    const RuleTable rule = build_rule(n);
    EvalOutput o = evaluate_batch(fn.f, b, rule);
    std::memcpy(est, o.estimates.data(), m * 8);
    std::memcpy(raw, o.raw_errors.data(), m * 8);
    std::memcpy(axes, o.split_axes.data(), m * 4);
    if (eval_count) *eval_count = o.eval_count;
    return 0;
  })
}

int ref_two_level_refine(int64_t m, const double* est, const double* raw,
                         const double* pest, const double* perr, double* out) {
  REF_TRY({
    two_level_refine(std::span<const double>(est, m), std::span<const double>(raw, m),
                     std::span<const double>(pest, m), std::span<const double>(perr, m),
                     std::span<double>(out, m));
    return 0;
  })
}

int ref_rel_err_classify(int64_t m, const double* est, const double* err, double tau,
                         int enabled, uint8_t* flags) {
  REF_TRY({
    auto f = rel_err_classify(std::span<const double>(est, m),
                              std::span<const double>(err, m), tau, enabled != 0);
    std::memcpy(flags, f.data(), m);
    return 0;
  })
}

struct ref_threshold_out {
  int32_t success, attempts, direction_changes, pad;
  double threshold, discarded_error, budget_limit;
  int64_t finished_count;
};

int ref_threshold_classify(int64_t m, const uint8_t* active, const double* errors,
                           double v_tot, double e_tot, double e_it, int64_t s_it,
                           double tau, const ref_config* lim, uint8_t* flags_out,
                           ref_threshold_out* out) {
  REF_TRY({
    ClassifyFlags a(active, active + m);
    ThresholdLimits L;
    if (lim) {
      L.direction_change_limit = lim->direction_change_limit;
      L.attempt_limit = lim->attempt_limit;
      L.p_max_start = lim->p_max_start;
      L.p_max_step = lim->p_max_step;
      L.p_max_cap = lim->p_max_cap;
    }
    auto r = threshold_classify(a, std::span<const double>(errors, m), v_tot, e_tot,
                                e_it, s_it, tau, L);
    std::memcpy(flags_out, r.flags.data(), r.flags.size());
    out->success = r.success;
    out->attempts = r.attempts;
    out->direction_changes = r.direction_changes;
    out->threshold = r.threshold;
    out->discarded_error = r.discarded_error;
    out->budget_limit = r.budget_limit;
    out->finished_count = r.finished_count;
    return 0;
  })
}

// filter(): batch arrays region-major; outputs sized m (kept prefix used).
int ref_filter(int n, int64_t m, const double* lows, const double* lengths,
               const double* est, const double* err, const int* axis,
               const double* pest, const double* perr, const uint8_t* flags,
               double* k_lows, double* k_lengths, double* k_est, double* k_err,
               int* k_axis, double* k_pest, double* k_perr, int64_t* kept,
               double* fin_est, double* fin_err, double* fin_vol) {
  REF_TRY({
    RegionBatch b;
    b.resize(n, m);
    std::memcpy(b.lows.data(), lows, m * n * 8);
    std::memcpy(b.lengths.data(), lengths, m * n * 8);
    std::memcpy(b.estimates.data(), est, m * 8);
    std::memcpy(b.errors.data(), err, m * 8);
    std::memcpy(b.split_axis.data(), axis, m * 4);
    std::memcpy(b.parent_estimates.data(), pest, m * 8);
    std::memcpy(b.parent_errors.data(), perr, m * 8);
    ClassifyFlags f(flags, flags + m);
    FilterResult r = filter(b, f);
    const int64_t k = r.kept.count;
    std::memcpy(k_lows, r.kept.lows.data(), k * n * 8);
    std::memcpy(k_lengths, r.kept.lengths.data(), k * n * 8);
    std::memcpy(k_est, r.kept.estimates.data(), k * 8);
    std::memcpy(k_err, r.kept.errors.data(), k * 8);
    std::memcpy(k_axis, r.kept.split_axis.data(), k * 4);
    std::memcpy(k_pest, r.kept.parent_estimates.data(), k * 8);
    std::memcpy(k_perr, r.kept.parent_errors.data(), k * 8);
    *kept = k;
    *fin_est = r.finished_estimate;
    *fin_err = r.finished_error;
    *fin_vol = r.finished_volume;
    return 0;
  })
}

int ref_bisect(int n, int64_t m, const double* lows, const double* lengths,
               const double* est, const double* err, const int* axis,
               int64_t max_regions, double* c_lows, double* c_lengths,
               double* c_pest, double* c_perr) {
  REF_TRY({
    RegionBatch b;
    b.resize(n, m);
    std::memcpy(b.lows.data(), lows, m * n * 8);
    std::memcpy(b.lengths.data(), lengths, m * n * 8);
    std::memcpy(b.estimates.data(), est, m * 8);
    std::memcpy(b.errors.data(), err, m * 8);
    std::memcpy(b.split_axis.data(), axis, m * 4);
    RegionBatch o = bisect(b, max_regions);
    std::memcpy(c_lows, o.lows.data(), 2 * m * n * 8);
    std::memcpy(c_lengths, o.lengths.data(), 2 * m * n * 8);
    std::memcpy(c_pest, o.parent_estimates.data(), 2 * m * 8);
    std::memcpy(c_perr, o.parent_errors.data(), 2 * m * 8);
    return 0;
  })
}

int ref_uniform_split(int n, const double* lo, const double* hi, int d,
                      int64_t max_regions, int64_t* count, double* lows,
                      double* lengths, int64_t cap) {
  REF_TRY({
    Bounds b(std::vector<double>(lo, lo + n), std::vector<double>(hi, hi + n));
    RegionBatch o = uniform_split(b, d, max_regions);
    *count = o.count;
    if (o.count <= cap) {
      std::memcpy(lows, o.lows.data(), o.count * n * 8);
      std::memcpy(lengths, o.lengths.data(), o.count * n * 8);
    }
    return 0;
  })
}

int ref_initial_subdivisions(int n, int64_t target) { return initial_subdivisions(n, target); }

double ref_block_sum(int64_t m, const double* x) {
  return block_sum(std::span<const double>(x, m));
}

double ref_block_sum_where(int64_t m, const double* x, const uint8_t* f, int which) {
  return block_sum_where(std::span<const double>(x, m), std::span<const uint8_t>(f, m),
                         static_cast<uint8_t>(which));
}

int ref_digits_converged(double a, double b, int digits) {
  return digits_converged(a, b, digits) ? 1 : 0;
}

int ref_convergence_digits(double tau) {
  Config c;
  c.tau_rel = tau;
  return c.convergence_digits();
}

double ref_reference_value(const char* id, int dim) {
  try {
    return reference_value(id, dim);
  } catch (const std::exception& e) {
    g_err = e.what();
    return std::numeric_limits<double>::quiet_NaN();
  }
}

// The platform libm, vectorised (glibc IFUNC-resolved exp/cos): the ground
// truth the device restatement in glibc_math.cuh must equal bit-for-bit.
void ref_libm_exp(int64_t m, const double* x, double* y) {
  for (int64_t i = 0; i < m; ++i) y[i] = std::exp(x[i]);
}
void ref_libm_cos(int64_t m, const double* x, double* y) {
  for (int64_t i = 0; i < m; ++i) y[i] = std::cos(x[i]);
}

double ref_call_integrand(int fid, const double* params, int nparams, const double* x,
                          int n) {
  Fn fn;
  if (!make_fn(fid, params, nparams, fn)) return std::numeric_limits<double>::quiet_NaN();
  return fn.f(x, n);
}

}  // extern "C"
