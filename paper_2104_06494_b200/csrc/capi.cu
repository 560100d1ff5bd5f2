// extern "C" boundary (include/pagani.h).  Exceptions map to the codes the
// reference's exception classes correspond to; CUDA failures get their own.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "driver.hpp"

namespace pgn {
double suite_reference_value(const std::string& id, int n, bool corrected, bool extended);
}  // namespace pgn

namespace {
thread_local std::string g_last_error;
}  // namespace

void pgn::set_last_error(const std::string& msg) { g_last_error = msg; }

namespace {

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return PAGANI_OK;
  } catch (const pgn::CudaError& e) {
    g_last_error = e.what();
    return PAGANI_E_CUDA;
  } catch (const pgn::NcclError& e) {
    g_last_error = e.what();
    return PAGANI_E_NCCL;
  } catch (const pgn::UnsupportedError& e) {
    g_last_error = e.what();
    return PAGANI_E_UNSUPPORTED;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return PAGANI_E_INVALID;
  } catch (const std::logic_error& e) {
    g_last_error = e.what();
    return PAGANI_E_LOGIC;
  } catch (const std::runtime_error& e) {
    g_last_error = e.what();
    return PAGANI_E_RUNTIME;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PAGANI_E_RUNTIME;
  }
}

// Batch-API device context: device 0's workspace stream.
struct Ctx {
  pgn::Workspace& ws;
  cudaStream_t st;
  Ctx() : ws(pgn::workspace_for(0)), st(ws.st) { PGN_CK(cudaSetDevice(ws.device)); }
};

template <class T>
void h2d(pgn::DevBuf<T>& d, const T* h, size_t n, cudaStream_t st) {
  d.alloc(n ? n : 1);
  if (n) PGN_CK(cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
}
template <class T>
void d2h(T* h, const T* d, size_t n, cudaStream_t st) {
  if (n) PGN_CK(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, st));
}

// region-major host (m x n) <-> axis-major device (n x cap)
std::vector<double> to_axis_major(const double* rm, int n, int64_t m, int64_t cap) {
  std::vector<double> am(static_cast<size_t>(n) * cap, 0.0);
  for (int64_t j = 0; j < m; ++j)
    for (int a = 0; a < n; ++a) am[a * cap + j] = rm[j * n + a];
  return am;
}
void to_region_major(const std::vector<double>& am, int n, int64_t m, int64_t cap, double* rm) {
  for (int64_t j = 0; j < m; ++j)
    for (int a = 0; a < n; ++a) rm[j * n + a] = am[a * cap + j];
}

double fold_scalar(Ctx& c, int64_t m, const double* d_x, const uint8_t* d_flag, int which,
                   int64_t* count) {
  const int64_t nblk = pgn::nblocks_of(m);
  pgn::DevBuf<double> part(nblk + 1), scratch(2 * nblk + 2);
  pgn::DevBuf<int64_t> cnt(nblk + 1);
  pgn::DevBuf<pgn::FoldScalars> sc(1);
  pgn::launch_fold_one(c.st, m, d_x, d_flag, which, part.p, cnt.p);
  pgn::launch_finalize(c.st, nblk, 1, part.p, d_flag ? cnt.p : nullptr, nullptr, scratch.p, sc.p);
  pgn::FoldScalars h{};
  d2h(&h, sc.p, 1, c.st);
  PGN_CK(cudaStreamSynchronize(c.st));
  if (count) *count = h.count;
  return h.sum[0];
}

}  // namespace

extern "C" {

int pagani_abi_version(void) { return PAGANI_ABI_VERSION; }
const char* pagani_last_error(void) { return g_last_error.c_str(); }

void pagani_config_default(pagani_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->tau_rel = 1e-3;
  c->tau_abs = 1e-20;
  c->it_max = 100;
  c->init_subdiv = 0;
  c->max_regions = int64_t{1} << 22;
  c->init_target = int64_t{1} << 14;
  c->rel_filtering_enabled = 1;
  c->threads = 0;
  c->validate_invariants = 0;
  c->refiner = PAGANI_REFINER_TWO_LEVEL;
  c->direction_change_limit = 4;
  c->attempt_limit = 40;
  c->p_max_start = 0.25;
  c->p_max_step = 0.10;
  c->p_max_cap = 0.95;
  c->mode = PAGANI_MODE_PARITY;
}

void pagani_integrand_builtin(pagani_integrand* f, int builtin_id, const double* params,
                              int n_params) {
  std::memset(f, 0, sizeof(*f));
  f->magic = PAGANI_INTEGRAND_MAGIC;
  f->kind = PAGANI_BUILTIN;
  f->builtin_id = builtin_id;
  f->n_params = n_params < 0 ? 0 : (n_params > PAGANI_MAX_PARAMS ? PAGANI_MAX_PARAMS : n_params);
  for (int i = 0; i < f->n_params; ++i) f->params[i] = params[i];
}

int pagani_device_count(int* count) {
  return guarded([&] { PGN_CK(cudaGetDeviceCount(count)); });
}

int pagani_release(void) {
  return guarded([&] { pgn::release_workspaces(); });
}

int pagani_integrate(const pagani_integrand* f, int ndim, const double* lower,
                     const double* upper, const pagani_config* cfg, pagani_result* out) {
  return guarded([&] { pgn::integrate(f, ndim, lower, upper, cfg, out); });
}

int64_t pagani_rule_point_count(int n) { return pgn::rule_point_count(n); }

int pagani_build_rule(int n, double* orbit_weights, double* generators, double* points,
                      double* weight_sets) {
  return guarded([&] {
    const pgn::RuleOrbits r = pgn::build_rule_orbits(n);
    if (orbit_weights)
      for (int k = 0; k < 5; ++k)
        for (int o = 0; o < 5; ++o) orbit_weights[k * 5 + o] = r.w[k][o];
    if (generators)
      for (int i = 0; i < 4; ++i) generators[i] = r.gen[i];
    pgn::expand_rule(r, points, weight_sets);
  });
}

int pagani_evaluate_batch(const pagani_integrand* f, int n, int64_t m, const double* lows,
                          const double* lengths, double* estimates, double* raw_errors,
                          int32_t* split_axes, int64_t* eval_count, int32_t mode) {
  return guarded([&] {
    if (n < 1 || n > 16) throw std::invalid_argument("evaluate_batch: dimension mismatch");
    const pgn::DeviceIntegrand di = pgn::resolve_integrand(f);
    const pgn::EvalLaunch k = pgn::evaluate_kernel(di, n, mode);
    if (!k.valid()) throw pgn::UnsupportedError("no device kernel for this integrand/dimension");
    const pgn::RuleOrbits rule = pgn::build_rule_orbits(n);
    if (eval_count) *eval_count = m * rule.point_count;
    if (m <= 0) return;
    Ctx c;
    const int64_t cap = m;
    std::vector<double> al = to_axis_major(lows, n, m, cap), an = to_axis_major(lengths, n, m, cap);
    pgn::DevBuf<double> dl, dn, est(m), err(m), raw(m);
    pgn::DevBuf<uint8_t> ax(m), fl(m);
    pgn::DevBuf<int32_t> ax32(m);
    h2d(dl, al.data(), al.size(), c.st);
    h2d(dn, an.data(), an.size(), c.st);
    pgn::EvalParams ep{};
    ep.m = m;
    ep.cap = cap;
    ep.low = dl.p;
    ep.len = dn.p;
    ep.est = est.p;
    ep.err = err.p;
    ep.raw = raw.p;
    ep.axis = ax.p;
    ep.flag = fl.p;
    ep.axis32 = ax32.p;
    ep.n = n;
    ep.tau = 1e-3;
    for (int kk = 0; kk < 5; ++kk)
      for (int o = 0; o < 5; ++o) ep.w[kk][o] = rule.w[kk][o];
    for (int i = 0; i < 4; ++i) ep.gen[i] = rule.gen[i];
    ep.ip = di.params;
    pgn::launch_evaluate(k, c.st, ep);
    PGN_CK(cudaGetLastError());
    d2h(estimates, est.p, m, c.st);
    d2h(raw_errors, raw.p, m, c.st);
    d2h(split_axes, ax32.p, m, c.st);
    PGN_CK(cudaStreamSynchronize(c.st));
  });
}

int pagani_two_level_refine(int64_t m, const double* est, const double* raw, const double* pest,
                            const double* perr, double* refined) {
  (void)perr;  // errorest.cpp:27-35 never reads parent errors
  return guarded([&] {
    if (m % 2 != 0) throw std::invalid_argument("two_level_refine: batch must pair siblings");
    if (m == 0) return;
    Ctx c;
    pgn::DevBuf<double> a, b, p, o(m);
    h2d(a, est, m, c.st);
    h2d(b, raw, m, c.st);
    h2d(p, pest, m, c.st);
    pgn::launch_refine(c.st, m, a.p, b.p, p.p, o.p);
    d2h(refined, o.p, m, c.st);
    PGN_CK(cudaStreamSynchronize(c.st));
  });
}

int pagani_rel_err_classify(int64_t m, const double* est, const double* err, double tau,
                            int32_t enabled, uint8_t* flags) {
  return guarded([&] {
    if (m == 0) return;
    Ctx c;
    pgn::DevBuf<double> a, b;
    pgn::DevBuf<uint8_t> f(m);
    h2d(a, est, m, c.st);
    h2d(b, err, m, c.st);
    pgn::launch_classify(c.st, m, a.p, b.p, tau, enabled, f.p);
    d2h(flags, f.p, m, c.st);
    PGN_CK(cudaStreamSynchronize(c.st));
  });
}

int pagani_apply_threshold(int64_t m, const double* err, double t, uint8_t* flags) {
  return guarded([&] {
    if (m == 0) return;
    Ctx c;
    pgn::DevBuf<double> b;
    pgn::DevBuf<uint8_t> f(m);
    h2d(b, err, m, c.st);
    pgn::launch_apply_threshold(c.st, m, b.p, t, f.p);
    d2h(flags, f.p, m, c.st);
    PGN_CK(cudaStreamSynchronize(c.st));
  });
}

int pagani_threshold_classify(int64_t m, const uint8_t* active, const double* errors,
                              double v_tot, double e_tot, double e_it, int64_t s_it,
                              double tau_rel, const pagani_config* limits, uint8_t* flags_out,
                              pagani_threshold_result* out) {
  return guarded([&] {
    if (s_it != m) throw std::invalid_argument("threshold_classify: array length mismatch");
    std::memset(out, 0, sizeof(*out));
    if (m > 0) std::memcpy(flags_out, active, m);
    if (m <= 0) return;
    pgn::Limits lim;
    if (limits) {
      lim.direction_change_limit = limits->direction_change_limit;
      lim.attempt_limit = limits->attempt_limit;
      lim.p_max_start = limits->p_max_start;
      lim.p_max_step = limits->p_max_step;
      lim.p_max_cap = limits->p_max_cap;
    }
    pgn::Workspace& ws = pgn::workspace_for(0);
    std::lock_guard<std::mutex> lock(ws.mu);
    PGN_CK(cudaSetDevice(ws.device));
    ws.ensure(1, m);
    pgn::DevBuf<double> d_err, d_est(m);
    pgn::DevBuf<uint8_t> d_fl, d_out(m);
    h2d(d_err, errors, m, ws.st);
    h2d(d_fl, active, m, ws.st);
    PGN_CK(cudaMemsetAsync(d_est.p, 0, m * sizeof(double), ws.st));
    const pgn::ThresholdOutcome r = pgn::device_threshold(ws, m, d_est.p, d_err.p, d_fl.p, v_tot,
                                                          e_tot, e_it, s_it, tau_rel, lim, nullptr);
    out->success = r.success;
    out->attempts = r.attempts;
    out->direction_changes = r.direction_changes;
    out->threshold = r.threshold;
    out->discarded_error = r.discarded;
    out->budget_limit = r.budget_limit;
    out->finished_count = r.finished_count;
    if (r.success) {
      pgn::launch_candidates(ws.st, m, r.threshold, d_fl.p, d_err.p, d_out.p);
      d2h(flags_out, d_out.p, m, ws.st);
      PGN_CK(cudaStreamSynchronize(ws.st));
    }
  });
}

int pagani_filter(int n, int64_t m, const double* lows, const double* lengths,
                  const double* estimates, const double* errors, const int32_t* split_axis,
                  const double* parent_estimates, const double* parent_errors,
                  const uint8_t* flags, double* kept_lows, double* kept_lengths,
                  double* kept_estimates, double* kept_errors, int32_t* kept_axis,
                  double* kept_parent_estimates, double* kept_parent_errors, int64_t* kept,
                  double* finished_estimate, double* finished_error, double* finished_volume) {
  return guarded([&] {
    *kept = 0;
    *finished_estimate = *finished_error = *finished_volume = 0.0;
    if (m <= 0) return;
    Ctx c;
    const int64_t cap = ((m + pgn::kBlock - 1) / pgn::kBlock) * pgn::kBlock;
    std::vector<double> al = to_axis_major(lows, n, m, cap), an = to_axis_major(lengths, n, m, cap);
    pgn::DevBuf<double> dl, dn, de, dr, dp, dq;
    pgn::DevBuf<int32_t> dax;
    pgn::DevBuf<uint8_t> df;
    h2d(dl, al.data(), al.size(), c.st);
    h2d(dn, an.data(), an.size(), c.st);
    h2d(de, estimates, m, c.st);
    h2d(dr, errors, m, c.st);
    h2d(dax, split_axis, m, c.st);
    h2d(dp, parent_estimates, m, c.st);
    h2d(dq, parent_errors, m, c.st);
    h2d(df, flags, m, c.st);
    // classify.cpp:104-105 finished sums; :108 kept count
    *finished_estimate = fold_scalar(c, m, de.p, df.p, 0, nullptr);
    int64_t kcount = 0;
    const int64_t nblk = pgn::nblocks_of(m);
    pgn::DevBuf<double> part(4 * nblk), scratch(2 * nblk + 2);
    pgn::DevBuf<int64_t> cnt(nblk), off(nblk);
    pgn::DevBuf<pgn::FoldScalars> sc(1);
    pgn::launch_fold_one(c.st, m, dr.p, df.p, 0, part.p, nullptr);
    pgn::launch_fold_one(c.st, m, dr.p, df.p, 1, part.p + nblk, cnt.p);  // counts of flag==1
    pgn::launch_finalize(c.st, nblk, 1, part.p, cnt.p, off.p, scratch.p, sc.p);
    pgn::FoldScalars h{};
    d2h(&h, sc.p, 1, c.st);
    PGN_CK(cudaStreamSynchronize(c.st));
    *finished_error = h.sum[0];
    kcount = h.count;
    pgn::DevBuf<double> kl(static_cast<size_t>(n) * cap), kn(static_cast<size_t>(n) * cap),
        ke(m), kr(m), kp(m), kq(m), fv(1);
    pgn::DevBuf<int32_t> ka(m);
    pgn::launch_compact(c.st, n, m, cap, df.p, off.p, dl.p, dn.p, de.p, dr.p, dax.p, dp.p, dq.p,
                        kl.p, kn.p, ke.p, kr.p, ka.p, kp.p, kq.p);
    pgn::launch_serial_volume(c.st, n, m, cap, dn.p, df.p, 0, fv.p);
    std::vector<double> hl(static_cast<size_t>(n) * cap), hn(static_cast<size_t>(n) * cap);
    d2h(hl.data(), kl.p, hl.size(), c.st);
    d2h(hn.data(), kn.p, hn.size(), c.st);
    d2h(kept_estimates, ke.p, kcount, c.st);
    d2h(kept_errors, kr.p, kcount, c.st);
    d2h(kept_axis, ka.p, kcount, c.st);
    d2h(kept_parent_estimates, kp.p, kcount, c.st);
    d2h(kept_parent_errors, kq.p, kcount, c.st);
    d2h(finished_volume, fv.p, 1, c.st);
    PGN_CK(cudaStreamSynchronize(c.st));
    to_region_major(hl, n, kcount, cap, kept_lows);
    to_region_major(hn, n, kcount, cap, kept_lengths);
    *kept = kcount;
  });
}

int pagani_bisect(int n, int64_t m, const double* lows, const double* lengths,
                  const double* estimates, const double* errors, const int32_t* split_axis,
                  int64_t max_regions, double* child_lows, double* child_lengths,
                  double* child_parent_estimates, double* child_parent_errors) {
  return guarded([&] {
    if (2 * m > max_regions) throw std::logic_error("bisect: doubling would exceed max_regions");
    if (m <= 0) return;
    Ctx c;
    const int64_t cap = ((m + pgn::kBlock - 1) / pgn::kBlock) * pgn::kBlock;
    const int64_t cap2 = 2 * cap;
    std::vector<double> al = to_axis_major(lows, n, m, cap), an = to_axis_major(lengths, n, m, cap);
    std::vector<uint8_t> ax8(m);
    for (int64_t j = 0; j < m; ++j) {
      if (split_axis[j] < 0 || split_axis[j] >= n)
        throw std::invalid_argument("bisect: split axis out of range");
      ax8[j] = static_cast<uint8_t>(split_axis[j]);
    }
    pgn::DevBuf<double> dl, dn, de, dr, cl(static_cast<size_t>(n) * cap2),
        cn(static_cast<size_t>(n) * cap2), cp(cap2), cq(cap2);
    pgn::DevBuf<uint8_t> dax;
    h2d(dl, al.data(), al.size(), c.st);
    h2d(dn, an.data(), an.size(), c.st);
    h2d(de, estimates, m, c.st);
    h2d(dr, errors, m, c.st);
    h2d(dax, ax8.data(), m, c.st);
    pgn::launch_split(c.st, n, m, cap, cap2, nullptr, 0, 0.0, nullptr, de.p, dr.p, dax.p, dl.p,
                      dn.p, cl.p, cn.p, cp.p, cq.p);
    PGN_CK(cudaGetLastError());
    std::vector<double> hl(static_cast<size_t>(n) * cap2), hn(static_cast<size_t>(n) * cap2);
    d2h(hl.data(), cl.p, hl.size(), c.st);
    d2h(hn.data(), cn.p, hn.size(), c.st);
    d2h(child_parent_estimates, cp.p, 2 * m, c.st);
    d2h(child_parent_errors, cq.p, 2 * m, c.st);
    PGN_CK(cudaStreamSynchronize(c.st));
    to_region_major(hl, n, 2 * m, cap2, child_lows);
    to_region_major(hn, n, 2 * m, cap2, child_lengths);
  });
}

int pagani_uniform_split(int n, const double* lower, const double* upper, int d,
                         int64_t max_regions, int64_t* count, double* lows, double* lengths,
                         int64_t capacity) {
  return guarded([&] {
    if (d < 1) throw std::invalid_argument("uniform_split: d must be >= 1");
    if (n < 1 || n > 16) throw std::invalid_argument("Bounds: dimension must be in [1, 16]");
    for (int a = 0; a < n; ++a) {
      if (!(lower[a] < upper[a]))
        throw std::invalid_argument("Bounds: lower must be < upper on every axis");
      if (!std::isfinite(lower[a]) || !std::isfinite(upper[a]))
        throw std::invalid_argument("Bounds: entries must be finite");
    }
    int64_t m = 1;
    for (int a = 0; a < n; ++a) {
      if (m > max_regions / d) throw std::runtime_error("uniform_split: d^n exceeds max_regions");
      m *= d;
    }
    if (m > max_regions) throw std::runtime_error("uniform_split: d^n exceeds max_regions");
    *count = m;
    if (m > capacity) return;
    Ctx c;
    double step[16];
    for (int a = 0; a < n; ++a) step[a] = (upper[a] - lower[a]) / d;
    pgn::DevBuf<double> dlo, dst, l(static_cast<size_t>(n) * m), ln(static_cast<size_t>(n) * m);
    h2d(dlo, lower, n, c.st);
    h2d(dst, static_cast<const double*>(step), n, c.st);
    pgn::launch_uniform_split(c.st, n, d, m, m, l.p, ln.p, dlo.p, dst.p);
    std::vector<double> hl(static_cast<size_t>(n) * m), hn(static_cast<size_t>(n) * m);
    d2h(hl.data(), l.p, hl.size(), c.st);
    d2h(hn.data(), ln.p, hn.size(), c.st);
    PGN_CK(cudaStreamSynchronize(c.st));
    to_region_major(hl, n, m, m, lows);
    to_region_major(hn, n, m, m, lengths);
  });
}

int pagani_initial_subdivisions(int n, int64_t init_target) {
  return pgn::initial_subdivisions(n, init_target);
}

int pagani_block_sum(int64_t m, const double* x, double* out) {
  return guarded([&] {
    *out = 0.0;
    if (m <= 0) return;
    Ctx c;
    pgn::DevBuf<double> d;
    h2d(d, x, m, c.st);
    *out = fold_scalar(c, m, d.p, nullptr, 0, nullptr);
  });
}

int pagani_block_sum_where(int64_t m, const double* x, const uint8_t* flags, int32_t which,
                           double* out) {
  return guarded([&] {
    *out = 0.0;
    if (m <= 0) return;
    Ctx c;
    pgn::DevBuf<double> d;
    pgn::DevBuf<uint8_t> f;
    h2d(d, x, m, c.st);
    h2d(f, flags, m, c.st);
    *out = fold_scalar(c, m, d.p, f.p, which, nullptr);
  });
}

int pagani_count_flags(int64_t m, const uint8_t* flags, int32_t which, int64_t* out) {
  return guarded([&] {
    *out = 0;
    if (m <= 0) return;
    Ctx c;
    pgn::DevBuf<double> z(m);
    pgn::DevBuf<uint8_t> f;
    PGN_CK(cudaMemsetAsync(z.p, 0, m * sizeof(double), c.st));
    h2d(f, flags, m, c.st);
    fold_scalar(c, m, z.p, f.p, which, out);
  });
}

int pagani_min_max(int64_t m, const double* x, double* lo, double* hi) {
  return guarded([&] {
    *lo = *hi = 0.0;
    if (m <= 0) return;
    Ctx c;
    pgn::DevBuf<double> d, o(2);
    pgn::DevBuf<unsigned long long> keys(2);
    h2d(d, x, m, c.st);
    pgn::launch_minmax(c.st, m, d.p, keys.p, o.p);
    double h[2];
    d2h(h, o.p, 2, c.st);
    PGN_CK(cudaStreamSynchronize(c.st));
    *lo = h[0];
    *hi = h[1];
  });
}

int pagani_check_termination(double v, double e, double v_f, double e_f, double tau_rel,
                             double tau_abs) {
  const double err = e + e_f;  // driver.cpp:43-46
  return (err <= std::fabs(v + v_f) * tau_rel || err <= tau_abs) ? 1 : 0;
}

int pagani_digits_converged(double v_prev, double v_curr, int digits) {
  return pgn::digits_converged(v_prev, v_curr, digits) ? 1 : 0;
}

int pagani_convergence_digits(double tau_rel) { return pgn::convergence_digits(tau_rel); }

int pagani_integrate_sequential(const pagani_integrand* f, int ndim, const double* lower,
                                const double* upper, double tau_rel, double tau_abs,
                                int64_t max_evals, int32_t validate_invariants, int32_t device,
                                int32_t mode, pagani_result* out) {
  return guarded([&] {
    pgn::integrate_sequential(f, ndim, lower, upper, tau_rel, tau_abs, max_evals,
                              validate_invariants, device, mode, out);
  });
}

int pagani_reference_value(const char* id, int n, int32_t flags, double* out) {
  return guarded([&] {
    if (!id || !out) throw std::invalid_argument("reference_value: null argument");
    *out = pgn::suite_reference_value(id, n, (flags & PAGANI_REFVAL_CORRECTED) != 0,
                                      (flags & PAGANI_REFVAL_EXTENDED) != 0);
  });
}

int pagani_math_exp(int64_t m, const double* x, double* y, int32_t on_device) {
  return guarded([&] {
    if (!on_device) {
      static const uint64_t T[] = PGN_EXP_TAB_INIT;
      for (int64_t i = 0; i < m; ++i) y[i] = pgn::gm_exp(x[i], T);
      return;
    }
    if (m <= 0) return;
    Ctx c;
    pgn::DevBuf<double> dx, dy(m);
    h2d(dx, x, m, c.st);
    pgn::launch_math(c.st, on_device == 2 ? 3 : 0, m, dx.p, dy.p);
    d2h(y, dy.p, m, c.st);
    PGN_CK(cudaStreamSynchronize(c.st));
  });
}

int pagani_math_cos(int64_t m, const double* x, double* y, int32_t on_device) {
  // on_device: 0 host build, 1 device gm_cos, 2 device branch-free gm_cos_bf,
  // 3 host build of gm_cos_bf
  return guarded([&] {
    if (on_device == 0 || on_device == 3) {
      static const uint64_t SC[] = PGN_SINCOS_TAB_INIT;
      const double* sc = reinterpret_cast<const double*>(SC);
      for (int64_t i = 0; i < m; ++i)
        y[i] = on_device ? pgn::gm_cos_bf(x[i], sc) : pgn::gm_cos(x[i], sc);
      return;
    }
    if (m <= 0) return;
    Ctx c;
    pgn::DevBuf<double> dx, dy(m);
    h2d(dx, x, m, c.st);
    pgn::launch_math(c.st, on_device == 2 ? 2 : (on_device == 4 ? 4 : 1), m, dx.p, dy.p);
    d2h(y, dy.p, m, c.st);
    PGN_CK(cudaStreamSynchronize(c.st));
  });
}

int pagani_call_integrand(const pagani_integrand* f, int n, int64_t m, const double* x,
                          double* y) {
  return guarded([&] {
    if (n < 1 || n > 16) throw std::invalid_argument("dimension out of range");
    const pgn::DeviceIntegrand di = pgn::resolve_integrand(f);
    if (m <= 0) return;
    Ctx c;
    pgn::DevBuf<double> dx, dy(m);
    h2d(dx, x, static_cast<size_t>(m) * n, c.st);
    pgn::launch_call_integrand(c.st, di.fid, n, m, dx.p, di.params, dy.p);
    PGN_CK(cudaGetLastError());
    d2h(y, dy.p, m, c.st);
    PGN_CK(cudaStreamSynchronize(c.st));
  });
}

}  // extern "C"
