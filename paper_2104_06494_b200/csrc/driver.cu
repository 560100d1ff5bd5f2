// The PAGANI iteration (Alg. 2) on one B200 (or R sharded GPUs): host C++
// makes every scalar decision exactly as /root/reference/proj/src/driver.cpp:83-215
// does; the region list never leaves HBM.  Per iteration:
//
//   k_evaluate  (prologue: the deferred bisection -- region j's row derived
//                from kept parent link[j >> 1] and stored; then rule +
//                integrand + 4th differences + two-level refine + rel-err
//                classify, fused; its tail folds each 2048-block serially:
//                partials of est, err, finished est/err, active counts,
//                error min/max)
//   k_finalize  (pairwise trees, kept offsets; programmatic launch) -> 64
//                bytes into mapped host memory, a published sequence number
//                (zero-copy hand-off)
//   -- host decisions --
//   [threshold search: per pass k_probe_multi (15 speculative thresholds) ->
//    k_finalize_multi -> 360 bytes zero-copy; the host replays the decisions]
//   k_link      (the filter: link + parent estimate per kept region)
//   [sharded: allgathered block records before the trees; k_split_bulk
//    (fused filter + bisect, TMA-staged rows) and the boundary exchange
//    after it -- DESIGN.md 7]
//
// Host arithmetic is compiled with -ffp-contract=off and uses the same
// expression order as the reference, so v, e, v_f, e_f, budgets and
// thresholds are bit-identical (tests/test_gpu_parity.py compares every
// per-iteration trace field with the reference library).
#include "driver.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <memory>

namespace pgn {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw CudaError(std::string("CUDA error: ") + cudaGetErrorString(e) + " at " + what);
  }
}

// ---------------------------------------------------------------------------
// Workspace
void Workspace::ensure(int n_, int64_t cap_) {
  cap_ = ((cap_ + kBlock - 1) / kBlock) * kBlock;
  if (cap_ <= cap && n_ <= n) return;
  PGN_CK(cudaSetDevice(device));
  const int64_t nc = cap_ > cap ? cap_ : cap;
  const int nn = n_ > n ? n_ : n;
  const int64_t nb = nc / kBlock;
  for (int b = 0; b < 2; ++b) {
    low[b].alloc(static_cast<size_t>(nn) * nc);
    len[b].alloc(static_cast<size_t>(nn) * nc);
  }
  pest.alloc(nc);
  link.alloc(nc / 2 + 1);
  est.alloc(nc);
  err.alloc(nc);
  axis.alloc(nc);
  flag.alloc(nc);
  flag2.alloc(nc);
  part_eval.alloc(4 * nb);
  part_probe.alloc(4 * nb);
  scratch.alloc(2 * nb + 2);
  cnt_eval.alloc(nb);
  cnt_probe.alloc(nb);
  off_eval.alloc(nb);
  off_probe.alloc(nb);
  blk_done.alloc(nb);
  PGN_CK(cudaMemset(blk_done.p, 0, nb * sizeof(int)));
  mm_blk.alloc(2 * nb);
  part_multi.alloc(2 * kMaxProbes * nb);
  cnt_multi.alloc(kMaxProbes * nb);
  scratch_multi.alloc(2 * 2 * kMaxProbes * nb + 2);
  if (!d_sc.p) {
    d_sc.alloc(2);
    mm_keys.alloc(2);
    mm_out.alloc(2);
    d_lower.alloc(16);
    d_step.alloc(16);
    d_tmp.alloc(4);
    PGN_CK(cudaMallocHost(&h_sc, 2 * sizeof(FoldScalars)));
    PGN_CK(cudaMallocHost(&h_mm, 4 * sizeof(double)));
    d_probe.alloc(1);
    PGN_CK(cudaMallocHost(&h_probe, sizeof(ProbeScalars)));
    PGN_CK(cudaHostAlloc(&h_probe_zc, sizeof(ProbeScalars), cudaHostAllocMapped));
    PGN_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_probe_zc), h_probe_zc, 0));
    spec_ps.alloc(1);
    probe_done.alloc(1);
    PGN_CK(cudaMemset(probe_done.p, 0, sizeof(int)));
    PGN_CK(cudaHostAlloc(&h_zc, sizeof(FoldScalars), cudaHostAllocMapped));
    PGN_CK(cudaHostAlloc(&h_ready, 64, cudaHostAllocMapped));
    *reinterpret_cast<volatile unsigned*>(h_ready) = 0;
    PGN_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_zc), h_zc, 0));
    PGN_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_ready), h_ready, 0));
  }
  n = nn;
  cap = nc;
  nblk_cap = nb;
}

cudaEvent_t Workspace::event(size_t i) {
  while (ev.size() <= i) {
    cudaEvent_t e;
    PGN_CK(cudaEventCreate(&e));
    ev.push_back(e);
  }
  return ev[i];
}

Workspace::~Workspace() {
  for (auto e : ev) cudaEventDestroy(e);
  if (h_sc) cudaFreeHost(h_sc);
  if (h_mm) cudaFreeHost(h_mm);
  if (h_probe) cudaFreeHost(h_probe);
  if (h_probe_zc) cudaFreeHost(h_probe_zc);
  if (h_zc) cudaFreeHost(h_zc);
  if (h_ready) cudaFreeHost(h_ready);
  if (h_kb) cudaFreeHost(h_kb);
  if (h_kbzc) cudaFreeHost(h_kbzc);
  if (st) cudaStreamDestroy(st);
}

void Workspace::ensure_shard(int R, int n_, int64_t nb_global, int64_t nblk_max_cap,
                             int64_t stage) {
  stage = ((stage + kBlock - 1) / kBlock) * kBlock;
  if (nb_global <= nb_global_cap && stage <= stage_cap && n_ <= stage_n &&
      rec_send.n >= static_cast<size_t>(nblk_max_cap + 1) &&
      rec_recv.n >= static_cast<size_t>(R) * (nblk_max_cap + 1))
    return;
  PGN_CK(cudaSetDevice(device));
  nb_global_cap = nb_global > nb_global_cap ? nb_global : nb_global_cap;
  stage_cap = stage > stage_cap ? stage : stage_cap;
  const int64_t nb = nb_global_cap;
  g_part.alloc(4 * nb);
  g_err0.alloc(1);
  g_cnt.alloc(nb);
  g_off.alloc(nb);
  g_off_probe.alloc(nb);
  g_mm.alloc(2 * nb);
  g_part_multi.alloc(2 * kMaxProbes * nb);
  g_cnt_multi.alloc(kMaxProbes * nb);
  g_scratch_multi.alloc(2 * 2 * kMaxProbes * nb + 2);
  g_scratch.alloc(2 * nb + 2);
  g_kb.alloc(kMaxRanks + 1);
  g_val.alloc(kMaxRanks);
  rec_send.alloc(nblk_max_cap + 1);
  rec_recv.alloc(static_cast<size_t>(R) * (nblk_max_cap + 1));
  prec_send.alloc(nblk_max_cap + 1);
  prec_recv.alloc(static_cast<size_t>(R) * (nblk_max_cap + 1));
  const int nn = n_ > stage_n ? n_ : stage_n;
  stage_n = nn;
  st_low.alloc(static_cast<size_t>(nn) * stage_cap);
  st_len.alloc(static_cast<size_t>(nn) * stage_cap);
  st_pest.alloc(stage_cap);
  if (!h_kb) PGN_CK(cudaMallocHost(&h_kb, (kMaxRanks + 1) * sizeof(int64_t)));
  if (!h_kbzc) {
    PGN_CK(cudaHostAlloc(&h_kbzc, (kMaxRanks + 1) * sizeof(int64_t), cudaHostAllocMapped));
    PGN_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_kbzc), h_kbzc, 0));
  }
}

void ShardCtx::set_bounds(std::vector<int64_t> b) {
  bounds = std::move(b);
  rb.R = R;
  nblk_max = max_blocks(bounds);
  nblk_global = nblocks_of(bounds[R]);
  for (int r = 0; r < R; ++r) {
    rb.first[r] = bounds[r] / kBlock;
    rb.nblk[r] = nblocks_of(bounds[r + 1] - bounds[r]);
  }
}

namespace {
std::mutex g_ws_mu;
std::map<int, std::unique_ptr<Workspace>>& ws_map() {
  static std::map<int, std::unique_ptr<Workspace>> m;
  return m;
}
}  // namespace

Workspace& workspace_for(int device) {
  std::lock_guard<std::mutex> g(g_ws_mu);
  auto& m = ws_map();
  auto it = m.find(device);
  if (it != m.end()) return *it->second;
  int count = 0;
  PGN_CK(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) throw CudaError("no CUDA device " + std::to_string(device));
  auto ws = std::make_unique<Workspace>();
  ws->device = device;
  PGN_CK(cudaSetDevice(device));
  PGN_CK(cudaStreamCreateWithFlags(&ws->st, cudaStreamNonBlocking));
  Workspace& r = *ws;
  m[device] = std::move(ws);
  return r;
}

void release_workspaces() {
  std::lock_guard<std::mutex> g(g_ws_mu);
  ws_map().clear();
}

// ---------------------------------------------------------------------------
// Integrand resolution: the device has no CPU fallback.
DeviceIntegrand resolve_integrand(const pagani_integrand* f) {
  if (!f) throw std::invalid_argument("integrand is null");
  if (f->magic != PAGANI_INTEGRAND_MAGIC)
    throw std::invalid_argument("integrand: bad magic (use pagani_integrand_builtin)");
  if (f->kind == PAGANI_HOST_FN)
    throw UnsupportedError(
        "host function-pointer integrands cannot run on the GPU (no CPU fallback); "
        "use a builtin integrand");
  if (f->kind == PAGANI_DEVICE_FN) {
    const pagani_device_fn* d = f->device_fn;
    if (!d || d->magic != PAGANI_DEVICE_FN_MAGIC || !d->launch)
      throw std::invalid_argument("integrand: PAGANI_DEVICE_FN without a valid device_fn");
    if (d->params_size != sizeof(EvalParams))
      throw std::invalid_argument(
          "integrand: device_fn was compiled against a different pagani_device.cuh "
          "(parameter block size mismatch)");
    DeviceIntegrand di;
    di.ext = d;
    return di;
  }
  if (f->kind != PAGANI_BUILTIN) throw std::invalid_argument("integrand: unknown kind");
  const int id = f->builtin_id;
  const bool ok = (id >= 1 && id <= 8) || (id >= 100 && id <= 106);
  if (!ok) throw std::invalid_argument("unknown integrand id " + std::to_string(id));
  DeviceIntegrand d;
  d.fid = id;
  const int np = f->n_params < 0 ? 0 : (f->n_params > 32 ? 32 : f->n_params);
  for (int i = 0; i < np; ++i) d.params.p[i] = f->params[i];
  return d;
}

EvalLaunch evaluate_kernel(const DeviceIntegrand& di, int n, int mode) {
  if (di.ext) {
    EvalLaunch k;
    k.ext = di.ext;
    k.mode = mode;
    k.fused_fold = true;  // k_evaluate_fn folds its 2048-blocks (pagani_device.cuh)
    return k;
  }
  return lookup_evaluate(di.fid, n, mode);
}

// PAGANI_SPLIT_BULK=0 selects the per-region-load split kernel (A/B runs).
// PAGANI_PROBE_STREAM=1: the streamed threshold passes (exact counts, fast
// sums, exact fold of the accepted threshold only).  Bit-identical results,
// but measured slower than the exact 15-node passes on B200,
// so the exact passes are the default.
bool probe_stream() {
  static const bool on = [] {
    const char* e = std::getenv("PAGANI_PROBE_STREAM");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

// Deferred bisection on one GPU (k_link + children derived in k_evaluate,
// DESIGN.md 4); PAGANI_DEFER_BISECT=0 selects the explicit split kernel.
// Speculative first probe pass: after an iteration that ran a
// threshold search, the next iteration's first pass is queued behind
// k_finalize, its thresholds built on the device.  Opt-in
// (PAGANI_SPEC_PROBE=1): bit-identical, but measured neutral on B200 (bench
// step 2034 vs 2032 ms) -- the host round trip it hides is about what the
// wasted passes (7% of them) and the serial build in k_finalize cost.
bool spec_probe() {
  static const bool on = [] {
    const char* e = std::getenv("PAGANI_SPEC_PROBE");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

bool defer_bisect() {
  static const bool on = [] {
    const char* e = std::getenv("PAGANI_DEFER_BISECT");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

int split_bulk_mode() {
  static const int mode = [] {
    const char* e = std::getenv("PAGANI_SPLIT_BULK");
    return e ? std::atoi(e) : -1;
  }();
  return mode;
}

// ---------------------------------------------------------------------------
// Scalar helpers (driver.cpp:28-58)
int convergence_digits(double tau_rel) {
  const double d = std::ceil(std::log10(1.0 / tau_rel));
  if (!(d >= 1.0)) return 1;
  if (d > 17.0) return 17;
  return static_cast<int>(d);
}

bool digits_converged(double v_prev, double v_curr, int digits) {
  if (!std::isfinite(v_prev) || !std::isfinite(v_curr)) return false;
  if (v_prev == 0.0 && v_curr == 0.0) return true;
  if ((v_prev < 0.0) != (v_curr < 0.0)) return false;
  if (digits < 1) digits = 1;
  if (digits > 17) digits = 17;
  char a[40], b[40];
  std::snprintf(a, sizeof a, "%.*e", digits - 1, v_prev);
  std::snprintf(b, sizeof b, "%.*e", digits - 1, v_curr);
  return std::strcmp(a, b) == 0;
}

int initial_subdivisions(int n, int64_t init_target) {  // geometry.cpp:67-81
  int d = 1;
  for (;;) {
    int64_t p = 1;
    bool over = false;
    for (int a = 0; a < n; ++a) {
      if (p > init_target / (d + 1)) {
        over = true;
        break;
      }
      p *= d + 1;
    }
    if (over || p > init_target) break;
    ++d;
  }
  return d;
}

// ---------------------------------------------------------------------------
// Spin until the device publishes `seq` at *flag (k_finalize's zero-copy
// hand-off), checking the stream for errors now and then so a failed launch
// cannot hang the host.
void wait_host_flag(const unsigned* flag, unsigned seq, cudaStream_t st) {
  // `seq` or later: a kernel queued behind the awaited one (the speculative
  // first probe pass) may already have published the next number
  const volatile unsigned* f = flag;
  auto reached = [&] { return static_cast<int>(*f - seq) >= 0; };
  for (uint64_t i = 0;; ++i) {
    if (reached()) break;
    if ((i & 4095) == 4095) {
      const cudaError_t e = cudaStreamQuery(st);
      if (e == cudaSuccess) {
        if (reached()) break;
        throw CudaError("zero-copy hand-off: stream idle but the scalars were not published");
      }
      if (e != cudaErrorNotReady) cuda_check(e, "k_finalize (zero-copy hand-off)");
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
}

// ---------------------------------------------------------------------------
// Threshold search (classify.cpp:37-95) with device probes.
ThresholdOutcome device_threshold(Workspace& ws, int64_t m, const double* d_est,
                                  const double* d_err, const uint8_t* d_flag, double v_tot,
                                  double e_tot, double e_it, int64_t s_it, double tau_rel,
                                  const Limits& lim, double* probe_ms, const double* minmax,
                                  ShardCtx* sh, unsigned spec_seq) {
  ThresholdOutcome r;
  if (s_it <= 0) return r;
  const double e_budget = e_tot - std::fabs(v_tot) * tau_rel;
  double p_max = lim.p_max_start;
  r.budget_limit = p_max * e_budget;
  if (!(e_budget > 0.0)) return r;

  cudaStream_t st = ws.st;
  double min_err, max_err;
  if (minmax) {
    min_err = minmax[0];
    max_err = minmax[1];
  } else {
    launch_minmax(st, m, d_err, ws.mm_keys.p, ws.mm_out.p);
    r.minmax_launches = 3;
    PGN_CK(cudaMemcpyAsync(ws.h_mm, ws.mm_out.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    PGN_CK(cudaStreamSynchronize(st));
    min_err = ws.h_mm[0];
    max_err = ws.h_mm[1];
  }
  double t = e_it / static_cast<double>(s_it);

  // The search is a walk down a binary tree: from threshold t the next probe
  // is (t + max)/2 if too few regions finish, (t + min)/2 if too much error
  // would be discarded (classify.cpp:82-89).  p_max only changes acceptance,
  // never the t sequence, so a pass evaluates the whole depth-4 subtree (15
  // thresholds) and the host replays the reference's sequential decisions on
  // the results -- identical outcomes, up to 4 probes per round trip.
  enum Dir { kNone, kTowardMax, kTowardMin };
  const int64_t nblk = nblocks_of(m);
  // The walk's state; a pass replays it on a copy and commits the copy.
  struct Walk {
    Dir last = kNone;
    bool done = false;
    int attempts = 0, direction_changes = 0;
    double p_max = 0.0, t = 0.0;
    int accepted = -1;  // node accepted in this pass
  };
  Walk w;
  w.p_max = p_max;
  w.t = t;
  // Replay the reference's sequential decisions over one pass's 15 nodes.
  // fast: the sums are the fast ones -- a comparison within their rounding
  // bound of the budget is undecidable, and the replay reports it (returns
  // false) without committing anything.
  auto replay = [&](const ProbeSet& ps, const ProbeScalars& pr, bool fast, Walk& out) -> bool {
    Walk v = out;
    int node = 0;
    for (;;) {
      ++v.attempts;
      const int64_t inactive = s_it - pr.count[node];
      const bool memory_ok = 2 * inactive > s_it;
      const double discarded = pr.err_sum[node];
      const double budget = v.p_max * e_budget;
      if (fast && memory_ok && std::isfinite(discarded) && std::isfinite(budget) &&
          std::fabs(discarded - budget) <= 1e-12 * std::fabs(discarded) + 1e-300)
        return false;  // too close to call on a fast sum
      if (memory_ok && discarded <= budget) {
        v.accepted = node;
        out = v;
        return true;
      }
      const Dir dir = memory_ok ? kTowardMin : kTowardMax;
      if (v.last != kNone && dir != v.last) {
        ++v.direction_changes;
        if (v.direction_changes > lim.direction_change_limit) {
          v.t = ps.t[node];
          v.done = true;
          break;
        }
        const double stepped = v.p_max + lim.p_max_step;
        v.p_max = (stepped < lim.p_max_cap) ? stepped : lim.p_max_cap;  // std::min(cap, p+step)
      }
      v.last = dir;
      const int child = dir == kTowardMax ? 2 * node + 1 : 2 * node + 2;
      v.t = child < kMaxProbes ? ps.t[child]
                               : (dir == kTowardMax ? (ps.t[node] + max_err) * 0.5
                                                    : (ps.t[node] + min_err) * 0.5);
      if (v.attempts >= lim.attempt_limit) {
        v.done = true;
        break;
      }
      if (child >= kMaxProbes) break;  // next pass rooted at t
      node = child;
    }
    out = v;
    return true;
  };
  const bool fast_ok = !sh && probe_stream();
  while (!w.done && w.attempts < lim.attempt_limit) {
    ProbeSet ps{};
    ps.T = kMaxProbes;
    ps.t[0] = w.t;
    for (int k = 0; 2 * k + 2 < kMaxProbes; ++k) {
      ps.t[2 * k + 1] = (ps.t[k] + max_err) * 0.5;
      ps.t[2 * k + 2] = (ps.t[k] + min_err) * 0.5;
    }
    prepare_probes(ps);
    cudaEvent_t e0 = ws.event(0), e1 = ws.event(1);
    auto timed_wait = [&](unsigned seq) {
      if (probe_ms) PGN_CK(cudaEventRecord(e1, st));
      wait_host_flag(ws.h_ready, seq, st);
      ++r.passes;
      if (probe_ms) {
        float ms = 0;
        PGN_CK(cudaEventSynchronize(e1));  // recorded right behind the published kernel
        PGN_CK(cudaEventElapsedTime(&ms, e0, e1));
        *probe_ms += ms;
      }
    };
    bool decided = false;
    if (fast_ok) {  // streaming pass: exact counts, fast sums
      if (probe_ms) PGN_CK(cudaEventRecord(e0, st));
      const unsigned seq = ++ws.seq;
      launch_probe_fast(st, m, ps, d_err, d_flag, ws.part_multi.p, ws.cnt_multi.p,
                        ws.d_probe_zc, ws.d_ready, seq);
      r.bytes += 9.0 * m;  // flag + err
      timed_wait(seq);
      *ws.h_probe = *ws.h_probe_zc;
      decided = replay(ps, *ws.h_probe, true, w);
      if (!decided) ++r.exact_fallbacks;
      if (decided && w.accepted >= 0) {
        // the accepted threshold's sums exactly: the serial 2048-block folds
        // under its final flags + the pairwise trees + the kept offsets
        const int node = w.accepted;
        if (probe_ms) PGN_CK(cudaEventRecord(e0, st));
        const unsigned seq2 = ++ws.seq;
        launch_fold_threshold(st, m, d_est, d_err, d_flag, ps.t[node], ws.part_probe.p,
                              ws.cnt_probe.p);
        r.bytes += 17.0 * m;  // flag + err + est
        launch_finalize(st, nblk, 2, ws.part_probe.p, ws.cnt_probe.p, ws.off_probe.p,
                        ws.scratch.p, ws.d_zc, nullptr, nullptr, ws.d_ready, seq2);
        timed_wait(seq2);
        const FoldScalars fs = *ws.h_zc;
        if (s_it - fs.count != s_it - ws.h_probe->count[node])
          throw std::logic_error("threshold search: exact and streamed candidate counts differ");
        r.success = true;
        r.threshold = ps.t[node];
        r.discarded = fs.sum[1];  // sum err where final flag == 0
        r.fin_v = fs.sum[0];      // sum est where final flag == 0
        r.budget_limit = w.p_max * e_budget;
        r.finished_count = s_it - fs.count;
        r.node = node;
        r.attempts = w.attempts;
        r.direction_changes = w.direction_changes;
        return r;
      }
    }
    if (!decided && spec_seq != 0 && r.passes == 0) {
      // the first pass already ran on the device, queued right behind
      // k_finalize with the ProbeSet it built from the same scalars by the
      // same code (build_probe_tree; event 0 was recorded before it)
      r.spec_used = true;
      r.bytes += 17.0 * m;
      timed_wait(spec_seq);
      *ws.h_probe = *ws.h_probe_zc;
      decided = true;
      const ProbeScalars& pr = *ws.h_probe;
      replay(ps, pr, false, w);
      if (w.accepted >= 0) {
        const int node = w.accepted;
        r.success = true;
        r.threshold = ps.t[node];
        r.discarded = pr.err_sum[node];
        r.budget_limit = w.p_max * e_budget;
        r.finished_count = s_it - pr.count[node];
        r.fin_v = pr.est_sum[node];
        r.node = node;
        r.attempts = w.attempts;
        r.direction_changes = w.direction_changes;
        launch_scan_counts(st, nblk, ws.cnt_multi.p + node * nblk, ws.off_probe.p);
        return r;
      }
      continue;
    }
    if (!decided) {  // the exact pass: the strict folds of every node
      if (probe_ms) PGN_CK(cudaEventRecord(e0, st));
      // zero-copy hand-off of the pass results (as k_finalize's scalars): the
      // last tree CTA publishes a sequence number into mapped host memory
      const unsigned seq = ++ws.seq;
      r.bytes += 17.0 * m;  // flag + err + est
      if (!sh) {
        launch_probe_multi(st, m, ps, d_est, d_err, d_flag, ws.part_multi.p, ws.cnt_multi.p,
                           ws.scratch_multi.p, ws.d_probe_zc, ws.d_ready, seq, ws.probe_done.p);
      } else {  // local blocks -> allgather of block records -> global trees on every rank
        launch_probe_only(st, m, ps, d_est, d_err, d_flag, ws.part_multi.p, ws.cnt_multi.p);
        launch_pack_probe(st, nblocks_of(m), sh->nblk_max, kMaxProbes, ws.part_multi.p,
                          ws.cnt_multi.p, ws.prec_send.p);
        sh->comm->allgather(ws.prec_send.p, ws.prec_recv.p, sh->nblk_max * sizeof(ProbeRec), st);
        launch_unpack_probe(st, sh->rb, sh->nblk_max, sh->nblk_global, kMaxProbes,
                            ws.prec_recv.p, ws.g_part_multi.p, ws.g_cnt_multi.p);
        launch_finalize_multi(st, sh->nblk_global, kMaxProbes, ws.g_part_multi.p,
                              ws.g_cnt_multi.p, ws.g_scratch_multi.p, ws.d_probe_zc, ws.d_ready,
                              seq, ws.probe_done.p);
      }
      timed_wait(seq);
      *ws.h_probe = *ws.h_probe_zc;
      const ProbeScalars& pr = *ws.h_probe;
      replay(ps, pr, false, w);
      if (w.accepted >= 0) {
        const int node = w.accepted;
        r.success = true;
        r.threshold = ps.t[node];
        r.discarded = pr.err_sum[node];
        r.budget_limit = w.p_max * e_budget;
        r.finished_count = s_it - pr.count[node];
        r.fin_v = pr.est_sum[node];
        r.node = node;
        r.attempts = w.attempts;
        r.direction_changes = w.direction_changes;
        if (!sh) {
          launch_scan_counts(st, nblk, ws.cnt_multi.p + node * nblk, ws.off_probe.p);
        } else {
          const int64_t ng = sh->nblk_global;
          launch_scan_counts(st, ng, ws.g_cnt_multi.p + node * ng, ws.g_off_probe.p);
          launch_gather_bounds(st, sh->rb, ws.g_off_probe.p, ws.g_cnt_multi.p + node * ng, ng,
                               ws.g_kb.p);
        }
        return r;
      }
    }
  }
  t = w.t;
  p_max = w.p_max;
  r.attempts = w.attempts;
  r.direction_changes = w.direction_changes;
  r.threshold = t;
  r.budget_limit = p_max * e_budget;
  return r;
}

// ---------------------------------------------------------------------------
namespace {

struct Bounds {
  std::vector<double> lower, upper;
};

void validate_bounds(int n, const double* lower, const double* upper) {  // geometry.cpp:9-23
  if (!lower || !upper) throw std::invalid_argument("Bounds: lower/upper size mismatch");
  if (n < 1 || n > kMaxDim)
    throw std::invalid_argument("Bounds: dimension must be in [1, 16]");
  for (int a = 0; a < n; ++a) {
    if (!(lower[a] < upper[a]))
      throw std::invalid_argument("Bounds: lower must be < upper on every axis");
    if (!std::isfinite(lower[a]) || !std::isfinite(upper[a]))
      throw std::invalid_argument("Bounds: entries must be finite");
  }
}

void validate_config(const pagani_config& c) {  // driver.cpp:35-41
  if (!(c.tau_rel > 0.0)) throw std::invalid_argument("Config: tau_rel must be > 0");
  if (!(c.tau_abs >= 0.0)) throw std::invalid_argument("Config: tau_abs must be >= 0");
  if (c.it_max < 1) throw std::invalid_argument("Config: it_max must be >= 1");
  if (c.init_subdiv == 0 && c.max_regions < 2 * c.init_target)
    throw std::invalid_argument("Config: max_regions must be >= 2 * init_target");
}

// Event slots: 0/1 probe loop, 2/3 whole-call span, 4.. per-kernel marks.
constexpr size_t kSpanBegin = 2, kSpanEnd = 3, kFirstMark = 4;

struct KTimer {
  Workspace& ws;
  bool on;         // profile 1: every kernel class
  bool eval_only;  // profile 2: k_evaluate's span only
  std::vector<std::pair<int, std::pair<size_t, size_t>>> spans;
  size_t next = kFirstMark;
  KTimer(Workspace& w, int level) : ws(w), on(level == 1), eval_only(level == 2) {}
  size_t mark() {
    if (!on) return 0;
    const size_t i = next++;
    PGN_CK(cudaEventRecord(ws.event(i), ws.st));
    return i;
  }
  size_t mark_eval() {  // the marks around k_evaluate: recorded at either level
    if (!on && !eval_only) return 0;
    const size_t i = next++;
    PGN_CK(cudaEventRecord(ws.event(i), ws.st));
    return i;
  }
  void span(int slot, size_t a, size_t b) {
    if ((on || eval_only) && a != 0 && b != 0) spans.push_back({slot, {a, b}});
  }
  void collect(pagani_result* out) {
    if (!on && !eval_only) return;
    for (auto& s : spans) {
      float ms = 0;
      PGN_CK(cudaEventElapsedTime(&ms, ws.event(s.second.first), ws.event(s.second.second)));
      out->kernel_ms[s.first] += ms;
    }
    spans.clear();
    next = kFirstMark;
  }
};

}  // namespace

void integrate(const pagani_integrand* f, int ndim, const double* lower, const double* upper,
               const pagani_config* cfg_in, pagani_result* out) {
  const auto t_wall0 = std::chrono::steady_clock::now();
  if (!cfg_in || !out) throw std::invalid_argument("null config or result");
  const pagani_config cfg = *cfg_in;
  validate_config(cfg);
  validate_bounds(ndim, lower, upper);
  const int n = ndim;
  const DeviceIntegrand di = resolve_integrand(f);
  if (cfg.mode != PAGANI_MODE_PARITY && cfg.mode != PAGANI_MODE_FAST)
    throw std::invalid_argument("Config: unknown mode");
  EvalLaunch eval_k = evaluate_kernel(di, n, cfg.mode);
  if (!eval_k.valid()) throw UnsupportedError("no device kernel for this integrand/dimension");
  if (std::getenv("PAGANI_UNFUSED_FOLD")) eval_k.fused_fold = false;  // A/B experiments

  // ---- ranks ------------------------------------------------------------------
  Comm* comm = comm_from_handle(cfg.comm);
  const int R = comm ? comm->size() : 1;
  ShardCtx shard;
  ShardCtx* sh = nullptr;
  // A communicator always selects the sharded path (R = 1 included: this is
  // how the NCCL transport is exercised on a single-GPU host).
  if (comm) {
    if (R > kMaxRanks) throw std::invalid_argument("too many ranks");
    if (!eval_k.fused_fold)  // only under the PAGANI_UNFUSED_FOLD experiment switch
      throw UnsupportedError("multi-GPU runs need the evaluate kernel's fused block folds");
    shard.comm = comm;
    shard.R = R;
    shard.rank = comm->rank();
    sh = &shard;
  }
  const int rank = sh ? sh->rank : 0;

  std::memset(out, 0, sizeof(*out));
  Workspace& ws = workspace_for(comm ? comm->device() : cfg.device);
  std::lock_guard<std::mutex> lock(ws.mu);
  PGN_CK(cudaSetDevice(ws.device));
  cudaStream_t st = ws.st;

  // driver.cpp:92-99 -- work on the unit cube, scale at the end.
  bool mapped = false;
  double jacobian = 1.0;
  double dom_len[kMaxDim];
  for (int a = 0; a < n; ++a) {
    if (lower[a] != 0.0 || upper[a] != 1.0) mapped = true;
    jacobian *= upper[a] - lower[a];
    dom_len[a] = upper[a] - lower[a];
  }
  const double tau_abs = mapped ? cfg.tau_abs / jacobian : cfg.tau_abs;

  const RuleOrbits rule = build_rule_orbits(n);  // rule.cpp:166
  const int d = cfg.init_subdiv > 0 ? cfg.init_subdiv : initial_subdivisions(n, cfg.init_target);
  int64_t M = 1;  // global batch size (geometry.cpp:86-94)
  for (int a = 0; a < n; ++a) {
    if (M > cfg.max_regions / d) throw std::runtime_error("uniform_split: d^n exceeds max_regions");
    M *= d;
  }
  if (M > cfg.max_regions) throw std::runtime_error("uniform_split: d^n exceeds max_regions");

  // capacity: the whole cap on one GPU; a balanced block share (+ the staging
  // of this rank's children) when sharded
  const int64_t glob_cap = cfg.max_regions > M ? cfg.max_regions : M;
  int64_t cap_local = glob_cap;
  if (sh) {
    const int64_t nbg = nblocks_of(glob_cap);
    cap_local = ((nbg + R - 1) / R) * kBlock;
    sh->set_bounds(shard_bounds(M, R));
    ws.ensure(n, cap_local);
    // staging for the children that leave this rank: at most all of its
    // children, 2 * (local kept) <= 2 * cap_local (not the cached ws.cap, which
    // may be left over from a larger single-GPU run)
    ws.ensure_shard(R, n, nbg + 1, (nbg + R - 1) / R + 1, 2 * cap_local);
  } else {
    ws.ensure(n, cap_local);
  }
  const int64_t cap = ws.cap;
  int64_t m = sh ? sh->local() : M;  // local batch size
  const bool prof = cfg.profile == 1;
  KTimer kt(ws, cfg.profile);
  cudaEvent_t ev_begin = ws.event(kSpanBegin), ev_end = ws.event(kSpanEnd);
  PGN_CK(cudaEventRecord(ev_begin, st));

  {  // uniform split of the unit cube (this rank's slice of it)
    double lo[kMaxDim], step[kMaxDim];
    for (int a = 0; a < n; ++a) {
      lo[a] = 0.0;
      step[a] = (1.0 - 0.0) / d;
    }
    PGN_CK(cudaMemcpyAsync(ws.d_lower.p, lo, n * sizeof(double), cudaMemcpyHostToDevice, st));
    PGN_CK(cudaMemcpyAsync(ws.d_step.p, step, n * sizeof(double), cudaMemcpyHostToDevice, st));
    const size_t a0 = kt.mark();
    launch_uniform_split(st, n, d, m, cap, ws.low[0].p, ws.len[0].p, ws.d_lower.p, ws.d_step.p,
                         sh ? sh->first() : 0);
    kt.span(PAGANI_K_INIT, a0, kt.mark());
    out->kernel_launches[PAGANI_K_INIT]++;
    out->h2d_bytes += 2 * n * sizeof(double);
  }

  EvalParams ep{};
  ep.cap = cap;
  ep.pest = ws.pest.p;
  ep.est = ws.est.p;
  ep.err = ws.err.p;
  ep.axis = ws.axis.p;
  ep.flag = ws.flag.p;
  ep.rel_filter = cfg.rel_filtering_enabled ? 1 : 0;
  ep.tau = cfg.tau_rel;
  ep.n = n;
  ep.mapped = mapped ? 1 : 0;
  for (int k = 0; k < 5; ++k)
    for (int o = 0; o < 5; ++o) ep.w[k][o] = rule.w[k][o];
  for (int i = 0; i < 4; ++i) ep.gen[i] = rule.gen[i];
  for (int a = 0; a < n; ++a) {
    ep.map_lo[a] = lower[a];
    ep.map_len[a] = dom_len[a];
  }
  ep.ip = di.params;

  Limits lim;
  lim.direction_change_limit = cfg.direction_change_limit;
  lim.attempt_limit = cfg.attempt_limit;
  lim.p_max_start = cfg.p_max_start;
  lim.p_max_step = cfg.p_max_step;
  lim.p_max_cap = cfg.p_max_cap;

  double acc_v = 0.0, acc_e = 0.0, acc_vf = 0.0, acc_ef = 0.0;  // Accumulators
  double prev_total = std::numeric_limits<double>::quiet_NaN();
  const int digits = convergence_digits(cfg.tau_rel);
  out->regions_generated = M;
  out->peak_regions = m;
  int cur = 0;  // which low/len buffer holds the batch
  double finished_volume = 0.0;
  std::vector<int64_t> kb(R + 1, 0);  // global kept offsets at rank boundaries

  // validate_invariants on a sharded run: the per-rank values of a check are
  // allgathered and added in rank order (the checks are tolerances, not
  // bit-exact quantities; one GPU uses the reference's exact sums).
  auto global_sum = [&](double* dval) -> double {
    double hv[kMaxRanks] = {};
    if (!sh) {
      PGN_CK(cudaMemcpyAsync(hv, dval, sizeof(double), cudaMemcpyDeviceToHost, st));
      PGN_CK(cudaStreamSynchronize(st));
      return hv[0];
    }
    comm->allgather(dval, ws.g_val.p, sizeof(double), st);
    PGN_CK(cudaMemcpyAsync(hv, ws.g_val.p, R * sizeof(double), cudaMemcpyDeviceToHost, st));
    PGN_CK(cudaStreamSynchronize(st));
    double tot = 0.0;
    for (int r = 0; r < R; ++r) tot += hv[r];
    return tot;
  };

  auto finish = [&](int status, int it) {
    out->status = status;
    out->iterations = it;
    out->estimate = (acc_v + acc_vf) * jacobian;
    out->errorest = (acc_e + acc_ef) * jacobian;
  };

  bool done = false;
  bool linked = false;  // this batch's geometry still lives in its parents' rows (k_link)
  bool searched_last = false;  // the previous iteration ran a threshold search
  for (int it = 1; it <= cfg.it_max && !done; ++it) {
    // ---- evaluate (+ refine + classify + block folds) -------------------------
    ep.m = m;
    ep.low = ws.low[cur].p;
    ep.len = ws.len[cur].p;
    // deferred bisection: the children are derived from the parent rows in
    // the other buffer and written to this one by k_evaluate
    ep.link = linked ? ws.link.p : nullptr;
    ep.plow = linked ? ws.low[cur ^ 1].p : nullptr;
    ep.plen = linked ? ws.len[cur ^ 1].p : nullptr;
    ep.refine = (it > 1 && cfg.refiner == PAGANI_REFINER_TWO_LEVEL) ? 1 : 0;
    const size_t k0 = kt.mark_eval();
    const int64_t nblk = nblocks_of(m);
    ep.nblk = nblk;
    if (eval_k.fused_fold) {  // block folds + min/max run in k_evaluate's tail
      ep.part = ws.part_eval.p;
      ep.cnt = ws.cnt_eval.p;
      ep.mm = ws.mm_blk.p;
      ep.blk_done = ws.blk_done.p;
    }
    if (m > 0) {
      launch_evaluate(eval_k, st, ep);
      PGN_CK(cudaGetLastError());
    }
    const size_t k1 = kt.mark_eval();
    kt.span(PAGANI_K_EVALUATE, k0, k1);
    out->kernel_launches[PAGANI_K_EVALUATE] += m > 0;
    // reads low/len (16n) [+ pest 8], writes est, err (16) + flag, axis (2)
    // (+ deferred bisection: the link (8 per sibling pair) and the child's
    // row written back, 16n; the parent rows are counted as the read)
    out->kernel_bytes[PAGANI_K_EVALUATE] +=
        static_cast<double>(m) * (16.0 * n + (ep.refine ? 8 : 0) + 18) +
        (linked ? static_cast<double>(m) * (16.0 * n + 4.0) : 0.0);
    out->eval_count += M * rule.point_count;
    out->region_evals += m;

    // ---- global scalars: v, e, finished sums, active counts, min/max ----------
    if (!eval_k.fused_fold) {
      launch_fold_eval(st, m, ws.est.p, ws.err.p, ws.flag.p, ws.part_eval.p, ws.cnt_eval.p);
      out->kernel_launches[PAGANI_K_FOLD]++;
    }
    const size_t k2 = kt.mark();
    const int64_t* offsets = ws.off_eval.p;  // kept offsets, indexed by (global) block
    // the next search's first pass, queued behind k_finalize before the host
    // has decided whether a search runs (it usually does once one has)
    const bool spec = !sh && eval_k.fused_fold && searched_last && it < cfg.it_max && m > 0 &&
                      spec_probe() && !probe_stream();
    unsigned spec_seq = 0;
    size_t sx0 = 0, sx1 = 0, k3 = 0;
    if (!sh) {
      SpecProbe sp;
      if (spec) sp = SpecProbe{ws.spec_ps.p, M};
      launch_finalize(st, nblk, 4, ws.part_eval.p, ws.cnt_eval.p, ws.off_eval.p, ws.scratch.p,
                      ws.d_zc, eval_k.fused_fold ? ws.mm_blk.p : nullptr, ws.err.p, ws.d_ready,
                      ++ws.seq, sp);
      out->kernel_launches[PAGANI_K_FINALIZE]++;
      k3 = kt.mark();
      if (spec) {
        sx0 = k3;
        if (prof) PGN_CK(cudaEventRecord(ws.event(0), st));  // device_threshold's pass timer
        spec_seq = ++ws.seq;
        out->spec_probe_passes++;
        launch_probe_multi_dev(st, m, ws.spec_ps.p, ws.est.p, ws.err.p, ws.flag.p,
                               ws.part_multi.p, ws.cnt_multi.p, ws.scratch_multi.p,
                               ws.d_probe_zc, ws.d_ready, spec_seq, ws.probe_done.p);
        sx1 = kt.mark();
      }
    } else {  // allgather the block records; every rank runs the same global trees
      launch_pack_blocks(st, nblk, sh->nblk_max, ws.part_eval.p, ws.cnt_eval.p, ws.mm_blk.p,
                         ws.err.p, ws.rec_send.p);
      comm->allgather(ws.rec_send.p, ws.rec_recv.p, (sh->nblk_max + 1) * sizeof(BlockRec), st);
      launch_unpack_blocks(st, sh->rb, sh->nblk_max, sh->nblk_global, ws.rec_recv.p, ws.g_part.p,
                           ws.g_cnt.p, ws.g_mm.p, ws.g_err0.p);
      // zero-copy hand-off as on one GPU: the scalars and the kept bounds at
      // the rank boundaries go to mapped host memory; k_gather_bounds
      // publishes the sequence number after both (seq 0 = fence, no publish)
      launch_finalize(st, sh->nblk_global, 4, ws.g_part.p, ws.g_cnt.p, ws.g_off.p, ws.g_scratch.p,
                      ws.d_zc, ws.g_mm.p, ws.g_err0.p, ws.d_ready, 0);
      launch_gather_bounds(st, sh->rb, ws.g_off.p, ws.g_cnt.p, sh->nblk_global, ws.d_kbzc,
                           ws.d_ready, ++ws.seq);
      out->kernel_launches[PAGANI_K_FINALIZE] += 4;
      offsets = ws.g_off.p;
    }
    if (sh) k3 = kt.mark();
    kt.span(PAGANI_K_FOLD, k1, k2);
    kt.span(PAGANI_K_FINALIZE, k2, k3);
    wait_host_flag(ws.h_ready, spec ? spec_seq - 1 : ws.seq, st);
    ws.h_sc[0] = *ws.h_zc;
    out->d2h_bytes += sizeof(FoldScalars);
    if (sh) {
      const volatile int64_t* hk = ws.h_kbzc;
      for (int r = 0; r <= R; ++r) kb[r] = hk[r];
      out->d2h_bytes += (R + 1) * sizeof(int64_t);
    }
    const FoldScalars sc = ws.h_sc[0];
    acc_v = sc.sum[0];  // block_sum(estimates)
    acc_e = sc.sum[1];  // block_sum(errors)

    pagani_trace_row row{};
    row.it = it;
    row.m = M;
    row.active_rel = sc.count;

    if (cfg.validate_invariants) {  // driver.cpp:75-79,148
      launch_serial_volume(st, n, m, cap, ws.len[cur].p, nullptr, 0, ws.d_tmp.p);
      const double tv = global_sum(ws.d_tmp.p);
      if (std::fabs(tv + finished_volume - 1.0) > 1e-10)
        throw std::logic_error("invariant violated: volume not conserved");
    }

    // check_termination (driver.cpp:43-46,150-152)
    {
      const double err_tot = acc_e + acc_ef;
      if (err_tot <= std::fabs(acc_v + acc_vf) * cfg.tau_rel || err_tot <= tau_abs) {
        row.v = acc_v, row.e = acc_e, row.v_f = acc_vf, row.e_f = acc_ef;
        row.active_final = row.active_rel;
        if (cfg.trace) cfg.trace(&row, cfg.trace_user);
        finish(PAGANI_CONVERGED, it);
        done = true;
        break;
      }
    }
    if (it == cfg.it_max) {
      row.v = acc_v, row.e = acc_e, row.v_f = acc_vf, row.e_f = acc_ef;
      row.active_final = row.active_rel;
      if (cfg.trace) cfg.trace(&row, cfg.trace_user);
      break;
    }

    // ---- triggers + threshold search (driver.cpp:154-172) --------------------
    const int64_t active_count = sc.count;
    const bool trig_memory = 2 * active_count > cfg.max_regions;
    const bool trig_digits = digits_converged(prev_total, acc_v + acc_vf, digits);
    row.trig_digits = trig_digits;
    row.trig_memory = trig_memory;
    bool use_t = false;
    double t_accepted = 0.0;
    double fin_v = sc.sum[2], fin_e = sc.sum[3];
    int64_t kept = sc.count;
    bool spec_used = false;
    searched_last = trig_digits || trig_memory;
    if (trig_digits || trig_memory) {
      double pms = 0.0;
      const double known_mm[2] = {sc.mn, sc.mx};
      const ThresholdOutcome tr = device_threshold(
          ws, m, ws.est.p, ws.err.p, ws.flag.p, acc_v + acc_vf, acc_e + acc_ef, acc_e, M,
          cfg.tau_rel, lim, prof ? &pms : nullptr, eval_k.fused_fold ? known_mm : nullptr, sh,
          spec_seq);
      spec_used = tr.spec_used;
      out->kernel_ms[PAGANI_K_PROBE] += pms;
      out->kernel_bytes[PAGANI_K_PROBE] += tr.bytes;
      out->kernel_launches[PAGANI_K_PROBE] += (sh ? 5 : 2) * tr.passes + (tr.success ? 1 : 0);
      out->kernel_launches[PAGANI_K_MINMAX] += tr.minmax_launches;
      out->d2h_bytes += tr.passes * sizeof(ProbeScalars);
      out->probe_fallbacks += tr.exact_fallbacks;
      if (out->n_events < PAGANI_MAX_EVENTS) {
        pagani_threshold_event& ev = out->events[out->n_events];
        ev.iteration = it;
        ev.success = tr.success;
        ev.batch_size = M;
        ev.finished_count = tr.finished_count;
        ev.discarded_error = tr.discarded;
        ev.budget_limit = tr.budget_limit;
      }
      out->n_events++;
      const bool affordable = acc_ef + tr.discarded <= 0.25 * cfg.tau_rel * std::fabs(acc_v + acc_vf);
      row.thr_invoked = 1;
      row.thr_success = tr.success;
      row.thr_attempts = tr.attempts;
      row.thr_dir_changes = tr.direction_changes;
      row.thr_threshold = tr.threshold;
      row.thr_discarded = tr.discarded;
      row.thr_budget = tr.budget_limit;
      row.thr_finished = tr.finished_count;
      if (tr.success && (trig_memory || affordable)) {
        row.thr_accepted = 1;
        use_t = true;
        t_accepted = tr.threshold;
        fin_e = tr.discarded;  // sum err[final flag == 0]
        fin_v = tr.fin_v;
        kept = M - tr.finished_count;
        offsets = sh ? ws.g_off_probe.p : ws.off_probe.p;
        if (sh) {  // kept offsets of the accepted candidates at rank boundaries
          PGN_CK(cudaMemcpyAsync(ws.h_kb, ws.g_kb.p, (R + 1) * sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, st));
          PGN_CK(cudaStreamSynchronize(st));
          for (int r = 0; r <= R; ++r) kb[r] = ws.h_kb[r];
        }
      }
    }
    if (spec && !spec_used) {  // the speculative pass ran for nothing: account for it
      kt.span(PAGANI_K_PROBE, sx0, sx1);
      out->kernel_launches[PAGANI_K_PROBE] += 2;
      out->kernel_bytes[PAGANI_K_PROBE] += 17.0 * static_cast<double>(m);
      out->spec_probe_wasted++;
    }
    row.v = acc_v, row.e = acc_e, row.v_f = acc_vf, row.e_f = acc_ef;
    row.active_final = kept;
    row.fin_v = fin_v;
    row.fin_e = fin_e;
    row.kept = kept;
    if (cfg.trace) cfg.trace(&row, cfg.trace_user);

    if (cfg.validate_invariants) {  // driver.cpp:185-198
      const uint8_t* fflag = ws.flag.p;
      if (use_t) {
        launch_candidates(st, m, t_accepted, ws.flag.p, ws.err.p, ws.flag2.p);
        fflag = ws.flag2.p;
      }
      launch_serial_volume(st, n, m, cap, ws.len[cur].p, fflag, 0, ws.d_tmp.p);
      finished_volume += global_sum(ws.d_tmp.p);
      // driver.cpp:185-190: the filter conserves the estimate.  kept_v =
      // block_sum of the kept estimates in compacted order.
      const int64_t kept_local = sh ? kb[rank + 1] - kb[rank] : kept;
      const int64_t nbk = nblocks_of(kept_local);
      if (nbk > 0) {
        launch_kept_partials(st, m, ws.flag.p, use_t ? 1 : 0, t_accepted, ws.err.p, ws.est.p,
                             ws.part_probe.p);
        launch_finalize(st, nbk, 1, ws.part_probe.p, nullptr, nullptr, ws.scratch.p, ws.d_sc.p);
      } else {
        PGN_CK(cudaMemsetAsync(ws.d_sc.p, 0, sizeof(FoldScalars), st));
      }
      const double kept_v = global_sum(ws.d_sc.p->sum);
      const double scale = std::max({1e-30, std::fabs(acc_v), std::fabs(fin_v)});
      if (std::fabs(kept_v + fin_v - acc_v) > 1e-10 * scale)
        throw std::logic_error("invariant violated: estimate not conserved by filter");
      if (fin_e < 0.0) throw std::logic_error("invariant violated: negative finished error");
    }

    // ---- filter accounting (driver.cpp:194-202) -------------------------------
    const double prev_e_f = acc_ef;
    acc_vf += fin_v;
    acc_ef += fin_e;
    if (cfg.validate_invariants && acc_ef < prev_e_f)
      throw std::logic_error("invariant violated: finished error decreased");
    acc_v -= fin_v;
    acc_e -= fin_e;
    prev_total = acc_v + acc_vf;

    if (kept == 0) {
      finish(PAGANI_MAX_ITERATIONS, it);
      done = true;
      break;
    }
    if (2 * kept > cfg.max_regions) {
      finish(PAGANI_MEMORY_EXHAUSTED, it);
      done = true;
      break;
    }

    // ---- fused filter + bisect (+ the exchange that re-balances the shards) ---
    const size_t k4 = kt.mark();
    const bool defer = !sh && defer_bisect() && eval_k.fn_link != nullptr;
    if (defer) {
      // flag, axis, est (+ err under a threshold) per region; link + pest per kept
      out->kernel_bytes[PAGANI_K_SPLIT] +=
          static_cast<double>(m) * (use_t ? 18.0 : 10.0) + static_cast<double>(kept) * 16.0;
    } else {  // flag (+ err under a threshold) for every region; est, axis, low, len of
              // each kept one; two children (low, len, parent est) per kept region.
      const double kl = sh ? static_cast<double>(kb[rank + 1] - kb[rank]) : static_cast<double>(kept);
      out->kernel_bytes[PAGANI_K_SPLIT] += static_cast<double>(m) * (use_t ? 9.0 : 1.0) +
                                           kl * (16.0 * n + 9.0) + 2.0 * kl * (16.0 * n + 8.0);
    }
    // k_split_bulk (TMA-staged rows; measured 3-4% faster than k_split_n per
    // bench step); PAGANI_SPLIT_BULK=0 selects k_split_n
    const bool bulk = split_bulk_mode() != 0;
    if (defer) {
      launch_link(st, m, ws.flag.p, use_t ? 1 : 0, t_accepted, offsets, ws.est.p, ws.err.p,
                  ws.axis.p, ws.link.p, ws.pest.p);
      PGN_CK(cudaGetLastError());
      out->kernel_launches[PAGANI_K_SPLIT]++;
      m = 2 * kept;
    } else if (!sh) {
      launch_split(st, n, m, cap, cap, ws.flag.p, use_t ? 1 : 0, t_accepted, offsets, ws.est.p,
                   ws.err.p, ws.axis.p, ws.low[cur].p, ws.len[cur].p, ws.low[cur ^ 1].p,
                   ws.len[cur ^ 1].p, ws.pest.p, nullptr, 0, SplitWindow{}, bulk, kept);
      PGN_CK(cudaGetLastError());
      out->kernel_launches[PAGANI_K_SPLIT]++;
      m = 2 * kept;
    } else {
      const int64_t sc_cap = ws.stage_cap;
      const std::vector<int64_t> next = shard_bounds(2 * kept, R);
      std::vector<Piece> sends, recvs;
      exchange_plan(R, rank, kb, next, sends, recvs);
      double* dlow = ws.low[cur ^ 1].p;
      double* dlen = ws.len[cur ^ 1].p;
      // the piece that stays on this rank is written straight into the next
      // batch; only the pieces that change owner go through the staging area
      SplitWindow win;
      for (const Piece& p : recvs)
        if (p.peer == rank) {
          win.low = dlow, win.len = dlen, win.pest = ws.pest.p, win.cap = cap;
          win.lo = p.src_off, win.hi = p.src_off + p.count, win.dst = p.dst_off;
        }
      launch_split(st, n, m, cap, sc_cap, ws.flag.p, use_t ? 1 : 0, t_accepted,
                   offsets + sh->rb.first[rank], ws.est.p, ws.err.p, ws.axis.p, ws.low[cur].p,
                   ws.len[cur].p, ws.st_low.p, ws.st_len.p, ws.st_pest.p, nullptr, kb[rank], win,
                   bulk, kb[rank + 1]);
      PGN_CK(cudaGetLastError());
      out->kernel_launches[PAGANI_K_SPLIT] += m > 0;
      std::vector<Transfer> ts, tr;
      double sent = 0.0;
      for (const Piece& p : sends) {
        if (p.peer == rank) continue;
        for (int a = 0; a < n; ++a) {
          ts.push_back({p.peer, ws.st_low.p + a * sc_cap + p.src_off, p.count * sizeof(double)});
          ts.push_back({p.peer, ws.st_len.p + a * sc_cap + p.src_off, p.count * sizeof(double)});
        }
        ts.push_back({p.peer, ws.st_pest.p + p.src_off, p.count * sizeof(double)});
        sent += static_cast<double>(p.count) * (16.0 * n + 8.0);
      }
      for (const Piece& p : recvs) {
        if (p.peer == rank) continue;
        for (int a = 0; a < n; ++a) {
          tr.push_back({p.peer, dlow + a * cap + p.dst_off, p.count * sizeof(double)});
          tr.push_back({p.peer, dlen + a * cap + p.dst_off, p.count * sizeof(double)});
        }
        tr.push_back({p.peer, ws.pest.p + p.dst_off, p.count * sizeof(double)});
      }
      out->kernel_bytes[PAGANI_K_EXCHANGE] += sent;
      out->kernel_launches[PAGANI_K_EXCHANGE] += !ts.empty() || !tr.empty();
      const size_t x0 = kt.mark();
      comm->exchange(ts, tr, st);
      kt.span(PAGANI_K_SPLIT, k4, x0);
      kt.span(PAGANI_K_EXCHANGE, x0, kt.mark());
      sh->set_bounds(next);
      m = sh->local();
    }
    if (!sh) kt.span(PAGANI_K_SPLIT, k4, kt.mark());
    linked = defer;
    cur ^= 1;
    M = 2 * kept;
    out->regions_generated += M;
    if (m > out->peak_regions) out->peak_regions = m;
  }
  if (!done) finish(PAGANI_MAX_ITERATIONS, cfg.it_max);
  PGN_CK(cudaEventRecord(ev_end, st));
  PGN_CK(cudaStreamSynchronize(st));
  {
    float span = 0;
    PGN_CK(cudaEventElapsedTime(&span, ev_begin, ev_end));
    out->device_ms = span;
  }
  kt.collect(out);
  out->wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_wall0).count();
}

}  // namespace pgn
