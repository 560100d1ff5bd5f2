// The sequential (globally adaptive, Alg. 1) engine -- the reference's
// comparison oracle integrate_sequential (/root/reference/proj/src/sequential.cpp:45-139),
// with the rule evaluation on the GPU.
//
// The algorithm is inherently one region at a time: pop the region with the
// largest error, bisect it along its split axis, evaluate the two children,
// push them back.  The heap stays on the host -- std::priority_queue with the
// reference's comparator, so ties pop in the same order -- and each step is
// one k_evaluate launch over the two children, fused with their two-level
// refinement (the siblings are lanes j, j^1 of one warp, errorest.cpp:10-37).
// The children's geometry and the kernel's outputs live in mapped pinned host
// memory, so a step is a launch plus a stream synchronisation and no copies.
// Results are bit-identical to the reference (tests/test_gpu_parity.py).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <queue>
#include <vector>

#include "driver.hpp"

namespace pgn {

namespace {

struct HeapRegion {  // sequential.cpp:16-22
  double estimate;
  double error;
  int split_axis;
  std::vector<double> low;
  std::vector<double> len;
};

struct ByError {  // sequential.cpp:24-28
  bool operator()(const HeapRegion& a, const HeapRegion& b) const { return a.error < b.error; }
};

// Mapped pinned buffers of one step (two regions, axis-major [a * 2 + j]).
struct StepBufs {
  double* h = nullptr;  // [low 2*16 | len 2*16 | pest 2 | est 2 | err 2]
  double* d = nullptr;
  uint8_t* hb = nullptr;  // [axis 2 | flag 2]
  uint8_t* db = nullptr;
  StepBufs() {
    PGN_CK(cudaHostAlloc(&h, 70 * sizeof(double), cudaHostAllocMapped));
    PGN_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d), h, 0));
    PGN_CK(cudaHostAlloc(&hb, 4, cudaHostAllocMapped));
    PGN_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&db), hb, 0));
  }
  ~StepBufs() {
    if (h) cudaFreeHost(h);
    if (hb) cudaFreeHost(hb);
  }
  double* low() { return h; }
  double* len() { return h + 32; }
  double* pest() { return h + 64; }
  double* est() { return h + 66; }
  double* err() { return h + 68; }
  int axis_at(int j) const { return hb[j]; }
};

}  // namespace

void integrate_sequential(const pagani_integrand* f, int ndim, const double* lower,
                          const double* upper, double tau_rel, double tau_abs, int64_t max_evals,
                          int validate_invariants, int device, int mode, pagani_result* out) {
  const auto t_wall0 = std::chrono::steady_clock::now();
  if (!out) throw std::invalid_argument("null result");
  if (!(tau_rel > 0.0)) throw std::invalid_argument("tau_rel must be > 0");
  if (!lower || !upper) throw std::invalid_argument("Bounds: lower/upper size mismatch");
  const int n = ndim;
  if (n < 1 || n > kMaxDim) throw std::invalid_argument("Bounds: dimension must be in [1, 16]");
  for (int a = 0; a < n; ++a) {  // geometry.cpp:9-23
    if (!(lower[a] < upper[a]))
      throw std::invalid_argument("Bounds: lower must be < upper on every axis");
    if (!std::isfinite(lower[a]) || !std::isfinite(upper[a]))
      throw std::invalid_argument("Bounds: entries must be finite");
  }
  const DeviceIntegrand di = resolve_integrand(f);
  const EvalLaunch eval_k = evaluate_kernel(di, n, mode);
  if (!eval_k.valid()) throw UnsupportedError("no device kernel for this integrand/dimension");

  std::memset(out, 0, sizeof(*out));
  Workspace& ws = workspace_for(device);
  std::lock_guard<std::mutex> lock(ws.mu);
  PGN_CK(cudaSetDevice(ws.device));
  cudaStream_t st = ws.st;
  StepBufs sb;

  bool mapped = false;  // sequential.cpp:53-60
  double jacobian = 1.0;
  for (int a = 0; a < n; ++a) {
    if (lower[a] != 0.0 || upper[a] != 1.0) mapped = true;
    jacobian *= upper[a] - lower[a];
  }
  const double tau_abs_int = mapped ? tau_abs / jacobian : tau_abs;
  const RuleOrbits rule = build_rule_orbits(n);

  EvalParams ep{};
  ep.cap = 2;
  ep.low = sb.d;
  ep.len = sb.d + 32;
  ep.pest = sb.d + 64;
  ep.est = sb.d + 66;
  ep.err = sb.d + 68;
  ep.axis = sb.db;
  ep.flag = sb.db + 2;
  ep.n = n;
  ep.tau = tau_rel;
  ep.mapped = mapped ? 1 : 0;
  for (int k = 0; k < 5; ++k)
    for (int o = 0; o < 5; ++o) ep.w[k][o] = rule.w[k][o];
  for (int i = 0; i < 4; ++i) ep.gen[i] = rule.gen[i];
  for (int a = 0; a < n; ++a) {
    ep.map_lo[a] = lower[a];
    ep.map_len[a] = upper[a] - lower[a];
  }
  ep.ip = di.params;

  auto evaluate = [&](int64_t m, bool refine) {
    ep.m = m;
    ep.refine = refine ? 1 : 0;
    launch_evaluate(eval_k, st, ep);
    PGN_CK(cudaGetLastError());
    PGN_CK(cudaStreamSynchronize(st));
    out->kernel_launches[PAGANI_K_EVALUATE]++;
    out->region_evals += m;
    out->eval_count += m * rule.point_count;
  };

  std::priority_queue<HeapRegion, std::vector<HeapRegion>, ByError> heap;
  // the whole (normalised) domain, raw error as-is (sequential.cpp:66-75)
  for (int a = 0; a < n; ++a) {
    sb.low()[a * 2] = 0.0 + 0.0 * ((1.0 - 0.0) / 1);  // uniform_split(unit cube, 1)
    sb.len()[a * 2] = (1.0 - 0.0) / 1;
  }
  evaluate(1, false);
  out->regions_generated = 1;
  double v = sb.est()[0];
  double e = sb.err()[0];
  heap.push({sb.est()[0], sb.err()[0], sb.axis_at(0), std::vector<double>(n, 0.0),
             std::vector<double>(n, 1.0)});
  out->peak_regions = 1;

  auto finish = [&](int status) {
    out->status = status;
    out->estimate = v * jacobian;
    out->errorest = e * jacobian;
  };

  for (;;) {
    if (e <= std::fabs(v) * tau_rel || e <= tau_abs_int) {
      finish(PAGANI_CONVERGED);
      break;
    }
    if (out->eval_count > max_evals) {
      finish(PAGANI_MAX_ITERATIONS);
      break;
    }
    HeapRegion top = heap.top();
    heap.pop();
    for (int child = 0; child < 2; ++child)  // sequential.cpp:85-95
      for (int a = 0; a < n; ++a) {
        double lo = top.low[a], ln = top.len[a];
        if (a == top.split_axis) {
          ln = top.len[a] * 0.5;
          if (child == 1) lo += ln;
        }
        sb.low()[a * 2 + child] = lo;
        sb.len()[a * 2 + child] = ln;
      }
    sb.pest()[0] = sb.pest()[1] = top.estimate;
    evaluate(2, true);  // + two_level_refine of the pair (errorest.cpp:10-37)
    out->regions_generated += 2;
    ++out->iterations;
    const double est0 = sb.est()[0], est1 = sb.est()[1];
    const double ref0 = sb.err()[0], ref1 = sb.err()[1];
    v += est0 + est1 - top.estimate;  // sequential.cpp:104-105
    e += ref0 + ref1 - top.error;
    for (int child = 0; child < 2; ++child) {
      std::vector<double> low(n), len(n);
      for (int a = 0; a < n; ++a) {
        low[a] = sb.low()[a * 2 + child];
        len[a] = sb.len()[a * 2 + child];
      }
      heap.push({child ? est1 : est0, child ? ref1 : ref0, sb.axis_at(child), std::move(low),
                 std::move(len)});
    }
    if (static_cast<int64_t>(heap.size()) > out->peak_regions) out->peak_regions = heap.size();

    if (validate_invariants && (out->iterations & 63) == 0) {  // sequential.cpp:114-130
      auto copy = heap;
      double hv = 0.0, he = 0.0;
      while (!copy.empty()) {
        hv += copy.top().estimate;
        he += copy.top().error;
        copy.pop();
      }
      const double scale = std::max({1e-30, std::fabs(v), std::fabs(hv)});
      if (std::fabs(hv - v) > 1e-10 * scale)
        throw std::logic_error("invariant violated: heap estimate drift");
      if (std::fabs(he - e) > 1e-8 * std::max(1e-30, e))
        throw std::logic_error("invariant violated: heap error drift");
    }
  }
  out->wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_wall0).count();
}

}  // namespace pgn
