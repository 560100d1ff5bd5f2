// Host-side PAGANI driver (C++): the reference's integrate() loop
// (/root/reference/proj/src/driver.cpp:83-215) over device-resident batches.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pagani.h"
#include "comm.hpp"
#include "kernels.cuh"
#include "rule.hpp"
#include "shard.hpp"

namespace pgn {

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& s) : std::runtime_error(s) {}
};
struct UnsupportedError : std::runtime_error {
  explicit UnsupportedError(const std::string& s) : std::runtime_error(s) {}
};

void cuda_check(cudaError_t e, const char* what);
#define PGN_CK(x) ::pgn::cuda_check((x), #x)

// Device buffer with RAII (batch API temporaries).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    free();
    n = count;
    if (count) PGN_CK(cudaMalloc(&p, count * sizeof(T)));
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { free(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// Per-device cached workspace: the region store (double-buffered, axis-major)
// and the scratch of the folds.  Sized once for `cap` regions of dimension
// n and reused by every later call with cap' <= cap.
struct Workspace {
  int device = -1;
  cudaStream_t st = nullptr;
  std::mutex mu;
  int n = 0;
  int64_t cap = 0;
  int64_t nblk_cap = 0;
  DevBuf<double> low[2], len[2];
  DevBuf<double> pest, est, err;
  DevBuf<uint64_t> link;               // deferred bisection: kept parent rows (k_link)
  DevBuf<uint8_t> axis, flag, flag2;
  DevBuf<double> part_eval, part_probe, scratch;
  DevBuf<int64_t> cnt_eval, cnt_probe, off_eval, off_probe;
  DevBuf<int> blk_done;                 // fused-fold arrival counters (self-resetting)
  DevBuf<unsigned long long> mm_blk;    // per-block min/max error keys
  DevBuf<double> part_multi, scratch_multi;
  DevBuf<int64_t> cnt_multi;
  DevBuf<ProbeScalars> d_probe;
  ProbeScalars* h_probe = nullptr;      // pinned
  ProbeScalars* h_probe_zc = nullptr;   // mapped: zero-copy pass results
  ProbeScalars* d_probe_zc = nullptr;   // device alias of h_probe_zc
  DevBuf<ProbeSet> spec_ps;  // the speculative first pass's thresholds (k_finalize builds them)
  DevBuf<int> probe_done;               // k_finalize_multi's CTA arrival counter
  // multi-GPU (sharded) buffers: global-order block arrays, records, staging
  int64_t nb_global_cap = 0, stage_cap = 0;
  int stage_n = 0;
  DevBuf<double> g_part, g_err0, g_part_multi, g_scratch_multi, g_scratch;
  DevBuf<double> g_val;  // [kMaxRanks]: per-rank scalars of the validate_invariants checks
  DevBuf<int64_t> g_cnt, g_off, g_off_probe, g_cnt_multi, g_kb;
  DevBuf<unsigned long long> g_mm;
  DevBuf<BlockRec> rec_send, rec_recv;
  DevBuf<ProbeRec> prec_send, prec_recv;
  DevBuf<double> st_low, st_len, st_pest;
  int64_t* h_kb = nullptr;  // pinned [kMaxRanks + 1]
  int64_t* h_kbzc = nullptr;  // mapped pinned [kMaxRanks + 1]: zero-copy kept bounds
  int64_t* d_kbzc = nullptr;  // device alias of h_kbzc
  void ensure_shard(int R, int n, int64_t nb_global, int64_t nblk_max_cap, int64_t stage);
  DevBuf<FoldScalars> d_sc;
  DevBuf<unsigned long long> mm_keys;
  DevBuf<double> mm_out, d_lower, d_step, d_tmp;
  FoldScalars* h_sc = nullptr;  // pinned [2]
  // zero-copy per-iteration scalars (mapped pinned memory, see k_finalize)
  FoldScalars* h_zc = nullptr;
  FoldScalars* d_zc = nullptr;  // device alias of h_zc
  unsigned* h_ready = nullptr;
  unsigned* d_ready = nullptr;
  unsigned seq = 0;
  double* h_mm = nullptr;       // pinned [4]
  std::vector<cudaEvent_t> ev;
  void ensure(int n, int64_t cap);
  cudaEvent_t event(size_t i);
  ~Workspace();
};

Workspace& workspace_for(int device);

// sequential.cu: integrate_sequential (sequential.cpp:45-139) on the device.
void integrate_sequential(const pagani_integrand* f, int ndim, const double* lower,
                          const double* upper, double tau_rel, double tau_abs, int64_t max_evals,
                          int validate_invariants, int device, int mode, pagani_result* out);
void release_workspaces();

// Integrand descriptor resolved to a device kernel.
struct DeviceIntegrand {
  int fid = 0;
  IntegrandParams params{};
  const pagani_device_fn* ext = nullptr;  // PAGANI_DEVICE_FN
};
// The evaluation kernel of an integrand for dimension n and mode.
EvalLaunch evaluate_kernel(const DeviceIntegrand& di, int n, int mode);
DeviceIntegrand resolve_integrand(const pagani_integrand* f);

struct ThresholdOutcome {
  bool success = false;
  double threshold = 0.0, discarded = 0.0, budget_limit = 0.0;
  int64_t finished_count = 0;
  int attempts = 0, direction_changes = 0;
  double fin_v = 0.0;  // sum of estimates where candidate == 0 (valid on success)
  int minmax_launches = 0;  // kernels launched by min_max (0 or 3)
  int passes = 0;           // speculative probe passes (2 kernels + 1 D2H each)
  int node = -1;            // accepted node of the last pass
  int exact_fallbacks = 0;  // streamed passes too close to call (re-run exactly)
  bool spec_used = false;   // the first pass was the speculative one
  double bytes = 0.0;       // algorithmic HBM bytes read by the search's kernels
};

struct Limits {
  int direction_change_limit = 4, attempt_limit = 40;
  double p_max_start = 0.25, p_max_step = 0.10, p_max_cap = 0.95;
};

// Multi-GPU context of one integrate() call (R > 1).
struct ShardCtx {
  Comm* comm = nullptr;
  int R = 1, rank = 0;
  std::vector<int64_t> bounds;  // global partition of the current batch
  RankBlocks rb{};
  int64_t nblk_max = 0, nblk_global = 0;
  void set_bounds(std::vector<int64_t> b);
  int64_t first() const { return bounds[rank]; }
  int64_t local() const { return bounds[rank + 1] - bounds[rank]; }
};

// classify.cpp:37-95 over device arrays (flags unchanged; candidates are
// re-derived from the returned threshold).  Leaves, on success, the probe's
// block offsets in ws.off_probe (1 GPU) or ws.g_off (sharded, global blocks).
// minmax: {min, max} of the errors if already known (fused fold), else null.
ThresholdOutcome device_threshold(Workspace& ws, int64_t m, const double* d_est,
                                  const double* d_err, const uint8_t* d_flag, double v_tot,
                                  double e_tot, double e_it, int64_t s_it, double tau_rel,
                                  const Limits& lim, double* probe_ms,
                                  const double* minmax = nullptr, ShardCtx* sh = nullptr,
                                  unsigned spec_seq = 0);

void integrate(const pagani_integrand* f, int ndim, const double* lower, const double* upper,
               const pagani_config* cfg, pagani_result* out);

bool digits_converged(double v_prev, double v_curr, int digits);
int convergence_digits(double tau_rel);
int initial_subdivisions(int n, int64_t init_target);

}  // namespace pgn
