// Region-store kernels around k_evaluate: deterministic block folds, the
// pairwise tree, min/max, threshold probes, fused filter+bisect, uniform split.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pagani.h"
#include "evaluate.cuh"

namespace pgn {

// reduce.cpp:10 -- block size of the deterministic sums.  Every global fp64
// sum in the loop is "serial inside fixed 2048-element blocks, then a fixed
// pairwise tree over the block partials" (reduce.cpp:13-64); reproducing that
// exactly is what makes v, e, v_f, e_f and the threshold sums bit-identical.
constexpr int64_t kBlock = 2048;

inline int64_t nblocks_of(int64_t m) { return (m + kBlock - 1) / kBlock; }

// Launch with programmatic stream serialization (the kernel calls pdl_wait()
// before touching its predecessor's outputs); PAGANI_PDL=0 launches plainly.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// Scalars produced by k_finalize (device) and copied to pinned host memory.
struct FoldScalars {
  double sum[4];
  int64_t count;
  int64_t pad;
  double mn, mx;  // min/max of the errors (when block keys are supplied)
};

// Speculative probe set: a level-order binary tree of candidate thresholds.
constexpr int kMaxProbes = 15;
struct ProbeSet {
  int T;
  int nan_cnt;           // thresholds that are NaN (they occupy sorted positions 0..nan_cnt-1)
  double t[kMaxProbes];  // tree order (node j)
  // Filled by prepare_probes(): finite thresholds ascending, NaN-padded to 16,
  // and the sorted position of every node.  A region's code is
  // flag ? (err NaN ? 16 : nan_cnt + #{s_k <= err}) : 0, and it is a
  // candidate of node j  <=>  code > pos[j]  <=>  flag && !(err < t[j]).
  double s[16];
  int pos[kMaxProbes];
  int pad2;
};
// Host: sort the node thresholds into ps.s / ps.pos / ps.nan_cnt.
void prepare_probes(ProbeSet& ps);

// The first pass of a search (classify.cpp:61-89): root t0 = e_it / s_it and
// the depth-4 subtree of its next steps, (t + max) / 2 toward max and
// (t + min) / 2 toward min.  One definition for the host (device_threshold)
// and the device (k_finalize's speculative pass), so both build the same bits.
__host__ __device__ inline void build_probe_tree(ProbeSet& ps, double t0, double mn, double mx) {
  ps.T = kMaxProbes;
  ps.t[0] = t0;
  for (int k = 0; 2 * k + 2 < kMaxProbes; ++k) {
    ps.t[2 * k + 1] = P_MUL(P_ADD(ps.t[k], mx), 0.5);
    ps.t[2 * k + 2] = P_MUL(P_ADD(ps.t[k], mn), 0.5);
  }
}

// Where k_finalize builds the speculative first pass of the next search
// (the ProbeSet the probe kernel reads; nullptr = off).
struct SpecProbe {
  ProbeSet* dev = nullptr;
  int64_t s_it = 0;  // the global batch size (the search's s_it)
};
struct ProbeScalars {
  double err_sum[kMaxProbes];  // sum err where candidate == 0 (discarded)
  double est_sum[kMaxProbes];  // sum est where candidate == 0
  long long count[kMaxProbes]; // #candidate == 1
};

using EvalKernel = void (*)(const EvalParams, const uint64_t*, const double*);
struct EvalLaunch {
  EvalKernel fn = nullptr;
  size_t smem = 0;          // dynamic shared memory bytes
  bool fused_fold = false;  // kernel runs the 2048-block folds in its tail
  const pagani_device_fn* ext = nullptr;  // caller-compiled kernel (PAGANI_DEVICE_FN)
  int mode = 0;                           // for ext
  EvalKernel fn_link = nullptr;  // deferred-bisection form (EvalParams.link), when it exists
  bool valid() const { return fn != nullptr || ext != nullptr; }
};

// ---- launchers (kernels.cu) ------------------------------------------------
// uniform_split of the unit cube (geometry.cpp:83-112), axis-major.
void launch_uniform_split(cudaStream_t st, int n, int d, int64_t m, int64_t cap, double* low,
                          double* len, const double* lower, const double* step,
                          int64_t first = 0);

// Post-evaluation block folds: q0 = sum est, q1 = sum err,
// q2 = sum est[flag==0] (+ count flag==1), q3 = sum err[flag==0].
// use_t: under the final flags of threshold t (flag && !(err < t)).
void launch_fold_eval(cudaStream_t st, int64_t m, const double* est, const double* err,
                      const uint8_t* flag, double* part, int64_t* cnt, int use_t = 0,
                      double t = 0.0);

// Candidate flags of an accepted threshold (classify.cpp:63-66), batch API.
void launch_candidates(cudaStream_t st, int64_t m, double t, const uint8_t* flag,
                       const double* err, uint8_t* out);

// Generic fold of one array with optional mask (block_sum / block_sum_where).
void launch_fold_one(cudaStream_t st, int64_t m, const double* x, const uint8_t* flag,
                     int which, double* part, int64_t* cnt);

// Pairwise trees over nq partial arrays (stride nblk) + exclusive scan of cnt
// (+ min/max of the errors from per-block keys mm, if given; err0 = &err[0]).
// With `ready`, `out` is mapped pinned host memory and the kernel publishes
// `seq` at *ready once every field is visible to the host (zero-copy hand-off).
void launch_finalize(cudaStream_t st, int64_t nblk, int nq, const double* part,
                     const int64_t* cnt, int64_t* offsets, double* scratch, FoldScalars* out,
                     const unsigned long long* mm = nullptr, const double* err0 = nullptr,
                     unsigned* ready = nullptr, unsigned seq = 0,
                     const SpecProbe& spec = SpecProbe{});

// The speculative first pass: k_probe_multi + its trees with the ProbeSet
// k_finalize left in device memory (both programmatic launches).
void launch_probe_multi_dev(cudaStream_t st, int64_t m, const ProbeSet* dts, const double* est,
                            const double* err, const uint8_t* flag, double* part, int64_t* cnt,
                            double* scratch, ProbeScalars* out, unsigned* ready, unsigned seq,
                            int* done);

// T speculative probes in one pass + their trees; part [2][kMaxProbes][nblk],
// cnt [kMaxProbes][nblk], scratch 2*3*kMaxProbes*nblk doubles.
// With `ready`, `out` is mapped host memory and the last tree CTA publishes
// `seq` there (zero-copy hand-off; `done` = a zeroed device counter).
void launch_probe_multi(cudaStream_t st, int64_t m, const ProbeSet& ts, const double* est,
                        const double* err, const uint8_t* flag, double* part, int64_t* cnt,
                        double* scratch, ProbeScalars* out, unsigned* ready = nullptr,
                        unsigned seq = 0, int* done = nullptr);
void launch_scan_counts(cudaStream_t st, int64_t nblk, const int64_t* cnt, int64_t* offsets);

// Fast probe pass (exact counts, fast sums of the discarded error per node)
// into mapped `out`, published with `seq`.  part / cnt: kMaxProbes x
// probe_fast_grid(m) scratch.
int probe_fast_grid(int64_t m);
// Exact block folds of est (q = 0) and err (q = 1) over the non-candidates
// of threshold t, and per-block candidate counts: part[q * nblk + b], cnt[b].
void launch_fold_threshold(cudaStream_t st, int64_t m, const double* est, const double* err,
                           const uint8_t* flag, double t, double* part, int64_t* cnt);
void launch_probe_fast(cudaStream_t st, int64_t m, const ProbeSet& ts, const double* err,
                       const uint8_t* flag, double* part, int64_t* cnt, ProbeScalars* out,
                       unsigned* ready, unsigned seq);

// min_max over err (reduce.cpp:74-82).  out[0] = min, out[1] = max, as doubles.
void launch_minmax(cudaStream_t st, int64_t m, const double* x, unsigned long long* keys,
                   double* out);

// Sharded runs: children whose (local) index c lies in [lo, hi) stay on this
// rank and are written straight into the next batch at c - lo + dst (stride
// cap); the others go to the staging buffers for the exchange.
struct SplitWindow {
  double* low = nullptr;
  double* len = nullptr;
  double* pest = nullptr;
  int64_t cap = 0, lo = 0, hi = 0, dst = 0;
};

// Fused filter (classify.cpp:97-129) + bisect (geometry.cpp:114-143): region
// j with flag 1 and rank k among the kept writes children 2k, 2k+1 into dst.
// kbase: subtracted from the (global) kept rank before writing children.
// bulk: the TMA-staged form (k_split_bulk); it needs the kept offsets and
// kept_end = the kept rank just past this launch's regions.
void launch_split(cudaStream_t st, int n, int64_t m, int64_t cap_src, int64_t cap_dst,
                  const uint8_t* flag, int use_t, double t, const int64_t* offsets,
                  const double* est,
                  const double* err, const uint8_t* axis, const double* low, const double* len,
                  double* dlow, double* dlen, double* dpest, double* dperr, int64_t kbase = 0,
                  const SplitWindow& win = SplitWindow{}, bool bulk = false,
                  int64_t kept_end = -1);

// Filter only, bisection deferred into the next k_evaluate (EvalParams.link):
// link[k] = j | axis[j] << 56, pest[k] = est[j] for the k-th kept region j.
void launch_link(cudaStream_t st, int64_t m, const uint8_t* flag, int use_t, double t,
                 const int64_t* offsets, const double* est, const double* err,
                 const uint8_t* axis, uint64_t* link, double* pest);

// Compaction only (filter() for the batch API).
void launch_compact(cudaStream_t st, int n, int64_t m, int64_t cap, const uint8_t* flag,
                    const int64_t* offsets, const double* low, const double* len,
                    const double* est, const double* err, const int32_t* axis,
                    const double* pest, const double* perr, double* klow, double* klen,
                    double* kest, double* kerr, int32_t* kaxis, double* kpest, double* kperr);

// Elementwise helpers for the batch API.
void launch_refine(cudaStream_t st, int64_t m, const double* est, const double* raw,
                   const double* pest, double* out);
void launch_classify(cudaStream_t st, int64_t m, const double* est, const double* err,
                     double tau, int enabled, uint8_t* flags);
void launch_apply_threshold(cudaStream_t st, int64_t m, const double* err, double t,
                            uint8_t* flags);
void launch_serial_volume(cudaStream_t st, int n, int64_t m, int64_t cap, const double* len,
                          const uint8_t* flag, int which, double* out);
// Serial 2048-block partials of the kept estimates in compacted order.
void launch_kept_partials(cudaStream_t st, int64_t m, const uint8_t* flag, int use_t, double t,
                          const double* err, const double* est, double* part);
void launch_math(cudaStream_t st, int which, int64_t m, const double* x, double* y);
void launch_call_integrand(cudaStream_t st, int fid, int n, int64_t m, const double* x,
                           const IntegrandParams& ip, double* y);

// ---- multi-GPU block records (allgathered once per fold / probe pass) ----
struct BlockRec {  // per 2048-block fold results of k_evaluate's tail
  double part[4];
  long long cnt;
  unsigned long long mn, mx;
  double pad;
};
struct ProbeRec {  // per 2048-block results of a speculative probe pass
  double err_sum[kMaxProbes];
  double est_sum[kMaxProbes];
  long long cnt[kMaxProbes];
};
constexpr int kMaxRanks = 64;
struct RankBlocks {  // global block index of each rank's first block, and counts
  int R;
  int pad;
  long long first[kMaxRanks];
  long long nblk[kMaxRanks];
};
// recs[0] is a header: part[0] = err[0] of the slice, cnt = #local blocks.
void launch_pack_blocks(cudaStream_t st, int64_t nblk_local, int64_t nblk_max, const double* part,
                        const int64_t* cnt, const unsigned long long* mm, const double* err,
                        BlockRec* recs);
void launch_unpack_blocks(cudaStream_t st, const RankBlocks& rb, int64_t nblk_max,
                          int64_t nblk_global, const BlockRec* all, double* part, int64_t* cnt,
                          unsigned long long* mm, double* err0);
void launch_pack_probe(cudaStream_t st, int64_t nblk_local, int64_t nblk_max, int T,
                       const double* part, const int64_t* cnt, ProbeRec* recs);
void launch_unpack_probe(cudaStream_t st, const RankBlocks& rb, int64_t nblk_max,
                         int64_t nblk_global, int T, const ProbeRec* all, double* part,
                         int64_t* cnt);
void launch_probe_only(cudaStream_t st, int64_t m, const ProbeSet& ts, const double* est,
                       const double* err, const uint8_t* flag, double* part, int64_t* cnt);
void launch_finalize_multi(cudaStream_t st, int64_t nblk, int T, const double* part,
                           const int64_t* cnt, double* scratch, ProbeScalars* out,
                           unsigned* ready = nullptr, unsigned seq = 0, int* done = nullptr);
// out[r] = offsets[first_block[r]] (r < R), out[R] = total (from FoldScalars-like count)
// With `ready`, `out` is mapped host memory and the kernel publishes `seq`.
void launch_gather_bounds(cudaStream_t st, const RankBlocks& rb, const int64_t* offsets,
                          const int64_t* cnt, int64_t nblk_global, int64_t* out,
                          unsigned* ready = nullptr, unsigned seq = 0);

// Device copies of the glibc tables.
const uint64_t* device_exp_table();
const double* device_sincos_table();

// k_evaluate dispatch (eval_*.cu): fn == nullptr if (fid, n, mode) is unsupported.
EvalLaunch lookup_evaluate(int fid, int n, int mode);
// Launch k_evaluate for m regions on `st` (sets the dynamic-smem attribute once).
void launch_evaluate(const EvalLaunch& k, cudaStream_t st, const EvalParams& ep);

}  // namespace pgn
