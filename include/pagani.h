/*
 * pagani.h -- C ABI of the B200-native PAGANI hot path (libpagani_b200.so).
 *
 * Drop-in boundary for the reference library `bfcub` (arXiv 2104.06494 CPU
 * implementation, /root/reference/proj).  Every entry point below names the
 * reference interface it replaces (file:line under /root/reference/proj).
 * All pointers are HOST pointers; the library owns device memory, streams and
 * NCCL communicators internally.  Return codes: 0 = ok, negative = error, with
 * the message in pagani_last_error() (thread-local):
 *   PAGANI_E_INVALID  (-1)  std::invalid_argument in the reference
 *   PAGANI_E_RUNTIME  (-2)  std::runtime_error    (e.g. uniform_split cap)
 *   PAGANI_E_LOGIC    (-3)  std::logic_error      (bisect cap, invariants)
 *   PAGANI_E_CUDA     (-10) CUDA error (no device, launch failure, OOM)
 *   PAGANI_E_NCCL     (-11) NCCL error (multi-GPU)
 *   PAGANI_E_UNSUPPORTED (-12) integrand kind the device cannot evaluate
 *                          (e.g. a host function pointer: there is NO CPU fallback)
 */
#ifndef PAGANI_H_
#define PAGANI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* The library is built with -fvisibility=hidden; everything declared in this
 * header is exported. */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define PAGANI_ABI_VERSION 3

#define PAGANI_OK 0
#define PAGANI_E_INVALID (-1)
#define PAGANI_E_RUNTIME (-2)
#define PAGANI_E_LOGIC (-3)
#define PAGANI_E_CUDA (-10)
#define PAGANI_E_NCCL (-11)
#define PAGANI_E_UNSUPPORTED (-12)

/* Status, driver.hpp:14 (enum class Status { Converged, MaxIterations, MemoryExhausted }) */
#define PAGANI_CONVERGED 0
#define PAGANI_MAX_ITERATIONS 1
#define PAGANI_MEMORY_EXHAUSTED 2

/* ---- integrand (replaces bfcub::Integrand, integrand.hpp:8-13) ----------
 * The reference takes a host function pointer called once per (region,point).
 * A GPU cannot call host code, so the device evaluates one of:
 *   PAGANI_BUILTIN: f1..f8 of the reference suite (integrands.cpp:24-79),
 *                   builtin_id 1..8, and the reference unit-test integrands
 *                   PAGANI_TEST_* (tests/test_*.cpp lambdas), parameterised by
 *                   params[].
 *   PAGANI_HOST_FN: rejected with PAGANI_E_UNSUPPORTED (no CPU fallback).
 *   PAGANI_DEVICE_FN: a user integrand compiled for the GPU by the caller
 *                   (include/pagani_device.cuh instantiates the evaluation
 *                   kernel for a C++ functor and fills device_fn); this is
 *                   the device counterpart of the reference's arbitrary
 *                   {fn, ctx} integrand (integrand.hpp:8-13).
 * `magic` must be PAGANI_INTEGRAND_MAGIC.                                     */
#define PAGANI_INTEGRAND_MAGIC 0x50474e49u /* 'PGNI' */
#define PAGANI_BUILTIN 0
#define PAGANI_HOST_FN 1
#define PAGANI_DEVICE_FN 2

/* A caller-compiled evaluation kernel (PAGANI_DEVICE_FN).  `launch` runs the
 * PAGANI evaluation of one batch of m regions on `stream` (a cudaStream_t):
 * `params` points at the library's parameter block of `params_size` bytes,
 * which the kernel was compiled against (a size mismatch means a header /
 * library version mismatch and is rejected); the two table pointers are the
 * device copies of glibc's exp / sincos tables.  Returns 0 or a cudaError_t. */
#define PAGANI_DEVICE_FN_MAGIC 0x50474e44u /* 'PGND' */
typedef struct pagani_device_fn {
  uint32_t magic;
  uint32_t params_size;
  int (*launch)(const void* params, uint32_t params_size, const void* exp_table,
                const void* sincos_table, void* stream, int64_t m, int32_t mode, void* user);
  void* user;
} pagani_device_fn;

#define PAGANI_F1 1 /* cos(sum (i+1) x_i)                 integrands.cpp:24-28 */
#define PAGANI_F2 2 /* prod 1/(1/2500 + (x_i - 1/2)^2)    integrands.cpp:30-37 */
#define PAGANI_F3 3 /* (1 + sum (i+1) x_i)^-(n+1)         integrands.cpp:39-43 */
#define PAGANI_F4 4 /* exp(-625 sum (x_i - 1/2)^2)        integrands.cpp:45-52 */
#define PAGANI_F5 5 /* exp(-10 sum |x_i - 1/2|)           integrands.cpp:54-58 */
#define PAGANI_F6 6 /* exp(sum (i+5) x_i) inside the box  integrands.cpp:60-67 */
#define PAGANI_F7 7 /* (sum x_i^2)^11                     integrands.cpp:69-73 */
#define PAGANI_F8 8 /* (sum x_i^2)^7 sqrt(sum x_i^2)      integrands.cpp:75-79 */
#define PAGANI_TEST_CONST 100    /* p0                              test_driver.cpp:22-32 */
#define PAGANI_TEST_MONOMIAL 101 /* prod x_i^p_i (repeated mult.)   test_rule.cpp:40-49   */
#define PAGANI_TEST_ROUGH 102    /* sum cos(p0 x^p1) + p2 n         test_driver.cpp:61-80 */
#define PAGANI_TEST_NANBOX 103   /* NaN if x0>p0 (&& x1>p1 if p1>=0) test_rule.cpp:237-254 */
#define PAGANI_TEST_POCKET 104   /* 1 if x0,x1,x2 > p0              test_rule.cpp:217-235 */
#define PAGANI_TEST_COSSUM 105   /* p0 sum cos(p_{1+i} 3 x_i)       test_rule.cpp:191-215 */
#define PAGANI_TEST_EXPSQ 106    /* sum exp(x_i/3) + x_i^2          test_rule.cpp:154-189 */

#define PAGANI_MAX_PARAMS 32
#define PAGANI_MAX_DIM 16 /* geometry.hpp:8 kMaxDim */

typedef struct pagani_integrand {
  uint32_t magic;
  int32_t kind;       /* PAGANI_BUILTIN | PAGANI_HOST_FN | PAGANI_DEVICE_FN */
  int32_t builtin_id; /* PAGANI_F1.. / PAGANI_TEST_* */
  int32_t n_params;
  double params[PAGANI_MAX_PARAMS];
  double (*host_fn)(const double* x, int n, void* ctx); /* PAGANI_HOST_FN only */
  void* host_ctx;
  const pagani_device_fn* device_fn; /* PAGANI_DEVICE_FN only */
} pagani_integrand;

/* ---- config (replaces bfcub::Config, driver.hpp:30-45, and ThresholdLimits,
 *      classify.hpp:23-29).  pagani_config_default() fills the reference
 *      defaults.                                                             */
#define PAGANI_REFINER_TWO_LEVEL 0 /* errorest.cpp:10-37 (default) */
#define PAGANI_REFINER_IDENTITY 1  /* refined = raw                  */

#define PAGANI_MODE_PARITY 0 /* bit-exact with the reference (default) */
#define PAGANI_MODE_FAST 1   /* per-orbit sums + FMA; final within 1e-12 */

typedef struct pagani_config {
  double tau_rel;               /* 1e-3  */
  double tau_abs;               /* 1e-20 */
  int32_t it_max;               /* 100   */
  int32_t init_subdiv;          /* 0 = derive from init_target */
  int64_t max_regions;          /* 2^22  */
  int64_t init_target;          /* 2^14  */
  int32_t rel_filtering_enabled;/* 1     */
  int32_t threads;              /* ignored on the GPU (OpenMP knob in the reference) */
  int32_t validate_invariants;  /* 0     */
  int32_t refiner;              /* PAGANI_REFINER_*  (Config::refiner fn pointer) */
  int32_t direction_change_limit; /* 4  */
  int32_t attempt_limit;          /* 40 */
  double p_max_start;             /* 0.25 */
  double p_max_step;              /* 0.10 */
  double p_max_cap;               /* 0.95 */
  /* B200 extensions */
  int32_t mode;                 /* PAGANI_MODE_* */
  int32_t device;               /* CUDA device ordinal (single-process) */
  int32_t profile;              /* 1 = record per-kernel CUDA-event times; 2 = k_evaluate's
                                   only (two event records per iteration instead of ~8:
                                   the host-side record calls sit on the GPU's critical path
                                   between host decisions and the next launch) */
  int32_t reserved0;
  /* per-iteration trace callback (full-precision BFCUB_TRACE, driver.cpp:174-182) */
  void (*trace)(const struct pagani_trace_row* row, void* user);
  void* trace_user;
  /* multi-GPU: one process per GPU.  comm == NULL -> single GPU. */
  void* comm; /* from pagani_comm_init_rank() */
} pagani_config;

/* ThresholdEvent, driver.hpp:47-58 */
typedef struct pagani_threshold_event {
  int32_t iteration;
  int32_t success;
  int64_t batch_size;
  int64_t finished_count;
  double discarded_error;
  double budget_limit;
} pagani_threshold_event;

#define PAGANI_MAX_EVENTS 256
#define PAGANI_N_KERNEL_SLOTS 8
/* kernel slots of pagani_result.kernel_ms / kernel_launches */
#define PAGANI_K_EVALUATE 0
#define PAGANI_K_FOLD 1     /* block partial folds (rel-err classify + block_sum) */
#define PAGANI_K_FINALIZE 2 /* pairwise trees + offsets */
#define PAGANI_K_MINMAX 3
#define PAGANI_K_PROBE 4    /* threshold probes */
#define PAGANI_K_SPLIT 5    /* filter + bisect */
#define PAGANI_K_INIT 6     /* uniform split */
#define PAGANI_K_EXCHANGE 7 /* sharded runs: post-bisection region exchange; kernel_bytes =
                               bytes this rank sent to peers (region geometry + parent est),
                               kernel_launches = exchanges with a peer transfer */

/* IntegrationResult, driver.hpp:60-68 (+ timing) */
typedef struct pagani_result {
  double estimate;
  double errorest;
  int32_t status;
  int32_t iterations;
  int64_t regions_generated;
  int64_t eval_count;
  int32_t n_events; /* may exceed PAGANI_MAX_EVENTS; events[] holds the first ones */
  int32_t probe_fallbacks; /* threshold passes whose streamed sums were too close to the
                              budget to decide and were re-run with the exact folds */
  pagani_threshold_event events[PAGANI_MAX_EVENTS];
  double wall_ms;                              /* host wall time of the call */
  double kernel_ms[PAGANI_N_KERNEL_SLOTS];     /* CUDA-event time per kernel kind (profile=1) */
  int64_t kernel_launches[PAGANI_N_KERNEL_SLOTS];
  int64_t region_evals;                        /* sum over iterations of batch sizes */
  int64_t peak_regions;
  int64_t h2d_bytes, d2h_bytes;
  double device_ms; /* CUDA-event span on the driver stream: first kernel -> last */
  /* Algorithmic HBM bytes per kernel kind (what each launch must read and
   * write), for the HBM rooflines of the memory kernels. */
  double kernel_bytes[PAGANI_N_KERNEL_SLOTS];
  /* Speculative first threshold passes: launched behind
   * k_finalize before the host decided whether a search runs, and how many of
   * them ran for nothing (no search that iteration). */
  int32_t spec_probe_passes;
  int32_t spec_probe_wasted;
} pagani_result;

/* One row per iteration (the BFCUB_TRACE point, driver.cpp:174-182, in full
 * precision, plus the filter outcome).  Layout shared with the oracle shim. */
typedef struct pagani_trace_row {
  int32_t it, trig_digits, trig_memory, thr_invoked;
  int64_t m, active_rel, active_final, kept;
  double v, e, v_f, e_f;
  double fin_v, fin_e;
  int32_t thr_success, thr_accepted, thr_attempts, thr_dir_changes;
  double thr_threshold, thr_discarded, thr_budget;
  int64_t thr_finished;
} pagani_trace_row;

/* ---- library ------------------------------------------------------------- */
int pagani_abi_version(void);
const char* pagani_last_error(void);
void pagani_config_default(pagani_config* cfg);
void pagani_integrand_builtin(pagani_integrand* f, int builtin_id, const double* params,
                              int n_params);
int pagani_device_count(int* count);
/* Frees cached device workspaces (they are reused across calls). */
int pagani_release(void);

/* ---- the hot path: bfcub::integrate (driver.hpp:77-79, driver.cpp:83-215) -- */
int pagani_integrate(const pagani_integrand* f, int ndim, const double* lower,
                     const double* upper, const pagani_config* cfg, pagani_result* out);

/* ---- batch-level entry points (device-backed; host arrays in/out) ---------
 * Region batches are REGION-MAJOR (m x n) on the host, as RegionBatch stores
 * them (geometry.hpp:32-33); the device stores them axis-major.            */

/* rule.hpp:51 rule_point_count */
int64_t pagani_rule_point_count(int n);
/* rule.hpp:53 build_rule: orbit weights [5 sets x 5 orbits] (set-major:
 * w[k*5+o]), generator magnitudes l2..l5, expanded points (N x n, may be NULL)
 * and packed weight sets (5 x N, may be NULL). */
int pagani_build_rule(int n, double* orbit_weights, double* generators, double* points,
                      double* weight_sets);
/* rule.hpp:67-68 evaluate_batch */
int pagani_evaluate_batch(const pagani_integrand* f, int n, int64_t m, const double* lows,
                          const double* lengths, double* estimates, double* raw_errors,
                          int32_t* split_axes, int64_t* eval_count, int32_t mode);
/* errorest.hpp:20-24 two_level_refine */
int pagani_two_level_refine(int64_t m, const double* estimates, const double* raw_errors,
                            const double* parent_estimates, const double* parent_errors,
                            double* refined);
/* classify.hpp:16-18 rel_err_classify */
int pagani_rel_err_classify(int64_t m, const double* estimates, const double* errors,
                            double tau_rel, int32_t filtering_enabled, uint8_t* flags);
/* classify.hpp:21 apply_threshold */
int pagani_apply_threshold(int64_t m, const double* errors, double t, uint8_t* flags);
/* classify.hpp:31-50 ThresholdResult + threshold_classify */
typedef struct pagani_threshold_result {
  int32_t success, attempts, direction_changes, reserved0;
  double threshold, discarded_error, budget_limit;
  int64_t finished_count;
} pagani_threshold_result;
int pagani_threshold_classify(int64_t m, const uint8_t* active, const double* errors,
                              double v_tot, double e_tot, double e_it, int64_t s_it,
                              double tau_rel, const pagani_config* limits, uint8_t* flags_out,
                              pagani_threshold_result* out);
/* classify.hpp:52-62 filter (kept_* arrays sized m; the first *kept used) */
int pagani_filter(int n, int64_t m, const double* lows, const double* lengths,
                  const double* estimates, const double* errors, const int32_t* split_axis,
                  const double* parent_estimates, const double* parent_errors,
                  const uint8_t* flags, double* kept_lows, double* kept_lengths,
                  double* kept_estimates, double* kept_errors, int32_t* kept_axis,
                  double* kept_parent_estimates, double* kept_parent_errors, int64_t* kept,
                  double* finished_estimate, double* finished_error, double* finished_volume);
/* geometry.hpp:50-52 bisect (children arrays sized 2m) */
int pagani_bisect(int n, int64_t m, const double* lows, const double* lengths,
                  const double* estimates, const double* errors, const int32_t* split_axis,
                  int64_t max_regions, double* child_lows, double* child_lengths,
                  double* child_parent_estimates, double* child_parent_errors);
/* geometry.hpp:45-48 uniform_split (arrays sized d^n) and :55 initial_subdivisions */
int pagani_uniform_split(int n, const double* lower, const double* upper, int d,
                         int64_t max_regions, int64_t* count, double* lows, double* lengths,
                         int64_t capacity);
int pagani_initial_subdivisions(int n, int64_t init_target);
/* reduce.hpp:13-22 */
int pagani_block_sum(int64_t m, const double* x, double* out);
int pagani_block_sum_where(int64_t m, const double* x, const uint8_t* flags, int32_t which,
                           double* out);
int pagani_count_flags(int64_t m, const uint8_t* flags, int32_t which, int64_t* out);
int pagani_min_max(int64_t m, const double* x, double* lo, double* hi);
/* driver.hpp:71-75 */
int pagani_check_termination(double v, double e, double v_f, double e_f, double tau_rel,
                             double tau_abs);
int pagani_digits_converged(double v_prev, double v_curr, int digits);
int pagani_convergence_digits(double tau_rel);

/* integrate_sequential (sequential.hpp:15-18, sequential.cpp:45-139): the
 * reference's globally adaptive comparison engine (Alg. 1) -- one region per
 * step from a max-error heap -- with each step's two children evaluated and
 * refined on the GPU.  Bit-identical to the reference.  mode: PAGANI_MODE_*.
 * out->iterations = steps; status CONVERGED or MAX_ITERATIONS (eval budget). */
int pagani_integrate_sequential(const pagani_integrand* f, int ndim, const double* lower,
                                const double* upper, double tau_rel, double tau_abs,
                                int64_t max_evals, int32_t validate_invariants, int32_t device,
                                int32_t mode, pagani_result* out);

/* Reference value of suite integrand `id` ("f1".."f8") in dimension n
 * (integrands.cpp:178-188 reference_for, long double, bit-identical).
 * flags: PAGANI_REFVAL_CORRECTED clamps f6's cut-off to the cube (the
 * reference does not, integrands.cpp:133-140); PAGANI_REFVAL_EXTENDED allows
 * f8 outside n in {2,3,8} (values from the reference's golden_box_values). */
#define PAGANI_REFVAL_CORRECTED 1
#define PAGANI_REFVAL_EXTENDED 2
int pagani_reference_value(const char* id, int n, int32_t flags, double* out);

/* glibc-exact math used by the device integrands, exported for verification.
 * exp: on_device 0 = host build of the same source, 1 = GPU, 2 = GPU paired
 * form (gm_exp2_s: x[2i], x[2i+1] as one pair, as the evaluator calls it).
 * cos: 0 = host gm_cos, 1 = GPU gm_cos, 2 = GPU branch-free gm_cos_bf, 3 =
 * host gm_cos_bf, 4 = GPU paired form (gm_cos2_s, f1's hot path). */
int pagani_math_exp(int64_t m, const double* x, double* y, int32_t on_device);
int pagani_math_cos(int64_t m, const double* x, double* y, int32_t on_device);
/* Evaluate a builtin integrand at host points (m x n), on the device. */
int pagani_call_integrand(const pagani_integrand* f, int n, int64_t m, const double* x,
                          double* y);

/* FP64 roofline denominator: a DFMA-chain microbenchmark over every SM of
 * `device` for about `seconds`; returns the achieved FP64 TFLOP/s (2 flops
 * per DFMA) and the SM clock (MHz) seen by the kernel. */
int pagani_fp64_peak(int device, double seconds, double* tflops, double* sm_mhz);

/* ---- multi-GPU (one process per GPU) ----------------------
 * unique_id: 128 bytes produced by pagani_comm_unique_id() on rank 0 and
 * broadcast by the caller (e.g. torch.distributed).  The communicator binds
 * `device` and is passed in pagani_config.comm.                              */
#define PAGANI_COMM_ID_BYTES 128
int pagani_comm_unique_id(uint8_t* unique_id);
int pagani_comm_init_rank(const uint8_t* unique_id, int nranks, int rank, int device,
                          void** comm);
/* Host-callback transport (e.g. torch.distributed / gloo): the library stages
 * device buffers through host memory and calls back.  Lets R ranks share one
 * GPU (tests) or run where NCCL is unavailable.  Callbacks return 0 on success.
 *   allgather: recv holds size * bytes, rank-major.
 *   exchange : one group of point-to-point sends and receives. */
typedef struct pagani_host_transport {
  int32_t rank, size;
  void* user;
  int (*allgather)(const void* send, void* recv, size_t bytes, void* user);
  int (*exchange)(int n_send, const int* send_peer, const void* const* send_buf,
                  const size_t* send_bytes, int n_recv, const int* recv_peer,
                  void* const* recv_buf, const size_t* recv_bytes, void* user);
} pagani_host_transport;
int pagani_comm_init_host(const pagani_host_transport* transport, int device, void** comm);
int pagani_comm_destroy(void* comm);

/* Shard logic (host only; exported so it can be tested without a GPU).
 * pagani_shard_bounds: balanced 2048-block-aligned partition of m regions,
 * nranks+1 boundaries.  pagani_shard_plan: given kept[r] (global kept index of
 * rank r's first kept region, nranks+1 entries), the pieces rank `rank` sends
 * and receives when the 2*kept[nranks] children are re-partitioned; each piece
 * is 4 int64 {peer, src_offset, dst_offset, count}. */
int pagani_shard_bounds(int64_t m, int nranks, int64_t* bounds);
int pagani_shard_plan(int nranks, int rank, const int64_t* kept, int max_pieces, int32_t* n_send,
                      int64_t* sends, int32_t* n_recv, int64_t* recvs);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* PAGANI_H_ */
