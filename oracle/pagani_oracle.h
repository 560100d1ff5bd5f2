/*
 * TEST INFRASTRUCTURE ONLY -- the plain-C restatement of the reference's
 * PAGANI hot path (/root/reference/proj/src), used as a checker by tests/ and
 * never linked into the product.  Same orc_* surface as oracle/ref_shim.cpp's
 * ref_* functions so tests can run one check against either.
 *
 * Parity status: pinned.  tests/test_oracle.py checks this restatement bit
 * for bit against the unmodified reference library (oracle/_ref) on full
 * per-iteration traces, batch functions, and the 300-instance threshold
 * trace-oracle workload of test_classify.cpp.
 */
#ifndef PAGANI_ORACLE_H_
#define PAGANI_ORACLE_H_

#include <stdint.h>

typedef struct {
  double tau_rel, tau_abs;
  int32_t it_max, init_subdiv;
  int64_t max_regions, init_target;
  int32_t rel_filtering_enabled, threads, validate_invariants, refiner;
  int32_t direction_change_limit, attempt_limit;
  double p_max_start, p_max_step, p_max_cap;
} orc_config;

typedef struct {
  int32_t iteration, success;
  int64_t batch_size, finished_count;
  double discarded_error, budget_limit;
} orc_event;

typedef struct {
  double estimate, errorest;
  int32_t status, iterations;
  int64_t regions_generated, eval_count;
  int32_t n_events, pad;
} orc_result;

typedef struct {
  int32_t it, trig_digits, trig_memory, thr_invoked;
  int64_t m, active_rel, active_final, kept;
  double v, e, v_f, e_f;
  double fin_v, fin_e;
  int32_t thr_success, thr_accepted, thr_attempts, thr_dir_changes;
  double thr_threshold, thr_discarded, thr_budget;
  int64_t thr_finished;
} orc_trace_row;

typedef struct {
  int32_t success, attempts, direction_changes, pad;
  double threshold, discarded_error, budget_limit;
  int64_t finished_count;
} orc_threshold_out;

#endif
