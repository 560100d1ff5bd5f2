"""B200-native PAGANI (arXiv 2104.06494) hot path.

The breadth-first cubature iteration of the reference library `bfcub`
(/root/reference/proj) rebuilt as hand-written sm_100a kernels behind the
reference's own integrate(integrand, bounds, config) API.  See DESIGN.md.
"""
from .api import (Bounds, Config, FilterResult, IntegrationResult, Integrand, RegionBatch,
                  Status, ThresholdEvent, ThresholdLimits, ThresholdResult, apply_threshold,
                  bisect, block_sum, block_sum_where, build_rule, check_termination,
                  count_flags, device_count, digits_converged, evaluate_batch, filter,
                  glibc_cos, glibc_exp, initial_subdivisions, integrand_by_id, integrate, integrate_sequential,
                  known_integrand, min_max, rel_err_classify, release, rule_point_count,
                  threshold_classify, to_string, two_level_refine, uniform_split)
from .suite import IntegrandSpec, reference_value, suite

__all__ = [
    "Bounds", "Config", "FilterResult", "IntegrationResult", "Integrand", "RegionBatch",
    "Status", "ThresholdEvent", "ThresholdLimits", "ThresholdResult", "apply_threshold",
    "bisect", "block_sum", "block_sum_where", "build_rule", "check_termination", "count_flags",
    "device_count", "digits_converged", "evaluate_batch", "filter", "glibc_cos", "glibc_exp",
    "initial_subdivisions", "integrand_by_id", "integrate", "integrate_sequential", "known_integrand", "min_max",
    "rel_err_classify", "release", "rule_point_count", "threshold_classify", "to_string",
    "two_level_refine", "uniform_split", "IntegrandSpec", "reference_value", "suite",
]
