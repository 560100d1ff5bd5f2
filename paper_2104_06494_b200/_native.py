"""ctypes view of include/pagani.h and the in-tree libpagani_b200.so.

The product path is this library and nothing else: importing fails loudly if
the shared object is missing (no CPU fallback exists).
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PAGANI_LIB") or os.path.join(PKG_DIR, "libpagani_b200.so")
REPO_ROOT = os.path.dirname(PKG_DIR)

PAGANI_OK = 0
PAGANI_E_INVALID = -1
PAGANI_E_RUNTIME = -2
PAGANI_E_LOGIC = -3
PAGANI_E_CUDA = -10
PAGANI_E_NCCL = -11
PAGANI_E_UNSUPPORTED = -12

PAGANI_INTEGRAND_MAGIC = 0x50474E49
PAGANI_BUILTIN = 0
PAGANI_HOST_FN = 1
PAGANI_MAX_PARAMS = 32
PAGANI_MAX_EVENTS = 256
PAGANI_N_KERNEL_SLOTS = 8
KERNEL_SLOTS = ["evaluate", "fold", "finalize", "minmax", "probe", "split", "init", "exchange"]

PAGANI_REFVAL_CORRECTED = 1
PAGANI_REFVAL_EXTENDED = 2

MODE_PARITY = 0
MODE_FAST = 1
REFINER_TWO_LEVEL = 0
REFINER_IDENTITY = 1


class Integrand(C.Structure):
    _fields_ = [("magic", C.c_uint32), ("kind", C.c_int32), ("builtin_id", C.c_int32),
                ("n_params", C.c_int32), ("params", C.c_double * PAGANI_MAX_PARAMS),
                ("host_fn", C.c_void_p), ("host_ctx", C.c_void_p), ("device_fn", C.c_void_p)]


class TraceRow(C.Structure):
    _fields_ = [("it", C.c_int32), ("trig_digits", C.c_int32), ("trig_memory", C.c_int32),
                ("thr_invoked", C.c_int32),
                ("m", C.c_int64), ("active_rel", C.c_int64), ("active_final", C.c_int64),
                ("kept", C.c_int64),
                ("v", C.c_double), ("e", C.c_double), ("v_f", C.c_double), ("e_f", C.c_double),
                ("fin_v", C.c_double), ("fin_e", C.c_double),
                ("thr_success", C.c_int32), ("thr_accepted", C.c_int32),
                ("thr_attempts", C.c_int32), ("thr_dir_changes", C.c_int32),
                ("thr_threshold", C.c_double), ("thr_discarded", C.c_double),
                ("thr_budget", C.c_double), ("thr_finished", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


TRACE_FN = C.CFUNCTYPE(None, C.POINTER(TraceRow), C.c_void_p)


class Config(C.Structure):
    _fields_ = [("tau_rel", C.c_double), ("tau_abs", C.c_double),
                ("it_max", C.c_int32), ("init_subdiv", C.c_int32),
                ("max_regions", C.c_int64), ("init_target", C.c_int64),
                ("rel_filtering_enabled", C.c_int32), ("threads", C.c_int32),
                ("validate_invariants", C.c_int32), ("refiner", C.c_int32),
                ("direction_change_limit", C.c_int32), ("attempt_limit", C.c_int32),
                ("p_max_start", C.c_double), ("p_max_step", C.c_double),
                ("p_max_cap", C.c_double),
                ("mode", C.c_int32), ("device", C.c_int32), ("profile", C.c_int32),
                ("reserved0", C.c_int32),
                ("trace", TRACE_FN), ("trace_user", C.c_void_p), ("comm", C.c_void_p)]


class ThresholdEvent(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("success", C.c_int32),
                ("batch_size", C.c_int64), ("finished_count", C.c_int64),
                ("discarded_error", C.c_double), ("budget_limit", C.c_double)]


class Result(C.Structure):
    _fields_ = [("estimate", C.c_double), ("errorest", C.c_double),
                ("status", C.c_int32), ("iterations", C.c_int32),
                ("regions_generated", C.c_int64), ("eval_count", C.c_int64),
                ("n_events", C.c_int32), ("probe_fallbacks", C.c_int32),
                ("events", ThresholdEvent * PAGANI_MAX_EVENTS),
                ("wall_ms", C.c_double),
                ("kernel_ms", C.c_double * PAGANI_N_KERNEL_SLOTS),
                ("kernel_launches", C.c_int64 * PAGANI_N_KERNEL_SLOTS),
                ("region_evals", C.c_int64), ("peak_regions", C.c_int64),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("device_ms", C.c_double),
                ("kernel_bytes", C.c_double * PAGANI_N_KERNEL_SLOTS),
                ("spec_probe_passes", C.c_int32), ("spec_probe_wasted", C.c_int32)]


class ThresholdResult(C.Structure):
    _fields_ = [("success", C.c_int32), ("attempts", C.c_int32),
                ("direction_changes", C.c_int32), ("reserved0", C.c_int32),
                ("threshold", C.c_double), ("discarded_error", C.c_double),
                ("budget_limit", C.c_double), ("finished_count", C.c_int64)]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p),
                          C.POINTER(C.c_size_t), C.c_int, C.POINTER(C.c_int),
                          C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.c_void_p)


class HostTransport(C.Structure):
    _fields_ = [("rank", C.c_int32), ("size", C.c_int32), ("user", C.c_void_p),
                ("allgather", ALLGATHER_FN), ("exchange", EXCHANGE_FN)]


PAGANI_COMM_ID_BYTES = 128

_D = C.POINTER(C.c_double)
_U8 = C.POINTER(C.c_uint8)
_I32 = C.POINTER(C.c_int32)
_I64 = C.POINTER(C.c_int64)

# name -> (restype, argtypes); mirrors include/pagani.h one to one.
SIGNATURES = {
    "pagani_abi_version": (C.c_int, []),
    "pagani_last_error": (C.c_char_p, []),
    "pagani_config_default": (None, [C.POINTER(Config)]),
    "pagani_integrand_builtin": (None, [C.POINTER(Integrand), C.c_int, _D, C.c_int]),
    "pagani_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "pagani_release": (C.c_int, []),
    "pagani_integrate": (C.c_int, [C.POINTER(Integrand), C.c_int, _D, _D, C.POINTER(Config),
                                   C.POINTER(Result)]),
    "pagani_integrate_sequential": (C.c_int, [C.POINTER(Integrand), C.c_int, _D, _D, C.c_double,
                                              C.c_double, C.c_int64, C.c_int32, C.c_int32,
                                              C.c_int32, C.POINTER(Result)]),
    "pagani_rule_point_count": (C.c_int64, [C.c_int]),
    "pagani_build_rule": (C.c_int, [C.c_int, _D, _D, _D, _D]),
    "pagani_evaluate_batch": (C.c_int, [C.POINTER(Integrand), C.c_int, C.c_int64, _D, _D, _D,
                                        _D, _I32, _I64, C.c_int32]),
    "pagani_two_level_refine": (C.c_int, [C.c_int64, _D, _D, _D, _D, _D]),
    "pagani_rel_err_classify": (C.c_int, [C.c_int64, _D, _D, C.c_double, C.c_int32, _U8]),
    "pagani_apply_threshold": (C.c_int, [C.c_int64, _D, C.c_double, _U8]),
    "pagani_threshold_classify": (C.c_int, [C.c_int64, _U8, _D, C.c_double, C.c_double,
                                            C.c_double, C.c_int64, C.c_double,
                                            C.POINTER(Config), _U8,
                                            C.POINTER(ThresholdResult)]),
    "pagani_filter": (C.c_int, [C.c_int, C.c_int64, _D, _D, _D, _D, _I32, _D, _D, _U8, _D, _D,
                                _D, _D, _I32, _D, _D, _I64, _D, _D, _D]),
    "pagani_bisect": (C.c_int, [C.c_int, C.c_int64, _D, _D, _D, _D, _I32, C.c_int64, _D, _D,
                                _D, _D]),
    "pagani_uniform_split": (C.c_int, [C.c_int, _D, _D, C.c_int, C.c_int64, _I64, _D, _D,
                                       C.c_int64]),
    "pagani_initial_subdivisions": (C.c_int, [C.c_int, C.c_int64]),
    "pagani_block_sum": (C.c_int, [C.c_int64, _D, _D]),
    "pagani_block_sum_where": (C.c_int, [C.c_int64, _D, _U8, C.c_int32, _D]),
    "pagani_count_flags": (C.c_int, [C.c_int64, _U8, C.c_int32, _I64]),
    "pagani_min_max": (C.c_int, [C.c_int64, _D, _D, _D]),
    "pagani_check_termination": (C.c_int, [C.c_double] * 6),
    "pagani_digits_converged": (C.c_int, [C.c_double, C.c_double, C.c_int]),
    "pagani_convergence_digits": (C.c_int, [C.c_double]),
    "pagani_reference_value": (C.c_int, [C.c_char_p, C.c_int, C.c_int32,
                                         C.POINTER(C.c_double)]),
    "pagani_math_exp": (C.c_int, [C.c_int64, _D, _D, C.c_int32]),
    "pagani_math_cos": (C.c_int, [C.c_int64, _D, _D, C.c_int32]),
    "pagani_call_integrand": (C.c_int, [C.POINTER(Integrand), C.c_int, C.c_int64, _D, _D]),
    "pagani_fp64_peak": (C.c_int, [C.c_int, C.c_double, _D, _D]),
    "pagani_comm_unique_id": (C.c_int, [_U8]),
    "pagani_comm_init_rank": (C.c_int, [_U8, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(C.c_void_p)]),
    "pagani_comm_init_host": (C.c_int, [C.POINTER(HostTransport), C.c_int,
                                        C.POINTER(C.c_void_p)]),
    "pagani_comm_destroy": (C.c_int, [C.c_void_p]),
    "pagani_shard_bounds": (C.c_int, [C.c_int64, C.c_int, _I64]),
    "pagani_shard_plan": (C.c_int, [C.c_int, C.c_int, _I64, C.c_int, C.POINTER(C.c_int32), _I64,
                                    C.POINTER(C.c_int32), _I64]),
}

_lib = None


class PaganiError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class CudaUnavailable(PaganiError):
    pass


def load(path: str = LIB_PATH):
    """Load libpagani_b200.so (raises if it is not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (make -C paper_2104_06494_b200/csrc). There is no CPU fallback.")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int):
    if rc == PAGANI_OK:
        return rc
    msg = load().pagani_last_error().decode(errors="replace")
    if rc == PAGANI_E_INVALID:
        raise ValueError(msg)
    if rc == PAGANI_E_LOGIC:
        raise AssertionError(msg)
    if rc == PAGANI_E_CUDA:
        raise CudaUnavailable(rc, msg)
    if rc == PAGANI_E_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise PaganiError(rc, msg)
