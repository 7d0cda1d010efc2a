"""ctypes binding of the C-ABI in include/edaa_b200.h (libedaa_cuda.so).

There is no CPU fallback: if the library is missing or no CUDA device is
present, loading fails loudly with EdaaError.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
CUDA_LIB = os.path.join(PKG, "libedaa_cuda.so")

EDAA_OK, EDAA_ERR_INVALID, EDAA_ERR_CUDA, EDAA_ERR_UNSUPPORTED, EDAA_ERR_STATE, \
    EDAA_ERR_ALL_FAILED = range(6)


class EdaaError(RuntimeError):
    """Error raised by the C-ABI (the reference's archetype::Error text where one applies)."""

    def __init__(self, msg, code=None):
        super().__init__(msg)
        self.code = code


class SolveParams(C.Structure):
    _fields_ = [("endmembers", C.c_size_t), ("outer_iters", C.c_size_t),
                ("inner_iters_a", C.c_size_t), ("inner_iters_b", C.c_size_t),
                ("runs", C.c_size_t), ("seeds", C.POINTER(C.c_uint64)),
                ("gammas", C.POINTER(C.c_double))]


class RunRecordC(C.Structure):
    _fields_ = [("fit_l1", C.c_double), ("coherence", C.c_double), ("eta_a", C.c_double),
                ("eta_b", C.c_double), ("ok", C.c_int), ("fail_code", C.c_int),
                ("fail_outer", C.c_size_t), ("message", C.c_char * 192)]


class ProfileC(C.Structure):
    _fields_ = [("ms", C.c_double * 5), ("launches", C.c_uint64 * 5)]


OBSERVER_FN = C.CFUNCTYPE(None, C.c_size_t, C.c_char, C.c_size_t, C.POINTER(C.c_double),
                          C.POINTER(C.c_double), C.c_size_t, C.c_size_t, C.c_void_p)

# (name, restype, argtypes) for every symbol include/edaa_b200.h declares.
SIGNATURES = [
    ("edaa_create", C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    ("edaa_destroy", C.c_int, [C.c_void_p]),
    ("edaa_last_error", C.c_char_p, [C.c_void_p]),
    ("edaa_stream", C.c_void_p, [C.c_void_p]),
    ("edaa_set_image_host", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t]),
    ("edaa_set_image_host_f64", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t]),
    ("edaa_set_image_host_checked", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t]),
    ("edaa_set_image_device", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t,
                                        C.c_size_t]),
    ("edaa_ingest_host", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_void_p,
                                   C.c_size_t, C.POINTER(C.c_size_t)]),
    ("edaa_ingest_host_f32", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_int,
                                       C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("edaa_image_get", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int)]),
    ("edaa_solve_async", C.c_int, [C.c_void_p, C.POINTER(SolveParams)]),
    ("edaa_finish", C.c_int, [C.c_void_p]),
    ("edaa_solve", C.c_int, [C.c_void_p, C.POINTER(SolveParams)]),
    ("edaa_run_record_get", C.c_int, [C.c_void_p, C.c_size_t, C.POINTER(RunRecordC)]),
    ("edaa_traces", C.c_int, [C.c_void_p, C.c_void_p]),
    ("edaa_factors", C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("edaa_select", C.c_int, [C.c_void_p, C.c_double, C.c_void_p, C.POINTER(C.c_size_t),
                              C.POINTER(C.c_double)]),
    ("edaa_solve_observed", C.c_int, [C.c_void_p, C.POINTER(SolveParams), OBSERVER_FN,
                                      C.c_void_p]),
    ("edaa_xb", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    ("edaa_objective", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    ("edaa_grad_abundances", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    ("edaa_grad_contributions", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                          C.c_void_p]),
    ("edaa_fit_l1", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    ("edaa_estimate_abundances", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t,
                                           C.c_double, C.c_void_p]),
    ("edaa_check_iterate", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t,
                                     C.c_int, C.POINTER(C.c_int), C.c_char_p, C.c_size_t]),
    ("edaa_profile_enable", C.c_int, [C.c_void_p, C.c_int]),
    ("edaa_profile_read", C.c_int, [C.c_void_p, C.POINTER(ProfileC)]),
    ("edaa_launch_count", C.c_uint64, [C.c_void_p]),
    ("edaa_probe_fp64_peak", C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    ("edaa_nccl_unique_id", C.c_int, [C.c_void_p, C.c_size_t]),
    ("edaa_set_pixel_shard", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int]),
    ("edaa_shard_pixels", C.c_int, [C.c_void_p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    ("edaa_set_shard_emulation", C.c_int, [C.c_void_p, C.c_int]),
    ("edaa_set_shard_exchange", C.c_int, [C.c_void_p, C.c_int]),
    ("edaa_set_pass_order", C.c_int, [C.c_void_p, C.c_int]),
    ("edaa_version", C.c_char_p, []),
    ("edaa_max_endmembers", C.c_size_t, []),
    ("edaa_max_bands", C.c_size_t, []),
]

_LIB = None


def load(path: str = CUDA_LIB):
    """Load libedaa_cuda.so (once). Raises EdaaError if it is not built.
    EDAA_CUDA_LIB (development) names an alternative in-tree build of the same ABI."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.environ.get("EDAA_CUDA_LIB", path)
    if not os.path.exists(path):
        raise EdaaError("libedaa_cuda.so is not built (run __graft_entry__.build()); "
                        "there is no CPU fallback")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _LIB = lib
    return lib
