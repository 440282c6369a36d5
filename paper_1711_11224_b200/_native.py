"""ctypes binding of the C-ABI in include/ndconv_b200.h (libndconv_b200.so).

The library is built in-tree by ``paper_1711_11224_b200.build``; importing this module
never compiles and never falls back to anything else -- a missing library is an error.
"""
from __future__ import annotations

import ctypes as C
import os

# NDC_LIB_PATH overrides the in-tree library (kernel-variant experiments in tools/).
LIB_PATH = os.environ.get("NDC_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                           "libndconv_b200.so")

size_t_p = C.POINTER(C.c_size_t)
dbl_p = C.POINTER(C.c_double)
flt_p = C.POINTER(C.c_float)


class DeconvConfig(C.Structure):
    """ndc_deconv_config == ndconv::DeconvConfig (solvers.hpp:20-28)."""
    _fields_ = [
        ("max_iters", C.c_size_t),
        ("tol_rel_objective", C.c_double),
        ("has_initial_step", C.c_int),
        ("initial_step", C.c_double),
        ("backtrack_factor", C.c_double),
        ("max_backtracks", C.c_size_t),
        ("power_iters", C.c_size_t),
    ]


class RlConfig(C.Structure):
    """ndc_rl_config == ndconv::RlConfig (solvers.hpp:30-35)."""
    _fields_ = [("max_iters", C.c_size_t), ("tol_rel_change", C.c_double)]


class Report(C.Structure):
    """ndc_deconv_report (solvers.hpp:48-61 minus the tensors)."""
    _fields_ = [
        ("iterations_run", C.c_size_t),
        ("stop_reason", C.c_int),
        ("wall_time_seconds", C.c_double),
        ("negative_pixels_clamped", C.c_size_t),
        ("trace_len", C.c_size_t),
        ("backtracks", C.c_size_t),
        ("step0", C.c_double),
    ]


# (name, restype, argtypes)
_SIGS = [
    ("ndc_last_error", C.c_char_p, []),
    ("ndc_version", C.c_char_p, []),
    ("ndc_stop_reason_name", C.c_char_p, [C.c_int]),
    ("ndc_deconv_config_default", None, [C.POINTER(DeconvConfig)]),
    ("ndc_rl_config_default", None, [C.POINTER(RlConfig)]),
    ("ndc_device_count", C.c_int, [C.POINTER(C.c_int)]),
    ("ndc_set_device", C.c_int, [C.c_int]),
    ("ndc_set_max_threads", None, [C.c_uint]),
    ("ndc_max_threads", C.c_uint, []),
    ("ndc_conv_output_shape", C.c_int, [C.c_int, size_t_p, size_t_p, size_t_p]),
    ("ndc_conv_full_f64", C.c_int, [C.c_int, size_t_p, dbl_p, size_t_p, dbl_p, dbl_p]),
    ("ndc_adjoint_apply_f64", C.c_int, [C.c_int, size_t_p, dbl_p, size_t_p, dbl_p, size_t_p, dbl_p]),
    ("ndc_normal_gradient_f64", C.c_int, [C.c_int, size_t_p, dbl_p, dbl_p, size_t_p, dbl_p, dbl_p]),
    ("ndc_objective_f64", C.c_int, [C.c_int, size_t_p, dbl_p, dbl_p, size_t_p, dbl_p, dbl_p]),
    ("ndc_estimate_step_f64", C.c_int, [C.c_int, size_t_p, dbl_p, size_t_p, C.c_size_t, dbl_p]),
    ("ndc_kkt_residual_f64", C.c_int, [C.c_int, size_t_p, dbl_p, dbl_p, size_t_p, dbl_p, dbl_p]),
    ("ndc_deconv_pg_f64", C.c_int, [C.c_int, size_t_p, dbl_p, size_t_p, dbl_p, size_t_p,
                                    C.POINTER(DeconvConfig), dbl_p, dbl_p, dbl_p, C.c_size_t,
                                    C.POINTER(Report)]),
    ("ndc_deconv_pg_batch_f64", C.c_int, [C.c_size_t, C.c_int, size_t_p, dbl_p, size_t_p, dbl_p,
                                          size_t_p, C.POINTER(DeconvConfig), dbl_p, dbl_p, dbl_p,
                                          C.c_size_t, C.POINTER(Report)]),
    ("ndc_deconv_pg_batch_f32", C.c_int, [C.c_size_t, C.c_int, size_t_p, flt_p, size_t_p, dbl_p,
                                          size_t_p, C.POINTER(DeconvConfig), flt_p, dbl_p, dbl_p,
                                          C.c_size_t, C.POINTER(Report)]),
    ("ndc_deconv_rl_f64", C.c_int, [C.c_int, size_t_p, dbl_p, size_t_p, dbl_p, size_t_p,
                                    C.POINTER(RlConfig), dbl_p, dbl_p, dbl_p, C.c_size_t,
                                    C.POINTER(Report)]),
    ("ndc_plan_create", C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_size_t, C.c_int, size_t_p,
                                  size_t_p, dbl_p]),
    ("ndc_plan_destroy", C.c_int, [C.c_void_p]),
    ("ndc_plan_set_observation_f64", C.c_int, [C.c_void_p, dbl_p]),
    ("ndc_plan_set_observation_f32", C.c_int, [C.c_void_p, flt_p]),
    ("ndc_plan_pg_begin", C.c_int, [C.c_void_p, C.POINTER(DeconvConfig)]),
    ("ndc_plan_pg_iterate", C.c_int, [C.c_void_p, C.c_size_t, size_t_p]),
    ("ndc_plan_pg_end", C.c_int, [C.c_void_p]),
    ("ndc_plan_pg_run", C.c_int, [C.c_void_p, C.POINTER(DeconvConfig)]),
    ("ndc_plan_rl_run", C.c_int, [C.c_void_p, C.POINTER(RlConfig)]),
    ("ndc_probe_fp32_peak", C.c_int, [C.c_int, C.POINTER(C.c_double)]),
    ("ndc_plan_check_guards", C.c_int, [C.c_void_p, C.POINTER(C.c_size_t)]),
    ("ndc_debug_guard_violations", C.c_int, [C.POINTER(C.c_ulonglong)]),
    ("ndc_plan_debug_corrupt_guard", C.c_int, [C.c_void_p]),
    ("ndc_plan_get_report", C.c_int, [C.c_void_p, C.c_size_t, C.POINTER(Report), dbl_p, dbl_p,
                                      C.c_size_t]),
    ("ndc_plan_get_estimate_f64", C.c_int, [C.c_void_p, dbl_p]),
    ("ndc_plan_get_estimate_f32", C.c_int, [C.c_void_p, flt_p]),
    ("ndc_plan_load_observation_ndtensor", C.c_int, [C.c_void_p, C.c_char_p]),
    ("ndc_plan_save_estimate_ndtensor", C.c_int, [C.c_void_p, C.c_char_p]),
    ("ndc_ndtensor_info", C.c_int, [C.c_char_p, C.POINTER(C.c_int), size_t_p]),
    ("ndc_ndtensor_read_f64", C.c_int, [C.c_char_p, dbl_p, C.c_size_t]),
    ("ndc_ndtensor_write_f64", C.c_int, [C.c_char_p, C.c_int, size_t_p, dbl_p]),
    ("ndc_pgm_info", C.c_int, [C.c_char_p, size_t_p, size_t_p]),
    ("ndc_pgm_read_f64", C.c_int, [C.c_char_p, dbl_p, C.c_size_t]),
    ("ndc_conv_full_batch_f32", C.c_int, [C.c_size_t, C.c_int, size_t_p, flt_p, size_t_p, dbl_p, flt_p]),
    ("ndc_adjoint_apply_batch_f32", C.c_int, [C.c_size_t, C.c_int, size_t_p, flt_p, size_t_p, dbl_p, size_t_p,
                                              flt_p]),
    ("ndc_pgm_write_f64", C.c_int, [C.c_char_p, C.c_size_t, C.c_size_t, dbl_p, C.c_int]),
    ("ndc_plan_get_observation_f64", C.c_int, [C.c_void_p, dbl_p]),
    ("ndc_plan_add_gaussian_noise", C.c_int, [C.c_void_p, C.c_double, C.c_double, C.c_uint64]),
    ("ndc_sim_phantom_lines_f64", C.c_int, [C.c_size_t, C.c_size_t, C.c_size_t, C.c_double, dbl_p]),
    ("ndc_sim_phantom_texture_f64", C.c_int, [C.c_size_t, C.c_size_t, dbl_p]),
    ("ndc_sim_gaussian_psf_f64", C.c_int, [C.c_int, size_t_p, C.c_double, dbl_p]),
    ("ndc_sim_delta_psf_f64", C.c_int, [C.c_int, size_t_p, dbl_p]),
    ("ndc_sim_add_gaussian_noise_f64", C.c_int, [C.c_size_t, dbl_p, C.c_double, C.c_double, C.c_uint64, dbl_p]),
    ("ndc_sim_mt19937_64", C.c_int, [C.c_uint64, C.c_size_t, C.c_size_t, C.POINTER(C.c_uint64)]),
    ("ndc_plan_forward", C.c_int, [C.c_void_p]),
    ("ndc_plan_adjoint", C.c_int, [C.c_void_p]),
    ("ndc_plan_set_timing", C.c_int, [C.c_void_p, C.c_int]),
    ("ndc_plan_reset_stats", C.c_int, [C.c_void_p]),
    ("ndc_plan_stats", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_uint64), dbl_p]),
    ("ndc_plan_stream", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    ("ndc_slab_range", C.c_int, [C.c_size_t, C.c_size_t, C.c_int, C.c_int, size_t_p, size_t_p,
                                 size_t_p, size_t_p]),
    ("ndc_nccl_unique_id", C.c_int, [C.c_char_p]),
    ("ndc_plan_create_sharded", C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int, size_t_p, size_t_p,
                                          dbl_p, C.c_int, C.c_int, C.c_char_p]),
    ("ndc_local_group_create", C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    ("ndc_local_group_destroy", C.c_int, [C.c_void_p]),
    ("ndc_plan_create_local", C.c_int, [C.POINTER(C.c_void_p), C.c_void_p, C.c_int, C.c_int, C.c_int,
                                        size_t_p, size_t_p, dbl_p]),
]

EXPORTED = [s[0] for s in _SIGS]

_lib = None


def lib() -> C.CDLL:
    """Load libndconv_b200.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1711_11224_b200.build` "
                "(the ndconv B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in _SIGS:
            if os.environ.get("NDC_LIB_PATH") and not hasattr(L, name):
                continue  # an older library variant (A/B timing) may lack newer entry points
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
