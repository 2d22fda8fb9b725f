"""ctypes binding of libasyncdiff_b200.so (include/asyncdiff_b200.h).

The shared library is built in-tree by __graft_entry__.build() /
paper_2406_06911_b200/csrc/Makefile.  There is no fallback: if the library is
missing, importing the product path raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libasyncdiff_b200.so")
if os.environ.get("ADX_LIB_VARIANT"):  # A/B tooling only: tools/ builds variant libraries beside the product one
    SO_PATH = os.path.join(_HERE, "libasyncdiff_b200." + os.environ["ADX_LIB_VARIANT"] + ".so")


class AdxError(Exception):
    """Base class; subclasses mirror the reference's std:: exception classes."""


class InvalidArgument(AdxError, ValueError):
    """std::invalid_argument"""


class OutOfRange(AdxError, IndexError):
    """std::out_of_range"""


class DomainError(AdxError, ArithmeticError):
    """std::domain_error"""


class AdxRuntimeError(AdxError, RuntimeError):
    """std::runtime_error"""


class LogicError(AdxError, RuntimeError):
    """std::logic_error"""


class CudaError(AdxRuntimeError):
    """CUDA / NCCL failure"""


_STATUS = {1: InvalidArgument, 2: OutOfRange, 3: DomainError, 4: AdxRuntimeError, 5: LogicError, 6: CudaError}


class adx_run_options(C.Structure):
    _fields_ = [
        ("round_timeout_s", C.c_double),
        ("jitter_seed", C.c_uint64),
        ("max_jitter_s", C.c_double),
        ("segment_delay_s", C.POINTER(C.c_double)),
        ("n_delays", C.c_int),
        ("use_graph", C.c_int),
        ("instrument", C.c_int),
    ]


class adx_run_stats(C.Structure):
    _fields_ = [
        ("broadcast_count", C.c_int),
        ("n_rounds", C.c_int),
        ("warmup_wall_s", C.c_double),
        ("total_wall_s", C.c_double),
        ("round_wall_s", C.POINTER(C.c_double)),
        ("round_comm_s", C.POINTER(C.c_double)),
        ("device_busy_s", C.POINTER(C.c_double)),
        ("device_evals", C.POINTER(C.c_longlong)),
        ("store_entries_per_round", C.POINTER(C.c_int)),
    ]


class adx_plan_counts_t(C.Structure):
    _fields_ = [
        ("broadcasts_paper_convention", C.c_int),
        ("broadcasts_strictly_needed", C.c_int),
        ("device_count", C.c_int),
        ("max_device_macs", C.c_longlong),
        ("sequential_total_macs", C.c_longlong),
    ]


# every symbol the header declares (checked by tests/test_capi_symbols.py)
EXPORTS = [
    "adx_last_error", "adx_version", "adx_device_count", "adx_random_normals", "adx_build_schedule", "adx_ddim_step",
    "adx_model_build_toy", "adx_model_shell", "adx_model_destroy", "adx_model_info", "adx_model_widths",
    "adx_model_links", "adx_model_stage_shape", "adx_model_set_stage_macs", "adx_model_tensor", "adx_sinusoid",
    "adx_partition_balanced", "adx_partition_create", "adx_partition_destroy", "adx_partition_num_segments",
    "adx_partition_strategy", "adx_partition_segment", "adx_partition_contiguous",
    "adx_partition_segment_of_stage", "adx_partition_validate", "adx_crossing_links",
    "adx_plan_async", "adx_plan_from_flat", "adx_plan_to_flat", "adx_plan_destroy", "adx_plan_validate",
    "adx_plan_counts", "adx_shift_embeddings", "adx_render_plan",
    "adx_engine_create", "adx_engine_destroy", "adx_engine_weight_bytes", "adx_engine_time_eval", "adx_bench_gemv", "adx_eval_full", "adx_eval_segment",
    "adx_run_options_default", "adx_session_create", "adx_session_destroy", "adx_session_run",
    "adx_session_upload", "adx_session_time", "adx_session_kernel_count", "adx_session_weight_bytes",
    "adx_session_download", "adx_run_serial", "adx_run_parallel", "adx_sequential_denoise",
    "adx_compare_trajectories", "adx_rank_program", "adx_nccl_unique_id", "adx_rank_session_create",
    "adx_rank_session_destroy", "adx_rank_session_run", "adx_rank_session_time", "adx_rank_session_kernel_count",
    "adx_model_save_checkpoint", "adx_model_load_checkpoint", "adx_plan_to_json", "adx_plan_from_json",
    "adx_predict_async", "adx_calibrate_and_compare", "adx_round_exchange_bytes", "adx_tc_gemm", "adx_tc_conv3x3",
    "adx_model_build_unet", "adx_unet_stage_info", "adx_unet_stage_params", "adx_unet_context", "adx_tc_attention", "adx_tc_attention_f32", "adx_tc_ln_fold_bf16", "adx_tc_ln_fold_supported", "adx_tc_geglu_group", "adx_sk_timeline", "adx_tc_gemm_cat_bf16", "adx_tc_conv3x3_s2_bf16", "adx_temporal_attention",
    "adx_engine_profile_pass", "adx_profile_records", "adx_tc_plan_override", "adx_engine_stage_times", "adx_partition_by_cost",
    "adx_tc_timeline", "adx_tc_gemm_bf16", "adx_tc_conv3x3_bf16", "adx_group_norm_bf16", "adx_gn_timeline",
]


class adx_unet_spec(C.Structure):
    _fields_ = [("H", C.c_int), ("W", C.c_int), ("c_lat", C.c_int), ("n_levels", C.c_int), ("ch", C.c_int * 8),
                ("attn", C.c_int * 8), ("n_res", C.c_int), ("head_dim", C.c_int), ("ctx_len", C.c_int),
                ("ctx_dim", C.c_int), ("temb_dim", C.c_int), ("groups", C.c_int), ("mid_attn", C.c_int),
                ("seed", C.c_uint64), ("cfg", C.c_int), ("cfg_scale", C.c_float), ("frames", C.c_int),
                ("motion", C.c_int)]


class adx_latency_report(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("sequential_total_s", "async_total_s", "warmup_s", "comm_total_s",
                                           "speedup", "comm_ratio", "approx_step_s", "approx_total_s")]


class adx_cost_comparison(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("predicted_total_s", "measured_total_s", "rel_error_total",
                                           "predicted_comm_ratio", "measured_comm_ratio", "rel_error_comm_ratio",
                                           "calibrated_comm_cost_s")]

_lib = None


def lib():
    """Load the C-ABI library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise ImportError(
            f"{SO_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the product path)")
    L = C.CDLL(SO_PATH)
    i, d, ll, u64, vp = C.c_int, C.c_double, C.c_longlong, C.c_uint64, C.c_void_p
    P = C.POINTER
    sig = {
        "adx_last_error": (C.c_char_p, []),
        "adx_version": (i, []),
        "adx_device_count": (i, []),
        "adx_random_normals": (i, [u64, ll, P(d)]),
        "adx_build_schedule": (i, [i, d, d, i, P(d), P(d), P(d)]),
        "adx_ddim_step": (i, [i, i, P(d), P(d), i, i, P(d), i, P(d)]),
        "adx_model_build_toy": (i, [i, P(i), i, i, u64, i, P(vp)]),
        "adx_model_shell": (i, [i, P(i), i, P(i), i, i, P(vp)]),
        "adx_model_destroy": (None, [vp]),
        "adx_model_info": (i, [vp, P(i), P(i), P(i)]),
        "adx_model_widths": (i, [vp, P(i)]),
        "adx_model_links": (i, [vp, P(i)]),
        "adx_model_stage_shape": (i, [vp, i, P(i), P(i), P(i), P(ll)]),
        "adx_model_set_stage_macs": (i, [vp, i, ll]),
        "adx_model_tensor": (i, [vp, i, i, P(P(d)), P(i), P(i)]),
        "adx_sinusoid": (i, [i, i, P(d)]),
        "adx_partition_balanced": (i, [vp, i, i, P(vp)]),
        "adx_partition_create": (i, [i, P(i), P(i), P(i), P(ll), i, P(vp)]),
        "adx_partition_destroy": (None, [vp]),
        "adx_partition_num_segments": (i, [vp]),
        "adx_partition_strategy": (i, [vp]),
        "adx_partition_segment": (i, [vp, i, P(i), i, P(i), P(ll), P(i)]),
        "adx_partition_contiguous": (i, [vp]),
        "adx_partition_segment_of_stage": (i, [vp, i, P(i)]),
        "adx_partition_validate": (i, [vp, vp]),
        "adx_crossing_links": (i, [vp, vp, P(i), i, P(i)]),
        "adx_plan_async": (i, [i, i, i, i, i, P(vp)]),
        "adx_plan_from_flat": (i, [P(i), i, P(vp)]),
        "adx_plan_to_flat": (i, [vp, P(i), i, P(i)]),
        "adx_plan_destroy": (None, [vp]),
        "adx_plan_validate": (i, [vp, C.c_char_p, i, P(i)]),
        "adx_plan_counts": (i, [vp, vp, P(adx_plan_counts_t), P(ll), P(ll)]),
        "adx_shift_embeddings": (i, [P(i), i, i, P(i)]),
        "adx_render_plan": (i, [vp, C.c_char_p, i, P(i)]),
        "adx_engine_create": (i, [vp, i, P(i), i, P(vp)]),
        "adx_engine_destroy": (None, [vp]),
        "adx_engine_weight_bytes": (i, [vp, i, P(ll)]),
        "adx_engine_time_eval": (i, [vp, i, i, P(d), P(ll), P(i)]),
        "adx_bench_gemv": (i, [i, i, i, i, i, i, P(d)]),
        "adx_engine_profile_pass": (i, [vp, i, P(d)]),
        "adx_profile_records": (i, [P(d), i, P(i)]),
        "adx_eval_full": (i, [vp, P(d), i, P(d)]),
        "adx_eval_segment": (i, [vp, vp, i, P(d), i, i, i, P(i), P(d), i, i, P(d), i, P(i), P(i), P(i),
                                 P(d), i, i, P(i)]),
        "adx_run_options_default": (None, [P(adx_run_options)]),
        "adx_session_create": (i, [vp, vp, vp, P(d), i, i, i, P(adx_run_options), P(vp)]),
        "adx_session_destroy": (None, [vp]),
        "adx_session_run": (i, [vp, P(d), P(d), P(d), P(adx_run_stats)]),
        "adx_session_upload": (i, [vp, P(d)]),
        "adx_session_time": (i, [vp, i, P(d)]),
        "adx_session_kernel_count": (i, [vp, P(i)]),
        "adx_session_weight_bytes": (i, [vp, P(ll)]),
        "adx_session_download": (i, [vp, P(d), P(d)]),
        "adx_run_serial": (i, [vp, vp, vp, P(d), P(d), i, P(adx_run_options), P(d), P(d), P(adx_run_stats)]),
        "adx_run_parallel": (i, [vp, vp, vp, P(d), P(d), i, i, P(adx_run_options), P(d), P(d),
                                 P(adx_run_stats)]),
        "adx_sequential_denoise": (i, [vp, P(d), P(d), i, P(d), P(d)]),
        "adx_compare_trajectories": (i, [P(d), P(d), i, i, P(d), P(d), P(d)]),
        "adx_rank_program": (i, [vp, vp, vp, i, P(i), i, P(i)]),
        "adx_nccl_unique_id": (i, [C.c_char_p]),
        "adx_rank_session_create": (i, [vp, vp, vp, P(d), i, i, C.c_char_p, P(adx_run_options), P(vp)]),
        "adx_rank_session_destroy": (None, [vp]),
        "adx_rank_session_run": (i, [vp, P(d), P(d), P(d)]),
        "adx_rank_session_time": (i, [vp, i, P(d)]),
        "adx_rank_session_kernel_count": (i, [vp, P(i)]),
        "adx_model_save_checkpoint": (i, [vp, C.c_char_p]),
        "adx_model_load_checkpoint": (i, [C.c_char_p, P(vp)]),
        "adx_plan_to_json": (i, [vp, C.c_char_p, i, P(i)]),
        "adx_plan_from_json": (i, [C.c_char_p, P(vp)]),
        "adx_predict_async": (i, [vp, P(d), i, d, d, d, d, P(ll), P(adx_latency_report), P(d), P(d)]),
        "adx_calibrate_and_compare": (i, [vp, P(d), i, P(d), i, i, d, P(adx_cost_comparison)]),
        "adx_round_exchange_bytes": (i, [vp, vp, vp, i, P(ll)]),
        "adx_model_build_unet": (i, [P(adx_unet_spec), P(vp)]),
        "adx_unet_stage_info": (i, [vp, i, P(i)]),
        "adx_unet_stage_params": (i, [vp, i, C.c_char_p, i, P(i), P(i), P(C.c_float), ll, P(ll)]),
        "adx_unet_context": (i, [vp, P(C.c_float)]),
        "adx_tc_gemm": (i, [i, i, i, i, P(C.c_uint16), P(C.c_uint16), P(C.c_float), i, P(C.c_float), i, i, P(d)]),
        "adx_tc_attention": (i, [i, i, i, i, P(C.c_uint16), P(C.c_uint16), P(C.c_uint16), i, P(C.c_uint16), i,
                                 P(d)]),
        "adx_tc_conv3x3_s2_bf16": (i, [i, i, i, i, i, i, P(C.c_uint16), P(C.c_uint16), P(C.c_float), P(C.c_uint16),
                                       i, i, i, P(d)]),
        "adx_tc_ln_fold_supported": (i, []),
        "adx_tc_geglu_group": (i, []),
        "adx_sk_timeline": (i, [P(C.c_ulonglong), i]),
        "adx_tc_gemm_cat_bf16": (i, [i, i, i, i, i, P(C.c_uint16), P(C.c_uint16), P(C.c_uint16), P(C.c_float),
                                     P(C.c_uint16), i, i]),
        "adx_tc_ln_fold_bf16": (i, [i, i, i, i, P(C.c_uint16), P(C.c_uint16), P(C.c_float), P(C.c_float), i,
                                    C.c_float, P(C.c_uint16), i, i, P(d)]),
        "adx_tc_attention_f32": (i, [i, i, i, i, i, P(C.c_float), P(C.c_float), P(C.c_float), P(C.c_float), i,
                                     P(d)]),
        "adx_temporal_attention": (i, [i, i, i, i, P(C.c_uint16), P(C.c_uint16), i, P(d)]),
        "adx_tc_conv3x3": (i, [i, i, i, i, i, i, P(C.c_uint16), P(C.c_uint16), P(C.c_float), P(C.c_float), i,
                               P(d)]),
        "adx_tc_plan_override": (i, [i, i]),
        "adx_tc_timeline": (i, [P(C.c_ulonglong), i]),
        "adx_gn_timeline": (i, [P(C.c_ulonglong), i]),
        "adx_group_norm_bf16": (i, [i, i, i, i, i, i, P(C.c_uint16), P(C.c_uint16), P(C.c_float), P(C.c_float),
                                    C.c_float, i, P(C.c_uint16), i, P(d)]),
        "adx_tc_gemm_bf16": (i, [i, i, i, i, P(C.c_uint16), P(C.c_uint16), P(C.c_float), P(C.c_uint16), i,
                                 P(C.c_uint16), i, i, i, i, P(d)]),
        "adx_tc_conv3x3_bf16": (i, [i, i, i, i, i, i, P(C.c_uint16), P(C.c_uint16), P(C.c_float), P(C.c_uint16),
                                    P(C.c_uint16), i, i, i, P(d)]),
        "adx_engine_stage_times": (i, [vp, i, i, P(d)]),
        "adx_partition_by_cost": (i, [vp, i, P(d), P(vp)]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("ADX_LIB_VARIANT") and not hasattr(L, name):
            continue  # A/B tooling: an older variant build may predate this entry point
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().adx_last_error().decode()
        raise _STATUS.get(rc, AdxRuntimeError)(msg)
