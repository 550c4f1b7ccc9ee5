"""ctypes description of the primkit C ABI (include/primkit/primkit.h).

Section 1 of the header is byte-compatible with the reference ABI
(/root/reference/proj/include/primkit/primkit.h), so the same description
binds both this library and the reference build used as the parity oracle.
"""
from __future__ import annotations

import ctypes as C

STATUS = {
    0: "OK", 1: "SHAPE_MISMATCH", 2: "INVALID_SHAPE", 3: "GROUP_MISMATCH",
    4: "ALGO_NOT_APPLICABLE", 5: "WORKSPACE_TOO_SMALL", 6: "DUPLICATE_SOLVER",
    7: "NO_APPLICABLE_SOLVER", 8: "NOT_TUNABLE", 9: "NO_VALID_CONFIG", 10: "IO_ERROR",
    11: "PARSE_ERROR", 12: "LAYOUT_NOT_DESCENDING", 13: "INVALID_EPSILON",
    14: "INVALID_AXIS", 15: "FUSION_NOT_SUPPORTED", 16: "ALREADY_COMPILED",
    17: "NOT_COMPILED", 18: "MISSING_ARGS", 19: "INVALID_VALUE", 20: "INTERNAL",
}
STATUS_CODE = {v: k for k, v in STATUS.items()}

F32, BF16 = 0, 1
CONVOLUTION, TRANSPOSE = 0, 1
FORWARD, BACKWARD_DATA, BACKWARD_WEIGHTS = 0, 1, 2
ALGO = {"Im2colGemm": 0, "Direct": 1, "Winograd": 2, "FFT": 3, "ImplicitGemm": 4}
RELU, LEAKY_RELU, SIGMOID, TANH = 0, 1, 2, 3
BN_PER_ACTIVATION, BN_SPATIAL = 0, 1


class ConvProblem(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "n", "c", "h", "w", "k", "y", "x", "pad_h", "pad_w", "stride_h", "stride_w",
        "dilation_h", "dilation_w", "groups")] + [
        ("direction", C.c_int), ("mode", C.c_int), ("etype", C.c_int)]


class AlgoPerf(C.Structure):
    _fields_ = [("solver_name", C.c_char * 64), ("algo", C.c_int), ("time_ms", C.c_double),
                ("workspace_bytes", C.c_uint64)]


class Counters(C.Structure):
    _fields_ = [("gemm_calls", C.c_uint64), ("scalar_muls", C.c_uint64),
                ("buffer_roundtrips", C.c_uint64)]


P = C.c_void_p
FP = C.POINTER(C.c_float)
I64P = C.POINTER(C.c_int64)
ST = C.c_int

# name -> (restype, argtypes); section 1 (reference ABI, 31 functions)
SECTION1 = {
    "primkit_last_error": (C.c_char_p, []),
    "primkit_handle_create": (ST, [C.POINTER(P)]),
    "primkit_handle_destroy": (None, [P]),
    "primkit_handle_use_fake_clock": (ST, [P]),
    "primkit_handle_now_ms": (ST, [P, C.POINTER(C.c_double)]),
    "primkit_handle_set_cache_dir": (ST, [P, C.c_char_p]),
    "primkit_handle_counters": (ST, [P, C.POINTER(Counters)]),
    "primkit_handle_reset_counters": (ST, [P]),
    "primkit_handle_set_seed": (ST, [P, C.c_uint64]),
    "primkit_problem_key": (ST, [C.POINTER(ConvProblem), C.c_char_p, C.c_size_t]),
    "primkit_conv_output_dims": (ST, [C.POINTER(ConvProblem), I64P]),
    "primkit_solver_count": (ST, [P, C.POINTER(C.c_int)]),
    "primkit_solver_name": (ST, [P, C.c_int, C.c_char_p, C.c_size_t]),
    "primkit_solver_is_applicable": (ST, [P, C.c_char_p, C.POINTER(ConvProblem), C.POINTER(C.c_int)]),
    "primkit_solver_is_tunable": (ST, [P, C.c_char_p, C.POINTER(C.c_int)]),
    "primkit_solver_workspace_bytes": (ST, [P, C.c_char_p, C.POINTER(ConvProblem), C.POINTER(C.c_uint64)]),
    "primkit_find_convolution": (ST, [P, C.POINTER(ConvProblem), FP, FP, C.c_size_t,
                                      C.POINTER(AlgoPerf), C.c_int, C.POINTER(C.c_int)]),
    "primkit_conv_run": (ST, [P, C.POINTER(ConvProblem), C.c_char_p, FP, FP, FP, C.c_size_t]),
    "primkit_tune": (ST, [P, C.POINTER(ConvProblem), C.c_char_p, C.c_int64, C.c_int, I64P]),
    "primkit_perfdb_save": (ST, [P, C.c_char_p]),
    "primkit_perfdb_load": (ST, [P, C.c_char_p]),
    "primkit_fusion_plan_create": (ST, [I64P, C.c_int, C.POINTER(P)]),
    "primkit_fusion_plan_destroy": (None, [P]),
    "primkit_fusion_add_conv": (ST, [P, I64P, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                     C.c_int64, C.c_int]),
    "primkit_fusion_add_bias": (ST, [P, C.c_int64]),
    "primkit_fusion_add_batchnorm": (ST, [P, C.c_int]),
    "primkit_fusion_add_activation": (ST, [P, C.c_int, C.c_float]),
    "primkit_fusion_compile": (ST, [P, P]),
    "primkit_fusion_output_dims": (ST, [P, I64P]),
    "primkit_fusion_set_args": (ST, [P, FP, FP, FP, FP, FP, FP, C.c_float, FP]),
    "primkit_fusion_execute": (ST, [P, P, FP, FP, C.c_int]),
}

POOL_MAX, POOL_AVG = 0, 1

# section 2 (B200 additions)
SECTION2 = {
    "primkit_handle_create_with_stream": (ST, [P, C.c_int, C.POINTER(P)]),
    "primkit_handle_set_stream": (ST, [P, P]),
    "primkit_channel_pitch": (C.c_int64, [C.c_int64]),
    "primkit_conv_device_workspace": (ST, [P, C.POINTER(ConvProblem), C.c_char_p, C.POINTER(C.c_uint64)]),
    "primkit_conv_run_device": (ST, [P, C.POINTER(ConvProblem), C.c_char_p, P, P, P, P, C.c_size_t]),
    "primkit_fusion_execute_device": (ST, [P, P, P, P, C.c_int]),
    "primkit_batchnorm_forward_train": (ST, [P, C.c_int, I64P, C.c_int, FP, FP, FP, FP, FP,
                                             C.c_float, C.c_float, FP, FP, FP]),
    "primkit_batchnorm_forward_infer": (ST, [P, C.c_int, I64P, C.c_int, FP, FP, FP, FP, FP,
                                             C.c_float, FP]),
    "primkit_batchnorm_backward": (ST, [P, C.c_int, I64P, C.c_int, FP, FP, FP, FP, FP, FP, FP, FP]),
    "primkit_batchnorm_forward_train_device": (ST, [P, I64P, C.c_int, P, P, P, P, P, C.c_float,
                                                    C.c_float, P, P, P, C.c_int]),
    "primkit_batchnorm_backward_device": (ST, [P, I64P, C.c_int, P, P, P, P, P, P, P, P, P, P,
                                               C.c_int]),
    "primkit_conv_bn_workspace": (ST, [P, C.POINTER(ConvProblem), C.c_char_p, C.POINTER(C.c_uint64)]),
    "primkit_conv_bn_forward_train_device": (ST, [P, C.POINTER(ConvProblem), C.c_char_p, P, P, P, P,
                                                  P, P, C.c_float, C.c_float, P, P, P, P, C.c_int,
                                                  P, C.c_size_t]),
    "primkit_conv_backward_data_bn_device": (ST, [P, C.POINTER(ConvProblem), C.c_char_p, P, P, P,
                                                  P, P, P, P, P, C.c_int, P, P, P, P, C.c_size_t]),
    "primkit_activation_forward": (ST, [P, C.c_int, C.c_float, I64P, C.c_int, FP, FP]),
    "primkit_activation_backward": (ST, [P, C.c_int, C.c_float, I64P, C.c_int, FP, FP, FP]),
    "primkit_nchw_to_device": (ST, [P, I64P, C.c_int, P, P]),
    "primkit_device_to_nchw": (ST, [P, I64P, C.c_int, P, P]),
    "primkit_handle_kernel_launches": (ST, [P, C.POINTER(C.c_uint64)]),
    "primkit_handle_last_device_ms": (ST, [P, C.POINTER(C.c_double)]),
    "primkit_handle_last_kernel": (ST, [P, C.c_char_p, C.c_size_t]),
    "primkit_handle_last_variant": (ST, [P, C.c_char_p, C.c_size_t]),
    "primkit_tune_kernels": (ST, [P, C.POINTER(ConvProblem), C.c_char_p, C.c_int64, C.c_char_p,
                                  C.c_size_t, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "primkit_plan_kernel_config": (ST, [P, C.POINTER(ConvProblem), C.c_char_p, C.c_char_p,
                                        C.c_size_t]),
    "primkit_handle_load_system_db": (ST, [P, C.c_char_p]),
    "primkit_handle_system_db": (ST, [P, C.c_char_p, C.c_size_t, C.POINTER(C.c_uint64)]),
    "primkit_handle_plan_cache_stats": (ST, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                             C.POINTER(C.c_uint64)]),
    "primkit_pooling_output_dims": (ST, [I64P, I64P, I64P, I64P, I64P]),
    "primkit_pooling_forward": (ST, [P, C.c_int, I64P, I64P, I64P, I64P, C.c_int, FP, FP, I64P]),
    "primkit_pooling_backward": (ST, [P, C.c_int, I64P, I64P, I64P, I64P, C.c_int, FP, I64P, FP]),
    "primkit_pooling_forward_device": (ST, [P, C.c_int, I64P, I64P, I64P, I64P, C.c_int, P, P, P]),
    "primkit_pooling_backward_device": (ST, [P, C.c_int, I64P, I64P, I64P, I64P, C.c_int, P, P, P]),
    "primkit_softmax_forward": (ST, [P, C.c_int, I64P, C.c_int, C.c_int64, FP, FP]),
    "primkit_softmax_backward": (ST, [P, C.c_int, I64P, C.c_int, C.c_int64, FP, FP, FP]),
    "primkit_softmax_forward_device": (ST, [P, C.c_int, I64P, C.c_int, C.c_int64, P, P]),
    "primkit_softmax_backward_device": (ST, [P, C.c_int, I64P, C.c_int, C.c_int64, P, P, P]),
    # section 3: data-parallel all-reduce
    "primkit_dp_unique_id": (ST, [C.c_char_p]),
    "primkit_dp_create": (ST, [P, C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(P)]),
    "primkit_dp_destroy": (None, [P]),
    "primkit_dp_set_bucket_bytes": (ST, [P, C.c_uint64]),
    "primkit_dp_register": (ST, [P, P, C.c_uint64, C.c_int, C.POINTER(C.c_int)]),
    "primkit_dp_grad_ready": (ST, [P, C.c_int]),
    "primkit_dp_finish": (ST, [P]),
    "primkit_dp_check": (ST, [P]),
    "primkit_dp_buckets": (ST, [P, C.POINTER(C.c_int)]),
    "primkit_dp_bucket_of": (ST, [P, C.c_int, C.POINTER(C.c_int)]),
}


def bind(lib: C.CDLL, sections=(SECTION1, SECTION2)) -> C.CDLL:
    for table in sections:
        for name, (res, args) in table.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
    return lib


def header_symbols(header_path: str) -> list[str]:
    """Every PRIMKIT_API function declared in a primkit header."""
    import re
    text = open(header_path).read()
    return re.findall(r"PRIMKIT_API[^;(]*?\b(primkit_\w+)\s*\(", text, flags=re.S)
