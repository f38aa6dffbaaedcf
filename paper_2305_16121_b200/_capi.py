"""ctypes binding of the C-ABI in include/oases.h (liboases.so, built in-tree).

This module is the only place Python touches the native library. It fails
loudly when the library is missing: there is no Python or CPU fallback for any
compute entry point.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OASES_LIB") or os.path.join(_HERE, "liboases.so")

OK, ERR_CONFIG, ERR_INFEASIBLE, ERR_IO, ERR_CUDA, ERR_NCCL = 0, 2, 3, 4, 5, 6
F32, BF16 = 0, 1
EPI_NONE, EPI_BIAS, EPI_BIAS_GELU, EPI_DGELU, EPI_BIAS_GELU_GRAD, EPI_MUL, EPI_ROWDOT = 0, 1, 2, 3, 4, 5, 6
CAUSAL_NONE, CAUSAL_SKIP_UPPER, CAUSAL_K_UPTO_M, CAUSAL_K_FROM_M = 0, 1, 2, 3


class OasesError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[oases status {status}] {msg}")
        self.status = status


class GemmOperand(C.Structure):
    _fields_ = [
        ("ptr", C.c_void_p),
        ("rows", C.c_int64),
        ("cols", C.c_int64),
        ("ld", C.c_int64),
        ("mn_major", C.c_int32),
        ("pad_", C.c_int32),
        ("row_off", C.c_int64 * 2),
        ("col_off", C.c_int64 * 2),
    ]


class GemmDesc(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32),
        ("c_dtype", C.c_int32),
        ("M", C.c_int64),
        ("N", C.c_int64),
        ("K", C.c_int64),
        ("batch", C.c_int64),
        ("batch_inner", C.c_int64),
        ("a", GemmOperand),
        ("b", GemmOperand),
        ("c", C.c_void_p),
        ("ldc", C.c_int64),
        ("c_row_off", C.c_int64 * 2),
        ("c_col_off", C.c_int64 * 2),
        ("epilogue", C.c_int32),
        ("causal", C.c_int32),
        ("alpha", C.c_float),
        ("accumulate", C.c_int32),
        ("bias", C.c_void_p),
        ("aux", C.c_void_p),
        ("c2", C.c_void_p),
        ("max_ctas", C.c_int32),
        ("pad_", C.c_int32),
        ("rowdot", C.c_void_p),
        ("rowdot_group", C.c_int32),
        ("rowdot_seq", C.c_int32),
        ("rowdot_heads", C.c_int32),
        ("pad2_", C.c_int32),
        ("colsum", C.c_void_p),
    ]


class AttnDesc(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32),
        ("samples", C.c_int32),
        ("heads_local", C.c_int32),
        ("heads_total", C.c_int32),
        ("head_offset", C.c_int32),
        ("head_dim", C.c_int32),
        ("seq", C.c_int32),
        ("max_ctas", C.c_int32),
        ("qkv", C.c_void_p),
        ("ld_qkv", C.c_int64),
        ("out", C.c_void_p),
        ("ld_out", C.c_int64),
        ("lse", C.c_void_p),
        ("dout", C.c_void_p),
        ("ld_dout", C.c_int64),
        ("dqkv", C.c_void_p),
        ("ld_dqkv", C.c_int64),
        ("ds", C.c_void_p),
        ("workspace", C.c_void_p),
        ("scale", C.c_float),
        ("dropout_p", C.c_float),
        ("seed", C.c_uint64),
        ("offset", C.c_uint64),
        ("mask_bits", C.c_void_p),
        ("mask_mode", C.c_int32),
        ("dsum_ready", C.c_int32),
        ("sample_offset", C.c_int32),
        ("pad_", C.c_int32),
    ]


class CtxDesc(C.Structure):
    _fields_ = [
        ("tp", C.c_int32),
        ("rank", C.c_int32),
        ("device", C.c_int32),
        ("local_workers", C.c_int32),
        ("unique_id", C.c_void_p),
        ("nccl_max_ctas", C.c_int32),
        ("gemm_max_ctas", C.c_int32),
        ("comm_disabled", C.c_int32),
    ]


class ModelDesc(C.Structure):
    _fields_ = [
        ("hidden_size", C.c_int32),
        ("num_layers", C.c_int32),
        ("seq_len", C.c_int32),
        ("attention_heads", C.c_int32),
        ("global_batch", C.c_int32),
        ("bytes_per_element", C.c_int32),
        ("recompute_enabled", C.c_int32),
        ("ffn_hidden", C.c_int32),
        ("use_attention", C.c_int32),
        ("use_layernorm", C.c_int32),
        ("use_bias", C.c_int32),
        ("use_residual", C.c_int32),
        ("hidden_dropout", C.c_float),
        ("attention_dropout", C.c_float),
        ("ln_eps", C.c_float),
        ("pad_", C.c_int32),
        ("seed", C.c_uint64),
    ]


class BlockLayout(C.Structure):
    _fields_ = [
        ("degree", C.c_int32),
        ("group", C.c_int32),
        ("rank_in_group", C.c_int32),
        ("groups", C.c_int32),
        ("heads_local", C.c_int32),
        ("attention", C.c_int32),
        ("samples_per_sub_batch", C.c_int64),
        ("tokens_per_sub_batch", C.c_int64),
        ("token_row0", C.c_int64),
        ("col_width", C.c_int64),
        ("row_width", C.c_int64),
    ]


class PlanOp(C.Structure):
    _fields_ = [
        ("id", C.c_int32),
        ("base_id", C.c_int32),
        ("kind", C.c_int32),
        ("pass_", C.c_int32),
        ("stream", C.c_int32),
        ("block", C.c_int32),
        ("sub_batch", C.c_int32),
        ("blocking", C.c_int32),
        ("dep_begin", C.c_int32),
        ("dep_count", C.c_int32),
    ]


class FlatPlan(C.Structure):
    _fields_ = [
        ("variant", C.c_int32),
        ("split_batch", C.c_int32),
        ("has_recompute", C.c_int32),
        ("n_forward", C.c_int32),
        ("n_ops", C.c_int32),
        ("n_deps", C.c_int32),
        ("ops", C.POINTER(PlanOp)),
        ("deps", C.POINTER(C.c_int32)),
    ]


class TraceEventC(C.Structure):
    _fields_ = [("op_id", C.c_int32), ("stream", C.c_int32), ("start", C.c_double), ("end", C.c_double)]


class KernelStats(C.Structure):
    _fields_ = [("gemm_ms", C.c_double), ("gemm_flops", C.c_double), ("gemm_launches", C.c_int32),
                ("pad_", C.c_int32)]


class StepResult(C.Structure):
    _fields_ = [
        ("makespan", C.c_double),
        ("compute_busy_fraction", C.c_double),
        ("comm_exposed", C.c_double),
        ("peak_memory", C.c_double),
        ("loss", C.c_double),
        ("n_events", C.c_int32),
        ("pad_", C.c_int32),
        ("events", C.POINTER(TraceEventC)),
    ]


# (name, restype, argtypes) of every symbol include/oases.h declares.
_SIGNATURES = [
    ("oases_last_error", C.c_char_p, []),
    ("oases_version", C.c_char_p, []),
    ("oases_device_sm_count", C.c_int, []),
    ("oases_gemm", C.c_int, [C.POINTER(GemmDesc), C.c_void_p]),
    ("oases_gemm_grouped", C.c_int, [C.POINTER(GemmDesc), C.c_int32, C.c_void_p]),
    ("oases_attention_supported", C.c_int32, [C.c_int, C.c_int32, C.c_int32]),
    ("oases_attention_fwd", C.c_int, [C.POINTER(AttnDesc), C.c_void_p]),
    ("oases_attention_mask_bytes", C.c_size_t, [C.POINTER(AttnDesc)]),
    ("oases_attention_masks", C.c_int, [C.POINTER(AttnDesc), C.c_void_p]),
    ("oases_attention_bwd_workspace", C.c_size_t, [C.POINTER(AttnDesc)]),
    ("oases_attention_bwd", C.c_int, [C.POINTER(AttnDesc), C.c_void_p]),
    ("oases_layernorm_fwd", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                       C.c_float, C.c_void_p]),
    ("oases_layernorm_bwd", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                       C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_float, C.c_void_p]),
    ("oases_layernorm_bwd_workspace", C.c_size_t, [C.c_int64, C.c_int64]),
    ("oases_softmax_fwd", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_float,
                                     C.c_float, C.c_uint64, C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    ("oases_softmax_bwd", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_float,
                                     C.c_float, C.c_uint64, C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    ("oases_bias_dropout_residual_layernorm_fwd", C.c_int,
     [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
      C.c_int64, C.c_float, C.c_float, C.c_uint64, C.c_uint64, C.c_void_p]),
    ("oases_bias_dropout_residual_fwd", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                                   C.c_int64, C.c_float, C.c_uint64, C.c_uint64, C.c_void_p]),
    ("oases_bias_dropout_residual_bwd", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                                   C.c_int64, C.c_int64, C.c_float, C.c_uint64, C.c_uint64,
                                                   C.c_void_p]),
    ("oases_colsum_workspace", C.c_size_t, [C.c_int64, C.c_int64]),
    ("oases_colsum", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_int64,
                                C.c_void_p]),
    ("oases_colsum_finalize", C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int, C.c_void_p]),
    ("oases_gelu_fwd", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    ("oases_gelu_bwd", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    ("oases_gelu_sq_loss", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int64,
                                      C.c_void_p]),
    ("oases_local_allreduce", C.c_int, [C.c_int, C.POINTER(C.c_void_p), C.c_int, C.c_int64, C.c_void_p]),
    ("oases_get_unique_id", C.c_int, [C.c_void_p]),
    ("oases_ctx_create", C.c_int, [C.POINTER(CtxDesc), C.POINTER(C.c_void_p)]),
    ("oases_ctx_destroy", C.c_int, [C.c_void_p]),
    ("oases_stack_create", C.c_int, [C.c_void_p, C.POINTER(ModelDesc), C.POINTER(C.c_void_p)]),
    ("oases_stack_create_mixed", C.c_int,
     [C.c_void_p, C.POINTER(ModelDesc), C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_void_p)]),
    ("oases_stack_block_degree", C.c_int, [C.c_void_p, C.c_int]),
    ("oases_rank_layout", C.c_int,
     [C.POINTER(ModelDesc), C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.POINTER(BlockLayout)]),
    ("oases_stack_destroy", C.c_int, [C.c_void_p]),
    ("oases_stack_param_numel", C.c_int64, [C.c_void_p, C.c_int, C.c_int]),
    ("oases_stack_num_blocks", C.c_int, [C.c_void_p]),
    ("oases_stack_num_workers", C.c_int, [C.c_void_p]),
    ("oases_stack_set_param", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]),
    ("oases_stack_get_grad", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]),
    ("oases_stack_init_random", C.c_int, [C.c_void_p, C.c_uint64]),
    ("oases_plan_bind", C.c_int, [C.c_void_p, C.POINTER(FlatPlan)]),
    ("oases_step", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(StepResult)]),
    ("oases_stack_set_input", C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    ("oases_stack_get_input_grad", C.c_int, [C.c_void_p, C.c_void_p]),
    ("oases_stack_get_activation", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]),
    ("oases_stack_capture_graph", C.c_int, [C.c_void_p]),
    ("oases_stack_sync", C.c_int, [C.c_void_p]),
    ("oases_stack_kernel_launches", C.c_int, [C.c_void_p]),
    ("oases_stack_set_kernel_timing", C.c_int, [C.c_void_p, C.c_int]),
    ("oases_stack_kernel_stats", C.c_int, [C.c_void_p, C.POINTER(KernelStats)]),
    ("oases_stack_graph_kernel_stats", C.c_int, [C.c_void_p, C.POINTER(KernelStats)]),
]

SYMBOLS = [name for name, _, _ in _SIGNATURES]

_lib = None


def lib():
    """Load liboases.so (once) and declare every C-ABI signature."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                "there is no CPU fallback")
        # torch first: its bundled NCCL/cudart get resolved before ours.
        try:
            import torch  # noqa: F401
        except ImportError:
            pass
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, res, args in _SIGNATURES:
            if not hasattr(L, name):
                continue  # reported by missing_symbols(); calling it raises AttributeError
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def missing_symbols() -> list:
    L = lib()
    return [name for name in SYMBOLS if not hasattr(L, name)]


def check(status: int) -> None:
    if status != OK:
        msg = lib().oases_last_error().decode(errors="replace")
        raise OasesError(status, msg)
