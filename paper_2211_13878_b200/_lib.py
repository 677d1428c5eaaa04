"""ctypes binding of libgx.so (the C ABI declared in include/gx.h).

The library is built in-tree (``make``) and loaded from this package directory.  There is
no fallback: if the shared object is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_char_p, c_double, c_float, c_int, c_int64,
                    c_size_t, c_uint32, c_uint64, c_void_p)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgx.so")

GX_OK, GX_ERR_CONFIG, GX_ERR_INFEASIBLE, GX_ERR_CUDA, GX_ERR_NCCL = 0, 1, 2, 3, 4
GX_OUT_BF16, GX_OUT_F32, GX_OUT_F32_ACC = 0, 1, 2


class GxError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"gx error {code}: {msg}")
        self.code = code
        self.msg = msg


class ValidationError(GxError):
    """Mirrors parplan::ValidationError (proj/include/parplan/common.h:26-29)."""


class GuardError(GxError):
    """Mirrors parplan::GuardError (proj/include/parplan/common.h:33-36)."""


class GemmEpilogue(Structure):
    _fields_ = [
        ("out_kind", c_int), ("out", c_void_p), ("ldo", c_int64), ("alpha", c_float),
        ("bias", c_void_p), ("gelu", c_int), ("aux", c_void_p), ("ld_aux", c_int64),
        ("residual", c_void_p), ("ld_res", c_int64), ("row_offset", c_int64),
        ("col_offset", c_int64), ("drop_ld", c_int64), ("drop_threshold", c_uint32),
        ("drop_scale", c_float), ("seed", c_uint64), ("site", c_uint64), ("gelu_bwd", c_int),
        ("seed_offset", c_void_p),
        ("trace", c_void_p),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `make` (or __graft_entry__.build())")
        _lib = ctypes.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def _declare(L: ctypes.CDLL) -> None:
    L.gx_last_error.restype = c_char_p
    L.gx_version.restype = c_int
    L.gx_k_gemm_bf16.argtypes = [c_void_p, c_int64, c_int, c_void_p, c_int64, c_int, c_int,
                                 c_int, c_int, POINTER(GemmEpilogue), c_int, c_void_p]
    L.gx_k_gemm_bf16.restype = c_int
    L.gx_k_gemm_bf16_splitk.argtypes = [c_void_p, c_int64, c_int, c_void_p, c_int64, c_int, c_int,
                                        c_int, c_int, c_void_p, c_int64, c_int, c_int, c_void_p]
    L.gx_k_gemm_bf16_splitk.restype = c_int
    for name in ("gx_k_attention_fwd", "gx_k_attention_bwd", "gx_k_layernorm_fwd",
                 "gx_k_layernorm_bwd", "gx_k_bias_dropout_add", "gx_k_dropout_bwd_colsum",
                 "gx_k_colsum", "gx_k_mse_loss", "gx_k_adamw", "gx_k_cast_bf16",
                 "gx_k_patch_merge", "gx_k_window_roll", "gx_k_rpb_grad", "gx_k_relb_grad",
                 "gx_k_poison_smem"):
        getattr(L, name).restype = c_int
    vp = c_void_p
    L.gx_k_attention_fwd.argtypes = [vp, vp]
    L.gx_k_attention_bwd.argtypes = [vp, vp]
    L.gx_k_poison_smem.argtypes = [vp]
    L.gx_k_layernorm_fwd.argtypes = [vp, vp, vp, vp, vp, vp, c_int, c_int, vp]
    L.gx_k_layernorm_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, c_int, c_int, vp]
    L.gx_k_bias_dropout_add.argtypes = [vp, vp, vp, vp, c_int, c_int, vp, vp]
    L.gx_k_dropout_bwd_colsum.argtypes = [vp, vp, vp, c_int, c_int, vp, vp]
    L.gx_k_colsum.argtypes = [c_void_p, c_int64, c_void_p, c_int, c_int, c_void_p]
    L.gx_k_mse_loss.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_float, c_void_p]
    L.gx_k_adamw.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_float,
                             c_float, c_float, c_float, c_float, c_float, c_float, c_void_p]
    L.gx_k_cast_bf16.argtypes = [c_void_p, c_void_p, c_int64, c_void_p]
    L.gx_k_patch_merge.argtypes = [vp, vp, c_int, c_int, c_int, c_int, c_int, vp]
    L.gx_k_window_roll.argtypes = [vp, vp, c_int, c_int, c_int, c_int, c_int, c_int, vp]
    L.gx_k_rpb_grad.argtypes = [vp, c_int, c_int, c_int, vp, c_int, vp]
    L.gx_k_relb_grad.argtypes = [vp, c_int, c_int, c_int, vp, c_int, vp, c_int, vp]
    L.gx_exec_create.argtypes = [c_char_p, POINTER(c_void_p)]
    L.gx_exec_destroy.argtypes = [vp]
    L.gx_exec_set_layer_params.argtypes = [vp, c_int, vp, c_int64]
    L.gx_exec_export_layer.argtypes = [vp, c_int, c_int, vp, c_int64]
    L.gx_exec_load_batch.argtypes = [vp, vp, vp]
    L.gx_exec_load_batch_device.argtypes = [vp, vp, vp]
    L.gx_exec_run.argtypes = [vp, c_int]
    L.gx_exec_loss.argtypes = [vp, POINTER(c_float)]
    L.gx_exec_sync.argtypes = [vp, c_int64]
    L.gx_exec_step.argtypes = [vp, vp, vp, c_int, POINTER(c_float)]
    L.gx_exec_export_output.argtypes = [vp, c_int, vp]
    L.gx_exec_stream.argtypes = [vp, POINTER(c_void_p)]
    L.gx_exec_info.argtypes = [vp, c_char_p, c_size_t, POINTER(c_size_t)]
    L.gx_exec_canonical_size.argtypes = [c_int, c_int, POINTER(c_int64)]
    L.gx_nccl_unique_id.argtypes = [c_char_p, c_size_t]
    for name in ("gx_exec_create", "gx_exec_destroy", "gx_exec_set_layer_params",
                 "gx_exec_export_layer", "gx_exec_load_batch", "gx_exec_load_batch_device",
                 "gx_exec_run", "gx_exec_loss", "gx_exec_sync", "gx_exec_step", "gx_exec_export_output",
                 "gx_exec_stream", "gx_exec_info", "gx_exec_canonical_size",
                 "gx_nccl_unique_id"):
        getattr(L, name).restype = c_int
    L.gx_launch_count.restype = c_int64
    L.gx_exec_profile_report.argtypes = [vp, c_char_p, c_size_t, POINTER(c_size_t)]
    L.gx_exec_profile_report.restype = c_int
    L.gx_exec_init_params.argtypes = [vp, c_uint64, c_float]
    L.gx_exec_init_params.restype = c_int
    L.gx_exec_topology.argtypes = [c_char_p, c_char_p, c_size_t, POINTER(c_size_t)]
    L.gx_exec_topology.restype = c_int
    declare_plan_api(L, "gx_plan_")


def declare_plan_api(L: ctypes.CDLL, prefix: str) -> None:
    """Declares the plan/search C surface under `prefix` (gx_plan_ or the oracle's ref_plan_)."""
    getattr(L, prefix + "last_error").restype = c_char_p
    for name, args in _EXTRA_SIGNATURES.items():
        fn = getattr(L, prefix + name[len("gx_plan_"):], None)
        if fn is not None:
            fn.argtypes = args
            fn.restype = c_int


_EXTRA_SIGNATURES: dict = {
    "gx_plan_optimize": [c_char_p, c_char_p, c_char_p, POINTER(c_int), c_int, c_int, c_char_p,
                         c_int, c_char_p, c_size_t, POINTER(c_size_t)],
    "gx_plan_exhaustive": [c_char_p, c_char_p, c_char_p, POINTER(c_int), c_int, c_int,
                           c_char_p, c_char_p, c_size_t, POINTER(c_size_t)],
    "gx_plan_dp_search": [c_char_p, c_int, c_int, c_int64, c_int, c_int, c_int, c_double,
                          c_char_p, c_char_p, c_size_t, POINTER(c_size_t)],
    "gx_plan_estimate": [c_int64, c_int64, c_double, c_char_p, c_int, c_double, c_char_p,
                         c_char_p, c_size_t, POINTER(c_size_t)],
    "gx_plan_transformation_ms": [c_int64, c_int64, c_char_p, c_char_p, c_int, c_double,
                                  POINTER(c_double)],
    "gx_plan_enumerate": [c_int, c_int, c_char_p, c_size_t, POINTER(c_size_t)],
    "gx_plan_exhaustive_dp": [c_char_p, c_int, c_int, c_int64, c_int, c_int, c_int, c_double,
                              c_char_p, c_char_p, c_size_t, POINTER(c_size_t)],
    "gx_plan_partition": [c_char_p, c_int, c_char_p, c_char_p, c_size_t, POINTER(c_size_t)],
    "gx_plan_pipeline_cost": [POINTER(c_double), c_int, c_int, c_int, POINTER(c_double)],
    "gx_plan_collective_bytes": [c_int, c_int, c_double, POINTER(c_double)],
    "gx_plan_validate": [c_char_p, c_char_p],
    "gx_plan_bandwidth": [c_char_p, c_int, POINTER(c_double)],
}


def last_error() -> str:
    return lib().gx_last_error().decode()


def check(code: int) -> None:
    if code != GX_OK:
        raise GxError(code, last_error())


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
