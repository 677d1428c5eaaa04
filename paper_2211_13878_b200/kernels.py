"""Torch-tensor conveniences over the per-kernel C ABI (gx_k_* in include/gx.h).

Used by the parity tests and the profiler.  Tensors only supply device pointers and
strides; all compute runs in libgx.so.  There is no CPU fallback: a CPU tensor or a
missing library is an error.
"""
from __future__ import annotations

import ctypes

from . import _lib


def _ptr(t) -> int:
    if t is None:
        return 0
    if not t.is_cuda:
        raise ValueError("gx kernels take CUDA tensors only (no CPU fallback)")
    return t.data_ptr()


def dropout_threshold(p: float) -> int:
    """p * 2^32 rounded down, clamped; 0 disables dropout (matches the oracle)."""
    if p <= 0.0:
        return 0
    return min(int(p * 4294967296.0), 0xFFFFFFFF)


def gemm(a, b, *, a_mn_major=False, b_mn_major=False, out=None, out_kind="bf16", bias=None,
         gelu_aux=None, residual=None, alpha=1.0, dropout_p=0.0, seed=0, site=0,
         row_offset=0, col_offset=0, drop_ld=None, tile_n=0, stream=None):
    """C = A * B^T.  A is [M,K] (or [K,M] if a_mn_major); B is [N,K] (or [K,N])."""
    import torch
    M = a.shape[1] if a_mn_major else a.shape[0]
    K = a.shape[0] if a_mn_major else a.shape[1]
    N = b.shape[1] if b_mn_major else b.shape[0]
    Kb = b.shape[0] if b_mn_major else b.shape[1]
    if K != Kb:
        raise ValueError(f"gemm: K mismatch {K} vs {Kb}")
    kinds = {"bf16": _lib.GX_OUT_BF16, "f32": _lib.GX_OUT_F32, "f32_acc": _lib.GX_OUT_F32_ACC}
    if out is None:
        dt = torch.bfloat16 if out_kind == "bf16" else torch.float32
        out = torch.empty(M, N, device=a.device, dtype=dt)
    ep = _lib.GemmEpilogue()
    ep.out_kind = kinds[out_kind]
    ep.out = _ptr(out)
    ep.ldo = out.stride(0)
    ep.alpha = alpha
    ep.bias = _ptr(bias)
    ep.gelu = 1 if gelu_aux is not None else 0
    ep.aux = _ptr(gelu_aux)
    ep.ld_aux = gelu_aux.stride(0) if gelu_aux is not None else 0
    ep.residual = _ptr(residual)
    ep.ld_res = residual.stride(0) if residual is not None else 0
    ep.row_offset = row_offset
    ep.col_offset = col_offset
    ep.drop_ld = drop_ld if drop_ld is not None else N
    ep.drop_threshold = dropout_threshold(dropout_p)
    ep.drop_scale = 1.0 / (1.0 - dropout_p) if dropout_p > 0 else 1.0
    ep.seed = seed
    ep.site = site
    _lib.check(_lib.lib().gx_k_gemm_bf16(
        _ptr(a), a.stride(0), int(a_mn_major), _ptr(b), b.stride(0), int(b_mn_major),
        M, N, K, ctypes.byref(ep), tile_n, _lib.stream_ptr(stream)))
    return out
