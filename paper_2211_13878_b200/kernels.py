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
    """Byte threshold thr8 = round(p * 256) in [1, 255]; 0 disables dropout (philox.cuh)."""
    if p <= 0.0:
        return 0
    return max(1, min(255, int(p * 256.0 + 0.5)))


def dropout_scale(p: float) -> float:
    t = dropout_threshold(p)
    return 1.0 if t == 0 else 256.0 / (256 - t)


def gemm(a, b, *, a_mn_major=False, b_mn_major=False, out=None, out_kind="bf16", bias=None,
         gelu_aux=None, residual=None, alpha=1.0, dropout_p=0.0, seed=0, site=0,
         row_offset=0, col_offset=0, drop_ld=None, tile_n=0, stream=None, gelu_bwd_aux=None,
         trace=None, gelu_mode=1):
    """C = A * B^T.  A is [M,K] (or [K,M] if a_mn_major); B is [N,K] (or [K,N]).
    trace: optional int64 device tensor [grid*16] receiving per-CTA %globaltimer stamps.
    gelu_mode 2: gelu_aux receives gelu'(pre) (forward) / gelu_bwd_aux holds gelu'(pre) (backward)."""
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
    ep.gelu = gelu_mode if gelu_aux is not None else 0
    ep.gelu_bwd = gelu_mode if gelu_bwd_aux is not None else 0
    aux = gelu_aux if gelu_aux is not None else gelu_bwd_aux
    ep.aux = _ptr(aux)
    ep.ld_aux = aux.stride(0) if aux is not None else 0
    ep.residual = _ptr(residual)
    ep.ld_res = residual.stride(0) if residual is not None else 0
    ep.row_offset = row_offset
    ep.col_offset = col_offset
    ep.drop_ld = drop_ld if drop_ld is not None else N
    ep.drop_threshold = dropout_threshold(dropout_p)
    ep.drop_scale = dropout_scale(dropout_p)
    ep.seed = seed
    ep.site = site
    ep.trace = _ptr(trace)
    _lib.check(_lib.lib().gx_k_gemm_bf16(
        _ptr(a), a.stride(0), int(a_mn_major), _ptr(b), b.stride(0), int(b_mn_major),
        M, N, K, ctypes.byref(ep), tile_n, _lib.stream_ptr(stream)))
    return out


def gemm_splitk(a, b, *, a_mn_major=False, b_mn_major=False, out=None, splits=0, tile_n=0,
                stream=None):
    """out (fp32, zero-initialised here if None) += A * B^T over `splits` K-slices."""
    import torch
    M = a.shape[1] if a_mn_major else a.shape[0]
    K = a.shape[0] if a_mn_major else a.shape[1]
    N = b.shape[1] if b_mn_major else b.shape[0]
    if out is None:
        out = torch.zeros(M, N, device=a.device, dtype=torch.float32)
    _lib.check(_lib.lib().gx_k_gemm_bf16_splitk(
        _ptr(a), a.stride(0), int(a_mn_major), _ptr(b), b.stride(0), int(b_mn_major), M, N, K,
        _ptr(out), out.stride(0), splits, tile_n, _lib.stream_ptr(stream)))
    return out


class _AttnArgs(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int), ("seq", ctypes.c_int), ("heads", ctypes.c_int),
                ("head_dim", ctypes.c_int), ("heads_total", ctypes.c_int),
                ("head_offset", ctypes.c_int), ("sample_offset", ctypes.c_int64),
                ("scale", ctypes.c_float), ("qkv", ctypes.c_void_p), ("ld_qkv", ctypes.c_int64),
                ("ctx", ctypes.c_void_p), ("ld_ctx", ctypes.c_int64), ("lse", ctypes.c_void_p),
                ("dctx", ctypes.c_void_p), ("dqkv", ctypes.c_void_p),
                ("dq_accum", ctypes.c_void_p), ("dsum", ctypes.c_void_p),
                ("drop_threshold", ctypes.c_uint32), ("drop_scale", ctypes.c_float),
                ("seed", ctypes.c_uint64), ("site", ctypes.c_uint64),
                ("seed_offset", ctypes.c_void_p), ("mask", ctypes.c_void_p),
                ("trace", ctypes.c_void_p), ("causal", ctypes.c_int),
                ("win_grid", ctypes.c_int), ("win_side", ctypes.c_int), ("win_shift", ctypes.c_int),
                ("rpb", ctypes.c_void_p), ("rpb_dpart", ctypes.c_void_p), ("rpb_side", ctypes.c_int),
                ("relb", ctypes.c_void_p), ("relb_map", ctypes.c_void_p),
                ("relb_buckets", ctypes.c_int), ("relb_dpart", ctypes.c_void_p)]


class Dropout(ctypes.Structure):
    _fields_ = [("threshold", ctypes.c_uint32), ("scale", ctypes.c_float),
                ("seed", ctypes.c_uint64), ("site", ctypes.c_uint64),
                ("row_offset", ctypes.c_int64), ("col_offset", ctypes.c_int64),
                ("drop_ld", ctypes.c_int64), ("seed_offset", ctypes.c_void_p)]


def make_dropout(p, seed, site, row_offset=0, col_offset=0, drop_ld=0):
    d = Dropout()
    d.threshold = dropout_threshold(p)
    d.scale = dropout_scale(p)
    d.seed, d.site, d.row_offset, d.col_offset, d.drop_ld = seed, site, row_offset, col_offset, drop_ld
    return d


def _attn_args(qkv, batch, seq, heads, head_dim, p, seed, site, heads_total=None, head_offset=0,
               sample_offset=0, causal=False, win=None, rpb=None, rpb_dpart=None, relb=None,
               relb_map=None, relb_dpart=None):
    a = _AttnArgs()
    a.causal = int(causal)
    if relb is not None:  # T5 relative bias: bf16 [heads][buckets] + int8 bucket map [2 seq - 1]
        a.relb, a.relb_map, a.relb_buckets = _ptr(relb), _ptr(relb_map), relb.shape[1]
        a.relb_dpart = _ptr(relb_dpart) if relb_dpart is not None else None
    if rpb is not None:  # Swin relative-position bias table [heads][(2 side - 1)^2] (bf16)
        a.rpb, a.rpb_side = _ptr(rpb), int(round(seq ** 0.5))
        a.rpb_dpart = _ptr(rpb_dpart) if rpb_dpart is not None else None
    if win is not None:  # (grid, side, shift): Swin shifted-window region mask
        a.win_grid, a.win_side, a.win_shift = win
    a.batch, a.seq, a.heads, a.head_dim = batch, seq, heads, head_dim
    a.heads_total = heads_total or heads
    a.head_offset, a.sample_offset = head_offset, sample_offset
    a.scale = head_dim ** -0.5
    a.qkv, a.ld_qkv = _ptr(qkv), qkv.stride(0)
    a.drop_threshold = dropout_threshold(p)
    a.drop_scale = dropout_scale(p)
    a.seed, a.site = seed, site
    return a


def poison_smem():
    """Fill every SM's shared memory with NaN bytes (tests: catches reads of unwritten smem)."""
    _lib.check(_lib.lib().gx_k_poison_smem(_lib.stream_ptr()))


def attention_mask_buffer(batch, seq, heads, device):
    import torch
    return torch.zeros(batch * heads * seq * ((seq + 63) // 64) * 4, device=device,
                       dtype=torch.int16)


def attention_fwd(qkv, batch, seq, heads, head_dim, p=0.0, seed=0, site=0, mask=None, trace=None,
                  **kw):
    """Returns (ctx, lse, mask); mask (keep bits) feeds attention_bwd when p > 0."""
    import torch
    ctx = torch.empty(batch * seq, heads * head_dim, device=qkv.device, dtype=torch.bfloat16)
    lse = torch.empty(batch * heads, seq, device=qkv.device, dtype=torch.float32)
    if mask is None:
        mask = attention_mask_buffer(batch, seq, heads, qkv.device)
    a = _attn_args(qkv, batch, seq, heads, head_dim, p, seed, site, **kw)
    a.ctx, a.ld_ctx, a.lse, a.mask = _ptr(ctx), ctx.stride(0), _ptr(lse), _ptr(mask)
    a.trace = _ptr(trace)
    _lib.check(_lib.lib().gx_k_attention_fwd(ctypes.addressof(a), _lib.stream_ptr()))
    return ctx, lse, mask


def attention_bwd(qkv, ctx, lse, dctx, batch, seq, heads, head_dim, p=0.0, seed=0, site=0,
                  mask=None, trace=None, **kw):
    import torch
    dqkv = torch.zeros_like(qkv)
    # fp32 dQ partials (one slice per 128-key tile on the tcgen05 path) and D / ticket words
    # (zero-initialised: the tcgen05 path keeps per-head tickets there)
    # (short sequences are packed 128 // seq per tile: one spare sequence of slack)
    dq_acc = torch.empty(((seq + 127) // 128) * (batch + 1) * heads * ((seq + 3) // 4 * 4) * head_dim,
                         device=qkv.device, dtype=torch.float32)
    dsum = torch.zeros(batch * heads * seq, device=qkv.device, dtype=torch.float32)
    a = _attn_args(qkv, batch, seq, heads, head_dim, p, seed, site, **kw)
    a.ctx, a.ld_ctx, a.lse = _ptr(ctx), ctx.stride(0), _ptr(lse)
    a.dctx, a.dqkv, a.dq_accum, a.dsum = _ptr(dctx), _ptr(dqkv), _ptr(dq_acc), _ptr(dsum)
    a.mask = _ptr(mask)
    a.trace = _ptr(trace)
    _lib.check(_lib.lib().gx_k_attention_bwd(ctypes.addressof(a), _lib.stream_ptr()))
    return dqkv


def relb_grad(dpart, tiles, heads, seq, relb_map, buckets, out, accumulate=False):
    """T5 relative-bias table gradient from attention_bwd's relb_dpart partials."""
    _lib.check(_lib.lib().gx_k_relb_grad(_ptr(dpart), tiles, heads, seq, _ptr(relb_map), buckets,
                                         _ptr(out), int(accumulate), _lib.stream_ptr()))
    return out


def layernorm_fwd(x, gamma, beta):
    import torch
    rows, h = x.shape
    y = torch.empty_like(x)
    mean = torch.empty(rows, device=x.device, dtype=torch.float32)
    rstd = torch.empty(rows, device=x.device, dtype=torch.float32)
    _lib.check(_lib.lib().gx_k_layernorm_fwd(
        _ptr(x), _ptr(gamma), _ptr(beta), _ptr(y), _ptr(mean), _ptr(rstd), rows, h,
        ctypes.c_void_p(_lib.stream_ptr())))
    return y, mean, rstd


def layernorm_bwd(dy, x, mean, rstd, gamma, dres=None):
    import torch
    rows, h = x.shape
    dx = torch.empty_like(x)
    dg = torch.zeros(h, device=x.device, dtype=torch.float32)
    db = torch.zeros(h, device=x.device, dtype=torch.float32)
    _lib.check(_lib.lib().gx_k_layernorm_bwd(
        _ptr(dy), _ptr(x), _ptr(mean), _ptr(rstd), _ptr(gamma), _ptr(dres), _ptr(dx), _ptr(dg),
        _ptr(db), rows, h, ctypes.c_void_p(_lib.stream_ptr())))
    return dx, dg, db


def bias_dropout_add(x, bias, residual, d: Dropout):
    import torch
    out = torch.empty_like(x)
    rows, cols = x.shape
    _lib.check(_lib.lib().gx_k_bias_dropout_add(
        _ptr(x), _ptr(bias), _ptr(residual), _ptr(out), rows, cols, ctypes.addressof(d),
        ctypes.c_void_p(_lib.stream_ptr())))
    return out


def dropout_bwd_colsum(dy, d: Dropout):
    import torch
    rows, cols = dy.shape
    dz = torch.empty_like(dy)
    db = torch.zeros(cols, device=dy.device, dtype=torch.float32)
    _lib.check(_lib.lib().gx_k_dropout_bwd_colsum(
        _ptr(dy), _ptr(dz), _ptr(db), rows, cols, ctypes.addressof(d),
        ctypes.c_void_p(_lib.stream_ptr())))
    return dz, db


def mse_loss(y, target):
    import torch
    dy = torch.empty_like(y)
    loss = torch.zeros(1, device=y.device, dtype=torch.float32)
    _lib.check(_lib.lib().gx_k_mse_loss(_ptr(y), _ptr(target), _ptr(dy), _ptr(loss), y.numel(),
                                        ctypes.c_float(1.0 / y.numel()),
                                        ctypes.c_void_p(_lib.stream_ptr())))
    return loss, dy


def adamw(p, g, m, v, out_bf16, lr, b1, b2, eps, wd, step):
    _lib.check(_lib.lib().gx_k_adamw(
        _ptr(p), _ptr(g), _ptr(m), _ptr(v), _ptr(out_bf16), p.numel(), ctypes.c_float(lr),
        ctypes.c_float(b1), ctypes.c_float(b2), ctypes.c_float(eps), ctypes.c_float(wd),
        ctypes.c_float(1 - b1 ** step), ctypes.c_float(1 - b2 ** step),
        ctypes.c_void_p(_lib.stream_ptr())))


def patch_merge(x, samples, grid_out, window_side, backward=False):
    """Swin patch merging (gx_k_patch_merge): [samples*4*G^2, c] -> [samples*G^2, 4c], or the
    scatter of a merged gradient back when backward=True."""
    import torch
    c = x.shape[1] // 4 if backward else x.shape[1]
    rows_out = samples * grid_out * grid_out
    out = torch.empty((4 * rows_out, c) if backward else (rows_out, 4 * c), dtype=x.dtype,
                      device=x.device)
    _lib.check(_lib.lib().gx_k_patch_merge(_ptr(x), _ptr(out), samples, grid_out, window_side,
                                           c, int(backward), _lib.stream_ptr()))
    return out


def window_roll(x, samples, grid, window_side, shift, inverse=False):
    """Swin cyclic shift of window-major tokens (gx_k_window_roll)."""
    import torch
    out = torch.empty_like(x)
    _lib.check(_lib.lib().gx_k_window_roll(_ptr(x), _ptr(out), samples, grid, window_side, shift,
                                           x.shape[1], int(inverse), _lib.stream_ptr()))
    return out


def rpb_grad(dpart, batch, heads, side, grad, accumulate=True):
    """Relative-position-bias gradient: fixed-order batch sum of the per-(window, head) table
    gradients (attention_bwd's rpb_dpart) into grad (fp32 [heads][(2 side - 1)^2])."""
    _lib.check(_lib.lib().gx_k_rpb_grad(_ptr(dpart), batch, heads, side, _ptr(grad),
                                        int(accumulate), _lib.stream_ptr()))
    return grad
