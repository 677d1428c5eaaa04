"""TEST INFRASTRUCTURE ONLY — CPU restatement of the executor's Transformer-layer math.

PARITY UNPINNED BY THE REFERENCE: the reference (/root/reference/proj) is a planner only and
contains no layer implementation (SURVEY.md §8(c) "Layer-numerics oracle: NONE").  This
module restates the layer the executor runs (a pre-LN encoder layer, PAPER.md:136-157
semantics for how DP/SDP/TP/PP split it) in float64 numpy, and is itself pinned against
torch.autograd (float64, CPU) in tests/test_layer_oracle.py, with golden vectors committed
under tests/golden/.  Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
reference legs may use it.

Layer (h hidden, H heads of d, f ffn; x is [tokens, h], tokens = samples * seq):
    a   = LN1(x)                       (eps 1e-5)
    qkv = a Wqkv^T + bqkv              (Wqkv rows ordered [3][H][d])
    ctx = drop_attn(softmax(q k^T / sqrt(d))) v      per (sample, head)
    x1  = x + drop_h1(ctx Wo^T + bo)
    c   = LN2(x1)
    y   = x1 + drop_h2(gelu(c W1^T + b1) W2^T + b2)  (exact erf GeLU)
Window layers (Swin W-MSA, shape.window > 0): tokens are stored window-major and attention
runs per window of `window` consecutive tokens; shape.shift > 0 (SW-MSA) rolls LN1's output by
-shift in both grid axes first (roll_rows), masks q-k pairs from different regions of the rolled
grid (shift_regions) and rolls the attention output back.  Patch-merging layers (shape.merge) first map
their input [4*seq, h/2] to x = LN_m(gather_2x2(input)) W_m^T ([seq, h]; merge_rows).
Dropout uses the Philox4x32-10 byte scheme of csrc/kernels/philox.cuh: one call
philox({c lo, c hi, site lo, site hi}, {seed lo, seed hi}) yields 16 bytes; an element is
kept iff its byte >= thr8 = round(p * 256), kept values scale by 256 / (256 - thr8).
Hidden sites: element e -> call e >> 4, byte e & 15.  Attention sites: see _attn_mask.
Site ids per layer l: attn = 3l+0, hidden-1 = 3l+1, hidden-2 = 3l+2.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint64(0x9E3779B9), np.uint64(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 (Salmon et al. 2011); inputs uint32-valued arrays."""
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint64) & MASK32 for v in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint64) & MASK32
    k1 = np.asarray(k1, dtype=np.uint64) & MASK32
    for _ in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & MASK32, lo1, (hi0 ^ c3 ^ k1) & MASK32, lo0
        k0 = (k0 + W0) & MASK32
        k1 = (k1 + W1) & MASK32
    return c0, c1, c2, c3


def dropout_threshold(p: float) -> int:
    """Byte threshold thr8 = round(p * 256) in [1, 255]; 0 = dropout off (philox.cuh)."""
    return 0 if p <= 0 else max(1, min(255, int(p * 256.0 + 0.5)))


def dropout_scale(p: float) -> float:
    t = dropout_threshold(p)
    return 1.0 if t == 0 else 256.0 / (256 - t)


def keep_bytes(seed: int, site: int, call: np.ndarray, byte: np.ndarray, p: float) -> np.ndarray:
    """Keep flag of byte `byte` (0..15) of Philox call `call` of a dropout site."""
    call = np.asarray(call, dtype=np.uint64)
    if p <= 0:
        return np.ones(call.shape, dtype=bool)
    w = philox4x32_10(call & MASK32, call >> np.uint64(32), np.uint64(site & 0xFFFFFFFF),
                      np.uint64(site >> 32), np.uint64(seed & 0xFFFFFFFF), np.uint64(seed >> 32))
    byte = np.asarray(byte, dtype=np.uint64)
    words = np.stack(w, axis=-1)
    word = np.take_along_axis(words, (byte >> np.uint64(2)).astype(np.int64)[..., None], axis=-1)[..., 0]
    b = (word >> (np.uint64(8) * (byte & np.uint64(3)))) & np.uint64(0xFF)
    return b >= np.uint64(dropout_threshold(p))


def keep_mask(seed: int, site: int, index: np.ndarray, p: float) -> np.ndarray:
    """Hidden-state sites: element e uses byte e & 15 of call e >> 4."""
    index = np.asarray(index, dtype=np.uint64)
    return keep_bytes(seed, site, index >> np.uint64(4), index & np.uint64(15), p)


@dataclass
class LayerShape:
    hidden: int
    heads: int
    seq: int
    ffn: int
    window: int = 0  # > 0: Swin-style windowed attention over window-major token groups
    merge: bool = False  # Swin patch merging at the input: [4*seq, hidden/2] -> [seq, hidden]
    causal: bool = False  # decoder self-attention: query q sees keys k <= q
    cross: bool = False   # T5 decoder: + cross-attention sublayer over the memory
    shift: int = 0        # Swin SW-MSA: tokens rolled by -shift around the window attention
    rpb: bool = False     # Swin relative-position bias table [heads][(2 side - 1)^2]
    rms: bool = False     # T5: every LayerNorm of the layer is an RMSNorm (gain only, eps 1e-6)
    relb: int = 0         # T5 relative attention bias: buckets (0 = none), max distance 128

    @property
    def att_seq(self):
        return self.window or self.seq

    @property
    def head_dim(self):
        return self.hidden // self.heads


def merge_rows(seq: int, window: int) -> np.ndarray:
    """Patch merging index (csrc/kernels/patch_merge.cu): [seq, 4] input rows (within a
    sample of 4*seq tokens) gathered for each output token.  Tokens are window-major: token
    (y, x) of a G-grid with windows of side ws is row ((y//ws)*(G//ws) + x//ws)*ws^2 +
    (y%ws)*ws + x%ws; output (y, x) takes inputs (2y+dy, 2x+dx), (dy, dx) = (0,0) (1,0) (0,1)
    (1,1)."""
    g, ws = math.isqrt(seq), math.isqrt(window)
    assert g * g == seq and ws * ws == window and g % ws == 0

    def row(y, x, grid):
        return ((y // ws) * (grid // ws) + x // ws) * ws * ws + (y % ws) * ws + x % ws

    out = np.empty((seq, 4), dtype=np.int64)
    for y in range(g):
        for x in range(g):
            t = row(y, x, g)
            for q, (dy, dx) in enumerate(((0, 0), (1, 0), (0, 1), (1, 1))):
                out[t, q] = row(2 * y + dy, 2 * x + dx, 2 * g)
    return out


def _wm_row(y, x, grid, ws):
    return ((y // ws) * (grid // ws) + x // ws) * ws * ws + (y % ws) * ws + x % ws


def roll_rows(seq: int, window: int, shift: int) -> np.ndarray:
    """Window-major row permutation of torch.roll(grid, (-shift, -shift)): out[t] = in[perm[t]]
    (csrc/kernels/patch_merge.cu window_roll)."""
    g, ws = math.isqrt(seq), math.isqrt(window)
    perm = np.empty(seq, dtype=np.int64)
    for y in range(g):
        for x in range(g):
            perm[_wm_row(y, x, g, ws)] = _wm_row((y + shift) % g, (x + shift) % g, g, ws)
    return perm


def shift_regions(seq: int, window: int, shift: int) -> np.ndarray:
    """[windows, window] region id (0..8) of each token of the rolled grid; SW-MSA lets q
    and k attend only within one region."""
    g, ws = math.isqrt(seq), math.isqrt(window)
    reg = np.empty(seq, dtype=np.int64)
    band = lambda v: 0 if v < g - ws else (1 if v < g - shift else 2)  # noqa: E731
    for y in range(g):
        for x in range(g):
            reg[_wm_row(y, x, g, ws)] = 3 * band(y) + band(x)
    return reg.reshape(seq // window, window)


def rel_index(window: int) -> np.ndarray:
    """[window, window] relative-position index of (q, k) in a side x side window (Swin's
    relative_position_index): (dy + side - 1) * (2 side - 1) + dx + side - 1."""
    w = math.isqrt(window)
    y, x = np.arange(window) // w, np.arange(window) % w
    return (y[:, None] - y[None] + w - 1) * (2 * w - 1) + (x[:, None] - x[None] + w - 1)


def t5_buckets(seq: int, bidirectional: bool, num_buckets: int = 32,
               max_distance: int = 128) -> np.ndarray:
    """T5's relative-position bucket (Raffel et al. 2020; the published
    `_relative_position_bucket` of the T5 implementations) of each relative position
    k - q = d for d in [-(seq-1), seq-1] (index d + seq - 1): |d| < max_exact exact, then
    log-spaced up to max_distance, saturating; bidirectional splits the buckets by sign.
    Computed in float64 (the executor's host code does the same)."""
    d = np.arange(-(seq - 1), seq, dtype=np.int64)
    n = -d  # query - key
    nb = num_buckets
    ret = np.zeros_like(n)
    if bidirectional:
        nb //= 2
        ret = (n < 0).astype(np.int64) * nb
        n = np.abs(n)
    else:
        n = np.maximum(n, 0)
    max_exact = nb // 2
    large = max_exact + (np.log(np.maximum(n, 1) / max_exact) / math.log(max_distance / max_exact)
                         * (nb - max_exact)).astype(np.int64)
    large = np.minimum(large, nb - 1)
    return ret + np.where(n < max_exact, n, large)


def init_layer_params(shape: LayerShape, rng: np.random.Generator, std=0.02) -> dict:
    h, f = shape.hidden, shape.ffn
    if shape.rpb:
        n2 = (2 * math.isqrt(shape.window) - 1) ** 2
        rp = {"rpb": 0.5 * rng.standard_normal((shape.heads, n2))}
    else:
        rp = {}
    if shape.relb:
        rp["relb"] = 0.5 * rng.standard_normal((shape.heads, shape.relb))
    merge = {} if not shape.merge else {
        "mln_g": 1.0 + 0.1 * rng.standard_normal(2 * h), "mln_b": 0.1 * rng.standard_normal(2 * h),
        "w_m": std * rng.standard_normal((h, 2 * h))}
    if shape.cross:
        merge = {
            "ln3_g": 1.0 + 0.1 * rng.standard_normal(h), "ln3_b": 0.1 * rng.standard_normal(h),
            "w_q2": std * rng.standard_normal((h, h)), "b_q2": 0.02 * rng.standard_normal(h),
            "w_kv2": std * rng.standard_normal((2 * h, h)), "b_kv2": 0.02 * rng.standard_normal(2 * h),
            "w_o2": std * rng.standard_normal((h, h)), "b_o2": 0.02 * rng.standard_normal(h)}
    return rp | merge | {
        "ln1_g": 1.0 + 0.1 * rng.standard_normal(h), "ln1_b": 0.1 * rng.standard_normal(h),
        "w_qkv": std * rng.standard_normal((3 * h, h)), "b_qkv": 0.02 * rng.standard_normal(3 * h),
        "w_o": std * rng.standard_normal((h, h)), "b_o": 0.02 * rng.standard_normal(h),
        "ln2_g": 1.0 + 0.1 * rng.standard_normal(h), "ln2_b": 0.1 * rng.standard_normal(h),
        "w_1": std * rng.standard_normal((f, h)), "b_1": 0.02 * rng.standard_normal(f),
        "w_2": std * rng.standard_normal((h, f)), "b_2": 0.02 * rng.standard_normal(h),
    }


def _rms_fwd(x, g, eps=1e-6):
    """T5 RMSNorm: x * rsqrt(mean(x^2) + eps) * g (no centring, no bias)."""
    rstd = 1.0 / np.sqrt((x * x).mean(-1, keepdims=True) + eps)
    xh = x * rstd
    return xh * g, (xh, rstd, True)


def _norm_fwd(x, g, b, rms):
    return _rms_fwd(x, g) if rms else _ln_fwd(x, g, b)


def _ln_fwd(x, g, b, eps=1e-5):
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xh = (x - mu) * rstd
    return xh * g + b, (xh, rstd)


def _ln_bwd(dy, cache, g):
    """LayerNorm (or, for an RMSNorm cache, RMSNorm: no mean term, zero bias gradient)."""
    xh, rstd = cache[0], cache[1]
    rms = len(cache) > 2
    dxh = dy * g
    mean_term = 0.0 if rms else dxh.mean(-1, keepdims=True)
    dx = rstd * (dxh - mean_term - xh * (dxh * xh).mean(-1, keepdims=True))
    return dx, (dy * xh).sum(0), (np.zeros(dy.shape[-1]) if rms else dy.sum(0))


try:  # vectorised erf when scipy is present (CPU-baseline speed); identical math otherwise
    from scipy.special import erf as _erf
except ImportError:  # pragma: no cover
    _erf = np.vectorize(math.erf)


def _gelu(x):
    return 0.5 * x * (1.0 + _erf(x / math.sqrt(2.0)))


def _gelu_grad(x):
    return 0.5 * (1.0 + _erf(x / math.sqrt(2.0))) + x * np.exp(-0.5 * x * x) / math.sqrt(2 * math.pi)


@dataclass
class Dropout:
    p_attn: float = 0.0
    p_hidden: float = 0.0
    seed: int = 1234


def _hidden_mask(drop: Dropout, site: int, rows: int, cols: int, row_offset: int):
    idx = (np.arange(rows, dtype=np.uint64)[:, None] + np.uint64(row_offset)) * np.uint64(cols) + \
        np.arange(cols, dtype=np.uint64)[None, :]
    return keep_mask(drop.seed, site, idx, drop.p_hidden)


def _attn_mask(drop: Dropout, site: int, samples: int, heads: int, seq: int, sample_offset: int,
               heads_total=None, head_offset=0):
    """Attention sites (csrc/kernels/attention.cu): element (q, k) of global (sample, head)
    is byte j of call ((bh*s + q)*ceil(s/64) + k//64)*4 + t, with kk = k % 64,
    t = (kk % 8) // 2, j = (kk // 8) * 2 + kk % 2 and bh = sample*heads_total + head."""
    H = heads_total or heads
    nkb = (seq + 63) // 64
    b = np.arange(samples, dtype=np.uint64)[:, None, None, None] + np.uint64(sample_offset)
    h = np.arange(heads, dtype=np.uint64)[None, :, None, None] + np.uint64(head_offset)
    q = np.arange(seq, dtype=np.uint64)[None, None, :, None]
    k = np.arange(seq, dtype=np.uint64)[None, None, None, :]
    kk = k % np.uint64(64)
    t = (kk % np.uint64(8)) // np.uint64(2)
    j = (kk // np.uint64(8)) * np.uint64(2) + kk % np.uint64(2)
    call = (((b * np.uint64(H) + h) * np.uint64(seq) + q) * np.uint64(nkb) + k // np.uint64(64)) \
        * np.uint64(4) + t
    return keep_bytes(drop.seed, site, call, j, drop.p_attn)


def _attention(q2, k2, v2, n, s, H, d, am, ka, causal):
    """softmax(q k^T / sqrt(d)) (keys k > q masked when causal), dropout, times v."""
    q = q2.reshape(n, s, H, d).transpose(0, 2, 1, 3)
    k = k2.reshape(n, s, H, d).transpose(0, 2, 1, 3)
    v = v2.reshape(n, s, H, d).transpose(0, 2, 1, 3)
    sc = q @ k.transpose(0, 1, 3, 2) / math.sqrt(d)
    if causal:
        sc = np.where(np.triu(np.ones((s, s), dtype=bool), 1), -np.inf, sc)
    sc = sc - sc.max(-1, keepdims=True)
    pr = np.exp(sc)
    pr = pr / pr.sum(-1, keepdims=True)
    pd = pr * am * ka
    ctx = (pd @ v).transpose(0, 2, 1, 3).reshape(n * s, H * d)
    return ctx, dict(q=q, k=k, v=v, pr=pr, am=am, ka=ka, pd=pd)


def _attention_bwd(dctx, c, n, s, H, d):
    """-> dq, dk, dv as [n*s, H*d]."""
    dctx4 = dctx.reshape(n, s, H, d).transpose(0, 2, 1, 3)
    dv = c["pd"].transpose(0, 1, 3, 2) @ dctx4
    dpd = dctx4 @ c["v"].transpose(0, 1, 3, 2)
    dpr = dpd * c["am"] * c["ka"]
    pr = c["pr"]
    dsc = pr * (dpr - (dpr * pr).sum(-1, keepdims=True)) / math.sqrt(d)
    to2 = lambda t: t.transpose(0, 2, 1, 3).reshape(n * s, H * d)  # noqa: E731
    return to2(dsc @ c["k"]), to2(dsc.transpose(0, 1, 3, 2) @ c["q"]), to2(dv)


def cross_sites(layer_id: int, n_layers: int):
    """Philox sites of a decoder layer's cross sublayer (after every layer's 3l+0..2)."""
    return 3 * n_layers + 2 * layer_id, 3 * n_layers + 2 * layer_id + 1


def layer_forward(P: dict, x: np.ndarray, shape: LayerShape, layer_id: int = 0,
                  drop: Dropout = Dropout(), sample_offset: int = 0, memory=None,
                  n_layers: int = 0):
    """x: [samples*seq, h] float64.  Returns (y, cache).  Attention runs per (attention
    sequence, head); an attention sequence is a sample, or one window of a sample (window
    layers: tokens stored window-major, so a window is `window` consecutive rows)."""
    h, H, d, s = shape.hidden, shape.heads, shape.head_dim, shape.att_seq
    mcache = {}
    if shape.merge:  # patch merging: gather 2x2 -> LN(2h) -> x = mln W_m^T
        idx = merge_rows(shape.seq, shape.window)
        ns = x.shape[0] // (4 * shape.seq)
        rows_in = (np.arange(ns)[:, None, None] * 4 * shape.seq + idx[None]).reshape(-1, 4)
        mg = x[rows_in].reshape(ns * shape.seq, 2 * h)
        mln, lnm = _ln_fwd(mg, P["mln_g"], P["mln_b"])
        mcache = dict(rows_in=rows_in, mln=mln, lnm=lnm, x_in_shape=x.shape)
        x = mln @ P["w_m"].T
    n = x.shape[0] // s                      # attention sequences
    nw = shape.seq // s                      # per sample
    a, ln1 = _norm_fwd(x, P["ln1_g"], P["ln1_b"], shape.rms)
    ar, perm = a, None
    if shape.shift:  # SW-MSA: roll the tokens (per sample), attend in windows, roll back
        ns = n // nw
        perm = (np.arange(ns)[:, None] * shape.seq + roll_rows(shape.seq, s, shape.shift)[None]).ravel()
        ar = a[perm]
    qkv = ar @ P["w_qkv"].T + P["b_qkv"]
    q = qkv[:, :h].reshape(n, s, H, d).transpose(0, 2, 1, 3)
    k = qkv[:, h:2 * h].reshape(n, s, H, d).transpose(0, 2, 1, 3)
    v = qkv[:, 2 * h:].reshape(n, s, H, d).transpose(0, 2, 1, 3)
    sc = q @ k.transpose(0, 1, 3, 2) / math.sqrt(d)
    if shape.rpb:
        sc = sc + P["rpb"][:, rel_index(s)][None]
    if shape.relb:  # T5: bias of bucket(k - q), bidirectional unless causal
        bk = t5_buckets(s, not shape.causal, shape.relb)
        rel = (np.arange(s)[None, :] - np.arange(s)[:, None]) + s - 1  # [q, k] -> k - q + s - 1
        sc = sc + P["relb"][:, bk[rel]][None]
    if shape.causal:
        sc = np.where(np.triu(np.ones((s, s), dtype=bool), 1), -np.inf, sc)
    if shape.shift:
        reg = np.tile(shift_regions(shape.seq, s, shape.shift), (n // nw, 1))  # [n, s]
        sc = np.where((reg[:, :, None] != reg[:, None, :])[:, None], -np.inf, sc)
    sc = sc - sc.max(-1, keepdims=True)
    pr = np.exp(sc)
    pr = pr / pr.sum(-1, keepdims=True)
    am = _attn_mask(drop, 3 * layer_id, n, H, s, sample_offset * nw)
    ka = dropout_scale(drop.p_attn)
    pd = pr * am * ka
    ctx4 = pd @ v
    ctx = ctx4.transpose(0, 2, 1, 3).reshape(n * s, h)
    if perm is not None:
        ctx_u = np.empty_like(ctx)
        ctx_u[perm] = ctx
        ctx = ctx_u
    o = ctx @ P["w_o"].T + P["b_o"]
    m1 = _hidden_mask(drop, 3 * layer_id + 1, n * s, h, sample_offset * shape.seq)
    kh = dropout_scale(drop.p_hidden)
    x1 = x + o * m1 * kh
    xcache = {}
    xr = x1
    if shape.cross:  # cross sublayer: q from LN3(x1), k / v from the memory
        sa, sh = cross_sites(layer_id, n_layers)
        c3, ln3 = _norm_fwd(x1, P["ln3_g"], P["ln3_b"], shape.rms)
        q2 = c3 @ P["w_q2"].T + P["b_q2"]
        kv2 = memory @ P["w_kv2"].T + P["b_kv2"]
        am2 = _attn_mask(drop, sa, n, H, s, sample_offset)
        ctx2, ac = _attention(q2, kv2[:, :h], kv2[:, h:], n, s, H, d, am2, ka, False)
        m3 = _hidden_mask(drop, sh, n * s, h, sample_offset * shape.seq)
        xr = x1 + (ctx2 @ P["w_o2"].T + P["b_o2"]) * m3 * kh
        xcache = dict(c3=c3, ln3=ln3, ctx2=ctx2, ac=ac, m3=m3, memory=memory, x2=xr)
    c, ln2 = _norm_fwd(xr, P["ln2_g"], P["ln2_b"], shape.rms)
    pre = c @ P["w_1"].T + P["b_1"]
    g = _gelu(pre)
    z = g @ P["w_2"].T + P["b_2"]
    m2 = _hidden_mask(drop, 3 * layer_id + 2, n * s, h, sample_offset * shape.seq)
    y = xr + z * m2 * kh
    cache = dict(x=x, a=ar, ln1=ln1, perm=perm, q=q, k=k, v=v, pr=pr, am=am, ka=ka, pd=pd, ctx=ctx, m1=m1,
                 kh=kh, x1=x1, c=c, ln2=ln2, pre=pre, g=g, m2=m2, n=n, **mcache, **xcache)
    return y, cache


def layer_backward(P: dict, dy: np.ndarray, cache: dict, shape: LayerShape):
    """Returns (dx, grads dict with the same keys as P)."""
    h, H, d, s = shape.hidden, shape.heads, shape.head_dim, shape.att_seq
    n = cache["n"]
    G = {}
    dz = dy * cache["m2"] * cache["kh"]
    G["b_2"] = dz.sum(0)
    G["w_2"] = dz.T @ cache["g"]
    dg = dz @ P["w_2"]
    dpre = dg * _gelu_grad(cache["pre"])
    G["b_1"] = dpre.sum(0)
    G["w_1"] = dpre.T @ cache["c"]
    dc = dpre @ P["w_1"]
    dx1_ln, G["ln2_g"], G["ln2_b"] = _ln_bwd(dc, cache["ln2"], P["ln2_g"])
    dx1 = dy + dx1_ln
    if shape.cross:  # dx1 so far is dL/dx2: back through the cross sublayer
        dx2 = dx1
        do2 = dx2 * cache["m3"] * cache["kh"]
        G["b_o2"] = do2.sum(0)
        G["w_o2"] = do2.T @ cache["ctx2"]
        dq2, dk2, dv2 = _attention_bwd(do2 @ P["w_o2"], cache["ac"], cache["n"], s, H, d)
        dkv2 = np.concatenate([dk2, dv2], axis=1)
        G["b_q2"], G["w_q2"] = dq2.sum(0), dq2.T @ cache["c3"]
        G["b_kv2"], G["w_kv2"] = dkv2.sum(0), dkv2.T @ cache["memory"]
        G["_dmem"] = dkv2 @ P["w_kv2"]
        dx1_3, G["ln3_g"], G["ln3_b"] = _ln_bwd(dq2 @ P["w_q2"], cache["ln3"], P["ln3_g"])
        dx1 = dx2 + dx1_3
    do = dx1 * cache["m1"] * cache["kh"]
    G["b_o"] = do.sum(0)
    G["w_o"] = do.T @ cache["ctx"]
    dctx = do @ P["w_o"]
    perm = cache["perm"]
    if perm is not None:
        dctx = dctx[perm]
    dctx4 = dctx.reshape(n, s, H, d).transpose(0, 2, 1, 3)
    dv = cache["pd"].transpose(0, 1, 3, 2) @ dctx4
    dpd = dctx4 @ cache["v"].transpose(0, 1, 3, 2)
    dpr = dpd * cache["am"] * cache["ka"]
    pr = cache["pr"]
    dsc = pr * (dpr - (dpr * pr).sum(-1, keepdims=True))
    if shape.rpb:
        idx = rel_index(s).ravel()
        tot = dsc.sum(0).reshape(H, -1)  # [H, s*s]
        G["rpb"] = np.stack([np.bincount(idx, weights=tot[hh], minlength=P["rpb"].shape[1])
                             for hh in range(H)])
    if shape.relb:
        bk = t5_buckets(s, not shape.causal, shape.relb)
        rel = (np.arange(s)[None, :] - np.arange(s)[:, None]) + s - 1
        tot = dsc.sum(0).reshape(H, -1)  # [H, s*s]
        G["relb"] = np.stack([np.bincount(bk[rel].ravel(), weights=tot[hh], minlength=shape.relb)
                              for hh in range(H)])
    dsc = dsc / math.sqrt(d)
    dq = dsc @ cache["k"]
    dk = dsc.transpose(0, 1, 3, 2) @ cache["q"]
    to2 = lambda t: t.transpose(0, 2, 1, 3).reshape(n * s, h)  # noqa: E731
    dqkv = np.concatenate([to2(dq), to2(dk), to2(dv)], axis=1)
    G["b_qkv"] = dqkv.sum(0)
    G["w_qkv"] = dqkv.T @ cache["a"]
    da = dqkv @ P["w_qkv"]
    if perm is not None:
        da_u = np.empty_like(da)
        da_u[perm] = da
        da = da_u
    dx_ln, G["ln1_g"], G["ln1_b"] = _ln_bwd(da, cache["ln1"], P["ln1_g"])
    dx = dx1 + dx_ln
    if shape.merge:
        G["w_m"] = dx.T @ cache["mln"]
        dmln = dx @ P["w_m"]
        dmg, G["mln_g"], G["mln_b"] = _ln_bwd(dmln, cache["lnm"], P["mln_g"])
        dxin = np.zeros(cache["x_in_shape"])
        dxin[cache["rows_in"].ravel()] = dmg.reshape(-1, h // 2)
        dx = dxin
    return dx, G


def model_step(params: list, x: np.ndarray, target: np.ndarray, shape: LayerShape,
               drop: Dropout = Dropout(), sample_offset: int = 0, count=None):
    """Forward through all layers, MSE loss = sum((y-t)^2)/count, backward.
    Returns (loss, y, dx, grads per layer)."""
    shapes = shape if isinstance(shape, (list, tuple)) else [shape] * len(params)
    dec0 = next((l for l, sh in enumerate(shapes) if sh.cross), None)
    caches = []
    hcur = x
    memory = None
    for l, P in enumerate(params):
        if l == dec0:
            memory = hcur  # the first decoder layer's input is every decoder layer's memory
        hcur, c = layer_forward(P, hcur, shapes[l], l, drop, sample_offset, memory, len(params))
        caches.append(c)
    count = count if count is not None else hcur.size
    loss = float(((hcur - target) ** 2).sum() / count)
    dcur = 2.0 * (hcur - target) / count
    grads = [None] * len(params)
    dmem = 0.0
    for l in reversed(range(len(params))):
        dcur, grads[l] = layer_backward(params[l], dcur, caches[l], shapes[l])
        dmem = dmem + grads[l].pop("_dmem", 0.0)
        if l == dec0:
            dcur = dcur + dmem
    return loss, hcur, dcur, grads


def adamw_reference(p, g, m, v, step, lr=1e-4, b1=0.9, b2=0.999, eps=1e-8, wd=0.0):
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    mh = m / (1 - b1 ** step)
    vh = v / (1 - b2 ** step)
    p = p - lr * (mh / (np.sqrt(vh) + eps) + wd * p)
    return p, m, v
