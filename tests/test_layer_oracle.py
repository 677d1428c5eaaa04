"""Pins the CPU layer oracle (oracle/layer_oracle.py) before it is trusted as the checker.

The reference has no layer implementation, so the numpy restatement is pinned against
torch.autograd in float64 on CPU (an independent implementation of the same math, with the
same Philox dropout masks), against Philox known-answer vectors (Random123 KAT), and
against the committed golden vectors in tests/golden/layer_small.npz.
"""
import math
import os

import numpy as np
import pytest
import torch

from oracle import layer_oracle as lo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "layer_small.npz")


def test_philox_known_answers():
    # Random123 philox4x32-10 known-answer tests (kat_vectors)
    out = lo.philox4x32_10(0, 0, 0, 0, 0, 0)
    assert [int(v) for v in out] == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    out = lo.philox4x32_10(0xffffffff, 0xffffffff, 0xffffffff, 0xffffffff, 0xffffffff, 0xffffffff)
    assert [int(v) for v in out] == [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]
    out = lo.philox4x32_10(0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344, 0xa4093822, 0x299f31d0)
    assert [int(v) for v in out] == [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]


def test_dropout_rate():
    idx = np.arange(400_000, dtype=np.uint64)
    keep = lo.keep_mask(1234, 7, idx, 0.1)
    assert lo.dropout_threshold(0.1) == 26
    assert abs(1.0 - keep.mean() - 26 / 256) < 0.003
    m = lo._attn_mask(lo.Dropout(0.1, 0.0, 5), 0, 2, 3, 200, 1)
    assert abs(1.0 - m.mean() - 26 / 256) < 0.005


def _torch_merge(x, P, shape):
    """Swin PatchMerging written with reshapes (independent of lo.merge_rows): window-major
    -> raster grid, x0..x3 = x[0::2,0::2], x[1::2,0::2], x[0::2,1::2], x[1::2,1::2], concat,
    raster -> window-major, LayerNorm, projection."""
    h = shape.hidden
    c, g2 = h // 2, math.isqrt(shape.seq)
    g, ws = 2 * g2, math.isqrt(shape.window)
    n = x.shape[0] // (g * g)
    r = x.reshape(n, g // ws, g // ws, ws, ws, c).permute(0, 1, 3, 2, 4, 5).reshape(n, g, g, c)
    m = torch.cat([r[:, 0::2, 0::2], r[:, 1::2, 0::2], r[:, 0::2, 1::2], r[:, 1::2, 1::2]], -1)
    m = m.reshape(n, g2 // ws, ws, g2 // ws, ws, 4 * c).permute(0, 1, 3, 2, 4, 5)
    m = m.reshape(n * g2 * g2, 4 * c)
    m = torch.nn.functional.layer_norm(m, (4 * c,), P["mln_g"], P["mln_b"], 1e-5)
    return m @ P["w_m"].T


def _wm_to_raster(t, g, ws):
    c = t.shape[-1]
    n = t.shape[0] // (g * g)
    return t.reshape(n, g // ws, g // ws, ws, ws, c).permute(0, 1, 3, 2, 4, 5).reshape(n, g, g, c)


def _raster_to_wm(t, ws):
    n, g, _, c = t.shape
    return t.reshape(n, g // ws, ws, g // ws, ws, c).permute(0, 1, 3, 2, 4, 5).reshape(n * g * g, c)


def _swin_attn_mask(g, ws, sh):
    """Swin's SW-MSA mask, built the way the Swin reference does (img_mask slices)."""
    img = torch.zeros(1, g, g, 1)
    cnt = 0
    for hs in (slice(0, -ws), slice(-ws, -sh), slice(-sh, None)):
        for wsl in (slice(0, -ws), slice(-ws, -sh), slice(-sh, None)):
            img[:, hs, wsl, :] = cnt
            cnt += 1
    mw = _raster_to_wm(img, ws).reshape(-1, ws * ws)
    return mw[:, None, :] != mw[:, :, None]  # [nW, win, win] True = masked


def _torch_mha(q2, k2, v2, n, s, H, d, am, ka, causal, mask=None, bias=None):
    q, k, v = (t.reshape(n, s, H, d).transpose(1, 2) for t in (q2, k2, v2))
    sc = q @ k.transpose(-1, -2) / math.sqrt(d)
    if bias is not None:
        sc = sc + bias[None]
    if causal:
        sc = sc.masked_fill(torch.ones(s, s, dtype=torch.bool).triu(1), -math.inf)
    if mask is not None:
        sc = sc.masked_fill(mask[:, None], -math.inf)
    pr = torch.softmax(sc, -1)
    return (pr * am * ka @ v).transpose(1, 2).reshape(n * s, H * d)


def _torch_layer(P, x, shape, drop, layer_id=0, sample_offset=0, memory=None, n_layers=0):
    if shape.merge:
        x = _torch_merge(x, P, shape)
    h, H, d, s = shape.hidden, shape.heads, shape.head_dim, shape.att_seq
    n = x.shape[0] // s
    nw, S = shape.seq // s, shape.seq
    if shape.rms:  # T5LayerNorm: hidden * rsqrt(mean(hidden^2) + eps) * weight
        ln = lambda t, g, b: t * torch.rsqrt(t.pow(2).mean(-1, keepdim=True) + 1e-6) * g  # noqa: E731
    else:
        ln = lambda t, g, b: torch.nn.functional.layer_norm(t, (h,), g, b, 1e-5)  # noqa: E731
    a = ln(x, P["ln1_g"], P["ln1_b"])
    qkv = a @ P["w_qkv"].T + P["b_qkv"]
    am = torch.from_numpy(lo._attn_mask(drop, 3 * layer_id, n, H, s, sample_offset * nw)).double()
    ka = lo.dropout_scale(drop.p_attn)
    mask = None
    bias = None
    if shape.rpb:  # Swin's relative_position_index, built the Swin way (coords meshgrid)
        w = math.isqrt(s)
        coords = torch.stack(torch.meshgrid(torch.arange(w), torch.arange(w), indexing="ij")).flatten(1)
        rel = (coords[:, :, None] - coords[:, None, :]).permute(1, 2, 0) + (w - 1)
        rpi = rel[:, :, 0] * (2 * w - 1) + rel[:, :, 1]
        bias = P["rpb"][:, rpi]  # [H, s, s]
    if shape.relb:  # T5's own bucketing (transformers' T5Attention), bidirectional unless causal
        from transformers.models.t5.modeling_t5 import T5Attention
        rp = torch.arange(s)[None, :] - torch.arange(s)[:, None]  # memory - query position
        bk = T5Attention._relative_position_bucket(rp, bidirectional=not shape.causal,
                                                   num_buckets=shape.relb, max_distance=128)
        bias = P["relb"][:, bk]  # [H, s, s]
    if shape.shift:
        g, ws, sh = math.isqrt(S), math.isqrt(s), shape.shift
        a = _raster_to_wm(torch.roll(_wm_to_raster(a, g, ws), (-sh, -sh), (1, 2)), ws)
        qkv = a @ P["w_qkv"].T + P["b_qkv"]
        mask = _swin_attn_mask(g, ws, sh).repeat(n // nw, 1, 1)
    ctx = _torch_mha(qkv[:, :h], qkv[:, h:2 * h], qkv[:, 2 * h:], n, s, H, d, am, ka, shape.causal,
                     mask, bias)
    if shape.shift:
        ctx = _raster_to_wm(torch.roll(_wm_to_raster(ctx, g, ws), (sh, sh), (1, 2)), ws)
    kh = lo.dropout_scale(drop.p_hidden)
    m1 = torch.from_numpy(lo._hidden_mask(drop, 3 * layer_id + 1, n * s, h, sample_offset * S)).double()
    x1 = x + (ctx @ P["w_o"].T + P["b_o"]) * m1 * kh
    if shape.cross:
        sa, sh = lo.cross_sites(layer_id, n_layers)
        q2 = ln(x1, P["ln3_g"], P["ln3_b"]) @ P["w_q2"].T + P["b_q2"]
        kv2 = memory @ P["w_kv2"].T + P["b_kv2"]
        am2 = torch.from_numpy(lo._attn_mask(drop, sa, n, H, s, sample_offset)).double()
        ctx2 = _torch_mha(q2, kv2[:, :h], kv2[:, h:], n, s, H, d, am2, ka, False)
        m3 = torch.from_numpy(lo._hidden_mask(drop, sh, n * s, h, sample_offset * S)).double()
        x1 = x1 + (ctx2 @ P["w_o2"].T + P["b_o2"]) * m3 * kh
    c = ln(x1, P["ln2_g"], P["ln2_b"])
    g = torch.nn.functional.gelu(c @ P["w_1"].T + P["b_1"])
    m2 = torch.from_numpy(lo._hidden_mask(drop, 3 * layer_id + 2, n * s, h, sample_offset * S)).double()
    return x1 + (g @ P["w_2"].T + P["b_2"]) * m2 * kh


@pytest.mark.parametrize("p,window,seq,merge,shift,rpb", [
    (0.0, 0, 12, False, 0, False), (0.1, 0, 12, False, 0, False), (0.1, 4, 12, False, 0, False),
    (0.1, 4, 16, True, 0, False), (0.0, 9, 36, True, 0, False), (0.1, 9, 36, False, 1, False),
    (0.0, 16, 64, False, 2, False), (0.1, 4, 16, True, 1, False), (0.1, 9, 36, False, 1, True),
    (0.0, 4, 16, True, 0, True)])
def test_oracle_matches_autograd(p, window, seq, merge, shift, rpb):
    rng = np.random.default_rng(0)
    shape = lo.LayerShape(hidden=64, heads=4, seq=seq, ffn=128, window=window, merge=merge,
                          shift=shift, rpb=rpb)
    P = lo.init_layer_params(shape, rng, std=0.1)
    x = rng.standard_normal((2 * shape.seq * (4 if merge else 1), shape.hidden // (2 if merge else 1)))
    dy = rng.standard_normal((2 * shape.seq, shape.hidden))
    drop = lo.Dropout(p_attn=p, p_hidden=p, seed=99)
    y, cache = lo.layer_forward(P, x, shape, 0, drop, sample_offset=3)
    dx, G = lo.layer_backward(P, dy, cache, shape)

    tP = {k: torch.tensor(v, requires_grad=True) for k, v in P.items()}
    tx = torch.tensor(x, requires_grad=True)
    ty = _torch_layer(tP, tx, shape, drop, 0, 3)
    ty.backward(torch.tensor(dy))
    assert np.allclose(y, ty.detach().numpy(), rtol=1e-10, atol=1e-10)
    assert np.allclose(dx, tx.grad.numpy(), rtol=1e-9, atol=1e-10)
    for k in P:
        assert np.allclose(G[k], tP[k].grad.numpy(), rtol=1e-9, atol=1e-10), k


def test_golden_vectors():
    """Committed outputs of the oracle (tests/golden/make_layer_golden.py)."""
    z = np.load(GOLDEN)
    shape = lo.LayerShape(*[int(v) for v in z["shape"]])
    P = {k[2:]: z[k] for k in z.files if k.startswith("P_")}
    drop = lo.Dropout(float(z["p"]), float(z["p"]), int(z["seed"]))
    y, cache = lo.layer_forward(P, z["x"], shape, 1, drop, 0)
    dx, G = lo.layer_backward(P, z["dy"], cache, shape)
    assert np.allclose(y, z["y"], rtol=0, atol=1e-12)
    assert np.allclose(dx, z["dx"], rtol=0, atol=1e-12)
    for k in G:
        assert np.allclose(G[k], z["G_" + k], rtol=0, atol=1e-12)



@pytest.mark.parametrize("p", [0.0, 0.1])
def test_t5_encoder_decoder_model_matches_autograd(p):
    """Encoder + causal decoder layers with cross-attention over the memory (the first decoder
    layer's input), MSE loss: loss, dx and every parameter gradient vs torch.autograd."""
    rng = np.random.default_rng(5)
    enc = lo.LayerShape(hidden=32, heads=2, seq=8, ffn=64)
    dec = lo.LayerShape(hidden=32, heads=2, seq=8, ffn=64, causal=True, cross=True)
    shapes = [enc, enc, dec, dec]
    params = [lo.init_layer_params(sh, rng, std=0.2) for sh in shapes]
    x = rng.standard_normal((3 * 8, 32))
    t = rng.standard_normal((3 * 8, 32))
    drop = lo.Dropout(p, p, 21)
    loss, y, dx, grads = lo.model_step(params, x, t, shapes, drop, sample_offset=2)

    tP = [{k: torch.tensor(v, requires_grad=True) for k, v in P.items()} for P in params]
    tx = torch.tensor(x, requires_grad=True)
    hcur, mem = tx, None
    for l, sh in enumerate(shapes):
        if sh.cross and mem is None:
            mem = hcur
        hcur = _torch_layer(tP[l], hcur, sh, drop, l, 2, mem, len(shapes))
    tl = ((hcur - torch.tensor(t)) ** 2).sum() / hcur.numel()
    tl.backward()
    assert abs(loss - tl.item()) <= 1e-10 * abs(loss)
    assert np.allclose(y, hcur.detach().numpy(), rtol=1e-10, atol=1e-12)
    assert np.allclose(dx, tx.grad.numpy(), rtol=1e-8, atol=1e-12)
    for l in range(len(shapes)):
        assert set(grads[l]) == set(params[l])
        for k in params[l]:
            assert np.allclose(grads[l][k], tP[l][k].grad.numpy(), rtol=1e-8, atol=1e-12), (l, k)


def test_t5_buckets_match_transformers():
    """lo.t5_buckets equals the published T5 bucketing (transformers' T5Attention) over every
    relative position of a 512-token sequence, both directions."""
    from transformers.models.t5.modeling_t5 import T5Attention
    for bi in (True, False):
        d = torch.arange(-511, 512)
        hf = T5Attention._relative_position_bucket(d, bidirectional=bi, num_buckets=32,
                                                   max_distance=128).numpy()
        assert np.array_equal(hf, lo.t5_buckets(512, bi, 32)), bi


@pytest.mark.parametrize("p", [0.0, 0.1])
def test_t5_rmsnorm_relative_bias_model_matches_autograd(p):
    """T5 layers proper: RMSNorm everywhere and the bucketed relative attention bias (40
    tokens: exact and log-spaced buckets), encoder (bidirectional) + causal decoder with
    cross-attention; loss, dx and every parameter gradient vs torch.autograd."""
    rng = np.random.default_rng(8)
    enc = lo.LayerShape(hidden=32, heads=2, seq=40, ffn=64, rms=True, relb=32)
    dec = lo.LayerShape(hidden=32, heads=2, seq=40, ffn=64, causal=True, cross=True, rms=True,
                        relb=32)
    shapes = [enc, dec]
    params = [lo.init_layer_params(sh, rng, std=0.2) for sh in shapes]
    x = rng.standard_normal((2 * 40, 32))
    t = rng.standard_normal((2 * 40, 32))
    drop = lo.Dropout(p, p, 23)
    loss, y, dx, grads = lo.model_step(params, x, t, shapes, drop, sample_offset=1)

    tP = [{k: torch.tensor(v, requires_grad=True) for k, v in P.items()} for P in params]
    tx = torch.tensor(x, requires_grad=True)
    hcur, mem = tx, None
    for l, sh in enumerate(shapes):
        if sh.cross and mem is None:
            mem = hcur
        hcur = _torch_layer(tP[l], hcur, sh, drop, l, 1, mem, len(shapes))
    tl = ((hcur - torch.tensor(t)) ** 2).sum() / hcur.numel()
    tl.backward()
    assert abs(loss - tl.item()) <= 1e-10 * abs(loss)
    assert np.allclose(y, hcur.detach().numpy(), rtol=1e-10, atol=1e-12)
    assert np.allclose(dx, tx.grad.numpy(), rtol=1e-8, atol=1e-12)
    for l in range(len(shapes)):
        for k in params[l]:
            ref = tP[l][k].grad
            ref = np.zeros(params[l][k].shape) if ref is None else ref.numpy()  # RMSNorm: no beta
            assert np.allclose(grads[l][k], ref, rtol=1e-8, atol=1e-12), (l, k)
