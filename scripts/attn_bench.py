"""Device time of the tcgen05 attention forward / backward at the BASELINE shapes
(graph-replayed, preallocated buffers; one JSON line per shape).

FLOP per call: forward 4 s^2 hd per (sequence, head), backward 2.5x that
(five s x s x hd products).  Usage: python scripts/attn_bench.py
"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import _lib  # noqa: E402
from paper_2211_13878_b200 import kernels as K  # noqa: E402
from scripts.tile_sweep import timeit  # noqa: E402

dev = torch.device("cuda:0")
SHAPES = [  # (name, sequences, seq, heads, head_dim, kw)
    ("bert-huge B=1", 1, 512, 20, 64, {}),
    ("bert-huge B=4", 4, 512, 20, 64, {}),
    ("bert-huge B=2 (sdp:8 per GPU)", 2, 512, 20, 64, {}),
    ("vit-huge B=4", 4, 257, 16, 80, {}),
    ("t5 causal B=2", 2, 512, 16, 64, {"causal": True}),
    ("t5 encoder relb B=2", 2, 512, 16, 64, {"relb": True}),
    ("t5 decoder causal+relb B=2", 2, 512, 16, 64, {"causal": True, "relb": True}),
    ("swin stage0 8 samples (W-MSA+rpb)", 8 * 64, 49, 10, 32, {"rpb": True}),
]


def run(name, n, s, H, d, kw):
    qkv = (torch.randn(n * s, 3 * H * d, device=dev) * 0.5).to(torch.bfloat16)
    dctx = torch.randn(n * s, H * d, device=dev).to(torch.bfloat16)
    ctx = torch.empty(n * s, H * d, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(n * H, s, device=dev)
    mask = K.attention_mask_buffer(n, s, H, dev)
    dqkv = torch.zeros_like(qkv)
    dq_acc = torch.empty(((s + 127) // 128) * (n + 1) * H * ((s + 3) // 4 * 4) * d, device=dev)
    dsum = torch.zeros(n * H * s, device=dev)
    extra = {}
    tab = dpart = None
    if kw.get("rpb"):
        side = int(round(s ** 0.5))
        tab = torch.randn(H, (2 * side - 1) ** 2, device=dev).to(torch.bfloat16)
        dpart = torch.empty(n * H * (2 * side - 1) ** 2, device=dev)
        extra = {"rpb": tab, "rpb_dpart": dpart}
    if kw.get("causal"):
        extra["causal"] = True
    if kw.get("relb"):  # 32-bucket table; any in-range bucket map times the same
        extra["relb"] = torch.randn(H, 32, device=dev).to(torch.bfloat16)
        extra["relb_map"] = torch.tensor([min(abs(t) // 16, 31) for t in range(1 - s, s)],
                                         dtype=torch.int8, device=dev)
        extra["relb_dpart"] = torch.empty(n * H * ((s + 127) // 128) * (2 * s - 1), device=dev)
    a = K._attn_args(qkv, n, s, H, d, 0.1, 1234, 3, **extra)
    a.ctx, a.ld_ctx, a.lse, a.mask = K._ptr(ctx), ctx.stride(0), K._ptr(lse), K._ptr(mask)
    a.dctx, a.dqkv, a.dq_accum, a.dsum = K._ptr(dctx), K._ptr(dqkv), K._ptr(dq_acc), K._ptr(dsum)
    lib = _lib.lib()

    def fwd():
        _lib.check(lib.gx_k_attention_fwd(ctypes.addressof(a), _lib.stream_ptr()))

    def bwd():
        _lib.check(lib.gx_k_attention_bwd(ctypes.addressof(a), _lib.stream_ptr()))

    fwd()
    torch.cuda.synchronize()
    tf = timeit(fwd)
    tb = timeit(bwd)
    flop = 4.0 * n * H * s * s * d
    print(json.dumps({"shape": name, "fwd_us": round(tf, 2), "bwd_us": round(tb, 2),
                      "fwd_tflops": round(flop / tf / 1e6, 1),
                      "bwd_tflops": round(2.5 * flop / tb / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    for sh in SHAPES:
        run(*sh)
