"""Attention cost split: device time with and without dropout (the Philox share), B = 1 / 4,
plus the forward's per-CTA phase medians (globaltimer stamps).  python scripts/attn_probe.py"""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import kernels as K  # noqa: E402
from scripts.tile_sweep import timeit  # noqa: E402
dev = torch.device("cuda:0")
s, H, d = 512, 20, 64
for B in (1, 4):
    qkv = (torch.randn(B * s, 3 * H * d, device=dev) * 0.5).to(torch.bfloat16)
    dctx = torch.randn(B * s, H * d, device=dev).to(torch.bfloat16)
    for p in (0.1, 0.0):
        ctx, lse, mask = K.attention_fwd(qkv, B, s, H, d, p=p, seed=1)
        tf = timeit(lambda: K.attention_fwd(qkv, B, s, H, d, p=p, seed=1, mask=mask))
        tb = timeit(lambda: K.attention_bwd(qkv, ctx, lse, dctx, B, s, H, d, p=p, seed=1, mask=mask))
        nq = 4
        trf = torch.zeros(nq * B * H * 32, dtype=torch.int64, device=dev)
        for i in range(3):
            K.attention_fwd(qkv, B, s, H, d, p=p, seed=1, mask=mask, trace=trf if i == 2 else None)
        torch.cuda.synchronize()
        t = trf.view(-1, 32).cpu().double()
        t0 = t[:, 0][t[:, 0] > 0].min()
        ph = {n: round(float((t[:, i] - t0).median()) / 1000, 2) for i, n in
              enumerate(["entry", "pdl", "s_ready", "max_done", "p_done", "o_ready"])}
        ph["exit_max"] = round(float((t[:, 5] - t0).max()) / 1000, 2)
        print(json.dumps({"B": B, "p": p, "fwd_us": round(tf, 2),
                          "bwd_us": round(tb, 2), "fwd_phases_us": ph}), flush=True)
