"""Device time of the window attention (Swin stage-0 shapes) under its mask / bias variants."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import kernels as K  # noqa: E402
from scripts.tile_sweep import timeit  # noqa: E402

dev = torch.device("cuda:0")
grid, ws, H, d, samples = 56, 7, 10, 32, 8
n, s, n2 = samples * (grid // ws) ** 2, ws * ws, (2 * ws - 1) ** 2
qkv = torch.randn(n * s, 3 * H * d, device=dev).to(torch.bfloat16)
dctx = torch.randn(n * s, H * d, device=dev).to(torch.bfloat16)
tab = torch.randn(H, n2, device=dev).to(torch.bfloat16)
dpart = torch.empty(n * H * n2, device=dev)
for name, kw in [("plain", {}), ("shift", {"win": (grid, ws, 3)}), ("rpb", {"rpb": tab}),
                 ("shift+rpb", {"win": (grid, ws, 3), "rpb": tab})]:
    ctx, lse, mask = K.attention_fwd(qkv, n, s, H, d, p=0.1, seed=1, **kw)
    fwd = timeit(lambda: K.attention_fwd(qkv, n, s, H, d, p=0.1, seed=1, mask=mask, **kw))
    bkw = dict(kw)
    if "rpb" in kw:
        bkw["rpb_dpart"] = dpart
    bwd = timeit(lambda: K.attention_bwd(qkv, ctx, lse, dctx, n, s, H, d, p=0.1, seed=1,
                                         mask=mask, **bkw))
    print(json.dumps({"variant": name, "fwd_us": round(fwd, 1), "bwd_us": round(bwd, 1)}), flush=True)
