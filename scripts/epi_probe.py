"""Out-projection GEMM epilogue cost by stage (bias, residual, Philox dropout) at M = 512..8192."""
import json, os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2211_13878_b200 import kernels as K
from scripts.tile_sweep import timeit
dev, bf = torch.device("cuda:0"), torch.bfloat16
h = 1280
for M in (512, 2048, 8192):
    r = lambda *s: torch.randn(*s, device=dev).to(bf)
    ctx, wo, x, oh = r(M, h), r(h, h), r(M, h), r(M, h)
    bh = torch.zeros(h, device=dev).to(bf)
    cur = torch.cuda.current_stream
    res = {}
    res["plain"] = timeit(lambda: K.gemm(ctx, wo, out=oh, stream=cur()))
    res["bias"] = timeit(lambda: K.gemm(ctx, wo, out=oh, bias=bh, stream=cur()))
    res["bias+res"] = timeit(lambda: K.gemm(ctx, wo, out=oh, bias=bh, residual=x, stream=cur()))
    res["bias+res+drop"] = timeit(lambda: K.gemm(ctx, wo, out=oh, bias=bh, residual=x, dropout_p=0.1, seed=1, site=1, stream=cur()))
    print(json.dumps({"M": M, **{k: round(v, 2) for k, v in res.items()}}), flush=True)
