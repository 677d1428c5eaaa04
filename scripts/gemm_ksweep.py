"""Fixed-overhead vs per-k-block cost of the GEMM kernels (graph-timed device time)."""
import json, sys
import torch
sys.path.insert(0, ".")
from paper_2211_13878_b200 import kernels
from scripts.bench_gemm import timeit
dev = torch.device("cuda:0")
for M, N in [(512, 5120), (2048, 5120), (512, 1280)]:
    for tn in (-256, -128, 256, 128, 64):
        row = []
        for K in (64, 256, 640, 1280, 2560, 5120):
            A = torch.randn(M, K, device=dev).bfloat16()
            B = torch.randn(N, K, device=dev).bfloat16()
            out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
            ms = timeit(lambda: kernels.gemm(A, B, out=out, tile_n=tn))
            row.append(round(ms * 1e3, 2))
        print(json.dumps({"M": M, "N": N, "tile_n": tn, "us_for_K_64_256_640_1280_2560_5120": row}), flush=True)
