"""Per-chunk epilogue cost probe: one tile, K=64, N = 32..256 valid columns."""
import json, sys
import torch
sys.path.insert(0, ".")
from paper_2211_13878_b200 import kernels
from scripts.bench_gemm import timeit
dev = torch.device("cuda:0")
for tn, M in ((-256, 256), (256, 128)):
    row = []
    for N in (32, 64, 128, 256):
        A = torch.randn(M, 64, device=dev).bfloat16()
        B = torch.randn(N, 64, device=dev).bfloat16()
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        row.append(round(timeit(lambda: kernels.gemm(A, B, out=out, tile_n=tn)) * 1e3, 2))
    print(json.dumps({"tile": tn, "M": M, "us_for_N_32_64_128_256": row}))
# empty-ish kernels for reference: torch fill of small tensor
x = torch.empty(16, device=dev)
print(json.dumps({"torch_fill_us": round(timeit(lambda: x.fill_(1.0)) * 1e3, 2)}))
