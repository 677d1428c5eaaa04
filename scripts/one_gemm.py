"""Runs a few launches of one GEMM shape (for ncu captures)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2211_13878_b200 import kernels
M, N, K = (int(v) for v in sys.argv[1:4])
amn = len(sys.argv) > 4 and sys.argv[4] == "1"
bmn = len(sys.argv) > 5 and sys.argv[5] == "1"
tn = int(sys.argv[6]) if len(sys.argv) > 6 else 0
dev = torch.device("cuda:0")
A = (torch.randn(K, M, device=dev) if amn else torch.randn(M, K, device=dev)).bfloat16()
B = (torch.randn(K, N, device=dev) if bmn else torch.randn(N, K, device=dev)).bfloat16()
out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
for _ in range(5):
    kernels.gemm(A, B, a_mn_major=amn, b_mn_major=bmn, out=out, tile_n=tn)
torch.cuda.synchronize()
