"""One BERT-Huge attention forward + backward (B from argv, default 1) -- an ncu target."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import kernels as K  # noqa: E402
dev = torch.device("cuda:0")
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
s, H, d = 512, 20, 64
qkv = (torch.randn(B * s, 3 * H * d, device=dev) * 0.5).to(torch.bfloat16)
dctx = torch.randn(B * s, H * d, device=dev).to(torch.bfloat16)
for _ in range(2):
    ctx, lse, mask = K.attention_fwd(qkv, B, s, H, d, p=0.1, seed=1)
    K.attention_bwd(qkv, ctx, lse, dctx, B, s, H, d, p=0.1, seed=1, mask=mask)
torch.cuda.synchronize()
