"""One Swin stage-0 window-attention forward + backward (an ncu target)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import kernels as K  # noqa: E402
dev = torch.device("cuda:0")
n, s, H, d = 8 * 64, 49, 10, 32
qkv = (torch.randn(n * s, 3 * H * d, device=dev) * 0.5).to(torch.bfloat16)
dctx = torch.randn(n * s, H * d, device=dev).to(torch.bfloat16)
tab = torch.randn(H, 13 * 13, device=dev).to(torch.bfloat16)
dpart = torch.empty(n * H * 169, device=dev)
for _ in range(2):
    ctx, lse, mask = K.attention_fwd(qkv, n, s, H, d, p=0.1, seed=1, rpb=tab)
    K.attention_bwd(qkv, ctx, lse, dctx, n, s, H, d, p=0.1, seed=1, mask=mask, rpb=tab, rpb_dpart=dpart)
torch.cuda.synchronize()
