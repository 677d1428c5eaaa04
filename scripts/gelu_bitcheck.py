"""Bit-identity check of the GeLU forward epilogue between two libgx builds: run once per
build (argv[1] = tag), saving y and gelu'(pre); `compare` checks the saved pairs are equal."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import kernels as K  # noqa: E402

out = "gpurun_out/gelu_bits"
os.makedirs(out, exist_ok=True)
if sys.argv[1] == "compare":
    a, b = torch.load(f"{out}/old.pt"), torch.load(f"{out}/new.pt")
    for k in a:
        same = torch.equal(a[k].view(torch.int16), b[k].view(torch.int16))
        print(k, "bit-identical" if same else f"DIFFERS in {(a[k] != b[k]).sum().item()} elements")
    sys.exit(0)
torch.manual_seed(0)
dev = torch.device("cuda:0")
res = {}
for M, N, Kd in [(512, 5120, 1280), (2048, 5120, 1280), (200, 384, 256)]:
    X = (torch.randn(M, Kd, device=dev) * 0.5).to(torch.bfloat16)
    W = (torch.randn(N, Kd, device=dev) * 0.05).to(torch.bfloat16)
    b = (torch.randn(N, device=dev) * 0.5).to(torch.bfloat16)
    aux = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    y = K.gemm(X, W, bias=b, gelu_aux=aux, gelu_mode=2)
    torch.cuda.synchronize()
    res[f"y_{M}"], res[f"d_{M}"] = y.cpu(), aux.cpu()
torch.save(res, f"{out}/{sys.argv[1]}.pt")
