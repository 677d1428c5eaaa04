"""Per-CTA phase timeline of the tcgen05 attention backward (globaltimer stamps, us)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import kernels as K  # noqa: E402
dev = torch.device("cuda:0")
B, s, H, d = int(os.environ.get("B", 1)), 512, int(os.environ.get("H", 20)), 64
kw = {}
if os.environ.get("CAUSAL"):
    kw["causal"] = True
if os.environ.get("RELB"):  # T5 relative bias (any in-range bucket map times the same)
    kw["relb"] = torch.randn(H, 32, device=dev).to(torch.bfloat16)
    kw["relb_map"] = torch.tensor([min(abs(t) // 16, 31) for t in range(1 - s, s)],
                                  dtype=torch.int8, device=dev)
qkv = (torch.randn(B * s, 3 * H * d, device=dev) * 0.5).to(torch.bfloat16)
dctx = torch.randn(B * s, H * d, device=dev).to(torch.bfloat16)
ctx, lse, mask = K.attention_fwd(qkv, B, s, H, d, p=0.1, seed=1, **kw)
if "relb" in kw:
    kw["relb_dpart"] = torch.empty(B * H * 4 * (2 * s - 1), device=dev)
ncta = 4 * B * H
tr = torch.zeros(ncta * 32, dtype=torch.int64, device=dev)
for i in range(4):
    K.attention_bwd(qkv, ctx, lse, dctx, B, s, H, d, p=0.1, seed=1, mask=mask,
                    trace=tr if i == 3 else None, **kw)
torch.cuda.synchronize()
t = tr.view(ncta, 32).cpu().double()
t0 = t[:, 0][t[:, 0] > 0].min()
names = {0: "entry", 1: "pdl", 2: "prologue_done", 25: "epi_done", 26: "cluster_synced", 27: "exit"}
for j in range(4):
    for k, n in enumerate(["s_ready", "softmax_done", "mma_issued", "mm_done", "dq_stored"]):
        names[4 + 5 * j + k] = f"c{j}_{n}"
out = {}
for i, n in sorted(names.items()):
    col = t[:, i]
    col = col[col > 0]
    if len(col):
        out[n] = round(float((col - t0).median()) / 1000, 2)
print(json.dumps(out))

# forward: stamps 0 entry, 1 pdl, 2 S ready, 3 row max exchanged, 4 P + sums done, 5 O ready
nq = (s + 127) // 128
trf = torch.zeros(nq * B * H * 32, dtype=torch.int64, device=dev)
for i in range(4):
    K.attention_fwd(qkv, B, s, H, d, p=0.1, seed=1, trace=trf if i == 3 else None,
                    **{k: v for k, v in kw.items() if k != "relb_dpart"})
torch.cuda.synchronize()
t = trf.view(-1, 32).cpu().double()
t0 = t[:, 0][t[:, 0] > 0].min()
print(json.dumps({n: round(float((t[:, i] - t0).median()) / 1000, 2) for i, n in
                  enumerate(["entry", "pdl", "s_ready", "max_done", "p_done", "o_ready"])}))
