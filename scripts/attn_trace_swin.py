"""Per-CTA phase medians of the tcgen05 attention forward at the Swin stage-0 shape (49-token
windows packed two per tile, head_dim 32, relative-position bias): where a small tile's time goes."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import kernels as K  # noqa: E402
dev = torch.device("cuda:0")
n, s, H, d = 8 * 64, 49, 10, 32
qkv = (torch.randn(n * s, 3 * H * d, device=dev) * 0.5).to(torch.bfloat16)
tab = torch.randn(H, 13 * 13, device=dev).to(torch.bfloat16)
tiles = (n + 1) // 2
tr = torch.zeros(tiles * H * 32, dtype=torch.int64, device=dev)
for i in range(3):
    K.attention_fwd(qkv, n, s, H, d, p=0.1, seed=1, rpb=tab, trace=tr if i == 2 else None)
torch.cuda.synchronize()
t = tr.view(-1, 32).cpu().double()
t0 = t[:, 0][t[:, 0] > 0].min()
rel = (t - t0) / 1000.0
dur = (t[:, 5] - t[:, 0]) / 1000.0
print(json.dumps({"ctas": int((t[:, 0] > 0).sum()), "span_us": round(float(rel[:, 5].max()), 2),
                  "per_cta_us": {n_: round(float(((t[:, i] - t[:, 0]) / 1000.0).median()), 2) for i, n_ in
                                 enumerate(["entry", "pdl", "s_ready", "max_done", "p_done", "o_ready"])},
                  "cta_total_median_us": round(float(dur.median()), 2)}))

# backward: stamps 0 entry, 1 pdl, 2 prologue done, 4 chunk-0 scores ready, 5 softmax done,
# 7 Pd / dS stored, 25 epilogue done, 26 cluster barrier passed, 27 exit
ctx, lse, mask = K.attention_fwd(qkv, n, s, H, d, p=0.1, seed=1, rpb=tab)
dctx = torch.randn(n * s, H * d, device=dev).to(torch.bfloat16)
dpart = torch.empty(n * H * 169, device=dev)
trb = torch.zeros(tiles * H * 32, dtype=torch.int64, device=dev)
for i in range(3):
    K.attention_bwd(qkv, ctx, lse, dctx, n, s, H, d, p=0.1, seed=1, mask=mask, rpb=tab,
                    rpb_dpart=dpart, trace=trb if i == 2 else None)
torch.cuda.synchronize()
t = trb.view(-1, 32).cpu().double()
names = {0: "entry", 1: "pdl", 2: "prologue_done", 4: "s_ready", 5: "softmax_done",
         7: "pds_stored", 25: "epi_done", 26: "cluster_synced", 27: "exit"}
print(json.dumps({"bwd_per_cta_us": {n_: round(float(((t[:, i] - t[:, 0]) / 1000.0).median()), 2)
                                     for i, n_ in names.items()}}))
