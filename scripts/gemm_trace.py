"""Per-CTA phase timeline of one CTA-pair GEMM launch (globaltimer stamps, ns):
entry, after-PDL, first-TMA, first-stage, last-MMA-issued, first-acc-ready, epi-done, exit."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import kernels as K  # noqa: E402
dev = torch.device("cuda:0")
bf = torch.bfloat16
names = ["entry", "pdl", "tma0", "stage0", "mma_last", "acc0", "epi_done", "exit", "c0", "c0ld", "c1", "c1ld", "blk0_math0", "blk0_math1", "blk0_staged", "blk0_stored"]
Mt = int(sys.argv[1]) if len(sys.argv) > 1 else 512
shapes = {"up_fwd(gelu)": (Mt, 5120, 1280, False, "gelu"), "qkv_fwd": (Mt, 3840, 1280, False, None),
          "dgrad_down(gelu_bwd)": (Mt, 5120, 1280, True, "gelu_bwd"), "out_fwd plain": (Mt, 1280, 1280, False, None),
          "out_fwd residual+dropout": (Mt, 1280, 1280, False, "residual"),
          "up_fwd plain": (Mt, 5120, 1280, False, None)}
for name, (M, N, Kd, bmn, epi) in shapes.items():
    A = (torch.randn(M, Kd, device=dev) * 0.5).to(bf)
    B = (torch.randn(Kd, N, device=dev) if bmn else torch.randn(N, Kd, device=dev)).to(bf) * 0.05
    aux = torch.randn(M, N, device=dev).to(bf)
    bias = torch.randn(N, device=dev).to(bf)
    tr = torch.zeros(148 * 16, dtype=torch.int64, device=dev)
    kw = {}
    if epi == "gelu":
        kw = dict(bias=bias, gelu_aux=aux)
    elif epi == "gelu_bwd":
        kw = dict(gelu_bwd_aux=aux)
    elif epi == "residual":
        kw = dict(bias=bias, residual=aux, dropout_p=0.1, seed=1, site=1)
    for i in range(4):
        K.gemm(A, B, b_mn_major=bmn, trace=tr if i == 3 else None, **kw)
    torch.cuda.synchronize()
    t = tr.view(148, 16).cpu()
    used = t[:, 0] > 0
    if not bool(used.any()):
        print(json.dumps({"gemm": name, "trace": "none (1-CTA kernel)"}))
        continue
    t = t[used].double()
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0  # us
    med = [float(rel[t[:, i] > 0, i].median()) if (t[:, i] > 0).any() else None for i in range(8)]
    # slots 8..15 are SM clock cycles (epilogue warp 4, lane 0), relative to slot 8
    cyc = (t[:, 8:16] - t[:, 8:9]).median(dim=0).values.tolist()
    med += [round(c) for c in cyc]
    print(json.dumps({"gemm": name, "ctas": int(used.sum()),
                      "median_us(0-7) / cycles(8-15)": {n: round(v, 2) for n, v in zip(names, med) if v is not None}}), flush=True)
