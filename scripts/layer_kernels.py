"""Graph-timed device time of every kernel of one BERT-Huge layer step at M = B*s tokens.

Each kernel is captured 20x back to back in one CUDA graph (replayed 5x), so the number is
its steady-state cost inside a graph (launch overhead amortised, PDL overlap included).
Usage: python scripts/layer_kernels.py [M=512]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import kernels as K  # noqa: E402
from scripts.bench_gemm import timeit  # noqa: E402


def main():
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    h, f, s, H, hd = 1280, 5120, 512, 20, 64
    B = M // s
    dev = torch.device("cuda:0")
    bf = torch.bfloat16
    r = lambda *sh: (torch.randn(*sh, device=dev) * 0.5).to(bf)
    x, ln, ctx, dout, dz = r(M, h), r(M, h), r(M, h), r(M, h), r(M, h)
    qkv, dqkv = r(M, 3 * h), r(M, 3 * h)
    gel, pre, dpre = r(M, f), r(M, f), r(M, f)
    wqkv, wo, w1, w2 = r(3 * h, h), r(h, h), r(f, h), r(h, f)
    b3, bh, bf_ = r(3 * h), r(h), r(f)
    outs = {k: torch.empty(*v, device=dev, dtype=bf) for k, v in
            {"qkv": (M, 3 * h), "h": (M, h), "f": (M, f)}.items()}
    g32 = {k: torch.empty(*v, device=dev, dtype=torch.float32) for k, v in
           {"wqkv": (3 * h, h), "wo": (h, h), "w1": (f, h), "w2": (h, f), "mh": (M, h)}.items()}
    d = K.make_dropout(0.1, 1234, 1, drop_ld=h)
    rows = []

    only = os.environ.get("ONLY")  # run just this kernel 3x, untimed (for ncu captures)

    def add(name, flops, fn, bytes_=0):
        if only is not None:
            if only in name:
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
            return
        ms = timeit(fn)
        rows.append({"kernel": name, "us": round(ms * 1e3, 2),
                     "tflops": round(flops / ms / 1e9, 1) if flops else None,
                     "gbs": round(bytes_ / ms / 1e6, 1) if bytes_ else None})
        print(json.dumps(rows[-1]), flush=True)

    F = lambda m, n, k: 2.0 * m * n * k
    # forward
    add("ln_fwd", 0, lambda: K.layernorm_fwd(x, b3[:h], bh), 4 * M * h)
    add("qkv_fwd", F(M, 3 * h, h), lambda: K.gemm(ln, wqkv, out=outs["qkv"], bias=b3))
    add("attn_fwd", 4.0 * B * H * s * s * hd, lambda: K.attention_fwd(qkv, B, s, H, hd, p=0.1, seed=1))
    add("out_fwd(bias+drop+res)", F(M, h, h),
        lambda: K.gemm(ctx, wo, out=outs["h"], bias=bh, residual=x, dropout_p=0.1, seed=1, site=1))
    add("up_fwd(bias+gelu)", F(M, f, h), lambda: K.gemm(ln, w1, out=outs["f"], bias=bf_, gelu_aux=pre,
                                                         gelu_mode=2))  # as the executor
    add("down_fwd(bias+drop+res)", F(M, h, f),
        lambda: K.gemm(gel, w2, out=outs["h"], bias=bh, residual=x, dropout_p=0.1, seed=1, site=2))
    add("down_fwd splitk", F(M, h, f), lambda: K.gemm_splitk(gel, w2, out=g32["mh"]))
    # backward
    add("dropout_bwd_colsum", 0, lambda: K.dropout_bwd_colsum(dout, d), 4 * M * h)
    add("wgrad_down dW2", F(h, f, M), lambda: K.gemm(dz, gel, a_mn_major=True, b_mn_major=True,
                                                     out=g32["w2"], out_kind="f32"))
    add("dgrad_down(gelu_bwd)", F(M, f, h),
        lambda: K.gemm(dz, w2, b_mn_major=True, out=outs["f"], gelu_bwd_aux=pre, gelu_mode=2))
    add("wgrad_up dW1", F(f, h, M), lambda: K.gemm(dpre, ln, a_mn_major=True, b_mn_major=True,
                                                   out=g32["w1"], out_kind="f32"))
    add("dgrad_up splitk", F(M, h, f), lambda: K.gemm_splitk(dpre, w1, b_mn_major=True, out=g32["mh"]))
    add("dgrad_up bf16", F(M, h, f), lambda: K.gemm(dpre, w1, b_mn_major=True, out=outs["h"]))
    add("ln_bwd", 0, lambda: K.layernorm_bwd(dout, x, torch.zeros(M, device=dev),
                                             torch.ones(M, device=dev), bh, dres=dz), 8 * M * h)
    add("wgrad_out dWo", F(h, h, M), lambda: K.gemm(dout, ctx, a_mn_major=True, b_mn_major=True,
                                                    out=g32["wo"], out_kind="f32"))
    add("dgrad_out", F(M, h, h), lambda: K.gemm(dout, wo, b_mn_major=True, out=outs["h"]))
    ctx_, lse, mask = K.attention_fwd(qkv, B, s, H, hd, p=0.1, seed=1)
    add("attn_bwd", 10.0 * B * H * s * s * hd,
        lambda: K.attention_bwd(qkv, ctx_, lse, ctx, B, s, H, hd, p=0.1, seed=1, mask=mask))
    add("wgrad_qkv dWqkv", F(3 * h, h, M), lambda: K.gemm(dqkv, ln, a_mn_major=True, b_mn_major=True,
                                                          out=g32["wqkv"], out_kind="f32"))
    add("dgrad_qkv splitk", F(M, h, 3 * h),
        lambda: K.gemm_splitk(dqkv, wqkv, b_mn_major=True, out=g32["mh"]))
    n = 19_676_160
    p32 = torch.zeros(n, device=dev)
    add("adamw (1 layer)", 0, lambda: K.adamw(p32, p32, p32, p32, torch.empty(n, device=dev, dtype=bf),
                                              1e-4, 0.9, 0.999, 1e-8, 0.0, 1), 30 * n)
    if only is not None:
        return
    tot = sum(r_["us"] for r_ in rows if "splitk" not in r_["kernel"] or "down_fwd" in r_["kernel"])
    print(json.dumps({"M": M, "sum_us_listed": round(tot, 1)}))


if __name__ == "__main__":
    main()
