"""Time the layer GEMM shapes at M tokens under every N-tile option (pick_tile audit)."""
import json
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import kernels as K  # noqa: E402

def timeit(fn, n=20, reps=10):
    """Device time per call: n calls captured in one CUDA graph (no host launch cost)."""
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(n):
                fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (n * reps) * 1e3



def main():
    """Every layer GEMM of BERT-Huge (h 1280, ffn 5120) at M tokens under each N tile
    (0 = the automatic choice; > 0 one CTA per 128 x N tile; < 0 CTA pair per 256 x |N|)."""
    dev, bf = torch.device("cuda:0"), torch.bfloat16
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    h, f = 1280, 5120
    r = lambda *s: torch.randn(*s, device=dev).to(bf)  # noqa: E731
    x, ctx, gel = r(M, h), r(M, h), r(M, f)
    wqkv, wo, w1, w2 = r(3 * h, h), r(h, h), r(f, h), r(h, f)
    dout, dz, dpre, dqkv = r(M, h), r(M, h), r(M, f), r(M, 3 * h)
    bh, bf_ = torch.zeros(h, device=dev).to(bf), torch.zeros(f, device=dev).to(bf)
    o3, oh, of = r(M, 3 * h), r(M, h), r(M, f)
    pre = r(M, f)
    g_qkv, g_o, g_1, g_2 = (torch.empty(3 * h, h, device=dev), torch.empty(h, h, device=dev),
                            torch.empty(f, h, device=dev), torch.empty(h, f, device=dev))
    cs = torch.cuda.current_stream
    shapes = {
        "qkv_fwd": lambda t: K.gemm(x, wqkv, out=o3, tile_n=t, stream=cs()),
        "out_fwd": lambda t: K.gemm(ctx, wo, out=oh, bias=bh, residual=x, dropout_p=0.1, seed=1,
                                    site=1, tile_n=t, stream=cs()),
        "up_fwd": lambda t: K.gemm(x, w1, out=of, bias=bf_, gelu_aux=pre, gelu_mode=2, tile_n=t,
                                   stream=cs()),
        "down_fwd": lambda t: K.gemm(gel, w2, out=oh, bias=bh, residual=x, dropout_p=0.1, seed=1,
                                     site=2, tile_n=t, stream=cs()),
        "dgrad_down": lambda t: K.gemm(dz, w2, b_mn_major=True, out=of, gelu_bwd_aux=pre,
                                       gelu_mode=2, tile_n=t, stream=cs()),
        "dgrad_up": lambda t: K.gemm(dpre, w1, b_mn_major=True, out=oh, tile_n=t, stream=cs()),
        "dgrad_out": lambda t: K.gemm(dout, wo, b_mn_major=True, out=oh, tile_n=t, stream=cs()),
        "dgrad_qkv": lambda t: K.gemm(dqkv, wqkv, b_mn_major=True, out=oh, tile_n=t, stream=cs()),
        "wgrad_down": lambda t: K.gemm(dz, gel, a_mn_major=True, b_mn_major=True, out=g_2,
                                       out_kind="f32", tile_n=t, stream=cs()),
        "wgrad_up": lambda t: K.gemm(dpre, x, a_mn_major=True, b_mn_major=True, out=g_1,
                                     out_kind="f32", tile_n=t, stream=cs()),
        "wgrad_out": lambda t: K.gemm(dout, ctx, a_mn_major=True, b_mn_major=True, out=g_o,
                                      out_kind="f32", tile_n=t, stream=cs()),
        "wgrad_qkv": lambda t: K.gemm(dqkv, x, a_mn_major=True, b_mn_major=True, out=g_qkv,
                                      out_kind="f32", tile_n=t, stream=cs()),
    }
    for name, fn in shapes.items():
        res = {}
        for t in (0, 64, 128, 256, -128, -160, -256):
            try:
                res[t] = round(timeit(lambda: fn(t)), 2)
            except Exception as e:  # unsupported combination
                res[t] = str(e)[:40]
        best = min((v, k) for k, v in res.items() if isinstance(v, float))
        print(json.dumps({"M": M, "gemm": name, "auto_us": res[0], "best": best[1],
                          "best_us": best[0], "us_by_tile": res}), flush=True)


if __name__ == "__main__":
    main()
