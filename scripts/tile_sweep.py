"""Time the layer GEMM shapes at M = 512 tokens under every N-tile option (pick_tile audit)."""
import json, os, sys
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
    dev, bf = torch.device("cuda:0"), torch.bfloat16
    M, h, f = 512, 1280, 5120


    r = lambda *s: torch.randn(*s, device=dev).to(bf)  # noqa: E731
    x, ctx, gel = r(M, h), r(M, h), r(M, f)
    wqkv, wo, w1, w2 = r(3 * h, h), r(h, h), r(f, h), r(h, f)
    dout, dz, dpre = r(M, h), r(M, h), r(M, f)
    bh = torch.zeros(h, device=dev).to(bf)
    o3, oh, of = r(M, 3 * h), r(M, h), r(M, f)
    shapes = {
        "qkv_fwd": lambda t: K.gemm(x, wqkv, out=o3, tile_n=t, stream=torch.cuda.current_stream()),
        "out_fwd": lambda t: K.gemm(ctx, wo, out=oh, bias=bh, residual=x, dropout_p=0.1, seed=1,
                                    site=1, tile_n=t, stream=torch.cuda.current_stream()),
        "up_fwd": lambda t: K.gemm(x, w1, out=of, tile_n=t, stream=torch.cuda.current_stream()),
        "dgrad_out": lambda t: K.gemm(dout, wo, b_mn_major=True, out=oh, tile_n=t,
                                      stream=torch.cuda.current_stream()),
        "dgrad_down": lambda t: K.gemm(dz, w2, b_mn_major=True, out=of, tile_n=t,
                                       stream=torch.cuda.current_stream()),
    }
    for name, fn in shapes.items():
        res = {}
        for t in (0, 64, 128, 256, -128, -256, -160):
            try:
                res[t] = round(timeit(lambda: fn(t)), 2)
            except Exception as e:  # unsupported combination
                res[t] = str(e)[:40]
        print(json.dumps({"gemm": name, "us_by_tile": res}), flush=True)


if __name__ == "__main__":
    main()
