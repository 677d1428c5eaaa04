"""Micro-benchmark: gx tcgen05 GEMM vs cuBLAS (torch.matmul) on the BERT-Huge layer shapes.

Prints one JSON line per shape: TFLOP/s of both and the fraction of MEASURED_PEAKS bf16.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13878_b200 import kernels  # noqa: E402


def timeit(fn, iters=20, warm=3):
    """Device time per call: `iters` calls captured in one CUDA graph (no launch overhead)."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(iters):
                fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (5 * iters)


def main():
    dev = torch.device("cuda:0")
    h = int(os.environ.get("H", 1280))
    res = []
    for M in [512, 1024, 2048, 4096]:
        shapes = [("qkv", M, 3 * h, h, False, False), ("out", M, h, h, False, False),
                  ("up", M, 4 * h, h, False, False), ("down", M, h, 4 * h, False, False),
                  ("dgrad_up", M, h, 4 * h, False, True), ("wgrad_up", 4 * h, h, M, True, True)]
        for name, m, n, k, amn, bmn in shapes:
            A = torch.randn(k, m, device=dev).to(torch.bfloat16) if amn else \
                torch.randn(m, k, device=dev).to(torch.bfloat16)
            B = torch.randn(k, n, device=dev).to(torch.bfloat16) if bmn else \
                torch.randn(n, k, device=dev).to(torch.bfloat16)
            out = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
            ms = timeit(lambda: kernels.gemm(A, B, a_mn_major=amn, b_mn_major=bmn, out=out))
            ms1 = min(timeit(lambda: kernels.gemm(A, B, a_mn_major=amn, b_mn_major=bmn, out=out, tile_n=t))
                      for t in (64, 128, 256))
            At = A.t() if amn else A
            Bt = B if bmn else B.t()
            ms_cublas = timeit(lambda: torch.matmul(At, Bt, out=out))
            fl = 2.0 * m * n * k
            r = {"shape": name, "M": m, "N": n, "K": k, "gx_ms": round(ms, 5),
                 "gx_tflops": round(fl / ms / 1e9, 1), "gx_1cta_tflops": round(fl / ms1 / 1e9, 1), "cublas_tflops": round(fl / ms_cublas / 1e9, 1)}
            print(json.dumps(r), flush=True)
            res.append(r)


if __name__ == "__main__":
    main()
