import sys, torch
sys.path.insert(0, ".")
from paper_2211_13878_b200 import kernels
dev = torch.device("cuda:0")
torch.manual_seed(0)
for (M, N, K, bn, amn, bmn) in [(128, 128, 512, 64, False, False), (128, 128, 512, 0, False, False), (128,128,512,128,False,False),
                                (256, 128, 512, 64, False, False), (128, 384, 128, 64, False, False), (128, 512, 512, 64, True, True),
                                (512, 1280, 5120, 0, False, False), (128, 128, 1024, 64, False, False)]:
    A = torch.randn(K, M, device=dev).bfloat16() if amn else torch.randn(M, K, device=dev).bfloat16()
    B = torch.randn(K, N, device=dev).bfloat16() if bmn else torch.randn(N, K, device=dev).bfloat16()
    ref = (A.float().t() if amn else A.float()) @ (B.float() if bmn else B.float().t())
    bad = 0
    worst = 0.0
    for it in range(300):
        C = kernels.gemm(A, B, a_mn_major=amn, b_mn_major=bmn, tile_n=bn)
        e = ((C.float() - ref).norm() / ref.norm()).item()
        worst = max(worst, e)
        if e > 1e-2:
            bad += 1
    torch.cuda.synchronize()
    print(M, N, K, bn, amn, bmn, "bad", bad, "of 300 worst", worst, flush=True)
