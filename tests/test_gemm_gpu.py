"""tcgen05 GEMM parity against a plain PyTorch fp32 reference of the same op.

Tolerance (bf16 output, fp32 accumulate): ||C - C_ref||_2 / ||C_ref||_2 <= 1e-2 and
max |C - C_ref| <= 2e-2 * max|C_ref| + 1e-3.
"""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _rel(x, ref):
    return ((x.float() - ref).norm() / ref.norm().clamp_min(1e-30)).item()


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, True), (True, False)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (512, 3840, 1280), (520, 480, 160),
                                   (1024, 1280, 5120), (256, 200, 72), (1280, 5120, 512),
                                   (776, 640, 1280)])
@pytest.mark.parametrize("tile_n", [0, 64, 128, 256, -128, -256, -160])
def test_gemm_layouts(cuda, a_mn, b_mn, M, N, K, tile_n):
    from paper_2211_13878_b200 import kernels
    if tile_n == -160 and b_mn:
        pytest.skip("N tile 160 is for K-major B only")
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, generator=g).to(cuda, torch.bfloat16)
    B = torch.randn(N, K, generator=g).to(cuda, torch.bfloat16)
    ref = A.float() @ B.float().t()
    a_arg = A.t().contiguous() if a_mn else A
    b_arg = B.t().contiguous() if b_mn else B
    C = kernels.gemm(a_arg, b_arg, a_mn_major=a_mn, b_mn_major=b_mn, tile_n=tile_n)
    torch.cuda.synchronize()
    assert _rel(C, ref) <= 1e-2
    assert (C.float() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item() + 1e-3


def test_gemm_f32_accumulate(cuda):
    from paper_2211_13878_b200 import kernels
    g = torch.Generator(device="cpu").manual_seed(5)
    M, N, K = 1280, 3840, 512
    dY = torch.randn(K, N, generator=g).to(cuda, torch.bfloat16)   # tokens x out
    X = torch.randn(K, M, generator=g).to(cuda, torch.bfloat16)    # tokens x in
    # weight gradient dW[N, M] = dY^T X, accumulated twice
    out = torch.zeros(N, M, device=cuda, dtype=torch.float32)
    kernels.gemm(dY, X, a_mn_major=True, b_mn_major=True, out=out, out_kind="f32_acc")
    kernels.gemm(dY, X, a_mn_major=True, b_mn_major=True, out=out, out_kind="f32_acc")
    ref = 2.0 * (dY.float().t() @ X.float())
    torch.cuda.synchronize()
    assert _rel(out, ref) <= 1e-5


def test_gemm_bias_gelu(cuda):
    from paper_2211_13878_b200 import kernels
    g = torch.Generator(device="cpu").manual_seed(6)
    M, N, K = 512, 5120, 1280
    X = torch.randn(M, K, generator=g).to(cuda, torch.bfloat16)
    W = (0.03 * torch.randn(N, K, generator=g)).to(cuda, torch.bfloat16)
    b = torch.randn(N, generator=g).to(cuda, torch.bfloat16)
    pre = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    y = kernels.gemm(X, W, bias=b, gelu_aux=pre)
    ref_pre = X.float() @ W.float().t() + b.float()
    ref = torch.nn.functional.gelu(pre.float())
    torch.cuda.synchronize()
    assert _rel(pre, ref_pre) <= 1e-2
    assert _rel(y, ref) <= 1e-2


def test_gemm_gelu_derivative_mode(cuda):
    """gelu == 2 writes gelu'(pre) as the aux output; gelu_bwd == 2 multiplies by it."""
    from paper_2211_13878_b200 import kernels
    g = torch.Generator(device="cpu").manual_seed(16)
    M, N, K = 512, 5120, 1280
    X = torch.randn(M, K, generator=g).to(cuda, torch.bfloat16)
    W = (0.03 * torch.randn(N, K, generator=g)).to(cuda, torch.bfloat16)
    b = torch.randn(N, generator=g).to(cuda, torch.bfloat16)
    dgel = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    y = kernels.gemm(X, W, bias=b, gelu_aux=dgel, gelu_mode=2)
    pre = (X.float() @ W.float().t() + b.float()).to(torch.bfloat16).float().requires_grad_(True)
    ref = torch.nn.functional.gelu(pre)
    ref.backward(torch.ones_like(ref))
    torch.cuda.synchronize()
    assert _rel(y, ref.detach()) <= 1e-2
    assert _rel(dgel, pre.grad) <= 1e-2
    # backward: out = (dY W2-like product) * aux
    dZ = torch.randn(M, 1280, generator=g).to(cuda, torch.bfloat16)
    W2 = (0.03 * torch.randn(1280, N, generator=g)).to(cuda, torch.bfloat16)
    out = kernels.gemm(dZ, W2, b_mn_major=True, gelu_bwd_aux=dgel, gelu_mode=2)
    ref2 = (dZ.float() @ W2.float()) * dgel.float()
    torch.cuda.synchronize()
    assert _rel(out, ref2) <= 1e-2


def test_gemm_residual_dropout(cuda):
    from paper_2211_13878_b200 import kernels
    g = torch.Generator(device="cpu").manual_seed(7)
    M, N, K = 512, 1280, 1280
    X = torch.randn(M, K, generator=g).to(cuda, torch.bfloat16)
    W = (0.03 * torch.randn(N, K, generator=g)).to(cuda, torch.bfloat16)
    b = torch.randn(N, generator=g).to(cuda, torch.bfloat16)
    R = torch.randn(M, N, generator=g).to(cuda, torch.bfloat16)
    y0 = kernels.gemm(X, W, bias=b, residual=R)
    ref0 = R.float() + (X.float() @ W.float().t() + b.float())
    torch.cuda.synchronize()
    assert _rel(y0, ref0) <= 1e-2
    y1 = kernels.gemm(X, W, bias=b, residual=R, dropout_p=0.1, seed=1234, site=9)
    dropped = ((y1.float() - R.float()).abs() < 1e-6).float().mean().item()
    assert 0.08 < dropped < 0.12


@pytest.mark.parametrize("M,N,K,b_mn", [(512, 1280, 5120, False), (512, 1280, 3840, True),
                                         (128, 256, 512, False), (2048, 1280, 5120, True),
                                         (520, 640, 1000, False)])
@pytest.mark.parametrize("splits,tile", [(0, 0), (3, -256), (5, -128), (4, 128), (7, 64)])
def test_gemm_splitk(cuda, M, N, K, b_mn, splits, tile):
    from paper_2211_13878_b200 import kernels
    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    A = torch.randn(M, K, generator=g).to(cuda, torch.bfloat16)
    B = torch.randn(N, K, generator=g).to(cuda, torch.bfloat16)
    ref = A.float() @ B.float().t()
    b_arg = B.t().contiguous() if b_mn else B
    out = kernels.gemm_splitk(A, b_arg, b_mn_major=b_mn, splits=splits, tile_n=tile)
    torch.cuda.synchronize()
    assert _rel(out, ref) <= 1e-5
