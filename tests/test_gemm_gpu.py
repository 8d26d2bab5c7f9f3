"""tcgen05 GEMM parity: every majorness/group/epilogue combination against a
torch fp32 matmul of the same bf16 operands (the kernel computes bf16 x bf16
with fp32 accumulation, so the only difference is summation order)."""
import pytest
import torch

from paper_2602_04816_b200 import _lib as L

pytestmark = pytest.mark.gpu


def _desc(M, N, K, A, B, C, a_mn, b_mn, G=1, kgroup=0, a_grouped=0, b_grouped=0, epi=L.EPI_F32,
          R=None):
    d = L.HlmGemmDesc()
    d.M, d.N, d.K, d.G, d.kgroup = M, N, K, G, kgroup
    d.a_mn, d.b_mn, d.a_grouped, d.b_grouped, d.epi = a_mn, b_mn, a_grouped, b_grouped, epi
    d.A = A.data_ptr(); d.lda = A.shape[-1]; d.a_gstride = A[0].numel() if a_grouped else 0
    d.B = B.data_ptr(); d.ldb = B.shape[-1]; d.b_gstride = B[0].numel() if b_grouped else 0
    d.C = C.data_ptr(); d.ldc = C.shape[-1]
    d.c_gstride = C[0].numel() if (G > 1 and not kgroup) else 0
    if R is not None:
        d.R = R.data_ptr(); d.ldr = R.shape[-1]; d.r_gstride = d.c_gstride
    return d


def _ref(A, B, a_mn, b_mn):
    a = A.float().t() if a_mn else A.float()   # (M,K)
    b = B.float() if b_mn else B.float().t()   # (K,N)
    return a @ b


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 520, 200), (8, 11, 8), (1024, 768, 1536),
                                   (4, 16, 8)])
def test_gemm_single(a_mn, b_mn, M, N, K):
    torch.manual_seed(M * 7 + N + K)
    dev = "cuda"
    # ld padded to a multiple of 8 elements (16 B) as TMA requires
    def mk(rows, cols):
        ld = (cols + 7) // 8 * 8
        t = torch.randn(rows, ld, device=dev).to(torch.bfloat16)
        t[:, cols:] = 0
        return t, ld
    A, _ = mk(K, M) if a_mn else mk(M, K)
    B, _ = mk(K, N) if b_mn else mk(N, K)
    Av = A[:, :M] if a_mn else A[:, :K]
    Bv = B[:, :N] if b_mn else B[:, :K]
    C = torch.full((M, N), float("nan"), device=dev)
    d = _desc(M, N, K, A, B, C, a_mn, b_mn)
    L.gemm(d)
    torch.cuda.synchronize()
    ref = _ref(Av, Bv, a_mn, b_mn)
    err = (C - ref).abs().max().item()
    assert err <= 1e-3 * ref.abs().max().item() + 1e-4, err


def test_gemm_bf16_and_residual():
    dev = "cuda"
    M, N, K = 512, 512, 256
    A = torch.randn(M, K, device=dev).bfloat16()
    B = torch.randn(K, N, device=dev).bfloat16()
    C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    L.gemm(_desc(M, N, K, A, B, C, 0, 1, epi=L.EPI_BF16))
    ref = A.float() @ B.float()
    assert torch.allclose(C.float(), ref, rtol=1e-2, atol=1e-2)
    R = torch.randn(M, N, device=dev)
    C2 = R.clone()
    L.gemm(_desc(M, N, K, A, B, C2, 0, 1, epi=L.EPI_F32_ADD, R=C2))
    torch.cuda.synchronize()
    assert torch.allclose(C2, R + ref, rtol=1e-4, atol=1e-3)


def test_gemm_groups():
    dev = "cuda"
    T, h = 384, 256
    X = torch.randn(T, h, device=dev).bfloat16()
    W = (torch.randn(3, h, h, device=dev) * 0.05).bfloat16()    # w_q|w_k|w_v (in,out)
    # N-grouped forward: Y[g] = X . W[g]
    Y = torch.empty(3, T, h, device=dev)
    L.gemm(_desc(T, h, h, X, W, Y, 0, 1, G=3, b_grouped=1))
    for g in range(3):
        ref = X.float() @ W[g].float()
        assert torch.allclose(Y[g], ref, rtol=1e-3, atol=1e-3)
    # K-grouped dgrad: D = sum_g dY[g] . W[g]^T
    dY = torch.randn(3, T, h, device=dev).bfloat16()
    D = torch.empty(T, h, device=dev)
    L.gemm(_desc(T, h, h, dY, W, D, 0, 0, G=3, kgroup=1, a_grouped=1, b_grouped=1))
    ref = sum(dY[g].float() @ W[g].float().t() for g in range(3))
    assert torch.allclose(D, ref, rtol=1e-3, atol=1e-3)
    # N-grouped wgrad: dW[g] = X^T . dY[g]
    dW = torch.empty(3, h, h, device=dev)
    L.gemm(_desc(h, h, T, X, dY, dW, 1, 1, G=3, b_grouped=1))
    torch.cuda.synchronize()
    for g in range(3):
        ref = X.float().t() @ dY[g].float()
        assert torch.allclose(dW[g], ref, rtol=1e-3, atol=1e-2)
