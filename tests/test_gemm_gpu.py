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


_SCHED_SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
from paper_2602_04816_b200 import _lib as L
from test_gemm_gpu import _desc
torch.manual_seed(5)
dev = "cuda"
out = {{}}
# 8 x 16 = 128 pair tiles (more than the 74 pairs: several tiles per pair), plain + residual
M, N, K = 2048, 4096, 512
A = torch.randn(M, K, device=dev).bfloat16()
B = torch.randn(N, K, device=dev).bfloat16()
R = torch.randn(M, N, device=dev)
C = torch.empty(M, N, device=dev)
L.gemm(_desc(M, N, K, A, B, C, 0, 0))
out["plain"] = C.clone()
L.gemm(_desc(M, N, K, A, B, C, 0, 0, epi=L.EPI_F32_ADD, R=R))
out["resid"] = C.clone()
# N-grouped (3 outputs) and K-grouped (2 K groups) with MN-major operands
G = 3
Bg = torch.randn(G, K, 1024, device=dev).bfloat16()
Cg = torch.empty(G, M, 1024, device=dev)
L.gemm(_desc(M, 1024, K, A, Bg, Cg, 0, 1, G=G, b_grouped=1))
out["ngroup"] = Cg.clone()
Ak = torch.randn(2, M, K, device=dev).bfloat16()
Bk = torch.randn(2, 1024, K, device=dev).bfloat16()
Ck = torch.empty(M, 1024, device=dev)
L.gemm(_desc(M, 1024, K, Ak, Bk, Ck, 0, 0, G=2, kgroup=1, a_grouped=1, b_grouped=1))
out["kgroup"] = Ck.clone()
torch.cuda.synchronize()
torch.save({{k: v.cpu() for k, v in out.items()}}, sys.argv[1])
"""


def test_dynamic_tile_schedule_is_bitwise_identical(tmp_path):
    """HLM_GEMM_DYNAMIC=1 (CTA pairs claim tiles from a per-launch counter) computes every
    tile exactly as the static stride does: same tiles, same k order, bitwise-equal C."""
    import os
    import subprocess
    import sys
    tests = os.path.dirname(os.path.abspath(__file__))
    script = tmp_path / "s.py"
    script.write_text(_SCHED_SCRIPT.format(root=os.path.dirname(tests), tests=tests))
    outs = {}
    for name, env in (("static", {"HLM_GEMM_DYNAMIC": "0"}), ("dynamic", {"HLM_GEMM_DYNAMIC": "1"})):
        path = tmp_path / f"{name}.pt"
        subprocess.run([sys.executable, str(script), str(path)], check=True, timeout=300,
                       env={**os.environ, **env})
        outs[name] = torch.load(path)
    for key, v in outs["static"].items():
        assert torch.equal(v, outs["dynamic"][key]), key
        assert torch.isfinite(v).all(), key
