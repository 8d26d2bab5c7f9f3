"""Throughput of the tcgen05 GEMM at the C2 (Qwen2.5-7B-shaped) block shapes vs torch/cuBLAS."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_04816_b200 import _lib as L

def desc(M, N, K, A, B, C, a_mn, b_mn, G=1, kgroup=0, ag=0, bg=0, epi=L.EPI_BF16):
    d = L.HlmGemmDesc()
    d.M, d.N, d.K, d.G, d.kgroup, d.a_mn, d.b_mn, d.a_grouped, d.b_grouped, d.epi = M, N, K, G, kgroup, a_mn, b_mn, ag, bg, epi
    d.A, d.lda, d.a_gstride = A.data_ptr(), A.shape[-1], (A[0].numel() if ag else 0)
    d.B, d.ldb, d.b_gstride = B.data_ptr(), B.shape[-1], (B[0].numel() if bg else 0)
    d.C, d.ldc, d.c_gstride = C.data_ptr(), C.shape[-1], (C[0].numel() if (G > 1 and not kgroup) else 0)
    return d

def timeit(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it / 1e3

T, h, f = 16384, 3584, 18944
dev = "cuda"
bf = torch.bfloat16
X = torch.randn(T, h, device=dev, dtype=bf)
Wqkv = torch.randn(3, h, h, device=dev, dtype=bf)
Wug = torch.randn(2, h, f, device=dev, dtype=bf)
Wd = torch.randn(f, h, device=dev, dtype=bf)
Act = torch.randn(T, f, device=dev, dtype=bf)
dQKV = torch.randn(3, T, h, device=dev, dtype=bf)
dUG = torch.randn(2, T, f, device=dev, dtype=bf)
Y3 = torch.empty(3, T, h, device=dev, dtype=bf)
Y2 = torch.empty(2, T, f, device=dev, dtype=bf)
Yh = torch.empty(T, h, device=dev, dtype=torch.float32)
Yf = torch.empty(T, f, device=dev, dtype=bf)
dW3 = torch.empty(3, h, h, device=dev, dtype=torch.float32)
dW2 = torch.empty(2, h, f, device=dev, dtype=torch.float32)
dWd = torch.empty(f, h, device=dev, dtype=torch.float32)
cases = [
  ("fwd qkv  [N-grp3]", desc(T, h, h, X, Wqkv, Y3, 0, 1, G=3, bg=1), 2*T*h*h*3, lambda: torch.matmul(X, Wqkv.view(3*h, h).t())),
  ("fwd up|gate [N-grp2]", desc(T, f, h, X, Wug, Y2, 0, 1, G=2, bg=1), 2*T*h*f*2, lambda: torch.matmul(X, Wug.view(2*h, f)[:h])),
  ("fwd down", desc(T, h, f, Act, Wd, Yh, 0, 1, epi=L.EPI_F32), 2*T*h*f, lambda: torch.matmul(Act, Wd)),
  ("dgrad down (d_act)", desc(T, f, h, X, Wd, Yf, 0, 0), 2*T*h*f, lambda: torch.matmul(X, Wd.t())),
  ("dgrad up|gate [K-grp2]", desc(T, h, f, dUG, Wug, Yh, 0, 0, G=2, kgroup=1, ag=1, bg=1, epi=L.EPI_F32), 2*T*h*f*2, None),
  ("dgrad qkv [K-grp3]", desc(T, h, h, dQKV, Wqkv, Yh, 0, 0, G=3, kgroup=1, ag=1, bg=1, epi=L.EPI_F32), 2*T*h*h*3, None),
  ("wgrad qkv [N-grp3]", desc(h, h, T, X, dQKV, dW3, 1, 1, G=3, bg=1, epi=L.EPI_F32), 2*T*h*h*3, lambda: torch.matmul(X.t(), dQKV[0])),
  ("wgrad up|gate [N-grp2]", desc(h, f, T, X, dUG, dW2, 1, 1, G=2, bg=1, epi=L.EPI_F32), 2*T*h*f*2, None),
  ("wgrad down", desc(f, h, T, Act, X, dWd, 1, 1, epi=L.EPI_F32), 2*T*h*f, lambda: torch.matmul(Act.t(), X)),
]
only = os.environ.get("GEMM_CASE")   # substring filter, e.g. GEMM_CASE="wgrad down"
for name, d, flops, ref in cases:
    if only and only not in name:
        continue
    t = timeit(lambda: L.gemm(d))
    line = f"{name:26s} {t*1e3:8.3f} ms  {flops/t/1e12:7.1f} TFLOP/s"
    if ref is not None:
        tr = timeit(ref)
        # the torch reference covers one group only for grouped cases
        rf = flops / (3 if 'qkv' in name and 'wgrad' in name else 1)
        if 'up|gate' in name and 'fwd' in name: rf = flops / 2
        line += f"   | torch/cuBLAS {rf/tr/1e12:7.1f} TFLOP/s"
    print(line, flush=True)
