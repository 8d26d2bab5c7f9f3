"""Causal attention forward / backward timing at the C2 shape (B8 S2048 H28 hd128).
Kernel variants are chosen by environment (HLM_ATTN_EXP_EMU, HLM_ATTN_BWD_V1), read once
per process: run this once per variant. ATTN_HEAT: see below."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_04816_b200 import _lib as L
Lb = L.blib()
B, S, H, hd = (int(x) for x in os.environ.get("ATTN_SHAPE", "8,2048,28,128").split(","))
h, T = H * hd, B * S
dev = "cuda"
q, k, v = (torch.randn(T, h, device=dev).bfloat16() for _ in range(3))
dq, dk, dv = (torch.empty_like(q) for _ in range(3))
ld_in = h   # planar q / k / v (ld = h), as the engine's block lays them out
do = torch.randn(T, h, device=dev).bfloat16()
o = torch.empty(T, h, device=dev, dtype=torch.bfloat16); lse = torch.empty(B * H * S, device=dev)
ds = torch.empty_like(lse)
d = L.HlmBlockDims(B, S, h, 8, H, 0)
vp = lambda t: ctypes.c_void_p(t.data_ptr())
fwd = lambda: L.check(Lb.hlm_cuda_attention_fwd(ctypes.byref(d), vp(q), vp(k), vp(v), vp(o), vp(lse), ld_in, None))
bwd = lambda: L.check(Lb.hlm_cuda_attention_bwd(ctypes.byref(d), vp(q), vp(k), vp(v), vp(o), vp(do), vp(lse), vp(ds), vp(dq), vp(dk), vp(dv), ld_in, None))
# ATTN_HEAT=1: a large bf16 GEMM before every timed call (GPU at its power limit, L2 full of
# other data, as inside a training step); only the attention call is timed
heat = os.environ.get("ATTN_HEAT") == "1"
ga = torch.randn(8192, 8192, device=dev).bfloat16() if heat else None
def t(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    if heat:
        tot = 0.0
        for _ in range(it):
            ga @ ga
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record(); fn(); b.record(); torch.cuda.synchronize()
            tot += a.elapsed_time(b)
        return tot / it
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it
fl = 2.0 * B * S * S * h   # causal fwd: QK^T and PV over the lower triangle
tf = t(fwd); tb = t(bwd)
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith(("HLM_ATTN", "ATTN_")))
print(f"[{tag or 'default'}] fwd {tf:.3f} ms = {fl/tf/1e9:.0f} TFLOP/s ; bwd {tb:.3f} ms = "
      f"{2.5*fl/tb/1e9:.0f} TFLOP/s (2.5x fwd flops)")
