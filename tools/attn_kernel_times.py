"""Per-kernel device times of one attention backward at the C2 shape (torch profiler):
the D kernel, dK/dV and dQ separately. Variants via the HLM_ATTN_* environment switches
(INTEGRATION.md §7)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_04816_b200 import _lib as L
Lb = L.blib()
B, S, H, hd = 8, 2048, 28, 128
h, T = H * hd, B * S
q, k, v, do = (torch.randn(T, h, device="cuda").bfloat16() for _ in range(4))
o = torch.empty_like(q); lse = torch.empty(B * H * S, device="cuda")
dq, dk, dv = (torch.empty_like(q) for _ in range(3)); ds = torch.empty_like(lse)
d = L.HlmBlockDims(B, S, h, 8, H, 0)
vp = lambda t: ctypes.c_void_p(t.data_ptr())
L.check(Lb.hlm_cuda_attention_fwd(ctypes.byref(d), vp(q), vp(k), vp(v), vp(o), vp(lse), h, None))
bwd = lambda: L.check(Lb.hlm_cuda_attention_bwd(ctypes.byref(d), vp(q), vp(k), vp(v), vp(o), vp(do), vp(lse), vp(ds), vp(dq), vp(dk), vp(dv), h, None))
for _ in range(3): bwd()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(10): bwd()
    torch.cuda.synchronize()
for e in prof.key_averages():
    if e.device_time_total > 0: print(f"  {e.key[:50]:50s} {e.device_time_total/e.count:8.1f} us")
