"""One transformer block forward + backward at a workload width (default C2: B8 S2048
h3584 f18944 28 heads, RoPE), fused GEMM epilogues vs HLM_BLOCK_UNFUSED, CUDA-event
timed back to back (median of `iters`). Prints ms per fwd / bwd and the per-kernel
split from the in-library kernel timer.

    python tools/block_bench.py [c2|c4|c5] [iters]
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_04816_b200 import _lib as L  # noqa: E402

SHAPES = {"c2": (8, 2048, 3584, 18944, 28), "c4": (8, 2048, 8192, 29568, 64), "c5": (4, 4096, 12288, 49152, 96)}


def vp(t):
    return ctypes.c_void_p(t.data_ptr())


def run(cfg="c2", iters=10):
    B, S, h, f, H = SHAPES[cfg]
    T, n = B * S, 4 * h * h + 3 * h * f + 2 * h
    dev = "cuda"
    Lb = L.blib()
    W = torch.cat([torch.randn(n - 2 * h, device=dev) * 0.02, 1 + 0.1 * torch.randn(2 * h, device=dev)]).bfloat16()
    x = torch.randn(T, h, device=dev)
    g = torch.randn(T, h, device=dev) * 1e-2
    y, gi = torch.empty_like(x), torch.empty_like(x)
    grad = torch.empty(n, device=dev)
    hd = h // H
    cs = torch.empty(S * hd // 2, device=dev)
    sn = torch.empty_like(cs)
    L.check(Lb.hlm_cuda_rope_table(vp(cs), vp(sn), S, hd, 1e6))
    out = {}
    # the two variants alternate iteration by iteration so clock / power drift hits both
    runs = {}
    for name, flags in (("fused", 0), ("unfused", L.BLOCK_UNFUSED)):
        d = L.HlmBlockDims(B, S, h, f, H, flags)
        acts = torch.empty(Lb.hlm_cuda_block_acts_bytes(ctypes.byref(d)), dtype=torch.uint8, device=dev)
        ws = torch.empty(Lb.hlm_cuda_block_ws_bytes(ctypes.byref(d)), dtype=torch.uint8, device=dev)
        runs[name] = (d, acts, ws, [], [])
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for i in range(iters + 2):
        for name, (d, acts, ws, tf, tb) in runs.items():
            ev[0].record()
            L.check(Lb.hlm_cuda_block_fwd(ctypes.byref(d), vp(W), vp(x), vp(y), vp(acts), vp(ws), vp(cs), vp(sn),
                                          None))
            ev[1].record()
            L.check(Lb.hlm_cuda_block_bwd(ctypes.byref(d), vp(W), vp(x), vp(acts), vp(g), vp(gi), vp(grad), vp(ws),
                                          vp(cs), vp(sn), None))
            ev[2].record()
            torch.cuda.synchronize()
            if i >= 2:
                tf.append(ev[0].elapsed_time(ev[1]))
                tb.append(ev[1].elapsed_time(ev[2]))
    # per-kind split of one more iteration of each variant (in-library kernel timer)
    Lb.hlm_ktimer_enable.argtypes = [ctypes.c_int]
    Lb.hlm_ktimer_collect.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
    kinds = ("gemm", "attn_fwd", "attn_bwd", "rmsnorm_fwd", "rmsnorm_bwd", "swiglu_fwd", "swiglu_bwd", "rope",
             "cast")
    for name, (d, acts, ws, _, _) in runs.items():
        Lb.hlm_ktimer_reset()
        Lb.hlm_ktimer_enable(1)
        L.check(Lb.hlm_cuda_block_fwd(ctypes.byref(d), vp(W), vp(x), vp(y), vp(acts), vp(ws), vp(cs), vp(sn), None))
        L.check(Lb.hlm_cuda_block_bwd(ctypes.byref(d), vp(W), vp(x), vp(acts), vp(g), vp(gi), vp(grad), vp(ws),
                                      vp(cs), vp(sn), None))
        torch.cuda.synchronize()
        Lb.hlm_ktimer_enable(0)
        parts = []
        for k, kname in enumerate(kinds):
            ms_k, w_k, n_k = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
            Lb.hlm_ktimer_collect(k, ctypes.byref(ms_k), ctypes.byref(w_k), ctypes.byref(n_k))
            if n_k.value:
                rate = f" {w_k.value / ms_k.value / 1e9:.0f} TF/s" if k < 3 else ""
                parts.append(f"{kname} {ms_k.value:.3f} ms x{n_k.value}{rate}")
        print(f"{cfg} {name:8s} " + "; ".join(parts), flush=True)
        Lb.hlm_ktimer_reset()
    for name, (_, _, _, tf, tb) in runs.items():
        tf.sort(), tb.sort()
        out[name] = (tf[len(tf) // 2], tb[len(tb) // 2])
        print(f"{cfg} {name:8s} fwd {out[name][0]:7.3f} ms  bwd {out[name][1]:7.3f} ms  "
              f"total {sum(out[name]):7.3f} ms", flush=True)
    f0, u0 = sum(out["fused"]), sum(out["unfused"])
    print(f"{cfg} fused saves {u0 - f0:.3f} ms per block fwd+bwd ({(u0 - f0) / u0 * 100:.1f} %)")


if __name__ == "__main__":
    run(sys.argv[1] if len(sys.argv) > 1 else "c2", int(sys.argv[2]) if len(sys.argv) > 2 else 10)
