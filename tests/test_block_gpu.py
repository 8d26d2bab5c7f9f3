"""Block / head / embedding kernels through the C ABI against the CPU oracle
(oracle/liboracle.so, itself pinned bitwise to the reference) on identical
bf16 weights and fp32 inputs.

Tolerance (BF16-compute / FP32-accumulate): the GPU rounds every GEMM operand
to bf16 (activations and gradients), the oracle computes in FP32 on the same
bf16 weights. Per-tensor relative L2 error must stay below REL_L2 (5e-2 on
gradients; the q/k projections' gradients are two orders smaller at init and
get their own bound) and below 1e-2 on forward outputs."""
import ctypes

import numpy as np
import pytest
import torch

import oracle as O
from paper_2602_04816_b200 import _lib as L

pytestmark = pytest.mark.gpu

REL_FWD = 1e-2
REL_GRAD = 5e-2


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel(); b = np.asarray(b, np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def vp(t):
    return ctypes.c_void_p(t.data_ptr())


def block_regions(c):
    h, f = c.hidden, c.ffn
    names = [("w_q", h * h), ("w_k", h * h), ("w_v", h * h), ("w_o", h * h), ("w_up", h * f),
             ("w_gate", h * f), ("w_down", f * h), ("norm1", h), ("norm2", h)]
    out, o = [], 0
    for n, k in names:
        out.append((n, o, k)); o += k
    return out


def run_block(c, w_tile, h_in, g_out, flags=0):
    Lb = L.blib()
    dev = "cuda"
    d = L.HlmBlockDims(c.batch, c.seq, c.hidden, c.ffn, c.n_heads, flags)
    T = c.batch * c.seq
    w = torch.from_numpy(w_tile).to(dev).to(torch.bfloat16)
    assert torch.equal(w.float().cpu(), torch.from_numpy(w_tile)), "weights must be bf16-exact"
    x = torch.from_numpy(h_in).to(dev)
    y = torch.empty_like(x)
    acts = torch.empty(Lb.hlm_cuda_block_acts_bytes(ctypes.byref(d)), dtype=torch.uint8, device=dev)
    ws = torch.empty(Lb.hlm_cuda_block_ws_bytes(ctypes.byref(d)), dtype=torch.uint8, device=dev)
    cs = sn = None
    if c.rope_theta > 0:
        hd = c.hidden // c.n_heads
        cs = torch.empty(c.seq * hd // 2, device=dev); sn = torch.empty_like(cs)
        L.check(Lb.hlm_cuda_rope_table(vp(cs), vp(sn), c.seq, hd, c.rope_theta))
    rc_, rs_ = (vp(cs), vp(sn)) if cs is not None else (None, None)
    L.check(Lb.hlm_cuda_block_fwd(ctypes.byref(d), vp(w), vp(x), vp(y), vp(acts), vp(ws), rc_, rs_, None))
    g = torch.from_numpy(g_out).to(dev)
    gin = torch.empty_like(x)
    grad = torch.full((w_tile.size,), float("nan"), device=dev)
    L.check(Lb.hlm_cuda_block_bwd(ctypes.byref(d), vp(w), vp(x), vp(acts), vp(g), vp(gin), vp(grad),
                                  vp(ws), rc_, rs_, None))
    torch.cuda.synchronize()
    return y.cpu().numpy(), gin.cpu().numpy(), grad.cpu().numpy()


CASES = [
    ("ref-desk", O.cfg(1, 32, 64, 32, 16, 2)),
    ("ref-acc3", O.cfg(1, 16, 32, 13, 8, 2)),
    ("ref-tiny", O.cfg(1, 8, 16, 11, 4, 1)),
    ("ref-c1", O.cfg(1, 256, 1024, 1024, 128, 4)),
    ("qwen-c1", O.cfg(1, 256, 1024, 1024, 128, 4, n_heads=2, rope_theta=1e6)),
    ("qwen-hd64", O.cfg(1, 256, 512, 64, 64, 2, n_heads=4, rope_theta=1e4)),
]


@pytest.mark.parametrize("name,c", CASES, ids=[n for n, _ in CASES])
def test_block_matches_oracle(name, c):
    orc = O.Oracle()
    w_all = orc.init_weights(c, 5, True)
    off = c.vocab * c.hidden
    w_tile = w_all[off:off + O.block_params(c)].copy()
    rng = np.random.default_rng(1)
    T = c.batch * c.seq
    h_in = rng.standard_normal(T * c.hidden).astype(np.float32)
    g_out = (rng.standard_normal(T * c.hidden) * 1e-2).astype(np.float32)
    y, gin, grad = run_block(c, w_tile, h_in, g_out)
    y_ref, _ = orc.block_forward(c, w_tile, h_in)
    gin_ref, grad_ref = orc.block_backward(c, w_tile, h_in, g_out)
    assert rel_l2(y, y_ref) < REL_FWD
    assert rel_l2(gin, gin_ref) < REL_GRAD
    report = {}
    for n, o, k in block_regions(c):
        report[n] = rel_l2(grad[o:o + k], grad_ref[o:o + k])
    print(name, {k: f"{v:.2e}" for k, v in report.items()})
    for n, e in report.items():
        assert e < REL_GRAD, (n, e)


def test_generic_and_default_attention_agree():
    c = O.cfg(1, 256, 512, 64, 128, 2, n_heads=2, rope_theta=1e6)
    orc = O.Oracle()
    w_all = orc.init_weights(c, 9, True)
    off = c.vocab * c.hidden
    w_tile = w_all[off:off + O.block_params(c)].copy()
    rng = np.random.default_rng(2)
    T = c.batch * c.seq
    h_in = rng.standard_normal(T * c.hidden).astype(np.float32)
    g_out = (rng.standard_normal(T * c.hidden) * 1e-2).astype(np.float32)
    a = run_block(c, w_tile, h_in, g_out, flags=0)
    b = run_block(c, w_tile, h_in, g_out, flags=L.BLOCK_GENERIC_ATTENTION)
    for u, v in zip(a, b):
        assert rel_l2(u, v) < 2e-2


def test_head_loss_and_embedding_match_oracle():
    """Whole model with zero blocks' contribution isolated: embed -> head -> CE
    -> head bwd -> embed bwd, against the oracle's loss and table gradients."""
    Lb = L.blib()
    dev = "cuda"
    c = O.cfg(1, 64, 128, 300, 32, 4)
    orc = O.Oracle()
    w = orc.init_weights(c, 3, True)
    # zero the block so h_L == embedding rows (identity block, test_numerics_api.cpp:15)
    off = c.vocab * c.hidden
    nb = O.block_params(c)
    w[off:off + nb] = 0.0
    tok = orc.copy_task_tokens(c, 4)
    loss_ref, g_ref = orc.forward_backward(c, w, tok)
    T, h, V = c.batch * c.seq, c.hidden, c.vocab
    table = torch.from_numpy(w[:off]).to(dev).bfloat16()
    head = torch.from_numpy(w[off + nb:]).to(dev).bfloat16()
    tok_d = torch.from_numpy(tok).to(dev)
    x = torch.empty(T, h, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    L.check(Lb.hlm_cuda_embed_fwd(vp(tok_d), vp(table), vp(x), T, h, V, vp(err), None))
    ws = torch.empty(Lb.hlm_cuda_head_ws_bytes(T, h, V), dtype=torch.uint8, device=dev)
    dx = torch.empty(T, h, device=dev)
    dhead = torch.empty(V, h, device=dev)
    loss_rows = torch.empty(T, device=dev)
    L.check(Lb.hlm_cuda_head_loss(T, h, V, vp(head), vp(x), vp(tok_d), 1.0 / T, vp(dx), vp(dhead), 0,
                                  vp(loss_rows), vp(ws), None))
    rp = np.empty(V + 1, np.int32); pos = np.empty(T, np.int32)
    L.check(Lb.hlm_embed_csr(tok.ctypes.data, T, V, rp.ctypes.data, pos.ctypes.data))
    rp_d, pos_d = torch.from_numpy(rp).to(dev), torch.from_numpy(pos).to(dev)
    dtab = torch.empty(V, h, device=dev)
    L.check(Lb.hlm_cuda_embed_bwd(vp(rp_d), vp(pos_d), vp(dx), vp(dtab), V, h, 0, None))
    torch.cuda.synchronize()
    assert err.item() == 0
    loss = loss_rows.double().sum().item()
    assert abs(loss - loss_ref) / loss_ref < 1e-3
    assert rel_l2(dhead.cpu().numpy().ravel(), g_ref[off + nb:]) < REL_GRAD
    assert rel_l2(dtab.cpu().numpy().ravel(), g_ref[:off]) < REL_GRAD


def test_head_loss_is_chunked_and_matches_torch():
    """T*V large enough for several row chunks (2 GiB of logits + d_logits per
    chunk): loss, d_x and the chunk-accumulated d_head vs an fp32 torch reference."""
    Lb = L.blib()
    dev = "cuda"
    T, h, V = 8192, 256, 152064
    torch.manual_seed(0)
    x = torch.randn(T, h, device=dev)
    head = (torch.randn(V, h, device=dev) * 0.02).bfloat16()
    tgt = torch.randint(0, V, (T,), device=dev, dtype=torch.int32)
    ws = torch.empty(Lb.hlm_cuda_head_ws_bytes(T, h, V), dtype=torch.uint8, device=dev)
    assert ws.numel() < 3 * (1 << 30)      # never the whole (T, V) fp32 + bf16 pair (7.5 GB)
    dx = torch.empty(T, h, device=dev)
    dhead = torch.empty(V, h, device=dev)
    loss_rows = torch.empty(T, device=dev)
    L.check(Lb.hlm_cuda_head_loss(T, h, V, vp(head), vp(x), vp(tgt), 1.0 / T, vp(dx), vp(dhead), 0,
                                  vp(loss_rows), vp(ws), None))
    torch.cuda.synchronize()
    xb = x.bfloat16().float().requires_grad_(True)
    hf = head.float().requires_grad_(True)
    loss = torch.nn.functional.cross_entropy(xb @ hf.t(), tgt.long())
    loss.backward()
    assert abs(loss_rows.double().sum().item() - loss.item()) < 1e-3 * loss.item()
    assert rel_l2(dx.cpu().numpy(), xb.grad.cpu().numpy()) < 2e-2
    assert rel_l2(dhead.cpu().numpy(), hf.grad.cpu().numpy()) < 2e-2


_RMS_SCRIPT = r"""
import ctypes, sys, torch
sys.path.insert(0, {root!r})
from paper_2602_04816_b200 import _lib as L
Lb = L.blib()
torch.manual_seed(0)
B, S, h, f, H = 1, 512, 3584, 1024, 28
T, n = B * S, 4 * h * h + 3 * h * f + 2 * h
W = torch.cat([torch.randn(n - 2 * h, device="cuda") * 0.02, 1 + 0.1 * torch.randn(2 * h, device="cuda")]).bfloat16()
x = torch.randn(T, h, device="cuda"); g = torch.randn(T, h, device="cuda") * 1e-2
y, gi = torch.empty_like(x), torch.empty_like(x); grad = torch.empty(n, device="cuda")
d = L.HlmBlockDims(B, S, h, f, H, 0)
acts = torch.empty(Lb.hlm_cuda_block_acts_bytes(ctypes.byref(d)), dtype=torch.uint8, device="cuda")
ws = torch.empty(Lb.hlm_cuda_block_ws_bytes(ctypes.byref(d)), dtype=torch.uint8, device="cuda")
hd = h // H
cs = torch.empty(S * hd // 2, device="cuda"); sn = torch.empty_like(cs)
vp = lambda t: ctypes.c_void_p(t.data_ptr())
L.check(Lb.hlm_cuda_rope_table(vp(cs), vp(sn), S, hd, 1e6))
L.check(Lb.hlm_cuda_block_fwd(ctypes.byref(d), vp(W), vp(x), vp(y), vp(acts), vp(ws), vp(cs), vp(sn), None))
L.check(Lb.hlm_cuda_block_bwd(ctypes.byref(d), vp(W), vp(x), vp(acts), vp(g), vp(gi), vp(grad), vp(ws), vp(cs),
                              vp(sn), None))
torch.cuda.synchronize()
torch.save({{"gi": gi.cpu(), "grad": grad.cpu()}}, sys.argv[1])
"""


def test_rmsnorm_backward_variants_are_bitwise_equal(tmp_path):
    """The RMSNorm backward kernels (scale / scale-gradient partial in registers at 2 or 3
    CTAs per SM, or in shared memory) sum every column in the same row order: a whole
    block backward is bit-identical across them."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "rms.py"
    script.write_text(_RMS_SCRIPT.format(root=root))
    res = {}
    for m in ("2", "3", "5"):
        out = tmp_path / f"rms_{m}.pt"
        subprocess.run([sys.executable, str(script), str(out)], check=True,
                       env={**os.environ, "HLM_RMSNORM_BWD_MINB": m})
        res[m] = torch.load(out)
    for m in ("3", "5"):
        assert torch.equal(res[m]["gi"], res["2"]["gi"]), m
        assert torch.equal(res[m]["grad"], res["2"]["grad"]), m
