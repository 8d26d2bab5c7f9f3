"""Test infrastructure: a PyTorch restatement of the whole decoder step (embedding, blocks,
head + CE, and their backward) used to calibrate and pin the GPU path's BF16 tolerance.

Two modes over the same weights (store layout, the BF16 shadow widened to fp32):

* exact=True  — no rounding of activations or gradients: the model as the reference
  defines it (oracle/hlm_oracle.cpp forward_backward, which follows
  proj/include/hlm/kernels.hpp:129-446 and proj/src/oracle.cpp:549-566, plus the
  multi-head + rotate-half RoPE extension), in fp32 (TF32 off) or fp64.
* exact=False — the same math with every tensor rounded to BF16 exactly where the CUDA
  path rounds it (paper_2602_04816_b200/csrc/capi/block_capi.cpp):
    forward : n1, q/k/v (GEMM epilogue), q/k after RoPE (in place on BF16), softmax P
              before the P.V product, attention output o, n2, up|gate, act = up*silu(gate),
              the head input x;
    backward: the incoming gradient of every GEMM (g_out -> g_bf before the down
              projection's wgrad / dgrad, d_y -> d_y_bf before o-proj's, d_logits), d_act,
              d_up|d_gate, d_o, dS before dQ / dK, dq/dk/dv, dq/dk after the inverse RoPE.
  Residual streams, RMSNorm statistics and backward, softmax statistics and every
  accumulation stay fp32, as in the kernels.

The BF16-emulating run measures the *inherent* rounding noise of this precision recipe
(its distance to the exact run); the GPU path's distance to the exact run must stay
within a small multiple of that noise, per tensor (tests/test_parity_wide_gpu.py).
Only tests import this module; nothing in the product path does.
"""
import math

import torch

BLOCK_TENSORS = ("w_q", "w_k", "w_v", "w_o", "w_up", "w_gate", "w_down", "norm1", "norm2")


def block_layout(h, f):
    """(name, offset, shape) in the canonical tile order (proj/src/host_store.cpp:70-92)."""
    out, o = [], 0
    for name, shape in (("w_q", (h, h)), ("w_k", (h, h)), ("w_v", (h, h)), ("w_o", (h, h)),
                        ("w_up", (h, f)), ("w_gate", (h, f)), ("w_down", (f, h)),
                        ("norm1", (h,)), ("norm2", (h,))):
        n = math.prod(shape)
        out.append((name, o, shape))
        o += n
    return out, o


def model_tensors(L, h, f, V):
    """(name, offset, numel) of every named parameter tensor in store layout (untied)."""
    out = [("embed", 0, V * h)]
    o = V * h
    lay, n = block_layout(h, f)
    for layer in range(1, L + 1):
        for name, off, shape in lay:
            out.append((f"L{layer}.{name}", o + off, math.prod(shape)))
        o += n
    out.append(("head", o, V * h))
    return out


class _Round(torch.autograd.Function):
    """BF16 RNE in the forward; the backward rounds the gradient too when `grad`."""

    @staticmethod
    def forward(ctx, x, fwd, grad):
        ctx.grad = grad
        return x.to(torch.bfloat16).to(x.dtype) if fwd else x.clone()

    @staticmethod
    def backward(ctx, g):
        return (g.to(torch.bfloat16).to(g.dtype) if ctx.grad else g), None, None


def _bf(x):
    return x.to(torch.bfloat16).to(x.dtype)


class _Attention(torch.autograd.Function):
    """Causal multi-head attention, q/k/v (B, H, S, hd). Emulated mode follows the flash
    kernels: P = exp(s - max) rounded before P.V, O normalised by the fp32 row sum; the
    backward recomputes P from the log-sum-exp, D = rowsum(dO * o_bf16), dS rounded
    before dQ = scale dS K and dK = scale dS^T Q, dV = P_bf^T dO."""

    @staticmethod
    def forward(ctx, q, k, v, emulate):
        S, hd = q.shape[-2], q.shape[-1]
        scale = 1.0 / math.sqrt(hd)
        s = (q @ k.transpose(-1, -2)) * scale
        mask = torch.triu(torch.ones(S, S, dtype=torch.bool, device=q.device), 1)
        s = s.masked_fill(mask, float("-inf"))
        m = s.amax(-1, keepdim=True)
        p = torch.exp(s - m)
        l = p.sum(-1, keepdim=True)
        o = ((_bf(p) if emulate else p) @ v) / l
        lse = m + torch.log(l)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.emulate, ctx.scale = emulate, scale
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        S = q.shape[-2]
        emulate, scale = ctx.emulate, ctx.scale
        s = (q @ k.transpose(-1, -2)) * scale
        mask = torch.triu(torch.ones(S, S, dtype=torch.bool, device=q.device), 1)
        p = torch.exp(s.masked_fill(mask, float("-inf")) - lse)
        o_used = _bf(o) if emulate else o
        D = (do * o_used).sum(-1, keepdim=True)
        dv = (_bf(p) if emulate else p).transpose(-1, -2) @ do
        dp = do @ v.transpose(-1, -2)
        ds = p * (dp - D)
        if emulate:
            ds = _bf(ds)
        dq = (ds @ k) * scale
        dk = (ds.transpose(-1, -2) @ q) * scale
        return dq, dk, dv, None


def rope_tables(S, hd, theta, device, dtype):
    """hlm_cuda_rope_table / oracle Rope: fp64 inverse frequency, fp32 angle, fp64 cos/sin
    rounded to fp32."""
    half = hd // 2
    i = torch.arange(half, dtype=torch.float64, device=device)
    inv = theta ** (-2.0 * i / hd)
    ang = (torch.arange(S, dtype=torch.float64, device=device)[:, None] * inv).float().double()
    return ang.cos().float().to(dtype), ang.sin().float().to(dtype)


class _Ctx:
    """Rounding helpers and RoPE tables of one restatement run."""

    def __init__(self, S, B, h, H, theta, exact, dtype, device, eps=1e-6):
        self.emulate = not exact
        self.S, self.B, self.h, self.H, self.eps = S, B, h, H, eps
        self.hd = h // H
        self.cos, self.sin = rope_tables(S, self.hd, theta, device, dtype) if theta > 0 else (None, None)

    def rf(self, x):   # rounded forward, fp32 gradient
        return _Round.apply(x, self.emulate, False)

    def rb(self, x):   # rounded forward and gradient
        return _Round.apply(x, self.emulate, self.emulate)

    def rg(self, x):   # gradient rounded (the GEMM's incoming gradient operand)
        return _Round.apply(x, False, self.emulate)

    def rms(self, x, s):
        return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + self.eps) * s

    def rope(self, x):
        B, S, H, hd = self.B, self.S, self.H, self.hd
        half = hd // 2
        x = x.view(B, S, H, hd)
        a, b = x[..., :half], x[..., half:]
        c, s_ = self.cos[None, :, None, :], self.sin[None, :, None, :]
        return torch.cat([a * c - b * s_, b * c + a * s_], -1).view(B * S, self.h)

    def block(self, x, blk):
        """block_forward (kernels.hpp:313-332 + heads / RoPE) with the CUDA path's roundings."""
        rf, rb, rg = self.rf, self.rb, self.rg
        B, S, H, hd, h = self.B, self.S, self.H, self.hd, self.h
        n1 = rf(self.rms(x, blk["norm1"]))
        if self.cos is not None:
            q = rb(self.rope(rb(n1 @ blk["w_q"])))
            k = rb(self.rope(rb(n1 @ blk["w_k"])))
        else:
            q, k = rb(n1 @ blk["w_q"]), rb(n1 @ blk["w_k"])
        v = rb(n1 @ blk["w_v"])
        qh, kh, vh = (t.view(B, S, H, hd).permute(0, 2, 1, 3) for t in (q, k, v))
        att = _Attention.apply(qh, kh, vh, self.emulate).permute(0, 2, 1, 3).reshape(B * S, h)
        att = rb(att)
        y = x + rg(att @ blk["w_o"])
        n2 = rf(self.rms(y, blk["norm2"]))
        up = rb(n2 @ blk["w_up"])
        gate = rb(n2 @ blk["w_gate"])
        act = rb(up * torch.nn.functional.silu(gate))
        return y + rg(act @ blk["w_down"])


class _NoTF32:
    def __enter__(self):
        self.prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False

    def __exit__(self, *a):
        torch.backends.cuda.matmul.allow_tf32 = self.prev


def _views(Wd, base, h, f):
    lay, n = block_layout(h, f)
    return {name: Wd[base + off:base + off + math.prod(shape)].view(*shape) for name, off, shape in lay}, n


def block_forward_backward(x, Wtile, g_out, h, f, S, B, H, theta=1e6, exact=True, dtype=torch.float32):
    """One block (hlm_cuda_block_fwd / _bwd semantics): returns (h_out, g_in, tile gradient)."""
    with _NoTF32():
        ctx = _Ctx(S, B, h, H, theta, exact, dtype, x.device)
        Wd = Wtile.detach().to(dtype).requires_grad_(True)
        xd = x.detach().to(dtype).requires_grad_(True)
        blk, _ = _views(Wd, 0, h, f)
        y = ctx.block(xd, blk)
        y.backward(g_out.to(dtype))
        return y.detach(), xd.grad.detach(), Wd.grad.detach()


def forward_backward(W, tokens, L, h, f, V, S, B, H, theta=1e6, exact=True, dtype=torch.float32,
                     return_rows=False):
    """Loss and per-parameter gradients (flat, store layout, untied) of one step.
    W: flat parameters (the BF16 shadow values), tokens: (B*S,) int (targets = tokens,
    the copy task). Returns (loss: float, grad: flat tensor of `dtype`[, per-row losses])."""
    with _NoTF32():
        Wd = W.detach().to(dtype).requires_grad_(True)
        ctx = _Ctx(S, B, h, H, theta, exact, dtype, W.device)
        tok = tokens.to(W.device).long()
        x = Wd[:V * h].view(V, h)[tok]
        o = V * h
        for _ in range(L):
            blk, n = _views(Wd, o, h, f)
            o += n
            x = ctx.block(x, blk)
        head = Wd[o:o + V * h].view(V, h)
        logits = ctx.rg(ctx.rf(x) @ head.t())
        rows = torch.nn.functional.cross_entropy(logits, tok, reduction="none")
        loss = rows.mean()
        loss.backward()
        if return_rows:
            return float(loss.detach()), Wd.grad.detach(), rows.detach()
        return float(loss.detach()), Wd.grad.detach()


def adam_update(master, grad, t, lr, beta1=0.9, beta2=0.999, eps_=1e-8, wd=0.0):
    """Reference adam_update_tile (proj/src/host_store.cpp:334-362) from zero moments at
    step t == 1 (fp32); returns the new master."""
    g = grad.float()
    m = (1 - beta1) * g
    v = (1 - beta2) * g * g
    bc1 = 1 - beta1 ** t
    bc2 = 1 - beta2 ** t
    return master - lr * ((m / bc1) / (torch.sqrt(v / bc2) + eps_) + wd * master)
