"""Vocab-chunked head (hlm_cuda_head_stats + hlm_cuda_head_grad_chunk, the
engine's piecewise head gradient) against the row-chunked hlm_cuda_head_loss
(reference head_fwd / ce_loss_and_grad / head_bwd, kernels.hpp:410-446), its
up-front finiteness certificate, and the engine path against the oracle."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2602_04816_b200 import _lib as L
from paper_2602_04816_b200 import engine as E

pytestmark = pytest.mark.gpu
UNCERT = 0xFFFFFFFFFFFFFFFE
NONE = 0xFFFFFFFFFFFFFFFF


def vp(t):
    return t.data_ptr()


def rel_l2(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def _head_inputs(T, h, V, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(T, h, device="cuda", generator=g)
    head = (torch.randn(V, h, device="cuda", generator=g) * 0.05).bfloat16()
    tgt = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32, generator=g)
    return x, head, tgt


def _pieces(Lb, T, h, V, x, head, tgt, vc, ws):
    dx = torch.empty(T, h, device="cuda")
    dhead = torch.full((V, h), float("nan"), device="cuda")
    loss = torch.empty(T, device="cuda")
    cert = torch.zeros(1, dtype=torch.int64, device="cuda")
    L.check(Lb.hlm_cuda_head_stats(T, h, V, vp(head), vp(x), vp(tgt), 1.0 / T, vp(loss), vp(cert), vp(ws), None))
    for k, v0 in enumerate(range(0, V, vc)):
        L.check(Lb.hlm_cuda_head_grad_chunk(T, h, V, vp(head), vp(tgt), 1.0 / T, v0, min(vc, V - v0), vp(dx),
                                            int(k > 0), vp(dhead), 0, vp(ws), None))
    torch.cuda.synchronize()
    return loss, dx, dhead, int(cert.item()) & (2**64 - 1)


@pytest.mark.parametrize("T,h,V,vc", [(256, 64, 1003, 128), (512, 128, 4096, 1024), (64, 16, 13, 8),
                                      (4096, 256, 152064, 18688)])
def test_vocab_chunks_match_row_chunked_head(T, h, V, vc):
    Lb = L.blib()
    x, head, tgt = _head_inputs(T, h, V)
    ws = torch.empty(Lb.hlm_cuda_head_ws_bytes(T, h, V), dtype=torch.uint8, device="cuda")
    vc = min(vc, Lb.hlm_cuda_head_chunk_vocab(T, V))
    loss_p, dx_p, dh_p, cert = _pieces(Lb, T, h, V, x, head, tgt, vc, ws)
    dx = torch.empty(T, h, device="cuda")
    dh = torch.empty(V, h, device="cuda")
    loss = torch.empty(T, device="cuda")
    L.check(Lb.hlm_cuda_head_loss(T, h, V, vp(head), vp(x), vp(tgt), 1.0 / T, vp(dx), vp(dh), 0, vp(loss),
                                  vp(ws), None))
    torch.cuda.synchronize()
    assert cert == NONE
    assert torch.equal(loss_p, loss)                       # same pass-1 statistics, bit for bit
    assert rel_l2(dh_p.cpu().numpy(), dh.cpu().numpy()) < 1e-5
    # d_x sums the vocab chunks in a different order (fp32): a few ulps of rounding
    assert rel_l2(dx_p.cpu().numpy(), dx.cpu().numpy()) < 2e-4


def test_certificate_refuses_huge_or_non_finite_inputs():
    Lb = L.blib()
    T, h, V = 128, 32, 300
    ws = torch.empty(Lb.hlm_cuda_head_ws_bytes(T, h, V), dtype=torch.uint8, device="cuda")
    for bad in (float("nan"), float("inf"), 3e37):
        x, head, tgt = _head_inputs(T, h, V, seed=1)
        x[5, 7] = bad
        *_, cert = _pieces(Lb, T, h, V, x, head, tgt, 128, ws)
        assert cert == UNCERT, bad
    x, head, tgt = _head_inputs(T, h, V, seed=1)
    head[17, 3] = float("nan")           # poisons the logits -> row statistics
    *_, cert = _pieces(Lb, T, h, V, x, head, tgt, 128, ws)
    assert cert == UNCERT


def _cfg():
    return E.ModelConfig(2, 64, 128, 1000, 32, 2, k_ckpt=1, n_heads=2, rope_theta=1e6)


def test_engine_head_pieces_match_oracle_and_unchunked():
    c = _cfg()
    tok = E.make_copy_task_batch(c, 11)
    res = {}
    for pv in (-1, 128):
        s = E.Store(c, 21)
        e = E.Engine(s, E.Arena(c), E.HyperParams(), E.EngineOptions(skip_optimizer=True, head_piece_vocab=pv))
        r = e.train_step(tok)
        res[pv] = (r.loss, s.grads(), s.weights())
    assert res[-1][0] == res[128][0]
    # d_x sums the vocab chunks in another fp32 order; the BF16 casts downstream turn
    # those ulps into ~1e-3 relative differences of the block gradients
    assert rel_l2(res[128][1], res[-1][1]) < 1e-2
    oc = O.cfg(c.layers, c.hidden, c.ffn, c.vocab, c.seq, c.batch, 1, False, c.n_heads, c.rope_theta)
    loss_ref, g_ref = O.Oracle().forward_backward(oc, res[128][2], tok)
    assert abs(res[128][0] - loss_ref) / loss_ref < 2e-3
    assert rel_l2(res[128][1], g_ref) < 5e-2


def test_engine_head_pieces_train_and_trace():
    from paper_2602_04816_b200.trace import validate_trace
    c = _cfg()
    toks = [E.make_copy_task_batch(c, 5, skip=i) for i in range(4)]
    losses = {}
    for pv in (-1, 128):
        s = E.Store(c, 8)
        e = E.Engine(s, E.Arena(c), E.HyperParams(lr=2e-3),
                     E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=5,
                                     overlap_optimizer_tail=True, tail_blocks=2, head_piece_vocab=pv))
        losses[pv] = [e.train_step(t).loss for t in toks]
        e.sync()
        tr = e.last_trace()
        assert validate_trace(tr, c.layers) == []
        heads = [o for o in tr if o["stream"] == "d2h" and o["layer"] == c.layers + 1]
        assert len(heads) == (8 if pv == 128 else 1)
        assert sum(o["bytes"] for o in heads) == 4 * c.vocab * c.hidden
    assert losses[-1][0] == losses[128][0]
    assert np.allclose(losses[-1], losses[128], rtol=1e-4)


def test_engine_head_pieces_non_finite_still_aborts():
    c = E.ModelConfig(2, 16, 32, 13, 4, 1)
    s = E.Store(c, 5, "fp32")
    w = s.weights()
    w[-1] = np.nan   # head tile: poisons the logits, so no certificate; the full scan finds it
    s.import_master(w)
    e = E.Engine(s, E.Arena(c), E.HyperParams(), E.EngineOptions(eager_optim=True, head_piece_vocab=4))
    with pytest.raises(E.NumericsError, match="non-finite gradient in layer"):
        e.train_step(E.make_copy_task_batch(c, 2))
