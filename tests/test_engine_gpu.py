"""The streaming engine on the GPU through the C ABI, against the oracle
(pinned bitwise to the reference) and the reference engine's own contracts
(proj/tests/test_engine.cpp)."""
import ast
import os

import numpy as np
import pytest

import oracle as O
from paper_2602_04816_b200 import engine as E

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

REL_GRAD = 5e-2     # BF16-compute / FP32-accumulate bound on per-tensor relative L2
REL_LOSS = 2e-3


def rel_l2(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def ocfg(c):
    return O.cfg(c.layers, c.hidden, c.ffn, c.vocab, c.seq, c.batch, c.k_ckpt,
                 bool(c.tie_embeddings), c.n_heads, c.rope_theta)


def tiles(c):
    """(name, offset, size) of every logical gradient tile in store layout."""
    V, h = c.vocab, c.hidden
    out = [("embed", 0, V * h)]
    o = V * h
    for l in range(1, c.layers + 1):
        out.append((f"block{l}", o, c.block_params())); o += c.block_params()
    if not c.tie_embeddings:
        out.append(("head", o, V * h))
    return out


def grad_step(c, seed, tokens, dtype="bf16", **opt):
    s = E.Store(c, seed, dtype)
    a = E.Arena(c)
    e = E.Engine(s, a, E.HyperParams(), E.EngineOptions(skip_optimizer=True, **opt))
    r = e.train_step(tokens)
    return r, s.grads(), s


CFGS = [
    ("desk-K2", E.ModelConfig(4, 32, 64, 32, 16, 2, k_ckpt=2)),
    ("desk-K1", E.ModelConfig(4, 32, 64, 32, 16, 2, k_ckpt=1)),
    ("tied-K3", E.ModelConfig(4, 8, 24, 11, 8, 2, k_ckpt=3, tie_embeddings=True)),
    ("c1-ref", E.ModelConfig(4, 256, 1024, 1024, 128, 4, k_ckpt=1)),
    ("c1-qwen", E.ModelConfig(4, 256, 1024, 1024, 128, 4, k_ckpt=1, n_heads=2, rope_theta=1e6)),
    # the attention paths by shape: two-query-tile forward + 64-wide backward over several
    # tiles (S 512), the one-tile forward (S % 256 != 0), head_dim 64 (mma.sync kernels)
    ("qwen-s512", E.ModelConfig(2, 256, 512, 512, 512, 2, k_ckpt=1, n_heads=2, rope_theta=1e6)),
    ("qwen-s384", E.ModelConfig(2, 256, 512, 512, 384, 2, k_ckpt=1, n_heads=2, rope_theta=1e6)),
    ("qwen-hd64", E.ModelConfig(2, 256, 512, 512, 256, 2, k_ckpt=1, n_heads=4, rope_theta=1e6)),
]


@pytest.mark.parametrize("name,c", CFGS, ids=[n for n, _ in CFGS])
def test_one_step_matches_oracle(name, c):
    orc = O.Oracle()
    seed = 1000 + c.layers
    tok = E.make_copy_task_batch(c, seed + 1)
    r, g, s = grad_step(c, seed, tok)
    w = s.weights()
    loss_ref, g_ref = orc.forward_backward(ocfg(c), w, tok)
    assert abs(r.loss - loss_ref) / loss_ref < REL_LOSS, (r.loss, loss_ref)
    errs = {n: rel_l2(g[o:o + k], g_ref[o:o + k]) for n, o, k in tiles(c)}
    print(name, "loss", r.loss, loss_ref, {k: f"{v:.1e}" for k, v in errs.items()})
    assert max(errs.values()) < REL_GRAD, errs


def test_untrained_loss_near_ln_v_and_debug_hidden():
    c = E.ModelConfig(4, 32, 64, 32, 16, 2, k_ckpt=2)
    s = E.Store(c, 9)
    e = E.Engine(s, E.Arena(c))
    tok = E.make_copy_task_batch(c, 3)
    e.begin_step(tok)
    e.forward_streaming()
    loss = e.anchor_loss()
    assert abs(loss - np.log(32)) < 0.1
    e.backward_blockwise()
    e.finish_step()


def test_zero_blocks_pass_embedding_through():
    c = E.ModelConfig(2, 16, 32, 13, 4, 1)
    s = E.Store(c, 5, "fp32")
    w = s.weights()
    nb = c.block_params()
    w[13 * 16: 13 * 16 + 2 * nb] = 0.0
    s.import_master(w)
    e = E.Engine(s, E.Arena(c))
    tok = E.make_copy_task_batch(c, 2)
    e.begin_step(tok)
    e.forward_streaming()
    h = e.debug_hidden().reshape(-1, 16)
    table = s.export(E.FIELD_SHADOW)[:13 * 16].reshape(13, 16)
    assert np.array_equal(h, table[tok])
    e.anchor_loss(); e.backward_blockwise(); e.finish_step()


def test_phase_protocol_errors():
    c = E.ModelConfig(2, 16, 32, 13, 4, 1)
    e = E.Engine(E.Store(c, 1), E.Arena(c))
    with pytest.raises(E.ProtocolError):
        e.forward_streaming()
    tok = E.make_copy_task_batch(c, 2)
    e.begin_step(tok)
    with pytest.raises(E.ProtocolError):
        e.backward_blockwise()


def test_out_of_range_ids_raise_and_engine_recovers():
    c = E.ModelConfig(2, 16, 32, 13, 4, 1)
    e = E.Engine(E.Store(c, 1), E.Arena(c))
    bad = np.array([0, 1, 13, 2], np.int32)
    with pytest.raises(IndexError, match="token id out of range"):
        e.train_step(bad)
    with pytest.raises(IndexError, match="target id out of range"):
        e.train_step(np.array([0, 1, 2, 3], np.int32), np.array([0, -1, 2, 3], np.int32))
    r = e.train_step(np.array([0, 1, 2, 3], np.int32))
    assert np.isfinite(r.loss)


def test_k_invariance_bitwise():
    base = dict(layers=6, hidden=32, ffn=64, vocab=32, seq=16, batch=2)
    tok = E.make_copy_task_batch(E.ModelConfig(**base), 21)
    ref = None
    for k in range(1, 7):
        for fused in ([True, False] if k == 1 else [True]):
            c = E.ModelConfig(**base, k_ckpt=k)
            _, g, _ = grad_step(c, 42, tok, fused_recompute=fused)
            if ref is None:
                ref = g
            else:
                assert np.array_equal(g, ref), (k, fused)


def test_byte_counters_match_formula():
    c = E.ModelConfig(4, 32, 64, 32, 16, 2, k_ckpt=2)
    s = E.Store(c, 3)
    e = E.Engine(s, E.Arena(c))
    r = e.train_step(E.make_copy_task_batch(c, 2))
    n_table, n_blocks = c.vocab * c.hidden, c.layers * c.block_params()
    assert r.h2d_bytes == 2 * (2 * n_table + 3 * n_blocks)     # reference 3-pass schedule (K=2)
    assert r.d2h_bytes == 4 * (2 * n_table + n_blocks)         # fp32 gradients
    c1 = E.ModelConfig(4, 32, 64, 32, 16, 2, k_ckpt=1)
    e1 = E.Engine(E.Store(c1, 3), E.Arena(c1))
    r1 = e1.train_step(E.make_copy_task_batch(c1, 2))
    assert r1.h2d_bytes == 2 * (2 * n_table + 2 * n_blocks)    # fused K=1: two passes
    assert r1.recompute_forwards == c1.layers


def test_compute_schedule_L6_K3():
    """proj/tests/test_engine.cpp:62-97 hand-enumerated compute order."""
    c = E.ModelConfig(6, 8, 16, 11, 4, 1, k_ckpt=3)
    e = E.Engine(E.Store(c, 3, "fp32"), E.Arena(c))
    e.train_step(E.make_copy_task_batch(c, 1))
    got = [(op["kind"], op["layer"]) for op in e.last_trace() if op["stream"] == "compute"]
    F, R, B = "Forward", "Recompute", "LocalBackward"
    expect = [(F, 0), (F, 1), (F, 2), (F, 3), (F, 4), (F, 5), (F, 6), (F, 7), (B, 7),
              (R, 4), (R, 5), (R, 6), (B, 6), (B, 5), (B, 4),
              (R, 1), (R, 2), (R, 3), (B, 3), (B, 2), (B, 1), (B, 0)]
    assert got == expect
    ops = e.last_trace()
    assert all(op["t_end_us"] >= op["t_start_us"] >= 0 for op in ops if op["stream"] != "host")


def _train(c, seed, steps, **opt):
    s = E.Store(c, seed)
    e = E.Engine(s, E.Arena(c), E.HyperParams(lr=2e-3), E.EngineOptions(**opt))
    rng_tok = [E.make_copy_task_batch(c, 7, skip=i) for i in range(steps)]
    for t in rng_tok:
        e.train_step(t)
    return s, e


def test_eager_equals_lazy_and_threaded_equals_inline_and_slabs():
    c = E.ModelConfig(4, 32, 64, 32, 16, 2, k_ckpt=2, tie_embeddings=True)
    lazy, _ = _train(c, 55, 3)
    eager, _ = _train(c, 55, 3, eager_optim=True)
    assert lazy.bitwise_equal(eager)
    threaded, _ = _train(c, 55, 3, eager_optim=True, threaded_accum=True, n_slab=2,
                         accum_delay_us=500)
    assert lazy.bitwise_equal(threaded)
    one, e1 = _train(c, 55, 3, n_slab=1)
    assert lazy.bitwise_equal(one)


def test_no_device_state_persists_and_peak_settles():
    c = E.ModelConfig(4, 32, 64, 32, 16, 2, k_ckpt=2)
    e = E.Engine(E.Store(c, 3), E.Arena(c))
    r = [e.train_step(E.make_copy_task_batch(c, 2, skip=i)) for i in range(3)]
    assert r[1].arena_peak == r[2].arena_peak


def test_training_tracks_oracle_mixed_precision():
    """North-star numerics (FP32 master + Adam, BF16 shadow) for 20 steps vs
    the oracle's mixed mode: per-step loss within 1 %."""
    c = E.ModelConfig(4, 32, 64, 32, 16, 8, k_ckpt=2)
    out = E.train({"model": dict(layers=4, hidden=32, ffn=64, vocab=32, seq=16, batch=8, k_ckpt=2),
                   "hyper": {"lr": 3e-3}, "run": {"steps": 20, "seed": 1234, "dtype": "fp32",
                                                  "eager_optim": True, "threaded_accum": True,
                                                  "n_slab": 3}})
    ref, _ = O.Oracle().train(ocfg(c), O.hyper(lr=3e-3), 1234, "mixed", 20)
    l = np.array(out["losses"])
    assert np.all(np.abs(l - ref) / ref < 1e-2), (l, ref)
    assert l[-1] < 0.8 * l[0]


def test_weight_cache_is_bitwise_neutral_and_halves_h2d():
    """HBM weight cache: cached blocks cross PCIe once per step; gradients and
    the optimizer trajectory are bitwise unchanged."""
    c = E.ModelConfig(4, 32, 64, 32, 16, 2, k_ckpt=1)
    tok = [E.make_copy_task_batch(c, 7, skip=i) for i in range(3)]
    s0 = E.Store(c, 5)
    e0 = E.Engine(s0, E.Arena(c), E.HyperParams(lr=2e-3), E.EngineOptions(eager_optim=True))
    r0 = [e0.train_step(t) for t in tok]
    blk = 2 * c.block_params()
    for cache_layers in (2, 4):
        s1 = E.Store(c, 5)
        a1 = E.Arena(c, weight_cache_bytes=cache_layers * ((blk + 255) // 256 * 256))
        e1 = E.Engine(s1, a1, E.HyperParams(lr=2e-3), E.EngineOptions(eager_optim=True))
        r1 = [e1.train_step(t) for t in tok]
        assert s0.bitwise_equal(s1)
        assert [x.loss for x in r0] == [x.loss for x in r1]
        assert r0[-1].h2d_bytes - r1[-1].h2d_bytes == cache_layers * blk
        ops = e1.last_trace()
        xfer_layers = [o["layer"] for o in ops if o["kind"] == "WeightXfer"]
        for l in range(c.layers - cache_layers + 1, c.layers + 1):
            assert xfer_layers.count(l) == 1


def test_optimizer_tail_overlap_is_bitwise_neutral():
    c = E.ModelConfig(6, 32, 64, 32, 16, 2, k_ckpt=1)
    tok = [E.make_copy_task_batch(c, 9, skip=i) for i in range(4)]
    ref = E.Store(c, 3)
    e0 = E.Engine(ref, E.Arena(c), E.HyperParams(lr=2e-3), E.EngineOptions(eager_optim=True))
    l0 = [e0.train_step(t).loss for t in tok]
    s = E.Store(c, 3)
    e = E.Engine(s, E.Arena(c), E.HyperParams(lr=2e-3),
                 E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=5,
                                 overlap_optimizer_tail=True, tail_blocks=3, accum_delay_us=300))
    l1 = [e.train_step(t).loss for t in tok]
    e.sync()
    assert l0 == l1
    assert ref.bitwise_equal(s)


def test_non_finite_gradient_aborts_naming_the_layer():
    """A NaN weight poisons the gradients; the eager optimizer must refuse the
    update (host_store.cpp:371-382 contract, checked on the GPU before D2H)."""
    c = E.ModelConfig(2, 16, 32, 13, 4, 1)
    s = E.Store(c, 5, "fp32")
    w = s.weights()
    w[-1] = np.nan   # head tile, last element
    s.import_master(w)
    e = E.Engine(s, E.Arena(c), E.HyperParams(), E.EngineOptions(eager_optim=True))
    with pytest.raises(E.NumericsError, match="non-finite gradient in layer"):
        e.train_step(E.make_copy_task_batch(c, 2))


def test_save_load_resume_is_bitwise(tmp_path):
    """reference test_engine.cpp:376-407: 3 steps + save + load into a
    differently seeded store + 3 steps == 6 uninterrupted steps."""
    c = E.ModelConfig(4, 32, 64, 32, 16, 2, k_ckpt=2)
    hp = E.HyperParams(lr=2e-3)
    opts = E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=3)
    full = E.Store(c, 77)
    lf = full.run_training(hp, 77, 6, opts)
    part = E.Store(c, 77)
    l1 = part.run_training(hp, 77, 3, opts)
    part.save(tmp_path / "ck.hlm2")
    resumed = E.Store(c, 1)
    resumed.load(tmp_path / "ck.hlm2")
    l2 = resumed.run_training(hp, 77, 3, opts)
    assert resumed.bitwise_equal(full)
    assert list(l1) + list(l2) == list(lf)


@pytest.mark.parametrize("kw", [dict(k=1), dict(k=3), dict(k=1, cache=2), dict(k=1, tail=True),
                                dict(k=2, fused=False)])
def test_measured_traces_validate(kw):
    from paper_2602_04816_b200.trace import validate_trace
    c = E.ModelConfig(6, 32, 64, 32, 16, 2, k_ckpt=kw.get("k", 1))
    blk = (2 * c.block_params() + 255) // 256 * 256
    a = E.Arena(c, weight_cache_bytes=kw.get("cache", 0) * blk)
    opts = E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=6,
                           overlap_optimizer_tail=kw.get("tail", False), tail_blocks=2,
                           fused_recompute=kw.get("fused", True))
    e = E.Engine(E.Store(c, 3), a, E.HyperParams(), opts)
    for i in range(3):
        e.train_step(E.make_copy_task_batch(c, 1, skip=i))
    e.sync()
    v = validate_trace(e.last_trace(), c.layers)
    assert v == [], v[:5]


@pytest.mark.parametrize("res", [dict(resident_embed=True, resident_blocks=2),
                                 dict(resident_blocks=6), dict(resident_embed=True)])
def test_hbm_resident_optimizer_tiles_are_bitwise_neutral(res, tmp_path):
    """Embedding / first blocks optimised on the GPU from HBM-resident FP32 state:
    same losses and, after sync(), the same store bit for bit as the host Adam."""
    from paper_2602_04816_b200.trace import validate_trace
    c = E.ModelConfig(6, 32, 64, 32, 16, 2, k_ckpt=1, n_heads=2, rope_theta=1e4)
    toks = [E.make_copy_task_batch(c, 4, skip=i) for i in range(3)]
    ref = E.Store(c, 8)
    e0 = E.Engine(ref, E.Arena(c), E.HyperParams(lr=2e-3, weight_decay=0.01),
                  E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=4))
    l0 = [e0.train_step(t).loss for t in toks]
    s = E.Store(c, 8)
    e1 = E.Engine(s, E.Arena(c), E.HyperParams(lr=2e-3, weight_decay=0.01),
                  E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=4,
                                  overlap_optimizer_tail=True, tail_blocks=1, **res))
    l1 = [e1.train_step(t) for t in toks]
    assert validate_trace(e1.last_trace(), c.layers) == []
    # save brings the store up to date itself (quiesce hook: optimizer tail + resident
    # write-back), so the file holds the state after step 3 of every tile
    ck = str(tmp_path / "now.hlm2")
    s.save(ck)
    assert l0 == [r.loss for r in l1]
    assert ref.bitwise_equal(s)
    back = E.Store(c, 1)
    back.load(ck)
    assert back.bitwise_equal(ref)
    streamed = 2 * (c.vocab * c.hidden * (0 if res.get("resident_embed") else 1) +
                    c.vocab * c.hidden + 2 * (c.layers - res.get("resident_blocks", 0)) * c.block_params())
    assert l1[-1].h2d_bytes == streamed


@pytest.mark.parametrize("opts", [dict(saved_act_layers=2), dict(saved_act_layers=6),
                                  dict(saved_act_layers=3, resident_blocks=4, resident_embed=True)])
def test_saved_activations_are_bitwise_neutral(opts):
    """Top blocks' forward activations kept in HBM (no recompute in their backward):
    the same losses and store bit for bit, and that many fewer recompute forwards."""
    from paper_2602_04816_b200.trace import validate_trace
    c = E.ModelConfig(6, 32, 64, 32, 16, 2, k_ckpt=1, n_heads=2, rope_theta=1e4)
    toks = [E.make_copy_task_batch(c, 4, skip=i) for i in range(3)]
    hp = E.HyperParams(lr=2e-3, weight_decay=0.01)
    ref = E.Store(c, 8)
    e0 = E.Engine(ref, E.Arena(c), hp, E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=4))
    l0 = [e0.train_step(t).loss for t in toks]
    e0.sync()
    s = E.Store(c, 8)
    o = dict(eager_optim=True, threaded_accum=True, n_slab=4, overlap_optimizer_tail=True, tail_blocks=1)
    o.update(opts)
    e1 = E.Engine(s, E.Arena(c), hp, E.EngineOptions(**o))
    l1 = [e1.train_step(t) for t in toks]
    assert validate_trace(e1.last_trace(), c.layers) == []
    e1.sync()
    assert l0 == [r.loss for r in l1]
    assert ref.bitwise_equal(s)
    assert l1[-1].recompute_forwards == c.layers - opts["saved_act_layers"]


@pytest.mark.parametrize("pieces", [dict(piece_elems=1000), dict(piece_elems=4096, head_piece_vocab=8),
                                    dict(piece_elems=1000, grad_buffers=5), dict(sparse_embed_grad=True),
                                    dict(sparse_embed_grad=True, piece_elems=700, grad_buffers=3),
                                    dict(embed_gather_host=True, sparse_embed_grad=True)])
def test_piecewise_transfers_are_bitwise_neutral(pieces):
    """Gradients landing in pieces with the host Adam piece by piece, and the
    forward H2D of cached blocks copied piece by piece behind the optimizer:
    the same losses and store, bit for bit, as whole-tile transfers."""
    from paper_2602_04816_b200.trace import validate_trace
    c = E.ModelConfig(6, 32, 64, 40, 16, 2, k_ckpt=1, n_heads=2, rope_theta=1e4)
    toks = [E.make_copy_task_batch(c, 6, skip=i) for i in range(4)]
    blk = (2 * c.block_params() + 255) // 256 * 256
    hp = E.HyperParams(lr=2e-3)
    res = []
    for kw in (dict(head_piece_vocab=-1), pieces):
        s = E.Store(c, 12)
        e = E.Engine(s, E.Arena(c, weight_cache_bytes=c.layers * blk), hp,
                     E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=c.layers + 4,
                                     overlap_optimizer_tail=True, tail_blocks=c.layers, **kw))
        losses = [e.train_step(t).loss for t in toks]
        assert validate_trace(e.last_trace(), c.layers) == []
        e.sync()
        res.append((losses, s))
    if "head_piece_vocab" in pieces:     # vocab-chunked head: d_x summed in another order
        assert res[0][0][0] == res[1][0][0]
        assert np.allclose(res[0][0], res[1][0], rtol=1e-4)
    else:
        assert res[0][0] == res[1][0]
        assert res[0][1].bitwise_equal(res[1][1])


def test_sparse_embedding_gradient_non_finite_names_the_table_element():
    c = E.ModelConfig(2, 16, 32, 13, 4, 1)
    s = E.Store(c, 5, "fp32")
    w = s.weights()
    tok = E.make_copy_task_batch(c, 2)
    w[int(tok[0]) * c.hidden + 3] = np.inf   # an embedding row the batch reads
    s.import_master(w)
    e = E.Engine(s, E.Arena(c), E.HyperParams(), E.EngineOptions(eager_optim=True, sparse_embed_grad=True))
    with pytest.raises(E.NumericsError, match="non-finite gradient in layer"):
        e.train_step(tok)


def test_bench_feature_set_tracks_oracle_for_20_steps():
    """Every scheduling feature the bench turns on — gradient / weight pieces, the
    vocab-chunked head, row-sparse embedding gradient, zero-copy embedding gather, extra
    gradient buffers, the optimizer tail over every block, the weight cache, pinned
    optimizer threads — over 20 training steps of the Qwen-style config (2 heads, RoPE)
    against the oracle's mixed-precision trajectory (per-step loss within 1 %)."""
    c = E.ModelConfig(4, 64, 128, 96, 32, 4, k_ckpt=1, n_heads=2, rope_theta=1e4)
    s = E.Store(c, 1234)
    blk = (2 * c.block_params() + 255) // 256 * 256
    e = E.Engine(s, E.Arena(c, weight_cache_bytes=c.layers * blk), E.HyperParams(lr=3e-3),
                 E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=c.layers + 4,
                                 overlap_optimizer_tail=True, tail_blocks=c.layers, piece_elems=5000,
                                 head_piece_vocab=16, sparse_embed_grad=True, embed_gather_host=True,
                                 grad_buffers=6))
    toks = [E.make_copy_task_batch(c, 1235, skip=i) for i in range(20)]   # run_training's data stream
    losses = [e.train_step(t).loss for t in toks]
    e.sync()
    ref, _ = O.Oracle().train(ocfg(c), O.hyper(lr=3e-3), 1234, "mixed", 20)
    l = np.array(losses)
    assert np.all(np.abs(l - ref) / ref < 1e-2), (l, ref)
    assert l[-1] < 0.9 * l[0]


def test_save_right_after_train_step_waits_for_the_optimizer_tail(tmp_path):
    """with an overlapped optimizer tail, train_step returns while the head and
    top blocks are still being optimised on the worker; a save right then must not mix
    tiles from two steps under a header that says step t."""
    c = E.ModelConfig(6, 32, 64, 32, 16, 2, k_ckpt=1, n_heads=2, rope_theta=1e4)
    toks = [E.make_copy_task_batch(c, 4, skip=i) for i in range(3)]
    hp = E.HyperParams(lr=2e-3, weight_decay=0.01)
    ref = E.Store(c, 8)
    e0 = E.Engine(ref, E.Arena(c), hp, E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=4))
    for t in toks:
        e0.train_step(t)
    e0.sync()
    s = E.Store(c, 8)
    e1 = E.Engine(s, E.Arena(c), hp,
                  E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=4, overlap_optimizer_tail=True,
                                  tail_blocks=6, accum_delay_us=2000))
    for t in toks:
        e1.train_step(t)
    s.save(tmp_path / "tail.hlm2")   # no sync(): the tail is still running (accum_delay_us)
    r = E.Store(c, 1)
    r.load(tmp_path / "tail.hlm2")
    assert r.adam_steps == 3 and r.bitwise_equal(ref)


def test_load_checkpoint_reuploads_hbm_resident_tiles(tmp_path):
    """load_checkpoint into a store whose live engine keeps HBM-resident tiles:
    the engine must train on the loaded state, not on its stale device copy (which its
    next sync() would otherwise write over the load)."""
    c = E.ModelConfig(6, 32, 64, 32, 16, 2, k_ckpt=1, n_heads=2, rope_theta=1e4)
    toks = [E.make_copy_task_batch(c, 4, skip=i) for i in range(3)]
    hp = E.HyperParams(lr=2e-3, weight_decay=0.01)
    ref = E.Store(c, 8)
    e0 = E.Engine(ref, E.Arena(c), hp, E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=4))
    l0 = [e0.train_step(t).loss for t in toks]
    e0.sync()
    s = E.Store(c, 8)
    e1 = E.Engine(s, E.Arena(c), hp,
                  E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=4, resident_embed=True,
                                  resident_blocks=3, overlap_optimizer_tail=True, tail_blocks=1))
    e1.train_step(toks[0])
    e1.train_step(toks[1])
    s.save(tmp_path / "two.hlm2")
    first = e1.train_step(toks[2]).loss
    s.load(tmp_path / "two.hlm2")    # back to the state after step 2
    again = e1.train_step(toks[2]).loss
    e1.sync()
    assert first == l0[2] and again == l0[2]
    assert s.adam_steps == 3 and s.bitwise_equal(ref)


def test_removed_transit_field_is_rejected():
    """The removed transit-tile mode keeps its C-ABI field (layout) and refuses non-zero."""
    c = E.ModelConfig(2, 16, 32, 13, 4, 1)
    o = E.EngineOptions(eager_optim=True)
    o.reserved_transit_blocks = 1
    with pytest.raises(E.HlmConfigError, match="transit"):
        E.Engine(E.Store(c, 5), E.Arena(c), E.HyperParams(), o)
