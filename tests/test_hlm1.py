"""HLM1 (the reference's checkpoint container) through our store.

A reference user's checkpoints (/root/reference/proj/src/checkpoint.cpp:38-120) load into
our store with hlm_store_load / hlm::load_checkpoint, and hlm_store_save_hlm1 /
hlm::save_checkpoint_hlm1 writes files the reference's loader reads. Golden files
(tests/golden/ref_*.hlm1) were written by the reference's own save_checkpoint after 3
Adam steps of run_training (tests/golden/make_golden.py); the checker is
oracle.read_hlm1, a numpy restatement of the container that was itself checked against
the reference loader when the fixtures were made (and live below when oracle/_ref exists).
"""
import os

import numpy as np
import pytest

import oracle as O
from paper_2602_04816_b200 import engine as E

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CONFIGS = {   # tests/golden/make_golden.py CONFIGS
    "tiny": dict(layers=2, hidden=8, ffn=16, vocab=11, seq=4, batch=1, k_ckpt=1),
    "acc_tied": dict(layers=4, hidden=8, ffn=24, vocab=11, seq=8, batch=2, k_ckpt=3, tie=True),
}
FILES = [("tiny", "bf16"), ("acc_tied", "fp32")]


def ecfg(kw):
    return E.ModelConfig(kw["layers"], kw["hidden"], kw["ffn"], kw["vocab"], kw["seq"], kw["batch"],
                         k_ckpt=kw["k_ckpt"], tie_embeddings=kw.get("tie", False))


def flat(d, key):
    return np.concatenate([t[key] for t in d["tiles"]])


def shadow_f32(store):
    return store.export(E.FIELD_SHADOW)


@pytest.mark.parametrize("name,dtype", FILES)
def test_reference_hlm1_loads_bitwise(name, dtype):
    path = os.path.join(GOLD, f"ref_{name}_{dtype}.hlm1")
    want = O.read_hlm1(path)
    assert want["dtype"] == dtype and want["adam_steps"] == 3
    s = E.Store(ecfg(CONFIGS[name]), 99, dtype, pin=False)   # different init: every value comes from the file
    s.load(path)
    assert s.adam_steps == 3
    assert np.array_equal(s.weights().view(np.uint32), flat(want, "weights").view(np.uint32))
    assert np.array_equal(s.export(E.FIELD_M).view(np.uint32), flat(want, "m").view(np.uint32))
    assert np.array_equal(s.export(E.FIELD_V).view(np.uint32), flat(want, "v").view(np.uint32))
    if dtype == "bf16":   # the reference BF16 weights are already rounded: shadow == master
        assert np.array_equal(shadow_f32(s).view(np.uint32), s.weights().view(np.uint32))


def trained_store(name, dtype):
    kw = CONFIGS[name]
    c = ecfg(kw)
    s = E.Store(c, 5, dtype, pin=False)
    rng = np.random.default_rng(3)
    hp = E.HyperParams(lr=3e-3)
    for t in (1, 2):
        s.adam_step(rng.standard_normal(s.total_params).astype(np.float32) * 1e-2, hp, t)
    return s


@pytest.mark.parametrize("name,dtype", FILES)
def test_save_hlm1_layout_and_roundtrip(tmp_path, name, dtype):
    s = trained_store(name, dtype)
    path = tmp_path / "x.hlm1"
    s.save_hlm1(path)
    got = O.read_hlm1(str(path))
    assert got["dtype"] == dtype and got["adam_steps"] == 2
    want_alias = [0, 1, 2, 3, 4, 0] if CONFIGS[name].get("tie") else list(range(CONFIGS[name]["layers"] + 2))
    assert list(got["alias"]) == want_alias
    # weights as the reference store holds them: RNE(master) for BF16, the master for FP32
    w = shadow_f32(s) if dtype == "bf16" else s.weights()
    assert np.array_equal(flat(got, "weights").view(np.uint32), w.view(np.uint32))
    assert np.array_equal(flat(got, "m").view(np.uint32), s.export(E.FIELD_M).view(np.uint32))
    assert np.array_equal(flat(got, "v").view(np.uint32), s.export(E.FIELD_V).view(np.uint32))
    r = E.Store(ecfg(CONFIGS[name]), 77, dtype, pin=False)
    r.load(path)
    assert r.adam_steps == 2
    assert np.array_equal(r.weights().view(np.uint32), w.view(np.uint32))
    assert np.array_equal(r.export(E.FIELD_M).view(np.uint32), s.export(E.FIELD_M).view(np.uint32))
    assert np.array_equal(r.export(E.FIELD_V).view(np.uint32), s.export(E.FIELD_V).view(np.uint32))


@pytest.mark.skipif(not O.Reference.available(), reason="oracle/_ref not built (no reference tree)")
@pytest.mark.parametrize("name,dtype", FILES)
def test_reference_loader_reads_our_hlm1(tmp_path, name, dtype):
    s = trained_store(name, dtype)
    path = tmp_path / "ours.hlm1"
    s.save_hlm1(path)
    kw = CONFIGS[name]
    w, m, v, steps = O.Reference().load_hlm1(O.cfg(**kw), dtype == "bf16", str(path))
    assert steps == 2
    assert np.array_equal(w.view(np.uint32), (shadow_f32(s) if dtype == "bf16" else s.weights()).view(np.uint32))
    assert np.array_equal(m.view(np.uint32), s.export(E.FIELD_M).view(np.uint32))
    assert np.array_equal(v.view(np.uint32), s.export(E.FIELD_V).view(np.uint32))


def test_hlm1_mismatch_is_rejected_with_the_reference_messages():
    tiny = os.path.join(GOLD, "ref_tiny_bf16.hlm1")
    wrong_depth = E.Store(ecfg(dict(CONFIGS["tiny"], layers=3)), 1, "bf16", pin=False)
    with pytest.raises(Exception, match="tile count does not match the model"):
        wrong_depth.load(tiny)
    wrong_dtype = E.Store(ecfg(CONFIGS["tiny"]), 1, "fp32", pin=False)
    with pytest.raises(Exception, match="dtype does not match the store"):
        wrong_dtype.load(tiny)
    wrong_width = E.Store(ecfg(dict(CONFIGS["tiny"], ffn=24)), 1, "bf16", pin=False)
    with pytest.raises(Exception, match="parameter count does not match the model"):
        wrong_width.load(tiny)


@pytest.mark.gpu
def test_training_resumes_from_a_reference_checkpoint():
    """The reference trained 3 BF16 steps and saved HLM1; our engine loads it and runs steps
    4-5 of the same run_training (data stream replayed from the step count). Step 4 starts
    from the reference's exact state, so its loss differs only by BF16-compute noise; step 5
    also carries the FP32-master difference (the reference re-rounds weights every step).
    lr 1e-2: consecutive losses differ by 0.37 % / 0.72 %, so a resume from the wrong state
    (a step early or late) fails the bounds; the oracle's mixed-precision trajectory sits
    within 4e-5 of the reference's here."""
    z = np.load(os.path.join(GOLD, "ref_resume.npz"))
    c = E.ModelConfig(2, 32, 64, 32, 16, 2, k_ckpt=1)
    s = E.Store(c, 1)
    s.load(os.path.join(GOLD, "ref_resume_bf16.hlm1"))
    assert s.adam_steps == 3
    losses = s.run_training(E.HyperParams(lr=float(z["lr"])), int(z["seed"]), 2,
                            E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=4))
    ref = z["losses16"]
    rel = np.abs(losses - ref[3:5]) / ref[3:5]
    assert rel[0] < 1e-3 and rel[1] < 2e-3, (losses, ref)
    assert np.argmin(np.abs(ref - losses[0])) == 3 and np.argmin(np.abs(ref - losses[1])) == 4
