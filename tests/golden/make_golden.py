"""Regenerate tests/golden/*.npz from the REFERENCE library itself
(oracle/_ref/libhlm_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile). Run here (the reference tree is absent on the GPU box):

    make -C oracle && python tests/golden/make_golden.py

Every array is computed by reference code: build_store, make_copy_task_batch,
Engine::train_step (skip_optimizer), oracle_forward_backward, run_training and
bf16_bits_from_f32.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# Reference test fixtures (proj/tests/helpers.hpp:41-64, acceptance_main.cpp:94-135)
CONFIGS = {
    "tiny": dict(layers=2, hidden=8, ffn=16, vocab=11, seq=4, batch=1, k_ckpt=1),
    "desk": dict(layers=4, hidden=32, ffn=64, vocab=32, seq=16, batch=2, k_ckpt=2),
    "acc3": dict(layers=3, hidden=16, ffn=32, vocab=13, seq=8, batch=2, k_ckpt=2),
    "acc_tied": dict(layers=4, hidden=8, ffn=24, vocab=11, seq=8, batch=2, k_ckpt=3, tie=True),
    "copytask": dict(layers=4, hidden=32, ffn=64, vocab=32, seq=16, batch=8, k_ckpt=2),
}

# bf16 bit table of reference tests/test_bf16.cpp:74-88
BF16_TABLE = [
    (0x3F800000, 0x3F80), (0x3F800001, 0x3F80), (0x3F808000, 0x3F80), (0x3F818000, 0x3F82),
    (0x3F807FFF, 0x3F80), (0x3F808001, 0x3F81), (0x7F7FFFFF, 0x7F80), (0x7F7F0000, 0x7F7F),
    (0x00000000, 0x0000), (0x80000000, 0x8000), (0x7F800000, 0x7F80), (0xFF800000, 0xFF80),
    (0x7FC00000, 0x7FC0), (0x7F800001, 0x7FC0), (0x00008000, 0x0000), (0x00018000, 0x0002),
    (0x3DCCCCCD, 0x3DCD), (0xC2480000, 0xC248), (0x42F6E979, 0x42F7), (0xB8D1B717, 0xB8D2),
]


def main():
    ref = O.Reference()
    # bf16 table checked through the reference's own conversion
    rng = np.random.default_rng(7)
    rand_bits = rng.integers(0, 2**32, size=4096, dtype=np.uint64).astype(np.uint32)
    ref_bits = np.array([ref.bf16_bits(float(np.uint32(b).view(np.float32))) for b in rand_bits],
                        np.uint16)
    table_in = np.array([a for a, _ in BF16_TABLE], np.uint32)
    table_out = np.array([ref.bf16_bits(float(np.uint32(a).view(np.float32))) for a in table_in],
                         np.uint16)
    assert list(table_out) == [b for _, b in BF16_TABLE], "reference disagrees with its own table"
    np.savez_compressed(os.path.join(OUT, "bf16.npz"), table_in=table_in, table_out=table_out,
                        rand_in=rand_bits, rand_out=ref_bits)

    for name, kw in CONFIGS.items():
        c = O.cfg(**kw)
        seed = 1000 + kw["layers"]
        w32 = ref.init_weights(c, seed, False)
        w16 = ref.init_weights(c, seed, True)
        tokens = ref.copy_task_tokens(c, seed + 1, 0)
        loss32, g32 = ref.grad_step(c, seed, False, tokens)
        loss16, g16 = ref.grad_step(c, seed, True, tokens)
        ofb_loss, ofb_g = ref.oracle_fb(c, w16, tokens)   # tape oracle on bf16-widened weights
        hp = O.hyper(lr=3e-3)
        tl32, tw32 = ref.train(c, hp, seed, False, 8)
        tl16, tw16 = ref.train(c, hp, seed, True, 8)
        np.savez_compressed(os.path.join(OUT, f"ref_{name}.npz"), cfg_json=str(kw),
                            seed=seed, w32=w32, w16=w16, tokens=tokens, loss32=loss32, g32=g32,
                            loss16=loss16, g16=g16, ofb_loss=ofb_loss, ofb_g=ofb_g,
                            train_losses32=tl32, train_w32=tw32, train_losses16=tl16,
                            train_w16=tw16)
        print(name, "loss32", loss32, "loss16", loss16)

    # C1: store seed 1234, data seed 1235, lr 3e-3, 3 steps
    c1 = O.cfg(4, 256, 1024, 1024, 128, 4, k_ckpt=1)
    tok = ref.copy_task_tokens(c1, 1235, 0)
    l32, _ = ref.train(c1, O.hyper(lr=3e-3), 1234, False, 3)
    l16, _ = ref.train(c1, O.hyper(lr=3e-3), 1234, True, 3)
    np.savez_compressed(os.path.join(OUT, "ref_c1.npz"), tokens=tok, losses32=l32, losses16=l16)
    print("c1", l32, l16, tok[:8])

    # HLM1 checkpoints written by the reference's save_checkpoint after 3 Adam steps
    # (proj/src/checkpoint.cpp:38-69): a BF16 store, and a tied FP32 store (alias table)
    for name, bf16 in (("tiny", True), ("acc_tied", False)):
        kw = CONFIGS[name]
        path = os.path.join(OUT, f"ref_{name}_{'bf16' if bf16 else 'fp32'}.hlm1")
        ref.train_save_hlm1(O.cfg(**kw), O.hyper(lr=3e-3), 1000 + kw["layers"], bf16, 3, path)
        print("hlm1", path, os.path.getsize(path))
    # resume from a reference checkpoint on the GPU engine: HLM1 after 3 BF16 steps and the
    # reference's own 5-step loss trajectory from the same seed (steps 4-5 = the resume)
    rkw = dict(layers=2, hidden=32, ffn=64, vocab=32, seq=16, batch=2, k_ckpt=1)
    rc = O.cfg(**rkw)
    ref.train_save_hlm1(rc, O.hyper(lr=1e-2), 1234, True, 3, os.path.join(OUT, "ref_resume_bf16.hlm1"))
    rl, _ = ref.train(rc, O.hyper(lr=1e-2), 1234, True, 5)
    np.savez_compressed(os.path.join(OUT, "ref_resume.npz"), cfg_json=str(rkw), seed=1234, lr=1e-2,
                        losses16=rl)
    print("resume", rl)

    # acceptance criterion 8 (proj/test_output.txt:20): 200-step fp32 copy task, seed 1234
    cc = O.cfg(**CONFIGS["copytask"])
    l200, _ = ref.train(cc, O.hyper(lr=3e-3), 1234, False, 200)
    np.savez_compressed(os.path.join(OUT, "ref_copytask200.npz"), losses=l200)
    print("copytask200", l200[0], l200[-1])


if __name__ == "__main__":
    main()
