"""Host-side C++ (libhlm_b200.so) on CPU only: store init, Adam, token
stream, footprint formulas, C-ABI symbol surface. No GPU calls (pinning off)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_2602_04816_b200 import _lib
from paper_2602_04816_b200 import engine as E

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_declared_symbol_is_exported():
    hdr = open(os.path.join(ROOT, "include", "hlm_cuda.h")).read()
    names = set(re.findall(r"\b(hlm_[a-z0-9_]+)\s*\(", hdr))
    lib = _lib.lib()
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert len(names) > 30


@pytest.mark.parametrize("name", ["tiny", "desk", "acc_tied"])
def test_store_init_bitwise_reference(name):
    z = np.load(os.path.join(GOLD, f"ref_{name}.npz"))
    import ast
    kw = ast.literal_eval(str(z["cfg_json"]))
    c = E.ModelConfig(kw["layers"], kw["hidden"], kw["ffn"], kw["vocab"], kw["seq"], kw["batch"],
                      kw["k_ckpt"], kw.get("tie", False))
    seed = int(z["seed"])
    assert np.array_equal(E.Store(c, seed, "bf16", pin=False).weights().view(np.uint32),
                          z["w16"].view(np.uint32))
    s32 = E.Store(c, seed, "fp32", pin=False)
    assert np.array_equal(s32.weights().view(np.uint32), z["w32"].view(np.uint32))
    # the transfer shadow is RNE(master), reference bf16.hpp semantics
    assert np.array_equal(s32.export(E.FIELD_SHADOW), z["w16"])
    assert np.array_equal(E.make_copy_task_batch(c, seed + 1), z["tokens"])


def test_parallel_init_is_deterministic_and_trunc_normal():
    c = E.ModelConfig(2, 64, 128, 512, 8, 2)
    a = E.Store(c, 7, "fp32", init="parallel", pin=False).weights()
    b = E.Store(c, 7, "fp32", init="parallel", pin=False).weights()
    assert np.array_equal(a, b)
    mats = a[:512 * 64]
    assert abs(mats.mean()) < 1e-3 and 0.015 < mats.std() < 0.02 and np.abs(mats).max() <= 0.04
    # norms are 1.0
    blk = a[512 * 64: 512 * 64 + c.block_params()]
    assert np.all(blk[-2 * 64:] == 1.0)


def test_adam_bitwise_vs_oracle_and_known_answer():
    c = E.ModelConfig(2, 16, 32, 13, 4, 1)
    s = E.Store(c, 3, "fp32", pin=False)
    orc = O.Oracle()
    rng = np.random.default_rng(0)
    w = s.weights().copy(); m = np.zeros_like(w); v = np.zeros_like(w)
    for t in (1, 2, 3, 4):
        g = (rng.standard_normal(w.size) * 1e-2).astype(np.float32)
        s.adam_step(g, E.HyperParams(lr=3e-3, weight_decay=0.01), t)
        orc.adam(O.hyper(lr=3e-3, weight_decay=0.01), t, w, g, m, v)
    assert np.array_equal(s.weights(), w)
    assert np.array_equal(s.export(E.FIELD_M), m)
    assert np.array_equal(s.export(E.FIELD_V), v)
    assert s.adam_steps == 4
    # shadow tracks the master (RNE)
    sh = s.export(E.FIELD_SHADOW)
    assert np.array_equal(sh, (w.view(np.uint32) + 0x7FFF + ((w.view(np.uint32) >> 16) & 1) >> 16
                               << 16).astype(np.uint32).view(np.float32))


def test_adam_rejects_non_finite_gradient_without_mutation():
    c = E.ModelConfig(2, 16, 32, 13, 4, 1)
    s = E.Store(c, 3, "fp32", pin=False)
    before = s.weights().copy()
    g = np.zeros(s.total_params, np.float32)
    g[5] = np.nan
    with pytest.raises(E.NumericsError, match="non-finite gradient in layer 0 at element 5"):
        s.adam_step(g, E.HyperParams(), 1)
    assert np.array_equal(s.weights(), before)


def test_config_validation():
    with pytest.raises(E.HlmConfigError):
        E.Store(E.ModelConfig(2, 12, 32, 13, 4, 1), 1, pin=False)        # hidden % 8
    with pytest.raises(E.HlmConfigError):
        E.Store(E.ModelConfig(2, 16, 32, 13, 4, 1, k_ckpt=3), 1, pin=False)  # K > L
    with pytest.raises(E.HlmConfigError):
        E.Store(E.ModelConfig(2, 16, 32, 13, 4, 1, n_heads=3), 1, pin=False)


def test_footprint_is_depth_invariant_except_anchors():
    a = E.arena_footprint(E.ModelConfig(4, 64, 128, 100, 16, 2))
    b = E.arena_footprint(E.ModelConfig(40, 64, 128, 100, 16, 2))
    assert a["stream_buf"] == b["stream_buf"] and a["stack"] == b["stack"]
    assert a["workspace"] == b["workspace"]
    assert b["anchor_slots"] == 41 and a["anchor_slots"] == 5
    assert a["anchor_slot"] == 4 * 2 * 16 * 64


def test_train_rejects_unknown_keys():
    with pytest.raises(E.HlmConfigError):
        E.train({"model": {}, "bogus": 1})


def test_checkpoint_roundtrip_and_geometry_checks(tmp_path):
    c = E.ModelConfig(2, 16, 32, 13, 4, 1)
    s = E.Store(c, 3, "fp32", pin=False)
    rng = np.random.default_rng(0)
    for t in (1, 2):
        s.adam_step((rng.standard_normal(s.total_params) * 1e-2).astype(np.float32), E.HyperParams(), t)
    p = tmp_path / "a.hlm2"
    s.save(p)
    r = E.Store(c, 99, "bf16", pin=False)
    r.load(p)
    assert r.bitwise_equal(s) and r.adam_steps == 2
    with pytest.raises(E.HlmConfigError, match="geometry"):
        E.Store(E.ModelConfig(3, 16, 32, 13, 4, 1), 1, pin=False).load(p)
    (tmp_path / "bad").write_bytes(b"HLMxxxxxxxxx")
    with pytest.raises(E.HlmConfigError, match="not an HLM2 or HLM1"):
        r.load(tmp_path / "bad")
    # an HLM1 header is parsed as the reference's container (tests/test_hlm1.py), with its checks
    (tmp_path / "bad1").write_bytes(b"HLM1xxxxxxxx")
    with pytest.raises(E.HlmConfigError, match="unsupported HLM1 version"):
        r.load(tmp_path / "bad1")


def test_sparse_embedding_adam_is_bitwise_the_dense_adam():
    """The engine's row-sparse embedding update (zero rows optimised without reading a
    gradient) equals the dense host Adam on the same gradient, bit for bit, including
    the BF16 shadow; over several steps with weight decay."""
    from paper_2602_04816_b200 import engine as E
    c = E.ModelConfig(2, 48, 96, 57, 8, 2)
    dense, sparse = E.Store(c, 31), E.Store(c, 31)
    hp = E.HyperParams(lr=3e-3, weight_decay=0.05)
    rng = np.random.default_rng(0)
    n_tab = c.vocab * c.hidden
    for t in range(1, 4):
        rows = np.sort(rng.choice(c.vocab, size=13, replace=False)).astype(np.int32)
        compact = rng.standard_normal((len(rows), c.hidden)).astype(np.float32)
        g = np.zeros(dense.total_params, np.float32)
        g[:n_tab].reshape(c.vocab, c.hidden)[rows] = compact
        dense.adam_step(g, hp, t)
        sparse.adam_embed_rows(rows, compact, hp, t)
        wd, ws = dense.export(E.FIELD_MASTER), sparse.export(E.FIELD_MASTER)
        assert np.array_equal(wd[:n_tab].view(np.uint32), ws[:n_tab].view(np.uint32))
    for field in (E.FIELD_MASTER, E.FIELD_M, E.FIELD_V, E.FIELD_SHADOW):
        a, b = dense.export(field)[:n_tab], sparse.export(field)[:n_tab]
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), field


def _cpu_slice(rank, gpu_nodes, allowed, online, node_of_cpu):
    lib = _lib.lib()
    I = ctypes.c_int
    arr = lambda xs: (I * max(1, len(xs)))(*xs)
    out = (I * 256)()
    n = lib.hlm_rank_cpu_slice(I(rank), arr(gpu_nodes), I(len(gpu_nodes)), arr(allowed), I(len(allowed)), I(online),
                               arr(node_of_cpu), I(len(node_of_cpu)), out, I(256))
    assert n >= 0
    return list(out[:n])


def test_rank_cpu_slices_follow_gpu_numa_nodes_and_never_overlap():
    """N data-parallel ranks on one host split the optimizer CPUs: each rank takes
    its share of its GPU's socket; unknown topology splits the whole set; a process
    the launcher already bound, or a single rank, keeps its affinity."""
    node_of = [0] * 8 + [1] * 8
    two_socket = [_cpu_slice(r, [0, 0, 1, 1], list(range(16)), 16, node_of) for r in range(4)]
    assert two_socket == [[0, 1, 2, 3], [4, 5, 6, 7], [8, 9, 10, 11], [12, 13, 14, 15]]
    # 8 ranks, GPUs 0-3 on socket 0 and 4-7 on socket 1, hyperthreads numbered after cores
    node_of = ([0] * 4 + [1] * 4) * 2
    sl = [_cpu_slice(r, [0] * 4 + [1] * 4, list(range(16)), 16, node_of) for r in range(8)]
    assert all(len(s) == 2 and all(node_of[c] == (r >= 4) for c in s) for r, s in enumerate(sl))
    assert sorted(c for s in sl for c in s) == list(range(16))
    unknown = [_cpu_slice(r, [-1, -1], list(range(16)), 16, []) for r in range(2)]
    assert unknown == [list(range(8)), list(range(8, 16))]
    assert _cpu_slice(1, [0, 1], [2, 3, 4], 16, [0] * 8 + [1] * 8) == [2, 3, 4]   # launcher-bound
    assert _cpu_slice(0, [0], list(range(16)), 16, [0] * 16) == list(range(16))
    # a node with no allowed CPU (memory-only node) falls back to the whole set
    assert _cpu_slice(0, [2, 2], list(range(4)), 4, [0] * 4) == [0, 1]


_ISA_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2602_04816_b200 import engine as E, _lib
import ctypes
L = _lib.lib(); L.hlm_host_isa.restype = ctypes.c_char_p
c = E.ModelConfig(2, 64, 96, 37, 4, 1)
s = E.Store(c, 3, "fp32", pin=False, init="parallel")
rng = np.random.default_rng(0)
for t in (1, 2, 3):
    g = (rng.standard_normal(s.total_params) * 1e-2).astype(np.float32)
    g[::7] = 0.0
    s.adam_step(g, E.HyperParams(lr=3e-3, weight_decay=0.01), t)
rows = np.array([0, 3, 4, 36], np.int32)
s.adam_embed_rows(rows, (rng.standard_normal(4 * 64) * 1e-2).astype(np.float32), E.HyperParams(), 4)
bad = np.zeros(s.total_params, np.float32); bad[1001] = np.inf
try:
    s.adam_step(bad, E.HyperParams(), 5); rejected = False
except E.NumericsError:
    rejected = True
np.savez(sys.argv[2], isa=L.hlm_host_isa().decode(), rejected=rejected,
         **{f: s.export(k) for f, k in (("w", E.FIELD_MASTER), ("m", E.FIELD_M), ("v", E.FIELD_V),
                                       ("sh", E.FIELD_SHADOW))})
"""


def test_portable_host_isa_is_bitwise_equal_to_avx512(tmp_path):
    """The library targets x86-64-v3 and picks AVX-512 host loop bodies at run time; the
    portable bodies (HLM_HOST_ISA=generic, what a host without AVX-512 runs) give the
    same bits for Adam (dense and row-sparse), BF16 packing and the finiteness check."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "isa.py"
    script.write_text(_ISA_SCRIPT)
    out = {}
    for isa in ("default", "generic"):
        env = dict(os.environ)
        if isa == "generic":
            env["HLM_HOST_ISA"] = "generic"
        dst = tmp_path / f"{isa}.npz"
        subprocess.run([sys.executable, str(script), root, str(dst)], check=True, env=env)
        out[isa] = np.load(dst)
    assert str(out["generic"]["isa"]) == "generic"
    for f in ("w", "m", "v", "sh"):
        assert np.array_equal(out["default"][f].view(np.uint32), out["generic"][f].view(np.uint32)), f
    assert bool(out["default"]["rejected"]) and bool(out["generic"]["rejected"])
