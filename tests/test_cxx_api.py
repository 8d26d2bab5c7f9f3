"""The C++ boundary: a reference-style C++ caller (tests/cxx/integration_caller.cpp, the
INTEGRATION.md §1 snippet) compiles against include/hlm/*.hpp and links against
libhlm_b200.so — the drop-in the reference's own callers need
(proj/tools/hlm_main.cpp:191-236, proj/src/trainer.cpp:8-42,
proj/python/bindings.cpp:79-96) — and on the GPU trains bit-identically to the C-ABI path.

CPU: compile + link, the exported C++ symbol set, and a link next to the reference's
own object files (the inline namespace hlm::b200 keeps the two libraries apart).
GPU: the caller's losses equal the ctypes (C ABI) path's bit for bit, the phase API
matches train_step, and the reference's exception types cross the library boundary.
"""
import glob
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2602_04816_b200")
SRC = os.path.join(ROOT, "tests", "cxx", "integration_caller.cpp")
REF_OBJ = os.path.join(ROOT, "oracle", "_ref", "obj")

# The reference C++ API a caller binds (proj/include/hlm/*.hpp), by demangled prefix.
REQUIRED = [
    "hlm::b200::Engine::Engine(",
    "hlm::b200::Engine::train_step(",
    "hlm::b200::Engine::begin_step(",
    "hlm::b200::Engine::forward_streaming(",
    "hlm::b200::Engine::anchor_loss(",
    "hlm::b200::Engine::backward_blockwise(",
    "hlm::b200::Engine::finish_step(",
    "hlm::b200::Engine::~Engine(",
    "hlm::b200::build_store(",
    "hlm::b200::adam_step(",
    "hlm::b200::adam_step_tile(",
    "hlm::b200::DeviceArena::DeviceArena(",
    "hlm::b200::make_copy_task_batch(",
    "hlm::b200::run_training(",
    "hlm::b200::save_checkpoint(",
    "hlm::b200::load_checkpoint(",
    "hlm::b200::save_checkpoint_hlm1(",
    "typeinfo for hlm::b200::ArenaOomError",
    "typeinfo for hlm::b200::ProtocolError",
]


def _compile(out, extra=()):
    cmd = ["g++", "-std=c++17", "-O2", f"-I{ROOT}/include", SRC, *extra, f"-L{LIBDIR}",
           "-lhlm_b200", f"-Wl,-rpath,{LIBDIR}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return out


@pytest.fixture(scope="module")
def caller(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    return _compile(str(tmp_path_factory.mktemp("cxx") / "integration_caller"))


def test_caller_compiles_and_links(caller):
    r = subprocess.run([caller], capture_output=True, text=True)
    assert r.returncode == 64 and "usage" in r.stderr


def test_library_exports_the_reference_cxx_api():
    so = os.path.join(LIBDIR, "libhlm_b200.so")
    out = subprocess.run(["nm", "-DC", "--defined-only", so], capture_output=True, text=True,
                         check=True).stdout
    missing = [s for s in REQUIRED if s not in out]
    assert not missing, missing
    # nothing of the CUDA runtime or the kernels leaks out of the library
    names = [ln.split(" ", 2)[-1] for ln in out.splitlines() if ln.strip()]
    stray = [n for n in names if not (n.startswith("hlm_") or "hlm::b200::" in n)]
    assert not stray, stray[:10]


@pytest.mark.skipif(not glob.glob(os.path.join(REF_OBJ, "*.o")),
                    reason="reference objects not built (oracle/_ref is built only where "
                           "/root/reference exists)")
def test_links_beside_the_reference_core(tmp_path):
    """The reference's libhlm_core objects (namespace hlm) and libhlm_b200.so
    (hlm::b200) link into one executable without a duplicate or mis-bound symbol."""
    objs = sorted(glob.glob(os.path.join(REF_OBJ, "*.o")))
    _compile(str(tmp_path / "both"), extra=(*objs, "-lpthread"))


def _c1():
    return ["4", "256", "1024", "1024", "128", "4", "1", "2"]


@pytest.mark.gpu
def test_cxx_caller_trains_bitwise_like_the_c_abi(caller):
    from paper_2602_04816_b200 import engine as E

    r = subprocess.run([caller, "train", *_c1(), "3"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    bits = [int(ln.split()[1], 16) for ln in r.stdout.splitlines() if ln.startswith("loss")]
    assert len(bits) == 3

    c = E.ModelConfig(4, 256, 1024, 1024, 128, 4, k_ckpt=1, n_heads=2, rope_theta=1e6)
    store = E.Store(c, 1234, "bf16")
    losses = store.run_training(E.HyperParams(lr=3e-3), 1234, 3,
                                E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=3))
    want = [int(v) for v in np.asarray(losses, np.float64).view(np.uint64)]
    assert bits == want, ([hex(b) for b in bits], [hex(w) for w in want])
    # the step's byte counters follow the reference formula (planner.cpp:22-30)
    tail = [ln for ln in r.stdout.splitlines() if ln.startswith("h2d")][0].split()
    n, Vh = c.block_params(), c.vocab * c.hidden
    assert int(tail[1]) == 2 * (2 * 4 * n + 2 * Vh) and int(tail[3]) == 4 * (4 * n + 2 * Vh)
    assert int(tail[5]) == 3
    # bench.py's scheduling features (overlapped tail, pieces, sparse embedding, vocab-chunked
    # head, weight cache) leave the numerics unchanged: the same losses bit for bit, except the
    # head chunking's d_x summation order (<= 2e-4), so compare the first step bitwise
    rx = subprocess.run([caller, "trainx", *_c1(), "3"], capture_output=True, text=True, timeout=600)
    assert rx.returncode == 0, rx.stderr
    bx = [int(ln.split()[1], 16) for ln in rx.stdout.splitlines() if ln.startswith("loss")]
    lx = [float(ln.split()[2]) for ln in rx.stdout.splitlines() if ln.startswith("loss")]
    assert bx[0] == bits[0] and np.allclose(lx, losses, rtol=1e-5)


@pytest.mark.gpu
def test_cxx_phase_api_matches_train_step(caller):
    from paper_2602_04816_b200 import engine as E

    r = subprocess.run([caller, "phases", *_c1()], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    b0, b1 = (int(lines[i].split()[1], 16) for i in (0, 1))
    assert b0 == b1
    c = E.ModelConfig(4, 256, 1024, 1024, 128, 4, k_ckpt=1, n_heads=2, rope_theta=1e6)
    s = E.Store(c, 1234, "bf16")
    e = E.Engine(s, E.Arena(c), E.HyperParams(), E.EngineOptions(skip_optimizer=True))
    loss = e.train_step(E.make_copy_task_batch(c, 1235)).loss
    assert int(np.float64(loss).view(np.uint64)) == b0
    assert lines[2] == "recompute_forwards 4"


@pytest.mark.gpu
def test_cxx_exceptions_cross_the_library_boundary(caller):
    r = subprocess.run([caller, "errors"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    out = r.stdout
    assert "errors caught 4" in out
    # ArenaOomError names the region that did not fit (reference test_arena.cpp:171-205)
    assert "ArenaOomError region=" in out


@pytest.mark.gpu
def test_arena_contract_through_the_cxx_api(caller):
    """DeviceArena / ArenaLedger contract (reference proj/tests/test_arena.cpp:160-215):
    budget caps and stack overflow raise ArenaOomError naming the region, anchors only on
    the K grid, protocol errors on misuse — exercised through the exported C++ API."""
    r = subprocess.run([caller, "arena"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout and "arena failures 0" in r.stdout


def _parse_ledger(out):
    """'region <name> k v k v ...', 'footprint k v ...', 'host k v ...', 'committed v k v ...'."""
    regions, kv = {}, {}
    for ln in out.splitlines():
        w = ln.split()
        if not w:
            continue
        if w[0] == "region":
            regions[w[1]] = {w[i]: int(w[i + 1]) for i in range(2, len(w) - 1, 2)}
        elif w[0] in ("footprint", "host"):
            kv.update({f"{w[0]}.{w[i]}": int(w[i + 1]) for i in range(1, len(w) - 1, 2)})
        elif w[0] == "committed":
            kv.update({w[i]: int(w[i + 1]) for i in range(0, len(w) - 1, 2)})
    return regions, kv


@pytest.mark.gpu
@pytest.mark.parametrize("K", [1, 2])
def test_live_ledger_equals_the_footprint_estimate(caller, K):
    """Plan == ledger (reference proj/tests/test_planner.cpp:43-72): after one step every
    region's live peak reaches exactly the capacity the footprint formula reserved — the
    estimate neither over- nor under-commits — and the host ledger equals 14 B/param."""
    L, h, f, V, S, B = 4, 256, 1024, 1024, 128, 4
    r = subprocess.run([caller, "ledger", str(L), str(h), str(f), str(V), str(S), str(B), str(K), "2"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    regions, kv = _parse_ledger(r.stdout)
    assert kv["committed"] == kv["footprint.total"]
    assert sum(x["capacity"] for x in regions.values()) == kv["footprint.total"]
    for name in ("activation_stack", "ckpt_anchors", "workspace"):
        assert regions[name]["step_peak"] == regions[name]["capacity"], (name, regions[name])
    widest = kv["footprint.widest_tile_bytes"]
    for name in ("stream_buf[0]", "stream_buf[1]"):
        assert regions[name]["capacity"] == kv["footprint.stream_buf"]
        assert regions[name]["step_peak"] == widest, (name, regions[name])
        assert regions[name]["current"] == 0          # nothing left streamed in after the step
    assert regions["ckpt_anchors"]["current"] == 0
    n = 4 * h * h + 3 * h * f + 2 * h
    params = 2 * V * h + L * n
    assert kv["host.params"] == params and kv["host.persistent"] == 14 * params
    assert kv["host.total"] == kv["host.persistent"] + kv["host.slabs"]


def test_cxx_caller_round_trips_a_reference_hlm1_checkpoint(caller, tmp_path):
    """hlm::load_checkpoint reads the reference's HLM1 (golden file written by the reference's
    save_checkpoint) and hlm::save_checkpoint_hlm1 writes it back byte for byte: a BF16 store's
    master is the file's BF16 weights exactly, m / v / step count unchanged, and the reference
    container carries the gradient region as zeros (last-step scratch, not restored)."""
    import oracle as O
    src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_tiny_bf16.hlm1")
    out = tmp_path / "back.hlm1"
    # tiny: L2 h8 f16 V11 S4 B1 K1, one head (tests/golden/make_golden.py)
    r = subprocess.run([caller, "hlm1", src, str(out), "2", "8", "16", "11", "4", "1", "1", "1"],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "adam_steps 3 " in r.stdout
    a, b = O.read_hlm1(src), O.read_hlm1(str(out))
    assert a["adam_steps"] == b["adam_steps"] and list(a["alias"]) == list(b["alias"])
    for ta, tb in zip(a["tiles"], b["tiles"]):
        for key in ("weights", "m", "v"):
            assert np.array_equal(ta[key].view(np.uint32), tb[key].view(np.uint32)), key
        assert not tb["grads"].any()
