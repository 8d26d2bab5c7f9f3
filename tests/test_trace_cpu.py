"""Trace validator (paper_2602_04816_b200/trace.py) on a measured C2 trace
committed under profiles/ (clean) and on mutations of it, each of which must be
reported at the mutated op under the right rule — the reference's mutation
localisation tests (proj/tests/test_scheduler.cpp:208-287)."""
import copy
import json
import os

import pytest

from paper_2602_04816_b200.trace import overlap_report, validate_trace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TRACE = os.path.join(ROOT, "profiles", "r01_trace_c2_step.jsonl")


@pytest.fixture(scope="module")
def ops():
    return [json.loads(l) for l in open(TRACE)]


def test_measured_trace_is_clean_and_overlapped(ops):
    assert validate_trace(ops, 28) == []
    rep = overlap_report(ops)
    assert rep["overlap"] > 0.5 and rep["h2d_gbs"] > 20


def _first(ops, **kw):
    return next(o for o in ops if all(o[k] == v for k, v in kw.items()))


def _mut(ops, fn):
    m = copy.deepcopy(ops)
    fn(m)
    return m


def test_missing_weights_dependency_is_localised(ops):
    tgt = _first(ops, kind="Forward", layer=5)
    m = _mut(ops, lambda m: m[tgt["id"]].__setitem__("deps", []))
    v = validate_trace(m, 28)
    assert any(x.op_id == tgt["id"] and x.rule == "weights-ready" for x in v)


def test_missing_backward_done_dependency_is_localised(ops):
    tgt = _first(ops, kind="GradXfer", layer=10)
    m = _mut(ops, lambda m: m[tgt["id"]].__setitem__("deps", []))
    v = validate_trace(m, 28)
    assert any(x.op_id == tgt["id"] and x.rule == "backward-done" for x in v)


def _op(i, stream, kind, layer, buf=-1, deps=(), t=(-1.0, -1.0)):
    return {"id": i, "stream": stream, "kind": kind, "layer": layer, "buf": buf, "slab": -1,
            "bytes": 0, "flops": 0, "params": 0, "pinned": True, "deps": list(deps),
            "t_start_us": t[0], "t_end_us": t[1]}


def test_buffer_overwrite_without_reader_dependency():
    """embed -> buf0, block1 -> buf1, block2 -> buf0 must wait for embed's reader."""
    ops = [_op(0, "h2d", "WeightXfer", 0, 0), _op(1, "compute", "Forward", 0, 0, [0]),
           _op(2, "h2d", "WeightXfer", 1, 1), _op(3, "compute", "Forward", 1, 1, [2]),
           _op(4, "h2d", "WeightXfer", 2, 0, [1]), _op(5, "compute", "Forward", 2, 0, [4])]
    assert validate_trace(ops, 2) == []
    ops[4]["deps"] = []
    v = validate_trace(ops, 2)
    assert [x.rule for x in v] == ["buffer-free"] and v[0].op_id == 4
    # overwriting an occupant nobody read
    ops2 = [_op(0, "h2d", "WeightXfer", 0, 0), _op(1, "h2d", "WeightXfer", 1, 0)]
    assert any(x.rule == "buffer-free" and "never consumed" in x.detail
               for x in validate_trace(ops2, 2))


def test_lifo_violation(ops):
    lbs = [o for o in ops if o["kind"] == "LocalBackward" and 1 <= o["layer"] <= 28]
    a, b = lbs[2], lbs[3]
    def swap(m):
        m[a["id"]]["layer"], m[b["id"]]["layer"] = m[b["id"]]["layer"], m[a["id"]]["layer"]
    v = validate_trace(_mut(ops, swap), 28)
    assert any(x.rule == "stack-discipline" for x in v)


def test_measured_race_is_detected(ops):
    tgt = _first(ops, kind="Forward", layer=7)
    w = ops[tgt["deps"][0]]
    def early(m):
        m[tgt["id"]]["t_start_us"] = w["t_end_us"] - 500.0
    v = validate_trace(_mut(ops, early), 28)
    assert any(x.op_id == tgt["id"] and x.rule == "timing" for x in v)


def test_forward_pointing_dependency_is_malformed(ops):
    tgt = _first(ops, kind="Forward", layer=3)
    m = _mut(ops, lambda m: m[tgt["id"]]["deps"].append(len(m) - 1))
    v = validate_trace(m, 28)
    assert any(x.op_id == tgt["id"] and x.rule == "malformed" for x in v)


def test_exposed_weights_counts_only_waits_on_inflight_transfers():
    """h2d_overlap: compute idle while a weight transfer its op depends on is in
    flight is exposed; idle before the transfer even started (host-paced) is not."""
    from paper_2602_04816_b200.trace import exposed_weights
    ops = [
        {"id": 0, "stream": "compute", "kind": "Forward", "layer": 0, "deps": [], "t_start_us": 0.0, "t_end_us": 100.0,
         "bytes": 0},
        # host-paced: the transfer starts 400 us after compute went idle, runs 100 us
        {"id": 1, "stream": "h2d", "kind": "WeightXfer", "layer": 1, "deps": [], "t_start_us": 500.0,
         "t_end_us": 600.0, "bytes": 1000},
        {"id": 2, "stream": "compute", "kind": "Forward", "layer": 1, "deps": [1], "t_start_us": 600.0,
         "t_end_us": 700.0, "bytes": 0},
        # fully hidden transfer
        {"id": 3, "stream": "h2d", "kind": "WeightXfer", "layer": 2, "deps": [], "t_start_us": 600.0,
         "t_end_us": 650.0, "bytes": 1000},
        {"id": 4, "stream": "compute", "kind": "Forward", "layer": 2, "deps": [3], "t_start_us": 700.0,
         "t_end_us": 800.0, "bytes": 0},
    ]
    r = exposed_weights(ops)
    assert abs(r["compute_idle_ms"] - 0.5) < 1e-9        # 100 -> 600
    assert abs(r["h2d_exposed_ms"] - 0.1) < 1e-9         # only 500 -> 600 had the transfer in flight
    assert abs(r["h2d_overlap"] - (1 - 100.0 / 150.0)) < 1e-9


def test_exposed_gradient_drain_counts_waits_on_the_buffer_d2h():
    """d2h_overlap: a backward that waits for its gradient buffer's previous D2H to drain
    exposes that transfer; a D2H that drained under compute is hidden. transfer_overlap
    combines both directions."""
    from paper_2602_04816_b200.trace import exposed_weights
    ops = [
        {"id": 0, "stream": "compute", "kind": "LocalBackward", "layer": 3, "deps": [], "t_start_us": 0.0,
         "t_end_us": 100.0, "bytes": 0},
        {"id": 1, "stream": "d2h", "kind": "GradXfer", "layer": 3, "deps": [0], "t_start_us": 100.0,
         "t_end_us": 400.0, "bytes": 1000},
        # the next backward reuses the buffer: it starts only when the D2H is done (300 us exposed)
        {"id": 2, "stream": "compute", "kind": "LocalBackward", "layer": 2, "deps": [1], "t_start_us": 400.0,
         "t_end_us": 500.0, "bytes": 0},
        {"id": 3, "stream": "d2h", "kind": "GradXfer", "layer": 2, "deps": [2], "t_start_us": 500.0,
         "t_end_us": 600.0, "bytes": 1000},
        # a later backward on that buffer with the drain already hidden under other compute
        {"id": 4, "stream": "compute", "kind": "LocalBackward", "layer": 1, "deps": [3], "t_start_us": 500.0,
         "t_end_us": 700.0, "bytes": 0},
    ]
    r = exposed_weights(ops)
    assert abs(r["d2h_exposed_ms"] - 0.3) < 1e-9
    assert abs(r["d2h_overlap"] - (1 - 300.0 / 400.0)) < 1e-9
    assert r["h2d_overlap"] is None
    assert abs(r["transfer_overlap"] - (1 - 300.0 / 400.0)) < 1e-9
