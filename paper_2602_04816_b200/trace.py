"""Protocol validator and overlap metrics for MEASURED engine traces.

Port of the reference's logical-trace checker (validate_trace,
proj/src/scheduler.cpp:29-201) to the traces the B200 engine records with
CUDA-event timestamps (`Engine.last_trace()`, JSONL schema of
include/hlm/trace.hpp). Structural rules, replayed in issue order:

  malformed        dependencies reference earlier ops
  weights-ready    a weight consumer depends on the latest WeightXfer of its
                   layer (weight-cache hits reuse the forward's transfer)
  backward-done    a GradXfer depends on the LocalBackward that produced it
  buffer-free      a WeightXfer into stream buffer b depends on b's last reader
                   and never overwrites an unconsumed occupant (cache slots,
                   buf >= 2, are written once per step and are exempt)
  stack-discipline local backwards pop recomputed layers in LIFO order

and one rule the logical trace could not have, because the trace is measured:

  timing           an event-timed op never starts before any event-timed
                   dependency ended (tolerance `tol_us`): a race detector on
                   the real H2D / compute / D2H streams.
"""
from collections import namedtuple

Violation = namedtuple("Violation", "op_id rule detail")

GPU_STREAMS = ("h2d", "compute", "d2h")


def _consumes_weights(op, embed_tile):
    if op["buf"] in (-2, -3):    # HBM-resident optimizer tile / rows gathered zero-copy from host
        return False
    if op["kind"] in ("Forward", "Recompute"):
        return True
    return op["kind"] == "LocalBackward" and op["layer"] != embed_tile


def validate_trace(ops, n_layers, embed_tile=0, head_tile=None, n_stream_buffers=2, tol_us=50.0):
    head_tile = n_layers + 1 if head_tile is None else head_tile
    out = []
    by_id = {op["id"]: op for op in ops}
    n = len(ops)
    for op in ops:
        for d in op["deps"]:
            if d < 0 or d >= n:
                out.append(Violation(op["id"], "malformed", "dependency id out of range"))
            elif d >= op["id"]:
                out.append(Violation(op["id"], "malformed", "dependency points forward in issue order"))

    last_xfer = {}
    for op in ops:
        if _consumes_weights(op, embed_tile):
            w = last_xfer.get(op["layer"], -1)
            if w < 0:
                out.append(Violation(op["id"], "weights-ready",
                                     f"no prior weight transfer for layer {op['layer']}"))
            elif w not in op["deps"]:
                out.append(Violation(op["id"], "weights-ready",
                                     f"missing dependency on weights_ready[{op['layer']}] (op {w})"))
        if op["kind"] == "WeightXfer":
            last_xfer[op["layer"]] = op["id"]

    last_lb = {}
    for op in ops:
        if op["kind"] == "LocalBackward":
            last_lb[op["layer"]] = op["id"]
        if op["kind"] == "GradXfer":
            lb = last_lb.get(op["layer"], -1)
            if lb < 0:
                out.append(Violation(op["id"], "backward-done",
                                     f"gradient transfer with no prior local backward for layer {op['layer']}"))
            elif lb not in op["deps"]:
                out.append(Violation(op["id"], "backward-done",
                                     f"missing dependency on backward_done[{op['layer']}] (op {lb})"))

    into, reader, consumed = {}, {}, {}
    for op in ops:
        b = op["buf"]
        if op["kind"] == "WeightXfer":
            if b < 0:
                out.append(Violation(op["id"], "buffer-free", "weight transfer without a buffer"))
                continue
            if b >= n_stream_buffers:
                continue
            if b in into:
                if not consumed.get(b, True):
                    out.append(Violation(op["id"], "buffer-free",
                                         f"overwrites buffer {b} whose occupant was never consumed"))
                elif reader.get(b, -1) >= 0 and reader[b] not in op["deps"]:
                    out.append(Violation(op["id"], "buffer-free",
                                         f"missing dependency on buffer_free[{b}] (reader op {reader[b]})"))
            into[b], reader[b], consumed[b] = op["id"], -1, False
        elif 0 <= b < n_stream_buffers and op["stream"] == "compute" and op["kind"] != "OptStep":
            reader[b], consumed[b] = op["id"], True

    group, used = [], 0
    for op in ops:
        if op["stream"] != "compute":
            continue
        if op["kind"] == "Recompute":
            if used > 0 or not group:
                if 0 < used < len(group):
                    out.append(Violation(op["id"], "stack-discipline",
                                         "recompute begins before the previous block was consumed"))
                if used == len(group):
                    group = []
                used = 0
            group.append(op["layer"])
        elif op["kind"] == "LocalBackward" and 1 <= op["layer"] <= n_layers:
            expect = group[len(group) - 1 - used] if group and used < len(group) else -1
            if op["layer"] != expect:
                out.append(Violation(op["id"], "stack-discipline",
                                     f"local backward of layer {op['layer']} violates LIFO order "
                                     f"(expected {expect})"))
            else:
                used += 1

    for op in ops:
        if op["stream"] not in GPU_STREAMS or op.get("t_start_us", -1) < 0:
            continue
        for d in op["deps"]:
            dep = by_id.get(d)
            if dep is None or dep["stream"] not in GPU_STREAMS or dep.get("t_end_us", -1) < 0:
                continue
            if dep is op or (dep["t_start_us"] == op["t_start_us"] and dep["t_end_us"] == op["t_end_us"]):
                continue   # fused head forward/backward share one launch
            if op["t_start_us"] + tol_us < dep["t_end_us"]:
                out.append(Violation(op["id"], "timing",
                                     f"starts at {op['t_start_us']:.1f} us before dependency op {d} "
                                     f"ended at {dep['t_end_us']:.1f} us"))
    return out


def _union(intervals):
    merged = []
    for s, e in sorted(intervals):
        if merged and s <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], e)
        else:
            merged.append([s, e])
    return merged


def overlap_report(ops):
    """Per-step transfer/compute overlap from a measured trace: the fraction of
    H2D + D2H busy time during which the compute stream was also busy, the
    achieved copy bandwidths (GB/s over the streams' busy time) and the compute
    stream's busy time (union of its op intervals)."""
    comp = _union([(o["t_start_us"], o["t_end_us"]) for o in ops
                   if o["stream"] == "compute" and o["t_end_us"] > o["t_start_us"] >= 0])

    def covered(a, b):
        return sum(max(0.0, min(b, e) - max(a, s)) for s, e in comp)

    rep = {"compute_busy_ms": sum(e - s for s, e in comp) / 1e3}
    for st in ("h2d", "d2h"):
        xs = [o for o in ops if o["stream"] == st and o["t_end_us"] > o["t_start_us"] >= 0]
        busy = sum(o["t_end_us"] - o["t_start_us"] for o in xs)
        rep[f"{st}_gbs"] = sum(o["bytes"] for o in xs) / busy / 1e3 if busy > 0 else None
        rep[f"{st}_busy_ms"] = busy / 1e3
        rep[f"{st}_hidden_ms"] = sum(covered(o["t_start_us"], o["t_end_us"]) for o in xs) / 1e3
    total = rep["h2d_busy_ms"] + rep["d2h_busy_ms"]
    rep["overlap"] = (rep["h2d_hidden_ms"] + rep["d2h_hidden_ms"]) / total if total > 0 else None
    rep.update(exposed_weights(ops))
    return rep


def exposed_weights(ops):
    """Where the compute stream idles, and why: for every idle gap before a
    compute op, the part during which a weight transfer that op depends on was
    in flight is EXPOSED TRANSFER; the rest of the gap is waiting for the
    transfer to be issued at all (the host optimizer had not finished that tile)
    or for other work. h2d_overlap = 1 - exposed / H2D busy time: the per-layer
    compute/transfer overlap of the north-star target, separated from host-paced
    idling; d2h_overlap the same for the gradient D2H (a backward waiting for its gradient
    buffer to drain), transfer_overlap both directions together (SURVEY §8d's
    1 - exposed transfer / transfer)."""
    by_id = {o["id"]: o for o in ops}
    comp = sorted((o for o in ops if o["stream"] == "compute" and o["t_end_us"] > o["t_start_us"] >= 0),
                  key=lambda o: o["t_start_us"])
    prev, idle = 0.0, 0.0   # timestamps are relative to the step-start event
    exposed = {"h2d": 0.0, "d2h": 0.0}
    for c in comp:
        if c["t_start_us"] > prev:
            g0, g1 = prev, c["t_start_us"]
            idle += g1 - g0
            for st in exposed:
                spans = []
                for d in c["deps"]:
                    x = by_id.get(d)
                    if x and x["stream"] == st and x["t_end_us"] > x["t_start_us"] >= 0:
                        lo, hi = max(g0, x["t_start_us"]), min(g1, x["t_end_us"])
                        if hi > lo:
                            spans.append((lo, hi))
                exposed[st] += sum(e - s for s, e in _union(spans))
        prev = max(prev, c["t_end_us"])
    busy = {st: sum(o["t_end_us"] - o["t_start_us"] for o in ops
                    if o["stream"] == st and o["t_end_us"] > o["t_start_us"] >= 0) for st in exposed}
    both = busy["h2d"] + busy["d2h"]
    # d2h exposure: the compute stream idling on a gradient D2H that must drain before the
    # next backward can write that gradient buffer (the backward's dependency on it)
    return {"compute_idle_ms": idle / 1e3, "h2d_exposed_ms": exposed["h2d"] / 1e3,
            "h2d_overlap": 1.0 - exposed["h2d"] / busy["h2d"] if busy["h2d"] > 0 else None,
            "d2h_exposed_ms": exposed["d2h"] / 1e3,
            "d2h_overlap": 1.0 - exposed["d2h"] / busy["d2h"] if busy["d2h"] > 0 else None,
            "transfer_overlap": 1.0 - (exposed["h2d"] + exposed["d2h"]) / both if both > 0 else None}
