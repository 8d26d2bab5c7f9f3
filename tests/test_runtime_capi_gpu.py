"""The device-runtime entry points of the C ABI: init + caps, raw arena,
typed streams / events, pinned H2D / D2H, and the head + cross-entropy call in the
survey's argument order — driven through ctypes exactly as a host caller without CUDA
headers would."""
import ctypes

import pytest
import torch

from paper_2602_04816_b200 import _lib as L

pytestmark = pytest.mark.gpu

_vp = ctypes.c_void_p


class Caps(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("sm_count", ctypes.c_int), ("cc_major", ctypes.c_int),
                ("cc_minor", ctypes.c_int), ("hbm_bytes", ctypes.c_int64), ("l2_bytes", ctypes.c_int64),
                ("smem_per_block_optin", ctypes.c_int64), ("name", ctypes.c_char * 64)]


class HeadDims(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("hidden", ctypes.c_int64), ("vocab", ctypes.c_int64)]


def lib():
    Lb = L.blib()
    Lb.hlm_cuda_arena_create.argtypes = [ctypes.c_size_t, ctypes.POINTER(_vp)]
    Lb.hlm_cuda_h2d_async.argtypes = [_vp, _vp, ctypes.c_size_t, _vp]
    Lb.hlm_cuda_d2h_async.argtypes = [_vp, _vp, ctypes.c_size_t, _vp]
    for f in ("arena_destroy", "stream_destroy", "stream_sync", "event_destroy", "event_sync", "event_query"):
        getattr(Lb, "hlm_cuda_" + f).argtypes = [_vp]
    Lb.hlm_cuda_stream_create.argtypes = [ctypes.c_int, ctypes.POINTER(_vp)]
    Lb.hlm_cuda_event_create.argtypes = [ctypes.POINTER(_vp)]
    Lb.hlm_cuda_event_record.argtypes = [_vp, _vp]
    Lb.hlm_cuda_event_wait.argtypes = [_vp, _vp]
    Lb.hlm_cuda_event_elapsed_ms.argtypes = [_vp, _vp, ctypes.POINTER(ctypes.c_float)]
    Lb.hlm_cuda_head_fwd_ce_bwd.argtypes = [ctypes.POINTER(HeadDims), _vp, _vp, _vp, ctypes.c_float, _vp, _vp,
                                            _vp, ctypes.POINTER(ctypes.c_double), _vp, _vp]
    return Lb


def test_init_reports_the_b200():
    Lb = lib()
    caps = Caps()
    L.check(Lb.hlm_cuda_init(0, ctypes.byref(caps)))
    assert (caps.cc_major, caps.cc_minor) == (10, 0)
    assert caps.sm_count == 148
    assert caps.hbm_bytes > 170e9 and caps.l2_bytes > 100e6
    assert caps.smem_per_block_optin >= 227 * 1024
    assert b"B200" in caps.name


def test_streams_events_and_pinned_copies_round_trip():
    """H2D on the H2D stream -> the compute stream waits on its event -> the D2H stream
    waits on the compute stream's event -> the bytes come back unchanged; events time the
    copy and report completion."""
    Lb = lib()
    n = 64 << 20
    src = torch.randint(0, 256, (n,), dtype=torch.uint8).pin_memory()
    dst = torch.zeros(n, dtype=torch.uint8).pin_memory()
    base = _vp()
    L.check(Lb.hlm_cuda_arena_create(n, ctypes.byref(base)))
    streams = {}
    for k, name in ((0, "compute"), (1, "h2d"), (2, "d2h")):
        s = _vp()
        L.check(Lb.hlm_cuda_stream_create(k, ctypes.byref(s)))
        streams[name] = s
    ev = {}
    for name in ("t0", "in", "ready", "out"):
        e = _vp()
        L.check(Lb.hlm_cuda_event_create(ctypes.byref(e)))
        ev[name] = e
    L.check(Lb.hlm_cuda_event_record(ev["t0"], streams["h2d"]))
    L.check(Lb.hlm_cuda_h2d_async(base, src.data_ptr(), n, streams["h2d"]))
    L.check(Lb.hlm_cuda_event_record(ev["in"], streams["h2d"]))
    L.check(Lb.hlm_cuda_event_wait(streams["compute"], ev["in"]))
    L.check(Lb.hlm_cuda_event_record(ev["ready"], streams["compute"]))
    L.check(Lb.hlm_cuda_event_wait(streams["d2h"], ev["ready"]))
    L.check(Lb.hlm_cuda_d2h_async(dst.data_ptr(), base, n, streams["d2h"]))
    L.check(Lb.hlm_cuda_event_record(ev["out"], streams["d2h"]))
    L.check(Lb.hlm_cuda_event_sync(ev["out"]))
    assert Lb.hlm_cuda_event_query(ev["out"]) == 0
    assert torch.equal(src, dst)
    ms = ctypes.c_float()
    L.check(Lb.hlm_cuda_event_elapsed_ms(ev["t0"], ev["in"], ctypes.byref(ms)))
    assert ms.value > 0 and n / (ms.value * 1e-3) > 5e9   # a pinned 64 MiB H2D, well above 5 GB/s
    for e in ev.values():
        L.check(Lb.hlm_cuda_event_destroy(e))
    for s in streams.values():
        L.check(Lb.hlm_cuda_stream_sync(s))
        L.check(Lb.hlm_cuda_stream_destroy(s))
    L.check(Lb.hlm_cuda_arena_destroy(base))


def test_arena_oom_is_reported_as_oom():
    Lb = lib()
    base = _vp()
    rc = Lb.hlm_cuda_arena_create(1 << 50, ctypes.byref(base))
    assert rc == 3 and not base.value   # HLM_ERR_OOM
    assert b"out of memory" in L.lib().hlm_cuda_last_error()


def test_head_fwd_ce_bwd_equals_head_loss():
    """The survey-order entry point computes exactly what hlm_cuda_head_loss does, and its
    host loss sum is the row sum in double."""
    Lb = lib()
    dev = "cuda"
    torch.manual_seed(2)
    T, h, V = 256, 128, 1000
    head = (torch.randn(V, h, device=dev) * 0.05).bfloat16()
    x = torch.randn(T, h, device=dev)
    tgt = torch.randint(0, V, (T,), dtype=torch.int32, device=dev)
    ws = torch.empty(Lb.hlm_cuda_head_ws_bytes(T, h, V), dtype=torch.uint8, device=dev)
    vp = lambda t: _vp(t.data_ptr())  # noqa: E731
    outs = []
    for fused in (False, True):
        dx = torch.full((T, h), float("nan"), device=dev)
        dhead = torch.full((V, h), float("nan"), device=dev)
        lr = torch.empty(T, device=dev)
        if fused:
            tot = ctypes.c_double()
            d = HeadDims(T, h, V)
            L.check(Lb.hlm_cuda_head_fwd_ce_bwd(ctypes.byref(d), vp(head), vp(x), vp(tgt), 1.0 / T, vp(dx),
                                                vp(dhead), vp(lr), ctypes.byref(tot), vp(ws), None))
            want = 0.0
            for v in lr.cpu().numpy():   # row order, double accumulation
                want += float(v)
            assert tot.value == want
        else:
            L.check(Lb.hlm_cuda_head_loss(T, h, V, vp(head), vp(x), vp(tgt), 1.0 / T, vp(dx), vp(dhead), 0,
                                          vp(lr), vp(ws), None))
        torch.cuda.synchronize()
        outs.append((dx, dhead, lr))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
