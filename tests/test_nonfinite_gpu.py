"""The GPU finiteness scan (hlm_cuda_nonfinite — the reference's "validate every gradient
before any mutation", host_store.cpp:374-382, run on the device before the D2H) at any
alignment: a data-parallel shard starts at rank * n / world elements, which need not be
16-byte aligned."""
import ctypes

import pytest
import torch

from paper_2602_04816_b200 import _lib

pytestmark = pytest.mark.gpu


def _scan(t):
    lib = _lib.lib()
    first = torch.empty(1, dtype=torch.int64, device="cuda")
    lib.hlm_cuda_nonfinite.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    _lib.check(lib.hlm_cuda_nonfinite(ctypes.c_void_p(t.data_ptr()), t.numel(),
                                      ctypes.c_void_p(first.data_ptr()), None))
    torch.cuda.synchronize()
    return int(first.cpu().item()) & 0xFFFFFFFFFFFFFFFF


@pytest.mark.parametrize("offset", [0, 1, 2, 3])
@pytest.mark.parametrize("n", [1, 3, 5, 4096 + 7, 1 << 20])
def test_scan_finds_the_first_nonfinite_at_any_alignment(offset, n):
    base = torch.randn(n + 8, device="cuda")
    g = base[offset:offset + n]
    assert _scan(g) == 0xFFFFFFFFFFFFFFFF
    for pos, bad in ((n - 1, float("nan")), (n // 2, float("inf")), (0, float("-inf"))):
        g2 = g.clone() if offset == 0 else base.clone()[offset:offset + n]
        g2[pos] = bad
        if pos < n - 1:
            g2[n - 1] = float("nan")   # a later one must not win
        assert _scan(g2) == pos, (offset, n, pos)
