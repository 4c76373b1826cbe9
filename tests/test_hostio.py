"""Host-transfer helpers: the page-locked output pool must never hand out
a block the caller still references (CPU: allocation stubbed), and the
pooled / staged D2H paths must return identical bytes (GPU)."""

import numpy as np
import pytest

from paper_1711_03888_b200 import hostio


class _Pool(hostio.PinnedPool):
    allocs = 0

    def _alloc(self, nbytes):
        _Pool.allocs += 1
        return np.empty(nbytes, np.uint8)


def test_pool_first_request_is_staged_then_pooled():
    p = _Pool()
    assert p.take(1024) is None  # first miss: caller stages
    a = p.take(1024)
    assert a is not None and a.nbytes == 1024


def test_pool_never_aliases_live_views():
    p = _Pool(per_size=2)
    p.take(4096)
    a = p.take(4096)
    v = a.view(np.float32)[10:20]  # caller keeps only a derived view
    del a
    b = p.take(4096)
    assert b is not None and not np.shares_memory(b, v)
    c = p.take(4096)  # both blocks referenced, per_size reached
    assert c is None
    del v
    d = p.take(4096)  # the first block is free again
    assert d is not None and not np.shares_memory(d, b)


def test_pool_reuses_released_block():
    p = _Pool(per_size=1)
    p.take(256)
    a = p.take(256)
    addr = a.ctypes.data
    del a
    b = p.take(256)
    assert b.ctypes.data == addr


def test_pool_cap():
    p = _Pool(per_size=4, cap_bytes=1000)
    p.take(600)
    keep = p.take(600)
    assert keep is not None
    p.take(600)
    assert p.take(600) is None  # would exceed the cap


def test_new_bytes_in_place():
    b, view = hostio.new_bytes(10_000)
    view[:] = 7
    assert isinstance(b, bytes) and len(b) == 10_000 and set(b) == {7}
    assert hostio.new_bytes(0)[0] == b""


@pytest.mark.gpu
def test_host_output_pooled_and_staged_agree():
    import torch
    hostio.POOL.clear()
    src = torch.arange(1 << 20, dtype=torch.int32, device="cuda").view(torch.uint8)
    n = src.numel()
    outs = [hostio.host_output(n, src) for _ in range(4)]  # staged, pooled, pooled, staged
    ref = src.cpu().numpy()
    for o in outs:
        assert np.array_equal(o, ref)
    addrs = {o.ctypes.data for o in outs}
    assert len(addrs) == 4  # all live at once: no aliasing
