"""Host <-> device transfers for the public API's host-buffer paths.

PCIe moves pinned memory at ~50 GB/s but pageable memory far slower, and
the reference's API hands out plain ``bytes`` / numpy arrays.  Every large
transfer therefore goes through two grow-only pinned staging buffers: the
DMA of chunk k+1 overlaps the (multi-threaded) CPU copy of chunk k between
the staging buffer and the caller's pageable memory.  Already-pinned host
tensors are copied directly.

The staging buffers are process-wide, so staged copies hold a lock and
return only once the DMA that reads / writes the staging memory is done:
concurrent callers (host threads) never share a buffer in flight.
"""

from __future__ import annotations

import threading
from typing import Dict, Tuple

import numpy as np

CHUNK = 64 << 20  # bytes per staging chunk

_pinned: Dict[Tuple[str, int], object] = {}
_stage_lock = threading.RLock()  # the staging buffers, the pinned cache, the pool


def pinned(role: str, nbytes: int):
    """Grow-only pinned uint8 host buffer keyed by role."""
    import torch
    key = (role, 0)
    with _stage_lock:
        b = _pinned.get(key)
        if b is None or b.numel() < nbytes:
            b = torch.empty(max(int(nbytes), 4096), dtype=torch.uint8, pin_memory=True)
            _pinned[key] = b
        return b


def _host_u8(buf):
    """A uint8 CPU tensor viewing `buf` (bytes / bytearray / memoryview /
    numpy / CPU tensor) without copying."""
    import torch
    if isinstance(buf, torch.Tensor):
        return buf.reshape(-1).view(torch.uint8)
    if isinstance(buf, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(buf).reshape(-1).view(np.uint8))
    mv = memoryview(buf).cast("B")
    if mv.readonly:  # torch wants a writable buffer; numpy gives a read-only view
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            return torch.frombuffer(mv, dtype=torch.uint8)
    return torch.frombuffer(mv, dtype=torch.uint8)


def to_device(src, dst) -> None:
    """Copy host bytes `src` into the CUDA uint8 tensor `dst` (same length)."""
    import torch
    h = _host_u8(src)
    n = h.numel()
    if n == 0:
        return
    if h.is_pinned():
        dst[:n].copy_(h, non_blocking=True)
        return
    with _stage_lock:
        stage = [pinned("h2d0", CHUNK), pinned("h2d1", CHUNK)]
        ev = [None, None]
        stream = torch.cuda.current_stream()
        for k, off in enumerate(range(0, n, CHUNK)):
            m = min(CHUNK, n - off)
            s = k & 1
            if ev[s] is not None:
                ev[s].synchronize()  # the DMA that last read this buffer is done
            stage[s][:m].copy_(h[off:off + m])
            dst[off:off + m].copy_(stage[s][:m], non_blocking=True)
            ev[s] = torch.cuda.Event()
            ev[s].record(stream)
        for e in ev:  # the staging buffers are free before another caller writes them
            if e is not None:
                e.synchronize()


def to_host(src, dst) -> None:
    """Copy the CUDA uint8 tensor `src` into host memory `dst` (a writable
    buffer / numpy array / CPU tensor of the same byte length)."""
    import torch
    h = _host_u8(dst)
    n = h.numel()
    if n == 0:
        return
    if h.is_pinned():
        h.copy_(src[:n], non_blocking=False)
        return
    with _stage_lock:
        stage = [pinned("d2h0", CHUNK), pinned("d2h1", CHUNK)]
        stream = torch.cuda.current_stream()
        chunks = list(range(0, n, CHUNK))
        ev = [None, None]

        def issue(k):
            off = chunks[k]
            m = min(CHUNK, n - off)
            stage[k & 1][:m].copy_(src[off:off + m], non_blocking=True)
            e = torch.cuda.Event()
            e.record(stream)
            ev[k & 1] = e

        issue(0)
        for k, off in enumerate(chunks):
            if k + 1 < len(chunks):
                issue(k + 1)
            ev[k & 1].synchronize()
            m = min(CHUNK, n - off)
            h[off:off + m].copy_(stage[k & 1][:m])


def _advise_huge(addr: int, nbytes: int) -> None:
    """madvise(MADV_HUGEPAGE) on the 2 MiB-aligned interior of a fresh
    mapping, so first-touch faults cost ~1/512 as many traps (no-op where
    THP is disabled)."""
    import ctypes
    if nbytes < (4 << 20):
        return
    try:
        libc = ctypes.CDLL(None, use_errno=True)
        a0 = (addr + (2 << 20) - 1) & ~((2 << 20) - 1)
        ln = (addr + nbytes - a0) & ~((2 << 20) - 1)
        if ln > 0:
            libc.madvise(ctypes.c_void_p(a0), ctypes.c_size_t(ln), 14)  # MADV_HUGEPAGE
    except Exception:
        pass


def new_bytes(n: int):
    """A new uninitialised ``bytes`` object of length n and a writable uint8
    CPU tensor over its buffer.  PyBytes_FromStringAndSize(NULL, n) is the
    CPython idiom for building a bytes object in place; the caller fills the
    whole buffer before the object escapes."""
    import ctypes

    import torch
    if n == 0:
        return b"", torch.empty(0, dtype=torch.uint8)
    api = ctypes.pythonapi
    api.PyBytes_FromStringAndSize.restype = ctypes.py_object
    api.PyBytes_FromStringAndSize.argtypes = [ctypes.c_void_p, ctypes.c_ssize_t]
    api.PyBytes_AsString.restype = ctypes.c_void_p
    api.PyBytes_AsString.argtypes = [ctypes.py_object]
    b = api.PyBytes_FromStringAndSize(None, n)
    addr = api.PyBytes_AsString(b)
    _advise_huge(addr, n)
    view = torch.from_numpy(np.ctypeslib.as_array((ctypes.c_uint8 * n).from_address(addr)))
    return b, view


def bytes_from(src_u8, n: int) -> bytes:
    """A new ``bytes`` object holding the first n bytes of the CPU uint8
    tensor `src_u8`, filled by torch's multi-threaded copy."""
    b, view = new_bytes(n)
    if n:
        view.copy_(src_u8[:n])
    return b


def empty_host(numel: int, dtype=None):
    """Fresh pageable CPU tensor advised to transparent huge pages."""
    import torch
    dtype = dtype or torch.float32
    t = torch.empty(numel, dtype=dtype)
    _advise_huge(t.data_ptr(), t.numel() * t.element_size())
    return t


class PinnedPool:
    """Page-locked host blocks for repeated multi-GB outputs.

    A D2H into page-locked memory runs at the full PCIe rate (~50 GB/s)
    while a transfer into fresh pageable memory is staged and runs at about
    half that; but locking a fresh block costs ~0.5 s per GB, far more than
    one transfer saves.  The pool therefore only pays for a block once a
    size has been asked for repeatedly: the first request of a size class
    returns None (the caller stages into pageable memory), later ones get a
    pooled block.  Blocks are handed out as numpy arrays; every view the
    caller derives keeps that array as its ``base`` (numpy collapses view
    chains onto it), so a block is reused only once the pool holds the last
    reference.  At most `per_size` blocks per size class and `cap_bytes` in
    total are kept."""

    def __init__(self, per_size: int = 2, cap_bytes: int = 48 << 30):
        self.per_size = per_size
        self.cap_bytes = cap_bytes
        self.blocks = {}  # nbytes -> [np.ndarray over a pinned tensor]
        self.misses = {}  # nbytes -> count

    def take(self, nbytes: int):
        with _stage_lock:
            return self._take(nbytes)

    def _take(self, nbytes: int):
        import sys
        lst = self.blocks.setdefault(nbytes, [])
        for i in range(len(lst)):
            # references: the list slot + getrefcount's argument
            if sys.getrefcount(lst[i]) <= 2:
                return lst[i]
        self.misses[nbytes] = self.misses.get(nbytes, 0) + 1
        total = sum(k * len(v) for k, v in self.blocks.items())
        if self.misses[nbytes] < 2 or len(lst) >= self.per_size or total + nbytes > self.cap_bytes:
            return None
        a = self._alloc(nbytes)
        if a is not None:
            lst.append(a)
        return a

    @staticmethod
    def _alloc(nbytes: int):
        import torch
        try:
            return torch.empty(nbytes, dtype=torch.uint8, pin_memory=True).numpy()
        except RuntimeError:
            return None

    def clear(self) -> None:
        self.blocks.clear()
        self.misses.clear()


POOL = PinnedPool()


def host_output(nbytes: int, src) -> np.ndarray:
    """Copy the first nbytes of the CUDA uint8 tensor `src` into host
    memory the caller owns: a pooled page-locked block (direct D2H) or
    fresh pageable memory (staged D2H).  Returns a uint8 numpy array."""
    import torch
    a = POOL.take(nbytes)
    if a is not None:
        torch.from_numpy(a).copy_(src[:nbytes])
        return a
    h = empty_host(nbytes, torch.uint8)
    to_host(src[:nbytes], h)
    return h.numpy()
