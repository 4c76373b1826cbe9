"""Thin test-side wrappers around the stage-level C-ABI parity hooks
(include/nbzg.h).  Each mirrors one nbz._kernels / nbz module function so the
GPU tests read like the reference's test_kernels_equiv.py."""

import ctypes

import numpy as np
import torch

from paper_1711_03888_b200 import _native as N


def _dev(a, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def _sync():
    torch.cuda.synchronize()


def minmax6(fields):
    L = N.lib()
    ts = [_dev(f, torch.float32) for f in fields]
    n = ts[0].numel()
    arr = (ctypes.c_void_p * 6)(*[t.data_ptr() for t in ts])
    out = torch.zeros(12, dtype=torch.float32, device="cuda")
    N.check(L.nbzg_minmax6(arr, n, N.ptr(out), N.stream_handle()), "minmax6")
    return out.cpu().numpy()


def integerize(x, bound):
    L = N.lib()
    t = _dev(x, torch.float32)
    out = torch.zeros(max(t.numel(), 1), dtype=torch.int64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.check(L.nbzg_integerize(N.ptr(t), t.numel(), float(bound), N.ptr(out), N.ptr(st),
                              N.stream_handle()), "integerize")
    return out[:t.numel()].cpu().numpy(), int(st.item())


def rindex_keys(coords, bounds3, segment_size=16384):
    L = N.lib()
    ts = [_dev(c, torch.float32) for c in coords]
    n = ts[0].numel()
    nseg = (n + segment_size - 1) // segment_size
    keys = torch.zeros(max(n, 1), dtype=torch.int64, device="cuda")
    bits = torch.zeros(max(nseg, 1), dtype=torch.uint8, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    b3 = (ctypes.c_double * 3)(*[float(b) for b in bounds3])
    N.check(L.nbzg_rindex_keys(N.ptr(ts[0]), N.ptr(ts[1]), N.ptr(ts[2]), n, b3, segment_size,
                               N.ptr(keys), N.ptr(bits), N.ptr(st), N.stream_handle()),
            "rindex_keys")
    return (keys[:n].cpu().numpy().view(np.uint64), bits[:nseg].cpu().numpy(), int(st.item()))


def prx_order(keys, segment_size, seg_bits, ignored_groups):
    L = N.lib()
    k = _dev(np.asarray(keys, np.uint64).view(np.int64))
    b = _dev(np.asarray(seg_bits, np.uint8))
    n = k.numel()
    out = torch.zeros(max(n, 1), dtype=torch.int64, device="cuda")
    N.check(L.nbzg_prx_order(N.ptr(k), n, segment_size, N.ptr(b), ignored_groups, N.ptr(out),
                             N.stream_handle()), "prx_order")
    return out[:n].cpu().numpy()


def huffman_lengths(sorted_counts):
    L = N.lib()
    c = _dev(np.asarray(sorted_counts, np.uint32).view(np.int32))
    k = c.numel()
    out = torch.zeros(k, dtype=torch.uint8, device="cuda")
    np2 = 1 << max(0, (k - 1).bit_length())
    ws = torch.zeros(12 * np2 + 64, dtype=torch.uint8, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.check(L.nbzg_huffman_lengths(N.ptr(c), k, N.ptr(out), N.ptr(ws), ws.numel(), N.ptr(st),
                                   N.stream_handle()), "huffman_lengths")
    return out.cpu().numpy(), int(st.item())


def huffman_codebook(hist):
    L = N.lib()
    h = _dev(np.asarray(hist, np.uint32).view(np.int32))
    nb = h.numel()
    sym = torch.zeros(nb, dtype=torch.int32, device="cuda")
    lens = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    lut = torch.zeros(nb, dtype=torch.int64, device="cuda")
    meta = torch.zeros(ctypes.sizeof(N.Meta), dtype=torch.uint8, device="cuda")
    ws = torch.zeros(20 * nb + 64, dtype=torch.uint8, device="cuda")
    N.check(L.nbzg_huffman_codebook(N.ptr(h), nb, N.ptr(sym), N.ptr(lens), N.ptr(lut),
                                    N.ptr(meta), N.ptr(ws), ws.numel(), N.stream_handle()),
            "codebook")
    m = N.Meta.from_buffer_copy(meta.cpu().numpy().tobytes())
    k = m.f[0].k
    return (sym[:k].cpu().numpy(), lens[:k].cpu().numpy(), lut.cpu().numpy().view(np.uint64), m)


def huff_encode(codes_u16, lut_u64):
    L = N.lib()
    c = _dev(np.asarray(codes_u16, np.uint16).view(np.int16))
    lut = _dev(np.asarray(lut_u64, np.uint64).view(np.int64))
    n = c.numel()
    total = int((np.asarray(lut_u64, np.uint64)[np.asarray(codes_u16)] >> np.uint64(57))
                .astype(np.int64).sum())
    nchunks = (n + 16383) // 16384
    out = torch.zeros(4 * ((total + 31) // 32) + 16, dtype=torch.uint8, device="cuda")
    cb = torch.zeros(max(nchunks, 1), dtype=torch.int32, device="cuda")
    ws = torch.zeros(16 * nchunks + 64, dtype=torch.uint8, device="cuda")
    N.check(L.nbzg_huff_encode(N.ptr(c), n, N.ptr(lut), N.ptr(out), N.ptr(cb), N.ptr(ws),
                               ws.numel(), N.stream_handle()), "huff_encode")
    return out.cpu().numpy().tobytes()[:(total + 7) // 8], total, cb.cpu().numpy()[:nchunks]


def crc64(data: bytes):
    from paper_1711_03888_b200 import io as nio
    return nio.crc64(data)


def huff_decode(data: bytes, total_bits: int, n: int, tables: dict):
    """K.huff_decode hook: tables as returned by oracle.huffman_tables."""
    import ctypes as C
    L = N.lib()
    buf = _dev(np.frombuffer(bytearray(bytes(data) + b"\0" * 16), np.uint8))
    ss = _dev(np.asarray(tables["sorted_syms"], np.int32))
    out = torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    fc = np.ascontiguousarray(tables["first_code"], np.uint64)
    cb = np.ascontiguousarray(tables["counts_by_len"], np.uint32)
    fi = np.ascontiguousarray(tables["first_idx"], np.uint32)
    N.check(L.nbzg_huff_decode(N.ptr(buf), total_bits, n, tables["min_len"], tables["max_len"],
                               fc.ctypes.data_as(C.c_void_p), cb.ctypes.data_as(C.c_void_p),
                               fi.ctypes.data_as(C.c_void_p), N.ptr(ss), N.ptr(out), N.ptr(st),
                               N.stream_handle()), "huff_decode")
    return out[:n].cpu().numpy(), int(st.item())


def deinterleave3(keys):
    L = N.lib()
    k = _dev(np.asarray(keys, np.uint64).view(np.int64))
    n = k.numel()
    outs = [torch.zeros(max(n, 1), dtype=torch.int64, device="cuda") for _ in range(3)]
    N.check(L.nbzg_deinterleave3(N.ptr(k), n, *[N.ptr(o) for o in outs], N.stream_handle()),
            "deinterleave3")
    return [o[:n].cpu().numpy() for o in outs]
