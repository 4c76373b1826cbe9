"""CPU oracle for the nbz SZ-LV / SZ-LV-PRX hot path -- TEST INFRASTRUCTURE ONLY.

This package is the parity checker for the B200 path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` and
``--impl reference`` legs) may import it; the product package
``paper_1711_03888_b200`` never does, and fails loudly when its own CUDA
library is missing instead of falling back here.

The arithmetic lives in ``nbz_oracle.c`` (a plain-C restatement of the
reference's numba kernels, each function citing ``pkg/src/nbz/_kernels.py``
line ranges).  This module adds the numpy glue that mirrors the reference's
Python layer:

* ``resolve_field_bounds``   pipeline.py:157-181 / model.py:104-125
* ``compress``               pipeline.py:447-526 (SZ-LV and SZ-LV-PRX only)
* ``serialize``              io.py:105-125 (container v1; v2 = same layout,
                             version 2, stream kind 3 = SZ_DQ: dual-quant
                             codes, chain restart + chunk index every 16384
                             symbols, escapes inline in the bitstream)
* ``decompress``             pipeline.py:542-604 (SZ branch)

Parity is PINNED: ``tests/test_oracle_golden.py`` checks this oracle
against golden vectors dumped from the reference package itself
(``scripts/make_golden.py`` -> ``tests/golden/*.npz``), including
byte-identical v1 archives.
"""

from __future__ import annotations

import ctypes
import os
import struct
import subprocess
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_ref", "liboracle.so")

MODE_UIDS = {"sz-lcf": 0, "sz-lv": 1, "sz-lv-prx": 2, "sz-cpc2000": 3, "cpc2000": 4}
CPC_MODES = ("sz-cpc2000", "cpc2000")
KIND_SZ_FIELD = 0
KIND_VLC_FIELD = 1
KIND_RINDEX = 2
KIND_SZ_DQ = 3
NO_FIELD = 255
CHUNK_SYMBOLS = 16384

ORC_STATUS = {0: "ok", 1: "bound too small", 2: "code too long", 3: "invalid code",
              4: "truncated", 5: "bad stream", 6: "no memory"}


def build(force: bool = False) -> str:
    """Compile nbz_oracle.c into oracle/_ref/liboracle.so (gcc, no FMA)."""
    src = os.path.join(_HERE, "nbz_oracle.c")
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(src)):
        return _LIB_PATH
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    subprocess.check_call(["make", "-s", "-C", _HERE, "lib"])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        D = ctypes.c_double
        I = ctypes.c_int
        sig = {
            "orc_minmax": (None, [P, I64, P, P]),
            "orc_integerize": (I, [P, I64, D, P]),
            "orc_interleave3": (None, [P, P, P, I64, P]),
            "orc_build_rindex": (I, [P, P, P, I64, I64, I, P, P, P]),
            "orc_prx_order": (None, [P, I64, I64, P, I, I, P]),
            "orc_sz_quantize": (I64, [P, I64, D, I64, I, P, P, P]),
            "orc_sz_dequantize": (I64, [P, I64, P, I64, D, I64, I, P]),
            "orc_dq_quantize": (I64, [P, I64, D, I64, I64, I64, P, P, P]),
            "orc_dq_dequantize": (I64, [P, I64, P, I64, D, I64, I64, I64, P]),
            "orc_huffman_lengths": (None, [P, I64, P]),
            "orc_huffman_build": (I64, [P, I64, P, P]),
            "orc_huffman_tables": (None, [P, P, I64, P, P, P, P, P]),
            "orc_huff_encode": (I64, [P, I64, P, P]),
            "orc_huff_decode": (I, [P, I64, I64, I, I, P, P, P, P, P]),
            "orc_crc64": (ctypes.c_uint64, [P, I64]),
            "orc_sz_payload": (I64, [P, I64, P, I64, I64, I, P]),
            "orc_sz_decode": (I, [P, I64, I64, D, I64, I, P]),
            "orc_free": (None, [P]),
            "orc_compress": (I, [P, I64, I, P, ctypes.c_uint32, I64, I64, I, I, P, P, P, P]),
            "orc_compress_v": (I, [P, I64, I, I, I, P, ctypes.c_uint32, I64, I64, I, I, P, P, P, P]),
            "orc_sz_decode_p": (I, [P, I64, I64, D, I64, I, I, P]),
            "orc_dq_quantize_p": (I64, [P, I64, D, I64, I64, I, P, P]),
            "orc_dq_dequantize_p": (I64, [P, I64, P, I64, D, I64, I64, I, P]),
            "orc_build_rindex_n": (I, [P, I, I64, I64, I, P, P, P]),
            "orc_compress_shards": (I64, [P, I64, I, P, ctypes.c_uint32, I64, I64, I, I, I,
                                          I, I, P]),
            "orc_num_threads": (I, []),
            "orc_cpc_coord_stream": (I64, [P, I64, I64, P, P, P, P, I, P]),
            "orc_vlc_vel_stream": (I64, [P, P, I64, I64, D, I, P]),
            "orc_cpc_coord_decode": (I, [P, I64, I64, I64, P, P, P, P]),
            "orc_vlc_vel_decode": (I, [P, I64, I64, I64, D, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


# ----------------------------------------------------------------------
# stage-level restatements (each mirrors one reference function)
# ----------------------------------------------------------------------

def minmax(x: np.ndarray) -> Tuple[float, float]:
    x = _c(x, np.float32)
    lo = np.zeros(1, np.float32)
    hi = np.zeros(1, np.float32)
    lib().orc_minmax(_p(x), x.size, _p(lo), _p(hi))
    return float(lo[0]), float(hi[0])


def resolve_field_bounds(fields: Sequence[np.ndarray], kinds: Sequence[str],
                         values: Sequence[float]):
    """pipeline.py:157-181.  kinds[i] in {'abs','rel'}.  Returns
    (resolved list with None for constants/empty, constants, mask)."""
    resolved: List[Optional[float]] = []
    constants: List[float] = []
    mask = 0
    for i, arr in enumerate(fields):
        if arr.size == 0:
            resolved.append(None)
            constants.append(0.0)
            continue
        lo, hi = minmax(arr)
        if hi - lo == 0.0:
            mask |= 1 << i
            resolved.append(None)
            constants.append(float(arr[0]))
            continue
        if kinds[i] == "abs":
            resolved.append(float(values[i]))
        else:
            resolved.append(float(values[i]) * (hi - lo))
        constants.append(0.0)
    return resolved, constants, mask


def integerize(x: np.ndarray, bound: float) -> np.ndarray:
    x = _c(x, np.float32)
    out = np.empty(x.size, np.int64)
    st = lib().orc_integerize(_p(x), x.size, float(bound), _p(out))
    if st:
        raise OverflowError("bound too small for value magnitude")
    return out


def interleave3(x, y, z) -> np.ndarray:
    x, y, z = (_c(a, np.int64) for a in (x, y, z))
    keys = np.empty(x.size, np.uint64)
    lib().orc_interleave3(_p(x), _p(y), _p(z), x.size, _p(keys))
    return keys


def build_rindex(cols: Sequence[np.ndarray], segment_size: int, allow_clamp: bool = True):
    c = [_c(a, np.int64) for a in cols]
    n = c[0].size
    nseg = (n + segment_size - 1) // segment_size
    keys = np.empty(n, np.uint64)
    bits = np.zeros(max(nseg, 1), np.uint8)
    minima = np.zeros(3 * max(nseg, 1), np.int64)
    st = lib().orc_build_rindex(_p(c[0]), _p(c[1]), _p(c[2]), n, segment_size,
                                int(allow_clamp), _p(keys), _p(bits), _p(minima))
    if st:
        raise OverflowError("segment needs more than 21 index bits")
    return keys, bits[:nseg], minima[:3 * nseg].reshape(nseg, 3)


def prx_order(keys: np.ndarray, segment_size: int, seg_bits: np.ndarray,
              ignored_groups: int, group_width: int = 3) -> np.ndarray:
    keys = _c(keys, np.uint64)
    sb = _c(seg_bits, np.uint8)
    order = np.empty(keys.size, np.int64)
    lib().orc_prx_order(_p(keys), keys.size, segment_size, _p(sb), ignored_groups,
                        group_width, _p(order))
    return order


def sz_quantize(x: np.ndarray, bound: float, half: int, use_lcf: bool = False):
    """Exact reference chain (_kernels.py:150-184)."""
    x = _c(x, np.float32)
    codes = np.empty(x.size, np.int32)
    recon = np.empty(x.size, np.float32)
    esc = np.empty(max(x.size, 1), np.float32)
    ne = lib().orc_sz_quantize(_p(x), x.size, float(bound), half, int(use_lcf), _p(codes),
                               _p(recon), _p(esc))
    return codes, esc[:ne].copy(), recon


def sz_dequantize(codes, esc, bound: float, half: int, use_lcf: bool = False):
    codes = _c(codes, np.int32)
    esc = _c(esc, np.float32)
    out = np.empty(codes.size, np.float32)
    used = lib().orc_sz_dequantize(_p(codes), codes.size, _p(esc), esc.size, float(bound), half,
                                   int(use_lcf), _p(out))
    if used != esc.size:
        raise ValueError("escape count mismatch")
    return out


def dq_quantize(x: np.ndarray, bound: float, half: int, k_prev: int = 0,
                chunk: int = CHUNK_SYMBOLS):
    """Dual-quant restatement (v2 stream kind SZ_DQ; chain restarts every
    `chunk` symbols, 0 = never); returns codes, escapes, k_last."""
    x = _c(x, np.float32)
    codes = np.empty(x.size, np.int32)
    esc = np.empty(max(x.size, 1), np.float32)
    kl = np.zeros(1, np.int64)
    ne = lib().orc_dq_quantize(_p(x), x.size, float(bound), half, int(k_prev), int(chunk),
                               _p(codes), _p(esc), _p(kl))
    return codes, esc[:ne].copy(), int(kl[0])


def dq_dequantize(codes, esc, bound: float, half: int, k_prev: int = 0,
                  chunk: int = CHUNK_SYMBOLS):
    codes = _c(codes, np.int32)
    esc = _c(esc, np.float32)
    out = np.empty(codes.size, np.float32)
    escb = esc if esc.size else np.zeros(1, np.float32)
    used = lib().orc_dq_dequantize(_p(codes), codes.size, _p(escb), esc.size, float(bound), half,
                                   int(k_prev), int(chunk), _p(out))
    if used != esc.size:
        raise ValueError("escape count mismatch")
    return out


def huffman_lengths(sorted_counts: np.ndarray) -> np.ndarray:
    c = _c(sorted_counts, np.int64)
    out = np.empty(c.size, np.int64)
    lib().orc_huffman_lengths(_p(c), c.size, _p(out))
    return out


def huffman_build(hist: np.ndarray):
    """encode.py:199-219: ascending symbols + lengths from a bincount."""
    h = _c(hist, np.int64)
    syms = np.empty(max(h.size, 1), np.int32)
    lens = np.empty(max(h.size, 1), np.uint8)
    k = lib().orc_huffman_build(_p(h), h.size, _p(syms), _p(lens))
    if k < 0:
        raise OverflowError("huffman code length exceeds encoder limit")
    if k == 0:
        raise ValueError("empty frequencies")
    return syms[:k].copy(), lens[:k].copy()


def huffman_tables(symbols: np.ndarray, lengths: np.ndarray):
    s = _c(symbols, np.int32)
    l = _c(lengths, np.uint8)
    packed = np.zeros(int(s[-1]) + 1, np.uint64)
    fc = np.zeros(64, np.uint64)
    fi = np.zeros(64, np.int64)
    cbl = np.zeros(64, np.int64)
    ss = np.zeros(s.size, np.int32)
    lib().orc_huffman_tables(_p(s), _p(l), s.size, _p(packed), _p(fc), _p(fi), _p(cbl), _p(ss))
    return dict(enc_packed=packed, first_code=fc, first_idx=fi, counts_by_len=cbl,
                sorted_syms=ss, min_len=int(l.min()), max_len=int(l.max()))


def huff_encode(codes: np.ndarray, packed: np.ndarray) -> Tuple[bytes, int]:
    codes = _c(codes, np.int32)
    packed = _c(packed, np.uint64)
    total_bits = int((packed[codes] >> np.uint64(57)).astype(np.int64).sum()) if codes.size else 0
    out = np.zeros((total_bits + 7) // 8 + 8, np.uint8)
    nb = lib().orc_huff_encode(_p(codes), codes.size, _p(packed), _p(out))
    return out[:nb].tobytes(), total_bits


def huff_decode(data: bytes, total_bits: int, n: int, tables: dict) -> np.ndarray:
    d = np.frombuffer(bytes(data) + b"\0" * 8, np.uint8)
    out = np.zeros(n, np.int32)
    st = lib().orc_huff_decode(_p(d), total_bits, n, tables["min_len"], tables["max_len"],
                               _p(tables["first_code"]), _p(tables["counts_by_len"]),
                               _p(tables["first_idx"]), _p(tables["sorted_syms"]), _p(out))
    if st:
        raise ValueError("invalid huffman code" if st == 1 else "truncated huffman stream")
    return out


def crc64(data) -> int:
    b = np.frombuffer(bytes(data), np.uint8) if not isinstance(data, np.ndarray) else _c(data, np.uint8)
    if b.size == 0:
        b = np.zeros(1, np.uint8)
        return int(lib().orc_crc64(_p(b), 0))
    return int(lib().orc_crc64(_p(b), b.size))


def sz_payload(codes: np.ndarray, esc: np.ndarray, interval_count: int, fmt: int) -> bytes:
    codes = _c(codes, np.int32)
    esc = _c(esc, np.float32)
    if esc.size == 0:
        esc = np.zeros(1, np.float32)[:0]
    out = ctypes.c_void_p()
    escb = esc if esc.size else np.zeros(1, np.float32)
    ln = lib().orc_sz_payload(_p(codes), codes.size, _p(escb), esc.size, interval_count, fmt,
                              ctypes.byref(out))
    if ln < 0:
        raise ValueError(ORC_STATUS.get(-ln, str(ln)))
    data = ctypes.string_at(out, ln)
    lib().orc_free(out)
    return data


def sz_decode(payload: bytes, n: int, bound: float, interval_count: int, fmt: int,
              lcf: bool = False) -> np.ndarray:
    buf = np.frombuffer(bytes(payload) + b"\0" * 8, np.uint8)
    out = np.zeros(max(n, 1), np.float32)
    st = lib().orc_sz_decode_p(_p(buf), len(payload), n, float(bound), interval_count, fmt,
                               int(lcf), _p(out))
    if st:
        raise ValueError(ORC_STATUS.get(st, str(st)))
    return out[:n]


# ----------------------------------------------------------------------
# whole-snapshot path (pipeline.py:447-526) + container (io.py:105-125)
# ----------------------------------------------------------------------

_FIXED = struct.Struct("<4sHBBQIIBBH")


def serialize(mode: str, n: int, interval_count: int, segment_size: int, ignored_groups: int,
              bounds, mask: int, constants, seg_bits, payloads, fmt: int,
              variant: int = 0) -> bytes:
    """Container restatement of io.py:105-125; fmt 2 writes version 2 and kind 3
    (fmt 3, the chunk-restart chain, is a version-1 container of SZ_FIELD streams)."""
    sorted_mode = mode == "sz-lv-prx"
    variant_uid = variant if (sorted_mode and n > 0) else 255
    head = bytearray()
    head += _FIXED.pack(b"NBZ1", 1 if fmt == 3 else fmt, MODE_UIDS[mode], variant_uid, n,
                        interval_count,
                        segment_size, ignored_groups, mask, 0)
    head += struct.pack("<6d", *bounds)
    head += struct.pack("<6f", *constants)
    streams = [(f, p) for f, p in enumerate(payloads) if p is not None]
    segs = bytes(np.asarray(seg_bits, np.uint8)) if (sorted_mode and n > 0) else b""
    head += struct.pack("<II", len(segs), len(streams))
    head += segs
    kind = KIND_SZ_DQ if fmt == 2 else KIND_SZ_FIELD
    for f, p in streams:
        head += struct.pack("<BBHQQ", kind, f, 0, len(p), crc64(p))
    head += struct.pack("<Q", crc64(bytes(head)))
    return bytes(head) + b"".join(p for _, p in streams)


VARIANTS = {"coord": 0, "vel": 1, "coordvel": 2}


def build_rindex_n(cols: Sequence[np.ndarray], segment_size: int, allow_clamp: bool = True):
    """rindex.build_r_indices for 3 or 6 interleaved fields."""
    c = [_c(a, np.int64) for a in cols]
    f, n = len(c), c[0].size
    nseg = (n + segment_size - 1) // segment_size
    keys = np.empty(n, np.uint64)
    bits = np.zeros(max(nseg, 1), np.uint8)
    minima = np.zeros(f * max(nseg, 1), np.int64)
    ptrs = (ctypes.c_void_p * f)(*[a.ctypes.data for a in c])
    st = lib().orc_build_rindex_n(ptrs, f, n, segment_size, int(allow_clamp), _p(keys),
                                  _p(bits), _p(minima))
    if st:
        raise OverflowError("segment needs more index bits than the key budget")
    return keys, bits[:nseg], minima[:f * nseg].reshape(nseg, f)


def compress(fields: Sequence[np.ndarray], mode: str, kinds, values, interval_count: int = 65536,
             segment_size: int = 16384, ignored_groups: int = 6, fmt: int = 1,
             variant: str = "coord") -> dict:
    """Whole-snapshot oracle compress.  fmt 1 reproduces the reference's v1
    archive byte-for-byte; fmt 2 is the dual-quant v2 archive the GPU emits;
    fmt 3 is the reference-readable v1 archive the GPU emits on request
    (the reference's chain restarted by a forced escape every 16384 values)."""
    f32 = [_c(a, np.float32) for a in fields]
    n = int(f32[0].size)
    if isinstance(kinds, str):
        kinds = [kinds] * 6
    if np.isscalar(values):
        values = [values] * 6
    resolved, constants, mask = resolve_field_bounds(f32, kinds, values)
    bounds = np.array([b if b is not None else 0.0 for b in resolved], np.float64)
    sorted_mode = mode == "sz-lv-prx"
    nseg = (n + segment_size - 1) // segment_size if (sorted_mode and n > 0) else 0
    seg_bits = np.zeros(max(nseg, 1), np.uint8)
    order = np.empty(max(n, 1), np.int64) if sorted_mode else None
    ptrs = (ctypes.c_void_p * 6)(*[a.ctypes.data for a in f32])
    outs = (ctypes.c_void_p * 6)()
    lens = np.zeros(6, np.int64)
    st = lib().orc_compress_v(ptrs, n, int(sorted_mode), VARIANTS[variant],
                              int(mode == "sz-lcf"), _p(bounds), mask,
                              interval_count, segment_size, ignored_groups, fmt, outs,
                              _p(lens), _p(seg_bits), _p(order) if order is not None else None)
    payloads: List[Optional[bytes]] = []
    for f in range(6):
        if outs[f]:
            payloads.append(ctypes.string_at(outs[f], int(lens[f])))
            lib().orc_free(outs[f])
        else:
            payloads.append(None)
    if st:
        raise ValueError(ORC_STATUS.get(st, str(st)))
    if n == 0:
        payloads = [None] * 6
    wire = serialize(mode, n, interval_count, segment_size, ignored_groups, bounds, mask,
                     constants, seg_bits[:nseg], payloads, fmt, variant=VARIANTS[variant])
    return dict(wire=wire, payloads=payloads, bounds=bounds, constants=constants, mask=mask,
                seg_bits=seg_bits[:nseg].copy(), order=None if order is None else order[:n],
                ratio=(24.0 * n / len(wire)) if n else None)


def parse(wire: bytes) -> dict:
    """Minimal container parser (io.py:128-211 layout, no CRC re-check)."""
    (magic, version, mode_uid, variant_uid, n, ic, ss, ig, mask, _pad) = _FIXED.unpack_from(wire, 0)
    off = _FIXED.size
    bounds = struct.unpack_from("<6d", wire, off); off += 48
    consts = struct.unpack_from("<6f", wire, off); off += 24
    nseg, nst = struct.unpack_from("<II", wire, off); off += 8
    seg_bits = np.frombuffer(wire, np.uint8, nseg, off).copy(); off += nseg
    dirs = []
    for _ in range(nst):
        dirs.append(struct.unpack_from("<BBHQQ", wire, off)); off += 20
    off += 8
    payloads = [None] * 6
    kinds = [None] * 6
    for kind, fid, _p2, ln, _crc in dirs:
        payloads[fid] = wire[off:off + ln]
        kinds[fid] = kind
        off += ln
    return dict(version=version, mode_uid=mode_uid, n=n, interval_count=ic, segment_size=ss,
                ignored_groups=ig, mask=mask, bounds=bounds, constants=consts,
                seg_bits=seg_bits, payloads=payloads, kinds=kinds)


def decompress(wire: bytes) -> List[np.ndarray]:
    a = parse(wire)
    n = a["n"]
    out = []
    for f in range(6):
        if a["mask"] & (1 << f):
            out.append(np.full(n, np.float32(a["constants"][f]), np.float32))
        elif n == 0:
            out.append(np.zeros(0, np.float32))
        else:
            fmt = 1 if a["kinds"][f] == KIND_SZ_FIELD else 2
            out.append(sz_decode(a["payloads"][f], n, a["bounds"][f], a["interval_count"], fmt,
                                 lcf=a["mode_uid"] == 0))
    return out


# ----------------------------------------------------------------------
# CPC2000 family (pipeline.py:447-526 stores_minima branch, 316-428)
# ----------------------------------------------------------------------

_SEG_MIN = struct.Struct("<B3q")


def _take(ptr, ln) -> bytes:
    data = ctypes.string_at(ptr, int(ln))
    lib().orc_free(ptr)
    return data


def cpc_coord_stream(keys_sorted, segment_size: int, seg_bits, xs_sorted, ints_sorted, bounds,
                     fmt: int) -> bytes:
    """_build_coord_stream (pipeline.py:316-337); ints_sorted[c] None for a
    constant coordinate (no correction records)."""
    k = _c(keys_sorted, np.uint64)
    n = k.size
    sb = _c(seg_bits, np.uint8)
    xs = [_c(a, np.float32) for a in xs_sorted]
    ints = [None if a is None else _c(a, np.int64) for a in ints_sorted]
    xp = (ctypes.c_void_p * 3)(*[a.ctypes.data for a in xs])
    ip = (ctypes.c_void_p * 3)(*[None if a is None else a.ctypes.data for a in ints])
    b = _c(bounds, np.float64)
    out = ctypes.c_void_p()
    ln = lib().orc_cpc_coord_stream(_p(k), n, segment_size, _p(sb), xp, ip, _p(b), fmt,
                                    ctypes.byref(out))
    if ln < 0:
        raise ValueError(ORC_STATUS.get(-ln, str(ln)))
    return _take(out, ln)


def vlc_vel_stream(ints_sorted, x_sorted, segment_size: int, bound: float, fmt: int) -> bytes:
    """_build_vel_stream (pipeline.py:378-395)."""
    i = _c(ints_sorted, np.int64)
    x = _c(x_sorted, np.float32)
    out = ctypes.c_void_p()
    ln = lib().orc_vlc_vel_stream(_p(i), _p(x), i.size, segment_size, float(bound), fmt,
                                  ctypes.byref(out))
    if ln < 0:
        raise ValueError(ORC_STATUS.get(-ln, str(ln)))
    return _take(out, ln)


def cpc_coord_decode(payload: bytes, n: int, segment_size: int, seg_bits, minima, bounds,
                     mask: int) -> List[Optional[np.ndarray]]:
    buf = np.frombuffer(bytes(payload) + b"\0" * 8, np.uint8)
    sb = _c(seg_bits, np.uint8)
    mn = _c(minima, np.int64).reshape(-1)
    b = _c(bounds, np.float64)
    outs = [None if mask & (1 << c) else np.zeros(max(n, 1), np.float32) for c in range(3)]
    op = (ctypes.c_void_p * 3)(*[None if o is None else o.ctypes.data for o in outs])
    st = lib().orc_cpc_coord_decode(_p(buf), len(payload), n, segment_size, _p(sb), _p(mn),
                                    _p(b), op)
    if st:
        raise ValueError(ORC_STATUS.get(st, str(st)))
    return [None if o is None else o[:n] for o in outs]


def vlc_vel_decode(payload: bytes, n: int, segment_size: int, bound: float) -> np.ndarray:
    buf = np.frombuffer(bytes(payload) + b"\0" * 8, np.uint8)
    out = np.zeros(max(n, 1), np.float32)
    st = lib().orc_vlc_vel_decode(_p(buf), len(payload), n, segment_size, float(bound), _p(out))
    if st:
        raise ValueError(ORC_STATUS.get(st, str(st)))
    return out[:n]


def serialize_cpc(mode: str, n: int, interval_count: int, segment_size: int,
                  ignored_groups: int, bounds, mask: int, constants, seg_bits, minima,
                  streams, fmt: int) -> bytes:
    """io.py:105-125 for the stores_minima modes: segments carry (bits,
    minima[3]); streams = [(kind, field, payload)], RINDEX first."""
    head = bytearray()
    head += _FIXED.pack(b"NBZ1", fmt, MODE_UIDS[mode], 0 if n > 0 else 255, n, interval_count,
                        segment_size, ignored_groups, mask, 0)
    head += struct.pack("<6d", *bounds)
    head += struct.pack("<6f", *constants)
    nseg = len(seg_bits) if n > 0 else 0
    head += struct.pack("<II", nseg, len(streams))
    for s in range(nseg):
        head += _SEG_MIN.pack(int(seg_bits[s]), *[int(v) for v in minima[s]])
    for kind, f, p in streams:
        head += struct.pack("<BBHQQ", kind, f, 0, len(p), crc64(p))
    head += struct.pack("<Q", crc64(bytes(head)))
    return bytes(head) + b"".join(p for _, _, p in streams)


def compress_cpc(fields: Sequence[np.ndarray], mode: str, kinds, values,
                 interval_count: int = 65536, segment_size: int = 16384,
                 ignored_groups: int = 6, fmt: int = 1) -> dict:
    """pipeline.compress for sz-cpc2000 / cpc2000 (pipeline.py:447-526):
    full-key R-index sort (k = 0, no key clamp: BoundTooSmallError past 21
    bits), the coordinate stream (raw first key + unsigned VLC deltas per
    segment + float32 corrections), velocities as SZ streams (sz-cpc2000;
    v1 sequential chain for fmt 1, dual-quant v2 for fmt 2) or signed VLC
    streams (cpc2000).  fmt 1 reproduces the reference archive byte for byte;
    fmt 2 (the GPU's) adds u32 per-segment bit lengths after each VLC-family
    payload and writes container version 2."""
    f32 = [_c(a, np.float32) for a in fields]
    n = int(f32[0].size)
    if isinstance(kinds, str):
        kinds = [kinds] * 6
    if np.isscalar(values):
        values = [values] * 6
    resolved, constants, mask = resolve_field_bounds(f32, kinds, values)
    bounds = np.array([b if b is not None else 0.0 for b in resolved], np.float64)
    streams = []
    order = None
    seg_bits = np.zeros(0, np.uint8)
    minima = np.zeros((0, 3), np.int64)
    if n > 0:
        ints = [np.zeros(n, np.int64) if resolved[i] is None else integerize(f32[i], resolved[i])
                for i in range(3)]
        keys, seg_bits, minima = build_rindex(ints, segment_size, allow_clamp=False)
        order = prx_order(keys, segment_size, seg_bits, 0, 3)
        work = [f[order] for f in f32]
        if (mask & 0b111) != 0b111:
            ks = keys[order]
            isort = [None if mask & (1 << c) else ints[c][order] for c in range(3)]
            streams.append((KIND_RINDEX, NO_FIELD,
                            cpc_coord_stream(ks, segment_size, seg_bits, work[:3], isort,
                                             bounds[:3], fmt)))
        half = interval_count // 2
        for fi in (3, 4, 5):
            if mask & (1 << fi):
                continue
            if mode == "cpc2000":
                iv = integerize(work[fi], resolved[fi])
                streams.append((KIND_VLC_FIELD, fi,
                                vlc_vel_stream(iv, work[fi], segment_size, resolved[fi], fmt)))
            elif fmt == 1:
                codes, esc, _r = sz_quantize(work[fi], resolved[fi], half)
                streams.append((KIND_SZ_FIELD, fi, sz_payload(codes, esc, interval_count, 1)))
            else:
                codes, esc, _k = dq_quantize(work[fi], resolved[fi], half)
                streams.append((KIND_SZ_DQ, fi, sz_payload(codes, esc, interval_count, 2)))
    wire = serialize_cpc(mode, n, interval_count, segment_size, ignored_groups, bounds, mask,
                         constants, seg_bits, minima, streams, fmt)
    return dict(wire=wire, streams=streams, bounds=bounds, constants=constants, mask=mask,
                seg_bits=seg_bits, minima=minima, order=order,
                ratio=(24.0 * n / len(wire)) if n else None)


def parse_cpc(wire: bytes) -> dict:
    (magic, version, mode_uid, variant_uid, n, ic, ss, ig, mask, _pad) = _FIXED.unpack_from(wire, 0)
    off = _FIXED.size
    bounds = struct.unpack_from("<6d", wire, off); off += 48
    consts = struct.unpack_from("<6f", wire, off); off += 24
    nseg, nst = struct.unpack_from("<II", wire, off); off += 8
    seg_bits = np.zeros(nseg, np.uint8)
    minima = np.zeros((nseg, 3), np.int64)
    for s in range(nseg):
        b, m0, m1, m2 = _SEG_MIN.unpack_from(wire, off); off += _SEG_MIN.size
        seg_bits[s] = b
        minima[s] = (m0, m1, m2)
    dirs = []
    for _ in range(nst):
        dirs.append(struct.unpack_from("<BBHQQ", wire, off)); off += 20
    off += 8
    streams = []
    for kind, fid, _p2, ln, _crc in dirs:
        streams.append((kind, fid, wire[off:off + ln]))
        off += ln
    return dict(version=version, mode_uid=mode_uid, n=n, interval_count=ic, segment_size=ss,
                ignored_groups=ig, mask=mask, bounds=bounds, constants=consts,
                seg_bits=seg_bits, minima=minima, streams=streams)


def decompress_cpc(wire: bytes) -> List[np.ndarray]:
    """pipeline.decompress stores_minima branch (pipeline.py:559-590); the
    output stays in sorted order, as in the reference."""
    a = parse_cpc(wire)
    n, mask = a["n"], a["mask"]
    out: List[Optional[np.ndarray]] = [None] * 6
    for f in range(6):
        if mask & (1 << f):
            out[f] = np.full(n, np.float32(a["constants"][f]), np.float32)
    if n == 0:
        return [np.zeros(0, np.float32)] * 6
    for kind, fid, p in a["streams"]:
        if kind == KIND_RINDEX:
            rec = cpc_coord_decode(p, n, a["segment_size"], a["seg_bits"], a["minima"],
                                   a["bounds"][:3], mask)
            for c in range(3):
                if out[c] is None:
                    out[c] = rec[c]
        elif kind == KIND_VLC_FIELD:
            out[fid] = vlc_vel_decode(p, n, a["segment_size"], a["bounds"][fid])
        else:
            out[fid] = sz_decode(p, n, a["bounds"][fid], a["interval_count"],
                                 1 if kind == KIND_SZ_FIELD else 2)
    return out


def compress_shards(fields, mode: str, eb_rel: float, nshards: int, nthreads: int,
                    interval_count: int = 65536, segment_size: int = 16384,
                    ignored_groups: int = 6, fmt: int = 1, decompress_too: bool = False) -> int:
    """CPU baseline: global bounds, then one segment-aligned shard per thread.
    SZ modes run in one C call (OpenMP over shards); the CPC modes run the
    CPC restatement per shard on a thread pool (the C stages release the
    GIL).  Returns the total payload / wire bytes."""
    f32 = [_c(a, np.float32) for a in fields]
    n = int(f32[0].size)
    resolved, _c2, mask = resolve_field_bounds(f32, ["rel"] * 6, [eb_rel] * 6)
    bounds = np.array([b if b is not None else 0.0 for b in resolved], np.float64)
    if mode in ("sz-cpc2000", "cpc2000"):
        import concurrent.futures as cf
        per = -(-n // max(nshards, 1))
        per = -(-per // segment_size) * segment_size
        kinds = ["abs" if b is not None else "rel" for b in resolved]
        vals = [b if b is not None else eb_rel for b in resolved]

        def one(s):
            lo, hi = s * per, min(n, (s + 1) * per)
            if hi <= lo:
                return 0
            r = compress_cpc([a[lo:hi] for a in f32], mode, kinds, vals,
                             interval_count=interval_count, segment_size=segment_size, fmt=fmt)
            if decompress_too:
                decompress_cpc(r["wire"])
            return len(r["wire"])

        with cf.ThreadPoolExecutor(max_workers=max(1, nthreads)) as ex:
            return int(sum(ex.map(one, range(max(nshards, 1)))))
    ptrs = (ctypes.c_void_p * 6)(*[a.ctypes.data for a in f32])
    bad = np.zeros(1, np.int64)
    tot = lib().orc_compress_shards(ptrs, n, int(mode == "sz-lv-prx"), _p(bounds), mask,
                                    interval_count, segment_size, ignored_groups, fmt, nshards,
                                    nthreads, int(decompress_too), _p(bad))
    if tot < 0 or bad[0]:
        raise RuntimeError(f"oracle shard compress failed: {tot} bad={int(bad[0])}")
    return int(tot)


def num_threads() -> int:
    return int(lib().orc_num_threads())
