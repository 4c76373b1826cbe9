"""ctypes binding of the in-tree C-ABI library ``libnbzg.so`` (include/nbzg.h).

There is deliberately no fallback: if the library is missing or no CUDA
device is present, every entry point raises ``NativeUnavailable`` -- the
B200 path never silently degrades to a CPU implementation.

PyTorch is used only as plumbing: the caching allocator for device
buffers and the current CUDA stream handle.
"""

from __future__ import annotations

import ctypes
import os
import threading
from typing import Dict, Tuple

_HERE = os.path.dirname(os.path.abspath(__file__))
# NBZG_LIB selects another in-tree build of the same library (kernel
# experiments: scripts/dec_variants.py); it is never a different implementation
LIB_PATH = os.environ.get("NBZG_LIB") or os.path.join(_HERE, "libnbzg.so")

NBZG_OK = 0
NBZG_BOUND_TOO_SMALL = 1
NBZG_CODE_TOO_LONG = 2
NBZG_INVALID_CODE = 3
NBZG_TRUNCATED = 4
NBZG_BAD_ARG = 5
NBZG_CUDA_ERROR = 6
NBZG_UNSUPPORTED = 7
NBZG_BAD_STREAM = 8

STATUS_NAMES = {0: "ok", 1: "bound too small", 2: "code too long", 3: "invalid huffman code",
                4: "truncated stream", 5: "bad argument", 6: "cuda error",
                7: "unsupported parameter", 8: "malformed stream"}

EXPORTED = (
    "nbzg_compress", "nbzg_compress_workspace_size", "nbzg_compress_arena_bound",
    "nbzg_decompress", "nbzg_decompress_workspace_size", "nbzg_minmax6", "nbzg_integerize",
    "nbzg_rindex_keys", "nbzg_prx_order", "nbzg_order_expand", "nbzg_huffman_lengths",
    "nbzg_huffman_codebook", "nbzg_huff_encode", "nbzg_crc64", "nbzg_crc64_workspace_size",
    "nbzg_version", "nbzg_device_sm_count", "nbzg_launch_count", "nbzg_trace_enable",
    "nbzg_trace_read", "nbzg_cpc_workspace_size", "nbzg_cpc_plan", "nbzg_cpc_pack",
    "nbzg_cpc_decode", "nbzg_cpc_decode_workspace_size", "nbzg_huff_decode",
    "nbzg_deinterleave3", "nbzg_crc64_many", "nbzg_crc64_many_workspace_size",
    "nbzg_compress_workspace_size_fmt",
)


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing (no CPU fallback exists)."""


c_p = ctypes.c_void_p
c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_u32 = ctypes.c_uint32
c_u64 = ctypes.c_uint64
c_sz = ctypes.c_size_t
c_d = ctypes.c_double
c_f = ctypes.c_float


class FieldMeta(ctypes.Structure):
    _fields_ = [("bound", c_d), ("twob", c_d), ("inv", c_d), ("inv32", c_f), ("constant", c_f),
                ("lo", c_f), ("hi", c_f), ("is_const", c_u32), ("k", c_u32),
                ("min_len", c_u32), ("max_len", c_u32), ("n_esc", c_u64),
                ("total_bits", c_u64), ("payload_off", c_u64), ("payload_len", c_u64),
                ("index_off", c_u64), ("bits_off", c_u64), ("esc_off", c_u64)]


class Meta(ctypes.Structure):
    _fields_ = [("f", FieldMeta * 6), ("mask", c_u32), ("status", c_u32),
                ("arena_used", c_u64), ("nseg", c_u64), ("pad", c_u64)]


class CompressArgs(ctypes.Structure):
    _fields_ = [("fields", c_p * 6), ("n", c_i64), ("sorted", c_i32), ("bound_kind", c_i32 * 6),
                ("bound_value", c_d * 6), ("interval_count", c_i64), ("segment_size", c_i64),
                ("ignored_groups", c_i32), ("rindex_variant", c_i32), ("workspace", c_p),
                ("workspace_bytes", c_sz), ("arena", c_p), ("arena_bytes", c_sz),
                ("meta", c_p), ("seg_bits", c_p), ("perm", c_p), ("predictor", c_i32),
                ("cpc", c_i32), ("seg_minima", c_p), ("sz_skip", c_u32), ("phase", c_i32),
                ("h_minmax", c_f * 12), ("fmt", c_i32), ("pad3", c_i32),
                ("order32", c_p)]


class CpcMeta(ctypes.Structure):
    _fields_ = [("off", c_u64 * 4), ("len", c_u64 * 4), ("total_bits", c_u64 * 4),
                ("corr", (c_u64 * 3) * 4), ("status", c_u32), ("pad", c_u32)]


class CpcArgs(ctypes.Structure):
    _fields_ = [("fields", c_p * 6), ("n", c_i64), ("segment_size", c_i64), ("mode", c_i32),
                ("pad0", c_i32), ("perm", c_p), ("seg_bits", c_p), ("seg_minima", c_p),
                ("meta", c_p), ("workspace", c_p), ("workspace_bytes", c_sz), ("arena", c_p),
                ("cmeta", c_p)]


class CpcDecodeArgs(ctypes.Structure):
    _fields_ = [("payload", c_p), ("payload_len", c_i64), ("kind", c_i32), ("indexed", c_i32),
                ("n", c_i64), ("segment_size", c_i64), ("total_bits", c_u64),
                ("seg_bits", c_p), ("seg_minima", c_p), ("bound", c_d * 3), ("out", c_p * 3),
                ("workspace", c_p), ("workspace_bytes", c_sz), ("status", c_p)]


class DecompressArgs(ctypes.Structure):
    _fields_ = [("payload", c_p * 6), ("payload_len", c_i64 * 6), ("kind", c_i32 * 6),
                ("bound", c_d * 6), ("out", c_p * 6), ("nfields", c_i32), ("pad0", c_i32),
                ("n", c_i64), ("interval_count", c_i64), ("workspace", c_p),
                ("workspace_bytes", c_sz), ("status", c_p)]


_SIGS = {
    "nbzg_compress": (ctypes.c_int, [c_p, c_p]),
    "nbzg_compress_workspace_size": (c_sz, [c_i64, c_i32, c_i64, c_i64]),
    "nbzg_compress_workspace_size_fmt": (c_sz, [c_i64, c_i32, c_i64, c_i64, c_i32]),
    "nbzg_compress_arena_bound": (c_sz, [c_i64, c_i64]),
    "nbzg_decompress": (ctypes.c_int, [c_p, c_p]),
    "nbzg_decompress_workspace_size": (c_sz, [c_i64, c_i64, c_i32]),
    "nbzg_minmax6": (ctypes.c_int, [c_p, c_i64, c_p, c_p]),
    "nbzg_integerize": (ctypes.c_int, [c_p, c_i64, c_d, c_p, c_p, c_p]),
    "nbzg_rindex_keys": (ctypes.c_int, [c_p, c_p, c_p, c_i64, c_p, c_i64, c_p, c_p, c_p, c_p]),
    "nbzg_prx_order": (ctypes.c_int, [c_p, c_i64, c_i64, c_p, c_i32, c_p, c_p]),
    "nbzg_order_expand": (ctypes.c_int, [c_p, c_i64, c_i64, c_p, c_p]),
    "nbzg_huffman_lengths": (ctypes.c_int, [c_p, c_i64, c_p, c_p, c_sz, c_p, c_p]),
    "nbzg_huffman_codebook": (ctypes.c_int, [c_p, c_i64, c_p, c_p, c_p, c_p, c_p, c_sz, c_p]),
    "nbzg_huff_encode": (ctypes.c_int, [c_p, c_i64, c_p, c_p, c_p, c_p, c_sz, c_p]),
    "nbzg_crc64": (ctypes.c_int, [c_p, c_i64, c_p, c_p, c_sz, c_p]),
    "nbzg_crc64_workspace_size": (c_sz, [c_i64]),
    "nbzg_version": (ctypes.c_char_p, []),
    "nbzg_device_sm_count": (ctypes.c_int, []),
    "nbzg_launch_count": (ctypes.c_ulonglong, []),
    "nbzg_trace_enable": (ctypes.c_int, [ctypes.c_int]),
    "nbzg_trace_read": (ctypes.c_int, [c_p, ctypes.c_int, c_p, ctypes.c_int]),
    "nbzg_cpc_workspace_size": (c_sz, [c_i64, c_i64]),
    "nbzg_cpc_plan": (ctypes.c_int, [c_p, c_p]),
    "nbzg_cpc_pack": (ctypes.c_int, [c_p, c_p]),
    "nbzg_cpc_decode_workspace_size": (c_sz, [c_i64, c_i64]),
    "nbzg_cpc_decode": (ctypes.c_int, [c_p, c_p]),
    "nbzg_huff_decode": (ctypes.c_int, [c_p, c_u64, c_i64, c_i32, c_i32, c_p, c_p, c_p, c_p, c_p,
                                        c_p, c_p]),
    "nbzg_deinterleave3": (ctypes.c_int, [c_p, c_i64, c_p, c_p, c_p, c_p]),
    "nbzg_crc64_many": (ctypes.c_int, [c_p, c_p, c_i32, c_p, c_p, c_sz, c_p]),
    "nbzg_crc64_many_workspace_size": (c_sz, [c_p, c_i32]),
}

_lib = None
_lock = threading.Lock()


def load_library(require_cuda: bool = False):
    """dlopen libnbzg.so and declare every prototype.  Works without a GPU
    (symbols only); ``require_cuda`` additionally checks for a device."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (make -C paper_1711_03888_b200/csrc)")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    if require_cuda:
        import torch
        if not torch.cuda.is_available():
            raise NativeUnavailable("the nbz B200 path needs a CUDA device; none is visible")
    return _lib


def lib():
    return load_library(require_cuda=True)


def check(rc: int, what: str):
    if rc != NBZG_OK:
        from .errors import ValidationError
        if rc in (NBZG_BAD_ARG, NBZG_UNSUPPORTED):
            raise ValidationError(f"{what}: {STATUS_NAMES.get(rc, rc)}")
        raise RuntimeError(f"{what}: {STATUS_NAMES.get(rc, rc)} (status {rc})")


def stream_handle():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> int:
    return int(t.data_ptr())


def launch_count() -> int:
    return int(load_library().nbzg_launch_count())


def trace_enable(on: bool = True) -> None:
    load_library().nbzg_trace_enable(1 if on else 0)


def trace_read(max_entries: int = 65536):
    """[(stage name, ms)] recorded since trace_enable (synchronises)."""
    stride = 32
    names = ctypes.create_string_buffer(stride * max_entries)
    ms = (ctypes.c_float * max_entries)()
    cnt = load_library().nbzg_trace_read(names, stride, ms, max_entries)
    raw = names.raw
    return [(raw[i * stride:(i + 1) * stride].split(b"\0", 1)[0].decode(), float(ms[i]))
            for i in range(cnt)]


def workspace(nbytes: int):
    """Per-call device scratch (uint8) from torch's caching allocator on the
    current stream: repeated calls reuse the cached block, and concurrent
    calls (host threads, each on its own stream) never share one -- the
    C-ABI keeps all per-call state in this buffer."""
    import torch
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device="cuda")


_SIDE: Dict[Tuple[int, int], list] = {}
_side_lock = threading.Lock()


def side_streams(k: int):
    """k persistent side CUDA streams of the current device and host thread
    (overlapping independent per-stream decodes; a host thread never shares
    its side streams with another)."""
    import torch
    key = (torch.cuda.current_device(), threading.get_ident())
    with _side_lock:
        lst = _SIDE.setdefault(key, [])
        while len(lst) < k:
            lst.append(torch.cuda.Stream())
        return lst[:k]
