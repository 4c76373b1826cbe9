"""Multi-GPU sharding of the compress path.

One process per GPU.  Rank r owns the contiguous, segment-aligned particle
range ``shard_range(n_total, r, world)``; the only exchanges are

1. an all-gather of the per-shard exact f32 (min, max) of the six fields
   (48 B per rank) so every rank resolves the SAME bounds as a single-GPU
   run would (``model.py:104-125``: b = eb_rel * (hi - lo) in f64); a
   relative bound resolved on a shard's own range would be ~P x tighter on
   lattice-ordered data and break ratio/key parity;
2. an all-gather of the per-shard archive sizes (one u64 per rank) after
   compress, giving each rank its byte offset in the concatenated output.

Everything between (R-index sort, quantise, Huffman) is shard-local: the
sort is segment-local (``rindex.py:181-197``) and the v2 chain restarts at
every 16384-symbol chunk, so each shard's archive decodes on its own.

The collectives use whatever ``torch.distributed`` process group is active
(NCCL on the GPU box; gloo in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .errors import ValidationError
from .model import FIELD_NAMES, BoundKind, ErrorBoundSpec

SEGMENT = 16384


def shard_range(n_total: int, rank: int, world: int, align: int = SEGMENT) -> Tuple[int, int]:
    """[p0, p1) of rank `rank`: contiguous, boundaries on multiples of
    `align` (whole R-index segments / v2 chunks), sizes differing by at most
    one `align` block; the last rank takes the ragged tail."""
    if world < 1 or not 0 <= rank < world:
        raise ValidationError(f"bad rank {rank} / world {world}")
    if n_total < 0:
        raise ValidationError("n_total must be >= 0")
    blocks = (n_total + align - 1) // align
    b0 = blocks * rank // world
    b1 = blocks * (rank + 1) // world
    return min(n_total, b0 * align), min(n_total, b1 * align)


def merge_minmax(per_rank: np.ndarray) -> np.ndarray:
    """(world, 6, 2) per-shard (min, max) -> global (6, 2).  Empty shards
    carry (+inf, -inf) and drop out."""
    a = np.asarray(per_rank, np.float64).reshape(-1, 6, 2)
    return np.stack([a[:, :, 0].min(axis=0), a[:, :, 1].max(axis=0)], axis=1)


def global_bounds(mm: np.ndarray, specs: Sequence[ErrorBoundSpec]) -> List[ErrorBoundSpec]:
    """Resolve each field's bound on the GLOBAL range exactly as
    ``model.resolve_bound`` does (f64 product of the relative bound and the
    f32 range), returned as absolute specs for the shard-local compress.
    A globally constant field keeps its relative spec: every shard then
    sees a zero range and takes the reference's constant-field path."""
    out = []
    for i, spec in enumerate(specs):
        lo, hi = float(mm[i, 0]), float(mm[i, 1])
        if spec.kind is BoundKind.ABSOLUTE or not (hi > lo):
            out.append(spec)
        else:
            out.append(ErrorBoundSpec.absolute(float(spec.value) * (hi - lo)))
    return out


def _collective_device(group=None, device=None):
    """Where the collectives' tensors live: the caller's choice, else the
    current CUDA device under NCCL (which rejects CPU tensors), else CPU."""
    import torch
    import torch.distributed as dist
    if device is not None:
        return device
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return None


def _all_gather_f64(vals: np.ndarray, group=None, device=None) -> np.ndarray:
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(np.asarray(vals, np.float64).ravel(), dtype=torch.float64)
    device = _collective_device(group, device)
    if device is not None:
        t = t.to(device)
    world = dist.get_world_size(group)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    return torch.stack(outs).cpu().numpy()


def allgather_minmax(mm_local: np.ndarray, group=None, device=None) -> np.ndarray:
    """Collective 1: (6, 2) local (min, max) -> (world, 6, 2)."""
    g = _all_gather_f64(mm_local, group, device)
    return g.reshape(-1, 6, 2)


def exclusive_offsets(sizes: Sequence[int]) -> np.ndarray:
    s = np.asarray(sizes, np.int64)
    return np.concatenate([[0], np.cumsum(s)[:-1]]) if s.size else s


def local_minmax(fields) -> np.ndarray:
    """Exact f32 (min, max) per field of this shard, (6, 2) f64; an empty
    shard gives (+inf, -inf).  CUDA fields: one fused pass (nbzg_minmax6,
    the K1 kernel; fields re-allocated 16-byte aligned if a view is not);
    host arrays: numpy."""
    import torch
    out = np.empty((6, 2), np.float64)
    fields = list(fields)
    n = int(fields[0].shape[0])
    if n == 0:
        out[:, 0], out[:, 1] = np.inf, -np.inf
        return out
    if all(isinstance(f, torch.Tensor) and f.is_cuda for f in fields):
        import ctypes

        from . import _native as N
        ts = [f.contiguous() for f in fields]
        ts = [t if t.data_ptr() % 16 == 0 else t.clone() for t in ts]
        arr = (ctypes.c_void_p * 6)(*[t.data_ptr() for t in ts])
        mm = torch.empty(12, dtype=torch.float32, device=ts[0].device)
        N.check(N.lib().nbzg_minmax6(arr, n, N.ptr(mm), N.stream_handle()), "minmax6")
        return mm.cpu().numpy().astype(np.float64).reshape(6, 2)
    for i, f in enumerate(fields):
        a = f.cpu().numpy() if isinstance(f, torch.Tensor) else np.asarray(f, np.float32)
        out[i] = (float(a.min()), float(a.max()))
    return out


@dataclass
class ShardResult:
    result: object          # CompressResult of this rank's shard
    rank: int
    world: int
    bounds: List[ErrorBoundSpec]
    offset: int             # byte offset of this shard's archive in the concatenation
    total_bytes: int        # sum of all shards' archive sizes


def compress_shard(snapshot, mode, bounds, settings=None, group=None,
                   device=None) -> ShardResult:
    """Compress this rank's shard with bounds resolved on the GLOBAL range
    (collective 1), then all-gather the archive sizes (collective 2).

    The compress runs in two C-ABI phases on one workspace: K1 gives the
    shard's exact min/max, the ranks all-gather them, and the rest of the
    compress resumes with the global min/max -- K1 runs once per rank."""
    import torch.distributed as dist

    from .pipeline import DEFAULT_SETTINGS, _CompressCall, _specs

    specs = _specs(bounds)
    settings = settings or DEFAULT_SETTINGS
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    call = _CompressCall(snapshot, mode, bounds, settings)
    if world == 1:  # the shard is the snapshot: resolve locally, as compress does
        res = call.finish()
        size = res.archive.total_bytes()
        resolved = [ErrorBoundSpec.absolute(b) if b > 0 else s
                    for b, s in zip(res.archive.bounds, specs)]
        return ShardResult(res, 0, 1, resolved, 0, int(size))
    mm = merge_minmax(allgather_minmax(call.local_minmax(), group, device))
    resolved = global_bounds(mm, specs)
    res = call.finish(mm)
    size = res.archive.total_bytes()
    sizes = _all_gather_f64(np.array([float(size)]), group, device).ravel().astype(np.int64)
    offs = exclusive_offsets(sizes)
    return ShardResult(res, rank, world, resolved, int(offs[rank]), int(sizes.sum()))
