"""Multi-GPU host logic on CPU: shard ranges, and the two collectives of
the sharded compress (global bounds, archive offsets) over a gloo
world-size-2 process group.  No GPU needed."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1711_03888_b200 import datagen, shard  # noqa: E402
from paper_1711_03888_b200.model import ErrorBoundSpec, resolve_bound  # noqa: E402


@pytest.mark.parametrize("n", [0, 1, 16383, 16384, 16385, 1_000_000, 262_144_000])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_range_partition(n, world):
    prev = 0
    for r in range(world):
        p0, p1 = shard.shard_range(n, r, world)
        assert p0 == prev and p0 <= p1 <= n
        if p1 < n:
            assert p1 % shard.SEGMENT == 0
        prev = p1
    assert prev == n
    sizes = [shard.shard_range(n, r, world)[1] - shard.shard_range(n, r, world)[0]
             for r in range(world)]
    assert max(sizes) - min(sizes) <= shard.SEGMENT


def test_shard_range_rejects_bad_rank():
    with pytest.raises(Exception):
        shard.shard_range(10, 2, 2)


def test_global_bounds_match_single_process():
    f = datagen.small_hacc(20)
    specs = [ErrorBoundSpec.relative(1e-4)] * 3 + [ErrorBoundSpec.absolute(0.5)] * 3
    per = [shard.local_minmax([x[:4000] for x in f]), shard.local_minmax([x[4000:] for x in f])]
    g = shard.merge_minmax(np.stack(per))
    gb = shard.global_bounds(g, specs)
    for i in range(6):
        assert gb[i].value == resolve_bound(specs[i], f[i])


def test_exclusive_offsets():
    assert shard.exclusive_offsets([5, 7, 0, 3]).tolist() == [0, 5, 12, 12]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                           world_size=world)
    try:
        spec = datagen.HaccSpec((40, 40, 40), 2.56)
        p0, p1 = shard.shard_range(spec.n, rank, world)
        fields = datagen.generate(spec, p0, p1)
        mm = shard.local_minmax(fields)
        g = shard.merge_minmax(shard.allgather_minmax(mm))
        specs = [ErrorBoundSpec.relative(1e-4)] * 6
        gb = shard.global_bounds(g, specs)
        sizes = shard._all_gather_f64(np.array([1000.0 + rank])).ravel().astype(np.int64)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), p=np.array([p0, p1]),
                 b=np.array([s.value for s in gb]), sizes=sizes)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_global_bounds(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    spec = datagen.HaccSpec((40, 40, 40), 2.56)
    full = datagen.generate(spec)
    ref = [resolve_bound(ErrorBoundSpec.relative(1e-4), f) for f in full]
    rs = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    # shards tile [0, n) on segment boundaries
    assert rs[0]["p"][0] == 0 and rs[0]["p"][1] == rs[1]["p"][0] and rs[1]["p"][1] == spec.n
    for r in rs:
        # every rank resolves exactly the single-GPU bounds
        assert r["b"].tolist() == ref
        assert r["sizes"].tolist() == [1000, 1001]
        assert shard.exclusive_offsets(r["sizes"]).tolist() == [0, 1000]
