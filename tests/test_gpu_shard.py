"""The sharded compress on real archives: two ranks on one
B200, gloo collectives over CPU tensors (one GPU per rank is the production
layout; the data path has no collective, so two ranks sharing a device run
the same code).  Each rank's archive must equal the oracle's v2 archive of
its shard compressed with the GLOBAL bounds, and the shards' decoded values,
concatenated, must equal the single-GPU decode bit for bit (the R-index sort
is segment-local and the v2 chain restarts every 16384 symbols, so sharding
on segment boundaries changes nothing but the Huffman tables)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

SPEC = dict(lattice=(48, 64, 64), spacing=2.5)  # 196608 particles = 12 segments


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, mode):
    import paper_1711_03888_b200 as nbz
    from paper_1711_03888_b200 import datagen, shard
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        torch.cuda.set_device(0)
        spec = datagen.HaccSpec(**SPEC)
        p0, p1 = shard.shard_range(spec.n, rank, world)
        fields = datagen.generate(spec, p0, p1)
        snap = nbz.ParticleSnapshot(*[torch.from_numpy(f).cuda() for f in fields])
        sr = shard.compress_shard(snap, mode, nbz.ErrorBoundSpec.relative(1e-4))
        wire = sr.result.archive.serialized()
        out = nbz.decompress(sr.result.archive, device=False)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), p=np.array([p0, p1]),
                 wire=np.frombuffer(wire, np.uint8),
                 bounds=np.array(sr.result.archive.bounds),
                 resolved=np.array([b.value for b in sr.bounds]),
                 offset=np.array([sr.offset, sr.total_bytes]),
                 **{f"o{i}": np.asarray(out.field(i)) for i in range(6)})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["sz-lv", "sz-lv-prx"])
def test_world2_shards_match_oracle_and_single_gpu(tmp_path, oracle_lib, mode):
    import paper_1711_03888_b200 as nbz
    from paper_1711_03888_b200 import datagen
    O = oracle_lib
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), mode), nprocs=world, join=True)
    rs = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    spec = datagen.HaccSpec(**SPEC)
    full = datagen.generate(spec)
    single = nbz.compress(nbz.ParticleSnapshot(*full), mode, nbz.ErrorBoundSpec.relative(1e-4))
    sdec = nbz.decompress(single.archive, device=False)
    sizes = [int(r["wire"].size) for r in rs]
    for r, rr in enumerate(rs):
        p0, p1 = (int(v) for v in rr["p"])
        # the globally resolved bounds: exactly the single-GPU archive's
        assert tuple(rr["bounds"]) == single.archive.bounds
        # the oracle's v2 archive of this shard under the same (absolute) bounds
        shard_fields = [f[p0:p1] for f in full]
        ref = O.compress(shard_fields, mode, "abs", list(rr["bounds"]), fmt=2)
        assert rr["wire"].tobytes() == ref["wire"], (mode, r)
        # decoded shard values == the single-GPU decode of the same particles
        for fi in range(6):
            assert np.array_equal(rr[f"o{fi}"].view(np.uint32),
                                  np.asarray(sdec.field(fi))[p0:p1].view(np.uint32)), (r, fi)
        # collective 2: byte offsets of the concatenated archives
        assert int(rr["offset"][0]) == sum(sizes[:r])
        assert int(rr["offset"][1]) == sum(sizes)
