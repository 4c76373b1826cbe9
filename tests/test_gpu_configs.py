"""BASELINE configurations at their stated sizes, checked against the oracle
(SURVEY.md §8d acceptance; reference tests test_acceptance.py:55-90, 328-368).

* config 2 -- the 640^3 HACC-like snapshot ``bench.py`` times
  (``datagen.generate('C2')``): the GPU archive is byte-identical to the
  oracle's v2 archive, its ratio is within 0.5% of the reference algorithm's
  (oracle v1 = the reference's exact chain), and every reconstructed value
  is within its bound;
* config 3 -- 2^26 HACC-like (512 x 512 x 256) and 2^26 AMDF-like snapshots
  at eb_rel 1e-2 .. 1e-6, sz-lv and sz-lv-prx: the same three checks;
* the reference's acceptance c10: byte determinism across repeated and
  threaded calls, and 1000 of 1000 single-byte corruptions rejected.

The oracle runs are independent C calls (ctypes releases the GIL), so they
run on a thread pool beside the GPU work.
"""

import concurrent.futures as cf
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1711_03888_b200 as nbz  # noqa: E402
from paper_1711_03888_b200 import datagen  # noqa: E402
from paper_1711_03888_b200 import io as nio  # noqa: E402

MODES = ("sz-lv", "sz-lv-prx")
EBS = (1e-2, 1e-3, 1e-4, 1e-5, 1e-6)


@pytest.fixture(scope="module")
def pool():
    with cf.ThreadPoolExecutor(max_workers=max(2, min(12, os.cpu_count() or 2))) as ex:
        yield ex


def _oracle_jobs(pool, O, fields, mode, eb):
    """(v2 wire, v1 ratio) futures of the oracle on the same arrays."""
    v2 = pool.submit(lambda: O.compress(fields, mode, "rel", eb, fmt=2)["wire"])
    v1 = pool.submit(lambda: O.compress(fields, mode, "rel", eb, fmt=1)["ratio"])
    return v2, v1


def _check_bound(dsnap, res):
    """|x[order] - recon| <= b at every point (device-side, exact in f64)."""
    rec = nbz.decompress(res.archive, device=True)
    order = res.order_device()
    for fi in range(6):
        x = dsnap.field(fi)
        if order is not None:
            x = x[order]
        b = res.archive.bounds[fi]
        if res.archive.is_constant(fi):
            assert torch.equal(x, rec.field(fi)), fi
            continue
        err = (x.double() - rec.field(fi).double()).abs().max().item()
        assert err <= b, (fi, err, b)


def _compare(res, wire_f, v1_f, tag):
    wire = res.archive.serialized()
    ref_wire = wire_f.result()
    assert len(wire) == len(ref_wire), (tag, len(wire), len(ref_wire))
    assert wire == ref_wire, tag
    r1 = v1_f.result()
    r2 = nbz.ratio(res.archive)
    assert abs(r2 / r1 - 1.0) < 0.005, (tag, r2, r1)
    return r2, r1


def test_c2_benched_snapshot_matches_oracle(oracle_lib, pool):
    """The exact snapshot bench.py times (BASELINE config 2)."""
    O = oracle_lib
    fields = datagen.generate("C2")
    jobs = {mode: _oracle_jobs(pool, O, fields, mode, 1e-4) for mode in MODES}
    dsnap = nbz.ParticleSnapshot(*[torch.from_numpy(f).cuda() for f in fields])
    for mode in MODES:
        res = nbz.compress(dsnap, mode, nbz.ErrorBoundSpec.relative(1e-4))
        _check_bound(dsnap, res)
        r2, r1 = _compare(res, *jobs[mode], ("C2", mode))
        print(f"C2 {mode}: ratio {r2:.6f} (reference chain {r1:.6f}, {100 * (r2 / r1 - 1):+.4f}%)")
        del res
    del dsnap, fields, jobs
    torch.cuda.empty_cache()


@pytest.fixture(scope="module")
def c3_fields():
    return {p: datagen.generate(f"C3-{p}") for p in ("hacc", "amdf")}


@pytest.mark.parametrize("profile", ["hacc", "amdf"])
def test_c3_error_bound_sweep(oracle_lib, pool, c3_fields, profile):
    """BASELINE config 3: 2^26 particles, eb_rel 1e-2 .. 1e-6 (alphabet from
    tens to ~65K symbols, escapes up to ~66% at 1e-6), both modes."""
    O = oracle_lib
    fields = c3_fields[profile]
    assert fields[0].size == 1 << 26
    jobs = {(mode, eb): _oracle_jobs(pool, O, fields, mode, eb) for eb in EBS for mode in MODES}
    dsnap = nbz.ParticleSnapshot(*[torch.from_numpy(f).cuda() for f in fields])
    for eb in EBS:
        for mode in MODES:
            res = nbz.compress(dsnap, mode, nbz.ErrorBoundSpec.relative(eb))
            _check_bound(dsnap, res)
            r2, r1 = _compare(res, *jobs[(mode, eb)], (profile, mode, eb))
            print(f"C3-{profile} {mode} eb {eb:g}: ratio {r2:.4f} (reference chain {r1:.4f})")
            del res
    del dsnap
    torch.cuda.empty_cache()


def _random_snapshot(rng, n):
    """A mixed snapshot in the spirit of the reference's random_snapshot."""
    return nbz.ParticleSnapshot(*[rng.normal(0, 1 + 10 * i, n).astype(np.float32)
                                  for i in range(6)])


def test_c10_determinism_threaded():
    """Acceptance c10 (test_acceptance.py:328-343): sequential, repeated and
    4-thread pool calls give byte-identical archives in every mode -- also
    with each host thread on its own CUDA stream (the C-ABI keeps all
    per-call state in the caller's workspace)."""
    snaps = [_random_snapshot(np.random.default_rng(40 + i), 40000) for i in range(4)]
    spec = nbz.ErrorBoundSpec.relative(1e-4)

    def wire(s, mode, own_stream=False):
        if own_stream:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                w = nbz.compress(s, mode, spec).archive.serialized()
            st.synchronize()
            return w
        return nbz.compress(s, mode, spec).archive.serialized()

    for mode in ("sz-lcf", "sz-lv", "sz-lv-prx", "sz-cpc2000", "cpc2000"):
        sequential = [wire(s, mode) for s in snaps]
        again = [wire(s, mode) for s in snaps]
        with cf.ThreadPoolExecutor(max_workers=4) as ex:
            threaded = list(ex.map(lambda s: wire(s, mode), snaps))
            streamed = list(ex.map(lambda s: wire(s, mode, True), snaps))
        assert sequential == again == threaded == streamed, mode
        # and decoding concurrently gives the sequential values
        archives = [nio.deserialize_archive(w) for w in sequential]
        ref = [nbz.decompress(a) for a in archives]
        with cf.ThreadPoolExecutor(max_workers=4) as ex:
            par = list(ex.map(nbz.decompress, archives))
        for a, b in zip(ref, par):
            for fi in range(6):
                assert np.array_equal(np.asarray(a.field(fi)), np.asarray(b.field(fi))), mode


@pytest.mark.parametrize("mode", ["sz-lv-prx", "sz-cpc2000"])
def test_c10_single_byte_corruptions_all_rejected(mode):
    """1000 random single-byte corruptions of a serialized archive are all
    rejected with ArchiveError (test_acceptance.py:355-368): the CRC-64s
    cover the header and every payload byte."""
    rng = np.random.default_rng(1010)
    snap = _random_snapshot(np.random.default_rng(40), 4000)
    base = bytearray(nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(1e-4))
                     .archive.serialized())
    rejected = 0
    for _ in range(1000):
        pos = int(rng.integers(0, len(base)))
        delta = int(rng.integers(1, 256))
        bad = bytearray(base)
        bad[pos] ^= delta
        try:
            nio.deserialize_archive(bytes(bad))
        except nbz.ArchiveError:
            rejected += 1
    assert rejected == 1000, rejected
