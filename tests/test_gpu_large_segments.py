"""Sorted mode with segments longer than one 16384-particle tile
(Settings.segment_size > 16384; rindex.py:155-229 puts no cap on it).  The
B200 path switches to one device-wide stable radix sort of (segment, masked
key) composites (csrc/rlarge.cu); archives must still be byte-identical to
the oracle's, the permutation identical to the oracle's stable order, and the
decode exact and within bound."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1711_03888_b200 as nbz  # noqa: E402
from paper_1711_03888_b200 import datagen  # noqa: E402

REL4 = nbz.ErrorBoundSpec.relative(1e-4)


@pytest.fixture(scope="module")
def O(oracle_lib):
    return oracle_lib


def _check(O, fields, settings, eb=1e-4, variant="coord", version=2):
    snap = nbz.ParticleSnapshot(*fields)
    res = nbz.compress(snap, "sz-lv-prx", nbz.ErrorBoundSpec.relative(eb), settings,
                       version=version)
    ref = O.compress(fields, "sz-lv-prx", "rel", eb, interval_count=settings.interval_count,
                     segment_size=settings.segment_size, ignored_groups=settings.ignored_groups,
                     fmt=3 if version == 1 else 2, variant=variant)
    assert np.array_equal(res.order, ref["order"])
    assert res.archive.serialized() == ref["wire"]
    rec = nbz.decompress(res.archive)
    odec = O.decompress(ref["wire"])
    work = [f[res.order] for f in fields]
    for fi in range(6):
        got = np.asarray(rec.field(fi))
        assert np.array_equal(got, odec[fi]), fi
        if not res.archive.is_constant(fi):
            err = np.abs(work[fi].astype(np.float64) - got.astype(np.float64))
            assert float(err.max()) <= res.archive.bounds[fi], fi
    return res


@pytest.mark.parametrize("S,ig", [(16385, 6), (32768, 6), (65536, 0), (65536, 6), (100003, 3),
                                  (1 << 22, 6)])
def test_long_segments_byte_identical(O, S, ig):
    """Segment sizes above the tile: powers of two, ragged (16385, 100003:
    segments straddle the radix blocks and the 16384-symbol chunks) and one
    segment holding the whole snapshot."""
    fields = datagen.small_hacc(64)  # 262144 particles
    _check(O, fields, nbz.Settings(segment_size=S, ignored_groups=ig))


def test_long_segments_amdf_ragged_n(O):
    fields = datagen.small_amdf(300001)
    _check(O, fields, nbz.Settings(segment_size=50000))


@pytest.mark.parametrize("eb", [1e-2, 1e-6])
def test_long_segments_bounds(O, eb):
    """Few key bits (1e-2: many ties, stability decides the order) and many
    (1e-6: masked keys wider than 32 bits plus the segment bits)."""
    fields = datagen.small_hacc(48)
    _check(O, fields, nbz.Settings(segment_size=40000, ignored_groups=0), eb=eb)


def test_long_segments_velocity_keys(O):
    fields = datagen.small_hacc(40)
    _check(O, fields, nbz.Settings(segment_size=30000, rindex_variant=nbz.RIndexVariant.VELOCITY),
           variant="vel")


def test_long_segments_reference_readable(O):
    """version=1: the reference-readable container from the same sort."""
    fields = datagen.small_hacc(40)
    _check(O, fields, nbz.Settings(segment_size=32768), version=1)


def test_long_segments_auto_mode(O):
    """mode="auto" runs the sizing phase and resumes the encoding; the
    resumed call must read the sorted copies again."""
    fields = datagen.small_hacc(48)
    snap = nbz.ParticleSnapshot(*fields)
    st = nbz.Settings(segment_size=65536)
    a = nbz.compress(snap, "sz-lv", REL4, st).archive.serialized()
    b = nbz.compress(snap, "sz-lv-prx", REL4, st).archive.serialized()
    res = nbz.compress(snap, "auto", REL4, st)
    assert res.archive.serialized() == (b if len(b) < len(a) else a)


def test_long_segments_bound_too_small():
    x = np.array([1e30, -1e30, 5.0, 7.0], np.float32)
    snap = nbz.ParticleSnapshot(x, x, x, x, x, x)
    with pytest.raises(nbz.BoundTooSmallError):
        nbz.compress(snap, "sz-lv-prx", nbz.ErrorBoundSpec.absolute(1e-30),
                     nbz.Settings(segment_size=65536))


def test_long_segments_cpc_rejected():
    fields = datagen.small_hacc(16)
    snap = nbz.ParticleSnapshot(*fields)
    with pytest.raises(nbz.ValidationError):
        nbz.compress(snap, "cpc2000", REL4, nbz.Settings(segment_size=65536))
