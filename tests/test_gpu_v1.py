"""Reference-readable archives (``compress(..., version=1)``): container
version 1 of SZ_FIELD streams whose chain is the reference's, restarted by a
forced escape every 16384 values.  The GPU archive is
byte-identical to the oracle's restatement of that chain (oracle fmt 3,
pinned to the reference on CPU in test_oracle_golden.py), decodes within the
bound, its ratio is within 0.5% of the reference's own archive, and the
unmodified reference package (baseline/_ref, when installed) deserialises and
decodes it to the same values."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1711_03888_b200 as nbz  # noqa: E402
from paper_1711_03888_b200 import datagen  # noqa: E402
from paper_1711_03888_b200 import io as nio  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _reference_nbz():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "nbz")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbz_numba_cache")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import nbz as ref_nbz
        from nbz import io as ref_io
        return ref_nbz, ref_io
    except Exception:  # pragma: no cover
        return None


CASES = [("hacc34", lambda: datagen.small_hacc(34)),
         ("amdf40k", lambda: datagen.small_amdf(40000)),
         ("C0", lambda: datagen.generate("C0"))]


@pytest.mark.parametrize("name,gen", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("mode", ["sz-lv", "sz-lv-prx"])
def test_v1_archive_matches_oracle_and_reference(oracle_lib, name, gen, mode):
    O = oracle_lib
    fields = gen()
    snap = nbz.ParticleSnapshot(*fields)
    res = nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(1e-4), version=1)
    wire = res.archive.serialized()
    ref = O.compress(fields, mode, "rel", 1e-4, fmt=3)
    assert wire == ref["wire"], (name, mode)
    # ratio within 0.5% of the reference's own (unrestarted) archive
    v1 = O.compress(fields, mode, "rel", 1e-4, fmt=1)
    assert abs(nbz.ratio(res.archive) / v1["ratio"] - 1) < 0.005
    # the GPU decodes it (compat chain) to the oracle's values, within the bound
    out = nbz.decompress(nio.deserialize_archive(wire))
    odec = O.decompress(wire)
    order = res.order
    for fi in range(6):
        got = np.asarray(out.field(fi))
        assert np.array_equal(got.view(np.uint32), odec[fi].view(np.uint32)), fi
        x = fields[fi] if order is None else fields[fi][order]
        assert np.abs(x.astype(np.float64) - got).max() <= res.archive.bounds[fi]
    # the unmodified reference reads it
    r = _reference_nbz()
    if r is not None:
        ref_nbz, ref_io = r
        rout = list(ref_nbz.decompress(ref_io.deserialize_archive(wire)).fields())
        for fi in range(6):
            assert np.array_equal(rout[fi].view(np.uint32), odec[fi].view(np.uint32)), fi


def test_v1_rejects_other_modes():
    snap = nbz.ParticleSnapshot(*datagen.small_hacc(8))
    for mode in ("sz-lcf", "sz-cpc2000", "cpc2000"):
        with pytest.raises(nbz.ValidationError):
            nbz.compress(snap, mode, nbz.ErrorBoundSpec.relative(1e-4), version=1)
